"""tools/contraction_ab.py -- on the GPU box: the DFMA vs DMMA A/B of the
sum-factorisation contraction stage (tfem_contraction_ab), p = 2..8, next to
the measured DFMA / DMMA peaks and, per order, the FP64 rate the 3D element
kernel needs to stay HBM-bound (flops per element / qdata bytes per element
x measured HBM bandwidth).  Writes a markdown table to stdout."""
import ctypes as C
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_1911_09220_b200 as tf  # noqa: E402

dev = tf.Device(0)
lib = tf.lib()
fp, mm = C.c_double(), C.c_double()
tf.abi.check(lib.tfem_fp64_peak(dev.h, C.byref(fp)))
tf.abi.check(lib.tfem_dmma_peak(dev.h, C.byref(mm)))
peaks = json.loads((pathlib.Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
    if (pathlib.Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {}
hbm = None
for k, v in peaks.items():
    if "hbm" in k.lower() and isinstance(v, (int, float)):
        hbm = float(v)
        break
print(f"measured peaks: DFMA {fp.value:.1f} TFLOP/s, DMMA (m8n8k4) {mm.value:.1f} TFLOP/s"
      + (f", HBM {hbm:.0f} GB/s" if hbm else ""))
print()
print("| p | q | DFMA stage TFLOP/s | DMMA stage TFLOP/s | DMMA / DFMA | DMMA padding | max rel diff |"
      " 3D BP3 flop/B | FP64 TFLOP/s to stay HBM-bound |")
print("|---|---|---|---|---|---|---|---|---|")
res = (C.c_double * 4)()
for p in range(2, 9):
    tf.abi.check(lib.tfem_contraction_ab(dev.h, p, res))
    q, d1 = p + 2, p + 1
    # 3D BP3 element: forward 2QD1^3 + 3*... (bench.py op_flops_per_element)
    fwd = 2 * q * d1 * d1 * d1 + 3 * q * q * d1 * d1 + 3 * q * q * q * d1
    flops = 2 * (2 * fwd) + 15 * q ** 3  # forward + transpose (FMA = 2 flops), 3x3 point factors
    qbytes = 6 * q ** 3 * 8
    need = (flops / qbytes * hbm / 1e3) if hbm else float("nan")
    print(f"| {p} | {q} | {res[0]:.1f} | {res[1]:.1f} | {res[1] / res[0]:.2f} | {res[3]:.2f} | "
          f"{res[2]:.1e} | {flops / qbytes:.2f} | {need:.1f} |")
dev.close()
