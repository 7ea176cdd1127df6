#!/bin/bash
# tools/bp5_check.sh -- on the GPU box: BP5 (collocated GLL) parity tests and
# GDOF/s at ~10M and the C4 ~200M sizes, 2D and 3D p = 4.
python -m pytest tests -m gpu -q -k "bp5 or gll or collocated" 2>&1 | tail -3
run() {
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --steps 3 --iters 100 "$@" 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value'],2), 'op', round(d['roofline']['frac'],3), 'cg', round(d['cg_roofline']['frac'],3), 'op_us', round(d['roofline']['ms_per_launch']*1e3,1))" \
    || echo "$* FAILED"
}
run --dim 2 --order 4 --bp 5
run --dim 3 --order 4 --bp 5
run --dim 3 --order 2 --bp 5
run --dim 2 --order 4 --bp 5 --cells 3536
run --dim 3 --order 4 --bp 5 --cells 146
python - <<'PY'
import ctypes as C, paper_1911_09220_b200 as tf
d = tf.Device(0); v = C.c_double(); w = C.c_double()
tf.abi.check(tf.lib().tfem_fp64_peak(d.h, C.byref(v))); tf.abi.check(tf.lib().tfem_dmma_peak(d.h, C.byref(w)))
print("DFMA peak TFLOP/s", round(v.value, 2), "DMMA peak TFLOP/s", round(w.value, 2))
PY
