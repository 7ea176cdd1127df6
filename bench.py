#!/usr/bin/env python
"""BP3 benchmark: PA-diffusion + Jacobi-PCG throughput on B200.

metric  "BP3 PA-diffusion CG GDOF/s (p=3) at 1/2/4/8 B200; HBM GB/s vs roofline"
        (BASELINE.json).  GDOF/s = DOFs x CG iterations / time.
workload (N=1) configs[1]: BP3, p = 3, ~10M DOFs on one B200.  2D (the
        reference's dimension: make_cartesian(1054, 1054) -> 10,004,569 DOFs,
        q = p+2 Gauss-Legendre, kappa = 1, Dirichlet on the whole boundary),
        one step = one cg_solve of a fixed 200 iterations (
        rel_tol = 0 so max_iters is reached), rhs seeded U(-1, 1).
value   device-resident: b, diag, x in HBM when the timed region starts;
        CUDA events on the library's stream, max over ranks.
e2e     the same solve through the C ABI with HOST buffers
        (tfem_cg_solve_host: b and diag copied in, x copied out every step).
roofline  dominant kernel = the PA operator application (element kernel +
        shared-DOF scatter, one tfem_operator_mult): algorithmic bytes
        B_op = E (nc q^2 8 + D1^2 4) + 16 N / event-timed
        launch duration, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the reference itself (oracle/_ref, all host threads) on a
        bounded sample (a few CG iterations of the same problem).

--impl reference: times the reference's own CPU cg_solve on the host cores
(rank 0 only), same metric / config, a few iterations per step.
N > 1 (torchrun): the mesh is partitioned by element rows across ranks
(weak scaling: ~10M DOFs per rank); see paper_1911_09220_b200/dist.py.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "BP3 PA-diffusion CG GDOF/s (p=3) at 1/2/4/8 B200; HBM GB/s vs roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tfem", choices=["tfem", "reference"])
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--bp", type=int, default=3, choices=[1, 3, 5],
                    help="CEED problem: 1 mass (q=p+2 GL, plain CG), 3 diffusion (q=p+2 GL, "
                         "Jacobi), 5 diffusion (q=p+1 GLL, Jacobi)")
    ap.add_argument("--cells", type=int, default=0, help="cells per axis (0: ~10M DOFs)")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--numerics", default="fma", choices=["reference", "fma"])
    ap.add_argument("--cpu-iters", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-bitexact", action="store_true", help="skip the reference-numerics line")
    ap.add_argument("--strong", action="store_true",
                    help="N > 1: partition one n^dim mesh over the ranks (default: weak scaling, "
                         "~10M DOFs per rank)")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the extra configurations (3D BP3 p=3 ~10M, 2D BP3 p=3 ~100M DOFs)")
    return ap.parse_args()


def default_n(dim, p):
    # ~10M DOFs: (n p + 1)^dim
    return {2: round((10.0e6 ** 0.5 - 1) / p), 3: round((10.0e6 ** (1 / 3) - 1) / p)}[dim]


def workload(args):
    n = args.cells or default_n(args.dim, args.order)
    p = args.order
    ndofs = (n * p + 1) ** args.dim
    ne = n ** args.dim
    return n, p, ndofs, ne


class Clocks:
    """nvidia-smi sampling during a timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.file = None

    def __enter__(self):
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.file, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        try:
            for line in open(self.file.name):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    sm.append(float(f[0]))
                    mx.append(float(f[1]))
                except ValueError:
                    continue
                for name, v in zip(names, f[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(name)
        finally:
            os.unlink(self.file.name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def op_flops_per_element(dim, p, nq, kind):
    """Algorithmic FP64 flops of one element's sum-factorised PA action
    (tensor_kernels.cpp:67-110 in 2D, its 3D analogue): the forward
    contractions, the pointwise qdata product and the transposed
    contractions, a multiply-add counted as 2 flops."""
    D1, Q = p + 1, nq
    if dim == 2:
        if kind == "mass":
            return 2 * (2 * Q * D1 ** 2 + 2 * Q ** 2 * D1) + Q ** 2
        # T (2 chains), W (2), point (4 mul + 2 add), S (2), r (2) + final add
        return 2 * (4 * Q * D1 ** 2 + 4 * Q ** 2 * D1) + 6 * Q ** 2 + D1 ** 2
    fwd_m = Q * D1 ** 3 + Q ** 2 * D1 ** 2 + Q ** 3 * D1
    if kind == "mass":
        return 2 * 2 * fwd_m + Q ** 3
    # forward: (B, G) in x, three products in y, three gradients in z;
    # pointwise symmetric 3x3 (9 mul + 6 add); the transpose mirrors it
    fwd_d = 2 * Q * D1 ** 3 + 3 * Q ** 2 * D1 ** 2 + 3 * Q ** 3 * D1
    return 2 * 2 * fwd_d + 15 * Q ** 3 + 2 * D1 ** 3


def config_key(args, n):
    return f"{args.dim}d_bp{args.bp}_p{args.order}_n{n}_{args.numerics}"


def traffic_from_profile(args, n):
    """ncu-measured DRAM bytes per operator application for THIS workload
    (profiles/traffic.json, keyed by config_key), or None when no capture of
    this exact configuration exists -- never another config's number."""
    f = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(f.read_text())["configs"][config_key(args, n)]["operator"]
    except Exception:
        return None


# ------------------------------------------------------------ reference arm
def reference_problem(n, p, threads):
    from oracle.pyoracle import RefForm, RefSpace, RefSystem
    rs = RefSpace.cartesian(n, n, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)], threads=threads)
    sys_ = RefSystem(f, "front")
    b = np.random.default_rng(2020).uniform(-1.0, 1.0, rs.n_dofs)
    b[sys_.ess] = 0.0
    return rs, f, sys_, b


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference(n, p, iters, steps=1, warmup=0):
    """GDOF/s of the reference cg_solve (Jacobi) on this host; falls back to
    the C restatement when oracle/_ref is absent."""
    threads = host_threads()
    from oracle.pyoracle import Ref
    if Ref.available():
        rs, f, sys_, b = reference_problem(n, p, threads)
        kind = "reference"
        run = lambda: sys_.cg(0.0, iters, True, rhs=b)[3]
        ndofs = rs.n_dofs
    else:
        from oracle.pyoracle import OrcCartesian
        oc = OrcCartesian(2, (n, n), p)
        qd = oc.setup("diffusion")
        ess = oc.boundary_dofs()
        op = oc.operator(["diffusion"], [qd], ess)
        d = oc.diagonal("diffusion", qd)
        d[ess] = 1.0
        b = np.random.default_rng(2020).uniform(-1.0, 1.0, oc.ndofs)
        b[ess] = 0.0
        kind, threads, ndofs = "port", 1, oc.ndofs

        def run():
            t0 = time.perf_counter()
            oc.cg(op, b, 0.0, iters, d)
            return time.perf_counter() - t0
    for _ in range(warmup):
        run()
    secs = [run() for _ in range(steps)]
    return ndofs, secs, threads, kind


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.dim != 2:
        print(json.dumps({"impl": "reference",
                          "unavailable": "the reference supports 2D quadrilaterals only"}))
        return
    n, p, _, _ = workload(args)
    ndofs, secs, threads, kind = cpu_reference(n, p, args.cpu_iters, args.steps, args.warmup)
    t = sum(secs)
    value = ndofs * args.cpu_iters * args.steps / t / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "impl": "reference",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args, n, p, ndofs, per_step_iters=args.cpu_iters),
        "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": threads, "kind": kind,
                         "sample": f"{args.cpu_iters} Jacobi-CG iterations per step on the "
                                   f"same {ndofs}-DOF problem"},
        "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


def config_of(args, n, p, ndofs, per_step_iters=None, world=1):
    it = per_step_iters if per_step_iters is not None else args.iters
    dim = args.dim
    return {
        "workload": f"BP{args.bp} {dim}D p={p} n={n}^{dim} ({ndofs:,} DOFs/rank), "
                    + {1: "PA mass q=p+2 Gauss-Legendre, CG",
                       3: "PA diffusion q=p+2 Gauss-Legendre, Jacobi-PCG",
                       5: "PA diffusion q=p+1 Gauss-Lobatto, Jacobi-PCG"}[args.bp]
                    + f" {it} iterations per step",
        "dim": dim, "order": p, "cells_per_axis": n, "dofs_per_rank": ndofs,
        "dofs_total": ndofs * world, "iterations_per_step": it, "numerics": args.numerics,
        "l2": "inputs larger than L2 (qdata alone > 126 MB); no flush needed",
        "parallelism": f"element-partitioned x{world}" if world > 1 else "single GPU",
    }


# ---------------------------------------------------------------- our arm
def measure_config(tf, dev, dim, p, bp, n, iters, steps, warmup=1):
    """One more workload on the same device, device-resident, CUDA events:
    GDOF/s, the CG and the operator roofline fractions (tfem_cg_profile), and
    the true-residual check.  Used for the extra keys of the bench line."""
    import torch
    cells = (n,) * dim
    sp = tf.FeSpace.cartesian(dev, cells, p)
    a = tf.BilinearForm(sp)
    if bp == 1:
        a.add_mass(1.0)
    elif bp == 5:
        a.add_diffusion(1.0, rule="gauss_lobatto", nq=p + 1)
    else:
        a.add_diffusion(1.0)
    a.assemble()
    ess = sp.essential_true_dofs()
    op = tf.ConstrainedOperator(a, ess)
    diag = op.diagonal()
    pc = None if bp == 1 else diag
    N, E = sp.n_dofs, sp.n_elements
    b_host = np.random.default_rng(2020).uniform(-1.0, 1.0, N)
    b_host[ess] = 0.0
    b = tf.Vector.from_numpy(dev, b_host)
    x = tf.Vector(dev, N)
    for _ in range(warmup):
        res = tf.cg_solve(op, b, 0.0, iters, pc, x=x)
    stream = torch.cuda.ExternalStream(dev.stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev.sync()
    ev0.record(stream)
    for _ in range(steps):
        res = tf.cg_solve(op, b, 0.0, iters, pc, x=x)
    ev1.record(stream)
    ev1.synchronize()
    t = ev0.elapsed_time(ev1) / 1e3
    chk = result_check(tf, dev, op, b_host, res, iters)
    nc = 1 if bp == 1 else (3 if dim == 2 else 6)
    nq = p + 1 if bp == 5 else p + 2
    b_op = E * (nc * nq ** dim * 8 + (p + 1) ** dim * 4) + 16 * N
    b_it = b_op + (80 if bp == 1 else 96) * N
    seg = (C.c_double * 3)()
    xp = tf.Vector(dev, N)
    tf.abi.check(tf.lib().tfem_cg_profile(dev.h, op.h, b.h, min(iters, 100),
                                          pc.h if pc is not None else None, xp.h, seg))
    peak, _ = peaks()
    value = N * iters * steps / t / 1e9
    return {"workload": f"BP{bp} {dim}D p={p} n={n}^{dim}", "dofs": N, "value": value,
            "unit": "GDOF/s", "ms_per_step": 1e3 * t / steps, "iterations_per_step": iters,
            "steps": steps, "cg_frac": b_it * iters * steps / t / 1e9 / peak,
            "operator_frac": b_op / (seg[0] * 1e-6) / 1e9 / peak, "operator_us": seg[0],
            "result_check_drift": chk["drift"]}


def result_check(tf, dev, op, b_host, res, iters):
    """After the timed region: the last solve's x against its own claim.
    The true residual ||b - A x|| (one more device operator application,
    differences on the host) must equal the recursive residual the device CG
    tracked for the returned iterate (res.x_norm) up to the round-off drift of
    `iters` iterations; the iteration count must be the requested one."""
    N = b_host.size
    ax = tf.Vector(dev, N)
    op.mult(res.x, ax)
    r = b_host - ax.numpy()
    true_rel = float(np.linalg.norm(r) / np.linalg.norm(b_host))
    rec_rel = res.x_norm / res.initial_norm
    drift = abs(true_rel - rec_rel) / rec_rel
    ok = res.iterations == iters and drift <= 1e-6
    if not ok:
        raise SystemExit(f"bench: result check failed: iterations {res.iterations}/{iters}, "
                         f"true residual {true_rel:.6e} vs recursive {rec_rel:.6e}")
    return {"iterations": res.iterations, "true_rel_residual": true_rel,
            "recursive_rel_residual": rec_rel, "drift": drift, "ok": ok}


def run_tfem(args):
    import torch
    import paper_1911_09220_b200 as tf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        from paper_1911_09220_b200 import dist
        return dist.bench_distributed(args, rank, world, local)

    torch.cuda.set_device(local)
    dev = tf.Device(local, numerics=args.numerics)
    stream = torch.cuda.ExternalStream(dev.stream)
    n, p, _, _ = workload(args)
    cells = (n,) * args.dim

    t0 = time.perf_counter()
    sp = tf.FeSpace.cartesian(dev, cells, p)
    a = tf.BilinearForm(sp)
    if args.bp == 1:
        a.add_mass(1.0)
    elif args.bp == 5:
        a.add_diffusion(1.0, rule="gauss_lobatto", nq=p + 1)
    else:
        a.add_diffusion(1.0)
    a.assemble()
    ess = sp.essential_true_dofs()
    op = tf.ConstrainedOperator(a, ess)
    diag = op.diagonal()
    dev.sync()
    setup_s = time.perf_counter() - t0
    pc = None if args.bp == 1 else diag  # BP1: unpreconditioned CG
    N = sp.n_dofs
    E = sp.n_elements
    b_host = np.random.default_rng(2020).uniform(-1.0, 1.0, N)
    b_host[ess] = 0.0
    b = tf.Vector.from_numpy(dev, b_host)
    x = tf.Vector(dev, N)

    def step():
        return tf.cg_solve(op, b, 0.0, args.iters, pc, x=x)

    for _ in range(args.warmup):
        res = step()
    assert res.iterations == args.iters

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = dev.launch_count()
    dev.sync()
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res = step()
        ev1.record(stream)
        ev1.synchronize()
    t_value = ev0.elapsed_time(ev1) / 1e3
    launches = dev.launch_count() - launches0
    clocks = clk.summary()
    value = N * args.iters * args.steps / t_value / 1e9
    check = result_check(tf, dev, op, b_host, res, args.iters)

    # ---- the bit-exact numerics (reference operation order), same workload
    exact = None
    if args.numerics == "fma" and args.dim == 2 and not args.no_bitexact:
        dev.set_numerics("reference")
        for _ in range(2):
            step()
        dev.sync()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
        t_exact = ev0.elapsed_time(ev1) / 1e3
        exact = {"value": N * args.iters * args.steps / t_exact / 1e9, "unit": "GDOF/s",
                 "ms_per_step": 1e3 * t_exact / args.steps,
                 "note": "TFEM_NUMERICS_REFERENCE: bit-identical to the CPU reference"}
        dev.set_numerics(args.numerics)

    # ---- roofline of the dominant kernel: the operator application
    nc = 1 if args.bp == 1 else (3 if args.dim == 2 else 6)
    nq = p + 1 if args.bp == 5 else p + 2
    b_op = E * (nc * nq ** args.dim * 8 + (p + 1) ** args.dim * 4) + 16 * N
    xin = tf.Vector.from_numpy(dev, b_host)
    yout = tf.Vector(dev, N)
    lib = tf.lib()
    for _ in range(3):
        tf.abi.check(lib.tfem_operator_mult_async(dev.h, op.h, xin.h, yout.h))
    M = 50
    dev.sync()
    ev0.record(stream)
    for _ in range(M):
        tf.abi.check(lib.tfem_operator_mult_async(dev.h, op.h, xin.h, yout.h))
    ev1.record(stream)
    ev1.synchronize()
    t_op_alone = ev0.elapsed_time(ev1) / 1e3 / M
    # The operator as it runs inside the solve (tfem_cg_profile: eager CG
    # iterations with events between the launches); p arrives partly
    # L2-resident from the direction kernel, which the standalone loop above
    # does not see.
    seg = (C.c_double * 3)()
    xprof = tf.Vector(dev, N)
    tf.abi.check(lib.tfem_cg_profile(dev.h, op.h, xin.h, min(args.iters, 100),
                                     pc.h if pc is not None else None, xprof.h, seg))
    del xin, yout, xprof
    t_op = seg[0] * 1e-6
    # FP64 side of the same launch: algorithmic flops against the measured
    # CUDA-core DFMA peak (probe.cu; the element kernels use no tensor cores)
    fpeak = C.c_double(0.0)
    tf.abi.check(lib.tfem_fp64_peak(dev.h, C.byref(fpeak)))
    f_op = E * op_flops_per_element(args.dim, p, nq, "mass" if args.bp == 1 else "diffusion")
    fp64 = {"achieved": f_op / t_op / 1e12, "peak": fpeak.value, "unit": "TFLOP/s",
            "frac": f_op / t_op / 1e12 / fpeak.value if fpeak.value > 0 else None,
            "flops_per_launch": f_op, "flops_per_dof": f_op / N,
            "peak_source": "measured (tfem_fp64_peak: DFMA chains on every SM)"}
    peak, peak_kind = peaks()
    achieved = b_op / t_op / 1e9
    b_it = b_op + (80 if args.bp == 1 else 96) * N
    cg_achieved = b_it * args.iters * args.steps / t_value / 1e9
    # update: read r, q (, d), write r; direction: read x, p, r (, d), write
    # x', p (the x update runs in the direction kernel; no diag in BP1)
    bu, bd = (24, 40) if args.bp == 1 else (32, 48)
    cg_kernels = {
        "operator": {"us": seg[0], "bytes_per_dof": b_op / N, "frac": achieved / peak},
        "update": {"us": seg[1], "bytes_per_dof": bu,
                   "frac": bu * N / (seg[1] * 1e-6) / 1e9 / peak},
        "direction": {"us": seg[2], "bytes_per_dof": bd,
                      "frac": bd * N / (seg[2] * 1e-6) / 1e9 / peak},
        "standalone_operator_us": 1e6 * t_op_alone,
        "source": "tfem_cg_profile (CUDA events between the launches of eager iterations)",
    }

    # ---- end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        bp = torch.from_numpy(b_host).pin_memory()
        dp = torch.from_numpy(diag.numpy()).pin_memory()
        xp = torch.empty(N, dtype=torch.float64).pin_memory()
        bh, dh, xh = bp.numpy(), dp.numpy(), xp.numpy()
        if pc is None:
            dh = None
        # the device-resident legs are done: their vectors make room for the
        # API's own device copies of b / diag / x (1B DOFs fill the GPU)
        del res, b, x, diag, pc
        tf.cg_solve_host(op, bh, 0.0, args.iters, dh, out=xh)
        dev.sync()
        w0 = time.perf_counter()
        ev0.record(stream)
        for _ in range(args.steps):
            _, it, _ = tf.cg_solve_host(op, bh, 0.0, args.iters, dh, out=xh)
        ev1.record(stream)
        ev1.synchronize()
        t_e2e = max(ev0.elapsed_time(ev1) / 1e3, 0.0)
        t_wall = time.perf_counter() - w0
        t_e = max(t_e2e, t_wall)
        e2e = {"value": N * args.iters * args.steps / t_e / 1e9, "unit": "GDOF/s",
               "h2d_bytes_per_step": 16 * N, "d2h_bytes_per_step": 8 * N,
               "ms_per_step": 1e3 * t_e / args.steps,
               "api": "tfem_cg_solve_host (pinned host b, diag -> x)"}

    # ---- end to end through the reference's own C++ API (the drop-in build:
    # form_linear_system + cg_solve on host Vectors, integration/bench_dropin)
    dropin = None
    exe = ROOT / "integration" / "_build" / "bin" / "bench_dropin"
    if not args.no_e2e and args.dim == 2 and args.bp == 3 and exe.exists():
        del op, a, sp
        dev.sync()
        out = subprocess.run([str(exe), str(n), str(p), str(args.iters), str(args.steps),
                              str(args.warmup)], capture_output=True, text=True, timeout=900)
        try:
            dropin = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            dropin = {"error": (out.stdout + out.stderr)[-500:]}

    # ---- extra configurations the north star names (same device, after the
    # headline legs): 3D BP3 p=3 at ~10M DOFs and 2D BP3 p=3 at ~100M DOFs
    extra = None
    if not args.no_extra and args.dim == 2 and args.bp == 3 and args.order == 3 and not args.cells:
        extra = {}
        for key, (dim, nn, steps) in {"3d_bp3_p3_10M": (3, 72, 5),
                                      "2d_bp3_p3_100M": (2, 3334, 3)}.items():
            try:
                extra[key] = measure_config(tf, dev, dim, 3, 3, nn, args.iters, steps)
            except Exception as e:  # reported, never required
                extra[key] = {"error": str(e)[:300]}

    cpu = None
    if not args.no_cpu_baseline and args.dim == 2:
        try:
            ndofs_c, secs, threads, kind = cpu_reference(n, p, args.cpu_iters)
            cpu = {"value": ndofs_c * args.cpu_iters / secs[0] / 1e9, "unit": "GDOF/s",
                   "cores": threads, "kind": kind,
                   "sample": f"{args.cpu_iters} Jacobi-CG iterations of the same "
                             f"{ndofs_c:,}-DOF problem ({secs[0]:.2f} s)"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GDOF/s", "cores": host_threads(), "kind": "reference",
                   "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_value / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args, n, p, N),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_from_profile(args, n),
                     "kernel": "PA operator (element kernel + shared-DOF scatter)",
                     "bytes_per_launch": b_op, "ms_per_launch": 1e3 * t_op,
                     "peak_source": peak_kind, "fp64": fp64},
        "cg_roofline": {"achieved": cg_achieved, "frac": cg_achieved / peak, "unit": "GB/s",
                        "bytes_per_dof_iteration": b_it / N, "kernels": cg_kernels},
        "e2e": e2e, "e2e_dropin": dropin, "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": launches,
        "bit_exact_numerics": exact, "setup_s": setup_s, "result_check": check,
        "extra_configs": extra,
    }
    print(json.dumps(line))


def self_launch(args):
    """--gpus N without torchrun: re-launch this command as N ranks (one per
    GPU, torchrun, 127.0.0.1); a box with fewer GPUs is an error."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but this box has "
                                                     f"{have} CUDA device(s)"}))
        sys.exit(2)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


def main():
    args = parse()
    world = os.environ.get("WORLD_SIZE")
    if world is not None and int(world) != args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}))
        sys.exit(2)
    if world is None and args.gpus > 1 and args.impl != "reference":
        self_launch(args)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_tfem(args)


if __name__ == "__main__":
    main()
