"""Generate tests/golden/reference_2d.npz from the UNMODIFIED reference
(oracle/_ref/libtfem_ref.so built from /root/reference/proj/src).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixture is committed; tests/test_golden.py checks the C restatement (CPU)
and the device path (GPU) against it, so parity stays pinned on boxes that
have no /root/reference.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import Ref, RefForm, RefSpace, RefSystem, ref_cg_csr  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_2d.npz"


def x_for(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def main():
    g = {}
    for n in range(1, 11):
        g[f"gl_{n}_x"], g[f"gl_{n}_w"] = Ref.rule(n)
        if n >= 2:
            g[f"gll_{n}_x"], g[f"gll_{n}_w"] = Ref.rule(n, lobatto=True)
    for p in range(1, 9):
        g[f"B_{p}_gl"], g[f"G_{p}_gl"] = Ref.eval_matrices(p, p + 2, 0, 0)
        g[f"B_{p}_gll"], g[f"G_{p}_gll"] = Ref.eval_matrices(p, p + 1, 0, 1)
    # Cartesian 5 x 4 on [0,2] x [0,1], kappa / rho = 1 + x + 2y
    for p in (1, 2, 3, 4):
        rs = RefSpace.cartesian(5, 4, p, 2.0, 1.0)
        g[f"cart_{p}_dofs"] = rs.element_dofs()
        g[f"cart_{p}_ess"] = rs.essential()
        for kind in ("diffusion", "mass"):
            f = RefForm(rs, [(kind, "varying", 0.0)])
            x = x_for(rs.n_dofs, 10 * p)
            g[f"cart_{p}_{kind}_qdata"] = f.qdata()
            g[f"cart_{p}_{kind}_x"] = x
            g[f"cart_{p}_{kind}_y"] = f.mult(x)
            g[f"cart_{p}_{kind}_diag"] = f.diagonal()
        _, cnt = RefForm(RefSpace.cartesian(1, 1, p), [("diffusion", "const", 1.0)]).mult_count(
            x_for((p + 1) ** 2, 1))
        g[f"mults_{p}"] = np.array(cnt)
    # curved order-2 mesh (acceptance criterion 1 fixture)
    rs = RefSpace.curved(4, 2, 2)
    f = RefForm(rs, [("diffusion", "varying", 0.0)])
    x = x_for(rs.n_dofs, 77)
    g["curved_dofs"] = rs.element_dofs()
    g["curved_ctrl"] = rs.ctrl_points()
    g["curved_qdata"] = f.qdata()
    g["curved_x"] = x
    g["curved_y"] = f.mult(x)
    # driver system: front solution, 8 x 8, p = 2, Jacobi, tol 1e-12
    rs = RefSpace.cartesian(8, 8, 2)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    sysr = RefSystem(f, "front")
    x = x_for(rs.n_dofs, 5)
    g["sys_rhs"], g["sys_diag"], g["sys_ess"] = sysr.rhs, sysr.diag, sysr.ess
    g["sys_x"], g["sys_opx"] = x, sysr.op_mult(x)
    xs, it, conv, _ = sysr.cg(1e-12, 2000, True)
    g["sys_cg_x"], g["sys_cg_iters"], g["sys_cg_conv"] = xs, np.array(it), np.array(conv)
    # CG exhaustion on the tridiagonal matrix of test_linalg.cpp:283-304
    n = 50
    rows, cols, vals = [0], [], []
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                cols.append(j)
                vals.append(v)
        rows.append(len(cols))
    rp, cc, vv = np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals)
    xt, itt, ct = ref_cg_csr(rp, cc, vv, np.ones(n), 1e-14, 24)
    g["tri_rowptr"], g["tri_cols"], g["tri_vals"] = rp, cc, vv
    g["tri_x"], g["tri_iters"], g["tri_conv"] = xt, np.array(itt), np.array(ct)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
