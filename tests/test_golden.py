"""Golden vectors made from the unmodified reference (tests/golden/
make_golden.py -> reference_2d.npz, committed).

CPU: the C restatement reproduces every golden bit for bit (so the oracle is
pinned even where /root/reference is absent).  GPU: the device path through
the C ABI reproduces them bit for bit (CG: same iteration count, solution to
round-off)."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from oracle.pyoracle import Orc, OrcCartesian, _d, _i

G = np.load(Path(__file__).resolve().parent / "golden" / "reference_2d.npz")


@pytest.fixture(scope="module")
def orc(oracle_built):
    return Orc


def test_rules_and_tables(orc):
    for n in range(1, 11):
        x, w = Orc.rule(n)
        assert (x == G[f"gl_{n}_x"]).all() and (w == G[f"gl_{n}_w"]).all()
        if n >= 2:
            x, w = Orc.rule(n, lobatto=True)
            assert (x == G[f"gll_{n}_x"]).all() and (w == G[f"gll_{n}_w"]).all()
    for p in range(1, 9):
        B, Gm = Orc.eval_matrices(p, p + 2, 0, 0)
        assert (B == G[f"B_{p}_gl"]).all() and (Gm == G[f"G_{p}_gl"]).all()
        B, Gm = Orc.eval_matrices(p, p + 1, 0, 1)
        assert (B == G[f"B_{p}_gll"]).all() and (Gm == G[f"G_{p}_gll"]).all()


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
def test_cartesian_restatement(orc, p, kind):
    oc = OrcCartesian(2, (5, 4), p, ext=[2.0, 1.0])
    assert (oc.elem_dofs == G[f"cart_{p}_dofs"]).all()
    assert (oc.boundary_dofs() == G[f"cart_{p}_ess"]).all()
    pts = oc.points()
    qd = oc.setup(kind, coeff=1.0 + pts[..., 0] + 2.0 * pts[..., 1])
    assert (qd == G[f"cart_{p}_{kind}_qdata"]).all()
    x = G[f"cart_{p}_{kind}_x"]
    assert (oc.apply(kind, qd, x) == G[f"cart_{p}_{kind}_y"]).all()
    assert (oc.diagonal(kind, qd) == G[f"cart_{p}_{kind}_diag"]).all()


def test_curved_restatement(orc):
    oc = OrcCartesian(2, (4, 4), 2)
    pts = np.zeros((oc.ne, oc.nqd, 2))
    Orc.check(Orc.lib().orc_physical_points(2, 2, oc.ne, _d(np.ascontiguousarray(G["curved_ctrl"])),
                                            oc.nq, 0, _d(pts)))
    qd = oc.setup("diffusion", ctrl=G["curved_ctrl"], geom_order=2,
                  coeff=1.0 + pts[..., 0] + 2.0 * pts[..., 1])
    assert (qd == G["curved_qdata"]).all()
    assert (oc.apply("diffusion", qd, G["curved_x"]) == G["curved_y"]).all()


def test_system_and_cg_restatement(orc):
    oc = OrcCartesian(2, (8, 8), 2)
    qd = oc.setup("diffusion")
    op = oc.operator(["diffusion"], [qd], G["sys_ess"])
    assert (oc.op_mult(op, G["sys_x"]) == G["sys_opx"]).all()
    d = oc.diagonal("diffusion", qd)
    d[G["sys_ess"]] = 1.0
    assert (d == G["sys_diag"]).all()
    x, it, conv = oc.cg(op, G["sys_rhs"], 1e-12, 2000, G["sys_diag"])
    assert it == int(G["sys_cg_iters"]) and conv == bool(G["sys_cg_conv"])
    assert (x == G["sys_cg_x"]).all()
    n = 50
    xt = np.zeros(n)
    it, cv = C.c_int(), C.c_int()
    Orc.check(Orc.lib().orc_cg_csr(n, _i(G["tri_rowptr"]), _i(G["tri_cols"]), _d(G["tri_vals"]),
                                   _d(np.ones(n)), 1e-14, 24, None, _d(xt), C.byref(it),
                                   C.byref(cv)))
    assert it.value == int(G["tri_iters"]) and (xt == G["tri_x"]).all()


# ------------------------------------------------------------------ device
@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
def test_device_cartesian(dev, p, kind):
    import paper_1911_09220_b200 as tf
    sp = tf.FeSpace.cartesian(dev, (5, 4), p, extents=(2.0, 1.0))
    assert (sp.element_dofs() == G[f"cart_{p}_dofs"]).all()
    assert (sp.essential_true_dofs() == G[f"cart_{p}_ess"]).all()
    pa = tf.pa_setup(sp, kind, lambda q: 1.0 + q[..., 0] + 2.0 * q[..., 1])
    assert (pa.qdata() == G[f"cart_{p}_{kind}_qdata"]).all()
    y = tf.Vector(dev, sp.n_dofs)
    tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, G[f"cart_{p}_{kind}_x"]), y)
    assert (y.numpy() == G[f"cart_{p}_{kind}_y"]).all()
    assert (tf.pa_diagonal(pa, sp).numpy() == G[f"cart_{p}_{kind}_diag"]).all()
    if kind == "diffusion":
        s1 = tf.FeSpace.cartesian(dev, (1, 1), p)
        a = tf.BilinearForm(s1)
        a.add_diffusion(1.0)
        a.assemble()
        tf.reset_multiply_count()
        a.mult_true(tf.Vector(dev, s1.n_dofs), tf.Vector(dev, s1.n_dofs))
        assert tf.multiply_count() == int(G[f"mults_{p}"])


@pytest.mark.gpu
def test_device_curved(dev):
    import paper_1911_09220_b200 as tf
    sp = tf.FeSpace.from_mesh(dev, 2, 2, G["curved_dofs"], int(G["curved_dofs"].max()) + 1,
                              G["curved_ctrl"], 2)
    pa = tf.pa_setup(sp, "diffusion", lambda q: 1.0 + q[..., 0] + 2.0 * q[..., 1])
    assert (pa.qdata() == G["curved_qdata"]).all()
    y = tf.Vector(dev, sp.n_dofs)
    tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, G["curved_x"]), y)
    assert (y.numpy() == G["curved_y"]).all()


@pytest.mark.gpu
def test_device_system_and_cg(dev):
    import paper_1911_09220_b200 as tf
    sp = tf.FeSpace.cartesian(dev, (8, 8), 2)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    op = tf.ConstrainedOperator(a, G["sys_ess"])
    y = tf.Vector(dev, sp.n_dofs)
    op.mult(G["sys_x"], y)
    assert (y.numpy() == G["sys_opx"]).all()
    assert (op.diagonal().numpy() == G["sys_diag"]).all()
    res = tf.cg_solve(op, G["sys_rhs"], 1e-12, 2000, G["sys_diag"])
    assert res.iterations == int(G["sys_cg_iters"]) and res.converged == bool(G["sys_cg_conv"])
    xr = G["sys_cg_x"]
    assert np.abs(res.x.numpy() - xr).max() <= 1e-10 * np.abs(xr).max()
    tri = tf.SparseOperator(dev, G["tri_rowptr"], G["tri_cols"], G["tri_vals"])
    r2 = tf.cg_solve(tri, np.ones(50), 1e-14, 24)
    assert r2.iterations == int(G["tri_iters"]) and r2.converged == bool(G["tri_conv"])
    assert np.abs(r2.x.numpy() - G["tri_x"]).max() <= 1e-12
