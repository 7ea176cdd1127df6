"""GPU parity, 3D and BP5 (q = p+1 Gauss-Lobatto): the sm_100a path against
the C restatement (oracle/tfem_oracle.c; pinned by tests/test_oracle_3d.py,
no reference exists for 3D).

Bars: layout / boundary / quadrature data / diagonal bit-identical (the
setup and diagonal kernels evaluate the restatement's exact order); operator
action within 1e-12 relative (fused multiply-adds, different contraction
order); CG iteration counts identical at a fixed tolerance.
"""
import numpy as np
import pytest

from oracle.pyoracle import OrcCartesian
import paper_1911_09220_b200 as tf

pytestmark = pytest.mark.gpu


def varying3(pts):
    return 1.0 + pts[..., 0] + 2.0 * pts[..., 1] + 3.0 * pts[..., 2]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_layout_3d(dev, p):
    n = (3, 2, 2)
    oc = OrcCartesian(3, n, p)
    sp = tf.FeSpace.cartesian(dev, n, p)
    assert sp.n_dofs == oc.ndofs
    assert (sp.element_dofs() == oc.elem_dofs).all()
    assert (sp.essential_true_dofs() == oc.boundary_dofs()).all()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 8])
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
@pytest.mark.parametrize("rule", ["gl", "gll"])
def test_qdata_apply_diag_3d(dev, p, kind, rule):
    n = (3, 2, 2)
    ext = [1.0, 0.7, 1.3]
    oc = OrcCartesian(3, n, p, rule=rule, ext=ext)
    sp = tf.FeSpace.cartesian(dev, n, p, extents=ext)
    rname = "gauss_legendre" if rule == "gl" else "gauss_lobatto"
    pa = tf.pa_setup(sp, kind, varying3, rule=rname)
    qd = oc.setup(kind, coeff=varying3(oc.points()))
    assert (pa.qdata() == qd).all()
    x = np.random.default_rng(p).uniform(-1, 1, sp.n_dofs)
    y = tf.Vector(dev, sp.n_dofs)
    tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, x), y)
    assert rel(y.numpy(), oc.apply(kind, qd, x)) <= 1e-12
    d = tf.pa_diagonal(pa, sp).numpy()
    assert (d == oc.diagonal(kind, qd)).all()


def test_bp1_mass_cg_3d(dev):
    """BP1 (configs[0]): PA mass + CG on the 16^3 hex mesh, p = 2, no
    preconditioner; iteration count identical to the restatement."""
    n, p = (16, 16, 16), 2
    oc = OrcCartesian(3, n, p)
    sp = tf.FeSpace.cartesian(dev, n, p)
    assert sp.n_dofs == 35937
    a = tf.BilinearForm(sp)
    a.add_mass(1.0)
    a.assemble()
    op = a.operator()
    b = np.random.default_rng(7).uniform(-1, 1, sp.n_dofs)
    res = tf.cg_solve(op, b, 1e-10, 500)
    qd = oc.setup("mass")
    xo, ito, co = oc.cg(oc.operator(["mass"], [qd]), b, 1e-10, 500)
    assert res.converged and co
    assert res.iterations == ito
    assert np.abs(res.x.numpy() - xo).max() <= 1e-8 * np.abs(xo).max()


@pytest.mark.parametrize("p", [2, 3])
def test_bp3_diffusion_jacobi_cg_3d(dev, p):
    n = (6, 5, 4)
    oc = OrcCartesian(3, n, p)
    sp = tf.FeSpace.cartesian(dev, n, p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    ess = sp.essential_true_dofs()
    op = tf.ConstrainedOperator(a, ess)
    d = op.diagonal()
    b = np.random.default_rng(3).uniform(-1, 1, sp.n_dofs)
    b[ess] = 0.0
    res = tf.cg_solve(op, b, 1e-10, 2000, d)
    qd = oc.setup("diffusion")
    do = oc.diagonal("diffusion", qd)
    do[ess] = 1.0
    assert (d.numpy() == do).all()
    xo, ito, co = oc.cg(oc.operator(["diffusion"], [qd], ess), b, 1e-10, 2000, do)
    assert res.converged and co
    assert res.iterations == ito
    assert np.abs(res.x.numpy() - xo).max() <= 1e-8 * np.abs(xo).max()


def test_bp5_gll_3d_cg(dev):
    """BP5: collocated GLL diffusion (q = p+1), p = 4."""
    n, p = (3, 3, 2), 4
    oc = OrcCartesian(3, n, p, rule="gll")
    sp = tf.FeSpace.cartesian(dev, n, p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0, rule="gauss_lobatto")
    a.assemble()
    ess = sp.essential_true_dofs()
    op = tf.ConstrainedOperator(a, ess)
    b = np.random.default_rng(5).uniform(-1, 1, sp.n_dofs)
    b[ess] = 0.0
    d = op.diagonal()
    res = tf.cg_solve(op, b, 1e-10, 2000, d)
    qd = oc.setup("diffusion")
    do = oc.diagonal("diffusion", qd)
    do[ess] = 1.0
    xo, ito, co = oc.cg(oc.operator(["diffusion"], [qd], ess), b, 1e-10, 2000, do)
    assert res.converged and co and res.iterations == ito


def test_3d_large_properties(dev):
    """At a size the oracle cannot do quickly: the operator is symmetric and
    annihilates constants, the mass integrates the volume (size-independent
    properties)."""
    n, p = (24, 24, 24), 3
    sp = tf.FeSpace.cartesian(dev, n, p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    ones = tf.Vector(dev, sp.n_dofs, 1.0)
    y = tf.Vector(dev, sp.n_dofs)
    a.mult_true(ones, y)
    assert np.abs(y.numpy()).max() <= 1e-11
    rng = np.random.default_rng(0)
    x1, x2 = rng.uniform(-1, 1, (2, sp.n_dofs))
    y1 = tf.Vector(dev, sp.n_dofs)
    y2 = tf.Vector(dev, sp.n_dofs)
    a.mult_true(x1, y1)
    a.mult_true(x2, y2)
    assert x2 @ y1.numpy() == pytest.approx(x1 @ y2.numpy(), rel=1e-11)
    m = tf.BilinearForm(sp)
    m.add_mass(1.0)
    m.assemble()
    m.mult_true(ones, y)
    assert y.numpy().sum() == pytest.approx(1.0, rel=1e-12)


@pytest.mark.parametrize("p", [3, 7])
def test_contraction_ab_probe(dev, p):
    """The DFMA vs DMMA contraction A/B (tools/contraction_ab.py): both
    variants compute the same stage (<= 1e-13 relative) and report rates."""
    import ctypes as C
    res = (C.c_double * 4)()
    tf.abi.check(tf.lib().tfem_contraction_ab(dev.h, p, res))
    assert res[2] <= 1e-13
    assert res[0] > 0.5 and res[1] > 0.5
    assert res[3] >= 1.0
    with pytest.raises(tf.InvalidArgument):
        tf.abi.check(tf.lib().tfem_contraction_ab(dev.h, 9, res))
