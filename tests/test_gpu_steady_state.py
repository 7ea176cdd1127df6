"""GPU parity at steady-state sizes: every element-kernel family compared with
the oracle on meshes where each persistent block / warp runs several laps of
its bulk-copy ring, in the numerics that get benchmarked.

The round-1 parity tests used meshes small enough that most kernels ran one
tile per block (the empty-barrier waits and ring wrap never executed).  Here:

* full-size operator actions (the BASELINE configs[1] BP3 mesh, 2D p >= 4 at
  n = 300, 3D at n = 24) against the C restatement (oracle/tfem_oracle.c,
  bit-equal to the reference on every 2D rule -- tests/test_oracle_ref.py):
  `==` in TFEM_NUMERICS_REFERENCE (2D), <= 1e-12 relative in the FMA
  numerics (the default, the one bench.py times);
* CG iteration counts on the driver's `front` system (2D: the reference
  itself, oracle/_ref) and on seeded 3D systems (the restatement), with the
  persistent grids capped (tfem_ctx_set_max_blocks) so that even these
  oracle-affordable meshes wrap every ring many times; tol 1e-10, as in
  acceptance_main.cpp:187-234 criterion 1 style comparisons.
"""
import numpy as np
import pytest

from oracle.pyoracle import OrcCartesian, RefForm, RefSpace, RefSystem
import paper_1911_09220_b200 as tf

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def rng_vec(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


@pytest.fixture
def capped(request):
    """A device whose persistent element kernels run on `max_blocks` blocks."""
    numerics, blocks = request.param
    d = tf.Device(0, numerics=numerics)
    d.set_max_blocks(blocks)
    yield d
    d.close()


def _form(sp, kind, rule="gauss_legendre"):
    a = tf.BilinearForm(sp)
    if kind == "mass":
        a.add_mass(1.0, rule=rule)
    else:
        a.add_diffusion(1.0, rule=rule)
    a.assemble()
    return a


def _check_operator(dev, n, p, kind, exact, rule="gl", seed=1):
    """Unconstrained action, constrained (CG) action and diagonal."""
    dim = len(n)
    oc = OrcCartesian(dim, n, p, rule=rule)
    sp = tf.FeSpace.cartesian(dev, n, p)
    a = _form(sp, kind, "gauss_legendre" if rule == "gl" else "gauss_lobatto")
    qd = oc.setup(kind)
    x = rng_vec(sp.n_dofs, seed)
    y = tf.Vector(dev, sp.n_dofs)
    a.mult_true(x, y)
    want = oc.apply(kind, qd, x)
    if exact:
        assert (y.numpy() == want).all(), rel(y.numpy(), want)
    else:
        assert rel(y.numpy(), want) <= 1e-12
    ess = sp.essential_true_dofs()
    op = tf.ConstrainedOperator(a, ess)
    oop = oc.operator([kind], [qd], ess)
    op.mult(x, y)
    want = oc.op_mult(oop, x)
    if exact:
        assert (y.numpy() == want).all(), rel(y.numpy(), want)
    else:
        assert rel(y.numpy(), want) <= 1e-12
    d = a.diagonal_true().numpy()
    dref = oc.diagonal(kind, qd)
    assert (d == dref).all() if exact else rel(d, dref) <= 1e-12


# ------------------------------------------------------------- full size
@pytest.mark.parametrize("numerics", ["fma", "reference"])
def test_bp3_headline_mesh(numerics):
    """configs[1]: make_cartesian(1054, 1054), p = 3 (10,004,569 DOFs): the
    benchmarked kernel (apply2d_tma<3,5>, FMA: 5-stage ring, one x buffer)
    runs ~34 laps per block; unconstrained and constrained action, diagonal."""
    dev = tf.Device(0, numerics=numerics)
    try:
        _check_operator(dev, (1054, 1054), 3, "diffusion", numerics == "reference", seed=42)
    finally:
        dev.close()


@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
def test_2d_low_order_large(dev_fma, p, kind):
    n = {1: 1500, 2: 800}[p]
    _check_operator(dev_fma, (n, n), p, kind, False, seed=p)


@pytest.mark.parametrize("p", [4, 5, 6, 7, 8])
@pytest.mark.parametrize("numerics", ["fma", "reference"])
def test_2d_high_order_n300(p, numerics):
    """apply2d_hi at n = 300 (90,000 elements: 10-30 laps of each warp's
    two-slot ring), both numerics (their warp counts differ at p = 7)."""
    dev = tf.Device(0, numerics=numerics)
    try:
        _check_operator(dev, (300, 300), p, "diffusion", numerics == "reference", seed=p)
    finally:
        dev.close()


@pytest.mark.parametrize("p", [4, 7, 8])
def test_2d_high_order_mass_and_bp5(dev_fma, p):
    _check_operator(dev_fma, (300, 300), p, "mass", False, seed=3)
    _check_operator(dev_fma, (300, 300), p, "diffusion", False, rule="gll", seed=4)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_3d_n24(dev_fma, p):
    """3D BP3 at 24^3 elements: apply3d_tma (q <= 7) or apply_grp (q >= 8),
    several laps per warp; action, constrained action, diagonal."""
    _check_operator(dev_fma, (24, 24, 24), p, "diffusion", False, seed=p)


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6, 7, 8])
def test_3d_bp5_n24(dev_fma, p):
    _check_operator(dev_fma, (24, 24, 24), p, "diffusion", False, rule="gll", seed=10 + p)


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_3d_bp1_mass_n24(dev_fma, p):
    _check_operator(dev_fma, (24, 24, 24), p, "mass", False, seed=20 + p)


# ------------------------------------------------- CG, rings wrapped
def _cg_2d(dev, p, n, jacobi):
    rs = RefSpace.cartesian(n, n, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    rsys = RefSystem(f, "front")
    xr, itr, cr, _ = rsys.cg(1e-10, 5000, jacobi)
    sp = tf.FeSpace.cartesian(dev, (n, n), p)
    a = _form(sp, "diffusion")
    op = tf.ConstrainedOperator(a, sp.essential_true_dofs())
    res = tf.cg_solve(op, rsys.rhs, 1e-10, 5000, op.diagonal() if jacobi else None)
    assert res.converged == cr
    assert res.iterations == itr, (res.iterations, itr)
    assert np.abs(res.x.numpy() - xr).max() <= 1e-8 * np.abs(xr).max()


@pytest.mark.parametrize("capped", [("fma", 2), ("reference", 2)], indirect=True)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_cg_iterations_2d_wrapped(capped, p):
    """The driver's front system on a 48 x 48 (p <= 3) / 24 x 24 mesh with
    the element kernels on 2 blocks: every block runs >= 5 laps of its ring
    during each of the hundreds of CG iterations; iteration counts equal the
    reference's cg_solve."""
    _cg_2d(capped, p, 48 if p <= 3 else 24, True)


@pytest.mark.parametrize("capped", [("fma", 2)], indirect=True)
@pytest.mark.parametrize("p", [2, 3, 6])
def test_cg_iterations_2d_wrapped_no_jacobi(capped, p):
    _cg_2d(capped, p, 48 if p <= 3 else 24, False)


def test_numerics_switch_on_one_operator():
    """the element grid depends on the numerics (p = 7, q = 9:
    13 vs 11 warps per block); switching numerics on an existing operator must
    refit the CG workspace's dot sinks (meshes of 705-832 elements change the
    32-block chunk count).  Both solves must match the reference's count."""
    p, n = 7, 28  # 784 elements
    rs = RefSpace.cartesian(n, n, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    rsys = RefSystem(f, "front")
    _, itr, _, _ = rsys.cg(1e-10, 5000, True)
    dev = tf.Device(0, numerics="fma")
    try:
        for blocks in (0, 3):
            dev.set_max_blocks(blocks)
            sp = tf.FeSpace.cartesian(dev, (n, n), p)
            a = _form(sp, "diffusion")
            op = tf.ConstrainedOperator(a, sp.essential_true_dofs())
            d = op.diagonal()
            for mode in ("fma", "reference", "fma"):
                dev.set_numerics(mode)
                res = tf.cg_solve(op, rsys.rhs, 1e-10, 5000, d)
                assert res.converged and res.iterations == itr, (mode, blocks, res.iterations)
    finally:
        dev.close()


def _cg_3d(dev, n, p, kind, rule, jacobi, seed):
    oc = OrcCartesian(3, n, p, rule=rule)
    sp = tf.FeSpace.cartesian(dev, n, p)
    a = _form(sp, kind, "gauss_legendre" if rule == "gl" else "gauss_lobatto")
    qd = oc.setup(kind)
    if kind == "mass":
        ess = np.zeros(0, dtype=np.int32)
        op = a.operator()
        oop = oc.operator([kind], [qd])
    else:
        ess = sp.essential_true_dofs()
        op = tf.ConstrainedOperator(a, ess)
        oop = oc.operator([kind], [qd], ess)
    b = rng_vec(sp.n_dofs, seed)
    b[ess] = 0.0
    d = do = None
    if jacobi:
        d = op.diagonal()
        do = oc.diagonal(kind, qd)
        do[ess] = 1.0
    res = tf.cg_solve(op, b, 1e-10, 5000, d)
    xo, ito, co = oc.cg(oop, b, 1e-10, 5000, do)
    assert res.converged and co
    assert res.iterations == ito, (res.iterations, ito)
    assert np.abs(res.x.numpy() - xo).max() <= 1e-8 * np.abs(xo).max()


@pytest.mark.parametrize("capped", [("fma", 2)], indirect=True)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_cg_iterations_3d_wrapped(capped, p):
    """3D BP3 (Jacobi) on 2 blocks: tens of laps of every warp's ring per
    application; iteration count equal to the restatement's cg."""
    n = {1: 12, 2: 10, 3: 8, 4: 7, 5: 6, 6: 6, 7: 5, 8: 5}[p]
    _cg_3d(capped, (n, n, n), p, "diffusion", "gl", True, seed=p)


@pytest.mark.parametrize("capped", [("fma", 2)], indirect=True)
@pytest.mark.parametrize("p", [2, 4, 6, 7, 8])
def test_cg_iterations_3d_bp5_wrapped(capped, p):
    # p = 8 at n = 5 stops one iteration before the restatement (263 vs 264:
    # the device's relative residual 9.83e-11 crosses the 1e-10 threshold
    # within FMA-vs-reference rounding); n = 4 stays clear of the threshold.
    # The p = 8 operator itself is checked at 1e-12 in test_3d_bp5_n24.
    n = {2: 10, 4: 7, 6: 6, 7: 5, 8: 4}[p]
    _cg_3d(capped, (n, n, n), p, "diffusion", "gll", True, seed=30 + p)


@pytest.mark.parametrize("capped", [("fma", 2)], indirect=True)
def test_cg_iterations_3d_bp1_wrapped(capped):
    _cg_3d(capped, (16, 16, 16), 2, "mass", "gl", False, seed=7)
