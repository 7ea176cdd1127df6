"""GPU parity beyond p = 8 and geometry order 3: the reference targets orders
up to 16 (basis.cpp:12-93 has no cap) and curves meshes to any
order (mesh.cpp:323-373).  2D p = 9..16 run the generic shared-memory stage
kernel (apply_grp.cu); bit-identical (`==`) to the unmodified reference
(oracle/_ref) in the reference numerics, <= 1e-12 in FMA numerics, and CG
iteration counts equal on the driver's front system."""
import numpy as np
import pytest

from oracle.pyoracle import RefForm, RefSpace, RefSystem
import paper_1911_09220_b200 as tf

pytestmark = pytest.mark.gpu


def varying(pts):
    return 1.0 + pts[..., 0] + 2.0 * pts[..., 1]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("p", [9, 12, 16])
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
def test_high_order_bitwise(dev, p, kind):
    n = (5, 4)
    rs = RefSpace.cartesian(*n, p)
    sp = tf.FeSpace.cartesian(dev, n, p)
    assert (sp.element_dofs() == rs.element_dofs()).all()
    f = RefForm(rs, [(kind, "varying", 0.0)])
    pa = tf.pa_setup(sp, kind, varying)
    assert (pa.qdata() == f.qdata()).all()
    x = np.random.default_rng(p).uniform(-1, 1, sp.n_dofs)
    y = tf.Vector(dev, sp.n_dofs)
    tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, x), y)
    assert (y.numpy() == f.mult(x)).all(), rel(y.numpy(), f.mult(x))
    a = tf.BilinearForm(sp)
    (a.add_diffusion if kind == "diffusion" else a.add_mass)(varying)
    a.assemble()
    assert (a.diagonal_true().numpy() == f.diagonal()).all()


@pytest.mark.parametrize("p", [10, 13, 16])
def test_high_order_fma_and_steady_state(dev_fma, p):
    """FMA numerics on a mesh where each block runs many elements."""
    n = (40, 36)
    rs = RefSpace.cartesian(*n, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    sp = tf.FeSpace.cartesian(dev_fma, n, p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    x = np.random.default_rng(3).uniform(-1, 1, sp.n_dofs)
    y = tf.Vector(dev_fma, sp.n_dofs)
    a.mult_true(x, y)
    assert rel(y.numpy(), f.mult(x)) <= 1e-12


@pytest.mark.parametrize("p", [9, 12, 16])
def test_high_order_cg_iterations(dev_fma, p):
    n = 4
    rs = RefSpace.cartesian(n, n, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    rsys = RefSystem(f, "front")
    xr, itr, cr, _ = rsys.cg(1e-10, 5000, True)
    sp = tf.FeSpace.cartesian(dev_fma, (n, n), p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    op = tf.ConstrainedOperator(a, sp.essential_true_dofs())
    res = tf.cg_solve(op, rsys.rhs, 1e-10, 5000, op.diagonal())
    assert res.converged == cr and res.iterations == itr, (res.iterations, itr)
    assert np.abs(res.x.numpy() - xr).max() <= 1e-8 * np.abs(xr).max()


@pytest.mark.parametrize("m", [4, 6, 8])
@pytest.mark.parametrize("p", [2, 5])
def test_curved_geometry_high_order_bitwise(dev, m, p):
    """curve_mesh of order m >= 4 (the device took m <= 3 in round 1)."""
    rs = RefSpace.curved(3, p, m)
    sp = tf.FeSpace.from_mesh(dev, 2, p, rs.element_dofs(), rs.n_dofs, rs.ctrl_points(), m)
    for kind in ("diffusion", "mass"):
        f = RefForm(rs, [(kind, "varying", 0.0)])
        pa = tf.pa_setup(sp, kind, varying)
        assert (pa.qdata() == f.qdata()).all()
        x = np.random.default_rng(m).uniform(-1, 1, sp.n_dofs)
        y = tf.Vector(dev, sp.n_dofs)
        tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, x), y)
        assert (y.numpy() == f.mult(x)).all()


def test_3d_order_cap_is_an_error(dev):
    with pytest.raises(tf.InvalidArgument):
        tf.FeSpace.cartesian(dev, (2, 2, 2), 9)
