"""GPU parity of LinearForm (forms.cpp:400-431): the
driver's manufactured sources, evaluated by the reference's own functions at
the device-computed points, integrated and scattered on the device --
bit-identical to the reference's b on Cartesian, curved and forest spaces."""
import numpy as np
import pytest

from oracle.pyoracle import RefSpace, ref_solution_f
import paper_1911_09220_b200 as tf

pytestmark = pytest.mark.gpu


def src(solution):
    return lambda pts: ref_solution_f(solution, pts)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("solution", ["front", "sine"])
def test_linear_form_cartesian_bitwise(dev, p, solution):
    rs = RefSpace.cartesian(5, 4, p, 2.0, 1.0)
    sp = tf.FeSpace.cartesian(dev, (5, 4), p, extents=(2.0, 1.0))
    b = tf.LinearForm(sp, src(solution)).values().numpy()
    assert (b == rs.linear_form(solution)).all()


@pytest.mark.parametrize("p", [1, 3])
def test_linear_form_curved_and_forest_bitwise(dev, p):
    rs = RefSpace.curved(4, p)
    sp = tf.FeSpace.from_mesh(dev, 2, p, rs.element_dofs(), rs.n_dofs, rs.ctrl_points(),
                              rs.geom_order)
    assert (tf.LinearForm(sp, src("front")).values().numpy() == rs.linear_form("front")).all()
    rs = RefSpace.random_forest(4, p, 6, 3)
    rp, cols, vals = rs.prolongation()
    sp = tf.FeSpace.from_mesh(dev, 2, p, rs.element_dofs(), rs.n_dofs, rs.ctrl_points(),
                              rs.geom_order,
                              prolongation=(rp, cols, vals, rs.true_index(), rs.n_true))
    assert (tf.LinearForm(sp, src("front")).values().numpy() == rs.linear_form("front")).all()


def test_linear_form_errors(dev):
    sp = tf.FeSpace.cartesian(dev, (2, 2, 2), 1)
    with pytest.raises(tf.InvalidArgument, match="2D"):
        tf.LinearForm(sp, 1.0)
    sp2 = tf.FeSpace.cartesian(dev, (2, 2), 1)
    with pytest.raises(tf.InvalidArgument, match="empty"):
        tf.LinearForm(sp2, None)


def spaces(dev, p):
    """(reference space, device space) pairs: Cartesian, curved, forest."""
    out = [(RefSpace.cartesian(5, 4, p, 2.0, 1.0),
            tf.FeSpace.cartesian(dev, (5, 4), p, extents=(2.0, 1.0)))]
    rs = RefSpace.curved(4, p)
    out.append((rs, tf.FeSpace.from_mesh(dev, 2, p, rs.element_dofs(), rs.n_dofs,
                                         rs.ctrl_points(), rs.geom_order)))
    rs = RefSpace.random_forest(4, p, 6, 3)
    rp, cols, vals = rs.prolongation()
    out.append((rs, tf.FeSpace.from_mesh(dev, 2, p, rs.element_dofs(), rs.n_dofs,
                                         rs.ctrl_points(), rs.geom_order,
                                         prolongation=(rp, cols, vals, rs.true_index(),
                                                       rs.n_true))))
    return out


@pytest.mark.parametrize("p", [1, 2, 3, 5])
@pytest.mark.parametrize("solution", ["front", "sine"])
def test_project_and_l2_error_bitwise(dev, p, solution):
    """project_coefficient and compute_l2_error (fespace.cpp:334-394)."""
    from oracle.pyoracle import ref_solution_u
    u = lambda pts: ref_solution_u(solution, pts)
    for rs, sp in spaces(dev, p):
        g = tf.project_coefficient(sp, u).numpy()
        assert (g == rs.project(solution)).all()
        assert tf.compute_l2_error(sp, g, u) == rs.l2_error(g, solution)
        x = np.random.default_rng(p).uniform(-1, 1, rs.n_dofs)
        assert tf.compute_l2_error(sp, x, u) == rs.l2_error(x, solution)
