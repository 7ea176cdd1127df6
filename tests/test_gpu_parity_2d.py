"""GPU parity, 2D: the sm_100a path through the C ABI against the unmodified
reference (oracle/_ref/libtfem_ref.so) on the same inputs.

Bar (BASELINE.json north_star): operator action within 1e-12 relative; in the
default TFEM_NUMERICS_REFERENCE mode the 2D device path evaluates the
reference's exact operation order, so these tests demand bit equality
(`==`), and CG iteration counts identical at a fixed tolerance.
"""
import numpy as np
import pytest

from oracle.pyoracle import Ref, RefForm, RefSpace, RefSystem, OrcCartesian
import paper_1911_09220_b200 as tf

pytestmark = pytest.mark.gpu

ORDERS = [1, 2, 3, 4, 5, 6, 7, 8]


def rng_vec(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def varying(pts):
    # 1 + x + 2y (test_forms.cpp:31), evaluated in the reference's order
    return 1.0 + pts[..., 0] + 2.0 * pts[..., 1]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("p", ORDERS)
@pytest.mark.parametrize("n", [(1, 1), (3, 2), (8, 8)])
def test_layout_matches_reference(dev, p, n):
    rs = RefSpace.cartesian(n[0], n[1], p)
    sp = tf.FeSpace.cartesian(dev, n, p)
    assert sp.n_dofs == rs.n_dofs
    assert (sp.element_dofs() == rs.element_dofs()).all()
    assert (sp.essential_true_dofs() == rs.essential()).all()


@pytest.mark.parametrize("p", ORDERS)
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
@pytest.mark.parametrize("coeff", ["const", "varying"])
def test_qdata_bitwise(dev, p, kind, coeff):
    rs = RefSpace.cartesian(5, 4, p, 2.0, 1.0)
    sp = tf.FeSpace.cartesian(dev, (5, 4), p, extents=(2.0, 1.0))
    f = RefForm(rs, [(kind, coeff, 1.0)])
    pa = tf.pa_setup(sp, kind, 1.0 if coeff == "const" else varying)
    assert pa.stored_reals() == f.stored_reals()
    assert (pa.qdata() == f.qdata()).all()
    B, G = pa.b1d(), pa.g1d()
    Br, Gr = Ref.eval_matrices(p, p + 2)
    assert (B == Br).all() and (G == Gr).all()


@pytest.mark.parametrize("p", ORDERS)
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
def test_apply_bitwise(dev, p, kind):
    n = (7, 6)
    rs = RefSpace.cartesian(*n, p)
    sp = tf.FeSpace.cartesian(dev, n, p)
    f = RefForm(rs, [(kind, "varying", 0.0)])
    pa = tf.pa_setup(sp, kind, varying)
    for trial in range(3):
        x = rng_vec(sp.n_dofs, 100 * p + trial)
        yr = f.mult(x)
        y = tf.Vector(dev, sp.n_dofs)
        tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, x), y)
        assert (y.numpy() == yr).all(), rel(y.numpy(), yr)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6])
def test_apply_local_accumulates(dev, p):
    """pa_apply_local is y += ... (forms.hpp:70-71)."""
    sp = tf.FeSpace.cartesian(dev, (4, 5), p)
    rs = RefSpace.cartesian(4, 5, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    pa = tf.pa_setup(sp, "diffusion", 1.0)
    x = rng_vec(sp.n_dofs, 7)
    y0 = rng_vec(sp.n_dofs, 8)
    y = tf.Vector.from_numpy(dev, y0)
    tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, x), y)
    want = y0 + f.mult(x)
    assert np.abs(y.numpy() - want).max() <= 1e-13 * np.abs(want).max()


@pytest.mark.parametrize("p", ORDERS)
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
def test_diagonal_bitwise(dev, p, kind):
    rs = RefSpace.cartesian(6, 5, p)
    sp = tf.FeSpace.cartesian(dev, (6, 5), p)
    f = RefForm(rs, [(kind, "varying", 0.0)])
    a = tf.BilinearForm(sp)
    (a.add_diffusion if kind == "diffusion" else a.add_mass)(varying)
    a.assemble()
    assert (a.diagonal_true().numpy() == f.diagonal()).all()


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_two_integrators_bitwise(dev, p):
    """Diffusion then mass accumulate into one L-vector (forms.cpp:539-541)."""
    rs = RefSpace.cartesian(6, 6, p)
    sp = tf.FeSpace.cartesian(dev, (6, 6), p)
    f = RefForm(rs, [("diffusion", "varying", 0.0), ("mass", "const", 3.0)])
    a = tf.BilinearForm(sp)
    a.add_diffusion(varying)
    a.add_mass(3.0)
    a.assemble()
    x = rng_vec(sp.n_dofs, 11)
    y = tf.Vector(dev, sp.n_dofs)
    a.mult_true(x, y)
    assert (y.numpy() == f.mult(x)).all()
    assert (a.diagonal_true().numpy() == f.diagonal()).all()
    assert a.stored_reals() == f.stored_reals()


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
def test_curved_geometry_bitwise(dev, p, kind):
    """Order-2 curved mesh (acceptance_main.cpp:52-57, criterion 1 fixture)."""
    rs = RefSpace.curved(4, p, 2)
    sp = tf.FeSpace.from_mesh(dev, 2, p, rs.element_dofs(), rs.n_dofs, rs.ctrl_points(), 2)
    f = RefForm(rs, [(kind, "varying", 0.0)])
    pa = tf.pa_setup(sp, kind, varying)
    assert (pa.qdata() == f.qdata()).all()
    x = rng_vec(sp.n_dofs, 5 * p)
    y = tf.Vector(dev, sp.n_dofs)
    tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, x), y)
    assert (y.numpy() == f.mult(x)).all()


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_constrained_operator_bitwise(dev, p):
    rs = RefSpace.cartesian(8, 8, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    rsys = RefSystem(f, "front")
    sp = tf.FeSpace.cartesian(dev, (8, 8), p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    ess = sp.essential_true_dofs()
    assert (ess == rsys.ess).all()
    op = tf.ConstrainedOperator(a, ess)
    x = rng_vec(sp.n_dofs, 3)
    y = tf.Vector(dev, sp.n_dofs)
    op.mult(x, y)
    assert (y.numpy() == rsys.op_mult(x)).all()
    d = op.diagonal().numpy()
    assert (d == rsys.diag).all()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6])
def test_constrained_two_integrators_bitwise(dev, p):
    """Essential DOFs with two integrators: the first gathers with the mask
    and leaves y[ess] alone, the last sets y[ess] = x[ess] (the per-position
    essential words of the element kernels with mask_in != ess_out)."""
    rs = RefSpace.cartesian(8, 7, p)
    f = RefForm(rs, [("diffusion", "varying", 0.0), ("mass", "const", 2.0)])
    rsys = RefSystem(f, "front")
    sp = tf.FeSpace.cartesian(dev, (8, 7), p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(varying)
    a.add_mass(2.0)
    a.assemble()
    op = tf.ConstrainedOperator(a, sp.essential_true_dofs())
    x = rng_vec(sp.n_dofs, 13 + p)
    y = tf.Vector(dev, sp.n_dofs)
    op.mult(x, y)
    assert (y.numpy() == rsys.op_mult(x)).all()
    assert (op.diagonal().numpy() == rsys.diag).all()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6])
@pytest.mark.parametrize("jacobi", [True, False])
def test_cg_front_iterations_match(dev, p, jacobi):
    """Driver system (front solution, tol 1e-12): same iteration count as the
    reference cg_solve, solutions equal to round-off."""
    n = 16
    rs = RefSpace.cartesian(n, n, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    rsys = RefSystem(f, "front")
    xr, itr, cr, _ = rsys.cg(1e-12, 2000, jacobi)
    sp = tf.FeSpace.cartesian(dev, (n, n), p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    op = tf.ConstrainedOperator(a, sp.essential_true_dofs())
    res = tf.cg_solve(op, rsys.rhs, 1e-12, 2000, op.diagonal() if jacobi else None)
    assert res.converged == cr
    assert res.iterations == itr
    x = res.x.numpy()
    assert np.abs(x - xr).max() <= 1e-10 * np.abs(xr).max()
    assert rsys.l2_error(x) == pytest.approx(rsys.l2_error(xr), rel=1e-6)


def test_cg_best_iterate_on_exhaustion(dev):
    """Non-convergence returns the best iterate after exactly max_iters
    (test_linalg.cpp:283-304), on the tridiagonal system of that test."""
    n = 50
    rows, cols, vals = [0], [], []
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                cols.append(j)
                vals.append(v)
        rows.append(len(cols))
    rp, cc, vv = np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals)
    b = np.ones(n)
    from oracle.pyoracle import ref_cg_csr
    xr, itr, cr = ref_cg_csr(rp, cc, vv, b, 1e-14, 24)
    op = tf.SparseOperator(dev, rp, cc, vv)
    res = tf.cg_solve(op, b, 1e-14, 24)
    assert not res.converged and res.iterations == 24 == itr and not cr
    assert np.abs(res.x.numpy() - xr).max() <= 1e-12
    A = np.zeros((n, n))
    for i in range(n):
        A[i, cc[rp[i]:rp[i + 1]]] = vv[rp[i]:rp[i + 1]]
    assert np.linalg.norm(b - A @ res.x.numpy()) < 0.5 * np.linalg.norm(b)


def test_cg_errors(dev):
    rp = np.array([0, 1, 2], np.int32)
    cc = np.array([0, 1], np.int32)
    op = tf.SparseOperator(dev, rp, cc, np.array([1.0, 1.0]))
    with pytest.raises(tf.InvalidArgument, match="strictly positive"):
        tf.cg_solve(op, np.ones(2), 1e-12, 10, np.zeros(2))
    with pytest.raises(tf.InvalidArgument):
        tf.cg_solve(op, np.ones(3), 1e-12, 10)
    nan_op = tf.SparseOperator(dev, rp, cc, np.array([np.nan, 0.0]))
    with pytest.raises(tf.TfemRuntimeError, match="breakdown"):
        tf.cg_solve(nan_op, np.ones(2), 1e-12, 10)
    res = tf.cg_solve(op, np.zeros(2), 1e-12, 10)
    assert res.converged and res.iterations == 0


def test_cg_on_iterate_callback(dev):
    sp = tf.FeSpace.cartesian(dev, (6, 6), 2)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    op = tf.ConstrainedOperator(a, sp.essential_true_dofs())
    b = rng_vec(sp.n_dofs, 1)
    b[sp.essential_true_dofs()] = 0.0
    seen = []
    res = tf.cg_solve(op, b, 1e-10, 500, on_iterate=lambda it, x: seen.append((it, x)))
    assert [s[0] for s in seen] == list(range(1, res.iterations + 1))
    assert np.array_equal(seen[-1][1], res.x.numpy())


def test_cg_profile_matches_solve(dev_fma):
    """tfem_cg_profile (eager, events between launches) computes the same
    iterates as the graph-replayed solve, and reports positive segment times."""
    import ctypes as C
    sp = tf.FeSpace.cartesian(dev_fma, (40, 40), 3)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    op = tf.ConstrainedOperator(a, sp.essential_true_dofs())
    b = rng_vec(sp.n_dofs, 3)
    b[sp.essential_true_dofs()] = 0.0
    d = op.diagonal()
    res = tf.cg_solve(op, b, 0.0, 37, d)
    bv = tf.Vector.from_numpy(dev_fma, b)
    xv = tf.Vector(dev_fma, sp.n_dofs)
    seg = (C.c_double * 3)()
    tf.abi.check(tf.lib().tfem_cg_profile(dev_fma.h, op.h, bv.h, 37, d.h, xv.h, seg))
    assert np.array_equal(xv.numpy(), res.x.numpy())
    assert all(v > 0.0 for v in seg)


def test_setup_errors_match_reference(dev):
    sp = tf.FeSpace.cartesian(dev, (2, 2), 1)
    with pytest.raises(tf.InvalidArgument, match="coefficient must be positive"):
        tf.pa_setup(sp, "diffusion", 0.0)
    with pytest.raises(tf.InvalidArgument, match="coefficient must be positive"):
        tf.pa_setup(sp, "mass", lambda p: p[..., 0] - 0.5)
    # inverted element: swap two corners of element 0
    rs = RefSpace.cartesian(2, 2, 1)
    ctrl = rs.ctrl_points()
    ctrl[1, [0, 1]] = ctrl[1, [1, 0]]
    bad = tf.FeSpace.from_mesh(dev, 2, 1, rs.element_dofs(), rs.n_dofs, ctrl, 1)
    with pytest.raises(tf.TfemRuntimeError, match="inverted element 1"):
        tf.pa_setup(bad, "diffusion", 1.0)


def test_lifecycle_errors(dev):
    sp = tf.FeSpace.cartesian(dev, (2, 2), 1)
    a = tf.BilinearForm(sp)
    x = tf.Vector(dev, sp.n_dofs)
    y = tf.Vector(dev, sp.n_dofs)
    with pytest.raises(tf.LogicError):
        a.mult_true(x, y)
    a.add_diffusion(1.0)
    with pytest.raises(tf.InvalidArgument):
        a.assemble(0)
    a.assemble()
    with pytest.raises(tf.LogicError):
        a.assemble()
    with pytest.raises(tf.LogicError):
        a.add_mass(1.0)
    with pytest.raises(tf.InvalidArgument):
        a.mult_true(tf.Vector(dev, 3), y)


def test_multiply_count_and_storage(dev):
    """test_forms.cpp:374-412 contracts."""
    for p in (1, 2, 3):
        sp = tf.FeSpace.cartesian(dev, (1, 1), p)
        a = tf.BilinearForm(sp)
        a.add_diffusion(1.0)
        a.assemble()
        x = tf.Vector.from_numpy(dev, rng_vec(sp.n_dofs, 5))
        y = tf.Vector(dev, sp.n_dofs)
        tf.reset_multiply_count()
        a.mult_true(x, y)
        nd, nq = p + 1, p + 2
        assert tf.multiply_count() == 4 * (nq * nd * nd + nq * nq * nd) + 4 * nq * nq
        rs = RefSpace.cartesian(1, 1, p)
        _, cnt = RefForm(rs, [("diffusion", "const", 1.0)]).mult_count(x.numpy())
        assert cnt == tf.multiply_count()
        sp2 = tf.FeSpace.cartesian(dev, (2, 2), p)
        a2 = tf.BilinearForm(sp2)
        a2.add_diffusion(1.0)
        a2.assemble()
        assert a2.stored_reals() == 4 * 3 * nq * nq


@pytest.mark.parametrize("p", ORDERS)
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
def test_fma_numerics_within_tolerance(dev_fma, p, kind):
    """Default numerics (TFEM_NUMERICS_FMA): operator action and diagonal
    within the north-star 1e-12 relative of the reference."""
    rs = RefSpace.cartesian(9, 7, p)
    f = RefForm(rs, [(kind, "varying", 0.0)])
    sp = tf.FeSpace.cartesian(dev_fma, (9, 7), p)
    pa = tf.pa_setup(sp, kind, varying)
    x = rng_vec(sp.n_dofs, 9 + p)
    y = tf.Vector(dev_fma, sp.n_dofs)
    tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev_fma, x), y)
    assert rel(y.numpy(), f.mult(x)) <= 1e-12
    assert rel(tf.pa_diagonal(pa, sp).numpy(), f.diagonal()) <= 1e-12


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6])
@pytest.mark.parametrize("jacobi", [True, False])
def test_fma_numerics_cg_iterations_match(dev_fma, p, jacobi):
    """Default numerics: identical CG iteration counts to the reference at
    tol 1e-12 on the driver's front system."""
    n = 16
    rs = RefSpace.cartesian(n, n, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    rsys = RefSystem(f, "front")
    xr, itr, cr, _ = rsys.cg(1e-12, 2000, jacobi)
    sp = tf.FeSpace.cartesian(dev_fma, (n, n), p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    op = tf.ConstrainedOperator(a, sp.essential_true_dofs())
    res = tf.cg_solve(op, rsys.rhs, 1e-12, 2000, op.diagonal() if jacobi else None)
    assert res.converged == cr and res.iterations == itr
    assert np.abs(res.x.numpy() - xr).max() <= 1e-10 * np.abs(xr).max()


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_bp5_gll_collocated_bitwise_vs_restatement(dev, p):
    """q = p+1 Gauss-Lobatto (BP5) -- not expressible in the reference API;
    checked against the C restatement, itself bit-equal to the reference on
    every rule it can express."""
    n = (6, 5)
    oc = OrcCartesian(2, n, p, rule="gll")
    sp = tf.FeSpace.cartesian(dev, n, p)
    pa = tf.pa_setup(sp, "diffusion", 1.0, rule="gauss_lobatto")
    qd = oc.setup("diffusion")
    assert (pa.qdata() == qd).all()
    x = rng_vec(sp.n_dofs, 2)
    y = tf.Vector(dev, sp.n_dofs)
    tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, x), y)
    assert (y.numpy() == oc.apply("diffusion", qd, x)).all()


def test_restriction_roundtrip(dev):
    """ElementRestriction Mult / MultTranspose against the reference map."""
    p = 3
    rs = RefSpace.cartesian(5, 4, p)
    sp = tf.FeSpace.cartesian(dev, (5, 4), p)
    dofs = rs.element_dofs()
    x = rng_vec(sp.n_dofs, 4)
    e = sp.restrict(tf.Vector.from_numpy(dev, x)).numpy().reshape(dofs.shape)
    assert (e == x[dofs]).all()
    ev = rng_vec(dofs.size, 5)
    y = tf.Vector(dev, sp.n_dofs)
    sp.restrict_transpose(tf.Vector.from_numpy(dev, ev), y)
    want = np.zeros(sp.n_dofs)
    for k in range(dofs.shape[0]):           # element order, forms.cpp:289-295
        for i in range(dofs.shape[1]):
            want[dofs[k, i]] += ev[k * dofs.shape[1] + i]
    assert (y.numpy() == want).all()


def test_full_size_bp3_bitwise(dev):
    """BASELINE configs[1] size (make_cartesian(1054, 1054), p = 3,
    10,004,569 DOFs): device qdata, operator action and diagonal equal the C
    restatement (itself bit-equal to the reference) bit for bit."""
    n, p = (1054, 1054), 3
    sp = tf.FeSpace.cartesian(dev, n, p)
    assert sp.n_dofs == 10_004_569
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    x = rng_vec(sp.n_dofs, 42)
    y = tf.Vector(dev, sp.n_dofs)
    a.mult_true(x, y)
    oc = OrcCartesian(2, n, p)
    qd = oc.setup("diffusion")
    assert (a.pa_data()[0].qdata() == qd).all()
    assert (y.numpy() == oc.apply("diffusion", qd, x)).all()
    assert (a.diagonal_true().numpy() == oc.diagonal("diffusion", qd)).all()


def test_full_size_properties(dev):
    """Size-independent checks at full size: constants annihilated, symmetry,
    mass integrates the area, repeated applications bit-identical."""
    n, p = (1054, 1054), 3
    sp = tf.FeSpace.cartesian(dev, n, p, extents=(2.0, 0.5))
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    y = tf.Vector(dev, sp.n_dofs)
    a.mult_true(tf.Vector(dev, sp.n_dofs, 1.0), y)
    assert np.abs(y.numpy()).max() <= 1e-11
    x1, x2 = rng_vec(sp.n_dofs, 1), rng_vec(sp.n_dofs, 2)
    y1, y2 = tf.Vector(dev, sp.n_dofs), tf.Vector(dev, sp.n_dofs)
    a.mult_true(x1, y1)
    a.mult_true(x2, y2)
    assert x2 @ y1.numpy() == pytest.approx(x1 @ y2.numpy(), rel=1e-11)
    first = y1.numpy()
    a.mult_true(x1, y1)
    assert (y1.numpy() == first).all()
    m = tf.BilinearForm(sp)
    m.add_mass(1.0)
    m.assemble()
    m.mult_true(tf.Vector(dev, sp.n_dofs, 1.0), y)
    assert y.numpy().sum() == pytest.approx(1.0, rel=1e-12)


def test_fp64_peak_probe(dev):
    # diagnostics behind bench.py's FP64 roofline: the DFMA peak of a B200 is
    # ~37 TFLOP/s nominal; the probe must land in a physically sensible range
    import ctypes as C
    v = C.c_double(0.0)
    tf.abi.check(tf.lib().tfem_fp64_peak(dev.h, C.byref(v)))
    assert 5.0 < v.value < 100.0, v.value
