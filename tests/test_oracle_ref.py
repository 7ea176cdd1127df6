"""CPU: pin the C restatement (oracle/tfem_oracle.c) against the unmodified
reference built in place (oracle/_ref) -- bit equality on every 2D quantity
of the hot path: 1D rules, basis tables, DOF layout, essential DOFs,
quadrature data (straight and curved, constant and varying coefficient),
operator action, diagonal, constrained operator and full CG solves."""
import numpy as np
import pytest

from oracle.pyoracle import (Orc, OrcCartesian, Ref, RefForm, RefSpace, RefSystem,
                             orc_layout_quads)

pytestmark = pytest.mark.usefixtures("oracle_built")


def need_ref():
    if not Ref.available():
        pytest.skip("reference not built (no /root/reference here)")


def test_rules_and_tables():
    need_ref()
    for n in range(1, 13):
        for lob in (False, True):
            if lob and n < 2:
                continue
            a, b = Ref.rule(n, lob), Orc.rule(n, lob)
            assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    for p in range(1, 9):
        for nq in (p + 1, p + 2):
            for rk in (0, 1):
                for nk in (0, 1, 2):
                    a, b = Ref.eval_matrices(p, nq, nk, rk), Orc.eval_matrices(p, nq, nk, rk)
                    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()


@pytest.mark.parametrize("n", [(1, 1), (3, 2), (5, 7)])
@pytest.mark.parametrize("p", range(1, 9))
def test_layout_and_boundary(n, p):
    need_ref()
    rs = RefSpace.cartesian(*n, p)
    oc = OrcCartesian(2, n, p)
    assert oc.ndofs == rs.n_dofs
    assert (oc.elem_dofs == rs.element_dofs()).all()
    assert (oc.boundary_dofs() == rs.essential()).all()


def test_closed_form_layout_equals_discovery_layout():
    import ctypes as C
    for n in [(1, 1), (4, 3), (9, 2)]:
        for p in (1, 2, 5):
            oc = OrcCartesian(2, n, p)
            ev = np.zeros((oc.ne, 4), dtype=np.int32)
            Orc.lib().orc_cartesian_elements(2, oc.n.ctypes.data_as(C.POINTER(C.c_int)),
                                             ev.ctypes.data_as(C.POINTER(C.c_int)))
            d, nd = orc_layout_quads((n[0] + 1) * (n[1] + 1), ev, p)
            assert nd == oc.ndofs and (d == oc.elem_dofs).all()


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
@pytest.mark.parametrize("coeff", ["const", "varying"])
def test_setup_apply_diagonal_bitwise(p, kind, coeff):
    need_ref()
    n = (4, 3)
    rs = RefSpace.cartesian(*n, p, 2.0, 1.0)
    oc = OrcCartesian(2, n, p, ext=[2.0, 1.0])
    f = RefForm(rs, [(kind, coeff, 1.0)])
    cv = None
    if coeff == "varying":
        pts = oc.points()
        cv = 1.0 + pts[..., 0] + 2.0 * pts[..., 1]
    qo = oc.setup(kind, coeff=cv)
    assert (f.qdata() == qo).all()
    x = np.random.default_rng(p).uniform(-1, 1, rs.n_dofs)
    assert (f.mult(x) == oc.apply(kind, qo, x)).all()
    assert (f.diagonal() == oc.diagonal(kind, qo)).all()


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_curved_setup_bitwise(p):
    need_ref()
    rs = RefSpace.curved(4, p, 2)
    oc = OrcCartesian(2, (4, 4), p)
    for kind in ("diffusion", "mass"):
        f = RefForm(rs, [(kind, "const", 1.0)])
        assert (f.qdata() == oc.setup(kind, ctrl=rs.ctrl_points(), geom_order=2)).all()


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("jacobi", [True, False])
def test_constrained_operator_and_cg_bitwise(p, jacobi):
    need_ref()
    n = 8
    rs = RefSpace.cartesian(n, n, p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    rsys = RefSystem(f, "front")
    oc = OrcCartesian(2, (n, n), p)
    qd = oc.setup("diffusion")
    op = oc.operator(["diffusion"], [qd], rsys.ess)
    x = np.random.default_rng(1).uniform(-1, 1, rs.n_dofs)
    assert (oc.op_mult(op, x) == rsys.op_mult(x)).all()
    xr, itr, cr, _ = rsys.cg(1e-12, 2000, jacobi)
    xo, ito, co = oc.cg(op, rsys.rhs, 1e-12, 2000, rsys.diag if jacobi else None)
    assert (itr, cr) == (ito, co)
    assert (xr == xo).all()


def test_cg_exhaustion_returns_best_iterate():
    """test_linalg.cpp:283-304 on the restatement's CSR CG."""
    need_ref()
    from oracle.pyoracle import ref_cg_csr
    import ctypes as C
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
    xr, itr, cr = ref_cg_csr(rp, cc, vv, b, 1e-14, 24)
    x = np.zeros(n)
    it, conv = C.c_int(), C.c_int()
    from oracle.pyoracle import _d, _i
    Orc.check(Orc.lib().orc_cg_csr(n, _i(rp), _i(cc), _d(vv), _d(b), 1e-14, 24, None, _d(x),
                                   C.byref(it), C.byref(conv)))
    assert it.value == itr == 24 and not conv.value and not cr
    assert (x == xr).all()


def test_error_paths_match_reference():
    need_ref()
    from oracle.pyoracle import OracleError
    rs = RefSpace.cartesian(2, 2, 1)
    with pytest.raises(OracleError, match="coefficient must be positive"):
        RefForm(rs, [("diffusion", "const", 0.0)])
    oc = OrcCartesian(2, (2, 2), 1)
    with pytest.raises(OracleError, match="coefficient must be positive"):
        oc.setup("diffusion", const=0.0)
    ctrl = oc.ctrl.copy()
    ctrl[1, [0, 1]] = ctrl[1, [1, 0]]
    with pytest.raises(OracleError, match="inverted element 1"):
        oc.setup("diffusion", ctrl=ctrl)
