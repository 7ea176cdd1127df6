"""CPU: pin the 3D / BP5 restatement (no reference oracle exists for them,
SURVEY.md 0.3) with the checks SURVEY.md 7 lists: analytic element-matrix
KATs, PA action == dense element matrices, constants annihilated, volume,
symmetry, a polynomial patch test through CG, and the 2D restatement's own
reference pinning for every rule it shares (test_oracle_ref.py)."""
import numpy as np
import pytest

from oracle.pyoracle import Orc, OrcCartesian

pytestmark = pytest.mark.usefixtures("oracle_built")


def kron3(a, b, c):
    # lattice index i = a + D1 (b + D1 c): x fastest -> kron(z, y, x)
    return np.kron(c, np.kron(b, a))


def test_unit_cube_trilinear_kats():
    """q = p+2 Gauss integrates the p = 1 matrices exactly:
    M = Mz (x) My (x) Mx, K = Kx-terms with the 1D [[1,-1],[-1,1]] stiffness."""
    oc = OrcCartesian(3, (1, 1, 1), 1)
    m1 = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    k1 = np.array([[1.0, -1.0], [-1.0, 1.0]])
    qm = oc.setup("mass")
    qk = oc.setup("diffusion")
    M = oc.element_matrix("mass", qm[0])
    K = oc.element_matrix("diffusion", qk[0])
    assert np.abs(M - kron3(m1, m1, m1)).max() <= 1e-15
    want = kron3(k1, m1, m1) + kron3(m1, k1, m1) + kron3(m1, m1, k1)
    assert np.abs(K - want).max() <= 1e-14


def test_stretched_box_scaling():
    """J = diag(2, 1, 0.5): mass scales by det J = 1, diffusion terms by
    det J / J_ii^2 (the 3D analogue of test_forms.cpp:193-199)."""
    oc = OrcCartesian(3, (1, 1, 1), 1, ext=[2.0, 1.0, 0.5])
    m1 = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    k1 = np.array([[1.0, -1.0], [-1.0, 1.0]])
    K = oc.element_matrix("diffusion", oc.setup("diffusion")[0])
    want = (0.25 * kron3(k1, m1, m1) + kron3(m1, k1, m1) + 4.0 * kron3(m1, m1, k1))
    assert np.abs(K - want).max() <= 1e-14
    qd = oc.setup("diffusion")
    assert np.abs(qd[..., [1, 2, 4]]).max() <= 1e-16  # off-diagonal factors vanish


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("kind", ["diffusion", "mass"])
@pytest.mark.parametrize("rule", ["gl", "gll"])
def test_pa_equals_dense_element_matrices(p, kind, rule):
    # p >= 5: fewer elements keep the dense (p+1)^6 q^3 element matrices
    # affordable (two elements -- one shared face -- up to p = 6, one above)
    n = (3, 2, 2) if p <= 4 else ((2, 1, 1) if p <= 6 else (1, 1, 1))
    oc = OrcCartesian(3, n, p, rule=rule, ext=[1.0, 0.7, 1.3])
    pts = oc.points()
    coeff = 1.0 + pts[..., 0] + 2.0 * pts[..., 1] + 3.0 * pts[..., 2]
    qd = oc.setup(kind, coeff=coeff)
    x = np.random.default_rng(p).uniform(-1, 1, oc.ndofs)
    y = oc.apply(kind, qd, x)
    want = np.zeros(oc.ndofs)
    wd = np.zeros(oc.ndofs)
    for e in range(oc.ne):
        d = oc.elem_dofs[e]
        K = oc.element_matrix(kind, qd[e])
        want[d] += K @ x[d]
        wd[d] += np.diag(K)
    assert np.abs(y - want).max() <= 1e-13 * np.abs(want).max()
    # diagonal of the assembled operator
    dg = oc.diagonal(kind, qd)
    assert np.abs(dg - wd).max() <= 1e-13 * np.abs(wd).max()


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_constants_and_volume(p):
    ext = [2.0, 1.0, 0.5]
    oc = OrcCartesian(3, (2, 3, 2), p, ext=ext)
    ones = np.ones(oc.ndofs)
    y = oc.apply("diffusion", oc.setup("diffusion"), ones)
    scale = np.abs(oc.diagonal("diffusion", oc.setup("diffusion"))).max()
    assert np.abs(y).max() <= 1e-12 * scale
    m = oc.apply("mass", oc.setup("mass"), ones)
    assert m.sum() == pytest.approx(np.prod(ext), rel=1e-13)


@pytest.mark.parametrize("p", [2, 3])
def test_symmetry(p):
    oc = OrcCartesian(3, (2, 2, 3), p)
    qd = oc.setup("diffusion")
    rng = np.random.default_rng(3)
    x, z = rng.uniform(-1, 1, (2, oc.ndofs))
    a = z @ oc.apply("diffusion", qd, x)
    b = x @ oc.apply("diffusion", qd, z)
    assert a == pytest.approx(b, rel=1e-13)


def dof_coordinates(oc):
    """Physical coordinates of every DOF (GLL lattice of each element)."""
    p = oc.p
    nodes, _ = Orc.rule(p + 1, lobatto=True)
    X = np.zeros((oc.ndofs, 3))
    nx, ny, nz = oc.n
    for e in range(oc.ne):
        i, j, k = e % nx, (e // nx) % ny, e // (nx * ny)
        for l, d in enumerate(oc.elem_dofs[e]):
            a, b, c = l % (p + 1), (l // (p + 1)) % (p + 1), l // (p + 1) ** 2
            X[d] = [(i + nodes[a]) / nx * oc.ext[0], (j + nodes[b]) / ny * oc.ext[1],
                    (k + nodes[c]) / nz * oc.ext[2]]
    return X


@pytest.mark.parametrize("p", [1, 2, 3])
def test_patch_test_through_cg(p):
    """A linear field is reproduced to 1e-10 by Jacobi-CG on the constrained
    system (the 3D analogue of test_forms.cpp:537-581)."""
    oc = OrcCartesian(3, (3, 2, 2), p)
    X = dof_coordinates(oc)
    u = 1.0 + X[:, 0] + 2.0 * X[:, 1] - 0.5 * X[:, 2]
    ess = oc.boundary_dofs()
    qd = oc.setup("diffusion")
    x0 = np.zeros(oc.ndofs)
    x0[ess] = u[ess]
    plain = oc.operator(["diffusion"], [qd])
    rhs = -oc.op_mult(plain, x0)
    rhs[ess] = 0.0
    op = oc.operator(["diffusion"], [qd], ess)
    d = oc.diagonal("diffusion", qd)
    d[ess] = 1.0
    x, it, conv = oc.cg(op, rhs, 1e-14, 2000, d)
    assert conv
    assert np.abs(x + x0 - u).max() <= 1e-10


def test_layout_is_conforming_3d():
    """Shared lattice points get one DOF: count = (n p + 1)^3 and every DOF
    is reached from an element."""
    for p in (1, 2, 3, 4):
        n = (3, 2, 4)
        oc = OrcCartesian(3, n, p)
        assert oc.ndofs == np.prod([k * p + 1 for k in n])
        assert len(np.unique(oc.elem_dofs)) == oc.ndofs
        # neighbouring elements agree on the coordinates of shared DOFs
        X = dof_coordinates(oc)
        p1 = p + 1
        nodes, _ = Orc.rule(p + 1, lobatto=True)
        for e in range(oc.ne):
            i, j, k = e % n[0], (e // n[0]) % n[1], e // (n[0] * n[1])
            for l, dd in enumerate(oc.elem_dofs[e]):
                a, b, c = l % p1, (l // p1) % p1, l // p1 ** 2
                want = [(i + nodes[a]) / n[0], (j + nodes[b]) / n[1], (k + nodes[c]) / n[2]]
                assert np.allclose(X[dd], want, atol=1e-15)


def test_gll_rule_collocation():
    """BP5: q = p+1 Gauss-Lobatto makes B1d the identity."""
    for p in range(1, 9):
        B, G = Orc.eval_matrices(p, p + 1, 0, 1)
        assert (B == np.eye(p + 1)).all()
        assert np.abs(G.sum(axis=1)).max() <= 1e-12 * np.abs(G).max()
