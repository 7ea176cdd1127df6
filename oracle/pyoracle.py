"""ORACLE INFRASTRUCTURE -- ctypes wrappers for the two CPU checkers.

* ``Ref``: the unmodified reference library (oracle/_ref/libtfem_ref.so,
  built from /root/reference/proj/src by oracle/Makefile) behind
  oracle/ref_shim.cpp.
* ``Orc``: the C restatement (oracle/liboracle.so, oracle/tfem_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline / reference
legs may import this module.  It is never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libtfem_ref.so"
ORC_SO = HERE / "liboracle.so"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64 = C.c_int64


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_ip)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_EXC = {1: ValueError, 2: RuntimeError, 3: AssertionError}


def _raise(code, msg):
    kind = {1: "invalid_argument", 2: "runtime_error", 3: "logic_error"}.get(code, "error")
    e = OracleError(code, f"{kind}: {msg}")
    raise e


def build():
    """Builds liboracle.so (and _ref when the reference tree is present)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)


# --------------------------------------------------------------- reference
class Ref:
    """The reference tensorfem library (2D quads only)."""

    _lib = None

    @classmethod
    def available(cls):
        return REF_SO.exists()

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not REF_SO.exists():
                raise FileNotFoundError(f"{REF_SO} missing: run make -C oracle ref")
            L = C.CDLL(str(REF_SO))
            L.ref_last_error.restype = C.c_char_p
            for n in ("ref_space_cartesian", "ref_space_curved", "ref_space_random_forest",
                      "ref_form_create", "ref_system_create"):
                getattr(L, n).restype = C.c_void_p
            L.ref_space_cartesian.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double]
            L.ref_space_curved.argtypes = [C.c_int, C.c_int, C.c_int]
            L.ref_space_random_forest.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint]
            L.ref_space_free.argtypes = [C.c_void_p]
            L.ref_space_info.argtypes = [C.c_void_p] + [_ip] * 6
            L.ref_space_element_dofs.argtypes = [C.c_void_p, _ip]
            L.ref_space_true_index.argtypes = [C.c_void_p, _ip]
            L.ref_space_essential.argtypes = [C.c_void_p, _ip, _ip]
            L.ref_space_prolongation.argtypes = [C.c_void_p, _ip, _ip, _dp, C.POINTER(C.c_longlong)]
            L.ref_space_element_vertices.argtypes = [C.c_void_p, _dp]
            L.ref_space_geometry_nodes.argtypes = [C.c_void_p, _dp]
            L.ref_form_create.argtypes = [C.c_void_p, C.c_int, C.c_int, _ip, _ip, _dp, C.c_int]
            L.ref_form_free.argtypes = [C.c_void_p]
            L.ref_form_mult.argtypes = [C.c_void_p, _dp, _dp]
            L.ref_form_mult_count.argtypes = [C.c_void_p, _dp, _dp, C.POINTER(C.c_ulonglong)]
            L.ref_form_diag.argtypes = [C.c_void_p, _dp]
            L.ref_form_stored_reals.argtypes = [C.c_void_p]
            L.ref_form_stored_reals.restype = C.c_longlong
            L.ref_form_qdata.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _ip]
            L.ref_form_matrix.argtypes = [C.c_void_p, _ip, _ip, _dp, C.POINTER(C.c_longlong)]
            L.ref_pa_setup.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double]
            L.ref_system_create.argtypes = [C.c_void_p, C.c_int]
            L.ref_system_free.argtypes = [C.c_void_p]
            L.ref_system_vectors.argtypes = [C.c_void_p, _dp, _dp, _dp]
            L.ref_system_ess.argtypes = [C.c_void_p, _ip]
            L.ref_system_op_mult.argtypes = [C.c_void_p, _dp, _dp]
            L.ref_system_cg.argtypes = [C.c_void_p, _dp, C.c_double, C.c_int, C.c_int, _dp,
                                        _ip, _ip, _dp]
            L.ref_system_l2_error.argtypes = [C.c_void_p, _dp, _dp]
            L.ref_solve_poisson.argtypes = [C.c_int] * 4 + [C.c_double, C.c_int, C.c_int, _ip,
                                                            _ip, _dp, _dp,
                                                            C.POINTER(C.c_longlong)]
            L.ref_cg_csr.argtypes = [C.c_int, _ip, _ip, _dp, _dp, C.c_double, C.c_int, _dp,
                                     _dp, _ip, _ip]
            L.ref_linear_form.argtypes = [C.c_void_p, C.c_int, _dp]
            L.ref_project.argtypes = [C.c_void_p, C.c_int, _dp]
            L.ref_l2_error.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
            L.ref_solution_u.argtypes = [C.c_int, _dp, C.c_int, _dp]
            L.ref_solution_f.argtypes = [C.c_int, _dp, C.c_int, _dp]
            L.ref_gauss_legendre.argtypes = [C.c_int, _dp, _dp]
            L.ref_gauss_lobatto.argtypes = [C.c_int, _dp, _dp]
            L.ref_eval_matrices.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp]
            cls._lib = L
        return cls._lib

    @classmethod
    def check(cls, rc):
        if rc != 0:
            _raise(rc, cls.lib().ref_last_error().decode())

    # 1D tables
    @classmethod
    def rule(cls, n, lobatto=False):
        p = np.zeros(n)
        w = np.zeros(n)
        fn = cls.lib().ref_gauss_lobatto if lobatto else cls.lib().ref_gauss_legendre
        cls.check(fn(n, _d(p), _d(w)))
        return p, w

    @classmethod
    def eval_matrices(cls, p, nq, node_kind=0, rule_kind=0):
        B = np.zeros((nq, p + 1))
        G = np.zeros((nq, p + 1))
        cls.check(cls.lib().ref_eval_matrices(p, node_kind, nq, rule_kind, _d(B), _d(G)))
        return B, G


class RefSpace:
    def __init__(self, handle):
        if not handle:
            raise OracleError(9, Ref.lib().ref_last_error().decode())
        self.h = C.c_void_p(handle)
        vals = [C.c_int() for _ in range(6)]
        Ref.lib().ref_space_info(self.h, *[C.byref(v) for v in vals])
        (self.n_dofs, self.n_true, self.n_elem, self.order, conf, self.geom_order) = [
            v.value for v in vals]
        self.conforming = bool(conf)

    @classmethod
    def cartesian(cls, nx, ny, p, w=1.0, h=1.0):
        return cls(Ref.lib().ref_space_cartesian(nx, ny, p, w, h))

    @classmethod
    def curved(cls, n, p, m=2):
        return cls(Ref.lib().ref_space_curved(n, p, m))

    @classmethod
    def random_forest(cls, n, p, count, seed):
        return cls(Ref.lib().ref_space_random_forest(n, p, count, seed))

    def __del__(self):
        try:
            Ref.lib().ref_space_free(self.h)
        except Exception:
            pass

    def element_dofs(self):
        nd = (self.order + 1) ** 2
        out = np.zeros((self.n_elem, nd), dtype=np.int32)
        Ref.lib().ref_space_element_dofs(self.h, _i(out))
        return out

    def true_index(self):
        out = np.zeros(self.n_dofs, dtype=np.int32)
        Ref.lib().ref_space_true_index(self.h, _i(out))
        return out

    def essential(self):
        cnt = C.c_int()
        Ref.check(Ref.lib().ref_space_essential(self.h, None, C.byref(cnt)))
        out = np.zeros(cnt.value, dtype=np.int32)
        Ref.check(Ref.lib().ref_space_essential(self.h, _i(out), C.byref(cnt)))
        return out

    def prolongation(self):
        nnz = C.c_longlong()
        Ref.check(Ref.lib().ref_space_prolongation(self.h, None, None, None, C.byref(nnz)))
        rp = np.zeros(self.n_dofs + 1, dtype=np.int32)
        cols = np.zeros(nnz.value, dtype=np.int32)
        vals = np.zeros(nnz.value)
        Ref.check(Ref.lib().ref_space_prolongation(self.h, _i(rp), _i(cols), _d(vals),
                                                   C.byref(nnz)))
        return rp, cols, vals

    def linear_form(self, solution="front"):
        out = np.zeros(self.n_dofs)
        Ref.check(Ref.lib().ref_linear_form(self.h, 0 if solution == "sine" else 1, _d(out)))
        return out

    def project(self, solution="front"):
        out = np.zeros(self.n_dofs)
        Ref.check(Ref.lib().ref_project(self.h, 0 if solution == "sine" else 1, _d(out)))
        return out

    def l2_error(self, x, solution="front"):
        err = C.c_double()
        Ref.check(Ref.lib().ref_l2_error(self.h, 0 if solution == "sine" else 1,
                                         _d(np.ascontiguousarray(x, dtype=np.float64)),
                                         C.byref(err)))
        return err.value

    def element_vertices(self):
        out = np.zeros((self.n_elem, 4, 2))
        Ref.lib().ref_space_element_vertices(self.h, _d(out))
        return out

    def ctrl_points(self):
        """Geometry control points in lattice order, E x (m+1)^2 x 2."""
        if self.geom_order == 1:
            v = self.element_vertices()
            return np.ascontiguousarray(v[:, [0, 1, 3, 2], :])
        n2 = (self.geom_order + 1) ** 2
        out = np.zeros((self.n_elem, n2, 2))
        Ref.check(Ref.lib().ref_space_geometry_nodes(self.h, _d(out)))
        return out


KIND = {"diffusion": 0, "mass": 1}
COEFF = {"const": 0, "varying": 1}


class RefForm:
    """BilinearForm with integrators [(kind, coeff_id, coeff_value)]."""

    def __init__(self, space: RefSpace, integrators, mode="partial", threads=1):
        self.space = space
        kinds = np.array([KIND[k] for k, _, _ in integrators], dtype=np.int32)
        cids = np.array([COEFF[c] for _, c, _ in integrators], dtype=np.int32)
        cvals = np.array([v for _, _, v in integrators], dtype=np.float64)
        h = Ref.lib().ref_form_create(space.h, 0 if mode == "full" else 1, len(integrators),
                                      _i(kinds), _i(cids), _d(cvals), threads)
        if not h:
            raise OracleError(9, Ref.lib().ref_last_error().decode())
        self.h = C.c_void_p(h)
        self.n = space.n_true
        self.integrators = integrators

    def __del__(self):
        try:
            Ref.lib().ref_form_free(self.h)
        except Exception:
            pass

    def mult(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        Ref.check(Ref.lib().ref_form_mult(self.h, _d(x), _d(y)))
        return y

    def mult_count(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        c = C.c_ulonglong()
        Ref.check(Ref.lib().ref_form_mult_count(self.h, _d(x), _d(y), C.byref(c)))
        return y, c.value

    def diagonal(self):
        y = np.zeros(self.n)
        Ref.check(Ref.lib().ref_form_diag(self.h, _d(y)))
        return y

    def stored_reals(self):
        return Ref.lib().ref_form_stored_reals(self.h)

    def qdata(self, integ=0):
        nq = C.c_int()
        nc = C.c_int()
        Ref.check(Ref.lib().ref_form_qdata(self.h, integ, None, C.byref(nq), C.byref(nc)))
        out = np.zeros((self.space.n_elem, nq.value * nq.value, nc.value))
        Ref.check(Ref.lib().ref_form_qdata(self.h, integ, _d(out), C.byref(nq), C.byref(nc)))
        return out

    def matrix_csr(self):
        nnz = C.c_longlong()
        Ref.check(Ref.lib().ref_form_matrix(self.h, None, None, None, C.byref(nnz)))
        rp = np.zeros(self.n + 1, dtype=np.int32)
        cols = np.zeros(nnz.value, dtype=np.int32)
        vals = np.zeros(nnz.value)
        Ref.check(Ref.lib().ref_form_matrix(self.h, _i(rp), _i(cols), _d(vals), C.byref(nnz)))
        return rp, cols, vals


class RefSystem:
    """The driver's homogenised Poisson system (driver.cpp:129-159)."""

    def __init__(self, form: RefForm, solution="front"):
        h = Ref.lib().ref_system_create(form.h, 0 if solution == "sine" else 1)
        if not h:
            raise OracleError(9, Ref.lib().ref_last_error().decode())
        self.h = C.c_void_p(h)
        self.form = form
        n = form.n
        self.n = n
        self.rhs = np.zeros(n)
        self.diag = np.zeros(n)
        self.x0 = np.zeros(n)
        Ref.lib().ref_system_vectors(self.h, _d(self.rhs), _d(self.diag), _d(self.x0))
        ne = Ref.lib().ref_system_ess(self.h, None)
        self.ess = np.zeros(ne, dtype=np.int32)
        Ref.lib().ref_system_ess(self.h, _i(self.ess))

    def __del__(self):
        try:
            Ref.lib().ref_system_free(self.h)
        except Exception:
            pass

    def op_mult(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        Ref.check(Ref.lib().ref_system_op_mult(self.h, _d(x), _d(y)))
        return y

    def cg(self, tol, max_iters, jacobi=True, rhs=None):
        x = np.zeros(self.n)
        it = C.c_int()
        conv = C.c_int()
        sec = C.c_double()
        rhs = None if rhs is None else np.ascontiguousarray(rhs, dtype=np.float64)
        Ref.check(Ref.lib().ref_system_cg(self.h, _d(rhs), tol, max_iters, 1 if jacobi else 0,
                                          _d(x), C.byref(it), C.byref(conv), C.byref(sec)))
        return x, it.value, bool(conv.value), sec.value

    def l2_error(self, x_cg):
        e = C.c_double()
        Ref.check(Ref.lib().ref_system_l2_error(self.h, _d(np.ascontiguousarray(x_cg)),
                                                C.byref(e)))
        return e.value


def ref_solution_u(solution, xy):
    """The reference's manufactured solution u (driver.cpp) at points xy[..., 2]."""
    pts = np.ascontiguousarray(xy, dtype=np.float64)
    out = np.zeros(pts.shape[:-1])
    Ref.check(Ref.lib().ref_solution_u(0 if solution == "sine" else 1, _d(pts),
                                       int(np.prod(pts.shape[:-1])), _d(out)))
    return out


def ref_solution_f(solution, xy):
    """The reference's manufactured source f (driver.cpp) at points xy[..., 2]."""
    pts = np.ascontiguousarray(xy, dtype=np.float64)
    out = np.zeros(pts.shape[:-1])
    Ref.check(Ref.lib().ref_solution_f(0 if solution == "sine" else 1, _d(pts),
                                       int(np.prod(pts.shape[:-1])), _d(out)))
    return out


def ref_cg_csr(rowptr, cols, vals, b, tol, max_iters, diag=None):
    n = len(b)
    x = np.zeros(n)
    it = C.c_int()
    conv = C.c_int()
    Ref.check(Ref.lib().ref_cg_csr(n, _i(rowptr), _i(cols), _d(vals), _d(b), tol, max_iters,
                                   _d(diag), _d(x), C.byref(it), C.byref(conv)))
    return x, it.value, bool(conv.value)


# -------------------------------------------------------------- restatement
class _OrcOp(C.Structure):
    _fields_ = [("dim", C.c_int), ("p", C.c_int), ("nq", C.c_int),
                ("ne", C.c_int64), ("ndofs", C.c_int64),
                ("B", _dp), ("G", _dp), ("n_integ", C.c_int), ("kinds", _ip),
                ("qdata", C.POINTER(_dp)), ("elem_dofs", _ip),
                ("n_ess", C.c_int64), ("ess", _ip)]


class Orc:
    """The C restatement (2D + 3D)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not ORC_SO.exists():
                raise FileNotFoundError(f"{ORC_SO} missing: run make -C oracle")
            L = C.CDLL(str(ORC_SO))
            L.orc_last_error.restype = C.c_char_p
            L.orc_gauss_legendre.argtypes = [C.c_int, _dp, _dp]
            L.orc_gauss_lobatto.argtypes = [C.c_int, _dp, _dp]
            L.orc_basis_nodes.argtypes = [C.c_int, C.c_int, _dp, _dp]
            L.orc_eval_matrices.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp]
            L.orc_cartesian_nv.argtypes = [C.c_int, _ip]
            L.orc_cartesian_nv.restype = C.c_int64
            L.orc_cartesian_ne.argtypes = [C.c_int, _ip]
            L.orc_cartesian_ne.restype = C.c_int64
            L.orc_cartesian_vertices.argtypes = [C.c_int, _ip, _dp, _dp]
            L.orc_cartesian_elements.argtypes = [C.c_int, _ip, _ip]
            L.orc_cartesian_ctrl.argtypes = [C.c_int, _ip, _dp, _dp]
            L.orc_h1_layout_quads.argtypes = [C.c_int, C.c_int, _ip, C.c_int, _ip]
            L.orc_h1_layout_quads.restype = C.c_int64
            L.orc_h1_layout_cartesian.argtypes = [C.c_int, _ip, C.c_int, _ip]
            L.orc_h1_layout_cartesian.restype = C.c_int64
            L.orc_boundary_dofs_cartesian.argtypes = [C.c_int, _ip, C.c_int, _ip]
            L.orc_boundary_dofs_cartesian.restype = C.c_int64
            L.orc_physical_points.argtypes = [C.c_int, C.c_int, C.c_int64, _dp, C.c_int,
                                              C.c_int, _dp]
            L.orc_pa_setup.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64,
                                       _dp, _dp, C.c_double, _dp, C.POINTER(C.c_int64)]
            L.orc_pa_apply_local.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64,
                                             _dp, _dp, _dp, _ip, _dp, _dp,
                                             C.POINTER(C.c_uint64)]
            L.orc_pa_diagonal.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64,
                                          _dp, _dp, _dp, _ip, _dp]
            L.orc_element_matrix.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp,
                                             _dp, _dp]
            L.orc_op_mult.argtypes = [C.POINTER(_OrcOp), _dp, _dp]
            L.orc_cg_pa.argtypes = [C.POINTER(_OrcOp), _dp, C.c_double, C.c_int, _dp, _dp,
                                    _ip, _ip]
            L.orc_cg_csr.argtypes = [C.c_int, _ip, _ip, _dp, _dp, C.c_double, C.c_int, _dp,
                                     _dp, _ip, _ip]
            cls._lib = L
        return cls._lib

    @classmethod
    def check(cls, rc):
        if rc != 0:
            _raise(rc, cls.lib().orc_last_error().decode())

    @classmethod
    def rule(cls, n, lobatto=False):
        p = np.zeros(n)
        w = np.zeros(n)
        fn = cls.lib().orc_gauss_lobatto if lobatto else cls.lib().orc_gauss_legendre
        cls.check(fn(n, _d(p), _d(w)))
        return p, w

    @classmethod
    def eval_matrices(cls, p, nq, node_kind=0, rule_kind=0):
        B = np.zeros((nq, p + 1))
        G = np.zeros((nq, p + 1))
        cls.check(cls.lib().orc_eval_matrices(p, node_kind, nq, rule_kind, _d(B), _d(G)))
        return B, G


def _ivec(n):
    return np.ascontiguousarray(np.array(n, dtype=np.int32))


class OrcCartesian:
    """A Cartesian H1 problem in the restatement: mesh, layout, setup."""

    def __init__(self, dim, n, p, nq=None, rule="gl", ext=None):
        self.dim = dim
        self.n = _ivec(n)
        self.p = p
        self.nq = nq if nq is not None else (p + 2 if rule == "gl" else p + 1)
        self.rule_kind = 0 if rule == "gl" else 1
        L = Orc.lib()
        self.ext = np.ascontiguousarray(np.array(ext if ext else [1.0] * dim, dtype=np.float64))
        self.ne = L.orc_cartesian_ne(dim, _i(self.n))
        self.nd = (p + 1) ** dim
        self.nqd = self.nq ** dim
        self.elem_dofs = np.zeros((self.ne, self.nd), dtype=np.int32)
        self.ndofs = L.orc_h1_layout_cartesian(dim, _i(self.n), p, _i(self.elem_dofs))
        if self.ndofs < 0:
            Orc.check(int(-self.ndofs))
        self.ctrl = np.zeros((self.ne, 2 ** dim, dim))
        L.orc_cartesian_ctrl(dim, _i(self.n), _d(self.ext), _d(self.ctrl))
        self.B, self.G = Orc.eval_matrices(p, self.nq, 0, self.rule_kind)

    def boundary_dofs(self):
        L = Orc.lib()
        cnt = L.orc_boundary_dofs_cartesian(self.dim, _i(self.n), self.p, None)
        out = np.zeros(cnt, dtype=np.int32)
        L.orc_boundary_dofs_cartesian(self.dim, _i(self.n), self.p, _i(out))
        return out

    def points(self):
        out = np.zeros((self.ne, self.nqd, self.dim))
        Orc.check(Orc.lib().orc_physical_points(self.dim, 1, self.ne, _d(self.ctrl), self.nq,
                                                self.rule_kind, _d(out)))
        return out

    def setup(self, kind, coeff=None, const=1.0, ctrl=None, geom_order=1):
        ncomp = 1 if kind == "mass" else (3 if self.dim == 2 else 6)
        qd = np.zeros((self.ne, self.nqd, ncomp))
        bad = C.c_int64(-1)
        ctrl = self.ctrl if ctrl is None else np.ascontiguousarray(ctrl)
        coeff = None if coeff is None else np.ascontiguousarray(coeff, dtype=np.float64)
        Orc.check(Orc.lib().orc_pa_setup(self.dim, KIND[kind], self.nq, self.rule_kind,
                                         geom_order, self.ne, _d(ctrl), _d(coeff), const,
                                         _d(qd), C.byref(bad)))
        return qd

    def apply(self, kind, qdata, x, y=None):
        y = np.zeros(self.ndofs) if y is None else y
        m = C.c_uint64(0)
        Orc.lib().orc_pa_apply_local(self.dim, KIND[kind], self.p, self.nq, self.ne,
                                     _d(self.B), _d(self.G), _d(np.ascontiguousarray(qdata)),
                                     _i(self.elem_dofs), _d(np.ascontiguousarray(x)), _d(y),
                                     C.byref(m))
        return y

    def diagonal(self, kind, qdata, y=None):
        y = np.zeros(self.ndofs) if y is None else y
        Orc.lib().orc_pa_diagonal(self.dim, KIND[kind], self.p, self.nq, self.ne, _d(self.B),
                                  _d(self.G), _d(np.ascontiguousarray(qdata)),
                                  _i(self.elem_dofs), _d(y))
        return y

    def element_matrix(self, kind, qdata_e):
        m = np.zeros((self.nd, self.nd))
        Orc.lib().orc_element_matrix(self.dim, KIND[kind], self.p, self.nq, _d(self.B),
                                     _d(self.G), _d(np.ascontiguousarray(qdata_e)), _d(m))
        return m

    def operator(self, kinds, qdatas, ess=None):
        """Keeps the arrays alive and returns an _OrcOp."""
        self._keep = [np.ascontiguousarray(q) for q in qdatas]
        self._kinds = np.array([KIND[k] for k in kinds], dtype=np.int32)
        self._qptrs = (_dp * len(qdatas))(*[_d(q) for q in self._keep])
        self._ess = np.zeros(0, dtype=np.int32) if ess is None else np.ascontiguousarray(
            ess, dtype=np.int32)
        op = _OrcOp(self.dim, self.p, self.nq, self.ne, self.ndofs, _d(self.B), _d(self.G),
                    len(qdatas), _i(self._kinds), self._qptrs, _i(self.elem_dofs),
                    len(self._ess), _i(self._ess))
        return op

    def op_mult(self, op, x):
        y = np.zeros(self.ndofs)
        Orc.lib().orc_op_mult(C.byref(op), _d(np.ascontiguousarray(x)), _d(y))
        return y

    def cg(self, op, b, tol, max_iters, diag=None):
        x = np.zeros(self.ndofs)
        it = C.c_int()
        conv = C.c_int()
        Orc.check(Orc.lib().orc_cg_pa(C.byref(op), _d(np.ascontiguousarray(b)), tol, max_iters,
                                      _d(diag), _d(x), C.byref(it), C.byref(conv)))
        return x, it.value, bool(conv.value)


def orc_layout_quads(nv, elem_vertices, p):
    ev = np.ascontiguousarray(elem_vertices, dtype=np.int32)
    ne = ev.shape[0]
    out = np.zeros((ne, (p + 1) ** 2), dtype=np.int32)
    nd = Orc.lib().orc_h1_layout_quads(nv, ne, _i(ev), p, _i(out))
    if nd < 0:
        Orc.check(int(-nd))
    return out, nd
