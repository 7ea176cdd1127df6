"""tensorfem API over the sm_100a C ABI -- the host-side mirror of the
reference's PA / CG interface (/root/reference/proj/include/tensorfem).

Names, argument meaning and error behaviour follow the reference:

    reference (C++)                              here
    FeSpace(make_cartesian(n, n), {H1, p})       FeSpace.cartesian(dev, (n, n), p)
    FeSpace::element_dofs / n_dofs               FeSpace.element_dofs() / .n_dofs
    FeSpace::essential_true_dofs(all attrs)      FeSpace.essential_true_dofs()
    pa_setup(space, kind, coeff)                 pa_setup(space, kind, coeff)
    pa_apply_local(pa, space, x, y)   (y +=)     pa_apply_local(pa, space, x, y)
    pa_apply / pa_diagonal                       pa_apply / pa_diagonal
    BilinearForm(space, Partial)                 BilinearForm(space, "partial")
      add_diffusion / add_mass / assemble        same
      mult_true / diagonal_true / stored_reals   same
    form_linear_system(...).op (Partial)         ConstrainedOperator(form, ess)
    SparseOperator(csr)                          SparseOperator(dev, rowptr, cols, vals)
    cg_solve(op, b, tol, it, diag, on_iterate)   cg_solve(op, b, tol, it, diag, on_iterate)
    multiply_count / reset_multiply_count        same (analytic counts per apply)

Exceptions: std::invalid_argument -> InvalidArgument (a ValueError),
std::runtime_error -> TfemRuntimeError, std::logic_error -> LogicError.
Vectors are device resident (`Vector`); numpy arrays are accepted wherever the
reference takes a Vector and are copied in (host buffers).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from typing import Callable, Optional, Sequence, Union

import numpy as np

from . import abi
from .abi import (InvalidArgument, LogicError, TfemRuntimeError, CudaError, check, lib)

DIFFUSION = "diffusion"
MASS = "mass"
_KIND = {DIFFUSION: abi.DIFFUSION, MASS: abi.MASS}
_RULE = {"gauss_legendre": abi.GAUSS_LEGENDRE, "gauss_lobatto": abi.GAUSS_LOBATTO}

_tls = threading.local()


def multiply_count() -> int:
    """Multiplies the instrumented reference kernels would have counted since
    the last reset on this thread (tensor_kernels.hpp:20-26)."""
    return getattr(_tls, "mults", 0)


def reset_multiply_count() -> None:
    _tls.mults = 0


def count_multiplies(n: int) -> None:
    _tls.mults = multiply_count() + int(n)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(abi.dp)


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(abi.i32p)


# ----------------------------------------------------------------- device
class Device:
    """A CUDA device with one stream (tfem_ctx).  numerics: "fma" (default;
    fused multiply-adds, within 1e-15 of the reference) or "reference" (the
    reference's exact operation order: bit-identical 2D results)."""

    def __init__(self, device: int = 0, numerics: str = "fma"):
        h = abi.vp()
        check(lib().tfem_ctx_create(device, C.byref(h)))
        self.h = h
        self.set_numerics(numerics)

    def set_numerics(self, mode: str):
        m = {"reference": abi.NUMERICS_REFERENCE, "fma": abi.NUMERICS_FMA}[mode]
        check(lib().tfem_ctx_set_numerics(self.h, m))
        self.numerics = mode

    def sync(self):
        check(lib().tfem_ctx_sync(self.h))

    @property
    def stream(self) -> int:
        return lib().tfem_ctx_stream(self.h) or 0

    def launch_count(self) -> int:
        return lib().tfem_ctx_launch_count(self.h)

    def set_max_blocks(self, n: int):
        """Test hook: cap the persistent element kernels at n blocks (0: one
        per SM) so small meshes run many laps of each block's pipeline."""
        check(lib().tfem_ctx_set_max_blocks(self.h, n))

    def close(self):
        if getattr(self, "h", None):
            lib().tfem_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Optional[Device] = None


def default_device() -> Device:
    global _default
    if _default is None:
        _default = Device(0)
    return _default


# ----------------------------------------------------------------- vector
class Vector:
    """Vector (vector.hpp:14-48) resident in HBM."""

    def __init__(self, dev: Device, n: int, value: float = 0.0, _wrap=None):
        self.dev = dev
        self.h = abi.vp()
        if _wrap is not None:
            ptr, self._keep = _wrap
            check(lib().tfem_vec_wrap(dev.h, ptr, n, C.byref(self.h)))
        else:
            check(lib().tfem_vec_create(dev.h, n, C.byref(self.h)))
            if value != 0.0:
                check(lib().tfem_vec_fill(self.h, value))
        self.n = int(n)

    @classmethod
    def from_numpy(cls, dev: Device, a) -> "Vector":
        a = np.ascontiguousarray(a, dtype=np.float64)
        v = cls(dev, a.size)
        v.upload(a)
        return v

    @classmethod
    def wrap_torch(cls, dev: Device, t) -> "Vector":
        """Non-owning view of a contiguous float64 CUDA tensor."""
        assert t.is_cuda and t.dtype.is_floating_point and t.element_size() == 8
        return cls(dev, t.numel(), _wrap=(t.data_ptr(), t))

    def size(self) -> int:
        return self.n

    def __len__(self):
        return self.n

    @property
    def data_ptr(self) -> int:
        return lib().tfem_vec_data(self.h) or 0

    def upload(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        check(lib().tfem_vec_upload(self.h, _dptr(a), a.size))

    def numpy(self) -> np.ndarray:
        out = np.empty(self.n)
        check(lib().tfem_vec_download(self.h, _dptr(out), self.n))
        return out

    def set_zero(self):
        check(lib().tfem_vec_fill(self.h, 0.0))

    def fill(self, v: float):
        check(lib().tfem_vec_fill(self.h, v))

    def dot(self, other: "Vector") -> float:
        out = C.c_double()
        check(lib().tfem_vec_dot(self.dev.h, self.h, other.h, C.byref(out)))
        return out.value

    def norm2(self) -> float:
        return float(np.sqrt(self.dot(self)))

    def axpy(self, a: float, x: "Vector"):
        """this += a * x"""
        check(lib().tfem_vec_axpy(self.dev.h, a, x.h, self.h))

    def __del__(self):
        try:
            if self.h:
                lib().tfem_vec_destroy(self.h)
                self.h = None
        except Exception:
            pass


def as_vector(dev: Device, v) -> Vector:
    return v if isinstance(v, Vector) else Vector.from_numpy(dev, v)


# ------------------------------------------------------------------ space
class FeSpace:
    """H1 space: the element restriction G (ElementRestriction), the element
    geometry and the prolongation P -- the identity on conforming meshes
    (fespace.cpp:62-72), [I; W] on non-conforming forests (:166-203)."""

    def __init__(self, dev, dim, order, restriction, geometry, n_cells=None, prolongation=None,
                 n_true=None):
        self.dev = dev
        self.dim = dim
        self._order = order
        self.r = restriction
        self.g = geometry
        self.P = prolongation
        self.n_cells = n_cells
        self.n_dofs = lib().tfem_restriction_n_dofs(restriction)
        self.n_elements = lib().tfem_restriction_n_elem(restriction)
        self._n_true = self.n_dofs if prolongation is None else n_true

    @property
    def conforming(self) -> bool:
        return self.P is None

    @classmethod
    def cartesian(cls, dev: Device, n: Sequence[int], order: int,
                  extents: Optional[Sequence[float]] = None) -> "FeSpace":
        """H1 order-p space on make_cartesian(n..., extents) (mesh.cpp:283-321),
        generated on the device; 2D numbering identical to the reference."""
        dim = len(n)
        nn = (C.c_int * 3)(*(list(n) + [0] * (3 - dim)))
        r = abi.vp()
        check(lib().tfem_restriction_cartesian(dev.h, dim, nn, order, C.byref(r)))
        g = abi.vp()
        ext = (C.c_double * 3)(*(list(extents or [1.0] * dim) + [0.0] * (3 - dim)))
        rc = lib().tfem_geometry_cartesian(dev.h, dim, nn, ext, C.byref(g))
        if rc:
            lib().tfem_restriction_destroy(r)
            check(rc)
        return cls(dev, dim, order, r, g, tuple(n))

    @classmethod
    def cartesian_box(cls, dev: Device, n_local: Sequence[int], origin: Sequence[int],
                      n_global: Sequence[int], order: int,
                      extents: Optional[Sequence[float]] = None) -> "FeSpace":
        """The n_local block at cell offset `origin` of make_cartesian(n_global)
        (one rank's slab): local DOF numbering, global vertex coordinates."""
        dim = len(n_local)
        pad = lambda v: (C.c_int * 3)(*(list(v) + [0] * (3 - dim)))
        r = abi.vp()
        check(lib().tfem_restriction_cartesian(dev.h, dim, pad(n_local), order, C.byref(r)))
        g = abi.vp()
        ext = (C.c_double * 3)(*(list(extents or [1.0] * dim) + [0.0] * (3 - dim)))
        rc = lib().tfem_geometry_cartesian_box(dev.h, dim, pad(n_local), pad(origin),
                                               pad(n_global), ext, C.byref(g))
        if rc:
            lib().tfem_restriction_destroy(r)
            check(rc)
        return cls(dev, dim, order, r, g, tuple(n_local))

    @classmethod
    def from_mesh(cls, dev: Device, dim: int, order: int, elem_dofs: np.ndarray, n_dofs: int,
                  ctrl: np.ndarray, geom_order: int = 1, prolongation=None) -> "FeSpace":
        """A space from a host element -> DOF table (FeSpace::element_dofs,
        [e][i]) and geometry control points ([e][lattice][dim]).
        `prolongation` = (rowptr, cols, vals, true_index, n_true) of
        FeSpace::prolongation() / true_index() on non-conforming meshes."""
        P, n_true = None, None
        if prolongation is not None:
            rp, cols, vals, tix, n_true = prolongation
            arrs = [np.ascontiguousarray(rp, dtype=np.int32), np.ascontiguousarray(cols, dtype=np.int32),
                    np.ascontiguousarray(vals, dtype=np.float64), np.ascontiguousarray(tix, dtype=np.int32)]
            P = abi.vp()
            check(lib().tfem_prolongation_create(dev.h, n_dofs, n_true, _iptr(arrs[0]),
                                                 _iptr(arrs[1]), _dptr(arrs[2]), _iptr(arrs[3]),
                                                 C.byref(P)))
        ed = np.ascontiguousarray(elem_dofs, dtype=np.int32)
        r = abi.vp()
        check(lib().tfem_restriction_create(dev.h, dim, order, ed.shape[0], n_dofs, _iptr(ed),
                                            C.byref(r)))
        ct = np.ascontiguousarray(ctrl, dtype=np.float64)
        g = abi.vp()
        rc = lib().tfem_geometry_create(dev.h, dim, geom_order, ed.shape[0], _dptr(ct),
                                        C.byref(g))
        if rc:
            lib().tfem_restriction_destroy(r)
            check(rc)
        return cls(dev, dim, order, r, g, prolongation=P, n_true=n_true)

    def order(self) -> int:
        return self._order

    @property
    def n_true_dofs(self) -> int:
        return self._n_true

    def true_to_local(self, x) -> Vector:
        """P x (fespace.cpp:244-250)."""
        xv = as_vector(self.dev, x)
        if xv.n != self.n_true_dofs:
            raise InvalidArgument("true_to_local: size mismatch")
        y = Vector(self.dev, self.n_dofs)
        if self.P is None:
            y.axpy(1.0, xv)
        else:
            check(lib().tfem_prolongation_mult(self.dev.h, self.P, xv.h, y.h))
        return y

    def local_to_true(self, x) -> Vector:
        """X[t] = x[true_dofs[t]] (fespace.cpp:252-262)."""
        xv = as_vector(self.dev, x)
        if xv.n != self.n_dofs:
            raise InvalidArgument("local_to_true: size mismatch")
        X = Vector(self.dev, self.n_true_dofs)
        if self.P is None:
            X.axpy(1.0, xv)
        else:
            check(lib().tfem_prolongation_local_to_true(self.dev.h, self.P, xv.h, X.h))
        return X

    def prolongation_transpose(self, y_local: Vector) -> Vector:
        """P^T y (SparseMatrix::mult_transpose, sparse.cpp:89-102)."""
        if self.P is None:
            y = Vector(self.dev, self.n_dofs)
            y.axpy(1.0, y_local)
            return y
        y = Vector(self.dev, self.n_true_dofs)
        check(lib().tfem_prolongation_mult_transpose(self.dev.h, self.P, y_local.h, y.h))
        return y

    def element_dofs(self) -> np.ndarray:
        nd = (self._order + 1) ** self.dim
        out = np.empty((self.n_elements, nd), dtype=np.int32)
        check(lib().tfem_restriction_elem_dofs(self.r, _iptr(out)))
        return out

    def essential_true_dofs(self) -> np.ndarray:
        """Sorted DOFs on every boundary attribute (fespace.cpp:205-242)."""
        cnt = C.c_int64()
        check(lib().tfem_restriction_boundary_dofs(self.r, None, C.byref(cnt)))
        out = np.empty(cnt.value, dtype=np.int32)
        check(lib().tfem_restriction_boundary_dofs(self.r, _iptr(out), C.byref(cnt)))
        return out

    def physical_points(self, nq: int, rule: str = "gauss_legendre") -> np.ndarray:
        nqd = nq ** self.dim
        out = np.empty((self.n_elements, nqd, self.dim))
        check(lib().tfem_geometry_points(self.dev.h, self.g, nq, _RULE[rule], _dptr(out)))
        return out

    def restrict(self, x: Vector) -> Vector:
        """ElementRestriction::Mult: L -> E ([e][i])."""
        nd = (self._order + 1) ** self.dim
        e = Vector(self.dev, self.n_elements * nd)
        check(lib().tfem_restriction_mult(self.dev.h, self.r, x.h, e.h))
        return e

    def restrict_transpose(self, e: Vector, y: Vector):
        """ElementRestriction::MultTranspose: y += G^T e (element order)."""
        check(lib().tfem_restriction_mult_transpose(self.dev.h, self.r, e.h, y.h))

    def __del__(self):
        try:
            lib().tfem_restriction_destroy(self.r)
            lib().tfem_geometry_destroy(self.g)
            if self.P is not None:
                lib().tfem_prolongation_destroy(self.P)
        except Exception:
            pass


# ------------------------------------------------------------ PA (D data)
Coefficient = Union[float, int, Callable[[np.ndarray], np.ndarray], np.ndarray]


class PaData:
    """Quadrature-point factors of one integrator (forms.hpp:29-58)."""

    def __init__(self, space: FeSpace, kind: str, h):
        self.space = space
        self.h = h
        self._kind = kind
        k, d, p, nq, ne = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        check(lib().tfem_pa_info(h, C.byref(k), C.byref(d), C.byref(p), C.byref(nq),
                                 C.byref(ne)))
        self._order, self._nq, self.n_elements, self.dim = p.value, nq.value, ne.value, d.value

    def kind(self) -> str:
        return self._kind

    def order(self) -> int:
        return self._order

    def quad_1d(self) -> int:
        return self._nq

    def _basis(self):
        B = np.empty((self._nq, self._order + 1))
        G = np.empty_like(B)
        check(lib().tfem_pa_basis(self.h, _dptr(B), _dptr(G)))
        return B, G

    def b1d(self) -> np.ndarray:
        return self._basis()[0]

    def g1d(self) -> np.ndarray:
        return self._basis()[1]

    def stored_reals(self) -> int:
        return lib().tfem_pa_stored_reals(self.h)

    def multiplies_per_apply(self) -> int:
        return lib().tfem_pa_multiply_count(self.h)

    def qdata(self) -> np.ndarray:
        """All factors in the reference layout [e][q][c] (forms.cpp:219-225)."""
        nc = 1 if self._kind == MASS else (3 if self.dim == 2 else 6)
        out = np.empty((self.n_elements, self._nq ** self.dim, nc))
        check(lib().tfem_pa_qdata(self.h, _dptr(out)))
        return out

    def d(self, element: int) -> np.ndarray:
        return self.qdata()[element].reshape(-1)

    def __del__(self):
        try:
            lib().tfem_pa_destroy(self.h)
        except Exception:
            pass


def _coeff_values(space: FeSpace, coeff: Coefficient, nq: int, rule: str):
    """(per-point array or None, constant) for the C ABI."""
    if coeff is None:
        raise InvalidArgument("pa_setup: coefficient is empty")
    if isinstance(coeff, (int, float)):
        return None, float(coeff)
    if callable(coeff):
        pts = space.physical_points(nq, rule)
        vals = np.asarray(coeff(pts), dtype=np.float64)
        return np.ascontiguousarray(np.broadcast_to(vals, pts.shape[:2])), 0.0
    arr = np.ascontiguousarray(coeff, dtype=np.float64)
    return arr, 0.0


def pa_setup(space: FeSpace, kind: str, coeff: Coefficient, rule: str = "gauss_legendre",
             nq: Optional[int] = None) -> PaData:
    """pa_setup (forms.cpp:201-229).  Default rule: q = p+2 Gauss-Legendre;
    BP5: rule="gauss_lobatto", nq = p+1."""
    if kind not in _KIND:
        raise InvalidArgument(f"pa_setup: unknown integrator kind {kind!r}")
    p = space.order()
    if nq is None:
        nq = p + 2 if rule == "gauss_legendre" else p + 1
    arr, const = _coeff_values(space, coeff, nq, rule)
    h = abi.vp()
    bad = C.c_int64(-1)
    check(lib().tfem_pa_setup(space.dev.h, _KIND[kind], space.g, p, nq, _RULE[rule],
                              None if arr is None else _dptr(arr), const, C.byref(h),
                              C.byref(bad)))
    return PaData(space, kind, h)


def pa_apply_local(pa: PaData, space: FeSpace, x: Vector, y: Vector, threads: int = 1):
    """y += G^T B^T D B G x (forms.cpp:231-296).  `threads` is accepted for
    API parity; the result never depends on it."""
    if threads < 1:
        raise InvalidArgument("pa_apply_local: threads must be >= 1")
    check(lib().tfem_pa_apply_local(space.dev.h, pa.h, space.r, x.h, y.h))
    count_multiplies(pa.multiplies_per_apply())


def pa_apply(pa: PaData, space: FeSpace, x) -> Vector:
    """y = P^T G^T B^T D B G P x (forms.cpp:298-309)."""
    xv = as_vector(space.dev, x)
    if xv.n != space.n_true_dofs:
        raise InvalidArgument("pa_apply: size mismatch")
    if space.P is None:
        y = Vector(space.dev, space.n_dofs)
        pa_apply_local(pa, space, xv, y)
        return y
    yl = Vector(space.dev, space.n_dofs)
    pa_apply_local(pa, space, space.true_to_local(xv), yl)
    return space.prolongation_transpose(yl)


def pa_diagonal(pa: PaData, space: FeSpace) -> Vector:
    """Exact diagonal (forms.cpp:311-382), on the true DOFs."""
    d = Vector(space.dev, space.n_true_dofs)
    if space.P is None:
        check(lib().tfem_pa_diagonal(space.dev.h, pa.h, space.r, d.h))
    else:
        check(lib().tfem_pa_diagonal_p(space.dev.h, pa.h, space.r, space.P, d.h))
    return d


class LinearForm:
    """LinearForm(space, f) (forms.cpp:400-431): b_i = sum_q w detJ f(x_q)
    phi_i(x_q), q = p + 2 Gauss-Legendre points, f evaluated on the host at
    the device-computed physical points, contraction and element-ordered
    scatter on the device (bit-identical to the reference)."""

    def __init__(self, space: FeSpace, f: Coefficient):
        if f is None:
            raise InvalidArgument("LinearForm: load function is empty")
        self.space = space
        nq = space.order() + 2
        arr, const = _coeff_values(space, f, nq, "gauss_legendre")
        if arr is None:
            arr = np.full((space.n_elements, nq * nq), const)
        vals = np.ascontiguousarray(arr, dtype=np.float64)
        self._b = Vector(space.dev, space.n_dofs)
        check(lib().tfem_linear_form(space.dev.h, space.g, space.r, space.order(), _dptr(vals),
                                     self._b.h))

    def values(self) -> Vector:
        return self._b


def project_coefficient(space: FeSpace, f: Callable[[np.ndarray], np.ndarray]) -> Vector:
    """project_coefficient (fespace.cpp:334-356): nodal interpolation of f,
    the last element winning on shared DOFs (L-vector)."""
    if f is None:
        raise InvalidArgument("project_coefficient: function is empty")
    nd = space.order() + 1
    xy = np.empty((space.n_elements, nd * nd, 2))
    check(lib().tfem_geometry_node_points(space.dev.h, space.g, space.order(), _dptr(xy)))
    vals = np.ascontiguousarray(np.broadcast_to(np.asarray(f(xy), dtype=np.float64),
                                                xy.shape[:2]))
    out = Vector(space.dev, space.n_dofs)
    check(lib().tfem_project(space.dev.h, space.r, _dptr(vals), out.h))
    return out


def compute_l2_error(space: FeSpace, x, u_exact: Callable[[np.ndarray], np.ndarray]) -> float:
    """compute_l2_error (fespace.cpp:358-394) of the L-vector x against
    u_exact, q = p + 3 Gauss-Legendre points; bit-identical to the reference."""
    xv = as_vector(space.dev, x)
    nq = space.order() + 3
    pts = space.physical_points(nq, "gauss_legendre")
    ue = np.ascontiguousarray(np.broadcast_to(np.asarray(u_exact(pts), dtype=np.float64),
                                              pts.shape[:2]))
    err = C.c_double()
    check(lib().tfem_l2_error(space.dev.h, space.g, space.r, space.order(), xv.h, _dptr(ue),
                              C.byref(err)))
    return err.value


# --------------------------------------------------------------- operators
class LinearOperator:
    """The virtual mult seam cg_solve drives (solvers.hpp:16-23)."""

    h = None
    dev: Device

    def rows(self) -> int:
        return lib().tfem_operator_size(self.h)

    def cols(self) -> int:
        return self.rows()

    def mult(self, x, y: Vector):
        xv = as_vector(self.dev, x)
        check(lib().tfem_operator_mult(self.dev.h, self.h, xv.h, y.h))
        self._count()

    def _count(self):
        pass

    def __del__(self):
        try:
            if self.h:
                lib().tfem_operator_destroy(self.h)
        except Exception:
            pass


class SparseOperator(LinearOperator):
    """SparseOperator over a CSR matrix (solvers.hpp:26-35)."""

    def __init__(self, dev: Device, rowptr, cols, vals):
        self.dev = dev
        self._arrs = [np.ascontiguousarray(rowptr, dtype=np.int32),
                      np.ascontiguousarray(cols, dtype=np.int32),
                      np.ascontiguousarray(vals, dtype=np.float64)]
        h = abi.vp()
        check(lib().tfem_operator_create_csr(dev.h, len(self._arrs[0]) - 1,
                                             _iptr(self._arrs[0]), _iptr(self._arrs[1]),
                                             _dptr(self._arrs[2]), C.byref(h)))
        self.h = h


class _PaOperator(LinearOperator):
    def __init__(self, form: "BilinearForm", essential=None):
        self.form = form
        self.dev = form.space.dev
        ess = np.zeros(0, dtype=np.int32) if essential is None else np.ascontiguousarray(
            essential, dtype=np.int32)
        arr = (abi.vp * len(form._pa))(*[pa.h for pa in form._pa])
        h = abi.vp()
        check(lib().tfem_operator_create_p(self.dev.h, len(form._pa), arr, form.space.r,
                                           form.space.P, len(ess),
                                           _iptr(ess) if len(ess) else None, C.byref(h)))
        self.h = h
        self.essential = ess

    def _count(self):
        count_multiplies(sum(pa.multiplies_per_apply() for pa in self.form._pa))

    def diagonal(self) -> Vector:
        d = Vector(self.dev, self.rows())
        check(lib().tfem_operator_diagonal(self.dev.h, self.h, d.h))
        return d


class ConstrainedOperator(_PaOperator):
    """form_linear_system's Partial operator (forms.cpp:164-190): identity on
    the sorted, unique essential DOFs, A with essential couplings cut
    elsewhere."""

    def __init__(self, form: "BilinearForm", essential):
        form._require_assembled()
        super().__init__(form, essential)


class BilinearForm:
    """BilinearForm in AssemblyMode::Partial (forms.hpp:105-157)."""

    def __init__(self, space: FeSpace, mode: str = "partial"):
        if mode != "partial":
            raise InvalidArgument("BilinearForm: only partial assembly runs on the device "
                                  "(full assembly is outside the PA hot path)")
        self.space = space
        self._integ = []
        self._pa = []
        self._assembled = False
        self._op = None

    def mode(self) -> str:
        return "partial"

    def add_diffusion(self, kappa: Coefficient, rule: str = "gauss_legendre", nq=None):
        self._add(DIFFUSION, kappa, rule, nq)

    def add_mass(self, rho: Coefficient, rule: str = "gauss_legendre", nq=None):
        self._add(MASS, rho, rule, nq)

    def _add(self, kind, coeff, rule, nq):
        if self._assembled:
            raise LogicError("BilinearForm: already assembled")
        if coeff is None:
            raise InvalidArgument("BilinearForm: coefficient is empty")
        self._integ.append((kind, coeff, rule, nq))

    def assemble(self, threads: int = 1):
        if threads < 1:
            raise InvalidArgument("BilinearForm: threads must be >= 1")
        if self._assembled:
            raise LogicError("BilinearForm: already assembled")
        self._pa = [pa_setup(self.space, k, c, r, q) for k, c, r, q in self._integ]
        self._assembled = True

    def assembled(self) -> bool:
        return self._assembled

    def _require_assembled(self):
        if not self._assembled:
            raise LogicError("BilinearForm: assemble() has not been called")

    def true_size(self) -> int:
        return self.space.n_true_dofs

    def pa_data(self):
        return list(self._pa)

    def operator(self) -> _PaOperator:
        self._require_assembled()
        if self._op is None:
            self._op = _PaOperator(self)
        return self._op

    def mult_true(self, x, y: Vector):
        """y = A x on true-DOF vectors (forms.cpp:527-543)."""
        self._require_assembled()
        n = self.true_size()
        if len(x) != n or len(y) != n:
            raise InvalidArgument("BilinearForm::mult_true: size mismatch")
        self.operator().mult(x, y)

    def diagonal_true(self) -> Vector:
        self._require_assembled()
        return self.operator().diagonal()

    def stored_reals(self) -> int:
        return sum(pa.stored_reals() for pa in self._pa)

    def local_matrix_reals(self) -> int:
        return 0

    def global_matrix_nnz(self) -> int:
        return 0


# --------------------------------------------------------------------- CG
@dataclass
class CgResult:
    """CgResult (solvers.hpp:37-41)."""
    x: Vector
    iterations: int
    converged: bool
    final_norm: float = 0.0
    initial_norm: float = 0.0
    x_norm: float = 0.0  # recursive residual norm of the returned x


def cg_solve(op: LinearOperator, b, rel_tol: float, max_iters: int,
             jacobi_diag=None, on_iterate: Optional[Callable[[int, np.ndarray], None]] = None,
             x: Optional[Vector] = None) -> CgResult:
    """cg_solve (solvers.cpp:11-97), the whole loop on the device."""
    dev = op.dev
    bv = as_vector(dev, b)
    dv = None if jacobi_diag is None else as_vector(dev, jacobi_diag)
    xv = x if x is not None else Vector(dev, bv.n)
    res = abi.CgResult()
    cb = abi.CG_CALLBACK(0)
    if on_iterate is not None:
        def _cb(it, ptr, n, user):
            on_iterate(it, np.ctypeslib.as_array(ptr, shape=(n,)).copy())
        cb = abi.CG_CALLBACK(_cb)
    check(lib().tfem_cg_solve(dev.h, op.h, bv.h, rel_tol, max_iters,
                              None if dv is None else dv.h, xv.h, C.byref(res), cb, None))
    op._count_iters = res.iterations
    return CgResult(xv, res.iterations, bool(res.converged), res.final_norm, res.initial_norm,
                    res.x_norm)


def cg_solve_host(op: LinearOperator, b: np.ndarray, rel_tol: float, max_iters: int,
                  jacobi_diag: Optional[np.ndarray] = None, out: Optional[np.ndarray] = None):
    """cg_solve with host buffers end to end (H2D of b / diag, D2H of x)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = out if out is not None else np.empty_like(b)
    d = None if jacobi_diag is None else np.ascontiguousarray(jacobi_diag, dtype=np.float64)
    res = abi.CgResult()
    check(lib().tfem_cg_solve_host(op.dev.h, op.h, _dptr(b), rel_tol, max_iters,
                                   None if d is None else _dptr(d), _dptr(x), C.byref(res)))
    return x, res.iterations, bool(res.converged)
