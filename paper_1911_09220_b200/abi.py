"""ctypes binding of the C ABI in include/tfem_cuda.h (libtfem_cuda.so).

This is the whole Python <-> device boundary: plain pointers, sizes and int
status codes.  Status codes are mapped back to the reference's exception
classes (invalid_argument -> InvalidArgument(ValueError), runtime_error ->
TfemRuntimeError(RuntimeError), logic_error -> LogicError).  There is no
fallback: if the shared library is missing, importing fails.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

HERE = Path(__file__).resolve().parent
SO_PATH = HERE / "libtfem_cuda.so"


class TfemError(Exception):
    code = 0


class InvalidArgument(TfemError, ValueError):
    """std::invalid_argument"""
    code = 1


class TfemRuntimeError(TfemError, RuntimeError):
    """std::runtime_error"""
    code = 2


class LogicError(TfemError, RuntimeError):
    """std::logic_error"""
    code = 3


class CudaError(TfemError, RuntimeError):
    code = 4


_BY_CODE = {1: InvalidArgument, 2: TfemRuntimeError, 3: LogicError, 4: CudaError}

OK, INVALID_ARGUMENT, RUNTIME_ERROR, LOGIC_ERROR, CUDA_ERROR = range(5)
DIFFUSION, MASS = 0, 1
GAUSS_LEGENDRE, GAUSS_LOBATTO = 0, 1
NODES_GAUSS_LOBATTO, NODES_GAUSS_LEGENDRE, NODES_UNIFORM = 0, 1, 2
NUMERICS_REFERENCE, NUMERICS_FMA = 0, 1

vp = C.c_void_p
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
i32p = C.POINTER(C.c_int32)
i64 = C.c_int64
i64p = C.POINTER(C.c_int64)


class CgResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int),
                ("final_norm", C.c_double), ("initial_norm", C.c_double),
                ("x_norm", C.c_double)]


CG_CALLBACK = C.CFUNCTYPE(None, C.c_int, dp, i64, vp)

MAX_PEERS = 8
NCCL_ID_BYTES = 128
EXCHANGE_HOOK = C.CFUNCTYPE(None, vp)
ALLREDUCE_HOOK = C.CFUNCTYPE(None, C.c_int, vp)


class Comm(C.Structure):
    _fields_ = [("exchange", EXCHANGE_HOOK), ("allreduce", ALLREDUCE_HOOK), ("user", vp)]


class Halo(C.Structure):
    _fields_ = [("n_peers", C.c_int),
                ("n_send", i64 * MAX_PEERS), ("n_recv", i64 * MAX_PEERS),
                ("send_idx", i32p * MAX_PEERS), ("recv_idx", i32p * MAX_PEERS),
                ("send_buf", vp * MAX_PEERS), ("recv_buf", vp * MAX_PEERS),
                ("red", vp)]

_PROTOS = {
    "tfem_last_error": (C.c_char_p, []),
    "tfem_version": (C.c_char_p, []),
    "tfem_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "tfem_ctx_destroy": (C.c_int, [vp]),
    "tfem_ctx_sync": (C.c_int, [vp]),
    "tfem_ctx_stream": (vp, [vp]),
    "tfem_ctx_set_numerics": (C.c_int, [vp, C.c_int]),
    "tfem_ctx_launch_count": (i64, [vp]),
    "tfem_ctx_set_max_blocks": (C.c_int, [vp, C.c_int]),
    "tfem_mem_alloc": (C.c_int, [vp, C.c_size_t, C.POINTER(vp)]),
    "tfem_mem_free": (C.c_int, [vp, vp]),
    "tfem_mem_trim": (C.c_int, [vp]),
    "tfem_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
    "tfem_host_free": (C.c_int, [vp]),
    "tfem_copy": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "tfem_quadrature": (C.c_int, [C.c_int, C.c_int, dp, dp]),
    "tfem_eval_matrices": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, dp, dp]),
    "tfem_vec_create": (C.c_int, [vp, i64, C.POINTER(vp)]),
    "tfem_vec_wrap": (C.c_int, [vp, vp, i64, C.POINTER(vp)]),
    "tfem_vec_destroy": (C.c_int, [vp]),
    "tfem_vec_size": (i64, [vp]),
    "tfem_vec_data": (vp, [vp]),
    "tfem_vec_upload": (C.c_int, [vp, dp, i64]),
    "tfem_vec_download": (C.c_int, [vp, dp, i64]),
    "tfem_vec_fill": (C.c_int, [vp, C.c_double]),
    "tfem_vec_dot": (C.c_int, [vp, vp, vp, dp]),
    "tfem_vec_axpy": (C.c_int, [vp, C.c_double, vp, vp]),
    "tfem_restriction_create": (C.c_int, [vp, C.c_int, C.c_int, i64, i64, i32p, C.POINTER(vp)]),
    "tfem_restriction_cartesian": (C.c_int, [vp, C.c_int, ip, C.c_int, C.POINTER(vp)]),
    "tfem_restriction_destroy": (C.c_int, [vp]),
    "tfem_restriction_n_dofs": (i64, [vp]),
    "tfem_restriction_n_elem": (i64, [vp]),
    "tfem_restriction_elem_dofs": (C.c_int, [vp, i32p]),
    "tfem_restriction_boundary_dofs": (C.c_int, [vp, i32p, i64p]),
    "tfem_restriction_mult": (C.c_int, [vp, vp, vp, vp]),
    "tfem_restriction_mult_transpose": (C.c_int, [vp, vp, vp, vp]),
    "tfem_geometry_create": (C.c_int, [vp, C.c_int, C.c_int, i64, dp, C.POINTER(vp)]),
    "tfem_geometry_cartesian": (C.c_int, [vp, C.c_int, ip, dp, C.POINTER(vp)]),
    "tfem_geometry_cartesian_box": (C.c_int, [vp, C.c_int, ip, ip, ip, dp, C.POINTER(vp)]),
    "tfem_geometry_destroy": (C.c_int, [vp]),
    "tfem_geometry_points": (C.c_int, [vp, vp, C.c_int, C.c_int, dp]),
    "tfem_pa_setup": (C.c_int, [vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, dp, C.c_double,
                                C.POINTER(vp), i64p]),
    "tfem_pa_destroy": (C.c_int, [vp]),
    "tfem_pa_info": (C.c_int, [vp, ip, ip, ip, ip, i64p]),
    "tfem_pa_stored_reals": (i64, [vp]),
    "tfem_pa_multiply_count": (C.c_uint64, [vp]),
    "tfem_pa_qdata": (C.c_int, [vp, dp]),
    "tfem_pa_basis": (C.c_int, [vp, dp, dp]),
    "tfem_pa_set_basis": (C.c_int, [vp, dp, dp]),
    "tfem_pa_apply_local": (C.c_int, [vp, vp, vp, vp, vp]),
    "tfem_pa_diagonal": (C.c_int, [vp, vp, vp, vp]),
    "tfem_linear_form": (C.c_int, [vp, vp, vp, C.c_int, dp, vp]),
    "tfem_geometry_node_points": (C.c_int, [vp, vp, C.c_int, dp]),
    "tfem_project": (C.c_int, [vp, vp, dp, vp]),
    "tfem_l2_error": (C.c_int, [vp, vp, vp, C.c_int, vp, dp, dp]),
    "tfem_pa_diagonal_p": (C.c_int, [vp, vp, vp, vp, vp]),
    "tfem_prolongation_create": (C.c_int, [vp, i64, i64, i32p, i32p, dp, i32p, C.POINTER(vp)]),
    "tfem_prolongation_destroy": (C.c_int, [vp]),
    "tfem_prolongation_mult": (C.c_int, [vp, vp, vp, vp]),
    "tfem_prolongation_mult_transpose": (C.c_int, [vp, vp, vp, vp]),
    "tfem_prolongation_local_to_true": (C.c_int, [vp, vp, vp, vp]),
    "tfem_operator_create_p": (C.c_int, [vp, C.c_int, C.POINTER(vp), vp, vp, i64, i32p,
                                         C.POINTER(vp)]),
    "tfem_operator_create": (C.c_int, [vp, C.c_int, C.POINTER(vp), vp, i64, i32p,
                                       C.POINTER(vp)]),
    "tfem_operator_set_comm": (C.c_int, [vp, C.POINTER(Comm), C.POINTER(Halo), i64, i32p]),
    "tfem_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "tfem_nccl_create": (C.c_int, [vp, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)]),
    "tfem_nccl_destroy": (C.c_int, [vp]),
    "tfem_nccl_allreduce": (C.c_int, [vp, vp, vp, i64]),
    "tfem_operator_set_nccl": (C.c_int, [vp, vp, C.c_int, ip, i64p, C.POINTER(i32p), i64p,
                                         C.POINTER(i32p), i64, i32p]),
    "tfem_operator_create_csr": (C.c_int, [vp, i64, i32p, i32p, dp, C.POINTER(vp)]),
    "tfem_operator_destroy": (C.c_int, [vp]),
    "tfem_operator_size": (i64, [vp]),
    "tfem_operator_mult": (C.c_int, [vp, vp, vp, vp]),
    "tfem_operator_mult_async": (C.c_int, [vp, vp, vp, vp]),
    "tfem_operator_diagonal": (C.c_int, [vp, vp, vp]),
    "tfem_cg_solve": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, vp, vp, C.POINTER(CgResult),
                                CG_CALLBACK, vp]),
    "tfem_cg_profile": (C.c_int, [vp, vp, vp, C.c_int, vp, vp, dp]),
    "tfem_fp64_peak": (C.c_int, [vp, dp]),
    "tfem_dmma_peak": (C.c_int, [vp, dp]),
    "tfem_contraction_ab": (C.c_int, [vp, C.c_int, dp]),
    "tfem_cg_solve_host": (C.c_int, [vp, vp, dp, C.c_double, C.c_int, dp, dp,
                                     C.POINTER(CgResult)]),
}

_lib = None


def lib():
    """Loads libtfem_cuda.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not SO_PATH.exists():
            raise ImportError(f"{SO_PATH} is missing: build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(str(SO_PATH))
        for name, (res, args) in _PROTOS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_PROTOS)


def check(rc):
    if rc != 0:
        msg = lib().tfem_last_error().decode()
        raise _BY_CODE.get(rc, TfemError)(msg)
