"""B200-native (sm_100a) partial-assembly operator + Jacobi-CG for high-order
H1 finite elements -- the accelerator path of arXiv 1911.09220 (MFEM),
drop-in for the tensorfem reference's PA / CG interface.

Layers:
  include/tfem_cuda.h        C ABI (the drop-in boundary)
  csrc/*.cu                  sm_100a kernels + the ABI  -> libtfem_cuda.so
  abi.py                     ctypes binding (no fallback: fails if .so missing)
  tensorfem.py               the reference-named host API
"""
from .abi import (CudaError, InvalidArgument, LogicError, TfemError, TfemRuntimeError, lib,
                  SO_PATH)
from .tensorfem import (DIFFUSION, MASS, BilinearForm, CgResult, ConstrainedOperator, Device,
                        FeSpace, LinearForm, LinearOperator, PaData, SparseOperator, Vector,
                        cg_solve,
                        cg_solve_host, compute_l2_error, count_multiplies, default_device,
                        multiply_count, project_coefficient,
                        pa_apply, pa_apply_local, pa_diagonal, pa_setup, reset_multiply_count)

__all__ = [
    "CudaError", "InvalidArgument", "LogicError", "TfemError", "TfemRuntimeError", "lib",
    "SO_PATH", "DIFFUSION", "MASS", "BilinearForm", "CgResult", "ConstrainedOperator",
    "Device", "FeSpace", "LinearForm", "LinearOperator", "PaData", "SparseOperator", "Vector", "cg_solve",
    "cg_solve_host", "compute_l2_error", "project_coefficient", "count_multiplies", "default_device", "multiply_count", "pa_apply",
    "pa_apply_local", "pa_diagonal", "pa_setup", "reset_multiply_count",
]
