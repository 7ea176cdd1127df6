"""CPU: the C-ABI library loads and exports every symbol include/tfem_cuda.h
declares (no compute calls -- there is no GPU here)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tfem_cuda.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tfem_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("tfem_pa_setup", "tfem_pa_apply_local", "tfem_pa_diagonal", "tfem_cg_solve",
              "tfem_restriction_create", "tfem_operator_mult", "tfem_cg_solve_host"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1911_09220_b200 import abi
    L = abi.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    # and the Python binding covers the whole header
    assert set(declared_symbols()) <= set(abi.exported_symbols())


def test_library_is_sm100a():
    so = ROOT / "paper_1911_09220_b200" / "libtfem_cuda.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_errors_without_a_device_are_status_codes():
    """Context creation with no GPU returns a status (never a crash)."""
    from paper_1911_09220_b200 import abi
    L = abi.lib()
    h = C.c_void_p()
    rc = L.tfem_ctx_create(0, C.byref(h))
    if rc == 0:
        L.tfem_ctx_destroy(h)
        pytest.skip("a device is present")
    assert rc in (abi.CUDA_ERROR, abi.INVALID_ARGUMENT)
    assert L.tfem_last_error()


def test_host_tables_match_reference(oracle_built):
    """The library's host-side 1D tables (quadrature + Basis1D) are
    bit-identical to the reference (quadrature.cpp, basis.cpp)."""
    import numpy as np
    from paper_1911_09220_b200 import abi
    from oracle.pyoracle import Ref, Orc
    chk = Ref if Ref.available() else Orc
    L = abi.lib()
    for n in range(2, 11):
        for rule in (0, 1):
            x = np.zeros(n)
            w = np.zeros(n)
            abi.check(L.tfem_quadrature(rule, n, x.ctypes.data_as(abi.dp),
                                        w.ctypes.data_as(abi.dp)))
            xr, wr = chk.rule(n, lobatto=rule == 1)
            assert (x == xr).all() and (w == wr).all()
    for p in range(1, 9):
        for nq, rule in ((p + 2, 0), (p + 1, 1)):
            B = np.zeros((nq, p + 1))
            G = np.zeros((nq, p + 1))
            abi.check(L.tfem_eval_matrices(p, 0, nq, rule, B.ctypes.data_as(abi.dp),
                                           G.ctypes.data_as(abi.dp)))
            Br, Gr = chk.eval_matrices(p, nq, 0, rule)
            assert (B == Br).all() and (G == Gr).all()


def test_invalid_arguments_map_to_status(oracle_built):
    import numpy as np
    from paper_1911_09220_b200 import abi
    L = abi.lib()
    x = np.zeros(1)
    assert L.tfem_quadrature(0, 0, x.ctypes.data_as(abi.dp), None) == abi.INVALID_ARGUMENT
    assert b"gauss_legendre" in L.tfem_last_error()
    assert L.tfem_quadrature(1, 1, x.ctypes.data_as(abi.dp), None) == abi.INVALID_ARGUMENT
