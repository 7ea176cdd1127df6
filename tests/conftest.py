"""Shared fixtures.  `-m gpu` tests need a B200 and the built libtfem_cuda.so;
everything else runs on the CPU (oracle, host logic, ABI surface)."""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtfem_cuda.so")
    config.addinivalue_line("markers", "slow: larger CPU cases")


@pytest.fixture(scope="session")
def oracle_built():
    """Builds the CPU checkers (restatement always; reference when present)."""
    from oracle import pyoracle
    if not pyoracle.ORC_SO.exists() or (Path("/root/reference").exists()
                                        and not pyoracle.REF_SO.exists()):
        pyoracle.build()
    return pyoracle


def _device(numerics):
    """Device 0.  The library import is unconditional: on a GPU box a missing
    libtfem_cuda.so is an error, never a skip."""
    from paper_1911_09220_b200 import CudaError, Device, InvalidArgument
    try:
        return Device(0, numerics=numerics)
    except (CudaError, InvalidArgument) as e:  # no device in this container
        pytest.skip(f"no CUDA device: {e}")


@pytest.fixture(scope="session")
def dev():
    """Bit-exact numerics (the reference's operation order): `==` parity."""
    d = _device("reference")
    yield d
    d.close()


@pytest.fixture(scope="session")
def dev_fma():
    """The default numerics (fused multiply-adds): 1e-12 parity."""
    d = _device("fma")
    yield d
    d.close()
