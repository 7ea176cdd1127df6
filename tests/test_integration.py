"""GPU: the reference's own C++ objects (unmodified library, oracle/_ref)
driving the B200 path through integration/tensorfem_b200.hpp -- the
drop-in as a maintainer would wire it."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "integration" / "_build" / "drop_in_test"


@pytest.mark.gpu
def test_reference_objects_drive_the_device_path(dev):
    if not BIN.exists():
        pytest.skip("drop_in_test not built (needs /root/reference at build time)")
    out = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "[FAIL]" not in out.stdout
    assert out.stdout.count("[PASS]") >= 50
