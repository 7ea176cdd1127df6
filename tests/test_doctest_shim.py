"""CPU: the doctest-compatible shim that runs the reference's unit suites on
the drop-in build (integration/doctest/doctest.h) -- doctest's SUBCASE
traversal (every leaf once per run of the test case, nested subcases) and
the assertion / Approx semantics the suites rely on."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_doctest_shim(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("no g++")
    exe = tmp_path / "selftest"
    subprocess.run(["g++", "-std=c++20", "-O0", f"-I{ROOT / 'integration' / 'doctest'}",
                    str(ROOT / "tests" / "data" / "doctest_shim_selftest.cpp"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    # doctest runs the case once per leaf: A/A1, A/A2, B
    visits = [l for l in out.stdout.splitlines() if l.startswith("visits=")][0]
    assert visits == "visits=[A1][A2][B]", visits
    assert "| 0 failed" in out.stdout
