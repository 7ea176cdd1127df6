"""The drop-in as a maintainer would ship it: the reference library
(/root/reference/proj) compiled with -DTENSORFEM_B200 -- its own forms.cpp /
solvers.cpp / vector.hpp patched by integration/patch/tensorfem_b200.patch to
route the PA operator, the diagonal, the constrained operator and cg_solve
through libtfem_cuda.so -- running the reference's OWN test programs:

* acceptance (tests/acceptance_main.cpp): criteria 1-10,
  one PASS/FAIL line each, exit code = failures;
* the doctest unit suites test_quadrature ... test_driver
  (tests/CMakeLists.txt:1-19) over integration/doctest/doctest.h;
* bench_dropin: the BP3 solve through form_linear_system + cg_solve with host
  Vectors (the e2e leg bench.py reports as `e2e_dropin`).

Binaries are built here (integration/Makefile; the reference sources are
needed at build time only) and travel to the GPU box."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "integration" / "_build" / "bin"
UNIT = ["test_quadrature", "test_basis", "test_linalg", "test_mesh", "test_ncmesh",
        "test_fespace", "test_forms", "test_driver"]


def _run(name, *args, timeout=900):
    exe = BIN / name
    assert exe.exists(), f"{exe} not built: run `make -C integration` (needs /root/reference)"
    return subprocess.run([str(exe), *map(str, args)], capture_output=True, text=True,
                          timeout=timeout)


def test_dropin_binaries_link_the_device_library():
    """CPU: every drop-in program is built and resolves the C ABI from
    libtfem_cuda.so (no host fallback linked in)."""
    if not (BIN / "acceptance").exists() and not Path("/root/reference/proj").exists():
        pytest.skip("drop-in binaries are built where the reference sources exist")
    for name in ["acceptance", "bench_dropin", *UNIT]:
        assert (BIN / name).exists(), name
    # the programs that assemble forms or solve resolve the hot path from the
    # device library (the linker drops it from suites that never touch it)
    for name in ["acceptance", "bench_dropin", "test_forms", "test_linalg", "test_driver"]:
        exe = BIN / name
        undef = subprocess.run(["nm", "-D", "--undefined-only", str(exe)], capture_output=True,
                               text=True).stdout
        assert "tfem_host_alloc" in undef and "tfem_cg_solve" in undef, name
        ldd = subprocess.run(["ldd", str(exe)], capture_output=True, text=True).stdout
        assert "libtfem_cuda.so" in ldd, name


@pytest.mark.gpu
def test_reference_acceptance_on_the_device(dev):
    out = _run("acceptance")
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith(("PASS", "FAIL"))]
    assert len(lines) == 10 and all(l.startswith("PASS") for l in lines), lines


@pytest.mark.gpu
@pytest.mark.parametrize("suite", UNIT)
def test_reference_unit_suite_on_the_device(dev, suite):
    out = _run(suite)
    print(out.stdout[-2000:], out.stderr[-4000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-6000:]
    assert "| 0 failed" in out.stdout


@pytest.mark.gpu
def test_bench_dropin_small(dev):
    out = _run("bench_dropin", 64, 3, 20, 2, 1)
    assert out.returncode == 0, out.stdout + out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["iterations"] == 20
    assert line["device_cartesian"] is True
    assert line["value"] > 0
