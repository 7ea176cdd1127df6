"""CPU: bench.py's driver contract where it can run without a GPU -- the
reference arm (`--impl reference`: the unmodified reference, oracle/_ref, on
the host cores) prints one JSON line with the contract keys, and `--gpus N`
on a box with fewer GPUs fails loudly instead of running one rank."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASELINE = json.loads((ROOT / "BASELINE.json").read_text())


def _bench(*args, timeout=300):
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_json_line(oracle_built):
    out = _bench("--impl", "reference", "--cells", "96", "--steps", "1", "--warmup", "1")
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference"
    assert d["metric"] == BASELINE["metric"]
    assert d["unit"] == "GDOF/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["dim"] == 2 and d["config"]["order"] == 3
    assert d["dtype"] == "f64" and d["data"] == "synthetic"


def test_more_gpus_than_the_box_has_is_an_error():
    import torch
    want = max(2, torch.cuda.device_count() + 1) # --gpus 1 is the plain single-rank run
    out = _bench("--gpus", str(want), "--steps", "1", "--warmup", "1", timeout=120)
    assert out.returncode != 0
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert "error" in d and f"--gpus {want}" in d["error"]
