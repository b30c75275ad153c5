"""Host checks (no GPU) of bench.py's driver contract: the reference arm (the
CPU oracle on a bounded sample, the one leg that runs without a GPU) prints one
JSON line with the BASELINE.json metric and the keys the driver reads, and the
product arm fails loudly instead of falling back to the CPU."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, **env):
    e = dict(os.environ, **env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, cwd=ROOT, timeout=600)


def test_reference_arm_json_contract():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], TQR_REF_BUDGET_S="0.3")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["impl"] == "reference" and d["metric"] == base["metric"]
    assert d["unit"] == "GFLOP/s" and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] and "sample" in d["cpu_baseline"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "configs[2]" in d["config"]["workload"]


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_arm_fails_loudly_without_gpu():
    r = _run(["--steps", "1", "--warmup", "0", "--no-tall"])
    assert r.returncode != 0
    assert not any(ln.startswith("{") for ln in r.stdout.splitlines())
