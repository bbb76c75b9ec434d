"""bench.py's JSON-line contract on the CPU (the reference arm = the oracle on the host cores),
and that our arm refuses to run without a GPU (there is no CPU fallback)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                          text=True, timeout=timeout)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["steps"] == 1 and line["value"] > 0
    assert line["unit"] == line["e2e"]["unit"] and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert "workload" in line["config"] and line["config"]["M"] == 1024 and line["config"]["N"] == 32


@pytest.mark.skipif(os.path.exists("/dev/nvidiactl") or os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_our_arm_has_no_cpu_fallback():
    r = _run(["--steps", "1", "--warmup", "0", "--no-cpu-baseline", "--no-c3-sweep", "--no-e2e"])
    assert r.returncode != 0
    assert not any(l.startswith("{") and '"value"' in l for l in r.stdout.splitlines())
