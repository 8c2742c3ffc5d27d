"""bench.py's reference arm on CPU (the driver runs `bench.py --impl
reference`): one JSON line with the contract's keys, for cfg 2 (the
reference's own run_solve from oracle/_ref) and the 3D workload (the 3D
oracle port)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", *args], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_cfg2():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libwost_ref.so")):
        pytest.skip("oracle/_ref not built")
    d = _run("--workload", "cfg2", "--ref-rounds", "2")
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["metric"] == "guided WoSt walks/sec" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_cfg4():
    d = _run("--workload", "cfg4", "--ref-rounds", "2")
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port"
    # the cfg 2 block: the reference's own run_solve
    assert d["cfg2"]["cpu_baseline"]["kind"] == "reference" and d["cfg2"]["value"] > 0
