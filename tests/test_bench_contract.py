"""bench.py contract checks that need no GPU: the reference arm (the CPU oracle, the one place besides
cpu_baseline where bench.py may execute oracle/) prints one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _reference_line(config):
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", config, "--steps", "1",
                          "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line_small_config():
    d = _reference_line("C1")
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "gates/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "C1"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_both_arms_share_the_headline_metric():
    src = open(os.path.join(ROOT, "bench.py")).read()
    # the C4 metric string is defined once and printed by both arms
    assert src.count("C4_METRIC = ") == 1
    assert '"metric": C4_METRIC' in src
    assert 'metric = C4_METRIC if args.config == "C4"' in src
