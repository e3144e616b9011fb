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


def test_reference_arm_is_labelled_as_a_sample():
    """The oracle arm times a bounded sample (first G gates, no <H>), not the full C4 step: it prints
    its own metric string with the sample size, same_config = false, and the shared unit gates/s."""
    d = _reference_line("C1")
    assert d["same_config"] is False and "first" in d["sample"]
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert src.count("C4_METRIC = ") == 1 and '"metric": C4_METRIC' in src
    assert "oracle sample" in d["metric"] and d["metric"] != "gates/sec (30q random circuit C4 evolution + 50-term <H>), SV GB/s, grad evals/sec"


def test_gpus_flag_fails_loudly_without_enough_gpus():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks, but only when the box has
    2 GPUs: here (no GPU) it must exit non-zero instead of reporting a smaller run as N = 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "0"], cwd=ROOT,
                         capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 2, (out.returncode, out.stdout[-500:], out.stderr[-500:])
    assert "--gpus 2" in out.stderr and not [l for l in out.stdout.splitlines() if l.startswith("{")]


def test_world_size_must_match_gpus_flag():
    env = dict(os.environ, WORLD_SIZE="4", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "0"], cwd=ROOT,
                         capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=4" in (out.stderr + out.stdout)
