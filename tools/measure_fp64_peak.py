"""Measures the FP64 peaks used as bench.py's roofline denominators on THIS box and writes
profiles/fp64_peak.json (committed): DFMA (CUDA cores), DMMA (mma.sync m8n8k4 f64) and both mixed
(tools/microbench/fp64_mix.cu, best of 5 runs each), with the SM clock sampled by nvidia-smi while
it runs. Usage (on the GPU box): python tools/measure_fp64_peak.py"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "microbench", "fp64_mix.cu")
BIN = "/tmp/fp64_mix"


def main():
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", BIN, SRC])
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,power.draw",
                            "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    best = {}
    t0 = time.time()
    for _ in range(5):
        out = subprocess.run([BIN], capture_output=True, text=True, check=True).stdout
        for line in out.splitlines():
            if line.startswith("{"):
                d = json.loads(line)
                best[d["mode"]] = max(best.get(d["mode"], 0.0), d["tflops"])
    smi.terminate()
    rows = []
    for line in smi.communicate(timeout=5)[0].splitlines():
        p = [x.strip() for x in line.split(",")]
        try:
            rows.append((float(p[0]), float(p[1]), float(p[2])))
        except (ValueError, IndexError):
            pass
    load = [r for r in rows if r[2] > 300.0] or rows
    clk = sorted(r[0] for r in load)
    rec = {"dfma_tflops": best.get("dfma"), "dmma_tflops": best.get("dmma"), "mixed_tflops": best.get("mixed"),
           "peak_tflops": max(best.values()), "source": "tools/microbench/fp64_mix.cu, best of 5 (tools/measure_fp64_peak.py)",
           "sm_mhz_median_under_load": clk[len(clk) // 2] if clk else None,
           "sm_max_mhz": max(r[1] for r in rows) if rows else None, "samples": len(rows),
           "seconds": round(time.time() - t0, 1), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    path = os.path.join(ROOT, "gpurun_out", "fp64_peak.json") if len(sys.argv) < 2 else sys.argv[1]
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
