"""Summarise ncu outputs into text files for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches gpurun_out/launches.csv   > profiles/rNN_launches.txt
  python tools/ncu_summary.py full     gpurun_out/prof_pass30.ncu-rep > profiles/rNN_ncu_pass30_full.txt
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    total = 0.0
    n = 0
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "").strip()
        v = float(r[iv].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        v *= scale
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        total += v
        n += 1
    print(f"# ncu launch list: {n} launches, {total:.3f} ms total (cold-cache, serialised; compare SHARES)")
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>12s} {'share':>7s}")
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name[:60]:60s} {c:8d} {t:12.3f} {100 * t / total:6.1f}%")


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    want = [
        "Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
    ]
    for r in rows[2:]:
        print("# ncu --set full capture (one launch)")
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                print(f"{w:80s} {r[i]:>20s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h))
                except ValueError:
                    pass
        print("# top warp stall reasons (warps per issue)")
        for v, h in sorted(stalls, reverse=True)[:8]:
            print(f"{h:80s} {v:20.3f}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
