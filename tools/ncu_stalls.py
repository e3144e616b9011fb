"""Summarise an ncu report: key raw metrics, top stall reasons, per-opcode stall/exec shares.

usage: python tools/ncu_stalls.py REPORT.ncu-rep [N_TOP] [LAUNCH_INDEX]"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
sel = ["--launch-skip", sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", rep, *sel, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
for k in ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "gpu__time_duration.sum",
          "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.per_cycle_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "sm__cycles_elapsed.avg.per_second"]:
    print(f"{k:85s} {d.get(k)}")
st = [(float(d[k]), k) for k in h if k.startswith("smsp__average_warps_issue_stalled")
      and k.endswith("per_issue_active.ratio") and d[k] not in ("", "n/a")]
print("# top stall reasons (warps per issue)")
for x in sorted(st, reverse=True)[:8]:
    print(f"{x[1]:85s} {x[0]:.3f}")
src = subprocess.run(["ncu", "-i", rep, *sel, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
# one block per kernel ("Kernel Name" row, header row, instructions): the selected launch's block
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
blk = 0 if len(starts) <= 2 or not sel else min(int(sys.argv[3]), len(starts) - 2)
rows = rows[starts[blk]:starts[blk + 1]]
h = rows[1]
data = rows[2:]
iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(int(r[iS] or 0) for r in data)
tex = sum(int(r[iE] or 0) for r in data)
c, ce = Counter(), Counter()
for r in data:
    t = r[1].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    op = op.split(".")[0]
    c[op] += int(r[iS] or 0)
    ce[op] += int(r[iE] or 0)
print(f"# opcodes: {tex} warp instructions executed, {tot} stall samples")
for op, s in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 16):
    print(f"{op:10s} stall {100 * s / max(1, tot):5.1f}%  exec {ce[op]:>12d} ({100 * ce[op] / max(1, tex):4.1f}%)")

# stall reasons per opcode (samples)
reasons = [x for x in h if x.startswith("stall_") and "(Not Issued)" not in x]
idx = {r: h.index(r) for r in reasons}
agg = {}
for r in data:
    t = r[1].strip().split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
    a = agg.setdefault(op, Counter())
    for k, i in idx.items():
        a[k] += int(r[i] or 0)
print("# stall reasons by opcode (top 4 each)")
for op, _ in c.most_common(8):
    print(f"{op:8s}", ", ".join(f"{k[6:]}={v}" for k, v in agg[op].most_common(4)))
