"""Runs a BASELINE config's gradient evaluation a few times (for ncu launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = W.config(cfg)
sv = P.StateVector(w.n)
ga, pa = P.GateArray(w.gates), P.PauliArray(w.ham)
for _ in range(reps):
    E, g = P.sv_expectation_with_grad(sv.h, ga, w.params, pa)
print(cfg, E, sv.stats())
