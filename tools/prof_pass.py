"""Profiling driver: runs a C4-shaped random circuit (Haar 1q + CZ bricks) at n qubits through
sv_apply_circuit a few times so `ncu -k regex:k_pass` can capture a steady-state pass; also
prints CUDA-event timings per circuit and the plan shape. Usage: python tools/prof_pass.py [n] [depth]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mode = sys.argv[3] if len(sys.argv) > 3 else "fwd"
w = W.random_circuit(n, depth, seed=3040)
plan = P.sv_plan_info(n, w.gates)
print(f"n={n} depth={depth} gates={len(w.gates)} passes={len(plan)} stages={sum(p['n_stages'] for p in plan)}")
sv = P.StateVector(n)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
P.sv_set_stream(sv.h, stream.cuda_stream)
ga = P.GateArray(w.gates)
if mode == "grad":
    wg = W.hea(n, 2, seed=3030)
    gag, pag = P.GateArray(wg.gates), P.PauliArray(wg.ham)
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if mode == "grad":
        P.sv_expectation_with_grad(sv.h, gag, wg.params, pag)
    else:
        P.sv_apply_circuit(sv.h, ga, w.params)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"iter {it}: {ms:.3f} ms  ({len(w.gates) / ms * 1e3:.1f} gates/s, {ms / len(plan):.3f} ms/pass, "
          f"{32 * 2**n / (ms / len(plan) / 1e3) / 1e9:.1f} GB/s per pass)")
sv.close()
