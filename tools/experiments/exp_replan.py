"""Gradient evaluations with parameters that change every call (an optimiser loop) vs fixed
parameters (plan-cache hits): measures the host re-planning cost per evaluation."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

for cfg in sys.argv[1:] or ["C2", "C3", "C4g"]:
    w = W.config(cfg)
    ga, pa = P.GateArray(w.gates), P.PauliArray(w.ham)
    sv = P.StateVector(w.n)
    reps = 10 if w.n < 26 else 3
    P.sv_expectation_with_grad(sv.h, ga, w.params, pa)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        P.sv_expectation_with_grad(sv.h, ga, w.params, pa)
    fixed = (time.perf_counter() - t0) / reps
    rng = np.random.default_rng(0)
    t0 = time.perf_counter()
    for _ in range(reps):
        p = w.params + 1e-3 * rng.standard_normal(len(w.params))
        P.sv_expectation_with_grad(sv.h, ga, p, pa)
    moving = (time.perf_counter() - t0) / reps
    print(f"{cfg}: fixed params {1e3 * fixed:.2f} ms/eval, changing params {1e3 * moving:.2f} ms/eval", flush=True)
    sv.close()
