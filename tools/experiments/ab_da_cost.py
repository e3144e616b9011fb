"""A/B of the adjoint-dense-stage threshold (SV_OPT_ADJOINT_DENSE_COST) on a gradient config:
grad evals/s with fixed parameters (plans cached), CUDA-event timed."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1]
for cost in [int(x) for x in sys.argv[2:]]:
    w = W.config(cfg)
    sv = P.StateVector(w.n)
    sv.set_option(P.SV_OPT_ADJOINT_DENSE_COST, cost)
    ga, pa = P.GateArray(w.gates), P.PauliArray(w.ham)
    for _ in range(2):
        P.sv_expectation_with_grad(sv.h, ga, w.params, pa)
    torch.cuda.synchronize()
    reps = 3 if w.n >= 28 else 10
    t0 = time.perf_counter()
    for _ in range(reps):
        E, g = P.sv_expectation_with_grad(sv.h, ga, w.params, pa)
    dt = (time.perf_counter() - t0) / reps
    print(f"{cfg} da_cost={cost}: {1 / dt:.2f} grad evals/s ({dt * 1e3:.1f} ms)", flush=True)
    sv.close()
