"""C4 circuit time at 30q for forced tile sizes (SV_OPT_TILE_QUBITS) and CTA counts."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

w = W.config("C4")
ga = P.GateArray(w.gates)
sv = P.StateVector(w.n)
for k in [int(x) for x in sys.argv[1:]]:
    sv.set_option(P.SV_OPT_TILE_QUBITS, k)
    sv.reset()
    P.sv_apply_circuit(sv.h, ga, w.params)
    torch.cuda.synchronize()
    P.sv_reset_stats(sv.h)
    t0 = time.perf_counter()
    for _ in range(2):
        sv.reset()
        P.sv_apply_circuit(sv.h, ga, w.params)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 2
    st = sv.stats()
    print(f"tile {k}: {dt * 1e3:.1f} ms, passes {st['gate_passes'] / 2:.0f}, {len(w.gates) / dt:.0f} gates/s", flush=True)
