"""Times one tiled Pauli pass at 30 qubits for Hamiltonians of controlled shape (E only):
Z0 alone (diagonal entry, one term), k hopping terms X_a Z.. X_b confined to one tile, and the
20-term diagonal group of the JW generator; prints ms per pass (CUDA events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
sv = P.StateVector(n)
w = W.random_circuit(n, 2, seed=1)
sv.apply_circuit(w.gates)
rng = np.random.default_rng(5)
qs = [3, 7, 11, 13, 17, 19, 23, 25, 27]  # 9 qubits + the low 3 = one tile
def hop(a, b, kind):
    t = {a: kind, b: kind}
    for q in range(a + 1, b):
        t[q] = "Z"
    return t
shapes = {"Z0": [(1.0, {0: "Z"})],
          "diag20": [(c, t) for c, t in W.jw_hamiltonian(n, 50, 3030) if all(p == "Z" for p in t.values())]}
for k in (1, 2, 4, 6, 8, 12):
    terms = []
    for i in range(k):
        a, b = sorted(rng.choice(qs, 2, replace=False))
        terms.append((rng.uniform(-1, 1), hop(int(a), int(b), "XY"[i % 2])))
    shapes[f"hop{k}"] = terms
for name, ham in shapes.items():
    pa = P.PauliArray(ham)
    P.sv_expectation(sv.h, pa)
    P.sv_reset_stats(sv.h)
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        P.sv_expectation(sv.h, pa)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    st = sv.stats()
    print(f"{name:8s} terms={len(ham):3d} passes={st['expectation_passes'] / 5:.0f} {ms:.2f} ms/call", flush=True)
sv.close()
