"""Times sv_expectation and sv_expectation_with_grad pieces at n qubits (CUDA events)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ham = W.jw_hamiltonian(n, 50, 3030)
pa = P.PauliArray(ham)
sv = P.StateVector(n)
w = W.random_circuit(n, 2, seed=1)
sv.apply_circuit(w.gates)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    E = P.sv_expectation(sv.h, pa)
    dt = time.perf_counter() - t0
    st = sv.stats()
    print(f"expectation n={n}: {dt*1e3:.2f} ms E={E:.12f} passes_total={st['expectation_passes']}")
sv.close()
