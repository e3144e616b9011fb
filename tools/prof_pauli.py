"""Times the tiled Pauli passes at n qubits: sv_expectation (E-only passes) and lambda = H psi
(sv_expectation_with_grad of an empty circuit: lambda passes + Re<psi|lambda>, no sweep)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 3030
ham = W.jw_hamiltonian(n, 50, seed)
pa = P.PauliArray(ham)
sv = P.StateVector(n)
w = W.random_circuit(n, 2, seed=1)
sv.apply_circuit(w.gates)
torch.cuda.synchronize()
for label, fn in (("E-only", lambda: P.sv_expectation(sv.h, pa)),
                  ("lambda", lambda: P.sv_expectation_with_grad(sv.h, P.GateArray([]), np.zeros(0), pa)[0])):
    fn()
    P.sv_reset_stats(sv.h)
    reps = 5
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        E = fn()
    dt = (time.perf_counter() - t0) / reps
    st = sv.stats()
    passes = st["expectation_passes"] / reps
    byt = st["algorithmic_bytes"] / reps
    print(f"{label} n={n}: {dt*1e3:.2f} ms/call  passes={passes:.0f}  {dt*1e3/passes:.2f} ms/pass  "
          f"alg bytes {byt/1e9:.2f} GB -> {byt/dt/1e9:.0f} GB/s  E={E:.12f}", flush=True)
sv.close()
