"""Small end-to-end workload for compute-sanitizer runs (memcheck / racecheck / synccheck): every
kernel family at sizes that exercise multi-tile, dense / sequential / adjoint-dense stages."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

n = 13
w = W.random_circuit(n, 4, seed=1)
sv = P.StateVector(n)
sv.apply_circuit(w.gates)
cp = W.random_complex(n, 3, seed=2, n_params=3, extra_kinds=("MAT2", "PS", "SWAP"))
sv.apply_circuit(cp.gates, cp.params)
ham = W.jw_hamiltonian(n, 20, 3) + W.random_hamiltonian(n, 5, 4)
print("E", sv.expectation(ham))
hea = W.hea(n, 2, seed=5, nterms=10)
print("grad", sv.expectation_with_grad(hea.gates, hea.params, hea.ham)[0])
print("sample", sv.sample(list(range(n)), 64, seed=1)[:4])
sv.close()
small = P.StateVector(4)
c1 = W.c1_ghz_rx()
print("batch", small.expectation_with_grad_batch(c1.gates, np.tile(c1.params, (4, 1)), c1.ham)[0])
small.close()
dm = P.DensityMatrix(5)
dm.apply_circuit(W.random_complex(5, 3, seed=6).gates)
print("dm", dm.expectation(W.random_hamiltonian(5, 4, 7)))
dm.close()
vs = P.StateVector(12, handle=P.sv_create_virtual_shards(12, 4))
vs.apply_circuit(W.random_circuit(12, 3, seed=8).gates)
print("shards", vs.expectation(W.jw_hamiltonian(12, 10, 9)))
vs.close()
print("done")
