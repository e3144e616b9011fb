"""complex64 relative state error vs the oracle on C4-shaped circuits (depth 8), per SV_OPT_C64_SPLIT."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

for n in (19, 21):
    w = W.random_circuit(n, 8, seed=100 + n)
    ref = oracle.apply_circuit(n, w.gates)
    out = []
    for split in (3, 0):
        sv = P.StateVectorC64(n)
        sv.set_option(P.SV_OPT_C64_SPLIT, split)
        sv.apply_circuit(w.gates)
        out.append(float(np.linalg.norm(sv.get_state() - ref) / np.linalg.norm(ref)))
        sv.close()
    print(f"n={n} rel_err split3={out[0]:.3e} fp64={out[1]:.3e}", flush=True)
