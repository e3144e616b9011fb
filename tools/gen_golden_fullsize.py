"""Writes tests/golden/fullsize_<case>.npz: oracle results for the bench configs at (or near) their
full sizes, for the `-m gpu` parity tests in tests/test_gpu_fullsize_oracle.py.

Calls ONLY oracle/ (the plain C CPU oracle) and workloads/ (the seeded input generators); nothing
here touches the CUDA path. The GPU box's pytest run compares against these stored values, so the
tests take seconds instead of the oracle's tens of minutes (SURVEY.md §8(d) "Oracle timing": 30q
full depth is ~20 min of host time per evaluation).

Cases (§7.1 P:579 random circuits in double precision, §7.2
P:604-606 QAOA with the adjoint method):
  C3      24q QAOA p=8, seeded angles (BASELINE configs[2]): E and all 16 gradients
  C3dc    the DC-QAOA variant (reading c2.20): E and all 24 gradients
  C4_26   the C4 generator (Haar 1q + CZ bricks, depth 40, seed 3040) at 26q with the 50-term JW H
          (seed 3030): sampled amplitudes and E
  C4_30d4 the first 4 layers of C4 itself (30q, 178 gates): sampled amplitudes and E
  C4g_26  the C4g generator (HEA, 2 layers, seed 3030) at 26q: E and all 104 gradients

Usage: python tools/gen_golden_fullsize.py CASE [CASE ...]   (OMP_NUM_THREADS = cores)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
N_SAMPLED = 16384  # sampled amplitude indices (plus indices 0..255)


case_workload = W.fullsize_case


def sampled_indices(n, seed):
    rng = np.random.default_rng(seed)
    idx = np.concatenate([np.arange(min(256, 1 << n)), rng.integers(0, 1 << n, N_SAMPLED)])
    return np.unique(idx).astype(np.int64)


def run(name):
    w = case_workload(name)
    t0 = time.time()
    out = {"n": np.int64(w.n), "n_gates": np.int64(len(w.gates))}
    if name in ("C3", "C3dc", "C4g_26"):
        E, g = oracle.adjoint_grad(w.n, w.gates, w.params, w.ham)
        out["E"] = np.float64(E)
        out["grad"] = np.asarray(g, dtype=np.float64)
        out["params"] = np.asarray(w.params, dtype=np.float64)
    else:
        psi = oracle.apply_circuit(w.n, w.gates)
        idx = sampled_indices(w.n, seed=w.n * 1000 + len(w.gates))
        out["idx"] = idx
        out["amps"] = psi[idx].copy()
        out["norm2"] = np.float64(np.vdot(psi, psi).real)
        E, Ei = oracle.expectation(psi, w.ham)
        out["E"] = np.float64(E)
        out["E_im"] = np.float64(Ei)
        del psi
    out["oracle_seconds"] = np.float64(time.time() - t0)
    out["omp_threads"] = np.int64(int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)))
    path = os.path.join(GOLDEN, f"fullsize_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: n={w.n} gates={len(w.gates)} E={float(out['E']):.15f} in {time.time() - t0:.1f} s -> {path}",
          flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:]:
        run(c)
