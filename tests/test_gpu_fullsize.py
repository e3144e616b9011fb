"""Parity at BASELINE.json's full sizes in the launch configuration bench.py times (30 qubits,
16 GiB state, the default plan), where the oracle cannot run: properties that hold at any size.

* C4 followed by its inverse returns |0...0> exactly (a mirror circuit: every amplitude checked).
* The energy of C4's state through sv_expectation (E-only Pauli passes) equals the energy the
  gradient path reports (lambda = H psi passes + Re<psi|lambda>): two independent kernel paths.
* C4g's adjoint gradient at 30q equals the parameter-shift rule (two extra evaluations through the
  forward and expectation kernels per parameter) on sampled parameters (§4: the
  adjoint method computes the same derivative as the shift rule, reading 8 of DESIGN.md).
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2406_17248_b200 as P
    return P


def test_c4_mirror_30q(P):
    w = W.config("C4")
    sv = P.StateVector(w.n)
    sv.apply_circuit(w.gates)
    sv.apply_circuit(W.mirror(w.gates)[len(w.gates):])
    psi = sv.get_state()
    sv.close()
    assert abs(psi[0] - 1.0) < 1e-10
    assert np.max(np.abs(psi[1:])) < 1e-10


def test_c4_energy_two_paths_30q(P):
    w = W.config("C4")
    sv = P.StateVector(w.n)
    sv.apply_circuit(w.gates)
    e1 = sv.expectation(w.ham)
    sv.reset()
    e2, g = sv.expectation_with_grad(w.gates, np.zeros(0), w.ham)
    sv.close()
    assert g.size == 0
    assert abs(e1 - e2) < 1e-9


def test_c4g_gradient_vs_shift_rule_30q(P):
    w = W.config("C4g")
    sv = P.StateVector(w.n)
    E, g = sv.expectation_with_grad(w.gates, w.params, w.ham)
    rng = np.random.default_rng(30)
    for k in rng.choice(len(w.params), size=3, replace=False):
        vals = []
        for s in (+1, -1):
            p = np.array(w.params, dtype=np.float64)
            p[k] += s * np.pi / 2
            sv.reset()
            sv.apply_circuit(w.gates, p)
            vals.append(sv.expectation(w.ham))
        shift = 0.5 * (vals[0] - vals[1])  # R_P(theta) = exp(-i theta P / 2): exact two-term rule
        assert abs(g[k] - shift) < 1e-9, (k, g[k], shift)
    sv.reset()
    sv.apply_circuit(w.gates, w.params)
    assert abs(sv.expectation(w.ham) - E) < 1e-9
    sv.close()
