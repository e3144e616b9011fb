"""NEXT-3 complex64 mode ("single-precision and double-precision
simulation modes") vs the complex128 CPU oracle.

Tolerances are RELATIVE to the state (an absolute 1e-4 on amplitudes of size 2^(-n/2) would let a
5% error per amplitude through). Derivation: a stored complex64 value carries 2^-24 ~ 6e-8
relative rounding; a dense stage's 16-term products use the 3-product TF32 hi/lo split
(hi = v rounded to 10 mantissa bits, lo = v - hi exact with |lo| <= 2^-11 |v|, read by the tensor
core to 10 bits) whose per-product error is ~2^-21 ~ 5e-7 relative, FP32 accumulation adds ~2^-24 per term. Over the <= ~30 stages of
these circuits, independent errors add in quadrature: ||d psi||_2 / ||psi||_2 ~ sqrt(30) * 6e-7
~ 3e-6, so REL = 1e-5 holds with margin. A single hi x hi TF32 product (2^-11 ~ 5e-4 relative)
gives ~1e-3: `test_c64_tolerance_detects_single_tf32` shows the bound catches it. Energies are
FP64-accumulated over complex64 inputs: |dE| <= 2 * sum|c_t| * ||d psi||_2.
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
REL = 1e-5   # ||psi_gpu - psi_oracle||_2 <= REL * ||psi_oracle||_2 (module docstring)


def rel_err(got, ref):
    return float(np.linalg.norm(got - ref) / np.linalg.norm(ref))


def e_tol(ham):
    return 2.0 * REL * sum(abs(c) for c, _ in ham) + 1e-12


@pytest.fixture(scope="module")
def P():
    import paper_2406_17248_b200 as P
    return P



@pytest.mark.parametrize("n,depth,native", [(9, 6, True), (11, 8, True), (14, 10, False), (17, 12, True),
                                            (19, 8, True)])
def test_c64_dense_circuit(P, n, depth, native):
    """C4-shaped circuits (Haar 1q + CZ bricks: dense FP32 stages) over several tiles. States
    whose planner picks tiles below 2^8 amplitudes (n = 12..16) run on the complex128 copy."""
    w = W.random_circuit(n, depth, seed=100 + n)
    ref = oracle.apply_circuit(n, w.gates)
    sv = P.StateVectorC64(n)
    P.sv_reset_stats(sv.h)
    sv.apply_circuit(w.gates)
    got = sv.get_state()
    st = P.sv_get_stats(sv.h)
    sv.close()
    assert rel_err(got, ref) <= REL
    # native complex64 passes: 16 bytes per amplitude per pass, no widen/narrow traffic
    if native:
        assert st["algorithmic_bytes"] == pytest.approx(16.0 * (1 << n) * st["gate_passes"])
    else:
        assert st["algorithmic_bytes"] > 16.0 * (1 << n) * st["gate_passes"]


@pytest.mark.parametrize("n", [9, 12, 15])
def test_c64_controlled_random(P, n):
    """The paper's complex random circuits with controls (sequential + dense stages), a random
    start state."""
    w = W.random_complex(n, 6, seed=n, extra_kinds=("PS", "MAT1", "MAT2", "SWAP", "XLIKE", "ZLIKE"))
    psi0 = W.random_state(n, seed=n)
    ref = oracle.apply_circuit(n, w.gates, psi0=psi0)
    sv = P.StateVectorC64(n)
    sv.set_state(psi0)
    sv.apply_circuit(w.gates)
    got = sv.get_state()
    sv.close()
    assert rel_err(got, ref) <= REL


@pytest.mark.parametrize("n", [10, 14])
def test_c64_expectation(P, n):
    w = W.random_circuit(n, 4, seed=7 + n)
    ham = W.jw_hamiltonian(n, 30, seed=n) + W.random_hamiltonian(n, 6, seed=n + 1)
    psi = oracle.apply_circuit(n, w.gates)
    ref = oracle.expectation(psi, ham)[0]
    sv = P.StateVectorC64(n)
    sv.apply_circuit(w.gates)
    E = sv.expectation(ham)
    sv.close()
    assert abs(E - ref) <= e_tol(ham)


def test_c64_promoted_paths(P):
    """Operations without a complex64 kernel run on a complex128 copy: small states (tiles below
    2^9 amplitudes), Pauli strings wider than a tile, gradients, sampling."""
    # small n: complex128 passes on the scratch copy, rounded back
    w = W.random_complex(5, 4, seed=3)
    sv = P.StateVectorC64(5)
    sv.apply_circuit(w.gates)
    assert rel_err(sv.get_state(), oracle.apply_circuit(5, w.gates)) <= REL
    sv.close()
    # wide x-mask (X on every qubit of 16)
    n = 16
    w = W.random_circuit(n, 3, seed=5)
    ham = [(0.7, {q: "X" for q in range(n)}), (-0.4, {0: "Z", 15: "Z"})]
    sv = P.StateVectorC64(n)
    sv.apply_circuit(w.gates)
    psi = oracle.apply_circuit(n, w.gates)
    assert abs(sv.expectation(ham) - oracle.expectation(psi, ham)[0]) <= e_tol(ham)
    sv.close()
    # gradient on a complex64 handle (complex128 copy of the complex64 start state)
    h = W.hea(10, 2, seed=4, nterms=12)
    sv = P.StateVectorC64(10)
    E, g = sv.expectation_with_grad(h.gates, h.params, h.ham)
    Er, gr = oracle.adjoint_grad(10, h.gates, h.params, h.ham)
    sv.close()
    # the gradient runs in complex128 on the widened complex64 start state |0..0> (exact)
    assert abs(E - Er) <= 1e-9
    assert np.max(np.abs(g - gr)) <= 1e-9


def test_c64_sampling_and_reset(P):
    n = 12
    w = W.random_circuit(n, 3, seed=9)
    sv = P.StateVectorC64(n)
    sv.apply_circuit(w.gates)
    shots = sv.sample(list(range(n)), 2000, seed=3)
    assert shots.shape == (2000,) and shots.min() >= 0 and shots.max() < (1 << n)
    sv.reset()
    st = sv.get_state()
    assert st[0] == 1.0 and np.count_nonzero(st) == 1
    sv.close()


def test_c64_matches_c128_path(P):
    """Same circuit and H through both precisions: agreement within the complex64 tolerance."""
    n = 16
    w = W.random_circuit(n, 8, seed=21)
    ham = W.jw_hamiltonian(n, 40, seed=2)
    a = P.StateVector(n)
    b = P.StateVectorC64(n)
    a.apply_circuit(w.gates)
    b.apply_circuit(w.gates)
    assert rel_err(b.get_state(), a.get_state()) <= REL
    assert abs(a.expectation(ham) - b.expectation(ham)) <= e_tol(ham)
    a.close()
    b.close()


def test_c64_tolerance_detects_single_tf32(P):
    """The relative bound has the power to catch a precision bug: the same 19-qubit dense circuit
    with the dense stages reduced to the single hi x hi TF32 product (SV_OPT_C64_SPLIT = 1, ~2^-11
    relative per product) exceeds REL by orders of magnitude, while the default 3-product split
    stays inside it."""
    n = 19
    w = W.random_circuit(n, 8, seed=100 + n)
    ref = oracle.apply_circuit(n, w.gates)
    errs = {}
    for split in (3, 1):
        sv = P.StateVectorC64(n)
        sv.set_option(P.SV_OPT_C64_SPLIT, split)
        sv.apply_circuit(w.gates)
        errs[split] = rel_err(sv.get_state(), ref)
        sv.close()
    assert errs[3] <= REL, errs
    assert errs[1] > 10 * REL, errs


@pytest.mark.parametrize("n", [19, 21])
def test_c64_fp64_dense_stages(P, n):
    """SV_OPT_C64_SPLIT = 0: all-dense complex64 passes widen the tile to FP64 and run the Gauss DMMA
    stages of the complex128 kernel (k_pass_dense<float2>), rounding to FP32 once per stage (no
    2^-21 TF32 product error): inside REL and below the TF32 split's error on the same circuit (the
    strict inequality also shows the FP64 path ran: from 19 qubits the planner's tiles hold 2^10+
    amplitudes and passes of dense stages only appear)."""
    w = W.random_circuit(n, 8, seed=100 + n)
    ref = oracle.apply_circuit(n, w.gates)
    errs = {}
    for split in (0, 3):
        sv = P.StateVectorC64(n)
        sv.set_option(P.SV_OPT_C64_SPLIT, split)
        sv.apply_circuit(w.gates)
        errs[split] = rel_err(sv.get_state(), ref)
        sv.close()
    assert errs[0] <= REL, errs
    assert errs[0] < errs[3], errs
