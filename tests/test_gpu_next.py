"""NEXT-1 batch-mode gradients and NEXT-2 sampling vs the CPU oracle."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
E_TOL = 1e-9


@pytest.fixture(scope="module")
def P():
    import paper_2406_17248_b200 as P
    return P


def test_batch_c1_closed_form(P):
    """C1 at 256 parameter rows in one launch: E = cos t0 cos t1, g = (-sin t0 cos t1, -cos t0 sin t1, 0, 0)."""
    w = W.c1_ghz_rx()
    rows = np.random.default_rng(1).uniform(-np.pi, np.pi, (256, 4))
    sv = P.StateVector(4)
    E, G = sv.expectation_with_grad_batch(w.gates, rows, w.ham)
    sv.close()
    np.testing.assert_allclose(E, np.cos(rows[:, 0]) * np.cos(rows[:, 1]), atol=E_TOL)
    ref = np.stack([-np.sin(rows[:, 0]) * np.cos(rows[:, 1]), -np.cos(rows[:, 0]) * np.sin(rows[:, 1]),
                    np.zeros(256), np.zeros(256)], 1)
    np.testing.assert_allclose(G, ref, atol=E_TOL)


@pytest.mark.parametrize("n", [3, 7, 11, 13])
def test_batch_random_tasks(P, n):
    """Rows of a random controlled circuit (one-launch kernel for n <= 11, row loop above)."""
    w = W.random_complex(n, 5, seed=n, n_params=4, extra_kinds=("PS", "MAT1", "MAT2", "SWAP"))
    ham = W.random_hamiltonian(n, 8, seed=n)
    rows = np.random.default_rng(n).uniform(-3, 3, (6, 4))
    psi0 = W.random_state(n, n)
    sv = P.StateVector(n)
    sv.set_state(psi0)
    E, G = sv.expectation_with_grad_batch(w.gates, rows, ham)
    for r in range(rows.shape[0]):
        E0, g0 = oracle.adjoint_grad(n, w.gates, rows[r], ham, psi0)
        assert abs(E[r] - E0) < E_TOL
        np.testing.assert_allclose(G[r], g0, atol=E_TOL, rtol=0)
    assert np.max(np.abs(sv.get_state() - psi0)) == 0.0  # state unchanged
    sv.close()


@pytest.mark.parametrize("n", [1, 5, 12, 18, 21])
def test_sampling_matches_oracle_exactly(P, n):
    """Every draw equals the oracle's inverse CDF (oracle.sample, or_sample: Fig. 1 P:377,
    S:272-280) on the same counter-based uniforms. Both sides decide the index in fp64 from
    prefix sums of |psi|^2 taken in different orders (GPU: block tree; oracle: left to right);
    a draw could differ only if u lands within ~1e-15 of a CDF edge, which the test rules out
    explicitly by checking the distance of every draw to its nearest edge."""
    w = W.random_complex(n, 4, seed=100 + n)
    psi = oracle.apply_circuit(n, w.gates)
    sv = P.StateVector(n)
    sv.apply_circuit(w.gates)
    qubits = list(range(n))[::-1][: min(n, 7)]
    shots = 20000
    got = sv.sample(qubits, shots, seed=n)
    ref = oracle.sample(psi, qubits, shots, seed=n)
    cdf = np.cumsum(np.abs(psi) ** 2)
    u = np.array([(oracle.splitmix64(n + s) >> 11) * 2.0 ** -53 for s in range(shots)]) * cdf[-1]
    j = np.searchsorted(cdf, u)
    near = np.minimum(np.abs(cdf[np.minimum(j, cdf.size - 1)] - u), np.abs(cdf[np.maximum(j - 1, 0)] - u))
    assert np.min(near) > 1e-13  # no draw sits on a rounding-level tie
    assert np.array_equal(got, ref)
    full = sv.sample(list(range(n)), shots, seed=n)
    assert np.array_equal(full, oracle.sample_indices(psi, shots, seed=n).astype(np.uint64))
    again = sv.sample(qubits, shots, seed=n)
    assert np.array_equal(got, again)  # deterministic under the seed
    sv.close()


def test_sampling_spec_examples(P):
    """|0> -> all 0; |+> -> binomial within 5 sigma; Bell -> only 00 and 11."""
    sv = P.StateVector(3)
    assert np.all(sv.sample([0], 100, seed=1) == 0)
    sv.apply_circuit([W.Gate("H", (0,))])
    ones = int(np.sum(sv.sample([0], 100000, seed=2)))
    assert abs(ones - 50000) < 5 * np.sqrt(100000 * 0.25)
    sv.reset()
    sv.apply_circuit([W.Gate("H", (0,)), W.Gate("X", (1,), (0,))])
    outs = sv.sample([0, 1], 10000, seed=3)
    assert set(np.unique(outs).tolist()) == {0, 3}
    sv.close()


# ----------------------------------------------------------------------------- NEXT-4 density matrix

@pytest.mark.parametrize("n", [1, 2, 4, 6, 8])
def test_density_matches_oracle(P, n):
    """rho <- U rho U^dagger through the fused 2n-qubit passes vs the oracle's full-matrix
    definition (§3.2), from |0><0| and from a mixed state; tr(rho H)."""
    w = W.random_complex(n, 4, seed=300 + n, n_params=3, extra_kinds=("MAT1", "MAT2", "PS", "XLIKE"))
    ham = W.random_hamiltonian(n, 8, seed=n)
    dm = P.DensityMatrix(n)
    dm.apply_circuit(w.gates, w.params)
    ref = oracle.dm_apply_circuit(n, w.gates, w.params)
    assert np.max(np.abs(dm.get_state() - ref)) <= 1e-10
    assert abs(dm.expectation(ham) - oracle.dm_expectation(ref, ham)) < E_TOL
    a, b = W.random_state(n, 1), W.random_state(n, 2)
    mix = 0.25 * np.outer(a, a.conj()) + 0.75 * np.outer(b, b.conj())
    dm.set_state(mix)
    dm.apply_circuit(w.gates, w.params)
    ref = oracle.dm_apply_circuit(n, w.gates, w.params, mix)
    assert np.max(np.abs(dm.get_state() - ref)) <= 1e-10
    assert abs(dm.expectation(ham) - oracle.dm_expectation(ref, ham)) < E_TOL
    dm.reset()
    st = dm.get_state()
    assert st[0, 0] == 1 and np.count_nonzero(st) == 1
    dm.close()


def test_density_pure_state_equals_state_vector_12q(P):
    """Pure-state consistency at 12 qubits (a 24-qubit vector): rho = |psi><psi| of the
    state-vector path (S:700 criterion 5), checked on sampled entries; tr(rho H) = <psi|H|psi>."""
    n = 12
    w = W.random_complex(n, 5, seed=12)
    psi = oracle.apply_circuit(n, w.gates)
    dm = P.DensityMatrix(n)
    dm.apply_circuit(w.gates)
    rho = dm.get_state()
    idx = np.random.default_rng(0).integers(0, 1 << n, (2000, 2))
    np.testing.assert_allclose(rho[idx[:, 0], idx[:, 1]], psi[idx[:, 0]] * np.conj(psi[idx[:, 1]]), atol=1e-12)
    assert abs(np.trace(rho) - 1) < 1e-10
    ham = W.jw_hamiltonian(n, 20, seed=5)
    assert abs(dm.expectation(ham) - oracle.expectation(psi, ham)[0]) < E_TOL
    with pytest.raises(P.SvError):
        dm.expectation_with_grad(w.gates, [], ham)
    dm.close()
