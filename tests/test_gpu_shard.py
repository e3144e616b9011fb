"""GPU parity of the sharded executor: P virtual shards on one B200 (every shard its own device
buffer, exchanges as device swaps) run the same schedule, localisation and expectation / gradient
logic as the NCCL transport. Compared with the CPU oracle (and the 1-GPU path)."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_shard_gloo import _global_heavy_circuit

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10
E_TOL = 1e-9


@pytest.fixture(scope="module")
def P():
    import paper_2406_17248_b200 as P
    return P


def _sharded(P, n, world):
    return P.StateVector(n, handle=P.sv_create_virtual_shards(n, world))


@pytest.mark.parametrize("world,n", [(2, 9), (4, 11), (8, 14), (2, 16), (8, 17)])
def test_sharded_circuits(P, world, n):
    gates = _global_heavy_circuit(n, seed=world * 100 + n)
    ref = oracle.apply_circuit(n, gates)
    sv = _sharded(P, n, world)
    sv.apply_circuit(gates)
    got = sv.get_state()
    assert np.max(np.abs(got - ref)) <= AMP_TOL
    # a second call continues from the permuted layout
    more = W.random_complex(n, 3, seed=7).gates
    sv.apply_circuit(more)
    ref2 = oracle.apply_circuit(n, more, None, ref)
    assert np.max(np.abs(sv.get_state() - ref2)) <= AMP_TOL
    sv.close()


@pytest.mark.parametrize("world,n", [(2, 10), (4, 12), (8, 15)])
def test_sharded_expectation(P, world, n):
    psi = W.random_state(n, n)
    ham = W.jw_hamiltonian(n, 40, seed=n) + W.random_hamiltonian(n, 20, seed=world)
    sv = _sharded(P, n, world)
    sv.set_state(psi)
    got = sv.expectation(ham)
    ref = oracle.expectation(psi, ham)[0]
    assert abs(got - ref) < E_TOL
    # the expectation's own swaps leave the state (as observed through get_state) unchanged
    assert np.max(np.abs(sv.get_state() - psi)) <= AMP_TOL
    sv.close()


@pytest.mark.parametrize("world,n", [(2, 8), (4, 10), (8, 13)])
def test_sharded_gradient(P, world, n):
    w = W.random_complex(n, 6, seed=40 + n, n_params=5, extra_kinds=("PS",))
    top = n - 1
    gates = w.gates + [
        W.Gate("RZ", (top,), param=0, coeff=1.5), W.Gate("RX", (top,), (0,), param=1),
        W.Gate("RZZ", (top, 2), param=2, coeff=-0.5), W.Gate("PS", (top,), (1,), param=3),
        W.Gate("RYY", (top, top - 1), param=4), W.Gate("RZZ", (top, top - 1), (0,), param=1),
    ]
    ham = W.random_hamiltonian(n, 10, seed=n) + [(0.7, {top: "X", 0: "Z"}), (-0.3, {top: "Y", top - 1: "Z"})]
    psi0 = W.random_state(n, world)
    E0, g0 = oracle.adjoint_grad(n, gates, w.params, ham, psi0)
    sv = _sharded(P, n, world)
    sv.set_state(psi0)
    E, g = sv.expectation_with_grad(gates, w.params, ham)
    assert abs(E - E0) < E_TOL
    np.testing.assert_allclose(g, g0, atol=E_TOL, rtol=0)
    assert np.max(np.abs(sv.get_state() - psi0)) <= AMP_TOL  # state untouched
    sv.close()


def test_sharded_qaoa_matches_single_gpu(P):
    w = W.qaoa(20, 3, seed_graph=5, seed_angles=6)
    one = P.StateVector(20)
    E1, g1 = one.expectation_with_grad(w.gates, w.params, w.ham)
    one.close()
    sv = _sharded(P, 20, 8)
    E8, g8 = sv.expectation_with_grad(w.gates, w.params, w.ham)
    sv.close()
    assert abs(E1 - E8) < E_TOL
    np.testing.assert_allclose(g1, g8, atol=E_TOL, rtol=0)


def test_sharded_reset_and_ghz(P):
    n = 16
    sv = _sharded(P, n, 4)
    gates = [W.Gate("H", (n - 1,))] + [W.Gate("X", (q,), (q + 1,)) for q in reversed(range(n - 1))]
    sv.apply_circuit(gates)
    st = sv.get_state()
    assert abs(st[0] - 2 ** -0.5) < 1e-14 and abs(st[-1] - 2 ** -0.5) < 1e-14
    zz = [(1.0, {0: "Z", n - 1: "Z"})]
    assert abs(sv.expectation(zz) - 1.0) < 1e-12
    assert abs(sv.expectation([(1.0, {q: "X" for q in range(n)})]) - 1.0) < 1e-12
    sv.reset()
    st = sv.get_state()
    assert st[0] == 1 and np.all(st[1:] == 0)
    sv.close()


@pytest.mark.parametrize("world,n,chunk", [(2, 12, 1000), (4, 13, 333), (8, 15, 4096)])
def test_sharded_bounce_exchange(P, world, n, chunk, monkeypatch):
    """The NCCL transport's exchange sequence (pack the outgoing half into a bounce buffer, chunked
    with a ragged tail, unpack the partner's half) run between virtual shards with device copies
    in place of ncclSend / ncclRecv: circuits, expectation and gradient vs the oracle."""
    monkeypatch.setenv("SV_VIRTUAL_BOUNCE", str(chunk))
    gates = _global_heavy_circuit(n, seed=world * 31 + n)
    ref = oracle.apply_circuit(n, gates)
    sv = _sharded(P, n, world)
    sv.apply_circuit(gates)
    assert np.max(np.abs(sv.get_state() - ref)) <= AMP_TOL
    ham = W.jw_hamiltonian(n, 30, seed=n)
    assert abs(sv.expectation(ham) - oracle.expectation(ref, ham)[0]) < E_TOL
    sv.close()
    w = W.random_complex(n, 4, seed=70 + n, n_params=4, extra_kinds=("PS",))
    hm = W.random_hamiltonian(n, 8, seed=n)
    E0, g0 = oracle.adjoint_grad(n, w.gates, w.params, hm)
    sv = _sharded(P, n, world)
    E, g = sv.expectation_with_grad(w.gates, w.params, hm)
    sv.close()
    assert abs(E - E0) < E_TOL
    np.testing.assert_allclose(g, g0, atol=E_TOL, rtol=0)
