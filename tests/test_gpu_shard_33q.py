"""The sharded executor at (nearly) C5 scale on one B200: a 33-qubit state (128 GiB) as 8 virtual
shards of 2^30 amplitudes — the per-GPU shard size of C5 (34 qubits) on 16 GPUs, and the layout,
swap schedule, localisation and cross-shard Pauli streaming of the NCCL transport (SURVEY §8(c)
pins for the sharded path at scale: block products and GHZ).

* Block-product circuits: no gate couples block A (qubits 0..16) with block B (17..32), so
  psi = psi_B (x) psi_A. Block B contains the three global qubits (30..32): its 1q gates on them force
  half-shard swaps. 4096 sampled amplitudes (sv_get_amplitudes, un-permuted through the final
  layout) equal psi_A[i_A] psi_B[i_B] from two oracle runs (17 and 16 qubits) within 1e-10, and
  <P_A (x) P_B> = <P_A><P_B> within 1e-9, including X on all 33 qubits (an x-mask wider than a shard:
  the chunked cross-shard stream).
* GHZ-33: amplitudes 0 and 2^33 - 1 equal 1/sqrt(2), <Z_0 Z_32> = 1, <X^(x)33> = 1.
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
N, NA = 33, 17


@pytest.fixture(scope="module")
def P():
    import paper_2406_17248_b200 as P
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < (140 << 30):
        pytest.skip("needs ~140 GiB of free device memory")
    return P


def _block_circuit(lo, n, depth, seed):
    """C4-shaped layers on qubits lo .. lo + n - 1 only (Haar 1q + CZ bricks inside the block)."""
    w = W.random_circuit(n, depth, seed=seed)
    out = []
    for g in w.gates:
        out.append(W.Gate(g.kind, tuple(t + lo for t in g.targets), tuple(c + lo for c in g.controls), g.param,
                          g.coeff, g.offset, g.mat))
    return w.gates, out


def _term(spec):
    return {q: p for q, p in spec.items()}


@pytest.mark.parametrize("bounce", [None, 1 << 26])
def test_block_product_33q_virtual_shards(P, bounce, monkeypatch):
    """bounce: swaps run the NCCL transport's pipelined pack / 1 GiB bounce-buffer / unpack sequence
    (device copies on the transfer stream in place of send / recv) instead of the swap kernel."""
    if bounce:
        monkeypatch.setenv("SV_VIRTUAL_BOUNCE", str(bounce))
    ga_local, ga = _block_circuit(0, NA, 5, seed=331)
    gb_local, gb = _block_circuit(NA, N - NA, 5, seed=332)
    # interleave the blocks' gates (they commute), so the schedule sees both
    gates = []
    for i in range(max(len(ga), len(gb))):
        if i < len(ga):
            gates.append(ga[i])
        if i < len(gb):
            gates.append(gb[i])
    psi_a = oracle.apply_circuit(NA, ga_local)
    psi_b = oracle.apply_circuit(N - NA, gb_local)
    sv = P.StateVector(N, handle=P.sv_create_virtual_shards(N, 8))
    sv.apply_circuit(gates)
    st = sv.stats()
    assert st["exchanges"] >= 3  # 1q gates on the global qubits 30..32 swapped them local
    rng = np.random.default_rng(33)
    idx = np.concatenate([np.arange(64), rng.integers(0, 1 << N, 4096), [(1 << N) - 1]]).astype(np.uint64)
    got = sv.get_amplitudes(idx)
    ia = (idx & np.uint64((1 << NA) - 1)).astype(np.int64)
    ib = (idx >> np.uint64(NA)).astype(np.int64)
    ref = psi_b[ib] * psi_a[ia]
    assert np.max(np.abs(got - ref)) <= 1e-10
    # expectations factorise; the all-X string is wider than a shard (chunked cross-shard stream)
    pa = {0: "X", 3: "Y", 9: "Z"}
    pb = {NA + 2: "Z", 30: "X", 32: "Y"}
    allx_a = {q: "X" for q in range(NA)}
    allx_b = {q: "X" for q in range(N - NA)}
    for ta, tb in ((pa, {q - NA: p for q, p in pb.items()}), (allx_a, allx_b)):
        ea = oracle.expectation(psi_a, [(1.0, ta)])[0]
        eb = oracle.expectation(psi_b, [(1.0, tb)])[0]
        full = dict(ta)
        full.update({q + NA: p for q, p in tb.items()})
        e = sv.expectation([(1.0, full)])
        assert abs(e - ea * eb) <= 1e-9, (e, ea * eb)
    sv.close()


def test_ghz_33q_virtual_shards(P):
    gates = [W.Gate("H", (0,))] + [W.Gate("X", (q + 1,), (q,)) for q in range(N - 1)]
    sv = P.StateVector(N, handle=P.sv_create_virtual_shards(N, 8))
    sv.apply_circuit(gates)
    amps = sv.get_amplitudes(np.array([0, (1 << N) - 1, 1, 1 << 32, 12345], dtype=np.uint64))
    assert abs(amps[0] - 2 ** -0.5) < 1e-12 and abs(amps[1] - 2 ** -0.5) < 1e-12
    assert np.max(np.abs(amps[2:])) == 0.0
    assert abs(sv.expectation([(1.0, {0: "Z", N - 1: "Z"})]) - 1.0) < 1e-12
    assert abs(sv.expectation([(1.0, {q: "X" for q in range(N)})]) - 1.0) < 1e-12
    assert abs(sv.expectation([(1.0, {5: "Z"})])) < 1e-12
    sv.close()
