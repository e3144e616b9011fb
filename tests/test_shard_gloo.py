"""Multi-process CPU tests of the sharding host logic (gloo, world sizes 2 and 4, no GPU).

Each rank takes the schedule libsv.so would run for its shard (`sv_shard_plan`: local segments with
global controls resolved and diagonal factors on global qubits folded, plus global<->local swaps),
executes the segments on its numpy shard with the test oracle's plain gate application, performs
each swap as the pairwise half-shard exchange of include/sv_debug.h over torch.distributed (gloo)
— the same protocol the NCCL transport implements — and rank 0 reassembles the state through the
final logical->physical layout and compares it with the oracle's unsharded result.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W

P = pytest.importorskip("paper_2406_17248_b200")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _insert_zero(i, l):
    lo = i & ((1 << l) - 1)
    return ((i >> l) << (l + 1)) | lo


def _worker(rank, world, port, n, gates_spec, params, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gates = gates_spec
        g = world.bit_length() - 1
        nl = n - g
        steps, perm = P.sv_shard_plan(n, world, rank, gates, params)
        shard = np.zeros(1 << nl, dtype=np.complex128)
        if rank == 0:
            shard[0] = 1.0
        half_idx = {}
        for st in steps:
            if st[0] == "segment":
                for mat, targets, cmask in st[1]:
                    controls = [b for b in range(nl) if (cmask >> b) & 1]
                    shard = oracle.apply_matrix(shard, mat, targets, controls)
            else:
                _, gpos, lpos = st
                j = gpos - nl
                peer = rank ^ (1 << j)
                h_send = 0 if (rank >> j) & 1 else 1
                key = (lpos, h_send)
                if key not in half_idx:
                    half_idx[key] = np.array([_insert_zero(i, lpos) | (h_send << lpos) for i in range(1 << (nl - 1))])
                idx = half_idx[key]
                send = torch.from_numpy(np.ascontiguousarray(shard[idx]).view(np.float64).copy())
                recv = torch.empty_like(send)
                reqs = [dist.isend(send, peer), dist.irecv(recv, peer)]
                for r in reqs:
                    r.wait()
                shard[idx] = recv.numpy().view(np.complex128)
        t = torch.from_numpy(shard.view(np.float64).copy())
        if rank == 0:
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.gather(t, parts, dst=0)
            phys = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            full = np.empty(1 << n, dtype=np.complex128)
            for i in range(1 << n):
                x = 0
                for qq in range(n):
                    if (i >> qq) & 1:
                        x |= 1 << perm[qq]
                full[i] = phys[x]
            q.put(full)
        else:
            dist.gather(t, dst=0)
    finally:
        dist.destroy_process_group()


def _run(world, n, gates, params=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, gates, params, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return full


def _global_heavy_circuit(n, seed):
    """Random circuit plus gates that stress the global qubits: non-diagonal targets on them
    (swaps), controls on them (dropped / removed per shard), diagonal and RZZ factors on them."""
    rng = np.random.default_rng(seed)
    w = W.random_complex(n, 5, seed=seed, extra_kinds=("MAT1", "MAT2", "PS", "ZLIKE", "XLIKE"))
    top = n - 1
    extra = [
        W.Gate("H", (top,)), W.Gate("X", (0,), (top,)), W.Gate("RZ", (top,), offset=0.7),
        W.Gate("RZZ", (top, 1), offset=1.1), W.Gate("RZZ", (2, top), (0,), offset=-0.4),
        W.Gate("PS", (top,), (1,), offset=0.3), W.Gate("RX", (top,), (n - 2,), offset=0.9),
        W.Gate("MAT2", (top, 0), mat=W.haar_unitary(4, rng)), W.Gate("SWAP", (top, n - 2)),
        W.Gate("RZZ", (n - 2, top), offset=0.25), W.Gate("Y", (n - 2,), (top, 0)),
    ]
    return w.gates[: len(w.gates) // 2] + extra + w.gates[len(w.gates) // 2:]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,n,seed", [(2, 5, 1), (2, 7, 2), (4, 6, 3), (4, 8, 4)])
def test_sharded_schedule_matches_oracle(world, n, seed):
    gates = _global_heavy_circuit(n, seed)
    ref = oracle.apply_circuit(n, gates)
    got = _run(world, n, gates)
    np.testing.assert_allclose(got, ref, atol=1e-12, rtol=0)


def test_schedule_swaps_only_for_global_nondiagonal_targets():
    n, world = 6, 2
    diag_only = [W.Gate("H", (0,)), W.Gate("Z", (5,)), W.Gate("RZZ", (5, 0), offset=0.2), W.Gate("X", (1,), (5,))]
    steps, perm = P.sv_shard_plan(n, world, 0, diag_only)
    assert all(s[0] == "segment" for s in steps) and perm == list(range(n))
    steps, perm = P.sv_shard_plan(n, world, 1, [W.Gate("H", (5,))])
    assert [s[0] for s in steps] == ["swap", "segment"] and perm[5] < n - 1


# ----------------------------------------------------------------------------- cross-shard Pauli streaming
# The protocol of shard.cpp's cross-shard groups (x-mask wider than a shard): rank r and its partner
# p = r ^ x_g stream each other's shard in chunks (chunk c = amplitudes [off, off + cnt)), and each
# rank adds sum_j conj(psi_r[j ^ x_l]) C(j) partner[j] over the received chunk, with
# C(j) = sum_t c'_t (-1)^{popc(j & z_t,local)} and the partner's rank-bit signs (-1)^{popc(z_t,global & p)}
# folded into c'_t (c'_t = c_t i^{popc(x & z_t)}); one all-reduce finishes E. Here every step runs in
# numpy over gloo send/recv; rank 0 compares with the oracle's <psi|H|psi>.

def _cross_worker(rank, world, port, n, psi, terms, chunk, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        nl = n - g
        NL = 1 << nl
        lmask = NL - 1
        mine = psi[rank * NL:(rank + 1) * NL]
        E = 0.0
        for x, zs, cs in terms:  # one x-group: the x-mask and its terms' z masks / coefficients
            xg, xl = x >> nl, x & lmask
            assert xg != 0
            peer = rank ^ xg
            cfold = []
            for z, c in zip(zs, cs):
                cp = c * (1j ** (bin(x & z).count("1") % 4))
                cfold.append(cp * (-1.0 if bin((z >> nl) & peer).count("1") % 2 else 1.0))
            for off in range(0, NL, chunk):
                send = torch.from_numpy(np.ascontiguousarray(mine[off:off + chunk]).view(np.float64).copy())
                recv = torch.empty_like(send)
                reqs = [dist.isend(send, peer), dist.irecv(recv, peer)]
                for r in reqs:
                    r.wait()
                part = recv.numpy().view(np.complex128)
                j = np.arange(off, off + chunk, dtype=np.int64)
                C = np.zeros(chunk, dtype=np.complex128)
                for z, cf in zip(zs, cfold):
                    par = np.array([bin(v).count("1") & 1 for v in (j & (z & lmask))])
                    C += cf * np.where(par == 1, -1.0, 1.0)
                E += float(np.sum(np.conj(mine[j ^ xl]) * C * part).real)
        t = torch.tensor([E], dtype=torch.float64)
        dist.all_reduce(t)
        if rank == 0:
            q.put(float(t.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,n,chunk", [(2, 6, 8), (4, 7, 4), (4, 8, 64)])
def test_cross_shard_chunk_protocol(world, n, chunk):
    psi = W.random_state(n, 11 * n + world)
    # Pauli strings wider than a shard: X/Y on every qubit (and a mixed-Z variant sharing the x-mask)
    full = (1 << n) - 1
    ham = [(0.7, {q: "X" for q in range(n)}), (-0.4, {q: ("Y" if q % 3 == 0 else "X") for q in range(n)}),
           (0.25, {**{q: "X" for q in range(n)}, 1: "Y", n - 1: "Y"})]
    groups = {}
    for c, term in ham:
        x = sum(1 << q for q, p in term.items() if p in "XY")
        z = sum(1 << q for q, p in term.items() if p in "YZ")
        groups.setdefault(x, ([], []))
        groups[x][0].append(z)
        groups[x][1].append(c)
    terms = [(x, zs, cs) for x, (zs, cs) in groups.items()]
    assert all(x == full for x, _, _ in terms)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cross_worker, args=(r, world, port, n, psi, terms, chunk, q)) for r in range(world)]
    for p in procs:
        p.start()
    E = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.expectation(psi, ham)[0]
    assert abs(E - ref) < 1e-12, (E, ref)
