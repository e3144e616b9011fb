"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star; derivation in DESIGN.md §Tolerances): 1e-10 absolute per
amplitude, 1e-9 on expectations and gradients.
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10
E_TOL = 1e-9


@pytest.fixture(scope="module")
def P():
    import paper_2406_17248_b200 as P
    return P


def _gpu_run(P, n, gates, params=None, psi0=None, opts=None):
    sv = P.StateVector(n)
    for k, v in (opts or {}).items():
        sv.set_option(k, v)
    if psi0 is not None:
        sv.set_state(psi0)
    sv.apply_circuit(gates, params)
    out = sv.get_state()
    sv.close()
    return out


def _assert_amps(got, ref, tol=AMP_TOL):
    err = np.max(np.abs(got - ref)) if got.size else 0.0
    assert err <= tol, f"max |gpu - oracle| = {err:.3e} > {tol:.0e}"


# ----------------------------------------------------------------------------- single gates

def _positions(n):
    """Target positions covering the low (in-chunk), mid (tile) and high (outer) ranges."""
    cand = {0, 1, 2, 3, 4, 5, 7, 11, 12, n - 2, n - 1}
    return sorted(q for q in cand if 0 <= q < n)


@pytest.mark.parametrize("kind", W.ALL_KINDS)
@pytest.mark.parametrize("n", [1, 2, 5, 13, 16])
def test_every_kind_every_position(P, kind, n):
    rng = np.random.default_rng(n * 100 + W.ALL_KINDS.index(kind))
    two = kind in W.KINDS_2Q
    if two and n < 2:
        pytest.skip("two-qubit kind needs n >= 2")
    psi0 = W.random_state(n, int(rng.integers(1 << 30)))
    gates = []
    for t in _positions(n):
        for nctrl in (0, 1, 2):
            targets = [t]
            if two:
                others = [q for q in range(n) if q != t]
                targets.append(int(rng.choice(others)))
            free = [q for q in range(n) if q not in targets]
            if nctrl > len(free):
                continue
            controls = tuple(int(c) for c in rng.choice(free, nctrl, replace=False)) if nctrl else ()
            mat = None
            if kind == "MAT1":
                mat = W.haar_unitary(2, rng)
            elif kind == "MAT2":
                mat = W.haar_unitary(4, rng)
            elif kind in ("XLIKE", "ZLIKE"):
                mat = rng.standard_normal(2) + 1j * rng.standard_normal(2)
            gates.append(W.Gate(kind, tuple(targets), controls, offset=float(rng.uniform(-7, 7)), mat=mat))
    # one gate per call (sv_apply_gate) and the whole list fused (sv_apply_circuit)
    ref = oracle.apply_circuit(n, gates, None, psi0)
    _assert_amps(_gpu_run(P, n, gates, None, psi0), ref)
    sv = P.StateVector(n)
    sv.set_state(psi0)
    for g in gates:
        sv.apply_gate(g)
    _assert_amps(sv.get_state(), ref)
    sv.close()


def test_all_controls_max(P):
    """n-1 controls (a single pair updated) and controls on every tile/outer position."""
    n = 15
    psi0 = W.random_state(n, 3)
    gates = [W.Gate("H", (t,), tuple(q for q in range(n) if q != t)) for t in (0, 6, 14)]
    gates += [W.Gate("RXX", (2, 13), tuple(q for q in range(n) if q not in (2, 13)), offset=0.7)]
    _assert_amps(_gpu_run(P, n, gates, None, psi0), oracle.apply_circuit(n, gates, None, psi0))


# ----------------------------------------------------------------------------- circuits

@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 9, 12, 13, 14, 17, 20])
def test_random_complex_circuits(P, n):
    """The paper's "complex random circuit" shape (controls p=0.3) plus user matrices."""
    w = W.random_complex(n, 10, seed=1000 + n, n_params=5,
                         extra_kinds=("MAT1", "MAT2", "XLIKE", "ZLIKE", "PS", "SDG", "TDG"))
    ref = oracle.apply_circuit(n, w.gates, w.params)
    _assert_amps(_gpu_run(P, n, w.gates, w.params), ref)


@pytest.mark.parametrize("opts", [{1: 4}, {1: 7}, {1: 10}, {2: 0}, {3: 0}, {3: 5}, {1: 13}, {4: 0}, {5: 0},
                                  {1: 9}, {1: 11}, {4: 0, 1: 12}])
def test_plan_options_do_not_change_results(P, opts):
    """Tile width, fusion on/off and the low-qubit granule only change the schedule."""
    n = 16
    w = W.random_complex(n, 6, seed=77, extra_kinds=("MAT2", "PS"))
    ref = oracle.apply_circuit(n, w.gates, w.params)
    _assert_amps(_gpu_run(P, n, w.gates, w.params, opts=opts), ref)


@pytest.mark.parametrize("dense", [1, 0])
def test_c4_shape_at_22q(P, dense):
    """C4's generator (Haar 1q + CZ bricks) at 22 qubits, depth 12; dense MMA stages on and off."""
    w = W.random_circuit(22, 12, seed=3040)
    _assert_amps(_gpu_run(P, 22, w.gates, opts={4: dense}), oracle.apply_circuit(22, w.gates))


def test_dense_stages_are_used(P):
    """The C4 plan folds most register stages into dense FP64-MMA stages (planner introspection)."""
    w = W.random_circuit(22, 12, seed=3040)
    plan = P.sv_plan_info(22, w.gates)
    assert sum(p["n_dense"] for p in plan) > 0.5 * sum(p["n_stages"] for p in plan)


def test_mirror_and_norm_at_24q(P):
    w = W.random_circuit(24, 6, seed=11)
    gates = W.mirror(w.gates)
    out = _gpu_run(P, 24, gates)
    assert abs(out[0] - 1) < 1e-11 and np.max(np.abs(out[1:])) < 1e-11


def test_empty_circuit_and_reset(P):
    sv = P.StateVector(5)
    sv.apply_circuit([])
    st = sv.get_state()
    assert st[0] == 1 and np.all(st[1:] == 0)
    sv.apply_circuit([W.Gate("H", (0,))])
    sv.reset()
    st = sv.get_state()
    assert st[0] == 1 and np.all(st[1:] == 0)
    sv.close()


# ----------------------------------------------------------------------------- expectation

@pytest.mark.parametrize("n", [1, 3, 6, 12, 15, 20])
def test_expectation_random(P, n):
    psi = W.random_state(n, n)
    ham = W.random_hamiltonian(n, 30, seed=n) + W.jw_hamiltonian(n, 20, seed=n) if n >= 4 else W.random_hamiltonian(n, 10, n)
    ref = oracle.expectation(psi, ham)[0]
    sv = P.StateVector(n)
    sv.set_state(psi)
    got = sv.expectation(ham)
    sv.close()
    assert abs(got - ref) < E_TOL


def test_expectation_spec_values(P):
    sv = P.StateVector(2)
    sv.apply_circuit([W.Gate("H", (0,)), W.Gate("X", (1,), (0,))])
    assert abs(sv.expectation([(1.0, {0: "X", 1: "X"})]) - 1.0) < 1e-14
    assert sv.expectation([]) == 0.0
    assert abs(sv.expectation([(0.25, {})]) - 0.25) < 1e-15
    sv.close()


# ----------------------------------------------------------------------------- gradients

def test_c1_full(P):
    """BASELINE configs[0]: amplitudes, E and gradient vs oracle and the closed form."""
    w = W.c1_ghz_rx()
    ref = oracle.apply_circuit(w.n, w.gates, w.params)
    _assert_amps(_gpu_run(P, w.n, w.gates, w.params), ref)
    sv = P.StateVector(w.n)
    E, g = sv.expectation_with_grad(w.gates, w.params, w.ham)
    th = w.params
    assert abs(E - np.cos(th[0]) * np.cos(th[1])) < E_TOL
    np.testing.assert_allclose(g, [-np.sin(th[0]) * np.cos(th[1]), -np.cos(th[0]) * np.sin(th[1]), 0, 0], atol=E_TOL)
    # state untouched by _with_grad
    st = sv.get_state()
    assert st[0] == 1 and np.all(st[1:] == 0)
    sv.close()


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (4, 2), (6, 3), (9, 4), (13, 5), (15, 6)])
def test_gradient_random_tasks(P, n, seed):
    w = W.random_complex(n, 8, seed=500 + seed, n_params=6, extra_kinds=("PS", "MAT1", "MAT2"))
    ham = W.random_hamiltonian(n, 8, seed)
    psi0 = W.random_state(n, seed)
    E0, g0 = oracle.adjoint_grad(n, w.gates, w.params, ham, psi0)
    sv = P.StateVector(n)
    sv.set_state(psi0)
    E, g = sv.expectation_with_grad(w.gates, w.params, ham)
    sv.close()
    assert abs(E - E0) < E_TOL
    np.testing.assert_allclose(g, g0, atol=E_TOL, rtol=0)


@pytest.mark.parametrize("da_cost", [-1, 0, 1 << 20])
def test_gradient_c2_hea_20q(P, da_cost):
    """C2: 20q HEA, 10 layers, 50-term JW-shaped H (400 params): default plan, adjoint dense
    stages wherever eligible, and none."""
    w = W.config("C2")
    E0, g0 = oracle.adjoint_grad(w.n, w.gates, w.params, w.ham)
    sv = P.StateVector(w.n)
    sv.set_option(P.SV_OPT_ADJOINT_DENSE_COST, da_cost)
    E, g = sv.expectation_with_grad(w.gates, w.params, w.ham)
    sv.close()
    assert abs(E - E0) < E_TOL
    np.testing.assert_allclose(g, g0, atol=E_TOL, rtol=0)


@pytest.mark.parametrize("n,seed", [(12, 7), (16, 8)])
def test_gradient_adjoint_dense_forced(P, n, seed):
    """Adjoint dense stages (R = sum psi lambda^H by MMA, host contraction) at small n: HEA
    layers (dense-friendly) plus a random controlled tail, every eligible stage taken."""
    h = W.hea(n, 3, seed=seed, nterms=20)
    tail = W.random_complex(n, 2, seed=seed, n_params=0, extra_kinds=("PS",))
    gates = list(h.gates) + list(tail.gates)
    psi0 = W.random_state(n, seed)
    E0, g0 = oracle.adjoint_grad(n, gates, h.params, h.ham, psi0)
    sv = P.StateVector(n)
    sv.set_option(P.SV_OPT_ADJOINT_DENSE_COST, 0)
    sv.set_state(psi0)
    E, g = sv.expectation_with_grad(gates, h.params, h.ham)
    sv.close()
    assert abs(E - E0) < E_TOL
    np.testing.assert_allclose(g, g0, atol=E_TOL, rtol=0)


@pytest.mark.parametrize("n,dc", [(12, False), (14, True), (16, False)])
def test_gradient_qaoa_adjoint_dense_outer_variants(P, n, dc):
    """QAOA (RZZ edges leaving the tile): adjoint dense stages whose variant bits include outer
    qubits (one R accumulator per outer variant), forced on at small n."""
    w = W.qaoa(n, 3, seed_graph=n, seed_angles=n + 1, dc=dc)
    E0, g0 = oracle.adjoint_grad(n, w.gates, w.params, w.ham)
    sv = P.StateVector(n)
    sv.set_option(P.SV_OPT_ADJOINT_DENSE_COST, 0)
    E, g = sv.expectation_with_grad(w.gates, w.params, w.ham)
    sv.close()
    assert abs(E - E0) < E_TOL
    np.testing.assert_allclose(g, g0, atol=E_TOL, rtol=0)


def test_gradient_qaoa_p1_24q_closed_form(P):
    """C3 graph at p=1: E and the shared-parameter gradient vs the Wang et al. closed form."""
    from test_oracle import _qaoa_p1_closed_form
    w = W.qaoa(24, 1, seed_graph=2403, seed_angles=2404)
    edges = w.meta["edges"]
    sv = P.StateVector(24)
    E, g = sv.expectation_with_grad(w.gates, w.params, w.ham)
    sv.close()
    gam, bet = w.params
    assert abs(E - _qaoa_p1_closed_form(edges, 24, gam, bet)) < E_TOL
    h = 1e-6
    dg = (_qaoa_p1_closed_form(edges, 24, gam + h, bet) - _qaoa_p1_closed_form(edges, 24, gam - h, bet)) / (2 * h)
    db = (_qaoa_p1_closed_form(edges, 24, gam, bet + h) - _qaoa_p1_closed_form(edges, 24, gam, bet - h)) / (2 * h)
    np.testing.assert_allclose(g, [dg, db], atol=1e-7)


def test_gradient_qaoa_zero_params_24q(P):
    w = W.config("C3")
    sv = P.StateVector(24)
    E, g = sv.expectation_with_grad(w.gates, np.zeros_like(w.params), w.ham)
    sv.close()
    assert abs(E + len(w.meta["edges"]) / 2) < E_TOL
    np.testing.assert_allclose(g, 0, atol=E_TOL)


# ----------------------------------------------------------------------------- errors

def test_validation_errors(P):
    sv = P.StateVector(3)
    cases = [
        (W.Gate("X", (3,)), "SV_E_QUBIT_RANGE"),
        (W.Gate("X", (0,), (0,)), "SV_E_TARGET_CONTROL_OVERLAP"),
        (W.Gate("SWAP", (1, 1)), "SV_E_DUPLICATE_TARGET"),
        (W.Gate("RX", (0,), param=2), "SV_E_PARAM_RANGE"),
        (W.Gate("H", (0,), param=0), "SV_E_ARG"),
        (W.Gate("X", (0,), (5,)), "SV_E_QUBIT_RANGE"),
    ]
    for g, status in cases:
        with pytest.raises(P.SvError) as ei:
            sv.apply_circuit([W.Gate("H", (1,)), g], [0.1])
        assert ei.value.status == status
    # atomic: nothing applied by the failing calls
    st = sv.get_state()
    assert st[0] == 1
    with pytest.raises(P.SvError) as ei:
        sv.expectation_with_grad([W.Gate("MAT1", (0,), param=0, mat=np.eye(2))], [0.1], [(1.0, {0: "Z"})])
    assert ei.value.status == "SV_E_NOT_DIFFERENTIABLE"
    with pytest.raises(P.SvError) as ei:
        sv.expectation_with_grad([W.Gate("MAT1", (0,), mat=2 * np.eye(2))], [], [(1.0, {0: "Z"})])
    assert ei.value.status == "SV_E_NOT_UNITARY"
    with pytest.raises(P.SvError) as ei:
        sv.expectation([(1.0, {4: "Z"})])
    assert ei.value.status == "SV_E_QUBIT_RANGE"
    sv.close()


def test_determinism(P):
    w = W.config("C2")
    sv = P.StateVector(w.n)
    a = sv.expectation_with_grad(w.gates, w.params, w.ham)
    b = sv.expectation_with_grad(w.gates, w.params, w.ham)
    sv.close()
    assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_user_streams(P):
    """Work on caller-provided CUDA streams (switched between calls, and back to the handle's own)
    gives the same results as the default stream (sv_set_stream, include/sv.h)."""
    import torch
    n = 14
    w = W.random_complex(n, 5, seed=77, n_params=3, extra_kinds=("PS", "MAT2"))
    ham = W.jw_hamiltonian(n, 12, seed=3)
    ref_psi = oracle.apply_circuit(n, w.gates, w.params)
    E0, g0 = oracle.adjoint_grad(n, w.gates, w.params, ham)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    sv = P.StateVector(n)
    P.sv_set_stream(sv.h, s1.cuda_stream)
    sv.apply_circuit(w.gates, w.params)
    P.sv_set_stream(sv.h, s2.cuda_stream)
    assert np.max(np.abs(sv.get_state() - ref_psi)) <= AMP_TOL
    sv.reset()
    E, g = sv.expectation_with_grad(w.gates, w.params, ham)
    P.sv_set_stream(sv.h, None)
    E2, g2 = sv.expectation_with_grad(w.gates, w.params, ham)
    sv.close()
    assert abs(E - E0) < E_TOL and abs(E2 - E0) < E_TOL
    np.testing.assert_allclose(g, g0, atol=E_TOL, rtol=0)
    assert np.array_equal(g, g2)


def test_concurrent_handles_two_threads(P):
    """Distinct handles may be driven concurrently (include/sv.h): two threads evaluate gradients of
    different circuits with changing parameters at once (each call plans on the shared host worker
    pool and launches on its own stream; ctypes releases the GIL); every result equals the
    oracle's."""
    import threading

    cases = [W.qaoa(12, 3, seed_graph=5, seed_angles=6), W.hea(11, 3, seed=9, nterms=20)]
    refs = [[oracle.adjoint_grad(w.n, w.gates, w.params + 0.01 * r, w.ham) for r in range(4)] for w in cases]
    errs = [[], []]

    def worker(i):
        w = cases[i]
        sv = P.StateVector(w.n)
        try:
            for r in range(4):
                E, g = sv.expectation_with_grad(w.gates, w.params + 0.01 * r, w.ham)
                errs[i].append(max(abs(E - refs[i][r][0]), float(np.max(np.abs(g - refs[i][r][1])))))
        finally:
            sv.close()

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert len(errs[0]) == 4 and len(errs[1]) == 4
    assert max(errs[0] + errs[1]) <= 1e-9, errs


def test_adjoint_cost_contract(P):
    """S:478 / S:695 cost contract on the GPU path: one evaluation of sv_expectation_with_grad
    performs N (forward plan) + 2N (adjoint plan over psi and lambda) = 3N gate applications
    (instrumented counter sv_stats.gate_applications), and the same numbers of HBM passes,
    whatever the number of distinct parameters P the circuit's rotations share."""
    import dataclasses
    base = W.random_complex(14, 6, seed=3, n_params=12)
    ham = W.random_hamiltonian(14, 6, seed=3)
    N = len(base.gates)
    seen = set()
    for nparam in (1, 4, 12):
        gates = []
        for g in base.gates:
            gates.append(dataclasses.replace(g, param=g.param % nparam) if g.param >= 0 else g)
        params = base.params[:nparam]
        sv = P.StateVector(14)
        P.sv_reset_stats(sv.h)
        E, g = sv.expectation_with_grad(gates, params, ham)
        st = sv.stats()
        sv.close()
        E0, g0 = oracle.adjoint_grad(14, gates, params, ham)
        assert abs(E - E0) < 1e-9 and np.max(np.abs(g - g0)) < 1e-9
        assert st["gate_applications"] == 3 * N, (nparam, st["gate_applications"], N)
        seen.add((st["gate_passes"], st["adjoint_passes"]))
    assert len(seen) == 1, seen  # pass counts do not grow with P


def test_structural_plan_refresh(P):
    """An optimiser loop re-evaluates one circuit structure with new angles: the library reuses the
    cached plan's passes and stages and rewrites only its matrices (sv_stats.plan_refreshes). Every
    evaluation must equal the oracle's — including angles that flip value-dependent fast paths
    (RZ(0) = identity diagonal, RX(0)), dense stages (C4-shaped 1q matrices) and adjoint plans."""
    w = W.qaoa(16, 3, seed_graph=3, seed_angles=4, dc=True)
    sv = P.StateVector(16)
    P.sv_reset_stats(sv.h)
    for r, p in enumerate([w.params, w.params * 0.5 + 0.1, np.zeros_like(w.params), w.params[::-1].copy()]):
        E, g = sv.expectation_with_grad(w.gates, p, w.ham)
        E0, g0 = oracle.adjoint_grad(16, w.gates, p, w.ham)
        assert abs(E - E0) < 1e-9 and np.max(np.abs(g - g0)) < 1e-9, r
    st = sv.stats()
    assert st["plan_refreshes"] >= 6 and st["plan_builds"] == 2, st  # forward + adjoint built once
    sv.close()
    # forward: the same C4-shaped structure with new Haar matrices (dense-stage variants re-filled)
    a = W.random_circuit(18, 6, seed=1)
    b = W.random_circuit(18, 6, seed=2)
    sv = P.StateVector(18)
    sv.apply_circuit(a.gates)
    sv.reset()
    sv.apply_circuit(b.gates)
    got = sv.get_state()
    st = sv.stats()
    sv.close()
    assert st["plan_refreshes"] >= 1
    assert np.max(np.abs(got - oracle.apply_circuit(18, b.gates))) <= 1e-10
    # back to back without a synchronisation: b's refreshed plan is uploaded on the side stream into
    # the buffer a's passes are still reading; the copy must wait for them (CachedPlan::used_ev)
    sv = P.StateVector(18)
    sv.apply_circuit(a.gates)
    sv.apply_circuit(b.gates)
    sv.apply_circuit(a.gates)
    got = sv.get_state()
    sv.close()
    ref = oracle.apply_circuit(18, a.gates, None, oracle.apply_circuit(18, b.gates, None, oracle.apply_circuit(18, a.gates)))
    assert np.max(np.abs(got - ref)) <= 1e-10
