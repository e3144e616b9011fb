"""Pins of the CPU oracle (oracle/sv_oracle.c) against what the paper and mathematics fix.

Each pin is chosen so that a plausible mistake in the oracle (dropped term, wrong sign, wrong
index or transposed operand) fails at least one of them:
  * matrix table  vs  matrix exponentials exp(-i t P/2) (scipy) and SPEC printed values;
  * gate application  vs  brute-force Kronecker products (tests/_brute.py), every kind x 0-2
    controls x target positions, n = 1..6;
  * expectation  vs  dense H = sum c (x) sigma, and closed forms;
  * adjoint gradient  vs  exact shift rules, central finite differences, closed forms
    (C1, RX/Z, chain rule, shared parameters, QAOA p=1 (Wang et al. 2018), QAOA at 0);
  * invariants: norm after 10^3 gates, mirror circuits, linearity in H.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg

import oracle
import workloads as W
import _brute as B

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_values.json")))
C1G = json.load(open(os.path.join(GOLD, "c1_worked_example.json")))
RNG = np.random.default_rng(1234)


# ----------------------------------------------------------------------------- matrix table

@pytest.mark.parametrize("kind,gen", [("RX", "X"), ("RY", "Y"), ("RZ", "Z"), ("RXX", "XX"), ("RYY", "YY"), ("RZZ", "ZZ")])
def test_rotation_matrices_are_exponentials(kind, gen):
    """R_P(t) = exp(-i t P / 2) (reading c2.1), via scipy's matrix exponential."""
    P = B.PAULI[gen[0]] if len(gen) == 1 else np.kron(B.PAULI[gen[1]], B.PAULI[gen[0]])
    for t in np.concatenate([RNG.uniform(-7, 7, 5), [0.0, np.pi, -np.pi / 2]]):
        ref = scipy.linalg.expm(-0.5j * t * P)
        np.testing.assert_allclose(oracle.gate_matrix(kind, t), ref, atol=1e-14)


def test_phase_shift_is_exponential():
    for t in RNG.uniform(-7, 7, 5):
        np.testing.assert_allclose(oracle.gate_matrix("PS", t), scipy.linalg.expm(1j * t * B.P1), atol=1e-14)


def test_fixed_gates_relations():
    m = oracle.gate_matrix
    # X, Y, Z are i * R_P(pi)
    for k, r in (("X", "RX"), ("Y", "RY"), ("Z", "RZ")):
        np.testing.assert_allclose(m(k), 1j * m(r, np.pi), atol=1e-15)
    # S, T family as phase shifts
    for k, t in (("S", np.pi / 2), ("SDG", -np.pi / 2), ("T", np.pi / 4), ("TDG", -np.pi / 4), ("Z", np.pi)):
        np.testing.assert_allclose(m(k), m("PS", t), atol=1e-15)
    np.testing.assert_allclose(m("S") @ m("S"), m("Z"), atol=1e-15)
    np.testing.assert_allclose(m("T") @ m("T"), m("S"), atol=1e-15)
    # H = (X + Z)/sqrt2, H^2 = I, H Z H = X; the constant is the correctly rounded 1/sqrt2
    H = m("H")
    np.testing.assert_allclose(H, (m("X") + m("Z")) / np.sqrt(2), atol=1e-16)
    np.testing.assert_allclose(H @ H, np.eye(2), atol=1e-15)
    np.testing.assert_allclose(H @ m("Z") @ H, m("X"), atol=1e-15)
    assert H[0, 0].real == 0.7071067811865476
    # Pauli algebra XY = iZ
    np.testing.assert_allclose(m("X") @ m("Y"), 1j * m("Z"), atol=1e-15)
    # SWAP exchanges the two target bits
    S = m("SWAP")
    for b0 in (0, 1):
        for b1 in (0, 1):
            e = np.zeros(4); e[b0 + 2 * b1] = 1
            assert np.argmax(np.abs(S @ e)) == b1 + 2 * b0


def test_user_matrices_and_class_table():
    """X-like = [[0,a],[b,0]] (reading c2.3), Z-like = diag(a,b); the static
    class table (reading c2.6) agrees with the zero pattern of every kind."""
    a, b = np.exp(0.3j), 0.5 * np.exp(-1.1j)
    np.testing.assert_array_equal(oracle.gate_matrix("XLIKE", 0, [a, b]), np.array([[0, a], [b, 0]]))
    np.testing.assert_array_equal(oracle.gate_matrix("ZLIKE", 0, [a, b]), np.array([[a, 0], [0, b]]))
    U2 = W.haar_unitary(2, RNG)
    U4 = W.haar_unitary(4, RNG)
    np.testing.assert_array_equal(oracle.gate_matrix("MAT1", 0, U2), U2)
    np.testing.assert_array_equal(oracle.gate_matrix("MAT2", 0, U4), U4)
    xlike = {"X", "Y", "XLIKE"}
    zlike = {"Z", "S", "SDG", "T", "TDG", "ZLIKE", "RZ", "PS", "RZZ"}
    for k in W.ALL_KINDS:
        M = oracle.gate_matrix(k, 0.77, U4 if k == "MAT2" else (U2 if k == "MAT1" else [a, b]))
        off = M - np.diag(np.diag(M))
        if k in zlike:
            assert np.all(off == 0), k
        elif k in xlike:
            assert np.all(np.diag(M) == 0), k
        else:
            assert np.any(off != 0) and np.any(np.diag(M) != 0), k


def test_spec_printed_matrices():
    g = SPEC["rx_pi_matrix"]
    np.testing.assert_allclose(oracle.gate_matrix("RX", np.pi), np.array(g["re"]) + 1j * np.array(g["im"]), atol=1e-15)
    ph = np.array(SPEC["rzz_half_pi_diag_phase_over_pi"]["phase_over_pi"])
    np.testing.assert_allclose(oracle.gate_matrix("RZZ", np.pi / 2), np.diag(np.exp(1j * np.pi * ph)), atol=1e-15)


# ----------------------------------------------------------------------------- gate application

def _draw_gate(kind, n, nctrl, rng):
    k = 2 if kind in W.KINDS_2Q else 1
    qs = [int(x) for x in rng.choice(n, k + nctrl, replace=False)]
    mat = None
    if kind == "MAT1":
        mat = W.haar_unitary(2, rng)
    elif kind == "MAT2":
        mat = W.haar_unitary(4, rng)
    elif kind in ("XLIKE", "ZLIKE"):
        mat = rng.standard_normal(2) + 1j * rng.standard_normal(2)
    return qs[:k], qs[k:], mat


@pytest.mark.parametrize("kind", W.ALL_KINDS)
def test_apply_matches_kronecker(kind):
    """Every kind x 0..2 controls x n in 1..6 vs the dense Kronecker oracle, <= 1e-12."""
    rng = np.random.default_rng(hash(kind) % 2**32)
    k = 2 if kind in W.KINDS_2Q else 1
    for n in range(k, 7):
        for nctrl in range(0, min(2, n - k) + 1):
            for _ in range(4):
                targets, controls, mat = _draw_gate(kind, n, nctrl, rng)
                t = rng.uniform(-7, 7)
                M = oracle.gate_matrix(kind, t, mat)
                psi = W.random_state(n, int(rng.integers(1 << 30)))
                got = oracle.apply_matrix(psi, M, targets, controls)
                ref = B.controlled(M, targets, controls, n) @ psi
                np.testing.assert_allclose(got, ref, atol=1e-12, rtol=0)


def test_apply_circuit_vs_kronecker_product():
    """A whole random circuit (paper gate set + controls, shared params) vs U_total = U_N..U_1."""
    n = 5
    w = W.random_complex(n, 6, seed=77, n_params=3, extra_kinds=("MAT1", "MAT2", "XLIKE", "ZLIKE", "PS", "SDG", "TDG"))
    U = np.eye(1 << n, dtype=complex)
    for g in w.gates:
        ang = (g.coeff * w.params[g.param] if g.param >= 0 else 0.0) + g.offset
        U = B.controlled(oracle.gate_matrix(g.kind, ang, g.mat), list(g.targets), list(g.controls), n) @ U
    np.testing.assert_allclose(oracle.apply_circuit(n, w.gates, w.params), U[:, 0], atol=1e-12)


def test_layout_and_spec_states():
    """Qubit 0 = least-significant index bit (Fig. 3: a|00>+b|01>+c|10>+d|11> stored a,b,c,d)."""
    psi = oracle.apply_circuit(2, [W.Gate("X", (0,))])
    assert np.argmax(np.abs(psi)) == 1
    psi = oracle.apply_circuit(2, [W.Gate("X", (1,))])
    assert np.argmax(np.abs(psi)) == 2
    s = SPEC["h_on_zero"]
    np.testing.assert_allclose(oracle.apply_circuit(1, [W.Gate("H", (0,))]).real, s["amps"], atol=s["tol"])
    al, be = 0.6, 0.8j
    np.testing.assert_allclose(oracle.apply_matrix(np.array([al, be]), oracle.gate_matrix("X"), [0]), [be, al])
    s = SPEC["bell"]
    bell = oracle.apply_circuit(2, [W.Gate("H", (0,)), W.Gate("X", (1,), (0,))])
    np.testing.assert_allclose(bell.real, s["amps"], atol=s["tol"])
    np.testing.assert_allclose(bell.imag, 0, atol=1e-16)
    s = SPEC["rx_pi_on_zero"]
    np.testing.assert_allclose(oracle.apply_circuit(1, [W.Gate("RX", (0,), offset=np.pi)]),
                               np.array(s["re"]) + 1j * np.array(s["im"]), atol=1e-15)
    # control not set: CNOT on |00> leaves it unchanged
    np.testing.assert_array_equal(oracle.apply_circuit(2, [W.Gate("X", (1,), (0,))]), [1, 0, 0, 0])


def test_norm_and_mirror():
    """Norm 1 within 1e-9 after 10^3 gates; C C^-1 |0> = |0>."""
    w = W.random_complex(6, 170, seed=5, extra_kinds=("MAT1", "MAT2", "XLIKE", "PS"))
    gates = w.gates
    assert len(gates) >= 1000
    psi = oracle.apply_circuit(6, gates)
    assert abs(np.vdot(psi, psi).real - 1) < 1e-9
    m = oracle.apply_circuit(6, W.mirror(gates[:300]))
    assert abs(m[0] - 1) < 1e-11 and np.max(np.abs(m[1:])) < 1e-11
    back = oracle.apply_circuit_dagger(6, gates[:300], None, oracle.apply_circuit(6, gates[:300]))
    assert abs(back[0] - 1) < 1e-11


# ----------------------------------------------------------------------------- expectation

def test_expectation_spec_values():
    z = SPEC
    one = oracle.apply_circuit(1, [W.Gate("X", (0,))])
    assert oracle.expectation(oracle.zero_state(1), [(1.0, {0: "Z"})])[0] == z["z0_on_zero"]["value"]
    assert oracle.expectation(one, [(1.0, {0: "Z"})])[0] == z["z0_on_one"]["value"]
    s01 = oracle.apply_circuit(2, [W.Gate("X", (0,))])  # |01> in the paper's ket order: qubit 0 = 1
    assert abs(oracle.expectation(s01, [(0.5, {0: "Z"}), (0.5, {1: "Z"})])[0] - z["half_z0_z1_on_01"]["value"]) < 1e-15
    r = oracle.apply_circuit(1, [W.Gate("RX", (0,), offset=np.pi / 3)])
    assert abs(oracle.expectation(r, [(1.0, {0: "Z"})])[0] - z["rx_pi3_z"]["value"]) < 1e-15
    bell = oracle.apply_circuit(2, [W.Gate("H", (0,)), W.Gate("X", (1,), (0,))])
    assert abs(oracle.expectation(bell, [(1.0, {0: "X", 1: "X"})])[0] - z["x0x1_bell"]["value"]) < 1e-15


@pytest.mark.parametrize("seed", range(6))
def test_expectation_vs_dense(seed):
    """<psi|H|psi> vs the dense Kronecker H, and Im ~ 0 (Hermitian H)."""
    n = 1 + seed % 6
    psi = W.random_state(n, seed)
    ham = W.random_hamiltonian(n, 12, seed)
    re, im = oracle.expectation(psi, ham)
    ref = np.vdot(psi, B.dense_hamiltonian(ham, n) @ psi)
    assert abs(re - ref.real) < 1e-12 and abs(im) < 1e-12


def test_triangle_maxcut_ground():
    edges = [(0, 1), (1, 2), (0, 2)]
    ham = W.maxcut_hamiltonian(edges)
    vals = []
    for b in range(8):
        psi = np.zeros(8, dtype=complex); psi[b] = 1
        e = oracle.expectation(psi, ham)[0]
        cut = sum(((b >> u) & 1) != ((b >> v) & 1) for u, v in edges)
        assert e == -cut  # diagonal: E on a basis state is -cut exactly
        vals.append(e)
    assert min(vals) == SPEC["triangle_maxcut"]["ground"]


# ----------------------------------------------------------------------------- C1 worked example

def test_c1_worked_example():
    w = W.c1_ghz_rx(C1G["theta"])
    psi = oracle.apply_circuit(w.n, w.gates, w.params)
    amps = np.array([a + 1j * b for a, b in C1G["amps_0_to_7"]])
    np.testing.assert_allclose(psi[:8], amps, atol=C1G["tol"])
    np.testing.assert_allclose(psi[8:], psi[7::-1], atol=1e-15)
    E, g = oracle.adjoint_grad(w.n, w.gates, w.params, w.ham)
    assert abs(E - C1G["E"]) < C1G["tol"]
    np.testing.assert_allclose(g, C1G["grad"], atol=C1G["tol"])


def test_c1_closed_form_many_angles():
    rng = np.random.default_rng(1)
    for _ in range(20):
        th = rng.uniform(-np.pi, np.pi, 4)
        w = W.c1_ghz_rx(th)
        E, g = oracle.adjoint_grad(w.n, w.gates, w.params, w.ham)
        assert abs(E - np.cos(th[0]) * np.cos(th[1])) < 1e-13
        np.testing.assert_allclose(g, [-np.sin(th[0]) * np.cos(th[1]), -np.cos(th[0]) * np.sin(th[1]), 0, 0], atol=1e-13)


# ----------------------------------------------------------------------------- gradients

def test_rx_z_anchor_grid():
    """RX(t)/<Z>: (cos t, -sin t) at 20 grid points <= 1e-12 (S:452-453, S:700 criterion 3)."""
    for t in np.linspace(-np.pi, np.pi, 20):
        E, g = oracle.adjoint_grad(1, [W.Gate("RX", (0,), param=0)], [t], [(1.0, {0: "Z"})])
        assert abs(E - np.cos(t)) < 1e-12 and abs(g[0] + np.sin(t)) < 1e-12
    E, g = oracle.adjoint_grad(1, [W.Gate("RX", (0,), param=0)], [0.0], [(1.0, {0: "Z"})])
    assert E == SPEC["rx_zero_z"]["value"] and g[0] == SPEC["rx_zero_z"]["grad"]
    E, g = oracle.adjoint_grad(1, [W.Gate("RX", (0,), param=0)], [np.pi / 3], [(1.0, {0: "Z"})])
    assert abs(g[0] - SPEC["rx_pi3_z"]["grad"]) < SPEC["rx_pi3_z"]["tol"]


def test_chain_rule_and_shared_parameters():
    """2a + 0.5b feeding RX as RX(2a) RX(0.5b) (reading in DESIGN.md); shared RX(a) on q0, q1
    with H = Z0 + Z1 -> -2 sin a."""
    a, b = 0.4, -1.3
    gates = [W.Gate("RX", (0,), param=0, coeff=2.0), W.Gate("RX", (0,), param=1, coeff=0.5)]
    E, g = oracle.adjoint_grad(1, gates, [a, b], [(1.0, {0: "Z"})])
    ang = 2 * a + 0.5 * b
    assert abs(E - np.cos(ang)) < 1e-14
    np.testing.assert_allclose(g, [-2 * np.sin(ang), -0.5 * np.sin(ang)], atol=1e-14)
    gates = [W.Gate("RX", (0,), param=0), W.Gate("RX", (1,), param=0)]
    E, g = oracle.adjoint_grad(2, gates, [a], [(1.0, {0: "Z"}), (1.0, {1: "Z"})])
    assert abs(g[0] + 2 * np.sin(a)) < 1e-14


@pytest.mark.parametrize("seed", range(8))
def test_adjoint_vs_shift_and_fd(seed):
    """Three-way agreement on random tasks with controls (corrected for controlled R_P by
    the 4-term rule, reading c2.10): adjoint vs exact shift <= 1e-10, vs central FD <= 1e-6."""
    n = 3 + seed % 3
    w = W.random_complex(n, 5, seed=100 + seed, n_params=4, extra_kinds=("PS", "MAT1", "MAT2"))
    ham = W.random_hamiltonian(n, 6, seed)
    psi0 = W.random_state(n, seed)
    E, g = oracle.adjoint_grad(n, w.gates, w.params, ham, psi0)
    gs = oracle.shift_grad(n, w.gates, w.params, ham, psi0)
    np.testing.assert_allclose(g, gs, atol=1e-10)
    assert abs(E - oracle.energy(n, w.gates, w.params, ham, psi0)) < 1e-13
    h = 1e-5
    for p in range(len(w.params)):
        d = np.zeros_like(w.params); d[p] = h
        fd = (oracle.energy(n, w.gates, w.params + d, ham, psi0) - oracle.energy(n, w.gates, w.params - d, ham, psi0)) / (2 * h)
        assert abs(fd - g[p]) < 1e-6


def test_two_term_rule_fails_for_controlled_rotation():
    """Reading c2.10: the 2-term rule is NOT exact for controlled R_P — guards the 4-term branch."""
    gates = [W.Gate("H", (0,)), W.Gate("H", (1,)), W.Gate("RY", (1,), (0,), param=0)]
    ham = [(1.0, {0: "X"})]  # couples the control branches, so the frequency-1/2 component appears
    t = 0.9
    _, g = oracle.adjoint_grad(2, gates, [t], ham)
    two = 0.5 * (oracle.energy(2, gates, [t + np.pi / 2], ham) - oracle.energy(2, gates, [t - np.pi / 2], ham))
    assert abs(two - g[0]) > 1e-3
    assert abs(oracle.shift_grad(2, gates, [t], ham)[0] - g[0]) < 1e-14


def test_gradient_linear_in_h():
    n = 4
    w = W.random_complex(n, 5, seed=9, n_params=3)
    h1, h2 = W.random_hamiltonian(n, 4, 1), W.random_hamiltonian(n, 5, 2)
    e1, g1 = oracle.adjoint_grad(n, w.gates, w.params, h1)
    e2, g2 = oracle.adjoint_grad(n, w.gates, w.params, h2)
    e3, g3 = oracle.adjoint_grad(n, w.gates, w.params, h1 + h2)
    assert abs(e1 + e2 - e3) < 1e-12
    np.testing.assert_allclose(g1 + g2, g3, atol=1e-12)


def test_non_differentiable_rejected():
    with pytest.raises(ValueError):
        oracle.adjoint_grad(1, [W.Gate("MAT1", (0,), param=0, mat=np.eye(2))], [0.1], [(1.0, {0: "Z"})])


def _qaoa_p1_closed_form(edges, n, gamma, beta):
    """Wang, Hadfield, Jiang, Rieffel, PRA 97 022304 (2018), eq. for <C_uv> at p = 1, with the
    circuit's Rzz(2 gamma), RX(2 beta): gamma_W = -2 gamma, beta_W = beta. E = -sum <C_uv>."""
    adj = {q: set() for q in range(n)}
    for u, v in edges:
        adj[u].add(v); adj[v].add(u)
    gw, bw = -2 * gamma, beta
    tot = 0.0
    for u, v in edges:
        du, dv, lam = len(adj[u]) - 1, len(adj[v]) - 1, len(adj[u] & adj[v])
        tot += (0.5 + 0.25 * np.sin(4 * bw) * np.sin(gw) * (np.cos(gw) ** du + np.cos(gw) ** dv)
                - 0.25 * np.sin(2 * bw) ** 2 * np.cos(gw) ** (du + dv - 2 * lam) * (1 - np.cos(2 * gw) ** lam))
    return -tot


@pytest.mark.parametrize("n,seed", [(8, 3), (10, 5), (12, 7)])
def test_qaoa_p1_closed_form(n, seed):
    """E and the shared-parameter gradient of p=1 QAOA vs the closed form (and its derivative by
    central differences of the closed form)."""
    w = W.qaoa(n, 1, seed_graph=seed, seed_angles=seed)
    edges = w.meta["edges"]
    gam, bet = w.params
    E, g = oracle.adjoint_grad(n, w.gates, w.params, w.ham)
    assert abs(E - _qaoa_p1_closed_form(edges, n, gam, bet)) < 1e-12
    h = 1e-6
    dg = (_qaoa_p1_closed_form(edges, n, gam + h, bet) - _qaoa_p1_closed_form(edges, n, gam - h, bet)) / (2 * h)
    db = (_qaoa_p1_closed_form(edges, n, gam, bet + h) - _qaoa_p1_closed_form(edges, n, gam, bet - h)) / (2 * h)
    np.testing.assert_allclose(g, [dg, db], atol=1e-8)


def test_qaoa_zero_parameters():
    """All-zero parameters: psi = |+>^n, every amplitude 2^(-n/2), E = -|E|/2, g = 0."""
    w = W.qaoa(10, 2, seed_graph=11, seed_angles=11)
    z = np.zeros_like(w.params)
    psi = oracle.apply_circuit(w.n, w.gates, z)
    np.testing.assert_allclose(psi, 2 ** (-w.n / 2), atol=1e-14)
    E, g = oracle.adjoint_grad(w.n, w.gates, z, w.ham)
    assert abs(E + len(w.meta["edges"]) / 2) < 1e-12
    np.testing.assert_allclose(g, 0, atol=1e-12)


# ----------------------------------------------------------------------------- density matrices

def test_density_oracle_pins():
    """§3.2: pure-state rho equals |psi><psi| of the state-vector oracle (S:700 #5),
    tr(rho) = 1, <H> = tr(rho H) equals the state-vector expectation, and a mixture is the convex
    combination of its components (linearity of rho -> U rho U^dagger)."""
    n = 3
    w = W.random_complex(n, 4, seed=21, n_params=2)
    psi = oracle.apply_circuit(n, w.gates, w.params)
    rho = oracle.dm_apply_circuit(n, w.gates, w.params)
    np.testing.assert_allclose(rho, np.outer(psi, psi.conj()), atol=1e-13)
    assert abs(np.trace(rho) - 1) < 1e-13
    ham = W.random_hamiltonian(n, 6, seed=3)
    assert abs(oracle.dm_expectation(rho, ham) - oracle.expectation(psi, ham)[0]) < 1e-13
    a, b = W.random_state(n, 1), W.random_state(n, 2)
    mix = 0.3 * np.outer(a, a.conj()) + 0.7 * np.outer(b, b.conj())
    out = oracle.dm_apply_circuit(n, w.gates, w.params, mix)
    pa, pb = oracle.apply_circuit(n, w.gates, w.params, a), oracle.apply_circuit(n, w.gates, w.params, b)
    np.testing.assert_allclose(out, 0.3 * np.outer(pa, pa.conj()) + 0.7 * np.outer(pb, pb.conj()), atol=1e-13)
    # Pauli matrices vs Kronecker products (independent construction)
    term = {0: "X", 2: "Y"}
    np.testing.assert_allclose(oracle.pauli_matrix(n, term), B.kron_list({0: B.PX, 2: B.PY}, n), atol=1e-15)


# ----------------------------------------------------------------------------- sampling (NEXT-2)
# "Sampling Measurement" (Fig. 1): or_sample is the plain inverse
# CDF of |psi|^2 driven by the counter-based SplitMix64 uniforms of the sv_sample contract.

SPLITMIX = json.load(open(os.path.join(GOLD, "splitmix64.json")))


def test_splitmix64_reference_outputs():
    g = int(SPLITMIX["golden"], 16)
    for k, ref in enumerate(SPLITMIX["stream_from_state_0"]):
        assert oracle.splitmix64((k * g) % (1 << 64)) == int(ref, 16)


def test_sample_spec_examples():
    """|0> -> all 0; |+> -> count of 0 within 5 sigma of 50000 at 1e5 shots; Bell state
    -> only 00 and 11 appear (zero-probability outcomes are never drawn)."""
    zero = oracle.zero_state(1)
    assert np.all(oracle.sample(zero, [0], 100, seed=1) == 0)
    plus = np.array([1, 1], dtype=np.complex128) / np.sqrt(2)
    ones = int(np.sum(oracle.sample(plus, [0], 100000, seed=2)))
    assert abs(ones - 50000) < 5 * np.sqrt(100000 * 0.25)
    bell = np.array([1, 0, 0, 1], dtype=np.complex128) / np.sqrt(2)
    assert set(np.unique(oracle.sample(bell, [0, 1], 10000, seed=3)).tolist()) == {0, 3}


def test_sample_worked_draws():
    """Hand-worked: probabilities (1/4, 0, 3/4, 0). With seed 0 the uniforms are the published
    SplitMix64 outputs / 2^64 (u_0 = 0xe220a8397b1dcdaf >> 11 / 2^53 = 0.8833...): a draw lands on
    index 0 iff u <= 1/4, else on index 2; indices 1 and 3 (probability 0) never appear."""
    psi = np.array([0.5, 0, np.sqrt(0.75), 0], dtype=np.complex128)
    g = int(SPLITMIX["golden"], 16)
    # seed = k * golden makes shot 0 of each call the k-th published output
    for k, ref in enumerate(SPLITMIX["stream_from_state_0"]):
        u = (int(ref, 16) >> 11) / 2.0 ** 53
        idx = oracle.sample_indices(psi, 1, seed=(k * g) % (1 << 64))[0]
        assert idx == (0 if u * 1.0 <= 0.25 else 2), (k, u, idx)
    idx = oracle.sample_indices(psi, 20000, seed=5)
    assert set(np.unique(idx).tolist()) <= {0, 2}
    assert abs(np.mean(idx == 0) - 0.25) < 5 * np.sqrt(0.25 * 0.75 / 20000)


def test_sample_frequencies_match_probabilities():
    """Empirical frequencies of 2e5 shots on a random 4-qubit state match |psi_i|^2 (every outcome
    within 5 sigma); the marginal over a qubit subset is the bits of the full draw."""
    psi = W.random_state(4, 77)
    p = np.abs(psi) ** 2
    shots = 200000
    idx = oracle.sample_indices(psi, shots, seed=11)
    freq = np.bincount(idx, minlength=16) / shots
    assert np.all(np.abs(freq - p) < 5 * np.sqrt(p * (1 - p) / shots) + 1e-12)
    sub = oracle.sample(psi, [3, 1], shots, seed=11)
    assert np.array_equal(sub, ((idx >> 3) & 1) | (((idx >> 1) & 1) << 1))
    # deterministic under the seed, different under another seed
    assert np.array_equal(idx, oracle.sample_indices(psi, shots, seed=11))
    assert not np.array_equal(idx, oracle.sample_indices(psi, shots, seed=12))


def test_oracle_adjoint_cost_contract():
    """S:478 / S:695: the adjoint gradient performs one forward pass and one backward sweep with two
    un-applications per gate — 3N gate applications, independent of the parameter count P (the
    instrumented counter of or_apply_gate); parameter-shift needs O(N P)."""
    for P in (1, 4, 12):
        w = W.random_complex(6, 6, seed=P, n_params=P)
        ham = W.random_hamiltonian(6, 5, seed=P)
        N = len(w.gates)
        oracle.reset_gate_applications()
        oracle.adjoint_grad(6, w.gates, w.params, ham)
        assert oracle.gate_applications() == 3 * N, (P, oracle.gate_applications(), N)
        oracle.reset_gate_applications()
        oracle.shift_grad(6, w.gates, w.params, ham)
        assert oracle.gate_applications() > 3 * N  # the shift rule re-evaluates per occurrence
