"""Seeded synthetic input generators shared by the tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic: it only draws circuits (gate kind names,
qubit indices, parameter indices, linear angle coefficients, Haar-random user matrices) and
Pauli-sum Hamiltonians with numpy's PCG64. Gate matrices, index arithmetic, Pauli actions,
expectations and gradients live separately in `oracle/` (test oracle) and in
`paper_2406_17248_b200/` (the CUDA product path); each side maps kind NAMES to its own codes.

Workload shapes follow the paper's benchmarks (recipe in DESIGN.md §Inputs):
  * random "complex" circuits over the §7.1 gate set X,Y,Z,H,CNOT,S,T,RX,RY,RZ,Rxx,Ryy,Rzz,SWAP
    "and its control version";
  * QAOA max-cut with a one-step Trotter ansatz (§7.2);
  * hardware-efficient VQE ansatz + JW-shaped molecular Pauli sums (Fig. 1 "Ansatz Library",
    P:339; VQE);
  * configs C1..C5 of BASELINE.json.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

KINDS_1Q = ("X", "Y", "Z", "H", "S", "SDG", "T", "TDG", "RX", "RY", "RZ", "PS", "XLIKE", "ZLIKE", "MAT1")
KINDS_2Q = ("SWAP", "RXX", "RYY", "RZZ", "MAT2")
ALL_KINDS = KINDS_1Q + KINDS_2Q
PARAM_KINDS = ("RX", "RY", "RZ", "PS", "RXX", "RYY", "RZZ")


@dataclass(frozen=True)
class Gate:
    """One gate instruction (SPEC.md S:104 GateInstruction; Fig. 1 "Any control on any gate").

    angle = coeff * params[param] + offset (param >= 0), else offset (fixed angle).
    mat: XLIKE/ZLIKE -> complex (a, b); MAT1 -> complex 2x2; MAT2 -> complex 4x4 with matrix
    index bit j <-> targets[j]. Ignored for other kinds.
    """
    kind: str
    targets: Tuple[int, ...]
    controls: Tuple[int, ...] = ()
    param: int = -1
    coeff: float = 1.0
    offset: float = 0.0
    mat: Optional[np.ndarray] = field(default=None, compare=False)


# A Pauli term: (real coefficient, {qubit: 'X'|'Y'|'Z'}); identity where absent.
PauliTerm = Tuple[float, Dict[int, str]]


@dataclass
class Workload:
    name: str
    n: int
    gates: List[Gate]
    params: np.ndarray
    ham: List[PauliTerm]
    meta: dict = field(default_factory=dict)


# ----------------------------------------------------------------------------- primitives

def haar_unitary(d: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-random d x d unitary: QR of a complex Ginibre matrix with R's diagonal phases
    divided out (Mezzadri 2007)."""
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / np.sqrt(2.0)
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph[None, :]


def random_state(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return v / np.linalg.norm(v)


def random_regular_graph(n: int, d: int, seed: int) -> List[Tuple[int, int]]:
    """Random d-regular simple graph by the configuration model with rejection of self-loops and
    multi-edges (whole-draw restart)."""
    rng = np.random.default_rng(seed)
    assert (n * d) % 2 == 0
    while True:
        stubs = np.repeat(np.arange(n), d)
        rng.shuffle(stubs)
        pairs = stubs.reshape(-1, 2)
        edges = set()
        ok = True
        for u, v in pairs:
            u, v = int(min(u, v)), int(max(u, v))
            if u == v or (u, v) in edges:
                ok = False
                break
            edges.add((u, v))
        if ok:
            return sorted(edges)


# ----------------------------------------------------------------------------- Hamiltonians

def maxcut_hamiltonian(edges: Sequence[Tuple[int, int]]) -> List[PauliTerm]:
    """H = sum_(u,v) 1/2 (Z_u Z_v - I) (reading c2.21). The identity parts are
    merged into one identity term -|E|/2."""
    ham: List[PauliTerm] = [(0.5, {u: "Z", v: "Z"}) for (u, v) in edges]
    ham.append((-0.5 * len(edges), {}))
    return ham


def jw_hamiltonian(n: int, nterms: int, seed: int) -> List[PauliTerm]:
    """JW-shaped molecular Pauli sum (SURVEY.md §8(d) recipe): 20% Z_i, 20% Z_i Z_j, 40% hopping
    X_i Z..Z X_j or Y_i Z..Z Y_j, 20% four-body X/Y products with JW Z-strings; coefficients
    U[-1, 1]; duplicate strings redrawn."""
    rng = np.random.default_rng(seed)
    n_z = nterms // 5
    n_zz = nterms // 5
    n_four = nterms // 5
    n_hop = nterms - n_z - n_zz - n_four
    seen = set()
    out: List[PauliTerm] = []

    def add(term: Dict[int, str]) -> bool:
        key = tuple(sorted(term.items()))
        if key in seen or not term:
            return False
        seen.add(key)
        out.append((float(rng.uniform(-1.0, 1.0)), dict(term)))
        return True

    def draw_z():
        return {int(rng.integers(n)): "Z"}

    def draw_zz():
        i, j = rng.choice(n, 2, replace=False)
        return {int(i): "Z", int(j): "Z"}

    def draw_hop():
        i, j = sorted(int(x) for x in rng.choice(n, 2, replace=False))
        p = "X" if rng.random() < 0.5 else "Y"
        t = {i: p, j: p}
        for q in range(i + 1, j):
            t[q] = "Z"
        return t

    def draw_four():
        qs = sorted(int(x) for x in rng.choice(n, 4, replace=False))
        t = {q: ("X" if rng.random() < 0.5 else "Y") for q in qs}
        # JW strings between the two creation/annihilation pairs
        for q in range(qs[0] + 1, qs[1]):
            t[q] = "Z"
        for q in range(qs[2] + 1, qs[3]):
            t[q] = "Z"
        return t

    for count, draw in ((n_z, draw_z), (n_zz, draw_zz), (n_hop, draw_hop), (n_four, draw_four)):
        made = 0
        tries = 0
        while made < count and tries < 100000:
            tries += 1
            if add(draw()):
                made += 1
    return out


def random_hamiltonian(n: int, nterms: int, seed: int, max_weight: Optional[int] = None) -> List[PauliTerm]:
    """Uniformly random Pauli strings (weight 0..max_weight) with U[-1,1] coefficients."""
    rng = np.random.default_rng(seed)
    mw = n if max_weight is None else max_weight
    out: List[PauliTerm] = []
    for _ in range(nterms):
        w = int(rng.integers(0, mw + 1))
        qs = rng.choice(n, w, replace=False) if w else []
        out.append((float(rng.uniform(-1, 1)), {int(q): "XYZ"[int(rng.integers(3))] for q in qs}))
    return out


# ----------------------------------------------------------------------------- circuits

def c1_ghz_rx(theta: Sequence[float] = (0.3, -1.1, 2.0, 0.7)) -> Workload:
    """C1: n=4, H(0); CNOT(0->1),(1->2),(2->3); RX(theta_q) on each qubit q (param q);
    H = Z0 + Z0 Z1 (reading c2.19)."""
    g = [Gate("H", (0,))]
    g += [Gate("X", (q + 1,), (q,)) for q in range(3)]
    g += [Gate("RX", (q,), param=q) for q in range(4)]
    ham = [(1.0, {0: "Z"}), (1.0, {0: "Z", 1: "Z"})]
    return Workload("C1", 4, g, np.asarray(theta, dtype=np.float64), ham)


def hea(n: int, layers: int, seed: int, nterms: int = 50) -> Workload:
    """C2 (and C4g): hardware-efficient ansatz, each layer RY(theta) on every qubit, RZ(theta) on
    every qubit, CNOT(q -> q+1) ladder; theta ~ U[0, 2pi); JW-shaped H."""
    rng = np.random.default_rng(seed)
    g: List[Gate] = []
    p = 0
    for _ in range(layers):
        for kind in ("RY", "RZ"):
            for q in range(n):
                g.append(Gate(kind, (q,), param=p))
                p += 1
        for q in range(n - 1):
            g.append(Gate("X", (q + 1,), (q,)))
    params = rng.uniform(0, 2 * np.pi, p)
    return Workload(f"HEA{n}x{layers}", n, g, params, jw_hamiltonian(n, nterms, seed))


def qaoa(n: int, p: int, seed_graph: int, seed_angles: int, dc: bool = False, degree: int = 3) -> Workload:
    """C3: QAOA max-cut on a random `degree`-regular graph: H on every qubit, then p blocks of
    [Rzz(2 gamma_k) per edge, RX(2 beta_k) per node] (+ RY(2 alpha_k) per node for the DC-QAOA
    variant, reading c2.20). Params: gamma_0..p-1, beta_0..p-1 (, alpha_0..p-1)."""
    edges = random_regular_graph(n, degree, seed_graph)
    rng = np.random.default_rng(seed_angles)
    g: List[Gate] = [Gate("H", (q,)) for q in range(n)]
    for k in range(p):
        g += [Gate("RZZ", (u, v), param=k, coeff=2.0) for (u, v) in edges]
        g += [Gate("RX", (q,), param=p + k, coeff=2.0) for q in range(n)]
        if dc:
            g += [Gate("RY", (q,), param=2 * p + k, coeff=2.0) for q in range(n)]
    nparam = (3 if dc else 2) * p
    params = rng.uniform(0, np.pi, nparam)
    return Workload(f"QAOA{n}p{p}{'dc' if dc else ''}", n, g, params, maxcut_hamiltonian(edges),
                    meta={"edges": edges})


def random_circuit(n: int, depth: int, seed: int) -> Workload:
    """C4/C5: per layer l a Haar-random 1q matrix (MAT1) on every qubit, then CZ on
    (0,1),(2,3),... for even l and (1,2),(3,4),... for odd l (reading c2.18)."""
    rng = np.random.default_rng(seed)
    g: List[Gate] = []
    for layer in range(depth):
        for q in range(n):
            g.append(Gate("MAT1", (q,), mat=haar_unitary(2, rng)))
        for q in range(layer % 2, n - 1, 2):
            g.append(Gate("Z", (q + 1,), (q,)))
    return Workload(f"RAND{n}d{depth}", n, g, np.zeros(0), [])


PAPER_GATE_SET = ("X", "Y", "Z", "H", "S", "T", "RX", "RY", "RZ", "RXX", "RYY", "RZZ", "SWAP")


def random_complex(n: int, gates_per_qubit: int, seed: int, p_control: float = 0.3,
                   n_params: int = 0, extra_kinds: Sequence[str] = ()) -> Workload:
    """CP: the paper's "complex random circuit" shape — gates drawn uniformly from the §7.1 set
    X,Y,Z,H,S,T,RX,RY,RZ,Rxx,Ryy,Rzz,SWAP (CNOT = X + control) with each gate controlled with
    probability p_control (SPEC.md S:678 generator). Rotations take a shared parameter
    index when n_params > 0 (coeff ~ U[-2,2], offset ~ U[-1,1]), else a fixed random angle."""
    rng = np.random.default_rng(seed)
    kinds = tuple(PAPER_GATE_SET) + tuple(extra_kinds)
    g: List[Gate] = []
    for _ in range(gates_per_qubit):
        for q in range(n):
            kind = kinds[int(rng.integers(len(kinds)))]
            two = kind in KINDS_2Q
            if two and n < 2:
                kind, two = "H", False
            if two:
                other = int(rng.choice([x for x in range(n) if x != q]))
                targets = (q, other)
            else:
                targets = (q,)
            free = [x for x in range(n) if x not in targets]
            controls: Tuple[int, ...] = ()
            if free and rng.random() < p_control:
                nc = 1 if rng.random() < 0.7 or len(free) < 2 else 2
                controls = tuple(int(x) for x in rng.choice(free, nc, replace=False))
            mat = None
            if kind == "MAT1":
                mat = haar_unitary(2, rng)
            elif kind == "MAT2":
                mat = haar_unitary(4, rng)
            elif kind in ("XLIKE", "ZLIKE"):
                mat = np.exp(1j * rng.uniform(0, 2 * np.pi, 2))
            if kind in PARAM_KINDS:
                if n_params > 0:
                    g.append(Gate(kind, targets, controls, param=int(rng.integers(n_params)),
                                  coeff=float(rng.uniform(-2, 2)), offset=float(rng.uniform(-1, 1))))
                else:
                    g.append(Gate(kind, targets, controls, offset=float(rng.uniform(0, 2 * np.pi))))
            else:
                g.append(Gate(kind, targets, controls, mat=mat))
    params = rng.uniform(0, 2 * np.pi, n_params)
    return Workload(f"CP{n}x{gates_per_qubit}", n, g, params, [])


def mirror(gates: Sequence[Gate]) -> List[Gate]:
    """C followed by C^-1 expressed with gate-level inverses (needs only kind names):
    rotations negate coeff/offset, S<->SDG, T<->TDG, self-inverse kinds repeat, user matrices
    are conjugate-transposed (a pure data transform on the drawn input)."""
    inv: List[Gate] = []
    swap = {"S": "SDG", "SDG": "S", "T": "TDG", "TDG": "T"}
    for gt in reversed(gates):
        k = gt.kind
        if k in PARAM_KINDS:
            inv.append(Gate(k, gt.targets, gt.controls, gt.param, -gt.coeff, -gt.offset))
        elif k in swap:
            inv.append(Gate(swap[k], gt.targets, gt.controls))
        elif k in ("MAT1", "MAT2"):
            inv.append(Gate(k, gt.targets, gt.controls, mat=np.conj(np.asarray(gt.mat)).T))
        elif k == "XLIKE":  # [[0,a],[b,0]]^dagger = [[0, conj b],[conj a, 0]]
            a, b = gt.mat
            inv.append(Gate(k, gt.targets, gt.controls, mat=np.array([np.conj(b), np.conj(a)])))
        elif k == "ZLIKE":
            inv.append(Gate(k, gt.targets, gt.controls, mat=np.conj(np.asarray(gt.mat))))
        else:
            inv.append(gt)
    return list(gates) + inv


# ----------------------------------------------------------------------------- configs

def config(name: str) -> Workload:
    """BASELINE.json configs by name (seeds in DESIGN.md §Inputs)."""
    if name == "C1":
        return c1_ghz_rx()
    if name == "C2":
        return hea(20, 10, seed=2002)
    if name == "C3":
        return qaoa(24, 8, seed_graph=2403, seed_angles=2404)
    if name == "C3dc":
        return qaoa(24, 8, seed_graph=2403, seed_angles=2404, dc=True)
    if name == "C4":
        w = random_circuit(30, 40, seed=3040)
        w.ham = jw_hamiltonian(30, 50, 3030)
        return w
    if name == "C4g":
        return hea(30, 2, seed=3030)
    if name == "C5":
        w = random_circuit(34, 40, seed=3440)
        w.ham = jw_hamiltonian(34, 50, 3440)
        return w
    raise KeyError(name)


def fullsize_case(name: str) -> Workload:
    """Full-size oracle parity cases (tests/golden/fullsize_<name>.npz, tools/gen_golden_fullsize.py):
    C3 / C3dc as benched; the C4 generator at 26q full depth; C4 itself truncated to its first 4
    layers (30q, 178 gates); the C4g generator at 26q."""
    if name in ("C3", "C3dc"):
        return config(name)
    if name == "C4_26":
        w = random_circuit(26, 40, seed=3040)
        w.ham = jw_hamiltonian(26, 50, 3030)
        return w
    if name == "C4_30d4":
        w = config("C4")
        w.gates = w.gates[: 2 * (30 + 15 + 30 + 14)]  # layers 0..3 (even: 15 CZ, odd: 14 CZ)
        return w
    if name == "C4g_26":
        return hea(26, 2, seed=3030)
    raise KeyError(name)


# ----------------------------------------------------------------------------- neutral arrays

def gate_arrays(gates: Sequence[Gate]) -> dict:
    """Neutral column arrays (no arithmetic): kind names, targets (G,2) int32 (second = -1 for
    1q kinds), control masks uint64, param int32, coeff/offset float64, mats (G,32) float64 with
    the user matrix as row-major interleaved (re, im) (zeros when absent)."""
    G = len(gates)
    targets = np.full((G, 2), -1, dtype=np.int32)
    cmask = np.zeros(G, dtype=np.uint64)
    param = np.full(G, -1, dtype=np.int32)
    coeff = np.ones(G, dtype=np.float64)
    offset = np.zeros(G, dtype=np.float64)
    mats = np.zeros((G, 32), dtype=np.float64)
    kinds = []
    for i, gt in enumerate(gates):
        kinds.append(gt.kind)
        targets[i, : len(gt.targets)] = gt.targets
        m = 0
        for c in gt.controls:
            m |= 1 << int(c)
        cmask[i] = m
        param[i] = gt.param
        coeff[i] = gt.coeff
        offset[i] = gt.offset
        if gt.mat is not None:
            flat = np.asarray(gt.mat, dtype=np.complex128).reshape(-1)
            mats[i, 0: 2 * flat.size: 2] = flat.real
            mats[i, 1: 2 * flat.size: 2] = flat.imag
    return dict(kinds=kinds, targets=targets, cmask=cmask, param=param, coeff=coeff, offset=offset, mats=mats)
