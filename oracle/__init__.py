"""ctypes wrapper of the plain-C CPU oracle (oracle/sv_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs. Never imported by the product package
(paper_2406_17248_b200/), which must fail loudly rather than fall back to anything here.

Marshalling only: every step of the computation happens in sv_oracle.c (see its header for the
paper passage each function follows).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# Oracle-private kind codes — must match the enum at the top of sv_oracle.c.
KIND_CODE: Dict[str, int] = {k: i for i, k in enumerate(
    ["X", "Y", "Z", "H", "S", "SDG", "T", "TDG", "RX", "RY", "RZ", "PS", "XLIKE", "ZLIKE", "MAT1",
     "SWAP", "RXX", "RYY", "RZZ", "MAT2"])}
PAULI_CODE = {"X": 1, "Y": 2, "Z": 3}

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -ffp-contract=off, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, u64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        L.or_gate_matrix.argtypes = [ctypes.c_int, f64, P, P]
        L.or_gate_matrix.restype = ctypes.c_int
        L.or_apply_matrix.argtypes = [P, ctypes.c_int, ctypes.c_int, P, u64, P]
        L.or_apply_matrix.restype = None
        circ = [P, P, P, P, P, P, P]
        L.or_apply_circuit.argtypes = [P, ctypes.c_int, i64] + circ + [P, i64, f64]
        L.or_apply_circuit.restype = None
        L.or_apply_circuit_dagger.argtypes = [P, ctypes.c_int, i64] + circ + [P]
        L.or_apply_circuit_dagger.restype = None
        L.or_expectation.argtypes = [P, ctypes.c_int, i64, P, P, P, P]
        L.or_expectation.restype = None
        L.or_adjoint_grad.argtypes = [P, ctypes.c_int, i64] + circ + [P, i32, i64, P, P, P, P]
        L.or_adjoint_grad.restype = ctypes.c_int
        L.or_shift_grad.argtypes = [P, ctypes.c_int, i64] + circ + [P, i32, i64, P, P, P]
        L.or_shift_grad.restype = ctypes.c_int
        L.or_splitmix64.argtypes = [u64]
        L.or_splitmix64.restype = u64
        L.or_sample.argtypes = [P, ctypes.c_int, i64, u64, P]
        L.or_sample.restype = None
        L.or_get_gate_applications.argtypes = []
        L.or_get_gate_applications.restype = i64
        L.or_reset_gate_applications.argtypes = []
        L.or_reset_gate_applications.restype = None
        L.or_state_zero.argtypes = [P, ctypes.c_int]
        L.or_state_zero.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class _Circ:
    """Keeps the marshalled gate columns alive for the duration of a call."""

    def __init__(self, gates):
        G = len(gates)
        self.n = G
        self.kinds = np.array([KIND_CODE[g.kind] for g in gates], dtype=np.int32)
        self.targets = np.full((max(G, 1), 2), -1, dtype=np.int32)
        self.cmask = np.zeros(max(G, 1), dtype=np.uint64)
        self.pidx = np.full(max(G, 1), -1, dtype=np.int32)
        self.coeff = np.ones(max(G, 1))
        self.offset = np.zeros(max(G, 1))
        self.mats = np.zeros((max(G, 1), 32))
        for i, g in enumerate(gates):
            self.targets[i, : len(g.targets)] = g.targets
            m = 0
            for c in g.controls:
                m |= 1 << int(c)
            self.cmask[i] = m
            self.pidx[i] = g.param
            self.coeff[i] = g.coeff
            self.offset[i] = g.offset
            if g.mat is not None:
                f = np.asarray(g.mat, dtype=np.complex128).reshape(-1)
                self.mats[i, 0: 2 * f.size: 2] = f.real
                self.mats[i, 1: 2 * f.size: 2] = f.imag
        if G == 0:
            self.kinds = np.zeros(1, dtype=np.int32)

    def args(self):
        return [_p(self.kinds), _p(self.targets), _p(self.cmask), _p(self.pidx), _p(self.coeff),
                _p(self.offset), _p(self.mats)]


class _Ham:
    def __init__(self, n: int, ham):
        T = len(ham)
        self.n = T
        self.ops = np.zeros((max(T, 1), n), dtype=np.uint8)
        self.coeffs = np.zeros(max(T, 1))
        for t, (c, term) in enumerate(ham):
            self.coeffs[t] = c
            for q, p in term.items():
                self.ops[t, q] = PAULI_CODE[p]


def zero_state(n: int) -> np.ndarray:
    psi = np.empty(1 << n, dtype=np.complex128)
    lib().or_state_zero(_p(psi), n)
    return psi


def gate_matrix(kind: str, phi: float = 0.0, mat=None) -> np.ndarray:
    user = np.zeros(32)
    if mat is not None:
        f = np.asarray(mat, dtype=np.complex128).reshape(-1)
        user[0: 2 * f.size: 2] = f.real
        user[1: 2 * f.size: 2] = f.imag
    out = np.zeros(32)
    d = lib().or_gate_matrix(KIND_CODE[kind], float(phi), _p(user), _p(out))
    return (out[0: 2 * d * d: 2] + 1j * out[1: 2 * d * d: 2]).reshape(d, d)


def apply_matrix(psi: np.ndarray, M: np.ndarray, targets: Sequence[int], controls: Sequence[int] = ()) -> np.ndarray:
    """Returns (Pi_C (x) M + (1-Pi_C) (x) I) psi (a copy)."""
    out = np.array(psi, dtype=np.complex128, copy=True)
    n = int(out.size).bit_length() - 1
    M = np.ascontiguousarray(M, dtype=np.complex128)
    t = np.array(list(targets) + [-1] * (2 - len(targets)), dtype=np.int32)
    cm = 0
    for c in controls:
        cm |= 1 << int(c)
    lib().or_apply_matrix(_p(out), n, len(targets), _p(t), cm, _p(M.view(np.float64)))
    return out


def apply_circuit(n: int, gates, params=None, psi0: Optional[np.ndarray] = None,
                  shift_gate: int = -1, shift: float = 0.0) -> np.ndarray:
    psi = zero_state(n) if psi0 is None else np.array(psi0, dtype=np.complex128, copy=True)
    params = np.ascontiguousarray(np.zeros(1) if params is None or len(params) == 0 else params, dtype=np.float64)
    c = _Circ(gates)
    lib().or_apply_circuit(_p(psi), n, c.n, *c.args(), _p(params), shift_gate, shift)
    return psi


def apply_circuit_dagger(n: int, gates, params=None, psi0: Optional[np.ndarray] = None) -> np.ndarray:
    psi = zero_state(n) if psi0 is None else np.array(psi0, dtype=np.complex128, copy=True)
    params = np.ascontiguousarray(np.zeros(1) if params is None or len(params) == 0 else params, dtype=np.float64)
    c = _Circ(gates)
    lib().or_apply_circuit_dagger(_p(psi), n, c.n, *c.args(), _p(params))
    return psi


def expectation(psi: np.ndarray, ham) -> Tuple[float, float]:
    psi = np.ascontiguousarray(psi, dtype=np.complex128)
    n = int(psi.size).bit_length() - 1
    h = _Ham(n, ham)
    re, im = ctypes.c_double(), ctypes.c_double()
    lib().or_expectation(_p(psi), n, h.n, _p(h.ops), _p(h.coeffs), ctypes.byref(re), ctypes.byref(im))
    return re.value, im.value


def adjoint_grad(n: int, gates, params, ham, psi0: Optional[np.ndarray] = None) -> Tuple[float, np.ndarray]:
    psi0 = zero_state(n) if psi0 is None else np.ascontiguousarray(psi0, dtype=np.complex128)
    params = np.ascontiguousarray(params, dtype=np.float64)
    P = len(params)
    pbuf = params if P else np.zeros(1)
    c = _Circ(gates)
    h = _Ham(n, ham)
    e = ctypes.c_double()
    g = np.zeros(max(P, 1))
    rc = lib().or_adjoint_grad(_p(psi0), n, c.n, *c.args(), _p(pbuf), P, h.n, _p(h.ops), _p(h.coeffs),
                               ctypes.byref(e), _p(g))
    if rc != 0:
        raise ValueError("non-differentiable gate carries a parameter")
    return e.value, g[:P]


def shift_grad(n: int, gates, params, ham, psi0: Optional[np.ndarray] = None) -> np.ndarray:
    psi0 = zero_state(n) if psi0 is None else np.ascontiguousarray(psi0, dtype=np.complex128)
    params = np.ascontiguousarray(params, dtype=np.float64)
    P = len(params)
    pbuf = params if P else np.zeros(1)
    c = _Circ(gates)
    h = _Ham(n, ham)
    g = np.zeros(max(P, 1))
    rc = lib().or_shift_grad(_p(psi0), n, c.n, *c.args(), _p(pbuf), P, h.n, _p(h.ops), _p(h.coeffs), _p(g))
    if rc != 0:
        raise ValueError("non-differentiable gate carries a parameter")
    return g[:P]


def gate_applications() -> int:
    """The oracle's instrumented gate-application counter (or_apply_gate calls since the last reset)."""
    return int(lib().or_get_gate_applications())


def reset_gate_applications() -> None:
    lib().or_reset_gate_applications()


def splitmix64(x: int) -> int:
    return int(lib().or_splitmix64(int(x) & ((1 << 64) - 1)))


def sample_indices(psi: np.ndarray, shots: int, seed: int) -> np.ndarray:
    """Basis index of every shot by the inverse CDF of |psi|^2 (or_sample, Fig. 1)."""
    psi = np.ascontiguousarray(psi, dtype=np.complex128)
    n = int(psi.size).bit_length() - 1
    out = np.zeros(max(int(shots), 1), dtype=np.int64)
    lib().or_sample(_p(psi), n, int(shots), int(seed) & ((1 << 64) - 1), _p(out))
    return out[: int(shots)]


def sample(psi: np.ndarray, qubits: Sequence[int], shots: int, seed: int) -> np.ndarray:
    """Per shot, bit j = measured value of qubits[j] (the library's sv_sample output format)."""
    idx = sample_indices(psi, shots, seed).astype(np.uint64)
    out = np.zeros(idx.size, dtype=np.uint64)
    for j, q in enumerate(qubits):
        out |= ((idx >> np.uint64(q)) & np.uint64(1)) << np.uint64(j)
    return out


def energy(n: int, gates, params, ham, psi0=None) -> float:
    return expectation(apply_circuit(n, gates, params, psi0), ham)[0]


# ----------------------------------------------------------------------------- density matrices
# PAPER.md §3.2: rho = sum_i p_i |psi_i><psi_i|, rho' = U rho U^dagger (eq. at),
# <H> = tr(rho H) (eq. at). Plain definitions with full 2^n x 2^n matrices (small n only):
# each gate's full unitary is built column by column with the oracle's plain gate application.

def full_unitary(n: int, gate, params=None) -> np.ndarray:
    """The 2^n x 2^n matrix of one gate (columns = the gate applied to basis states)."""
    U = np.empty((1 << n, 1 << n), dtype=np.complex128)
    for c in range(1 << n):
        e = np.zeros(1 << n, dtype=np.complex128)
        e[c] = 1.0
        U[:, c] = apply_circuit(n, [gate], params, e)
    return U


def dm_apply_circuit(n: int, gates, params=None, rho0: Optional[np.ndarray] = None) -> np.ndarray:
    """rho <- U_k rho U_k^dagger for every gate in order; rho0 defaults to |0><0|."""
    rho = np.zeros((1 << n, 1 << n), dtype=np.complex128) if rho0 is None else np.array(rho0, dtype=np.complex128)
    if rho0 is None:
        rho[0, 0] = 1.0
    for g in gates:
        U = full_unitary(n, g, params)
        rho = U @ rho @ U.conj().T
    return rho


def pauli_matrix(n: int, term: dict) -> np.ndarray:
    """Dense matrix of one Pauli string (columns = the string applied to basis states)."""
    P = np.empty((1 << n, 1 << n), dtype=np.complex128)
    for c in range(1 << n):
        e = np.zeros(1 << n, dtype=np.complex128)
        e[c] = 1.0
        for q, p in term.items():
            e = apply_matrix(e, gate_matrix(p), [q])
        P[:, c] = e
    return P


def dm_expectation(rho: np.ndarray, ham) -> float:
    """<H> = tr(rho H) = sum_t c_t tr(rho P_t), real part."""
    n = int(rho.shape[0]).bit_length() - 1
    return float(sum(c * np.trace(rho @ pauli_matrix(n, term)) for c, term in ham).real)
