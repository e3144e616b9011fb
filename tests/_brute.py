"""Brute-force dense-matrix path used ONLY to pin the oracle (n <= 8).

Independent of oracle/sv_oracle.c's index arithmetic: the full 2^n x 2^n unitary of a gate is
assembled from explicit Kronecker products in qubit order (qubit 0 is the rightmost Kronecker
factor, i.e. the least-significant index bit — Fig. 3), with controls as
Pi_C (x) M + (I - Pi_C) (x) I. Textbook Pauli matrices are written here.
"""
import numpy as np

I2 = np.eye(2, dtype=complex)
PX = np.array([[0, 1], [1, 0]], dtype=complex)
PY = np.array([[0, -1j], [1j, 0]], dtype=complex)
PZ = np.array([[1, 0], [0, -1]], dtype=complex)
P0 = np.array([[1, 0], [0, 0]], dtype=complex)  # |0><0|
P1 = np.array([[0, 0], [0, 1]], dtype=complex)  # |1><1|
PAULI = {"X": PX, "Y": PY, "Z": PZ}


def kron_list(factors_by_qubit, n):
    """factors_by_qubit: dict qubit -> 2x2; identity elsewhere. Qubit n-1 leftmost."""
    out = np.array([[1.0 + 0j]])
    for q in reversed(range(n)):
        out = np.kron(out, factors_by_qubit.get(q, I2))
    return out


def embed_targets(M, targets, n):
    """Full-space operator of a k-qubit matrix M (index bit j <-> targets[j]) via a sum of
    Kronecker products of its 2x2 blocks' elementary matrices |r_j><c_j|."""
    k = len(targets)
    d = 1 << k
    full = np.zeros((1 << n, 1 << n), dtype=complex)
    for r in range(d):
        for c in range(d):
            if M[r, c] == 0:
                continue
            fac = {}
            for j, t in enumerate(targets):
                e = np.zeros((2, 2), dtype=complex)
                e[(r >> j) & 1, (c >> j) & 1] = 1
                fac[t] = e
            full += M[r, c] * kron_list(fac, n)
    return full


def controlled(M, targets, controls, n):
    U = embed_targets(M, targets, n)
    if not controls:
        return U
    proj = kron_list({c: P1 for c in controls}, n)
    eye = np.eye(1 << n, dtype=complex)
    return proj @ U + (eye - proj)


def dense_hamiltonian(ham, n):
    H = np.zeros((1 << n, 1 << n), dtype=complex)
    for c, term in ham:
        H += c * kron_list({q: PAULI[p] for q, p in term.items()}, n)
    return H
