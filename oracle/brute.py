"""Kronecker-product brute force for n <= 8 — TEST INFRASTRUCTURE ONLY (pins the C oracle).

Each gate becomes the full 2^n x 2^n operator built from tensor products, the textbook
construction that the paper's pair addressing is a fast way to evaluate:

  * a 1-qubit U on qubit k:       I_{2^{n-1-k}} (x) U (x) I_{2^k}
  * a 4x4 M on adjacent (k, k+1): I_{2^{n-2-k}} (x) M (x) I_{2^k}   (sub-index s = bit(k) + 2 bit(k+1))
  * M on arbitrary (q0, q1):      conjugate the adjacent form by a chain of adjacent-SWAP operators
  * a diagonal:                   the same, with the diagonal written as a matrix
Shares nothing with oracle/sv_oracle.c (different derivation, different language).
"""
from __future__ import annotations

import numpy as np

U1, U2, D1, D2, SWAP, CHUNK_SWAP, BEGIN, END = 1, 2, 3, 4, 5, 6, 7, 8
_SWAP4 = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)


def _eye(k: int) -> np.ndarray:
    return np.eye(1 << k, dtype=np.complex128)


def op_1q(u: np.ndarray, k: int, n: int) -> np.ndarray:
    return np.kron(_eye(n - 1 - k), np.kron(u, _eye(k)))


def op_2q_adjacent(m: np.ndarray, k: int, n: int) -> np.ndarray:
    return np.kron(_eye(n - 2 - k), np.kron(m, _eye(k)))


def op_2q(m: np.ndarray, q0: int, q1: int, n: int) -> np.ndarray:
    """Route q0 -> position 0 and q1 -> position 1 with adjacent swaps P, then P^T (M on 0,1) P."""
    pos = list(range(n))          # pos[j] = which original qubit sits at position j
    P = np.eye(1 << n, dtype=np.complex128)
    def bubble(target_qubit, dest):
        nonlocal P
        j = pos.index(target_qubit)
        while j > dest:
            P = op_2q_adjacent(_SWAP4, j - 1, n) @ P
            pos[j - 1], pos[j] = pos[j], pos[j - 1]
            j -= 1
    bubble(q0, 0)
    bubble(q1, 1)
    return P.conj().T @ op_2q_adjacent(m, 0, n) @ P


def _cplx(rec, count: int) -> np.ndarray:
    m = np.asarray(rec["m"], dtype=np.float64)
    return m[0:2 * count:2] + 1j * m[1:2 * count:2]


def full_operator(rec, n: int) -> np.ndarray:
    k, q0, q1 = int(rec["kind"]), int(rec["q0"]), int(rec["q1"])
    if k == U1:
        return op_1q(_cplx(rec, 4).reshape(2, 2), q0, n)
    if k == D1:
        return op_1q(np.diag(_cplx(rec, 2)), q0, n)
    if k == U2:
        return op_2q(_cplx(rec, 16).reshape(4, 4), q0, q1, n)
    if k == D2:
        return op_2q(np.diag(_cplx(rec, 4)), q0, q1, n)
    if k in (SWAP, CHUNK_SWAP):
        return op_2q(_SWAP4, q0, q1, n)
    if k in (BEGIN, END):
        return np.eye(1 << n, dtype=np.complex128)
    raise ValueError(f"kind {k}")


def apply_brute(circ, n: int, psi0: np.ndarray) -> np.ndarray:
    assert n <= 10, "brute force is for tiny n"
    psi = np.asarray(psi0, dtype=np.complex128).copy()
    for rec in circ:
        psi = full_operator(rec, n) @ psi
    return psi


def circuit_unitary(circ, n: int) -> np.ndarray:
    u = np.eye(1 << n, dtype=np.complex128)
    for rec in circ:
        u = full_operator(rec, n) @ u
    return u
