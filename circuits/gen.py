"""Seeded synthetic circuit generators — the shared INPUT module.

This module is the only code both the oracle (``oracle/``) and the CUDA path
(``paper_2102_02957_b200``) consume, and it holds none of the method's
arithmetic: it only *builds* gate records (matrices and qubit indices).
Applying gates, the cache-blocking pass, reductions and sampling live on each
side separately.

Record layout (``GATE_DTYPE``, 272 bytes) mirrors ``sv_gate`` in
``include/sv.h``::

    int32 kind, q0, q1, pad; float64 m[32]

``m`` is complex interleaved (re, im), ROW-major.  Kinds:

* ``U1``  2x2 unitary on ``q0`` (8 doubles).
* ``U2``  4x4 unitary on (q0, q1); sub-index ``s = bit(q0) + 2*bit(q1)``
  (so CNOT(control=c, target=t) = U2(q0=t, q1=c, Eq. 2 matrix)).
* ``D1``  diag(d0, d1) on ``q0`` (4 doubles).
* ``D2``  diag(d0..d3) on (q0, q1), same sub-index (8 doubles).
* ``SWAP`` on (q0, q1), no payload.

Citations (``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md):
u3 is Eq. (1); CNOT is Eq. (2) with the higher sub-bit as control
(P:96-107); u1 = diag(1, e^{i lambda}) (OpenQASM); controlled
phase = diag(1,1,1,e^{i lambda}).  QFT / QV shapes follow the
paper's two workloads with the gate orders fixed in DESIGN.md
(readings R13/R14).
"""
from __future__ import annotations

import math
from typing import Iterable, Sequence

import numpy as np

U1, U2, D1, D2, SWAP, CHUNK_SWAP, BEGIN, END = 1, 2, 3, 4, 5, 6, 7, 8
KIND_NAMES = {U1: "U1", U2: "U2", D1: "D1", D2: "D2", SWAP: "SW",
              CHUNK_SWAP: "CS", BEGIN: "BEGIN", END: "END"}

GATE_DTYPE = np.dtype([("kind", "<i4"), ("q0", "<i4"), ("q1", "<i4"),
                       ("pad", "<i4"), ("m", "<f8", (32,))])
assert GATE_DTYPE.itemsize == 272

MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------- matrices
def u3(theta: float, psi: float, lam: float) -> np.ndarray:
    """Eq. (1): [[cos t/2, -e^{i lam} sin t/2], [e^{i psi} sin t/2, e^{i(psi+lam)} cos t/2]]."""
    for v in (theta, psi, lam):
        if not math.isfinite(v):
            raise ValueError("u3 parameters must be finite")
    c, s = math.cos(theta / 2.0), math.sin(theta / 2.0)
    return np.array([[c, -np.exp(1j * lam) * s],
                     [np.exp(1j * psi) * s, np.exp(1j * (psi + lam)) * c]], dtype=np.complex128)


#: The Hadamard as the exact real matrix (the value u3(pi/2, 0, pi) approximates to 1 ulp).
H_MATRIX = np.array([[1.0, 1.0], [1.0, -1.0]], dtype=np.complex128) * (1.0 / math.sqrt(2.0))
X_MATRIX = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=np.complex128)

#: Eq. (2): rows/cols ordered by s = bit(target) + 2*bit(control) -> control = higher sub-bit.
CNOT_MATRIX = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=np.complex128)

SWAP_MATRIX = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)


def u1_diag(lam: float) -> np.ndarray:
    """u1(lambda) = diag(1, e^{i lambda}) (OpenQASM)."""
    return np.array([1.0, np.exp(1j * lam)], dtype=np.complex128)


def cphase_diag(lam: float) -> np.ndarray:
    """Controlled phase diag(1, 1, 1, e^{i lambda}) — QFT's diagonal block."""
    return np.array([1.0, 1.0, 1.0, np.exp(1j * lam)], dtype=np.complex128)


def haar_unitary(rng: np.random.Generator, dim: int) -> np.ndarray:
    """Haar-random U(dim): QR of a complex Ginibre matrix with the R-diagonal phase fixed (Mezzadri)."""
    z = (rng.standard_normal((dim, dim)) + 1j * rng.standard_normal((dim, dim))) / math.sqrt(2.0)
    q, r = np.linalg.qr(z)
    d = np.diagonal(r)
    return q * (d / np.abs(d))[None, :]


def haar_su(rng: np.random.Generator, dim: int) -> np.ndarray:
    """Haar U(dim) divided by det^{1/dim} on the principal branch -> SU(dim) (BASELINE north_star: SU(4))."""
    u = haar_unitary(rng, dim)
    det = np.linalg.det(u)
    return u / (det ** (1.0 / dim))


# ---------------------------------------------------------------- records
def _pack_matrix(mat: np.ndarray) -> np.ndarray:
    flat = np.asarray(mat, dtype=np.complex128).reshape(-1)
    out = np.zeros(32, dtype=np.float64)
    out[0:2 * flat.size:2] = flat.real
    out[1:2 * flat.size:2] = flat.imag
    return out


def gate(kind: int, q0: int, q1: int = -1, mat=None) -> np.ndarray:
    rec = np.zeros((), dtype=GATE_DTYPE)
    rec["kind"], rec["q0"], rec["q1"] = kind, q0, (q1 if kind in (U2, D2, SWAP, CHUNK_SWAP) else -1)
    if mat is not None:
        rec["m"] = _pack_matrix(mat)
    return rec


def records(gs: Iterable[np.ndarray]) -> np.ndarray:
    gs = list(gs)
    out = np.zeros(len(gs), dtype=GATE_DTYPE)
    for i, g in enumerate(gs):
        out[i] = g
    return out


def matrix_of(rec) -> np.ndarray:
    """Unpack the complex payload of one record (U1: 2x2, U2: 4x4, D1: 2, D2: 4)."""
    k = int(rec["kind"])
    m = np.asarray(rec["m"], dtype=np.float64)
    c = m[0::2] + 1j * m[1::2]
    if k == U1:
        return c[:4].reshape(2, 2)
    if k == U2:
        return c[:16].reshape(4, 4)
    if k == D1:
        return c[:2].copy()
    if k == D2:
        return c[:4].copy()
    raise ValueError(f"kind {k} has no matrix")


def qubits_of(rec) -> tuple:
    k = int(rec["kind"])
    if k in (U1, D1):
        return (int(rec["q0"]),)
    if k in (U2, D2, SWAP, CHUNK_SWAP):
        return (int(rec["q0"]), int(rec["q1"]))
    return ()


def is_diagonal(rec) -> bool:
    """Diagonality is declared by kind, never detected from matrices."""
    return int(rec["kind"]) in (D1, D2)


# ---------------------------------------------------------------- workloads
def qft(n: int) -> np.ndarray:
    """QFT(n) in the DESIGN.md R13 order: for q = n-1..0: H(q); for j = q-1..0:
    D2(q0=j, q1=q, diag(1,1,1,e^{i pi/2^{q-j}})); then SWAP(i, n-1-i), i < n//2.
    Gate count n + n(n-1)/2 + n//2."""
    gs = []
    for q in range(n - 1, -1, -1):
        gs.append(gate(U1, q, mat=H_MATRIX))
        for j in range(q - 1, -1, -1):
            gs.append(gate(D2, j, q, cphase_diag(math.pi / (1 << (q - j)))))
    for i in range(n // 2):
        gs.append(gate(SWAP, i, n - 1 - i))
    return records(gs)


def quantum_volume(n: int, depth: int, seed: int) -> np.ndarray:
    """QV(n, depth, seed): per layer p = rng.permutation(n), then
    U2(q0=p[2i], q1=p[2i+1], Haar SU(4)) for i < n//2.  Gate count depth * (n//2)."""
    rng = np.random.default_rng(seed)
    gs = []
    for _ in range(depth):
        p = rng.permutation(n)
        for i in range(n // 2):
            gs.append(gate(U2, int(p[2 * i]), int(p[2 * i + 1]), haar_su(rng, 4)))
    return records(gs)


def ghz(n: int) -> np.ndarray:
    """H(0) then CNOT(control=i, target=i+1): |0..0> + |1..1> over sqrt 2."""
    gs = [gate(U1, 0, mat=H_MATRIX)]
    for i in range(n - 1):
        gs.append(gate(U2, i + 1, i, CNOT_MATRIX))  # q0 = target, q1 = control
    return records(gs)


def random_circuit(n: int, n_gates: int, seed: int, kinds: Sequence[str] = ("u3", "cx", "cp", "swap", "su4", "u1", "d2")) -> np.ndarray:
    """Fuzz circuits over the kinds named: u3 (U1), cx (U2 CNOT), cp (D2 controlled phase),
    swap (SWAP), su4 (U2 Haar), u1 (D1), d2 (D2 with 4 random phases)."""
    rng = np.random.default_rng(seed)
    gs = []
    for _ in range(n_gates):
        k = kinds[int(rng.integers(len(kinds)))]
        if k in ("u3", "u1") or n < 2:
            q = int(rng.integers(n))
            if k == "u1":
                gs.append(gate(D1, q, mat=u1_diag(float(rng.uniform(-math.pi, math.pi)))))
            else:
                th, ps, la = (float(x) for x in rng.uniform(-math.pi, math.pi, 3))
                gs.append(gate(U1, q, mat=u3(th, ps, la)))
            continue
        a, b = (int(x) for x in rng.choice(n, 2, replace=False))
        if k == "cx":
            gs.append(gate(U2, a, b, CNOT_MATRIX))
        elif k == "cp":
            gs.append(gate(D2, a, b, cphase_diag(float(rng.uniform(-math.pi, math.pi)))))
        elif k == "swap":
            gs.append(gate(SWAP, a, b))
        elif k == "su4":
            gs.append(gate(U2, a, b, haar_su(rng, 4)))
        elif k == "d2":
            gs.append(gate(D2, a, b, np.exp(1j * rng.uniform(-math.pi, math.pi, 4))))
        else:
            raise ValueError(k)
    return records(gs)


def dagger(rec) -> np.ndarray:
    """Conjugate transpose of one gate record (same qubits)."""
    k = int(rec["kind"])
    out = np.array(rec, dtype=GATE_DTYPE)
    if k in (U1, U2):
        out["m"] = _pack_matrix(matrix_of(rec).conj().T)
    elif k in (D1, D2):
        out["m"] = _pack_matrix(matrix_of(rec).conj())
    return out


def mirror(circ: np.ndarray) -> np.ndarray:
    """C followed by C^dagger (gates reversed, each conjugate-transposed): returns any state to itself."""
    inv = [dagger(circ[i]) for i in range(len(circ) - 1, -1, -1)]
    return np.concatenate([circ, records(inv)]) if len(circ) else circ.copy()


# ---------------------------------------------------------------- seeds
def splitmix64(x: int) -> int:
    """SplitMix64 finaliser (Steele et al.): the counter-based generator both sides implement."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def basis_index(seed: int, n: int) -> int:
    """Seeded basis state |k>, k = splitmix64(seed) mod 2^n."""
    return splitmix64(seed) % (1 << n)


def sample_uniforms(seed: int, shots: int) -> np.ndarray:
    """u_s = (splitmix64(seed XOR s) >> 11) * 2^-53 — the random numbers sv_sample draws (DESIGN R16)."""
    return np.array([(splitmix64((seed ^ s) & MASK64) >> 11) * (2.0 ** -53) for s in range(shots)], dtype=np.float64)
