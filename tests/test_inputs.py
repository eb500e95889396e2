"""Pins for the shared input generators (circuits/gen.py)."""
import cmath
import math

import numpy as np
import pytest

import circuits as C


def test_u3_special_cases():
    # S:53-55 / Eq. (1): u3(0,0,0)=I, u3(pi,0,pi)=X, u3(pi/2,0,pi)=H.
    assert np.max(np.abs(C.u3(0, 0, 0) - np.eye(2))) <= 1e-15
    assert np.max(np.abs(C.u3(math.pi, 0, math.pi) - C.X_MATRIX)) <= 1e-15
    assert np.max(np.abs(C.u3(math.pi / 2, 0, math.pi) - C.H_MATRIX)) <= 1e-15


def test_u3_term_by_term():
    # Eq. (1) entries evaluated independently with cmath, 100 random triples.
    rng = np.random.default_rng(7)
    for th, ps, la in rng.uniform(-2 * math.pi, 2 * math.pi, (100, 3)):
        m = C.u3(th, ps, la)
        ref = [[math.cos(th / 2), -cmath.exp(1j * la) * math.sin(th / 2)],
               [cmath.exp(1j * ps) * math.sin(th / 2), cmath.exp(1j * (ps + la)) * math.cos(th / 2)]]
        assert np.max(np.abs(m - np.array(ref))) <= 1e-15
        assert np.max(np.abs(m.conj().T @ m - np.eye(2))) <= 1e-12


def test_cnot_is_eq2():
    # Eq. (2): rows (00,01,10,11) with the higher bit as control: |10> -> |11>.
    e2 = np.zeros(4); e2[2] = 1
    assert np.array_equal(np.abs(C.CNOT_MATRIX @ e2), np.array([0, 0, 0, 1.0]))
    assert np.array_equal(C.CNOT_MATRIX @ C.CNOT_MATRIX, np.eye(4))


def test_haar_su4():
    rng = np.random.default_rng(3)
    for _ in range(50):
        u = C.haar_su(rng, 4)
        assert np.max(np.abs(u.conj().T @ u - np.eye(4))) <= 1e-12
        assert abs(np.linalg.det(u) - 1) <= 1e-12


@pytest.mark.parametrize("n", [1, 2, 5, 10, 30, 36])
def test_qft_gate_count(n):
    # n H + n(n-1)/2 controlled phases + n//2 swaps (QFT36 = 684).
    g = C.qft(n)
    assert len(g) == n + n * (n - 1) // 2 + n // 2
    if n == 36:
        assert len(g) == 684


@pytest.mark.parametrize("n,depth", [(4, 10), (28, 10), (33, 10), (5, 3)])
def test_qv_gate_count_and_determinism(n, depth):
    # depth * floor(n/2) two-qubit gates; same seed -> identical list.
    a, b = C.quantum_volume(n, depth, 1), C.quantum_volume(n, depth, 1)
    assert len(a) == depth * (n // 2)
    assert a.tobytes() == b.tobytes()
    assert C.quantum_volume(n, depth, 2).tobytes() != a.tobytes()
    if (n, depth) == (33, 10):
        assert len(a) == 160
    for layer in range(depth):
        qs = [q for r in a[layer * (n // 2):(layer + 1) * (n // 2)] for q in (int(r["q0"]), int(r["q1"]))]
        assert len(set(qs)) == len(qs)  # each layer pairs distinct qubits


def test_splitmix64_reference_values():
    # SplitMix64 reference outputs for seed 0 stream (Vigna's splitmix64.c: x += golden; mix).
    assert C.splitmix64(0) == 0xE220A8397B1DCDAF
    assert C.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_mirror_structure():
    c = C.random_circuit(5, 30, 11)
    m = C.mirror(c)
    assert len(m) == 60
    for i in range(30):
        a, b = c[i], m[59 - i]
        assert (int(a["kind"]), int(a["q0"]), int(a["q1"])) == (int(b["kind"]), int(b["q0"]), int(b["q1"]))
