"""Pins for the C oracle (oracle/sv_oracle.c) against things other than itself:
the paper's worked pair, Kronecker brute force, closed forms, a library FFT, invariants."""
import math

import numpy as np
import pytest

import circuits as C
import oracle as O
from oracle import brute


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return v / np.linalg.norm(v)


def test_pair_address_worked_example():
    # indices 0011 and 0111 are the pair for k = 2.
    pairs = [O.pair_address(i, 2) for i in range(8)]
    assert (3, 7) in pairs


@pytest.mark.parametrize("n", range(1, 13))
def test_pair_address_partitions(n):
    # for each k the 2^(n-1) pairs partition [0, 2^n), each pair differs only in bit k.
    for k in range(n):
        seen = []
        for i in range(1 << (n - 1)):
            a, b = O.pair_address(i, k)
            assert b == a + (1 << k) and (a >> k) & 1 == 0
            seen += [a, b]
        assert sorted(seen) == list(range(1 << n))


def test_cnot_basis_action():
    # Eq. (2) + P:107: CNOT with control = q1 maps |10> (index 2) to |11> (index 3).
    g = C.records([C.gate(C.U2, 0, 1, C.CNOT_MATRIX)])
    out = O.apply_circuit(g, 2, basis=2)
    assert np.array_equal(out, np.array([0, 0, 0, 1], dtype=complex))
    assert np.array_equal(O.apply_circuit(g, 2, basis=0), np.array([1, 0, 0, 0], dtype=complex))


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8])
def test_oracle_matches_kronecker_brute_force(n):
    # BASELINE north_star: brute-force 2^n x 2^n products on n <= 8.  All gate kinds, asymmetric
    # matrices (catches transposes), both qubit orders (catches swapped sub-indices).
    for seed in range(3):
        circ = C.random_circuit(n, 40, 100 * n + seed) if n >= 2 else None
        psi = rand_state(n, seed)
        got = O.apply_circuit(circ, n, psi)
        ref = brute.apply_brute(circ, n, psi)
        assert np.max(np.abs(got - ref)) <= 1e-12


def test_oracle_u2_qubit_order_and_transpose():
    # A deliberately asymmetric non-unitary matrix exposes any transpose / sub-index mix-up.
    n = 4
    m = np.arange(16).reshape(4, 4) + 1j * np.arange(16).reshape(4, 4)[::-1]
    psi = rand_state(n, 5)
    for q0, q1 in [(0, 1), (1, 0), (0, 3), (3, 1), (2, 0)]:
        g = C.records([C.gate(C.U2, q0, q1, m)])
        assert np.max(np.abs(O.apply_circuit(g, n, psi) - brute.apply_brute(g, n, psi))) <= 1e-12
    m2 = np.array([[1, 2j], [3, 4 - 1j]])
    for k in range(n):
        g = C.records([C.gate(C.U1, k, mat=m2)])
        assert np.max(np.abs(O.apply_circuit(g, n, psi) - brute.apply_brute(g, n, psi))) <= 1e-12


def test_diagonal_equals_dense():
    # the diagonal kinds give exactly what the dense kinds give for the same matrix.
    n = 6
    rng = np.random.default_rng(2)
    for t in range(20):
        psi = rand_state(n, t)
        d = np.exp(1j * rng.uniform(-3, 3, 4))
        a, b = (int(x) for x in rng.choice(n, 2, replace=False))
        g_diag = C.records([C.gate(C.D2, a, b, d), C.gate(C.D1, b, mat=d[:2])])
        g_dense = C.records([C.gate(C.U2, a, b, np.diag(d)), C.gate(C.U1, b, mat=np.diag(d[:2]))])
        assert np.max(np.abs(O.apply_circuit(g_diag, n, psi) - O.apply_circuit(g_dense, n, psi))) <= 1e-14


def test_unitarity_long_circuit():
    # S:260, north_star: norm preserved to 1e-12 after many gates.
    n = 12
    a = O.apply_circuit(C.random_circuit(n, 1000, 9), n)
    assert abs(O.norm2(a) - 1) <= 1e-12


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_qft_closed_form_all_k(n):
    # QFT|k>_j = e^{+2 pi i jk / 2^n} / 2^{n/2} for the R13 gate order, every k.
    N = 1 << n
    j = np.arange(N)
    for k in range(N):
        out = O.apply_circuit(C.qft(n), n, basis=k)
        ref = np.exp(2j * np.pi * ((j * k) % N) / N) / math.sqrt(N)
        assert np.max(np.abs(out - ref)) <= 1e-12


@pytest.mark.parametrize("n", [8, 10, 14, 16])
def test_qft_closed_form_seeded_k(n):
    N = 1 << n
    k = C.basis_index(1, n)
    out = O.apply_circuit(C.qft(n), n, basis=k)
    j = np.arange(N, dtype=np.int64)
    ref = np.exp(2j * np.pi * ((j * k) % N) / N) / math.sqrt(N)
    assert np.max(np.abs(out - ref)) <= 1e-12


@pytest.mark.parametrize("n", [3, 7, 12])
def test_qft_is_scaled_inverse_dft(n):
    # Library routine: QFT(psi) = sqrt(N) * numpy.fft.ifft(psi) for any psi.
    psi = rand_state(n, n)
    out = O.apply_circuit(C.qft(n), n, psi)
    assert np.max(np.abs(out - math.sqrt(1 << n) * np.fft.ifft(psi))) <= 1e-13


@pytest.mark.parametrize("n", [2, 5, 11])
def test_ghz(n):
    a = O.apply_circuit(C.ghz(n), n)
    ref = np.zeros(1 << n, dtype=complex)
    ref[0] = ref[-1] = 1 / math.sqrt(2)
    assert np.max(np.abs(a - ref)) <= 1e-15


def test_mirror_returns_to_basis():
    n = 10
    k = C.basis_index(3, n)
    a = O.apply_circuit(C.mirror(C.quantum_volume(n, 6, 4)), n, basis=k)
    ref = np.zeros(1 << n, dtype=complex); ref[k] = 1
    assert np.max(np.abs(a - ref)) <= 1e-12


def test_unpermute_against_tensor_transpose():
    # R7 un-permute vs an independent numpy axis transpose of the (2,)*n tensor.
    n = 7
    rng = np.random.default_rng(1)
    for _ in range(10):
        pi = rng.permutation(n)
        phys = rand_state(n, int(rng.integers(1000)))
        got = O.unpermute(phys, pi)
        # logical bit q sits at physical bit pi[q]; C-order axis a <-> bit n-1-a
        t = phys.reshape((2,) * n)
        axes = [n - 1 - pi[n - 1 - a] for a in range(n)]
        ref = np.transpose(t, axes).reshape(-1)
        assert np.array_equal(got, ref)


def test_marginal_against_reshape_sum():
    n = 8
    psi = rand_state(n, 3)
    p = np.abs(psi) ** 2
    t = p.reshape((2,) * n)
    for Q in ([0], [7], [2, 5], [5, 2], [0, 1, 2, 3, 4, 5, 6, 7], [6, 0, 3]):
        got = O.marginal(psi, Q)
        keep = [n - 1 - q for q in Q]
        rest = tuple(a for a in range(n) if a not in keep)
        s = t.sum(axis=rest)  # remaining axes in increasing axis order
        remaining = sorted(keep)
        # reorder so that Q[0] is the least significant bit of y
        s = np.transpose(s, [remaining.index(k) for k in reversed(keep)]).reshape(-1)
        assert np.max(np.abs(got - s)) <= 1e-15


def test_marginals_closed_forms():
    n = 9
    a = O.apply_circuit(C.qft(n), n, basis=C.basis_index(1, n))
    for Q in ([0], [3, 8], [0, 1, 2, 3]):
        assert np.max(np.abs(O.marginal(a, Q) - 2.0 ** -len(Q))) <= 1e-13
    g = O.apply_circuit(C.ghz(n), n)
    p = O.marginal(g, [0, 4, 8])
    ref = np.zeros(8); ref[0] = ref[7] = 0.5
    assert np.max(np.abs(p - ref)) <= 1e-15


def test_sampling_against_searchsorted():
    n = 10
    psi = rand_state(n, 8)
    us = C.sample_uniforms(42, 5000)
    got = O.sample(psi, us)
    cdf = np.cumsum(np.abs(psi) ** 2)
    ref = np.searchsorted(cdf, us, side="right")
    assert np.array_equal(got, ref.astype(np.uint64))


def test_norm2_non_unit_vectors():
    # or_norm2 = sum_x |a_x|^2 (the definition, not sqrt of it): a hand-computed vector and the
    # quadratic scaling law norm2(c a) = |c|^2 norm2(a) on a random non-normalised state.
    a = np.array([3 + 4j, 0, 1j, -2, 0.5, 0, 0, -0.5j], dtype=np.complex128)
    assert O.norm2(a) == 25 + 0 + 1 + 4 + 0.25 + 0.25
    rng = np.random.default_rng(5)
    b = rng.standard_normal(1 << 10) + 1j * rng.standard_normal(1 << 10)
    ref = float(np.sum(b.real ** 2 + b.imag ** 2))
    assert abs(O.norm2(b) - ref) <= 1e-12 * ref
    assert abs(O.norm2(3.0 * b) - 9.0 * ref) <= 1e-12 * 9 * ref
    assert O.norm2(np.zeros(4, dtype=np.complex128)) == 0.0


def test_sampling_tail_beyond_total_mass():
    # u at or beyond the total mass (rounding, or a sub-normalised state) returns the last outcome
    # with nonzero probability, never a zero-probability index (R16).
    a = np.zeros(16, dtype=np.complex128)
    a[3] = 0.6
    a[9] = 0.8j * 0.999  # total mass 0.36 + 0.6387... < 1
    mass = abs(a[3]) ** 2 + abs(a[9]) ** 2
    us = np.array([0.0, 0.35, 0.37, mass - 1e-12, mass, 0.99999, 0.5])
    got = O.sample(a, us)
    assert list(got) == [3, 3, 9, 9, 9, 9, 9]
    # a state whose trailing amplitudes are zero: the tail goes to the last nonzero one, not 2^n - 1
    b = np.zeros(8, dtype=np.complex128)
    b[0] = b[2] = np.sqrt(0.5)
    assert list(O.sample(b, np.array([0.25, 0.75, 1.0 - 2 ** -53]))) == [0, 2, 2]
