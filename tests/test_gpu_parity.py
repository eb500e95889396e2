"""GPU parity: libsv.so (C-ABI, sm_100a kernels) vs the CPU oracle on the same seeded inputs.

Tolerances (north_star, DESIGN "Tolerances"): fp64 max|d| <= 1e-10; fp32 max|d| <= 1e-4 and
||d||_2 <= 1e-5 * ||a||_2 (reading R15)."""
import math

import numpy as np
import pytest

import circuits as C
import oracle as O

from conftest import gpu_available

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_2102_02957_b200")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")
    import torch
    torch.cuda.set_device(0)


def check(got, ref, prec):
    d = np.abs(got.astype(np.complex128) - ref)
    if prec == "fp64":
        assert d.max() <= 1e-10, d.max()
    else:
        assert d.max() <= 1e-4, d.max()
        assert np.linalg.norm(d) <= 1e-5 * max(1.0, np.linalg.norm(ref)), np.linalg.norm(d)


def rand_state_records(n, seed):
    return C.random_circuit(n, 4 * n, seed, kinds=("u3", "su4"))


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_qft10_cfg0(prec):
    n, c = 10, 6
    k = C.basis_index(1, n)
    with sv.StateVector(n, c, prec) as s:
        s.reset(k)
        s.apply(C.qft(n))
        got = s.state()
    ref = O.apply_circuit(C.qft(n), n, basis=k)
    check(got, ref, prec)
    j = np.arange(1 << n)
    closed = np.exp(2j * np.pi * ((j * k) % (1 << n)) / (1 << n)) / math.sqrt(1 << n)
    check(got, closed, prec)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_random_circuits(prec):
    rng = np.random.default_rng(11)
    for t in range(40):
        n = int(rng.integers(2, 17))
        c = int(rng.integers(2, n + 1)) if n >= 2 else 1
        if prec == "fp64":
            c = min(c, 13)
        else:
            c = min(c, 13)
        circ = C.random_circuit(n, int(rng.integers(0, 120)), 500 + t)
        with sv.StateVector(n, c, prec) as s:
            s.apply(circ)
            s.apply(circ[: len(circ) // 2])  # pi carried across calls
            got = s.state()
        ref = O.apply_circuit(circ[: len(circ) // 2], n, O.apply_circuit(circ, n))
        check(got, ref, prec)


@pytest.mark.parametrize("n,c", [(14, 12), (16, 8), (18, 12), (20, 10), (20, 13)])
def test_qv_and_qft_mid(n, c):
    for circ in (C.quantum_volume(n, 10, 1), C.qft(n)):
        with sv.StateVector(n, c, "fp64") as s:
            s.reset(C.basis_index(2, n))
            s.apply(circ)
            got = s.state()
        check(got, O.apply_circuit(circ, n, basis=C.basis_index(2, n)), "fp64")


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_unblocked_baseline(prec):
    n = 14
    circ = C.random_circuit(n, 80, 9)
    with sv.StateVector(n, 8, prec) as s:
        s.apply(circ, flags=sv.SV_UNBLOCKED)
        got = s.state()
        st = s.stats()
    check(got, O.apply_circuit(circ, n), prec)
    assert st["sections"] == 0 and st["kernel_launches"] >= 80


def test_restore_order_and_permutation():
    n, c = 12, 5
    circ = C.quantum_volume(n, 6, 4)
    with sv.StateVector(n, c) as s:
        s.apply(circ, flags=sv.SV_RESTORE_ORDER)
        assert list(s.permutation()) == list(range(n))
        got = s.state()
    check(got, O.apply_circuit(circ, n), "fp64")


def test_edge_cases():
    # empty circuit, diagonal-only circuit, tiny n, c = n
    for n, c in [(1, 1), (2, 2), (3, 2), (4, 4), (5, 3)]:
        circ = C.random_circuit(n, 30, n, kinds=("u3", "u1") if n == 1 else ("u3", "cx", "cp", "swap", "su4", "u1", "d2"))
        with sv.StateVector(n, c) as s:
            s.apply(circ[:0])
            s.apply(circ)
            got = s.state()
        check(got, O.apply_circuit(circ, n), "fp64")
    circ = C.random_circuit(16, 200, 3, kinds=("cp", "u1", "d2"))
    psi = C.random_circuit(16, 40, 4, kinds=("u3",))
    with sv.StateVector(16, 4) as s:
        s.apply(psi)
        s.apply(circ)
        got = s.state()
    check(got, O.apply_circuit(circ, 16, O.apply_circuit(psi, 16)), "fp64")


def test_readout_norm_probs_amplitudes():
    n, c = 16, 10
    circ = C.quantum_volume(n, 8, 3)
    ref = O.apply_circuit(circ, n)
    with sv.StateVector(n, c) as s:
        s.apply(circ)
        assert abs(s.norm() - 1.0) <= 1e-12
        for Q in ([0], [15, 3], [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15], [7, 2, 11]):
            assert np.max(np.abs(s.probabilities(Q) - O.marginal(ref, Q))) <= 1e-13
        idx = np.array([0, 1, 12345, (1 << n) - 1, 777], dtype=np.uint64)
        assert np.max(np.abs(s.amplitudes(idx) - ref[idx.astype(np.int64)])) <= 1e-10


def test_sampling():
    n, c = 14, 8
    # pi = identity (no blocking swaps needed: c = n) -> exact match with the oracle's inverse CDF
    circ = C.quantum_volume(n, 6, 5)
    with sv.StateVector(n, n) as s:
        s.apply(circ)
        assert list(s.permutation()) == list(range(n))
        shots = s.sample(20000, 99)
    ref = O.apply_circuit(circ, n)
    us = C.sample_uniforms(99, 20000)
    cdf = np.cumsum(np.abs(ref) ** 2)
    near_edge = np.min(np.abs(cdf[None, :] - us[:, None]), axis=1) < 1e-12
    exp = O.sample(ref, us)
    assert np.array_equal(shots[~near_edge], exp[~near_edge])
    # blocked (pi != id, so the GPU scans in memory order): a chi^2 test over ALL outcomes
    # (outcomes expected fewer than 5 times are pooled into one bin), every shot a nonzero outcome
    from scipy.stats import chi2 as chi2_dist
    for n2, c2, shots, seed in [(12, 6, 400_000, 7), (16, 8, 2_000_000, 8)]:
        circ2 = C.quantum_volume(n2, 6, 5)
        with sv.StateVector(n2, c2) as s:
            s.apply(circ2)
            assert list(s.permutation()) != list(range(n2))
            got = s.sample(shots, seed)
        p = np.abs(O.apply_circuit(circ2, n2)) ** 2
        assert np.all(p[got.astype(np.int64)] > 0)
        obs = np.bincount(got.astype(np.int64), minlength=1 << n2).astype(np.float64)
        exp = p * shots
        big = exp >= 5
        o2 = np.concatenate([obs[big], [obs[~big].sum()]])
        e2 = np.concatenate([exp[big], [exp[~big].sum()]])
        keep = e2 > 0
        stat = float(np.sum((o2[keep] - e2[keep]) ** 2 / e2[keep]))
        dof = int(keep.sum()) - 1
        assert chi2_dist.sf(stat, dof) > 1e-6, (n2, stat, dof)


def test_mirror_returns_to_basis_large():
    n, c = 24, 12
    k = C.basis_index(5, n)
    with sv.StateVector(n, c) as s:
        s.reset(k)
        s.apply(C.mirror(C.quantum_volume(n, 10, 2)))
        a = s.amplitudes(np.array([k], dtype=np.uint64))
        assert abs(a[0] - 1.0) <= 1e-10
        assert abs(s.norm() - 1.0) <= 1e-12


@pytest.mark.parametrize("mode", [0, 2])
def test_interpreter_and_async_modes(mode):
    # mode 0: every section runs the program interpreter (k_section); mode 2: the first apply of a
    # shape runs the interpreter while its kernels compile, later applies the generated kernels
    prev = sv.jit_mode(mode)
    try:
        for n, c, circ in [(14, 10, C.quantum_volume(14, 6, 5)), (16, 12, C.qft(16)),
                           (13, 9, C.random_circuit(13, 150, 77))]:
            for prec in ("fp64", "fp32"):
                for rep in range(2):
                    with sv.StateVector(n, c, prec) as s:
                        s.reset(C.basis_index(3, n))
                        s.apply(circ)
                        got = s.state()
                        st = s.stats()
                    check(got, O.apply_circuit(circ, n, basis=C.basis_index(3, n)), prec)
                    if mode == 0:
                        assert st["jit_launches"] == 0 and st["interp_launches"] > 0
                if mode == 2:
                    sv.jit_wait()
    finally:
        sv.jit_mode(prev)


def test_generated_kernels_run():
    # default mode: the generated kernels are the ones that run
    with sv.StateVector(14, 10, "fp64") as s:
        s.apply(C.quantum_volume(14, 4, 9))
        st = s.stats()
    assert st["jit_launches"] > 0 and st["interp_launches"] == 0


@pytest.mark.slow
def test_qv33_full_size_mirror():
    # BASELINE configs[3] at full size (2^33 fp64 amplitudes, 128 GiB) in the bench's configuration
    # (c = 9): the mirror circuit C C^dagger returns the seeded basis state exactly; the forward
    # circuit keeps the norm and its marginals sum to one.
    n, c = 33, 9
    k = C.basis_index(6, n)
    circ = C.quantum_volume(n, 10, 1)
    with sv.StateVector(n, c) as s:
        s.reset(k)
        s.apply(C.mirror(circ))
        a = s.amplitudes(np.array([k, (k + 1) % (1 << n)], dtype=np.uint64))
        assert abs(a[0] - 1.0) <= 1e-10 and abs(a[1]) <= 1e-10
        s.reset(0)
        s.apply(circ)
        assert abs(s.norm() - 1.0) <= 1e-12
        assert abs(s.probabilities([0, 16, 32]).sum() - 1.0) <= 1e-12


def test_deferred_basis_state_readers():
    # sv_reset defers writing |k> to the next circuit's first section; every reader, an empty
    # circuit, the unblocked path and a plan not starting with a section must still see |k>
    n, c = 12, 6
    k = C.basis_index(9, n)
    ref = np.zeros(1 << n, dtype=np.complex128)
    ref[k] = 1
    with sv.StateVector(n, c) as s:
        s.reset(k)
        check(s.state(), ref, "fp64")
        s.reset(k)
        assert abs(s.norm() - 1) <= 1e-15
        s.reset(k)
        assert abs(s.amplitudes(np.array([k], dtype=np.uint64))[0] - 1) <= 1e-15
        s.reset(k)
        s.apply(C.records([]))
        check(s.state(), ref, "fp64")
        s.reset(k)
        p = s.probabilities([0, 1, 2])
        assert abs(p[k & 7] - 1) <= 1e-15
        circ = C.random_circuit(n, 40, 3)
        for flags in (0, sv.SV_UNBLOCKED):
            s.reset(k)
            s.apply(circ, flags=flags)
            check(s.state(), O.apply_circuit(circ, n, basis=k), "fp64")
        s.reset(k)
        s.reset(k ^ 5)  # two resets in a row: the last one wins
        s.apply(circ)
        check(s.state(), O.apply_circuit(circ, n, basis=k ^ 5), "fp64")


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_host_memory_tier(prec):
    # NEXT-4: state in host memory, the GPU streaming 2^d-amplitude chunks through every section
    for n, c, d, circ, basis in [(14, 6, 11, C.quantum_volume(14, 8, 2), 0), (15, 5, 11, C.qft(15), C.basis_index(3, 15)),
                                 (13, 5, 10, C.random_circuit(13, 200, 21), 5)]:
        with sv.HostStateVector(n, c, d, prec) as s:
            s.reset(basis)
            s.apply(circ)
            ref = O.apply_circuit(circ, n, basis=basis)
            check(s.state(), ref, prec)
            tol = 1e-12 if prec == "fp64" else 1e-5
            assert abs(s.norm() - 1) <= tol
            Q = [0, n - 1, n // 2]
            assert np.max(np.abs(s.probabilities(Q) - O.marginal(ref, Q))) <= tol
            s.apply(C.mirror(circ))  # the layout carries over to the next circuit
            back = np.zeros(1 << n, dtype=np.complex128)
            back[:] = O.apply_circuit(C.mirror(circ), n, ref)
            check(s.state(), back, prec)


def test_absorb_swaps():
    # SV_ABSORB_SWAPS: user SWAPs relabel the tracked permutation instead of being gates (the
    # paper's bit reordering); QFT's terminal swap layer then costs no section
    for n, c, circ, basis in [(16, 8, C.qft(16), C.basis_index(4, 16)), (14, 6, C.random_circuit(14, 200, 12, kinds=("u3", "cx", "swap", "cp", "su4")), 0)]:
        with sv.StateVector(n, c) as s:
            s.reset(basis)
            s.apply(circ, flags=sv.SV_ABSORB_SWAPS)
            s.apply(circ[: len(circ) // 2], flags=sv.SV_ABSORB_SWAPS)  # pi carried into the next circuit
            got = s.state()
            st = s.stats()
        ref = O.apply_circuit(circ[: len(circ) // 2], n, O.apply_circuit(circ, n, basis=basis))
        check(got, ref, "fp64")
        assert st["sections"] > 0
