"""The section compiler on CPU: programs from sv_compile_circuit, executed by tests/emulator.py
(which mirrors section.cu's data flow and checks its invariants), must reproduce the oracle."""
import numpy as np
import pytest

import circuits as C
import oracle as O

from emulator import run

sv = pytest.importorskip("paper_2102_02957_b200")


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2102_02957_b200 import build
    build.build()


def emulate(recs, n, c, g=0, precision="fp64", seed=0, flags=0, pi0=None, sigma0=None, psi=None):
    """Run the compiled programs on a random (or given) logical state; returns (steps, pi, sigma, logical out)."""
    steps, ints, coefs, aux, pi, sigma = sv.compile_circuit(recs, n, c, g, 0, precision, flags, pi0, sigma0)
    if psi is None:
        rng = np.random.default_rng(seed)
        psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        psi /= np.linalg.norm(psi)
    mu0 = list(range(n)) if pi0 is None else [int(sigma0[int(p)]) for p in pi0]
    mem = np.empty_like(psi)
    mem[:] = psi[O.unpermute(np.arange(1 << n).astype(np.complex128), mu0).real.astype(np.int64).argsort()]

    def gate_fn(m, st):
        rec = np.array(recs[int(st[4])], dtype=C.GATE_DTYPE)
        rec["q0"], rec["q1"] = int(st[2]), int(st[3])
        m[:] = O.apply_circuit(C.records([rec]), n, m)

    run(steps, ints, coefs, aux, mem, gate_fn=gate_fn)
    got = O.unpermute(mem, [int(sigma[int(p)]) for p in pi])
    ref = O.apply_circuit(recs, n, psi)
    err = np.max(np.abs(got - ref))
    assert err <= 1e-12, err
    return steps, pi, sigma, got


def test_two_applies_carry_the_permutations():
    # the GPU test_random_circuits pattern: a second circuit starts from the first one's pi/sigma
    rng = np.random.default_rng(11)
    for t in range(40):
        n = int(rng.integers(2, 17))
        c = min(int(rng.integers(2, n + 1)), 13)
        circ = C.random_circuit(n, int(rng.integers(0, 120)), 500 + t)
        _, pi, sigma, out = emulate(circ, n, c, seed=t)
        emulate(circ[: len(circ) // 2], n, c, pi0=pi, sigma0=sigma, psi=out)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_random_circuits_emulated(prec):
    rng = np.random.default_rng(31)
    for t in range(25):
        n = int(rng.integers(4, 15))
        c = int(rng.integers(2, n + 1))
        recs = C.random_circuit(n, int(rng.integers(1, 90)), 900 + t)
        emulate(recs, n, c, precision=prec, seed=t)


def test_diagonal_heavy_emulated():
    for t, (n, c) in enumerate([(12, 4), (14, 6), (13, 12), (10, 3)]):
        psi_recs = C.random_circuit(n, 20, 50 + t, kinds=("u3", "su4"))
        recs = np.concatenate([psi_recs, C.random_circuit(n, 150, 60 + t, kinds=("cp", "u1", "d2", "u3"))])
        emulate(recs, n, c, seed=t)


@pytest.mark.parametrize("n,c", [(12, 6), (14, 8), (14, 12), (16, 12), (16, 10), (17, 11)])  # c >= 10: tiles with 2 low bits, direct
def test_qft_qv_emulated(n, c):
    emulate(C.qft(n), n, c)
    emulate(C.quantum_volume(n, 6, 2), n, c)


def test_ghz_permutation_ops_emulated():
    emulate(C.ghz(12), 12, 5)
    emulate(C.mirror(C.random_circuit(9, 60, 4, kinds=("cx", "swap", "u3"))), 9, 4)


def test_free_initial_layout_emulated():
    # sv_apply_circuit right after sv_reset(0): the planner picks the initial layout (NEXT-2);
    # |0> sits at memory address 0 under every layout, so the emulated start state is exact.
    rng = np.random.default_rng(11)
    for t in range(40):
        n = int(rng.integers(2, 17))
        c = min(int(rng.integers(2, n + 1)), 13)
        circ = C.random_circuit(n, int(rng.integers(0, 120)), 500 + t)
        psi = np.zeros(1 << n, dtype=np.complex128)
        psi[0] = 1
        for prec in ("fp64", "fp32"):
            emulate(circ, n, c, precision=prec, flags=sv.SV_FREE_LAYOUT, psi=psi.copy())
    for n, c in [(12, 6), (14, 12), (16, 12)]:
        psi = np.zeros(1 << n, dtype=np.complex128)
        psi[0] = 1
        emulate(C.qft(n), n, c, flags=sv.SV_FREE_LAYOUT, psi=psi.copy())
        emulate(C.quantum_volume(n, 6, 2), n, c, flags=sv.SV_FREE_LAYOUT, psi=psi.copy())


@pytest.mark.parametrize("prec,G", [("fp64", 3), ("fp32", 4)])
def test_section_smem_maps_conflict_free(prec, G):
    # every shared-memory round trip of the QV / QFT workloads hits distinct 16-/8-byte slots per
    # 128-byte wavefront (the per-section swizzle and thread-bit choice in compile.cpp)
    from emulator import smem_conflicts
    for recs, n, c in [(C.quantum_volume(22, 10, 1), 22, 12), (C.quantum_volume(22, 10, 2), 22, 10),
                       (C.qft(22), 22, 12), (C.qft(22), 22, 10), (C.random_circuit(16, 200, 3), 16, 9)]:
        steps, ints, coefs, aux, pi, sigma = sv.compile_circuit(recs, n, c, 0, 0, prec, sv.SV_FREE_LAYOUT)
        for st in steps:
            if st[0] == 1 and st[5] >= 4 + G:
                bad = smem_conflicts(ints[st[1]:st[1] + st[2]], G)
                assert not bad, (n, c, bad)


def test_two_rank_programs_emulated():
    # Two ranks' section programs (rank bits folded into constants per rank) run on their halves
    # of the full memory-ordered state, with each cross-GPU exchange emulated as a swap of the
    # local and rank memory bits (the plan's semantics): the result equals the oracle.
    from emulator import run_section, swap_bits
    exchanged = 0
    for n, c, circ in [(14, 6, C.quantum_volume(14, 6, 1)), (13, 5, C.qft(13)),
                       (12, 5, C.random_circuit(12, 160, 9, kinds=("u3", "su4", "cp", "d2", "swap")))]:
        g, nL = 1, n - 1
        per = [sv.compile_circuit(circ, n, c, g, r, "fp64") for r in (0, 1)]
        steps = [p[0] for p in per]
        assert np.array_equal(steps[0][:, [0, 5, 6, 7]], steps[1][:, [0, 5, 6, 7]])
        rng = np.random.default_rng(n)
        psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        psi /= np.linalg.norm(psi)
        mem = psi.copy()
        for i, st in enumerate(steps[0]):
            kind = int(st[0])
            if kind in (0, 3):
                swap_bits(mem, int(st[1]), int(st[2]))
                exchanged += kind == 0
            elif kind == 1:
                for r in (0, 1):
                    sr = steps[r][i]
                    _, ints, coefs, aux, _, _ = per[r]
                    off, cnt, coff, ccnt, T, n_out, flags, aoff, acnt = (int(x) for x in sr[1:10])
                    run_section(mem[r << nL:(r + 1) << nL], ints[off:off + cnt], coefs[coff:coff + ccnt], n_out, T,
                                flags, aux[aoff:aoff + acnt])
            else:
                raise AssertionError(kind)
        pi, sigma = per[0][4], per[0][5]
        got = O.unpermute(mem, [int(sigma[int(p)]) for p in pi])
        ref = O.apply_circuit(circ, n, psi)
        assert np.max(np.abs(got - ref)) <= 1e-12, (n, c)
    assert exchanged >= 2
