"""CPU tests of libsv.so: exports, the C++ blocking pass (bit-exact vs the oracle's independent
pass) and the executor plan (semantics vs the dense oracle).  No GPU is needed: these entry
points are host-only."""
import os
import re

import numpy as np
import pytest

import circuits as C
import oracle as O
from oracle import blocking as B

from blockutil import load_golden, parse_gates, triples
from libutil import lib_tokens, memory_perm, plan_to_dense_records

sv = pytest.importorskip("paper_2102_02957_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2102_02957_b200 import build
    build.build()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "sv.h")).read()
    names = set(re.findall(r"^\s*(?:int|void|const char\*)\s+(sv_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 19
    L = sv.lib()
    for nm in names:
        assert hasattr(L, nm), nm
    assert set(names) == set(sv._lib.EXPORTS)


def test_gate_dtype_matches_inputs():
    assert sv.GATE_DTYPE == C.GATE_DTYPE


def assert_same_pass(recs, n, c, flags=0, pi0=None):
    toks_o, pi_o = B.block_circuit(triples(recs), n, c, pi0=pi0, flags=flags)
    toks_l, pi_l = sv.block_circuit(recs, n, c, pi0=pi0, flags=flags)
    assert lib_tokens(toks_l) == toks_o
    assert list(pi_l) == list(pi_o)
    # gate payloads are copied bit-for-bit from the input records
    for r in toks_l:
        if int(r["kind"]) in (C.U1, C.U2, C.D1, C.D2, C.SWAP) and int(r["pad"]) >= 0:
            assert r["m"].tobytes() == recs[int(r["pad"])]["m"].tobytes()
    return toks_l, pi_l


@pytest.mark.parametrize("row", load_golden(os.path.join(ROOT, "tests", "golden", "blocking_traces.txt")))
def test_pass_golden(row):
    n, c, gates, expected, pi_expected, flags = row
    recs = parse_gates(gates, n)
    toks, pi = sv.block_circuit(recs, n, c, flags=flags)
    assert B.format_tokens(lib_tokens(toks)) == expected
    assert list(pi) == pi_expected


def test_pass_bit_exact_random_10k():
    # bit-exact with the independent pass on >= 10^4 random circuits.
    rng = np.random.default_rng(2024)
    for t in range(10000):
        n = int(rng.integers(2, 16))
        c = int(rng.integers(2, n + 1))
        ng = int(rng.integers(0, 40))
        kinds = ("u3", "cx", "cp", "swap", "su4", "u1", "d2") if t % 2 else ("cx", "su4", "cp")
        recs = C.random_circuit(n, ng, 77000 + t, kinds=kinds)
        pi0 = rng.permutation(n) if t % 5 == 0 else None
        flags = B.RESTORE_ORDER if t % 7 == 0 else 0
        assert_same_pass(recs, n, c, flags=flags, pi0=pi0)


@pytest.mark.parametrize("n,c", [(28, c) for c in range(8, 15)] + [(33, 12), (30, 10), (30, 12), (30, 13)])
def test_pass_bit_exact_qv(n, c):
    for seed in (1, 2, 3):
        assert_same_pass(C.quantum_volume(n, 10, seed), n, c)


@pytest.mark.parametrize("n,c", [(10, 6), (30, 10), (30, 11), (30, 12), (30, 13), (36, 12), (37, 12), (33, 12)])
def test_pass_bit_exact_qft(n, c):
    assert_same_pass(C.qft(n), n, c)


def test_pass_errors():
    with pytest.raises(sv.SvError, match="EINFEASIBLE"):
        sv.block_circuit(C.records([C.gate(C.U2, 0, 1, np.eye(4))]), 4, 1)
    with pytest.raises(sv.SvError, match="EINVAL"):
        sv.block_circuit(C.records([C.gate(C.U2, 0, 0, np.eye(4))]), 4, 2)
    with pytest.raises(sv.SvError, match="EINVAL"):
        sv.block_circuit(C.records([C.gate(C.U1, 5, mat=np.eye(2))]), 4, 2)
    bad = C.records([C.gate(C.U1, 0, mat=np.eye(2))])
    bad["kind"] = 42
    with pytest.raises(sv.SvError, match="EMALFORMED"):
        sv.block_circuit(bad, 4, 2)


def run_plan_dense(recs, n, c, g, flags=0, seed=0, basis_zero=False):
    """Execute the library's plan densely (exchange = SWAP of memory bits) and compare with the
    oracle on the original circuit, un-permuting through mu(q) = sigma[pi[q]]."""
    plan, pi, sigma = sv.plan_circuit(recs, n, c, g, flags=flags)
    nL = n - g
    # structural checks: section gates only on local memory bits unless diagonal; SWAP records
    # outside sections are physical memory-bit swaps (compaction / fused store swaps) on local
    # bits; every section tile can hold its bits plus the three lowest memory bits (coalescing)
    inside = False
    act = set()
    for r in plan:
        k = int(r["kind"])
        if k == C.BEGIN:
            inside, act = True, set()
        elif k == C.END:
            inside = False
            if len(act) <= 13 and nL >= 3:
                assert len(act | {0, 1, 2}) <= 13
        elif k == 9:
            assert not inside and int(r["q0"]) < nL <= int(r["q1"])
        elif k in (C.U1, C.U2):
            assert inside and int(r["q0"]) < nL and (k == C.U1 or int(r["q1"]) < nL)
            act |= {int(r["q0"])} | ({int(r["q1"])} if k == C.U2 else set())
        elif k == C.SWAP:
            assert (flags & sv.SV_UNBLOCKED) or (not inside and int(r["q0"]) < nL and int(r["q1"]) < nL)
    rng = np.random.default_rng(seed)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    if basis_zero:  # SV_FREE_LAYOUT plans assume a basis state; |0> sits at 0 under any layout
        psi = np.zeros(1 << n, dtype=np.complex128)
        psi[0] = 1
    ref = O.apply_circuit(recs, n, psi)
    mem = O.apply_circuit(plan_to_dense_records(plan), n, psi)
    got = O.unpermute(mem, memory_perm(pi, sigma))
    assert np.max(np.abs(got - ref)) <= 1e-12
    return plan


@pytest.mark.parametrize("g", [0, 1, 2, 3])
def test_plan_semantics_random(g):
    rng = np.random.default_rng(10 + g)
    for t in range(120):
        n = int(rng.integers(max(3, g + 2), 12))
        c = int(rng.integers(2, n - g + 1)) if n - g >= 2 else 1
        recs = C.random_circuit(n, int(rng.integers(0, 60)), 3000 + t + 1000 * g)
        run_plan_dense(recs, n, c, g, flags=B.RESTORE_ORDER if t % 3 == 0 else 0, seed=t)


@pytest.mark.parametrize("g", [0, 1, 2])
def test_plan_semantics_qv_qft(g):
    run_plan_dense(C.quantum_volume(10, 10, 1), 10, 5, g)
    plan = run_plan_dense(C.qft(10), 10, 6, g)
    if g == 0:  # single GPU: no data ever moves between sections
        assert not any(int(r["kind"]) == 9 for r in plan)


def test_plan_unblocked_matches():
    recs = C.random_circuit(8, 50, 5)
    plan = run_plan_dense(recs, 8, 4, 0, flags=sv.SV_UNBLOCKED)
    assert sum(1 for r in plan if int(r["kind"]) == C.BEGIN) == 50

    # several GPUs: the paper's unblocked multi-GPU baseline (NEXT-3) - a non-diagonal gate on a
    # global qubit is bracketed by two exchanges of its rank bit with a free local bit
    for g in (1, 2):
        recs = C.random_circuit(9, 60, 17 + g, kinds=("u3", "su4", "cx", "cp", "swap"))
        plan = run_plan_dense(recs, 9, 4, g, flags=sv.SV_UNBLOCKED)
        glob = set(range(9 - g, 9))
        want = 0
        for r in recs:
            k, qs = int(r["kind"]), {int(r["q0"])} | ({int(r["q1"])} if int(r["kind"]) in (C.U2, C.D2, C.SWAP) else set())
            if k in (C.D1, C.D2) or not (qs & glob):
                continue
            if k == C.SWAP and len(qs & glob) == 1:
                want += 1
            else:
                want += 2 * len(qs & glob)
        assert sum(1 for r in plan if int(r["kind"]) == 9) == want


def test_plan_splits_wide_sections():
    # chunk_bits above the 13-bit tile limit: sections are split (same pass at c = 13), never wider
    n = 18
    recs = C.quantum_volume(n, 8, 2)
    plan = run_plan_dense(recs, n, 16, 0)
    act, widest = set(), 0
    for r in plan:
        k = int(r["kind"])
        if k == C.BEGIN:
            act = set()
        elif k == C.END:
            widest = max(widest, len(act))
        elif k in (C.U1, C.U2):
            act |= {int(r["q0"])} | ({int(r["q1"])} if k == C.U2 else set())
    assert widest <= 13


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_jit_sources_compile_for_sm100a(prec, tmp_path):
    # the run-time specialised section kernels (jit.cpp) are generated and NVRTC-compiled on the
    # host; the GPU parity tests then run them.  Both the plain and the pipelined variant appear.
    n = 13
    recs = np.concatenate([C.qft(n), C.quantum_volume(n, 4, 3), C.random_circuit(n, 60, 5, kinds=("cp", "u3", "d2"))])
    k, ms = sv.jit_compile_circuit(recs, n, 10, precision=prec, flags=sv.SV_FREE_LAYOUT, dump_dir=str(tmp_path))
    assert k >= 3
    srcs = [open(p).read() for p in sorted(tmp_path.glob("section_*.cu"))]
    assert len(srcs) == k and len(list(tmp_path.glob("section_*.cubin"))) == k
    assert all("op_c<" in s for s in srcs)


@pytest.mark.parametrize("g", [1, 2, 3])
def test_two_level_and_free_layout_plans(g):
    # multi-GPU plans take the two-level form (outer pass at the shard size, NEXT-1) when it moves
    # fewer bytes; with SV_FREE_LAYOUT the first outer block starts local.  Dense semantics hold.
    for recs, n, c in [(C.quantum_volume(12, 8, 2), 12, 5), (C.qft(12), 12, 4),
                       (C.random_circuit(11, 150, 40 + g), 11, 4)]:
        run_plan_dense(recs, n, c, g, flags=sv.SV_FREE_LAYOUT, basis_zero=True)
        run_plan_dense(recs, n, c, g)


def test_two_level_exchange_volume_qv33():
    # QV(33, 10, 1), c = 9: cross-GPU exchanges per GPU in shard-equivalents (SURVEY §8(f) NEXT-1
    # predicted 1.5 / 2.25 / 2.62 for the two-level pass; the one-level Belady mapping needs
    # 2.5 / 4.5 / 6.1)
    circ = C.quantum_volume(33, 10, 1)
    for g, most in [(1, 1.0), (2, 1.5), (3, 2.5)]:
        plan, _, _ = sv.plan_circuit(circ, 33, 9, g, flags=sv.SV_FREE_LAYOUT)
        ex = plan[plan["kind"] == 9]
        batches = {}
        for r in ex:
            batches[int(r["pad"])] = batches.get(int(r["pad"]), 0) + 1
        vol = sum(1 - 2.0 ** -k for k in batches.values())
        assert vol <= most + 1e-9, (g, vol)


def test_nccl_exchange_plan_is_the_default_plan():
    # The NCCL send/recv exchange packs strided blocks into a staging buffer (kernels.cu
    # k_pack_bits), so it takes the same plan as the peer-memory exchange — the two-level plan
    # included — whatever local bits the exchanges pick (a victim restriction to the
    # top bits used to be ignored by the two-level plan).  QFT34 on 2 GPUs exchanges low bits.
    for n, g, circ in [(33, 2, C.quantum_volume(33, 10, 1)), (33, 3, C.quantum_volume(33, 10, 1)), (34, 1, C.qft(34))]:
        a, pa, sa = sv.plan_circuit(circ, n, 9, g, flags=sv.SV_EXCHANGE_NCCL | sv.SV_FREE_LAYOUT)
        b, pb, sb = sv.plan_circuit(circ, n, 9, g, flags=sv.SV_FREE_LAYOUT)
        assert np.array_equal(a, b) and np.array_equal(pa, pb) and np.array_equal(sa, sb)
        assert any(int(r["kind"]) == sv.SV_EXCHANGE for r in a)


def test_header_compiles_as_c_and_cpp():
    # include/sv.h is a plain C ABI: it must compile on its own as C99 and as C++
    import shutil
    import subprocess
    hdr = os.path.join(ROOT, "include", "sv.h")
    for cc, lang in (("gcc", ["-x", "c", "-std=c99"]), ("g++", ["-x", "c++", "-std=c++17"])):
        if shutil.which(cc):
            subprocess.run([cc, "-fsyntax-only", "-Wall", "-Werror", *lang, hdr], check=True)


def test_pass_absorb_swaps_bit_exact_and_plans():
    # SV_ABSORB_SWAPS (the paper's bit reordering P:287-289): the library's pass matches
    # the oracle's independent pass token for token on random swap-heavy circuits and QFT, and the
    # executor's plans built on it still compute the original circuit (dense, under pi / sigma).
    rng = np.random.default_rng(55)
    for t in range(3000):
        n = int(rng.integers(2, 14))
        c = int(rng.integers(2, n + 1))
        recs = C.random_circuit(n, int(rng.integers(0, 40)), 91000 + t, kinds=("u3", "cx", "swap", "cp", "su4"))
        flags = sv.SV_ABSORB_SWAPS | (B.RESTORE_ORDER if t % 6 == 0 else 0)
        assert_same_pass(recs, n, c, flags=flags, pi0=rng.permutation(n) if t % 4 == 0 else None)
    for n, c in [(10, 6), (16, 8), (30, 8), (36, 12)]:
        assert_same_pass(C.qft(n), n, c, flags=sv.SV_ABSORB_SWAPS)
        plain = sum(1 for r in sv.block_circuit(C.qft(n), n, c)[0] if int(r["kind"]) == C.BEGIN)
        absorbed = sum(1 for r in sv.block_circuit(C.qft(n), n, c, flags=sv.SV_ABSORB_SWAPS)[0] if int(r["kind"]) == C.BEGIN)
        assert absorbed < plain  # the terminal swap layer costs no section
    for g in (0, 1, 2):
        for t in range(40):
            n = int(rng.integers(g + 3, 11))
            c = int(rng.integers(2, n - g + 1))
            recs = C.random_circuit(n, int(rng.integers(0, 50)), 93000 + t, kinds=("u3", "cx", "swap", "cp", "su4"))
            run_plan_dense(recs, n, c, g, flags=sv.SV_ABSORB_SWAPS, seed=t)
