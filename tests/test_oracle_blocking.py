"""Pins for the oracle's independent blocking pass (oracle/blocking.py): golden traces, and the
semantic contract — the blocked circuit executed densely equals the input after un-permuting
by the final pi (DESIGN R7) — plus the structural properties of Listing 3."""
import os

import numpy as np
import pytest

import circuits as C
import oracle as O
from oracle import blocking as B

from blockutil import load_golden, parse_gates, tokens_to_records, triples

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "blocking_traces.txt")


@pytest.mark.parametrize("row", load_golden(GOLDEN))
def test_golden_traces(row):
    n, c, gates, expected, pi_expected, flags = row
    recs = parse_gates(gates, n)
    toks, pi = B.block_circuit(triples(recs), n, c, flags=flags)
    assert B.format_tokens(toks) == expected
    assert pi == pi_expected


def check_semantics(recs, n, c, flags=0, seed=0):
    toks, pi = B.block_circuit(triples(recs), n, c, flags=flags)
    assert B.verify_blocked(toks, c)
    rng = np.random.default_rng(seed)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    ref = O.apply_circuit(recs, n, psi)
    phys = O.apply_circuit(tokens_to_records(toks, recs), n, psi)
    assert np.max(np.abs(O.unpermute(phys, pi) - ref)) <= 1e-12
    if flags & B.RESTORE_ORDER:
        assert pi == list(range(n))
    return toks, pi


def test_semantic_equivalence_random():
    # 300 random circuits, n in [4, 12], c in [2, n]: blocked == original under pi.
    rng = np.random.default_rng(123)
    for t in range(300):
        n = int(rng.integers(4, 13)) if t % 3 else int(rng.integers(4, 9))
        c = int(rng.integers(2, n + 1))
        recs = C.random_circuit(n, int(rng.integers(0, 80)), 1000 + t)
        check_semantics(recs, n, c, flags=B.RESTORE_ORDER if t % 4 == 0 else 0, seed=t)


@pytest.mark.parametrize("n,c", [(8, 3), (10, 4), (10, 6), (12, 8)])
def test_semantics_qv_qft(n, c):
    check_semantics(C.quantum_volume(n, 10, 1), n, c)
    check_semantics(C.qft(n), n, c)


def test_per_qubit_order_preserved_and_structure():
    # per-qubit gate subsequences are preserved (reorder legality); chunk_swaps
    # have sq0 < c <= sq1; batches between sections act on disjoint qubits; every section is
    # non-empty and consecutive sections are separated by >= 1 chunk_swap (progress).
    rng = np.random.default_rng(5)
    for t in range(400):
        n = int(rng.integers(3, 14)); c = int(rng.integers(2, n + 1))
        recs = C.random_circuit(n, int(rng.integers(1, 120)), 5000 + t)
        toks, pi = B.block_circuit(triples(recs), n, c)
        emitted = [tk[3] for tk in toks if tk[0] not in ("CS", "BEGIN", "END")]
        assert sorted(emitted) == list(range(len(recs)))  # every gate exactly once
        for q in range(n):
            sub = [i for i in emitted if q in C.qubits_of(recs[i])]
            assert sub == sorted(sub)
        batch, sections, in_sec, cur = [], 0, False, 0
        for tk in toks:
            if tk[0] == "CS":
                assert tk[1] < c <= tk[2]
                batch.append(tk)
            elif tk[0] == "BEGIN":
                qs = [q for b_ in batch for q in b_[1:]]
                assert len(qs) == len(set(qs))
                if sections > 0:
                    assert batch, "consecutive sections need a chunk_swap between them"
                batch, in_sec, cur = [], True, 0
                sections += 1
            elif tk[0] == "END":
                assert cur > 0
                in_sec = False
            else:
                cur += 1


def test_idempotent_on_local_circuit():
    # a circuit already below c -> zero swaps, one section, pi = identity.
    n, c = 10, 6
    recs = C.random_circuit(c, 50, 77)
    toks, pi = B.block_circuit(triples(recs), n, c)
    assert [t for t in toks if t[0] == "CS"] == []
    assert sum(1 for t in toks if t[0] == "BEGIN") == 1
    assert pi == list(range(n))


def test_diagonals_never_force_swaps():
    # R5: a circuit of diagonal gates on any qubits blocks into one section, no swaps.
    n, c = 12, 3
    recs = C.random_circuit(n, 60, 3, kinds=("cp", "u1", "d2"))
    toks, pi = B.block_circuit(triples(recs), n, c)
    assert [t[0] for t in toks].count("CS") == 0 and pi == list(range(n))


def test_infeasible():
    with pytest.raises(B.Infeasible):
        B.block_circuit([(C.U2, 0, 1)], 4, 1)
    toks, _ = B.block_circuit([(C.D2, 0, 1), (C.U1, 3, -1)], 4, 1)
    assert B.verify_blocked(toks, 1)


def test_absorb_swaps_semantics():
    # ABSORB_SWAPS: user SWAPs become relabels of pi; the blocked circuit (no SWAP tokens left)
    # executed densely and un-permuted by the final pi equals the input circuit, and no emitted
    # section is empty.
    rng = np.random.default_rng(321)
    for t in range(300):
        n = int(rng.integers(3, 11))
        c = int(rng.integers(2, n + 1))
        recs = C.random_circuit(n, int(rng.integers(0, 60)), 5000 + t, kinds=("u3", "cx", "swap", "cp", "su4", "d2"))
        flags = B.ABSORB_SWAPS | (B.RESTORE_ORDER if t % 5 == 0 else 0)
        toks, pi = check_semantics(recs, n, c, flags=flags, seed=t)
        body = [tk for tk in toks if tk[0] not in ("BEGIN", "END", "CS")]
        if not flags & B.RESTORE_ORDER:
            assert all(tk[0] != B.SWAP for tk in body)
        for a, b in zip(toks, toks[1:]):
            assert not (a[0] == "BEGIN" and b[0] == "END")
