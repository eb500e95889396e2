"""Multi-rank parity on ONE GPU: the in-process virtual world (sv_world_create / sv_create_local).

G ranks, each a host thread with its own handle and shard on the same B200, run the multi-GPU path
end to end — the two-level plan, the packed-piece peer exchange and its pipeline with the sections,
the NCCL-style send/recv exchange (as device copies), the unblocked per-gate exchanges, every
collective readout — and rank 0's results are checked against the CPU oracle and against a
one-GPU run (tests/mgpu_cases.py).  PAPER.md P:137-166 (data distribution, pipelined exchange),
P:407-420 (chunk_swap across processes); SURVEY §8(a) a6, §8(f) NEXT-1..NEXT-3."""
import os

import numpy as np
import pytest

os.environ.setdefault("SV_COMM_TIMEOUT_S", "300")  # a failed rank thread must not hang the suite

import circuits as C  # noqa: E402
import mgpu_cases as M  # noqa: E402
from conftest import gpu_available  # noqa: E402

pytestmark = pytest.mark.gpu
sv = pytest.importorskip("paper_2102_02957_b200")

_REF, _ONE = {}, {}


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")
    import torch
    torch.cuda.set_device(0)


def run_world(world, case):
    name, recs, n, c, flags, basis, prec, second = case
    with sv.LocalWorld(world) as w:
        def body(r):
            with sv.StateVector(n, c, prec, rank=r, local_world=w) as s:
                return M.run_rank(s, case)
        return w.run(body)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("case", M.cases(), ids=[c[0] for c in M.cases()])
def test_local_world_parity(world, case):
    name = case[0]
    if name not in _REF:
        _REF[name] = M.reference(case)
        _ONE[name] = M.single_gpu(sv, case)
    res = run_world(world, case)
    checks, err, d1 = M.check(case, res[0], _REF[name], _ONE[name], world)
    bad = [k for k, ok in checks.items() if not ok]
    assert not bad, (name, world, bad, err, d1, res[0]["stats"])
    # every rank returned the same collective readouts
    for r in range(1, world):
        assert res[r]["state"] is None
        assert res[r]["norm"] == res[0]["norm"]
        assert np.array_equal(res[r]["probs"], res[0]["probs"])
        assert np.array_equal(res[r]["amps"], res[0]["amps"])
        assert np.array_equal(res[r]["shots"], res[0]["shots"])
        assert res[r]["stats"]["exchanges"] == res[0]["stats"]["exchanges"]


def test_local_world_two_level_volume():
    # The two-level plan (NEXT-1) moves fewer bytes than the one-level plan and the exchange byte
    # ledger matches the plan: bytes sent per rank = sum over batches of (1 - 2^-k) * shard bytes.
    n, c, world = 20, 8, 4
    circ = C.quantum_volume(n, 10, 3)
    recs, _, _ = sv.plan_circuit(circ, n, c, 2, flags=sv.SV_FREE_LAYOUT)
    batches = {}
    for r in recs:
        if int(r["kind"]) == sv.SV_EXCHANGE:
            batches.setdefault(int(r["pad"]), 0)
            batches[int(r["pad"])] += 1
    shard = 16 << (n - 2)
    want = sum((1 - 2.0 ** -k) * shard for k in batches.values())

    with sv.LocalWorld(world) as w:
        def body(r):
            with sv.StateVector(n, c, "fp64", rank=r, local_world=w) as s:
                s.reset(0)
                s.apply(circ)
                return s.stats()
        st = w.run(body)
    assert st[0]["exchange_batches"] == len(batches)
    assert st[0]["bytes_sent"] == int(want)


def test_local_world_errors():
    # a world of a non-power-of-two size and a rank outside the world are rejected (SV_EINVAL)
    with pytest.raises(sv.SvError):
        sv.LocalWorld(3)
    with sv.LocalWorld(2) as w:
        with pytest.raises(sv.SvError):
            sv.StateVector(12, 4, rank=2, local_world=w)


def test_local_world_interpreter_shared_constants():
    # The interpreter kernel reads its program from the module's one __constant__ bank; four ranks
    # on four streams copy and launch concurrently, serialised by the per-device event chain
    # (section.cu launch_section).  Without it a rank's launch could read another's program.
    import oracle as O
    prev = sv.jit_mode(0)
    try:
        for world, (n, c, circ) in [(4, (14, 6, C.quantum_volume(14, 6, 11))), (2, (13, 5, C.qft(13)))]:
            with sv.LocalWorld(world) as w:
                def body(r):
                    with sv.StateVector(n, c, "fp64", rank=r, local_world=w) as s:
                        s.reset(3)
                        s.apply(circ)
                        st = s.stats()
                        return s.state(), st
                res = w.run(body)
            got, st = res[0]
            assert st["interp_launches"] > 0 and st["jit_launches"] == 0
            assert float(np.max(np.abs(got - O.apply_circuit(circ, n, basis=3)))) <= 1e-10
    finally:
        sv.jit_mode(prev)


@pytest.mark.parametrize("xrun,xceu", [("16", "0"), ("16", "1"), ("1024", "1"), ("0", "1")])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_local_world_copy_engine_gather(world, xrun, xceu, monkeypatch):
    # The copy-engine form of the exchange (api.cpp exchange, kernels.cu copy_bits_ce): rows of the
    # block go straight from the state into the peer's slot as strided 2-D copies when its runs are
    # >= SV_XRUN bytes, and back into place the same way (SV_XCEU=0: the unpack kernel instead).
    # SV_XRUN=16 forces the copies for every exchanged bit (one-element rows), 1024 (the default)
    # only for bits >= 6, 0 packs and unpacks with kernels; all against the oracle.
    monkeypatch.setenv("SV_XRUN", xrun)
    monkeypatch.setenv("SV_XCEU", xceu)
    for case in [c for c in M.cases() if c[0] in ("qv", "qft", "rand", "qv-twice", "qft-fp32")]:
        name = case[0]
        if name not in _REF:
            _REF[name] = M.reference(case)
            _ONE[name] = M.single_gpu(sv, case)
        res = run_world(world, case)
        checks, err, d1 = M.check(case, res[0], _REF[name], _ONE[name], world)
        bad = [k for k, ok in checks.items() if not ok]
        assert not bad, (name, world, xrun, xceu, bad, err, d1)


@pytest.mark.parametrize("xchain", ["0", "1", "16"])
@pytest.mark.parametrize("world", [2, 4])
def test_local_world_pipeline_chains(world, xchain, monkeypatch):
    # The executor's pipeline plan (api.cpp apply_circuit / exchange): up to SV_XCHAIN section
    # launches on either side of an exchange run quarter by quarter around it (0: none, the pieces
    # still grouped by the split bits; 1: one launch each side; 16: long chains across sections).
    monkeypatch.setenv("SV_XCHAIN", xchain)
    for case in [c for c in M.cases() if c[0] in ("qv", "qft", "rand", "qv-twice", "qft-absorb")]:
        name = case[0]
        if name not in _REF:
            _REF[name] = M.reference(case)
            _ONE[name] = M.single_gpu(sv, case)
        res = run_world(world, case)
        checks, err, d1 = M.check(case, res[0], _REF[name], _ONE[name], world)
        bad = [k for k, ok in checks.items() if not ok]
        assert not bad, (name, world, xchain, bad, err, d1)


@pytest.mark.parametrize("xrun", ["16", "1024"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_local_world_inplace_exchange(world, xrun, monkeypatch):
    # The in-place form of the exchange (SV_XINPLACE=1, api.cpp exchange): per group of pieces one
    # rank of each pair stages its rows into the partner's slot, the partner writes its rows straight
    # into the stager's state after the piece's barrier and unpacks its slot; roles alternate.
    monkeypatch.setenv("SV_XINPLACE", "1")
    monkeypatch.setenv("SV_XRUN", xrun)
    for case in [c for c in M.cases() if c[0] in ("qv", "qft", "rand", "qv-twice", "qft-fp32", "qft-absorb")]:
        name = case[0]
        if name not in _REF:
            _REF[name] = M.reference(case)
            _ONE[name] = M.single_gpu(sv, case)
        res = run_world(world, case)
        checks, err, d1 = M.check(case, res[0], _REF[name], _ONE[name], world)
        bad = [k for k, ok in checks.items() if not ok]
        assert not bad, (name, world, xrun, bad, err, d1)
