"""Multi-rank parity cases, shared by tests/mgpu_worker.py (torchrun: one process per GPU, NCCL +
CUDA IPC peer memory) and tests/test_local_world.py (an in-process virtual world: G ranks on one
GPU, sv_create_local).  Both run every case through the C ABI on every rank and judge the result on
rank 0 against the CPU oracle and against a one-GPU run of the same circuit.

What the cases exercise (SURVEY §8(a) a6 / §8(f) NEXT-1..3):
  * qv / qft / rand / ghz: the blocked path — two-level plan when it moves less (NEXT-1), the
    pipelined peer-memory exchange, free initial layout after sv_reset (NEXT-2);
  * qv-nccl: the send/recv exchange through a staging buffer (SV_EXCHANGE_NCCL);
  * qv-restore: SV_RESTORE_ORDER (order restored physically);
  * qv-unblocked: the paper's unblocked multi-GPU baseline (per-gate exchanges, NEXT-3);
  * qv-twice: a second circuit on the layout the first one left (no free layout);
  * qft-fp32: the fp32 path; qft-absorb: SV_ABSORB_SWAPS (swaps as relabels of pi).
G-invariance (SURVEY P-G): a plan on G ranks relabels and exchanges bits differently from the
one-GPU plan, so sections group gates into different phases, DIAGSETs and slot orders; amplitudes
then agree to rounding (asserted: max |d| <= 1e-12), and bitwise only where every operation is
exact — GHZ (H, then CNOT permutations) is asserted bitwise.
"""
from __future__ import annotations

import numpy as np

import circuits as C


def cases():
    """(name, records, n, chunk_bits, flags, basis, precision, second circuit or None)."""
    SV_UNBLOCKED, SV_RESTORE_ORDER, SV_EXCHANGE_NCCL, SV_ABSORB_SWAPS = 1, 2, 4, 32
    return [
        ("qv", C.quantum_volume(20, 10, 1), 20, 10, 0, 0, "fp64", None),
        ("qv-nccl", C.quantum_volume(20, 10, 2), 20, 10, SV_EXCHANGE_NCCL, 0, "fp64", None),
        ("qft", C.qft(22), 22, 12, 0, C.basis_index(7, 22), "fp64", None),
        ("rand", C.random_circuit(18, 300, 5), 18, 8, 0, 0, "fp64", None),
        ("qv-restore", C.quantum_volume(16, 8, 3), 16, 6, SV_RESTORE_ORDER, 0, "fp64", None),
        ("ghz", C.ghz(21), 21, 5, 0, 0, "fp64", None),
        ("qv-unblocked", C.quantum_volume(16, 3, 4), 16, 6, SV_UNBLOCKED, 0, "fp64", None),
        ("qv-twice", C.quantum_volume(18, 6, 6), 18, 7, 0, C.basis_index(3, 18), "fp64", C.qft(18)),
        ("qft-fp32", C.qft(20), 20, 9, 0, C.basis_index(5, 20), "fp32", None),
        ("qft-nccl", C.qft(19), 19, 7, SV_EXCHANGE_NCCL, C.basis_index(2, 19), "fp64", None),
        ("qft-absorb", C.qft(20), 20, 8, SV_ABSORB_SWAPS, C.basis_index(6, 20), "fp64", None),
    ]


AMP_IDX = lambda n: np.array([0, 1, (1 << n) - 1, 12345 % (1 << n)], dtype=np.uint64)  # noqa: E731
MARG_Q = lambda n: [0, n - 1, n // 2]  # noqa: E731


def run_rank(s, case):
    """Every rank: simulate the case on its handle; returns the readouts (state on rank 0 only)."""
    name, recs, n, c, flags, basis, prec, second = case
    s.reset(basis)
    s.apply(recs, flags=flags)
    if second is not None:
        s.apply(second, flags=flags)
    st = s.stats()
    return dict(state=s.state(), norm=s.norm(), probs=s.probabilities(MARG_Q(n)), amps=s.amplitudes(AMP_IDX(n)),
                shots=s.sample(20000, 3), stats=st)


def reference(case):
    """The oracle's state for the case (O.apply_circuit: plain per-gate loops, no blocking)."""
    import oracle as O
    name, recs, n, c, flags, basis, prec, second = case
    ref = O.apply_circuit(recs, n, basis=basis)
    if second is not None:
        ref = O.apply_circuit(second, n, ref)
    return ref


def single_gpu(sv, case):
    """The same case on one GPU (sv_create) for the G-invariance check."""
    name, recs, n, c, flags, basis, prec, second = case
    with sv.StateVector(n, c, prec) as one:
        one.reset(basis)
        one.apply(recs, flags=flags)
        if second is not None:
            one.apply(second, flags=flags)
        return one.state()


def check(case, res, ref, single, world):
    """Judge rank 0's readouts; returns {check: ok} and the max deviation from the oracle."""
    import oracle as O
    name, recs, n, c, flags, basis, prec, second = case
    got = res["state"]
    tol, ntol = (1e-10, 1e-12) if prec == "fp64" else (1e-4, 1e-5)
    err = float(np.max(np.abs(got - ref)))
    d_single = float(np.max(np.abs(got.astype(np.complex128) - single.astype(np.complex128))))
    idx = AMP_IDX(n)
    checks = {
        "oracle": err <= tol,
        "oracle_l2": float(np.linalg.norm(got - ref)) <= (1e-12 if prec == "fp64" else 1e-5),
        "norm": abs(res["norm"] - 1) <= ntol,
        "probs": float(np.max(np.abs(res["probs"] - O.marginal(ref, MARG_Q(n))))) <= ntol,
        "amps": float(np.max(np.abs(res["amps"] - ref[idx.astype(np.int64)]))) <= tol,
        "shots_valid": bool(np.all(np.abs(ref[res["shots"].astype(np.int64)]) > 0)),
        "exchanged": world == 1 or res["stats"]["exchanges"] > 0 or name in ("ghz",),
        "g_invariant": d_single <= (1e-12 if prec == "fp64" else 1e-6),
    }
    if name == "ghz":
        checks["g_invariant_bitwise"] = bool(np.array_equal(got, single))
    return checks, err, d_single
