"""Helpers for tests that call the library's host-only entry points."""
import numpy as np

import circuits as C

TOKEN = {C.CHUNK_SWAP: "CS", C.BEGIN: "BEGIN", C.END: "END"}


def lib_tokens(recs):
    """libsv token records -> the oracle pass's tuple format."""
    out = []
    for r in recs:
        k = int(r["kind"])
        if k == C.CHUNK_SWAP:
            out.append(("CS", int(r["q0"]), int(r["q1"])))
        elif k in (C.BEGIN, C.END):
            out.append((TOKEN[k],))
        else:
            out.append((k, int(r["q0"]), int(r["q1"]) if k in (C.U2, C.D2, C.SWAP) else -1, int(r["pad"])))
    return out


def memory_perm(pi, sigma):
    """logical qubit q -> memory bit sigma[pi[q]]"""
    return [int(sigma[int(p)]) for p in pi]


def plan_to_dense_records(recs):
    """Plan records -> records the dense oracle can run on the full memory-ordered vector:
    EXCHANGE(m, b) is a SWAP of memory bits m and b; markers are kept (no-ops)."""
    out = []
    for r in recs:
        k = int(r["kind"])
        if k == 9:  # SV_EXCHANGE
            out.append(C.gate(C.SWAP, int(r["q0"]), int(r["q1"])))
        else:
            out.append(np.array(r, dtype=C.GATE_DTYPE))
    return C.records(out)
