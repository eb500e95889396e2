"""Helpers shared by the blocking-pass tests (parsing golden rows, converting token streams)."""
import re

import numpy as np

import circuits as C

_G = re.compile(r"(U1|U2|D1|D2|SW)\((\d+)(?:,(\d+))?\)")
KIND = {"U1": C.U1, "U2": C.U2, "D1": C.D1, "D2": C.D2, "SW": C.SWAP}


def parse_gates(text: str, n: int):
    if text.strip() == "QFT4":
        return C.qft(4)
    rng = np.random.default_rng(0)
    gs = []
    for m in _G.finditer(text):
        k = KIND[m.group(1)]
        q0 = int(m.group(2)); q1 = int(m.group(3)) if m.group(3) else -1
        if k == C.U1:
            gs.append(C.gate(k, q0, mat=C.u3(*rng.uniform(0, 3, 3))))
        elif k == C.U2:
            gs.append(C.gate(k, q0, q1, C.haar_su(rng, 4)))
        elif k == C.D1:
            gs.append(C.gate(k, q0, mat=C.u1_diag(0.3)))
        elif k == C.D2:
            gs.append(C.gate(k, q0, q1, C.cphase_diag(0.7)))
        else:
            gs.append(C.gate(k, q0, q1))
    return C.records(gs)


def load_golden(path):
    rows = []
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        head, gates, out, pi = (s.strip() for s in line.split("|"))
        words = head.split()
        n, c = int(words[0]), int(words[1])
        flags = 32 if "absorb" in words[2:] else 0  # SV_ABSORB_SWAPS / oracle.blocking.ABSORB_SWAPS
        rows.append((n, c, gates, out, [int(x) for x in pi.split()], flags))
    return rows


def triples(recs):
    return [(int(r["kind"]), int(r["q0"]), int(r["q1"])) for r in recs]


def tokens_to_records(tokens, recs):
    """Blocked token stream -> executable records (CS -> CHUNK_SWAP, markers kept, gates carry
    their input record's matrix bit-for-bit)."""
    out = []
    for t in tokens:
        if t[0] == "CS":
            out.append(C.gate(C.CHUNK_SWAP, t[1], t[2]))
        elif t[0] == "BEGIN":
            out.append(C.gate(C.BEGIN, -1))
        elif t[0] == "END":
            out.append(C.gate(C.END, -1))
        else:
            k, q0, q1, gi = t
            g = np.array(recs[gi], dtype=C.GATE_DTYPE) if gi >= 0 else C.gate(k, q0, q1)
            g["kind"], g["q0"], g["q1"] = k, q0, q1
            out.append(g)
    return C.records(out)
