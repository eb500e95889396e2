"""Independent cache-blocking pass — TEST INFRASTRUCTURE ONLY (the oracle's copy of the pass).

Follows Listing 3 of the paper with the prose of P:324-326 and P:350, in the
paper's order, with every ambiguity resolved by the DESIGN.md readings (R2-R6, R9):

    while REMAINING is not empty
      choose QB_CHUNK qubits                            (R2 all c slots, R3 in-order rule)
      put chunk_swap gates in OUTPUT                    (R4 descending free slot)
      clear QB_BLOCKED
      for gates in REMAINING
        if qubits in chunk and not blocked: OUTPUT      (R5 diagonals always local)
        else: set QB_BLOCKED on its qubits; NEXT        (R2' "set QB_BLOCKED")
      REMAINING <- NEXT

The GPU library's pass (paper_2102_02957_b200/csrc/blocking.cpp) is written separately in
C++; tests require the two token streams to be identical.  This module imports nothing from
the product package and holds no amplitude arithmetic.

Token stream: list of tuples
    ("CS", sq0, sq1)            chunk_swap, sq0 < sq1 (paper-physical qubits)
    ("BEGIN",) / ("END",)       section markers
    (kind, q0, q1, index)       an input gate (kind in U1..SWAP) on physical qubits, with the
                                index of the input record whose matrix it carries bit-for-bit.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

U1, U2, D1, D2, SWAP = 1, 2, 3, 4, 5
RESTORE_ORDER = 1 << 1
ABSORB_SWAPS = 1 << 5  # a user SWAP relabels pi instead of being a 2-qubit gate


class Infeasible(ValueError):
    """A non-diagonal two-qubit gate cannot fit a chunk of c < 2 qubits."""


def _qubits(kind: int, q0: int, q1: int) -> Tuple[int, ...]:
    return (q0,) if kind in (U1, D1) else (q0, q1)


def _diagonal(kind: int) -> bool:
    return kind in (D1, D2)


def block_circuit(gates: Sequence[Tuple[int, int, int]], n: int, c: int,
                  pi0: Optional[Sequence[int]] = None, flags: int = 0):
    """gates: sequence of (kind, q0, q1) in logical qubits.  Returns (tokens, pi_final) where
    pi_final[q] is the physical position of logical qubit q after the blocked circuit."""
    if not (1 <= c <= n):
        raise ValueError("need 1 <= c <= n")
    for (k, q0, q1) in gates:
        if not _diagonal(k) and k != U1 and c < 2:
            raise Infeasible("non-diagonal 2-qubit gate with c < 2")
    pi = list(range(n)) if pi0 is None else [int(x) for x in pi0]
    inv = [0] * n
    for q, p in enumerate(pi):
        inv[p] = q
    out: List[tuple] = []
    remaining = list(range(len(gates)))

    absorb = bool(flags & ABSORB_SWAPS)
    while remaining:
        # ---- choose QB_CHUNK (R3: in order, dependency aware, whole-gate admission).  With
        # ABSORB_SWAPS a swap is no gate: later gates on its qubits act on the state that was on
        # the other qubit at the start of the section (start[q]).
        S: List[int] = []
        blocked = set()
        start = list(range(n))
        for gi in remaining:
            k, q0, q1 = gates[gi]
            qs = _qubits(k, q0, q1)
            if blocked.intersection(qs):
                blocked.update(qs)
                continue
            if _diagonal(k):
                continue
            if absorb and k == SWAP:
                start[q0], start[q1] = start[q1], start[q0]
                continue
            need = [q for q in sorted(start[x] for x in qs) if q not in S]
            if len(S) + len(need) <= c:
                S.extend(need)
            else:
                blocked.update(qs)
            if len(S) == c:
                break
        # ---- chunk_swaps: bring each selected qubit outside the chunk into a free slot (R4)
        incoming = [q for q in S if pi[q] >= c]
        free = sorted((p for p in range(c) if inv[p] not in S), reverse=True)
        for i, q in enumerate(incoming):
            p = free[i]
            sq1 = pi[q]
            out.append(("CS", p, sq1))
            evicted = inv[p]
            pi[evicted], pi[q] = sq1, p
            inv[sq1], inv[p] = evicted, q
        # ---- emit the section
        out.append(("BEGIN",))
        opened = len(out)
        blocked = set()
        nxt: List[int] = []
        for gi in remaining:
            k, q0, q1 = gates[gi]
            qs = _qubits(k, q0, q1)
            if blocked.intersection(qs):
                blocked.update(qs)
                nxt.append(gi)
                continue
            if absorb and k == SWAP:  # relabel: the states of q0 and q1 trade physical positions
                pi[q0], pi[q1] = pi[q1], pi[q0]
                inv[pi[q0]], inv[pi[q1]] = q0, q1
                continue
            if _diagonal(k) or all(pi[q] < c for q in qs):
                out.append((k, pi[q0], pi[q1] if len(qs) == 2 else -1, gi))
            else:
                blocked.update(qs)
                nxt.append(gi)
        if len(out) == opened:
            out.pop()  # only absorbed swaps: no section
        else:
            out.append(("END",))
        remaining = nxt

    if flags & RESTORE_ORDER:
        # P:379 case (b) "only occurs when we reorder qubits for the output" (R7).
        for p in range(n):
            q = inv[p]
            if q == p:
                continue
            t = pi[p]  # physical position of logical p; t > p because positions < p are settled
            if t >= c:
                out.append(("CS", p, t))
            else:
                out.append(("BEGIN",))
                out.append((SWAP, p, t, -1))
                out.append(("END",))
            pi[q], pi[p] = t, p
            inv[t], inv[p] = q, p
    return out, pi


def verify_blocked(tokens, c: int) -> bool:
    """every non-marker non-diagonal gate acts only on physical qubits < c, chunk_swaps
    have sq0 < sq1 with sq1 >= c, and BEGIN/END nest properly."""
    inside = False
    for t in tokens:
        if t[0] == "BEGIN":
            if inside:
                return False
            inside = True
        elif t[0] == "END":
            if not inside:
                return False
            inside = False
        elif t[0] == "CS":
            if inside or not (t[1] < t[2] and t[2] >= c):
                return False
        else:
            k, q0, q1 = t[0], t[1], t[2]
            if not inside:
                return False
            if not _diagonal(k) and any(q >= c for q in _qubits(k, q0, q1)):
                return False
    return not inside


def format_tokens(tokens) -> str:
    names = {U1: "U1", U2: "U2", D1: "D1", D2: "D2", SWAP: "SW"}
    parts = []
    for t in tokens:
        if t[0] == "CS":
            parts.append(f"CS({t[1]},{t[2]})")
        elif t[0] == "BEGIN":
            parts.append("[")
        elif t[0] == "END":
            parts.append("]")
        else:
            k = t[0]
            parts.append(f"{names[k]}({t[1]})" if k in (U1, D1) else f"{names[k]}({t[1]},{t[2]})")
    return " ".join(parts)
