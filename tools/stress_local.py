"""Randomised multi-rank parity sweep on ONE GPU (not part of the test suite): fuzz circuits on an
in-process virtual world of G = 2, 4 or 8 ranks (sv_create_local), random chunk_bits, precision,
exchange transport (copy engine with or without the pack kernel, copy-engine unpack, NCCL-style send/recv), swap absorption, unblocked
mode, a second circuit on the left-over layout; rank 0's state against the oracle.
usage: python tools/stress_local.py [seed] [cases]"""
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
os.environ.setdefault("SV_COMM_TIMEOUT_S", "120")
import circuits as C  # noqa: E402
import oracle as O  # noqa: E402
import paper_2102_02957_b200 as sv  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
count = int(sys.argv[2]) if len(sys.argv) > 2 else 120
bad = 0
for t in range(count):
    world = int(rng.choice([2, 4, 8]))
    g = world.bit_length() - 1
    n = int(rng.integers(g + 6, 19))
    c = int(rng.integers(2, min(n - g, 12) + 1))
    prec = "fp64" if rng.random() < 0.75 else "fp32"
    flags = 0
    r = rng.random()
    if r < 0.2:
        flags |= sv.SV_EXCHANGE_NCCL
    elif r < 0.3:
        flags |= sv.SV_UNBLOCKED
    if rng.random() < 0.25 and not flags & sv.SV_UNBLOCKED:
        flags |= sv.SV_ABSORB_SWAPS
    kinds = [("u3", "cx", "cp", "swap", "su4", "u1", "d2"), ("u3", "su4"), ("cp", "u1", "d2", "u3", "swap")][t % 3]
    circ = C.random_circuit(n, int(rng.integers(1, 200)), 20000 + t, kinds=kinds)
    k = int(rng.integers(0, 1 << n))
    os.environ["SV_XRUN"] = str(rng.choice(["16", "256", "1024", "0"]))  # copy-engine gather threshold
    os.environ["SV_XCEU"] = str(rng.choice(["0", "1"]))  # copy-engine unpack
    os.environ["SV_XCHAIN"] = str(rng.choice(["0", "1", "4", "16"]))  # launches pipelined per exchange side
    os.environ["SV_XINPLACE"] = str(rng.choice(["0", "1"]))  # in-place exchange form
    try:
        with sv.LocalWorld(world) as w:
            def body(rank):
                with sv.StateVector(n, c, prec, rank=rank, local_world=w) as s:
                    s.reset(k)
                    s.apply(circ, flags=flags)
                    s.apply(circ[: len(circ) // 3], flags=flags)
                    return s.state()
            got = w.run(body)[0]
        ref = O.apply_circuit(circ[: len(circ) // 3], n, O.apply_circuit(circ, n, basis=k))
        err = float(np.max(np.abs(got.astype(np.complex128) - ref)))
        tol = 1e-10 if prec == "fp64" else 1e-4
        if not err <= tol:
            bad += 1
            print(f"FAIL t={t} G={world} n={n} c={c} {prec} flags={flags} gates={len(circ)} err={err:.3g} "
                  f"xrun={os.environ['SV_XRUN']} xceu={os.environ['SV_XCEU']} xchain={os.environ['SV_XCHAIN']} inplace={os.environ['SV_XINPLACE']}", flush=True)
    except Exception as e:  # noqa: BLE001
        bad += 1
        print(f"ERROR t={t} G={world} n={n} c={c} {prec} flags={flags}: {e}", flush=True)
print(f"stress_local: {count} cases, {bad} failures", flush=True)
