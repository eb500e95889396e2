"""Randomised parity sweep on one GPU (not part of the test suite): many (n, c, precision, mode)
combinations of fuzz circuits against the oracle; prints failures."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import circuits as C  # noqa: E402
import oracle as O  # noqa: E402
import paper_2102_02957_b200 as sv  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
count = int(sys.argv[2]) if len(sys.argv) > 2 else 200
bad = 0
for t in range(count):
    n = int(rng.integers(4, 19))
    c = int(rng.integers(2, min(n, 13) + 1))
    prec = "fp64" if rng.random() < 0.7 else "fp32"
    mode = 1 if rng.random() < 0.8 else 0
    kinds = [("u3", "cx", "cp", "swap", "su4", "u1", "d2"), ("u3", "su4"), ("cp", "u1", "d2", "u3", "swap")][t % 3]
    circ = C.random_circuit(n, int(rng.integers(1, 250)), 10000 + t, kinds=kinds)
    k = int(rng.integers(0, 1 << n))
    sv.jit_mode(mode)
    try:
        with sv.StateVector(n, c, prec) as s:
            s.reset(k)
            s.apply(circ)
            s.apply(circ[: len(circ) // 3])
            got = s.state()
        ref = O.apply_circuit(circ[: len(circ) // 3], n, O.apply_circuit(circ, n, basis=k))
        err = float(np.max(np.abs(got.astype(np.complex128) - ref)))
        tol = 1e-10 if prec == "fp64" else 1e-4
        if not err <= tol:
            bad += 1
            print(f"FAIL t={t} n={n} c={c} {prec} mode={mode} gates={len(circ)} err={err:.3g}", flush=True)
    except Exception as e:  # noqa: BLE001
        bad += 1
        print(f"ERROR t={t} n={n} c={c} {prec} mode={mode}: {e}", flush=True)
print(f"stress: {count} cases, {bad} failures", flush=True)
