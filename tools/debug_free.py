import sys, numpy as np
sys.path.insert(0, '.')
import circuits as C, oracle as O
import paper_2102_02957_b200 as sv
import torch
rng = np.random.default_rng(11)
for t in range(40):
    n = int(rng.integers(2, 17))
    c = min(int(rng.integers(2, n + 1)), 13)
    circ = C.random_circuit(n, int(rng.integers(0, 120)), 500 + t)
    ref = O.apply_circuit(circ, n)
    for pre in (False, True):
        with sv.StateVector(n, c, "fp64") as s:
            if pre: s.apply(circ[:0])
            s.apply(circ)
            got = s.state()
        e = np.abs(got - ref).max()
        if e > 1e-10:
            st = sv.compile_circuit(circ, n, c, 0, 0, "fp64", 0 if pre else sv.SV_FREE_LAYOUT)[0]
            print(f"t={t} n={n} c={c} gates={len(circ)} pre={pre} err={e:.3g} steps:\n{st[:, :10]}", flush=True)
print("done")
