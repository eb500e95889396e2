"""Small runs of every kernel family for compute-sanitizer (tools/sanitize.sh): generated section
kernels (QFT10 c=6, QV12 c=8, fp64 + fp32), the interpreter, the per-gate baseline, the readouts
(norm, marginals, sampling, amplitude gather) and a two-rank local world (exchange push / unpack
kernels, pipelined with the next section).  Checks parity against the oracle too."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import circuits as C  # noqa: E402
import oracle as O  # noqa: E402
import paper_2102_02957_b200 as sv  # noqa: E402


def run(n, c, circ, prec, flags=0, basis=0):
    with sv.StateVector(n, c, prec) as s:
        s.reset(basis)
        s.apply(circ, flags=flags)
        got = s.state()
        s.norm()
        s.probabilities([0, n - 1])
        s.sample(1000, 1)
        s.amplitudes(np.array([0, 3], dtype=np.uint64))
    ref = O.apply_circuit(circ, n, basis=basis)
    err = float(np.max(np.abs(got - ref)))
    assert err <= (1e-10 if prec == "fp64" else 1e-4), err
    return err


def main():
    import torch
    torch.cuda.set_device(0)
    print("qft10", run(10, 6, C.qft(10), "fp64", basis=C.basis_index(1, 10)))
    print("qv12", run(12, 8, C.quantum_volume(12, 4, 1), "fp64"))
    print("qv12 fp32", run(12, 8, C.quantum_volume(12, 4, 1), "fp32"))
    print("rand unblocked", run(11, 6, C.random_circuit(11, 40, 2), "fp64", flags=sv.SV_UNBLOCKED))
    prev = sv.jit_mode(0)
    print("qv12 interpreter", run(12, 8, C.quantum_volume(12, 3, 2), "fp64"))
    sv.jit_mode(prev)
    n, c, circ = 13, 6, C.quantum_volume(13, 4, 3)
    with sv.LocalWorld(2) as w:
        def body(r):
            with sv.StateVector(n, c, "fp64", rank=r, local_world=w) as s:
                s.reset(0)
                s.apply(circ)
                st = s.state()
                s.norm()
                return st
        res = w.run(body)
    err = float(np.max(np.abs(res[0] - O.apply_circuit(circ, n))))
    assert err <= 1e-10, err
    print("local world x2", err)
    print("SANITIZE_CASE_OK")


if __name__ == "__main__":
    main()
