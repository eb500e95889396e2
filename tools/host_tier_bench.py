"""Host-memory tier timing: QV(n, 10, 1) fp64 with the state in host memory and 2^d-amplitude
chunks streamed through one GPU, against the same circuit resident in HBM."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import circuits as C  # noqa: E402
import paper_2102_02957_b200 as sv  # noqa: E402

n, d, c = int(sys.argv[1]), int(sys.argv[2]), 9
circ = C.quantum_volume(n, 10, 1)
with sv.HostStateVector(n, c, d) as h:
    for rep in range(2):
        h.reset(0)
        t = time.perf_counter()
        h.apply(circ)
        dt = time.perf_counter() - t
    print(f"host tier QV{n} d={d}: {dt:.3f} s ({(1 << n) * 16 / 2**30:.0f} GiB state, {1 << (n - d)} chunks)", flush=True)
with sv.StateVector(n, c) as s:
    for rep in range(2):
        s.reset(0)
        t = time.perf_counter()
        s.apply(circ)
        s.synchronize()
        dt = time.perf_counter() - t
    print(f"HBM-resident QV{n}: {dt:.3f} s", flush=True)
