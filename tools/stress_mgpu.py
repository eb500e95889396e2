"""Randomised multi-GPU parity sweep (torchrun): fuzz circuits on a distributed state, gathered on
rank 0 and compared with the oracle; exchange paths P2P and NCCL, free and fixed layouts."""
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])


def main():
    import torch
    import torch.distributed as dist
    import circuits as C
    import paper_2102_02957_b200 as sv
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    g = world.bit_length() - 1
    if rank == 0:
        import oracle as O
    rng = np.random.default_rng(7)
    count = int(os.environ.get("ST_COUNT", "60"))
    bad = 0
    for t in range(count):
        n = int(rng.integers(g + 5, 19))
        c = int(rng.integers(2, min(n - g, 12) + 1))
        flags = sv.SV_EXCHANGE_NCCL if rng.random() < 0.25 else 0
        circ = C.random_circuit(n, int(rng.integers(1, 200)), 20000 + t)
        k = int(rng.integers(0, 1 << n))
        s = sv.create_distributed(n, c, "fp64")
        s.reset(k)
        if rng.random() < 0.5:
            s.apply(C.records([]))  # fixed initial layout
        s.apply(circ, flags=flags)
        s.apply(circ[: len(circ) // 2], flags=flags)
        got = s.state()
        nrm = s.norm()
        s.close()
        if rank == 0:
            ref = O.apply_circuit(circ[: len(circ) // 2], n, O.apply_circuit(circ, n, basis=k))
            err = float(np.max(np.abs(got - ref)))
            if not (err <= 1e-10 and abs(nrm - 1) <= 1e-12):
                bad += 1
                print(f"FAIL t={t} n={n} c={c} flags={flags} err={err:.3g} norm={nrm}", flush=True)
    if rank == 0:
        print(f"stress-mgpu world={world}: {count} cases, {bad} failures", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
