"""Exchange micro-benchmark (torchrun, N GPUs): circuits that force one exchange batch of k rank
bits (a 1-qubit gate on the top global qubit: k = 1; a 2-qubit gate on the two top global qubits:
k = 2), timed with the library's per-launch events.  Prints per-direction GB/s per rank 0."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist
    import circuits as C
    import paper_2102_02957_b200 as sv
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n = int(os.environ.get("XB_N", "32"))
    s = sv.create_distributed(n, 8, "fp64")
    s.set_timing(True)
    cases = [("k1", C.records([C.gate(C.U1, n - 1, mat=C.H_MATRIX)]))]
    if world >= 4:
        cases.append(("k2", C.records([C.gate(C.U2, n - 1, n - 2, mat=C.haar_su(np.random.default_rng(1), 4))])))
    for name, circ in cases:
        for rep in range(4):
            s.reset(0)
            s.apply(C.records([]))  # consume the free initial layout: the gate's qubits stay global
            s.reset_stats()
            s.apply(circ, flags=int(os.environ.get("XB_FLAGS", "0")))
            st = s.stats()
            if rank == 0 and rep > 0:
                gbs = st["bytes_sent"] / (st["exchange_ms"] / 1e3) / 1e9 if st["exchange_ms"] else 0
                print(f"[xb] {name} world={world} bytes/rank={st['bytes_sent'] / 2**30:.1f} GiB "
                      f"exchange={st['exchange_ms']:.2f} ms -> {gbs:.0f} GB/s; sections {st['section_ms']:.2f} ms",
                      flush=True)
    s.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
