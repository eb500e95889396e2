"""Peer-transfer ceilings the exchange is measured against (SURVEY §8(d) measurement protocol, item 4).

Two parts, both timed with CUDA events on the streams that carry the transfer:
  python tools/p2p_bench.py ce N      one process, N GPUs: copy-engine peer copies (tensor.copy_
                                      between devices = cudaMemcpyPeerAsync), pairs (0,1), (2,3)..
                                      in both directions at once, 64 MiB .. 4 GiB
  torchrun --nproc-per-node N tools/p2p_bench.py nccl
                                      NCCL send/recv between rank pairs (r, r ^ 1), both directions
                                      at once (batch_isend_irecv), 64 MiB .. 4 GiB
Prints one JSON line per size: GB/s per direction (bytes one GPU sends / time)."""
import json
import os
import sys

import torch

SIZES = [64 << 20, 256 << 20, 1 << 30, 4 << 30]


def ce(n):
    pairs = [(a, a + 1) for a in range(0, n - 1, 2)]
    for s in SIZES:
        bufs, streams = {}, {}
        for a, b in pairs:
            for x, y in ((a, b), (b, a)):
                bufs[(x, y)] = (torch.empty(s, dtype=torch.uint8, device=f"cuda:{x}"),
                                torch.empty(s, dtype=torch.uint8, device=f"cuda:{y}"))
                streams[(x, y)] = torch.cuda.Stream(device=f"cuda:{x}")
        reps = 10 if s <= (1 << 30) else 4
        for warm in (True, False):
            ev = {}
            for k, (src, dst) in bufs.items():
                with torch.cuda.device(k[0]), torch.cuda.stream(streams[k]):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(1 if warm else reps):
                        dst.copy_(src, non_blocking=True)
                    e1.record()
                    ev[k] = (e0, e1)
            for d in range(n):
                torch.cuda.synchronize(d)
        ms = max(e0.elapsed_time(e1) for e0, e1 in ev.values())
        print(json.dumps({"kind": "ce_peer_copy", "gpus": n, "pairs": pairs, "bytes": s,
                          "gbs_per_direction": round(reps * s / ms / 1e6, 1), "ms": round(ms / reps, 3)}), flush=True)
        del bufs


def nccl():
    import torch.distributed as dist
    dist.init_process_group("nccl")
    r, w = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", r)))
    peer = r ^ 1
    for s in SIZES:
        a = torch.empty(s, dtype=torch.uint8, device="cuda")
        b = torch.empty(s, dtype=torch.uint8, device="cuda")
        reps = 10 if s <= (1 << 30) else 4

        def once():
            ops = [dist.P2POp(dist.isend, a, peer), dist.P2POp(dist.irecv, b, peer)]
            for q in dist.batch_isend_irecv(ops):
                q.wait()

        once()
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            once()
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        if r == 0:
            t = float(ms.item())
            print(json.dumps({"kind": "nccl_send_recv", "gpus": w, "bytes": s,
                              "gbs_per_direction": round(reps * s / t / 1e6, 1), "ms": round(t / reps, 3)}), flush=True)
        del a, b
    dist.destroy_process_group()


if __name__ == "__main__":
    if sys.argv[1] == "ce":
        ce(int(sys.argv[2]) if len(sys.argv) > 2 else torch.cuda.device_count())
    else:
        nccl()
