"""The N > 1 path on CPU: world_size 2, 4 and 8 over gloo.

Each process is one rank: it compiles its own section programs (sv_compile_circuit with its rank,
so rank bits fold into constants exactly as on the GPU), runs them on its shard with the kernel
emulator, and performs every EXCHANGE step with real inter-process communication (all_gather of
the subcube's shards over gloo, then the bit exchange).  Rank 0 gathers the final shards and
compares the logical state with the dense oracle.  This covers the planner's multi-rank logic
(sigma bookkeeping, exchange pairs, rank-bit folding) without GPUs; the GPU exchange kernel itself
is covered by tests/test_multi_gpu.py."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import circuits as C
    import oracle as O
    import paper_2102_02957_b200 as sv
    from emulator import run_section

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = world.bit_length() - 1
    try:
        for (kind, n, c, seed) in cases:
            recs = {"qv": lambda: C.quantum_volume(n, 6, seed), "qft": lambda: C.qft(n),
                    "rand": lambda: C.random_circuit(n, 60, seed)}[kind]()
            nL = n - g
            rng = np.random.default_rng(seed)
            psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
            psi /= np.linalg.norm(psi)
            shard = psi[rank << nL:(rank + 1) << nL].copy()  # sigma = pi = id: memory == logical
            steps, ints, coefs, aux, pi, sigma = sv.compile_circuit(recs, n, c, g, rank)
            i = 0
            while i < len(steps):
                st = steps[i]
                kind_ = int(st[0])
                if kind_ == 1:
                    off, cnt, coff, ccnt, T, n_out, flags, aoff, acnt = (int(x) for x in st[1:10])
                    run_section(shard, ints[off:off + cnt], coefs[coff:coff + ccnt], n_out, T, flags,
                                aux[aoff:aoff + acnt])
                    i += 1
                elif kind_ == 3:
                    m1, m2 = int(st[1]), int(st[2])
                    x = np.arange(shard.size, dtype=np.int64)
                    y = x ^ ((((x >> m1) ^ (x >> m2)) & 1) * ((1 << m1) | (1 << m2)))
                    shard[:] = shard[y]
                    i += 1
                elif kind_ == 0:  # one exchange batch: consecutive records with the same batch id
                    batch = int(st[3])
                    pairs = []
                    while i < len(steps) and int(steps[i][0]) == 0 and int(steps[i][3]) == batch:
                        pairs.append((int(steps[i][1]), int(steps[i][2]) - nL))
                        i += 1
                    allsh = [torch.zeros(shard.size * 2, dtype=torch.float64) for _ in range(world)]
                    dist.all_gather(allsh, torch.from_numpy(shard.view(np.float64).copy()))
                    allsh = [a.numpy().view(np.complex128) for a in allsh]
                    # new[rank][x] = old[rank with b-bits := x's m-bits][x with m-bits := rank's b-bits]
                    x = np.arange(shard.size, dtype=np.int64)
                    src_rank = np.full(shard.size, rank, dtype=np.int64)
                    src_x = x.copy()
                    for m, b in pairs:
                        xm = (x >> m) & 1
                        rb = (rank >> b) & 1
                        src_rank = (src_rank & ~(1 << b)) | (xm << b)
                        src_x = (src_x & ~(1 << m)) | (rb << m)
                    new = np.empty_like(shard)
                    for r in range(world):
                        sel = src_rank == r
                        new[sel] = allsh[r][src_x[sel]]
                    shard = new
                else:
                    raise AssertionError("per-gate steps are not used by blocked plans with nL >= 4")
            out = [torch.zeros(shard.size * 2, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(out, torch.from_numpy(shard.view(np.float64).copy()))
            if rank == 0:
                mem = np.concatenate([o.numpy().view(np.complex128) for o in out])
                got = O.unpermute(mem, [int(sigma[int(p)]) for p in pi])
                ref = O.apply_circuit(recs, n, psi)
                err = float(np.max(np.abs(got - ref)))
                q.put((kind, n, c, err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_distributed_plan_over_gloo(world):
    import torch.multiprocessing as mp
    from paper_2102_02957_b200 import build
    build.build()
    import oracle
    oracle.build()
    cases = [("qv", 10, 5, 1), ("qft", 10, 5, 0), ("rand", 9, 4, 7), ("qv", 12, 8, 2)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=5) for _ in cases]
    for kind, n, c, err in res:
        assert err <= 1e-12, (kind, n, c, err)
