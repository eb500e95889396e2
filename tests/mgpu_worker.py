"""torchrun worker for tests/test_multi_gpu.py: one rank per GPU, NCCL process group.

Every rank runs the cases of tests/mgpu_cases.py through sv_create_dist / sv_apply_circuit; rank 0
gathers the logical state (sv_get_state) and judges it against the oracle and against a
single-GPU run of the same circuit on its own device.  Exit code 0 = all checks passed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist

    import mgpu_cases as M
    import paper_2102_02957_b200 as sv

    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    failures = []
    for case in M.cases():
        name, recs, n, c, flags, basis, prec, second = case
        s = sv.create_distributed(n, c, prec)
        res = M.run_rank(s, case)
        s.close()
        if rank == 0:
            checks, err, d1 = M.check(case, res, M.reference(case), M.single_gpu(sv, case), world)
            st = res["stats"]
            print(f"[mgpu] {name}: err={err:.2e} vs-1gpu={d1:.1e} exchanges={st['exchanges']} "
                  f"bytes={st['bytes_sent']} {checks}", flush=True)
            failures += [f"{name}:{k}" for k, ok in checks.items() if not ok]
    dist.barrier()
    dist.destroy_process_group()
    if failures:
        print("[mgpu] FAILURES:", failures, flush=True)
        sys.exit(1)


if __name__ == "__main__":
    main()
