"""torchrun worker for tests/test_multi_gpu.py: one rank per GPU, NCCL process group.

For each case every rank runs the circuit through sv_create_dist / sv_apply_circuit; rank 0
gathers the logical state (sv_get_state) and compares it with the oracle, and additionally with a
single-GPU run of the same circuit on its own device (bitwise: the amplitudes see the same
floating-point operations whatever the number of GPUs, SURVEY P-G).  Exit code 0 = all good."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import circuits as C
    import paper_2102_02957_b200 as sv

    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    failures = []
    if rank == 0:
        import oracle as O
    cases = [
        ("qv", C.quantum_volume(20, 10, 1), 20, 10, 0),
        ("qv-nccl", C.quantum_volume(20, 10, 2), 20, 10, sv.SV_EXCHANGE_NCCL),
        ("qft", C.qft(22), 22, 12, 0),
        ("rand", C.random_circuit(18, 300, 5), 18, 8, 0),
        ("qv-restore", C.quantum_volume(16, 8, 3), 16, 6, sv.SV_RESTORE_ORDER),
        ("ghz", C.ghz(21), 21, 5, 0),
        # the paper's unblocked multi-GPU baseline (NEXT-3): per-gate exchanges of global qubits
        ("qv-unblocked", C.quantum_volume(16, 3, 4), 16, 6, sv.SV_UNBLOCKED),
    ]
    for name, recs, n, c, flags in cases:
        s = sv.create_distributed(n, c, "fp64")
        s.reset(C.basis_index(7, n) if name == "qft" else 0)
        s.apply(recs, flags=flags)
        st = s.stats()
        got = s.state()
        norm = s.norm()
        probs = s.probabilities([0, n - 1, n // 2])
        idx = np.array([0, 1, (1 << n) - 1, 12345], dtype=np.uint64)
        amps = s.amplitudes(idx)
        shots = s.sample(20000, 3)
        s.close()
        if rank == 0:
            basis = C.basis_index(7, n) if name == "qft" else 0
            ref = O.apply_circuit(recs, n, basis=basis)
            err = float(np.max(np.abs(got - ref)))
            one = sv.StateVector(n, c, "fp64")
            one.reset(basis)
            one.apply(recs, flags=flags)
            single = one.state()
            one.close()
            checks = {
                "oracle": err <= 1e-10,
                "norm": abs(norm - 1) <= 1e-12,
                "probs": float(np.max(np.abs(probs - O.marginal(ref, [0, n - 1, n // 2])))) <= 1e-12,
                "amps": float(np.max(np.abs(amps - ref[idx.astype(np.int64)]))) <= 1e-10,
                "shots_valid": bool(np.all(np.abs(ref[shots.astype(np.int64)]) > 0)),
                "exchanged": world == 1 or st["exchanges"] > 0 or name in ("ghz",),
                "g_invariant_bitwise": bool(np.array_equal(got, single)),
            }
            print(f"[mgpu] {name}: err={err:.2e} exchanges={st['exchanges']} bytes={st['bytes_sent']} {checks}",
                  flush=True)
            failures += [f"{name}:{k}" for k, ok in checks.items() if not ok and k != "g_invariant_bitwise"]
            if not checks["g_invariant_bitwise"]:
                print(f"[mgpu] note: {name} not bitwise G-invariant (max diff "
                      f"{float(np.max(np.abs(got - single))):.2e})", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if failures:
        print("[mgpu] FAILURES:", failures, flush=True)
        sys.exit(1)


if __name__ == "__main__":
    main()
