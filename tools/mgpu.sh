#!/bin/bash
# multi-GPU on one box (under gpurun --gpus N): parity tests over NCCL + CUDA IPC, then bench lines —
# QV33 strong (copy-engine exchange pipelined with the sections / alone / the NCCL send/recv
# comparator), QFT weak, QV28 strong blocked vs unblocked (NEXT-3).  NVLink data counters
# (nvidia-smi) around the QV33 run.  Outputs gpurun_out/r02_mgpu_*_n$N.*
N=${1:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/r02_mgpu_tests_n$N.log 2>&1; echo mtests=$?
nvidia-smi nvlink -gt d > gpurun_out/r02_mgpu_nvlink_before_n$N.txt 2>&1
timeout 900 $R --master-port 29601 bench.py --gpus $N --steps 5 --warmup 3 --no-sub > gpurun_out/r02_mgpu_qv33_n$N.json 2> gpurun_out/r02_mgpu_qv33_n$N.err; echo qv33=$?
nvidia-smi nvlink -gt d > gpurun_out/r02_mgpu_nvlink_after_n$N.txt 2>&1
SV_XPIPE=0 timeout 900 $R --master-port 29602 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e > gpurun_out/r02_mgpu_qv33raw_n$N.json 2> gpurun_out/r02_mgpu_qv33raw_n$N.err; echo qv33raw=$?
timeout 900 $R --master-port 29603 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e --nccl > gpurun_out/r02_mgpu_qv33nccl_n$N.json 2> gpurun_out/r02_mgpu_qv33nccl_n$N.err; echo qv33nccl=$?
timeout 900 $R --master-port 29604 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e --workload qft_weak > gpurun_out/r02_mgpu_qftweak_n$N.json 2> gpurun_out/r02_mgpu_qftweak_n$N.err; echo qftweak=$?
SV_XPIPE=0 timeout 900 $R --master-port 29605 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e --workload qft_weak > gpurun_out/r02_mgpu_qftweakraw_n$N.json 2> gpurun_out/r02_mgpu_qftweakraw_n$N.err; echo qftweakraw=$?
timeout 900 $R --master-port 29606 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e --workload qv28 > gpurun_out/r02_mgpu_qv28_n$N.json 2> gpurun_out/r02_mgpu_qv28_n$N.err; echo qv28=$?
timeout 900 $R --master-port 29607 bench.py --gpus $N --steps 3 --warmup 3 --no-sub --no-e2e --workload qv28 --unblocked > gpurun_out/r02_mgpu_qv28unb_n$N.json 2> gpurun_out/r02_mgpu_qv28unb_n$N.err; echo qv28unb=$?
# peer-transfer ceilings (copy-engine peer copy, NCCL send/recv) on the same box
timeout 600 python tools/p2p_bench.py ce $N > gpurun_out/r02_p2p_ce_n$N.jsonl 2> gpurun_out/r02_p2p_ce_n$N.err; echo p2pce=$?
timeout 600 $R --master-port 29608 tools/p2p_bench.py nccl > gpurun_out/r02_p2p_nccl_n$N.jsonl 2> gpurun_out/r02_p2p_nccl_n$N.err; echo p2pnccl=$?
