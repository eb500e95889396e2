# 4 GPUs: the whole GPU suite (multi-GPU parity at 2 and 4 ranks included), then the pipelined
# QV33 / QFT35 lines with the exchange span timed from its first piece
set -x
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r02_final_gpu_suite_4gpu.log 2>&1; echo suite=$? secs=$(( $(date +%s) - T0 ))
N=4
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $R --master-port 29951 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r02_final_qv33_n4.json 2> gpurun_out/r02_final_qv33_n4.err; echo qv33=$?
timeout 900 $R --master-port 29952 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e --workload qft_weak > gpurun_out/r02_final_qftweak_n4.json 2> gpurun_out/r02_final_qftweak_n4.err; echo qftweak=$?
