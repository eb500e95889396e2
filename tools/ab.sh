# 1-GPU A/B of SV_STREAM_HINTS (device 0), then the 2-GPU exchange lines
set -x
for m in 0 1; do
  SV_STREAM_HINTS=$m CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload qft30 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/r02_ab2_qft30_h$m.json 2>/dev/null; echo qft30 h$m=$?
  SV_STREAM_HINTS=$m CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload qv28 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/r02_ab2_qv28_h$m.json 2>/dev/null; echo qv28 h$m=$?
done
N=2
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $R --master-port 29601 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e > gpurun_out/r02_ab2_qv33_n2.json 2>/dev/null; echo qv33=$?
timeout 900 $R --master-port 29603 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e --workload qft_weak > gpurun_out/r02_ab2_qftweak_n2.json 2>/dev/null; echo qftweak=$?
timeout 900 $R --master-port 29602 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e --nccl > gpurun_out/r02_ab2_qv33nccl_n2.json 2>/dev/null; echo qv33nccl=$?
