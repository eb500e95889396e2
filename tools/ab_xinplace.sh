#!/bin/bash
# In-place exchange form A/B on N GPUs (under gpurun --gpus N): default (copy engines at both ends,
# every rank unpacks) vs SV_XINPLACE=1; QFT weak and QV33, pipelined and alone.  On 2 GPUs the
# local-world parity and a randomised sweep run first.  Outputs gpurun_out/r02_abi_*_n$N.json
N=${1:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
B="bench.py --gpus $N --warmup 3 --no-sub --no-e2e"
if [ "$N" = 2 ]; then
timeout 900 python -m pytest tests/test_local_world.py -q -x -k "inplace or parity" > gpurun_out/r02_abi_localworld.log 2>&1; echo lw=$?
timeout 900 python tools/stress_local.py 11 80 > gpurun_out/r02_abi_stress.log 2>&1; echo stress=$?
fi
SV_XINPLACE=1 timeout 900 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/r02_abi_mgpu_tests_n$N.log 2>&1; echo mt=$?
port=29900
for r in 1 2; do
for v in 0 1; do
  for wl in qft_weak qv33; do
    port=$((port+1))
    SV_XINPLACE=$v timeout 900 $R --master-port $port $B --steps 5 --workload $wl > gpurun_out/r02_abi_${wl}_i${v}_r${r}_n$N.json 2> gpurun_out/r02_abi_${wl}_i${v}_r${r}_n$N.err; echo $wl-i$v-r$r=$?
  done
done
done
