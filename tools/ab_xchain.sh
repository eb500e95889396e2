#!/bin/bash
# Pipeline chain length A/B on N GPUs (under gpurun --gpus N): SV_XCHAIN = 1 (one launch on either
# side of an exchange, the earlier form), 4 (default), 16; QV33 strong and QFT weak.
# Outputs gpurun_out/r02_abc_*_n$N.json; first the local-world parity (incl. the chain tests).
N=${1:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
B="bench.py --gpus $N --warmup 3 --no-sub --no-e2e"
if [ "$N" = 2 ]; then
timeout 900 python -m pytest tests/test_local_world.py -q -x > gpurun_out/r02_abc_localworld.log 2>&1; echo lw=$?
timeout 600 python tools/stress_local.py 7 60 > gpurun_out/r02_abc_stress.log 2>&1; echo stress=$?
fi
timeout 900 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/r02_abc_mgpu_tests_n$N.log 2>&1; echo mt=$?
port=29800
for r in 1 2; do
for c in 1 4 16; do
  for wl in qv33 qft_weak; do
    port=$((port+1))
    SV_XCHAIN=$c timeout 900 $R --master-port $port $B --steps 5 --workload $wl > gpurun_out/r02_abc_${wl}_c${c}_r${r}_n$N.json 2> gpurun_out/r02_abc_${wl}_c${c}_r${r}_n$N.err; echo $wl-c$c-r$r=$?
  done
done
done
