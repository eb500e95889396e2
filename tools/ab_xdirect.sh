#!/bin/bash
# A/B of the exchange's copy-engine forms on N GPUs (under gpurun --gpus N): pack kernel + copy +
# unpack kernel (SV_XRUN=0 SV_XCEU=0), copy-engine gather straight from the state (SV_XCEU=0), and
# copy-engine gather + unpack (the default); QFT weak and QV33 strong, pipelined and alone.  Outputs gpurun_out/r02_abx_*_n$N.json
N=${1:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
B="bench.py --gpus $N --warmup 3 --no-sub --no-e2e"
timeout 900 python -m pytest tests/test_local_world.py -q -x -k "copy_engine or parity" > gpurun_out/r02_abx_localworld.log 2>&1; echo lw=$?
timeout 900 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/r02_abx_mgpu_tests_n$N.log 2>&1; echo mt=$?
port=29700
for cfg in "pack:SV_XRUN=0 SV_XCEU=0" "direct:SV_XRUN=1024 SV_XCEU=0" "directu:SV_XRUN=1024 SV_XCEU=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  for wl in qft_weak qv33; do
    port=$((port+1))
    env $envs timeout 900 $R --master-port $port $B --steps 5 --workload $wl > gpurun_out/r02_abx_${wl}_${name}_n$N.json 2> gpurun_out/r02_abx_${wl}_${name}_n$N.err; echo $wl-$name=$?
    port=$((port+1))
    env $envs SV_XPIPE=0 timeout 900 $R --master-port $port $B --steps 5 --workload $wl > gpurun_out/r02_abx_${wl}_${name}raw_n$N.json 2> gpurun_out/r02_abx_${wl}_${name}raw_n$N.err; echo $wl-${name}raw=$?
  done
done
