#!/bin/bash
# QFT weak lines at the workload's chunk_bits on N GPUs (under gpurun --gpus N), pipelined and with
# the exchange alone; on one GPU also the fp32 variant at c = 8 and 9.  gpurun_out/qfw_*_n$N.json
N=${1:-1}
if [ "$N" = 1 ]; then
  B="python bench.py --gpus 1 --warmup 3 --no-sub --no-cpu-baseline --no-e2e"
  timeout 600 $B --steps 5 --workload qft_weak > gpurun_out/qfw_qftweak_n1.json 2>/dev/null; echo w=$?
  for c in 8 9; do timeout 600 $B --steps 5 --workload qft_weak_fp32 --chunk-bits $c > gpurun_out/qfw_fp32_c${c}_n1.json 2>/dev/null; echo f$c=$?; done
else
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  timeout 900 $R --master-port 29951 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e --workload qft_weak > gpurun_out/qfw_qftweak_n$N.json 2> gpurun_out/qfw_qftweak_n$N.err; echo w=$?
  SV_XPIPE=0 timeout 900 $R --master-port 29952 bench.py --gpus $N --steps 5 --warmup 3 --no-sub --no-e2e --workload qft_weak > gpurun_out/qfw_qftweakraw_n$N.json 2> gpurun_out/qfw_qftweakraw_n$N.err; echo wr=$?
fi
