#!/bin/bash
# QV33 chunk_bits on one B200 with the final kernels (5 timed steps each).  gpurun_out/qv33c_*.json
B="python bench.py --gpus 1 --warmup 3 --no-sub --no-cpu-baseline --no-e2e"
for c in 8 9 10 11 12; do
  timeout 600 $B --steps 5 --chunk-bits $c > gpurun_out/qv33c_c$c.json 2>/dev/null; echo c=$c rc=$?
done
