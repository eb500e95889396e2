#!/bin/bash
# Peak micro-benchmarks on one B200 with nvidia-smi clocks sampled during the run.
# usage (under gpurun): bash tools/peaks.sh [tag]
T=${1:-peaks}
bash tools/hostinfo.sh > gpurun_out/${T}_host.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap \
  --format=csv -lms 100 > gpurun_out/${T}_clocks.csv &
SMI=$!
./tools/microbench > gpurun_out/${T}.jsonl 2>&1; echo microbench=$?
kill $SMI
