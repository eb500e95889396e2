#!/bin/bash
# Plain bench run, then one ncu --set full capture of the section kernel (1 GPU).
set -e
CMD="python bench.py --workload qv28 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
ncu --set full --clock-control none --import-source on -k regex:k_section -s 20 -c 2 -o gpurun_out/prof_section $CMD > gpurun_out/prof_ncu.log 2>&1
