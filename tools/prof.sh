#!/bin/bash
# usage: tools/prof.sh <workload> <launch-skip> <launch-count> [kernel-regex] [extra bench args]
# Plain bench run, then one ncu --set full capture of the section kernel (1 GPU).
set -e
W=$1; S=$2; C=$3; K=${4:-"sv_sec|k_section"}; shift 3; shift || true
CMD="python bench.py --workload $W --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $@"
$CMD > gpurun_out/prof_${W}_plain.json 2> gpurun_out/prof_${W}_plain.err
ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $C -o gpurun_out/prof_${W} $CMD > gpurun_out/prof_${W}_ncu.log 2>&1
