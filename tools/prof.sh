#!/bin/bash
# usage: tools/prof.sh <tag> <launch-skip> <launch-count> -- <bench args...>
# The plain bench command first (must exit 0), then one ncu --set full capture of section kernels
# (1 GPU).  Outputs gpurun_out/prof_<tag>.*
TAG=$1; S=$2; C=$3; shift 4
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sub $@"
$CMD > gpurun_out/prof_${TAG}_plain.json 2> gpurun_out/prof_${TAG}_plain.err && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sv_sec -s $S -c $C -o gpurun_out/prof_${TAG} $CMD \
  > gpurun_out/prof_${TAG}_ncu.log 2>&1; echo prof_${TAG}=$?
