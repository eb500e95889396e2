#!/bin/bash
# one ncu --set full capture of a QV28 section kernel per chunk_bits (after tools/sweep.sh ran the
# same commands without ncu); skip = the section launches of the warm-up steps
for c in 8 9 10 11 12 13 14; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sv_sec -s 40 -c 1 -o gpurun_out/sweep_ncu_qv28_c$c \
    python bench.py --workload qv28 --chunk-bits $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sub \
    > gpurun_out/sweep_ncu_qv28_c$c.log 2>&1; echo ncu c=$c rc=$?
done
