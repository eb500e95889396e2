#!/bin/bash
# BASELINE configs[1] chunk_bits sweep (QV28, c = 8..14) and the blocked-vs-unblocked comparison
# on one B200: one bench line per point, then one ncu --set full capture of a
# section kernel per c.  Outputs under gpurun_out/sweep_*.
mkdir -p gpurun_out
for c in 8 9 10 11 12 13 14; do
  timeout 900 python bench.py --workload qv28 --chunk-bits $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sub \
    > gpurun_out/sweep_qv28_c$c.json 2> gpurun_out/sweep_qv28_c$c.err; echo qv28 c=$c rc=$?
done
timeout 900 python bench.py --workload qv28 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sub --unblocked \
  > gpurun_out/sweep_qv28_unblocked.json 2> gpurun_out/sweep_qv28_unblocked.err; echo qv28 unblocked rc=$?
for c in 8 10 12; do
  timeout 900 python bench.py --workload qft30 --chunk-bits $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sub \
    > gpurun_out/sweep_qft30_c$c.json 2> gpurun_out/sweep_qft30_c$c.err; echo qft30 c=$c rc=$?
done
timeout 900 python bench.py --workload qft30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sub --unblocked \
  > gpurun_out/sweep_qft30_unblocked.json 2> gpurun_out/sweep_qft30_unblocked.err; echo qft30 unblocked rc=$?
