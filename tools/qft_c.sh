#!/bin/bash
# QFT chunk_bits on one B200: QFT30 (configs[2]) and QFT33 (the weak line's N = 1 point) at c = 8..12,
# then one ncu --set full capture of the QFT30 c=10 read + write sections.  gpurun_out/qftc_*
B="python bench.py --gpus 1 --warmup 3 --no-sub --no-cpu-baseline --no-e2e"
for c in 8 9 10 11 12; do
  timeout 600 $B --steps 10 --workload qft30 --chunk-bits $c > gpurun_out/qftc_qft30_c$c.json 2>/dev/null; echo qft30 c=$c rc=$?
done
for c in 8 9 10 11; do
  timeout 600 $B --steps 4 --workload qft_weak --chunk-bits $c > gpurun_out/qftc_qft33_c$c.json 2>/dev/null; echo qft33 c=$c rc=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sv_sec -s 1 -c 2 -o gpurun_out/qftc_ncu_c10 \
  $B --steps 1 --workload qft30 --chunk-bits 10 > gpurun_out/qftc_ncu_c10.log 2>&1; echo ncu=$?
