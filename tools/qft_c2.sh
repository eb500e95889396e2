#!/bin/bash
# QFT chunk_bits with direct HBM phases on 64-byte runs (tiles holding memory bits 0..1 only):
# GPU parity first, then QFT30 c = 8..11, QFT33 c = 9..11, one ncu capture of the QFT33 c=11 sections.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -q -x > gpurun_out/qftc2_parity.log 2>&1; echo parity=$?
B="python bench.py --gpus 1 --warmup 3 --no-sub --no-cpu-baseline --no-e2e"
for c in 8 9 10 11; do
  timeout 600 $B --steps 10 --workload qft30 --chunk-bits $c > gpurun_out/qftc2_qft30_c$c.json 2>/dev/null; echo qft30 c=$c rc=$?
done
for c in 9 10 11; do
  timeout 600 $B --steps 4 --workload qft_weak --chunk-bits $c > gpurun_out/qftc2_qft33_c$c.json 2>/dev/null; echo qft33 c=$c rc=$?
done
timeout 900 ncu --set full --clock-control none -k regex:sv_sec -s 1 -c 2 -o gpurun_out/qftc2_ncu_qft30_c10 \
  $B --steps 1 --workload qft30 --chunk-bits 10 > gpurun_out/qftc2_ncu.log 2>&1; echo ncu=$?
