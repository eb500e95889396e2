#!/bin/bash
# The one-GPU lines of DESIGN §7-§8 with the current code: QFT weak (QFT33 fp64, QFT34 fp32),
# QV28 and QFT30 blocked vs the unblocked per-gate baseline.  Outputs gpurun_out/r02_1gpu_*.json
o=gpurun_out/r02_1gpu
B="python bench.py --gpus 1 --warmup 3 --no-sub --no-cpu-baseline --no-e2e"
timeout 900 $B --steps 5 --workload qft_weak > ${o}_qftweak.json 2> ${o}_qftweak.err; echo qftweak=$?
timeout 900 $B --steps 5 --workload qft_weak_fp32 > ${o}_qftweak32.json 2> ${o}_qftweak32.err; echo qftweak32=$?
timeout 900 $B --steps 10 --workload qv28 > ${o}_qv28.json 2> ${o}_qv28.err; echo qv28=$?
timeout 900 $B --steps 3 --workload qv28 --unblocked > ${o}_qv28unb.json 2> ${o}_qv28unb.err; echo qv28unb=$?
timeout 900 $B --steps 10 --workload qft30 > ${o}_qft30.json 2> ${o}_qft30.err; echo qft30=$?
timeout 900 $B --steps 3 --workload qft30 --unblocked > ${o}_qft30unb.json 2> ${o}_qft30unb.err; echo qft30unb=$?
