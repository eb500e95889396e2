# A/B of the section-kernel variants (SV_TMA), one B200
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "qft10 or random or qv_and_qft or edge or generated" > gpurun_out/r02_ab_tests.log 2>&1; echo tests=$?
for m in 1 0 3; do SV_TMA=$m timeout 600 python bench.py --workload qft30 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_ab_qft30_tma$m.json 2>gpurun_out/r02_ab_qft30_tma$m.err; echo qft30 tma$m=$?; done
for m in 2 0; do SV_TMA=$m timeout 600 python bench.py --workload qv28 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_ab_qv28_tma$m.json 2>gpurun_out/r02_ab_qv28_tma$m.err; echo qv28 tma$m=$?; done
for m in 1 0; do SV_TMA=$m timeout 600 python bench.py --workload qft_weak --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_ab_qft33_tma$m.json 2>gpurun_out/r02_ab_qft33_tma$m.err; echo qft33 tma$m=$?; done
