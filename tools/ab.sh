set -x
bash tools/sweep_ncu.sh
bash tools/prof.sh qft30b 13 3 -- --workload qft30
timeout 900 python bench.py --workload qft30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sub --unblocked > gpurun_out/sweep_qft30_unblocked2.json 2>/dev/null; echo unb=$?
