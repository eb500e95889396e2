#!/bin/bash
# Round-end style run on one B200: smoke(), the default bench line as the driver runs it, the
# reference arm, the ncu launch list of one bench step, and one ncu --set full capture of sv_sec.
# Outputs gpurun_out/r02_final_*.
set -x
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_final_bench.json 2> gpurun_out/r02_final_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r02_final_ref.json 2> gpurun_out/r02_final_ref.err; echo ref=$?
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r02_final_ncu_plain.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_final_launches.csv $CMD > gpurun_out/r02_final_ncu_launch.log 2>&1; echo launches=$?
