timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 600 python tools/stress.py 5 120 > gpurun_out/stress.log 2>&1; echo stress=$?
for W in qft30 qv28; do timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_$W.json 2> gpurun_out/f_$W.err; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_qv33.json 2> gpurun_out/f_qv33.err
