timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 600 python bench.py --workload qv28 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_qv28.json 2> gpurun_out/c_qv28.err
timeout 900 python bench.py --workload qv33 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_qv33.json 2> gpurun_out/c_qv33.err
