timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests=$?
for W in qft30 qv28; do
timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c_$W.json 2> gpurun_out/c_$W.err
done
timeout 900 python bench.py --workload qv33 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c_qv33.json 2> gpurun_out/c_qv33.err
