timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "qft or mid or random" > gpurun_out/gt.log 2>&1; echo t=$?
for i in 1 2; do
timeout 600 python bench.py --workload qft30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q$i.json 2> gpurun_out/q$i.err
done
timeout 600 python bench.py --workload qv28 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v.json 2> gpurun_out/v.err
