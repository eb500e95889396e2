timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "prob or marg or qft10 or mid" > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 600 python bench.py --workload qft30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_qft30.json 2> gpurun_out/c_qft30.err
./tools/prof.sh qv28 66 2
