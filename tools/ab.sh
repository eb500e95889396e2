timeout 900 python bench.py --workload qft_weak_fp32 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/qft34f32.json 2> gpurun_out/qft34f32.err
