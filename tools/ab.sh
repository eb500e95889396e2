timeout 900 python bench.py --workload qft_weak --precision fp32 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f32_qft33.json 2> gpurun_out/f32_qft33.err
timeout 900 python bench.py --workload qft_weak --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f64_qft33.json 2> gpurun_out/f64_qft33.err
timeout 900 python bench.py --workload qv_weak --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f64_qv30.json 2> gpurun_out/f64_qv30.err
timeout 900 python bench.py --workload qv28 --precision fp32 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f32_qv28.json 2> gpurun_out/f32_qv28.err
