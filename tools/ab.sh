for C in 8 9 10; do
  timeout 900 python bench.py --workload qv33 --chunk-bits $C --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s_qv33_$C.json 2> gpurun_out/s_qv33_$C.err
  timeout 600 python bench.py --workload qv28 --chunk-bits $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s_qv28_$C.json 2> gpurun_out/s_qv28_$C.err
done
for C in 7 8 9; do
  timeout 600 python bench.py --workload qft30 --chunk-bits $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s_qft30_$C.json 2> gpurun_out/s_qft30_$C.err
done
