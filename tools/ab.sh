for C in 6 7; do
  SV_PREF_TILE=10 timeout 600 python bench.py --workload qft30 --chunk-bits $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/t10_qft30_$C.json 2> gpurun_out/t10_qft30_$C.err
done
SV_PREF_TILE=10 timeout 600 python bench.py --workload qv28 --chunk-bits 7 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/t10_qv28_7.json 2> gpurun_out/t10_qv28_7.err
timeout 600 python bench.py --workload qft30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/t11_qft30_8.json 2> gpurun_out/t11_qft30_8.err
