for TS in 384 512; do
  SV_JIT_CACHE=0 SV_JIT_THREADS_SM=$TS timeout 600 python bench.py --workload qv28 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ts_qv28_$TS.json 2> gpurun_out/ts_qv28_$TS.err
  SV_JIT_CACHE=0 SV_JIT_THREADS_SM=$TS timeout 600 python bench.py --workload qft30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ts_qft30_$TS.json 2> gpurun_out/ts_qft30_$TS.err
done
