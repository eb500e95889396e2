for P in 1 0; do
  SV_PIPE=$P timeout 600 python bench.py --workload qv28 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_qv28_$P.json 2> gpurun_out/p_qv28_$P.err
  SV_PIPE=$P timeout 600 python bench.py --workload qft30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_qft30_$P.json 2> gpurun_out/p_qft30_$P.err
done
