# A/B: interpreter (SV_JIT=0) vs run-time specialised kernels (SV_JIT=sync), then GPU tests.
for W in qft30 qv28; do
  for J in 0 sync; do
    SV_JIT=$J timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${W}_jit$J.json 2> gpurun_out/ab_${W}_jit$J.err
  done
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests=$?
