# 1 GPU: the GPU suite under the bounds-checking build (SV_CHECK=1), then dense-section occupancy A/B and fp32 lines
set -x
SV_CHECK=1 SV_JIT_CACHE=0 timeout 1700 python -m pytest tests -m gpu -q -x > gpurun_out/r02_gpu_checked.log 2>&1; echo checked=$?
for t in 384 512; do
  SV_DENSE_TSM=$t timeout 600 python bench.py --workload qv28 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/r02_ab6_qv28_t$t.json 2>/dev/null; echo qv28 t$t=$?
  SV_DENSE_TSM=$t timeout 900 python bench.py --workload qv33 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/r02_ab6_qv33_t$t.json 2>/dev/null; echo qv33 t$t=$?
done
timeout 900 python bench.py --workload qft_weak_fp32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/r02_ab6_qft34_fp32.json 2>/dev/null; echo qft34fp32=$?
timeout 900 python bench.py --workload qv28 --precision fp32 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/r02_ab6_qv28_fp32.json 2>/dev/null; echo qv28fp32=$?
