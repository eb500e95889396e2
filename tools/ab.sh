# 1 GPU: dense 2-qubit gate form A/B (Gauss three-multiply vs four-multiply)
set -x
for f in 4 3; do
  SV_U2_FORM=$f timeout 600 python bench.py --workload qv28 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/r02_ab7_qv28_f$f.json 2>/dev/null; echo qv28 f$f=$?
  SV_U2_FORM=$f timeout 900 python bench.py --workload qv33 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/r02_ab7_qv33_f$f.json 2>/dev/null; echo qv33 f$f=$?
done
SV_U2_FORM=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "random or qv_and_qft" > gpurun_out/r02_ab7_tests.log 2>&1; echo tests=$?
