# final one-GPU verification as the driver runs it: build, the GPU suite, smoke, the default bench line
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_last_build.log 2>&1; echo build=$?
T0=$(date +%s)
timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/r02_last_gpu_suite.log 2>&1; echo suite=$? secs=$(( $(date +%s) - T0 ))
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_last_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_last_bench.json 2> gpurun_out/r02_last_bench.err; echo bench=$?
