#!/bin/bash
# Last check of the round on one B200: the GPU suite, smoke(), the default bench line.
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_last_gpu_suite.txt 2>&1; echo suite=$?
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_last_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_last_bench.json 2> gpurun_out/r02_last_bench.err; echo bench=$?
