#!/bin/bash
# End-of-round evidence on one B200: the GPU suite, smoke(), the default bench line, the reference
# arm, the ncu launch list of one bench step, ncu --set full of one QV33 section and the QFT30
# read + write sections.  Outputs gpurun_out/r02_final_* and gpurun_out/prof_*.
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_final_gpu_suite.txt 2>&1; echo suite=$?
bash tools/round_bench.sh
bash tools/prof.sh qv33fin 90 1 -- --workload qv33
bash tools/prof.sh qft30fin 1 3 -- --workload qft30
