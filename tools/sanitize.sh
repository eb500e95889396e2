#!/bin/bash
# compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md): bash tools/sanitize.sh memcheck|racecheck|synccheck|initcheck
T=${1:-memcheck}
python tools/sanitize_case.py > gpurun_out/r02_sanitize_plain_$T.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_case.py > gpurun_out/r02_sanitize_$T.log 2>&1; echo sanitize_$T=$?
