# randomised parity sweeps on one GPU (logs for profiles/)
set -x
timeout 1200 python tools/stress.py 7 300 > gpurun_out/r02_stress.log 2>&1; echo stress=$?
timeout 1500 python tools/stress_local.py 8 150 > gpurun_out/r02_stress_local.log 2>&1; echo local=$?
SV_XCE=0 timeout 900 python tools/stress_local.py 9 60 > gpurun_out/r02_stress_local_push.log 2>&1; echo push=$?
SV_TMA=2 timeout 900 python tools/stress.py 10 100 > gpurun_out/r02_stress_tma.log 2>&1; echo tma=$?
