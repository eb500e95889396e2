N=${1:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/mgpu_tests_$N.log 2>&1; echo mtests=$?
timeout 900 $R --master-port 29601 bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo b=$?
timeout 900 $R --master-port 29602 bench.py --gpus $N --steps 3 --warmup 3 --workload qft_weak --no-e2e > gpurun_out/bench_qftweak_n$N.json 2> gpurun_out/bench_qftweak_n$N.err; echo bw=$?
timeout 900 $R --master-port 29603 bench.py --gpus $N --steps 3 --warmup 3 --workload qv28 --no-e2e > gpurun_out/bench_qv28_n$N.json 2> gpurun_out/bench_qv28_n$N.err; echo b28=$?
