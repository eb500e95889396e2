# multi-GPU: parity tests, strong-scaling bench (QV33), weak QFT, and the unblocked comparator
N=${1:-2}
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/mgpu_tests_$N.log 2>&1; echo mtests=$?
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 $R --master-port 29533 bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo bench=$?
timeout 1500 $R --master-port 29534 bench.py --gpus $N --steps 3 --warmup 3 --workload qft_weak --no-e2e > gpurun_out/bench_qftweak_n$N.json 2> gpurun_out/bench_qftweak_n$N.err; echo benchw=$?


