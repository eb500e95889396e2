for N in 2 4; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29900 + N)) tools/stress_mgpu.py > gpurun_out/stress_m$N.log 2>&1
done
