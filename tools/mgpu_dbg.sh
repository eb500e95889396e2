R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for F in 1 0; do
SV_FUSE=$F SV_DEBUG_TIMING=1 timeout 900 $R --master-port 2961$F bench.py --gpus 2 --steps 1 --warmup 3 --workload qv33 --no-e2e > gpurun_out/dbg_f$F.json 2> gpurun_out/dbg_f$F.err
done
