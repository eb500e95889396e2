# 2-GPU exchange transports: copy engine (default) vs push kernel, pipelined and alone
set -x
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_local_world.py -q -x > gpurun_out/r02_ab4_localworld.log 2>&1; echo lw=$?
N=2
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/r02_ab4_mgpu_tests.log 2>&1; echo mt=$?
P=29800
for w in qft_weak qv33; do
for v in "" "SV_XPIPE=0" "SV_XCE=0" "SV_XCE=0 SV_XPIPE=0"; do
  P=$((P+1)); tag=$(echo "$w $v" | tr ' =' '__')
  env $v timeout 900 $R --master-port $P bench.py --gpus $N --steps 3 --warmup 3 --no-sub --no-e2e --workload $w > gpurun_out/r02_ab4_$tag.json 2>/dev/null; echo "$w $v rc=$?"
done; done
