# 2-GPU exchange A/B (QFT34 weak) + 1-GPU QFT30 / QV28 with the straight-line DIAGSET prologue
set -x
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload qft30 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/r02_ab3_qft30.json 2>/dev/null; echo qft30=$?
N=2
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
P=29700
for v in "" "SV_XPIPE=0" "SV_XGRID=264" "SV_XSLOT_MB=4096" "SV_XGRID=528 SV_XPIPE=0" "SV_XGRID=66"; do
  P=$((P+1)); tag=$(echo "d $v" | tr ' =' '__')
  env $v timeout 900 $R --master-port $P bench.py --gpus $N --steps 3 --warmup 3 --no-sub --no-e2e --workload qft_weak > gpurun_out/r02_ab3_qftweak_$tag.json 2>/dev/null; echo "$v rc=$?"
done
