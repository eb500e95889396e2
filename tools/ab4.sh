R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for cfg in "4 128" "4 256" "4 512" "0 0" "4 128"; do
  set -- $cfg
  SV_XPIPE=$1 SV_XGRID=$2 timeout 900 $R --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 3 --warmup 3 --no-e2e > gpurun_out/x4_$1_$2.json 2> gpurun_out/x4_$1_$2.err
  tail -1 gpurun_out/x4_$1_$2.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg', round(d['ms_per_step'],1), d['nvlink']['achieved'], d['roofline']['avg_launch_ms'])"
done
