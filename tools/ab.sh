# 2 GPUs: local-world + NCCL parity, then the exchange pipelined with both neighbouring sections
set -x
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_local_world.py -q -x > gpurun_out/r02_ab5_localworld.log 2>&1; echo lw=$?
timeout 900 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/r02_ab5_mgpu_tests.log 2>&1; echo mt=$?
N=2
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
P=29900
for w in qft_weak qv33; do
for v in "" "SV_XPIPE=0"; do
  P=$((P+1)); tag=$(echo "$w $v" | tr ' =' '__')
  env $v timeout 900 $R --master-port $P bench.py --gpus $N --steps 3 --warmup 3 --no-sub --no-e2e --workload $w > gpurun_out/r02_ab5_$tag.json 2>/dev/null; echo "$w $v rc=$?"
done; done
python - <<'PY' > gpurun_out/r02_nvml_probe.txt 2>&1
import pynvml as N
N.nvmlInit(); h = N.nvmlDeviceGetHandleByIndex(0)
for fid, name in [(N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, "XMIT_BYTES"), (N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, "RCV_BYTES"), (N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, "THRU_DATA_TX")]:
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = N.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(name, scope, "ret", v.nvmlReturn, "type", v.valueType, "val", v.value.ullVal)
        except Exception as e:
            print(name, scope, "exc", e)
PY
echo probe=$?
