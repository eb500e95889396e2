R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
SV_XPIPE=0 timeout 600 $R --master-port 29811 tools/xbench.py > gpurun_out/xb_nopipe.log 2>&1
SV_XPIPE=4 timeout 600 $R --master-port 29812 tools/xbench.py > gpurun_out/xb_pipe.log 2>&1
