#!/bin/bash
# Record the GPU box's host resources (the oracle's CPU baseline runs there).
echo "nproc=$(nproc)"; free -g; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
