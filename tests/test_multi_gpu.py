"""Multi-GPU parity through the C ABI: torchrun with one rank per GPU (NCCL + CUDA IPC peer memory).
Skipped unless at least 2 GPUs are visible (run under `gpurun --gpus 2` or `--gpus 4`)."""
import os
import subprocess
import sys

import pytest

from conftest import gpu_available

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    if not gpu_available():
        return 0
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_parity(world):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world), os.path.join(ROOT, "tests", "mgpu_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(res.stdout[-4000:])
    print(res.stderr[-4000:])
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
