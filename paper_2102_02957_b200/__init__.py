"""B200-native cache-blocked state-vector simulator (arXiv 2102.02957 hot path).

The compute lives in libsv.so (include/sv.h): a host C++ cache-blocking pass and planner,
sm_100a section kernels, peer-memory / NCCL chunk exchange and reductions.  This package is a
thin binding; see DESIGN.md.
"""
from ._lib import (GATE_DTYPE, SV_BEGIN, SV_CHUNK_SWAP, SV_D1, SV_D2, SV_END, SV_EXCHANGE, SV_EXCHANGE_NCCL, SV_FREE_LAYOUT, SV_ABSORB_SWAPS,  # noqa: F401
                   SV_FP32, SV_FP64, SV_RESTORE_ORDER, SV_SWAP, SV_U1, SV_U2, SV_UNBLOCKED, HostStateVector, LocalWorld, StateVector, SvError,
                   block_circuit, compile_circuit, jit_compile_circuit, jit_mode, jit_wait, JIT_OFF, JIT_SYNC, JIT_ASYNC, lib, nccl_unique_id, plan_circuit)
from .dist import create_distributed  # noqa: F401
