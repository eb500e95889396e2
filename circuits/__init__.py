"""Shared seeded inputs (circuits, basis indices, sampling uniforms) — no method arithmetic here."""
from .gen import *  # noqa: F401,F403
from .gen import GATE_DTYPE, U1, U2, D1, D2, SWAP, CHUNK_SWAP, BEGIN, END  # noqa: F401
