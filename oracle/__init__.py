"""The oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It is the plain CPU definition of what the cache-blocked GPU path
computes:

  * sv_oracle.c  — dense complex128 simulator, one loop per gate in input order (C + OpenMP);
  * blocking.py  — an independent Python implementation of the paper's Listing 3 pass;
  * brute.py     — Kronecker-product brute force (n <= 8) that pins sv_oracle.c.

Nothing here is imported by paper_2102_02957_b200/, and nothing here imports it.
Parity status per function is listed in DESIGN.md ("Oracle pins"); every function is pinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile sv_oracle.c with gcc + OpenMP into oracle/liboracle.so (no CUDA involved)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fcx-limited-range", "-std=c11", "-shared", "-fPIC",
               "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            dp, ip, up = ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)
            L.or_pair_address.argtypes = [ctypes.c_uint64, ip, up, up]
            L.or_apply_circuit.argtypes = [dp, ip, ctypes.c_void_p, ctypes.c_int64]
            L.or_apply_circuit.restype = ctypes.c_int
            L.or_init_basis.argtypes = [dp, ip, ctypes.c_uint64]
            L.or_unpermute.argtypes = [dp, ip, ctypes.POINTER(ctypes.c_int32), dp]
            L.or_norm2.argtypes = [dp, ip]
            L.or_norm2.restype = ctypes.c_double
            L.or_marginal.argtypes = [dp, ip, ctypes.POINTER(ctypes.c_int32), ip, dp]
            L.or_sample_sorted.argtypes = [dp, ip, dp, ctypes.c_int64, up]
            _lib = L
        return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _nq(a: np.ndarray) -> int:
    n = int(a.size).bit_length() - 1
    assert a.size == 1 << n
    return n


def pair_address(i: int, k: int):
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    lib().or_pair_address(i, k, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def basis_state(n: int, k: int = 0) -> np.ndarray:
    a = np.empty(1 << n, dtype=np.complex128)
    lib().or_init_basis(_dp(a), n, k)
    return a


def apply_circuit(recs: np.ndarray, n: int, psi: np.ndarray = None, basis: int = 0, inplace: bool = False) -> np.ndarray:
    """Dense U_circuit |psi> (|basis> if psi is None).  recs: structured array of 272-byte records
    (circuits.GATE_DTYPE layout); BEGIN/END are ignored and CHUNK_SWAP acts as SWAP.  inplace=True
    updates a contiguous complex128 psi in place (for states too large to copy)."""
    if psi is None:
        a = basis_state(n, basis)
    elif inplace:
        assert psi.dtype == np.complex128 and psi.flags.c_contiguous
        a = psi
    else:
        a = np.array(psi, dtype=np.complex128, copy=True)
    assert a.size == 1 << n
    recs = np.ascontiguousarray(recs)
    rc = lib().or_apply_circuit(_dp(a), n, recs.ctypes.data_as(ctypes.c_void_p), len(recs))
    if rc != 0:
        raise ValueError("oracle: malformed gate record")
    return a


def unpermute(phys: np.ndarray, pi) -> np.ndarray:
    n = _nq(phys)
    pi = np.ascontiguousarray(pi, dtype=np.int32)
    out = np.empty_like(phys)
    lib().or_unpermute(_dp(np.ascontiguousarray(phys)), n, pi.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _dp(out))
    return out


def norm2(a: np.ndarray) -> float:
    return float(lib().or_norm2(_dp(np.ascontiguousarray(a)), _nq(a)))


def marginal(a: np.ndarray, qubits) -> np.ndarray:
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    p = np.empty(1 << len(q), dtype=np.float64)
    lib().or_marginal(_dp(np.ascontiguousarray(a)), _nq(a), q.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(q), _dp(p))
    return p


def sample(a: np.ndarray, us: np.ndarray) -> np.ndarray:
    """Inverse-CDF samples in logical index order for the given uniforms; out[s] answers us[s]."""
    us = np.asarray(us, dtype=np.float64)
    order = np.argsort(us, kind="stable")
    srt = np.ascontiguousarray(us[order])
    res = np.empty(len(us), dtype=np.uint64)
    lib().or_sample_sorted(_dp(np.ascontiguousarray(a)), _nq(a), _dp(srt), len(us),
                           res.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    out = np.empty_like(res)
    out[order] = res
    return out
