"""ctypes binding of libsv.so (include/sv.h) — argument marshalling only.

Every step of the path runs inside the library (host C++ pass/planner, sm_100a kernels); this
module only converts numpy arrays to pointers and error codes to exceptions.  There is no
fallback: if libsv.so is missing, or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsv.so")

# sv_gate: int32 kind, q0, q1, pad; double m[32]  (272 bytes)
GATE_DTYPE = np.dtype([("kind", "<i4"), ("q0", "<i4"), ("q1", "<i4"), ("pad", "<i4"), ("m", "<f8", (32,))])
SV_U1, SV_U2, SV_D1, SV_D2, SV_SWAP, SV_CHUNK_SWAP, SV_BEGIN, SV_END, SV_EXCHANGE = range(1, 10)
SV_FP32, SV_FP64 = 0, 1
SV_UNBLOCKED, SV_RESTORE_ORDER, SV_EXCHANGE_NCCL, SV_FREE_LAYOUT, SV_ABSORB_SWAPS = 1, 2, 4, 8, 32
ERRORS = {-1: "SV_EINVAL", -2: "SV_ECAPACITY", -3: "SV_EINFEASIBLE", -4: "SV_EMALFORMED", -5: "SV_ECUDA", -6: "SV_ENCCL"}


class SvError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [("circuits", ctypes.c_uint64), ("gates", ctypes.c_uint64), ("sections", ctypes.c_uint64),
                ("chunk_swaps", ctypes.c_uint64), ("exchanges", ctypes.c_uint64),
                ("exchange_batches", ctypes.c_uint64), ("bytes_sent", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64), ("pass_ms", ctypes.c_double), ("apply_ms", ctypes.c_double),
                ("timed_sections", ctypes.c_uint64), ("section_ms", ctypes.c_double), ("exchange_ms", ctypes.c_double),
                ("gate_ms", ctypes.c_double), ("section_bytes", ctypes.c_double), ("section_flops", ctypes.c_double),
                ("compactions", ctypes.c_uint64), ("store_swaps", ctypes.c_uint64),
                ("jit_launches", ctypes.c_uint64), ("interp_launches", ctypes.c_uint64),
                ("jit_compiled", ctypes.c_uint64), ("jit_compile_ms", ctypes.c_double),
                ("timed_input_sections", ctypes.c_uint64), ("input_section_ms", ctypes.c_double),
                ("input_section_bytes", ctypes.c_double), ("input_section_flops", ctypes.c_double)]


EXPORTS = ["sv_create", "sv_create_dist", "sv_world_create", "sv_world_destroy", "sv_create_local", "sv_destroy", "sv_nccl_unique_id", "sv_reset", "sv_apply_circuit",
           "sv_synchronize", "sv_get_amplitudes", "sv_get_state", "sv_norm", "sv_probabilities", "sv_sample",
           "sv_get_permutation", "sv_stats", "sv_stats_get", "sv_stats_reset", "sv_set_timing", "sv_last_error", "sv_block_circuit", "sv_plan_circuit",
           "sv_compile_circuit", "sv_jit_compile_circuit", "sv_jit_mode", "sv_jit_wait", "sv_host_create", "sv_host_destroy", "sv_host_reset",
           "sv_host_apply_circuit", "sv_host_get_state", "sv_host_norm", "sv_host_probabilities",
           "sv_host_last_error", "sv_free",
           "sv_abi_version"]

_lib = None


def lib():
    """Load libsv.so (built by __graft_entry__.build() / paper_2102_02957_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    vp, i32, u32, u64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int32)
    hp = ctypes.POINTER(vp)
    sig = {
        "sv_create": ([i32, i32, i32, hp], i32),
        "sv_create_dist": ([i32, i32, i32, i32, i32, vp, vp, sz, vp, hp], i32),
        "sv_world_create": ([i32, hp], i32),
        "sv_world_destroy": ([vp], i32),
        "sv_create_local": ([i32, i32, i32, vp, i32, vp, hp], i32),
        "sv_destroy": ([vp], i32),
        "sv_nccl_unique_id": ([vp], i32),
        "sv_reset": ([vp, u64], i32),
        "sv_apply_circuit": ([vp, vp, sz, u32], i32),
        "sv_synchronize": ([vp], i32),
        "sv_get_amplitudes": ([vp, vp, sz, vp], i32),
        "sv_get_state": ([vp, vp], i32),
        "sv_norm": ([vp, dp], i32),
        "sv_probabilities": ([vp, ip, i32, dp], i32),
        "sv_sample": ([vp, sz, u64, vp], i32),
        "sv_get_permutation": ([vp, ip], i32),
        "sv_stats": ([vp, ctypes.POINTER(Stats)], i32),
        "sv_stats_get": ([vp, ctypes.POINTER(Stats)], i32),
        "sv_stats_reset": ([vp], i32),
        "sv_set_timing": ([vp, i32], i32),
        "sv_last_error": ([vp], ctypes.c_char_p),
        "sv_block_circuit": ([vp, sz, i32, i32, ip, u32, hp, ctypes.POINTER(sz), ip], i32),
        "sv_plan_circuit": ([vp, sz, i32, i32, i32, ip, ip, u32, hp, ctypes.POINTER(sz), ip, ip], i32),
        "sv_compile_circuit": ([vp, sz, i32, i32, i32, i32, i32, ip, ip, u32, hp, ctypes.POINTER(sz), hp, ctypes.POINTER(sz),
                                hp, ctypes.POINTER(sz), hp, ctypes.POINTER(sz), ip, ip], i32),
        "sv_jit_compile_circuit": ([vp, sz, i32, i32, i32, i32, i32, u32, ctypes.c_char_p, ip,
                                    ctypes.POINTER(ctypes.c_double)], i32),
        "sv_jit_mode": ([i32], i32),
        "sv_host_create": ([i32, i32, i32, i32, ctypes.POINTER(vp)], i32),
        "sv_host_destroy": ([vp], i32),
        "sv_host_reset": ([vp, ctypes.c_uint64], i32),
        "sv_host_apply_circuit": ([vp, vp, sz, u32], i32),
        "sv_host_get_state": ([vp, vp], i32),
        "sv_host_norm": ([vp, ctypes.POINTER(ctypes.c_double)], i32),
        "sv_host_probabilities": ([vp, ip, i32, ctypes.POINTER(ctypes.c_double)], i32),
        "sv_host_last_error": ([vp], ctypes.c_char_p),
        "sv_jit_wait": ([], i32),
        "sv_free": ([vp], None),
        "sv_abi_version": ([], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.sv_abi_version() != 3:
        raise RuntimeError("libsv.so ABI version mismatch")
    _lib = L
    return L


def check(rc: int, handle=None):
    if rc != 0:
        msg = lib().sv_last_error(handle)
        raise SvError(rc, msg.decode() if msg else "")


def as_gates(gates) -> np.ndarray:
    g = np.ascontiguousarray(gates)
    if g.dtype.itemsize != GATE_DTYPE.itemsize:
        raise TypeError("gate records must be 272-byte sv_gate records")
    return g.view(GATE_DTYPE)


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def block_circuit(gates, n: int, c: int, pi0=None, flags: int = 0):
    """Host-only cache-blocking pass (sv_block_circuit) -> (token records, pi_final)."""
    g = as_gates(gates)
    out = ctypes.c_void_p()
    nout = ctypes.c_size_t()
    pif = np.zeros(n, dtype=np.int32)
    p0 = None if pi0 is None else np.ascontiguousarray(pi0, dtype=np.int32)
    rc = lib().sv_block_circuit(g.ctypes.data if len(g) else None, len(g), n, c, None if p0 is None else _ip(p0), flags,
                                ctypes.byref(out), ctypes.byref(nout), _ip(pif))
    check(rc)
    try:
        toks = np.frombuffer(ctypes.string_at(out.value, nout.value * GATE_DTYPE.itemsize), dtype=GATE_DTYPE).copy()
    finally:
        lib().sv_free(out)
    return toks, pif


def plan_circuit(gates, n: int, c: int, world_log2: int, pi0=None, sigma0=None, flags: int = 0):
    """Host-only executor plan (sv_plan_circuit) -> (records, pi_final, sigma_final)."""
    g = as_gates(gates)
    out = ctypes.c_void_p()
    nout = ctypes.c_size_t()
    pif = np.zeros(n, dtype=np.int32)
    sgf = np.zeros(n, dtype=np.int32)
    p0 = None if pi0 is None else np.ascontiguousarray(pi0, dtype=np.int32)
    s0 = None if sigma0 is None else np.ascontiguousarray(sigma0, dtype=np.int32)
    rc = lib().sv_plan_circuit(g.ctypes.data if len(g) else None, len(g), n, c, world_log2,
                               None if p0 is None else _ip(p0), None if s0 is None else _ip(s0), flags,
                               ctypes.byref(out), ctypes.byref(nout), _ip(pif), _ip(sgf))
    check(rc)
    try:
        recs = np.frombuffer(ctypes.string_at(out.value, nout.value * GATE_DTYPE.itemsize), dtype=GATE_DTYPE).copy()
    finally:
        lib().sv_free(out)
    return recs, pif, sgf


def compile_circuit(gates, n: int, c: int, world_log2: int = 0, rank: int = 0, precision: str = "fp64",
                    flags: int = 0, pi0=None, sigma0=None):
    """Host-only: the section programs sv_apply_circuit would launch (sv_compile_circuit) ->
    (steps int64[k, 12], ints int32[], coefs complex128[], aux complex128[], pi_final, sigma_final)."""
    g = as_gates(gates)
    st, ni, co, ax = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    nst, nin, nco, nax = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    pif = np.zeros(n, dtype=np.int32)
    sgf = np.zeros(n, dtype=np.int32)
    prec = {"fp64": SV_FP64, "fp32": SV_FP32}[precision]
    p0 = None if pi0 is None else np.ascontiguousarray(pi0, dtype=np.int32)
    s0 = None if sigma0 is None else np.ascontiguousarray(sigma0, dtype=np.int32)
    rc = lib().sv_compile_circuit(g.ctypes.data if len(g) else None, len(g), n, c, world_log2, rank, prec,
                                  None if p0 is None else _ip(p0), None if s0 is None else _ip(s0), flags,
                                  ctypes.byref(st), ctypes.byref(nst), ctypes.byref(ni), ctypes.byref(nin),
                                  ctypes.byref(co), ctypes.byref(nco), ctypes.byref(ax), ctypes.byref(nax),
                                  _ip(pif), _ip(sgf))
    check(rc)
    try:
        steps = np.frombuffer(ctypes.string_at(st.value, nst.value * 96), dtype=np.int64).reshape(-1, 12).copy()
        ints = np.frombuffer(ctypes.string_at(ni.value, nin.value * 4), dtype=np.int32).copy()
        coefs = np.frombuffer(ctypes.string_at(co.value, nco.value * 16), dtype=np.complex128).copy()
        aux = np.frombuffer(ctypes.string_at(ax.value, nax.value * 16), dtype=np.complex128).copy()
    finally:
        for p in (st, ni, co, ax):
            lib().sv_free(p)
    return steps, ints, coefs, aux, pif, sgf


def jit_compile_circuit(gates, n: int, c: int, world_log2: int = 0, rank: int = 0, precision: str = "fp64",
                        flags: int = 0, dump_dir: str = None):
    """Host-only: NVRTC-compile the run-time specialised kernel of every section launch
    (sv_jit_compile_circuit) -> (kernels, compile_ms)."""
    g = as_gates(gates)
    nk = np.zeros(1, dtype=np.int32)
    ms = ctypes.c_double()
    prec = {"fp64": SV_FP64, "fp32": SV_FP32}[precision]
    rc = lib().sv_jit_compile_circuit(g.ctypes.data if len(g) else None, len(g), n, c, world_log2, rank, prec, flags,
                                      dump_dir.encode() if dump_dir else None, _ip(nk), ctypes.byref(ms))
    check(rc)
    return int(nk[0]), ms.value


JIT_OFF, JIT_SYNC, JIT_ASYNC = 0, 1, 2


def jit_mode(mode: int = -1) -> int:
    """Set (0 interpreter, 1 sync, 2 async) or query (-1) the process-wide section-kernel mode;
    returns the previous mode (sv_jit_mode)."""
    return int(lib().sv_jit_mode(mode))


def jit_wait() -> None:
    check(lib().sv_jit_wait())


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().sv_nccl_unique_id(buf))
    return buf.raw


class LocalWorld:
    """In-process virtual world of `world` ranks on the current device (sv_world_create): the
    multi-GPU path (exchange kernels, plans, collectives) with every shard on one GPU.  Each rank's
    StateVector(..., rank=r, local_world=w) must be driven by its own thread: run(fn) calls fn(rank)
    on `world` threads and returns the per-rank results (re-raising the first exception)."""

    def __init__(self, world: int):
        h = ctypes.c_void_p()
        check(lib().sv_world_create(world, ctypes.byref(h)))
        self._h = h
        self.world = world

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sv_world_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def run(self, fn):
        import threading
        out = [None] * self.world
        errs = [None] * self.world

        def body(r):
            try:
                out[r] = fn(r)
            except BaseException as e:  # noqa: BLE001 - re-raised in the caller
                errs[r] = e

        th = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for e in errs:
            if e is not None:
                raise e
        return out


class StateVector:
    """One rank's handle on a chunk-sharded n-qubit state (sv_create / sv_create_dist /
    sv_create_local)."""

    def __init__(self, n_qubits: int, chunk_bits: int, precision: str = "fp64", *, rank: int = 0, world: int = 1,
                 nccl_id: bytes = None, stream: int = None, buffer_ptr: int = None, buffer_bytes: int = 0,
                 local_world: "LocalWorld" = None):
        self.n, self.c = n_qubits, chunk_bits
        self.precision = precision
        self.rank, self.world = rank, world
        prec = {"fp64": SV_FP64, "fp32": SV_FP32}[precision]
        self.cdtype = np.complex128 if prec == SV_FP64 else np.complex64
        h = ctypes.c_void_p()
        if local_world is not None:
            self.world = local_world.world
            rc = lib().sv_create_local(n_qubits, chunk_bits, prec, local_world._h, rank, stream, ctypes.byref(h))
        elif world == 1 and buffer_ptr is None and stream is None:
            rc = lib().sv_create(n_qubits, chunk_bits, prec, ctypes.byref(h))
        else:
            uid = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            rc = lib().sv_create_dist(n_qubits, chunk_bits, prec, rank, world, uid, buffer_ptr, buffer_bytes, stream,
                                      ctypes.byref(h))
        check(rc)
        self._h = h

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc):
        check(rc, self._h)

    # -- evolution
    def reset(self, basis_index: int = 0):
        self._check(lib().sv_reset(self._h, int(basis_index)))

    def apply(self, gates, flags: int = 0):
        g = as_gates(gates)
        self._check(lib().sv_apply_circuit(self._h, g.ctypes.data if len(g) else None, len(g), flags))

    def synchronize(self):
        self._check(lib().sv_synchronize(self._h))

    # -- readout
    def amplitudes(self, idx) -> np.ndarray:
        i = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.zeros(len(i), dtype=self.cdtype)
        if len(i):
            self._check(lib().sv_get_amplitudes(self._h, i.ctypes.data, len(i), out.ctypes.data))
        return out

    def state(self) -> np.ndarray:
        out = np.zeros(1 << self.n, dtype=self.cdtype) if self.rank == 0 else None
        self._check(lib().sv_get_state(self._h, out.ctypes.data if out is not None else None))
        return out

    def norm(self) -> float:
        d = ctypes.c_double()
        self._check(lib().sv_norm(self._h, ctypes.byref(d)))
        return d.value

    def probabilities(self, qubits) -> np.ndarray:
        q = np.ascontiguousarray(qubits, dtype=np.int32)
        out = np.zeros(1 << len(q), dtype=np.float64)
        self._check(lib().sv_probabilities(self._h, _ip(q), len(q), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def sample(self, shots: int, seed: int) -> np.ndarray:
        out = np.zeros(shots, dtype=np.uint64)
        self._check(lib().sv_sample(self._h, shots, seed, out.ctypes.data))
        return out

    def permutation(self) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.int32)
        self._check(lib().sv_get_permutation(self._h, _ip(out)))
        return out

    def set_timing(self, enable: bool = True):
        self._check(lib().sv_set_timing(self._h, 1 if enable else 0))

    def reset_stats(self):
        self._check(lib().sv_stats_reset(self._h))

    def stats(self) -> dict:
        s = Stats()
        self._check(lib().sv_stats_get(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in Stats._fields_}


class HostStateVector:
    """Host-memory tier (NEXT-4, sv_host_*): the state in pinned host memory, the current GPU
    caching 2^device_bits-amplitude chunks; every section streams all chunks through the GPU."""

    def __init__(self, n_qubits: int, chunk_bits: int, device_bits: int, precision: str = "fp64"):
        self.n = n_qubits
        self.precision = precision
        h = ctypes.c_void_p()
        prec = {"fp64": SV_FP64, "fp32": SV_FP32}[precision]
        rc = lib().sv_host_create(n_qubits, chunk_bits, prec, device_bits, ctypes.byref(h))
        if rc != 0:
            msg = lib().sv_host_last_error(None)
            raise SvError(rc, msg.decode() if msg else "")
        self._h = h

    def _check(self, rc):
        if rc != 0:
            msg = lib().sv_host_last_error(self._h)
            raise SvError(rc, msg.decode() if msg else "")

    def reset(self, basis_index: int = 0):
        self._check(lib().sv_host_reset(self._h, int(basis_index)))

    def apply(self, gates, flags: int = 0):
        g = as_gates(gates)
        self._check(lib().sv_host_apply_circuit(self._h, g.ctypes.data if len(g) else None, len(g), flags))

    def state(self) -> np.ndarray:
        out = np.empty(1 << self.n, dtype=np.complex128 if self.precision == "fp64" else np.complex64)
        self._check(lib().sv_host_get_state(self._h, out.ctypes.data))
        return out

    def norm(self) -> float:
        v = ctypes.c_double()
        self._check(lib().sv_host_norm(self._h, ctypes.byref(v)))
        return v.value

    def probabilities(self, qubits) -> np.ndarray:
        q = np.ascontiguousarray(qubits, dtype=np.int32)
        out = np.empty(1 << len(q), dtype=np.float64)
        self._check(lib().sv_host_probabilities(self._h, _ip(q), len(q),
                                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().sv_host_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
