#!/usr/bin/env python
"""bench.py — the driver's benchmark contract for the cache-blocked state-vector hot path.

    python bench.py --gpus N --steps K --warmup W [--impl reference] [--workload qv33]

One STEP = one pass of the whole hot path over the workload: the host blocking
pass + plan + program upload (a1-a3), every section kernel (a4, a7), every cross-GPU exchange
(a5/a6), and a readout of marginal probabilities (a8), all through the C ABI of libsv.so.
The default workload is BASELINE configs[3]: QV(33, depth 10, seed 1), fp64, chunk_bits 9,
strong scaling over N GPUs (2^33 amplitudes = 128 GiB in total; it fits one B200).  The state
(>= 4 GiB) is far larger than L2, so no flush is needed between steps.

Rank 0 prints ONE JSON line.  `value` = input gates per second of the whole job, timed with
CUDA events on the library's stream (max over ranks); `e2e` = the same metric measured through
the public API with host buffers (gate list H2D, probabilities + amplitudes D2H) and a host
clock; `roofline` = the section kernel (the dominant kernel) against its binding roofline;
`cpu_baseline` = the CPU oracle on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import circuits as C  # noqa: E402

METRIC = "QV/QFT circuit gates/s (fp64 state vector, cache-blocked)"
APPLY_FLAGS = 0  # SV_UNBLOCKED with --unblocked (the comparator), else the blocked path


def sv_flags_unblocked():
    return 1  # include/sv.h SV_UNBLOCKED
FALLBACK_HBM_GBS = 6650.0
# FP64 FMA pipe, derived (fallback when profiles/r02_peaks.json is absent): 64 DFMA/clk/SM x 148 SMs
# x 1.965 GHz x 2 flops
FP64_PEAK_TFLOPS = 2 * 64 * 148 * 1.965e9 / 1e12


# ----------------------------------------------------------------------------- workloads
def workload(name: str, world: int):
    g = world.bit_length() - 1
    if name == "qv33":
        n = 33
        return dict(name="qv33", desc="QV(33, depth 10, seed 1) fp64, strong scaling", n=n,
                    gates=C.quantum_volume(n, 10, 1), basis=0, scaling="strong", chunk_bits=9)
    if name == "qv28":
        return dict(name="qv28", desc="QV(28, depth 10, seed 1) fp64", n=28,
                    gates=C.quantum_volume(28, 10, 1), basis=0, scaling="strong", chunk_bits=9)
    if name == "qft30":
        return dict(name="qft30", desc="QFT(30) fp64 on |splitmix64(1) mod 2^30>", n=30, gates=C.qft(30),
                    basis=C.basis_index(1, 30), scaling="strong", chunk_bits=8)
    if name == "qft_weak":
        n = 33 + g
        # c = 9: one read + write pass fewer than c = 8 at 2^33 local amplitudes (QFT33 188 vs 228 ms,
        # profiles/r02_qft_chunk_bits.md)
        return dict(name="qft_weak", desc=f"QFT({n}) fp64, 2^33 amplitudes per GPU (weak)", n=n, gates=C.qft(n),
                    basis=C.basis_index(1, n), scaling="weak", chunk_bits=9)
    if name == "qft_weak_fp32":  # BASELINE configs[4]'s fp32 variant: 2^34 fp32 amplitudes per GPU (37q at 8)
        n = 34 + g
        return dict(name="qft_weak_fp32", desc=f"QFT({n}) fp32, 2^34 amplitudes per GPU (weak)", n=n, gates=C.qft(n),
                    basis=C.basis_index(1, n), scaling="weak", chunk_bits=8, precision="fp32")
    if name == "qv_weak":
        n = 30 + g
        return dict(name="qv_weak", desc=f"QV({n}, 10, 1) fp64, 2^30 amplitudes per GPU (weak)", n=n,
                    gates=C.quantum_volume(n, 10, 1), basis=0, scaling="weak", chunk_bits=9)
    raise SystemExit(f"unknown workload {name}")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", FALLBACK_HBM_GBS)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) < 9:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        load = [s for s in sm if s > 600] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ----------------------------------------------------------------------------- oracle timing
def oracle_sample(wl, target_s: float = 15.0, max_gates: int = None):
    """Time the CPU oracle (as it stands) on the first m gates of the workload from its basis
    state; m is chosen from a one-gate probe so the sample takes ~target_s."""
    import oracle as O
    n = wl["n"]
    gates = wl["gates"]
    a = O.basis_state(n, wl["basis"])
    t0 = time.perf_counter()
    O.apply_circuit(gates[:1], n, a, inplace=True)
    per = time.perf_counter() - t0
    m = max(1, min(len(gates) - 1, int(target_s / max(per, 1e-6))))
    if max_gates:
        m = min(m, max_gates)
    t0 = time.perf_counter()
    O.apply_circuit(gates[1:1 + m], n, a, inplace=True)
    dt = time.perf_counter() - t0
    del a
    return m, dt, per


def oracle_fits(wl):
    """The oracle holds the whole 2^n-amplitude complex128 state in host RAM; return None if it fits
    in MemAvailable (with 10% headroom), else a one-line reason."""
    need = 16 << wl["n"]
    try:
        with open("/proc/meminfo") as f:
            avail = next(int(l.split()[1]) * 1024 for l in f if l.startswith("MemAvailable:"))
    except (OSError, StopIteration):
        return None
    if need * 1.1 > avail:
        return f"oracle state for {wl['n']} qubits needs {need / 2**30:.0f} GiB of host RAM, {avail / 2**30:.0f} GiB available"
    return None


def cores():
    v = os.environ.get("OMP_NUM_THREADS")
    return int(v) if v else (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


def run_reference(args):
    """--impl reference: the oracle (plain C + OpenMP, no blocking) timed on the host cores, each step
    a bounded sample of the same workload (rank 0 only under torchrun)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = workload(args.workload, args.gpus)
    why = oracle_fits(wl)
    if why:
        print(json.dumps({"impl": "reference", "unavailable": why}), flush=True)
        return 0
    import oracle as O
    n, gates = wl["n"], wl["gates"]
    a = O.basis_state(n, wl["basis"])
    t0 = time.perf_counter()
    O.apply_circuit(gates[:1], n, a, inplace=True)
    per = time.perf_counter() - t0
    m = max(1, min(len(gates), int(args.ref_step_s / max(per, 1e-6))))
    gi = 1
    times = []
    for it in range(args.warmup + args.steps):
        sel = [(gi + j) % len(gates) for j in range(m)]
        gi = (gi + m) % len(gates)
        t0 = time.perf_counter()
        O.apply_circuit(gates[sel], n, a, inplace=True)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = args.steps * m / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded QV/QFT generator)",
            "config": {"workload": wl["desc"], "n_qubits": n, "gates_per_step": m, "chunk_bits": None},
            "cpu_baseline": {"value": value, "unit": "gates/s", "cores": cores(), "kind": "oracle",
                             "sample": f"{m} gates of {wl['desc']} per step from its basis state (dense C oracle, OpenMP)"},
            "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def fp64_peak():
    """Measured FP64 FMA peak (TFLOP/s) on this pool's B200 (tools/microbench.cu, 4 s of DFMA back to
    back at the 1965 MHz it held: profiles/r02_peaks.json); the derived 64 DFMA/clk/SM x 148 SMs x
    1.965 GHz x 2 = 37.2 TFLOP/s if that file is missing."""
    p = os.path.join(ROOT, "profiles", "r02_peaks.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["fp64_tflops"]), float(d.get("fp32_tflops", 2 * d["fp64_tflops"])), \
            "measured (profiles/r02_peaks.json: tools/microbench.cu DFMA 4 s at 1965 MHz)"
    return FP64_PEAK_TFLOPS, 2 * FP64_PEAK_TFLOPS, "derived: 64 DFMA/clk/SM x 148 SMs x 1.965 GHz x 2"


class Ctx:
    """Per-process state shared by the workloads of one bench run."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.args = torch, dist, args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def measure(ctx, wl, precision, c, steps, warmup, e2e_steps, with_clocks=True):
    """Time `steps` hot-path steps of workload wl on this rank's GPU(s); returns the raw numbers."""
    import paper_2102_02957_b200 as sv
    torch, world, rank = ctx.torch, ctx.world, ctx.rank
    n, gates = wl["n"], wl["gates"]
    stream = torch.cuda.Stream()
    uid = None
    if world > 1:
        u = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            u.copy_(torch.tensor(np.frombuffer(sv.nccl_unique_id(), dtype=np.uint8).copy()))
        ctx.dist.broadcast(u, 0)
        uid = bytes(u.cpu().numpy().tobytes())
    s = sv.StateVector(n, c, precision, rank=rank, world=world, nccl_id=uid, stream=stream.cuda_stream)
    Q = list(range(min(10, n)))

    def step():  # simulate the circuit from its basis state, then read out
        s.reset(wl["basis"])
        s.apply(gates, flags=APPLY_FLAGS)
        s.probabilities(Q)

    s.reset(wl["basis"])
    for _ in range(warmup):
        step()
    s.synchronize()
    # ---- timed region (device time, CUDA events on the library's stream)
    s.reset_stats()
    s.set_timing(True)
    clk = ClockSampler(ctx.local)
    if with_clocks:
        clk.start()
    ctx.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    e1.synchronize()
    ctx.barrier()
    clocks = clk.stop() if with_clocks else None
    ms = ctx.max_over_ranks(e0.elapsed_time(e1))
    st = s.stats()
    s.set_timing(False)
    # ---- e2e through the public API with host buffers
    e2e = None
    if e2e_steps:
        idx = np.arange(0, 1 << n, max(1, (1 << n) // 1024), dtype=np.uint64)[:1024]
        h2d = gates.nbytes + idx.nbytes
        d2h = (8 << len(Q)) + idx.size * (16 if precision == "fp64" else 8)
        times = []
        for it in range(e2e_steps + 1):
            ctx.barrier()
            t0 = time.perf_counter()
            s.reset(wl["basis"])
            s.apply(gates, flags=APPLY_FLAGS)
            s.probabilities(Q)
            s.amplitudes(idx)
            dt = ctx.max_over_ranks(time.perf_counter() - t0)
            if it > 0:
                times.append(dt)
        e2e = {"value": len(gates) / (sum(times) / len(times)), "unit": "gates/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": len(times)}
    s.close()
    return dict(ms=ms, ms_step=ms / steps, value=len(gates) / (ms / steps / 1e3), st=st, clocks=clocks, e2e=e2e)


def roofline(wl, precision, r, world):
    """The section kernel (K1, the dominant kernel) against the roofline that binds it."""
    st, ms = r["st"], r["ms"]
    if not st["timed_sections"]:
        return None
    hbm_peak, hbm_src = peaks()
    f64, f32, fsrc = fp64_peak()
    fpk = f64 if precision == "fp64" else f32
    t_launch = st["section_ms"] / st["timed_sections"] / 1e3
    bytes_l = st["section_bytes"] / st["timed_sections"]
    flops_l = st["section_flops"] / st["timed_sections"]
    # HBM roofline over the read + write launches; the first section after sv_reset generates its
    # input in-kernel (write only) and is reported beside them
    n_in = st.get("timed_input_sections", 0)
    n_rw = st["timed_sections"] - n_in
    rw = None
    if n_rw > 0 and n_in > 0:
        rw = ((st["section_bytes"] - st["input_section_bytes"]) / n_rw,
              (st["section_ms"] - st["input_section_ms"]) / n_rw / 1e3,
              (st["section_flops"] - st.get("input_section_flops", 0.0)) / n_rw)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "section_traffic.json")
    if os.path.exists(prof) and world == 1:  # captured on one GPU: the N = 1 launch shape only
        try:
            traffic = json.load(open(prof)).get(wl["name"])
        except Exception:
            traffic = None
    if bytes_l / (hbm_peak * 1e9) >= flops_l / (fpk * 1e12):
        b_rw, t_rw, _ = rw if rw else (bytes_l, t_launch, flops_l)
        ach = b_rw / t_rw / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "traffic": traffic, "peak_source": hbm_src,
                "launches_rw": n_rw, "avg_launch_ms_rw": round(t_rw * 1e3, 4), "alg_bytes_per_launch_rw": b_rw}
    else:
        _, t_rw, f_rw = rw if rw else (bytes_l, t_launch, flops_l)
        ach = f_rw / t_rw / 1e12
        roof = {"bound": "alu", "achieved": round(ach, 3), "peak": round(fpk, 2), "unit": "TFLOP/s",
                "frac": round(ach / fpk, 4), "traffic": traffic, "peak_source": fsrc,
                "launches_rw": n_rw, "avg_launch_ms_rw": round(t_rw * 1e3, 4), "alg_flops_per_launch_rw": f_rw}
    roof.update({"kernel": "sv_sec (run-time specialised section kernel; k_section when interpreted)",
                 "launches_timed": st["timed_sections"], "avg_launch_ms": round(t_launch * 1e3, 4),
                 "alg_bytes_per_launch": bytes_l, "alg_flops_per_launch": flops_l,
                 "hbm_frac_of_measured": round(bytes_l / t_launch / 1e9 / hbm_peak, 4),
                 "section_share_of_step": round(st["section_ms"] / ms, 4),
                 "input_sections": ({"launches": n_in, "avg_ms": round(st["input_section_ms"] / n_in, 4),
                                     "write_only_gbs": round(st["input_section_bytes"] / (st["input_section_ms"] / 1e3) / 1e9, 1)}
                                    if n_in else None),
                 "alg_bytes_note": "2 x shard bytes per section launch (read + write); the first section after "
                                   "sv_reset clears the shard and computes only the tile holding the basis amplitude "
                                   "(1 x shard bytes, one tile of flops): reported as input_sections, excluded from "
                                   "frac (the read + write launches, *_rw)"})
    clocks = r.get("clocks") or {}
    if roof["bound"] == "alu" and clocks.get("sm_mhz"):
        # the FP64 peak scales with the SM clock; under FP64 + HBM load the B200 runs below its
        # 1965 MHz maximum (sw_power_cap): the fraction at the clock it actually ran is context
        f = clocks["sm_mhz"] / 1965.0
        roof["peak_at_load_clock"] = round(roof["peak"] * f, 2)
        roof["frac_at_load_clock"] = round(roof["frac"] / f, 4)
    return roof


def nvlink(r, steps, wl_name=None, world=1):
    st, ms = r["st"], r["ms"]
    if not st["exchange_ms"]:
        return None
    gbs = st["bytes_sent"] / (st["exchange_ms"] / 1e3) / 1e9
    alone = None
    prof = os.path.join(ROOT, "profiles", "r02_exchange_alone.json")
    if os.path.exists(prof) and not APPLY_FLAGS:
        try:
            alone = json.load(open(prof)).get(f"{wl_name}_n{world}")
        except Exception:
            alone = None
    return {"achieved": round(gbs, 1), "peak": 900.0, "unit": "GB/s per direction", "frac": round(gbs / 900.0, 4),
            "counters": "unavailable: NVML NVLink byte counters report NOT_SUPPORTED on this pool's driver (profiles/r02_nvml_probe.txt)",
            "overlapped": os.environ.get("SV_XPIPE", "1") != "0",
            "alone_measured": alone,
            "frac_of_measured_peer_copy": round(gbs / 770.0, 4), "bytes_per_rank_per_step": st["bytes_sent"] / steps,
            "share_of_step": round(st["exchange_ms"] / ms, 4),
            "transport": "NCCL send/recv (packed)" if APPLY_FLAGS & 4 else ("copy engines over CUDA IPC: strided rows from the state into the peer's slot and back into place "
                          "(rows >= SV_XRUN bytes, default 1 KiB), else pack kernel + copy + unpack kernel"
                          if os.environ.get("SV_XCE", "1") != "0" else "peer-store push kernel (CUDA IPC)")}


def run_ours(args):
    ctx = Ctx(args)
    torch, world, rank = ctx.torch, ctx.world, ctx.rank
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(ctx.local)
    if world > 1:
        ctx.dist.init_process_group("nccl", device_id=torch.device("cuda", ctx.local))
    wl = workload(args.workload, world)
    if wl.get("precision"):
        args.precision = wl["precision"]
    wl["desc"] = wl["desc"].replace("fp64", args.precision)
    n, gates = wl["n"], wl["gates"]
    c = args.chunk_bits if args.chunk_bits else wl["chunk_bits"]
    r = measure(ctx, wl, args.precision, c, args.steps, args.warmup, 0 if args.no_e2e else args.e2e_steps)
    st, ms, clocks = r["st"], r["ms"], r["clocks"]
    roof = roofline(wl, args.precision, r, world)
    nvl = nvlink(r, args.steps, wl["name"], world) if world > 1 else None

    # ---- the HBM-bound workload beside it (BASELINE configs[2], QFT30 fp64 c = 8), same GPUs
    sub = {}
    if not args.no_sub and args.workload != "qft30":
        wq = workload("qft30", world)
        rq = measure(ctx, wq, "fp64", wq["chunk_bits"], 20, 3, 0, with_clocks=True)
        sub["qft30"] = {"workload": wq["desc"], "value": rq["value"], "unit": "gates/s", "ms_per_step": rq["ms_step"],
                        "steps": 20, "warmup": 3, "chunk_bits": wq["chunk_bits"],
                        "roofline": roofline(wq, "fp64", rq, world),
                        "nvlink": nvlink(rq, 20, "qft30", world) if world > 1 else None, "clocks": rq["clocks"],
                        "gpu_launches": int(rq["st"]["kernel_launches"])}

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and oracle_fits(wl):
        cpu = {"value": None, "unit": "gates/s", "cores": cores(), "kind": "oracle", "sample": oracle_fits(wl)}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        m, dt, per = oracle_sample(wl, target_s=args.cpu_target_s)
        cpu = {"value": m / dt, "unit": "gates/s", "cores": cores(), "kind": "oracle",
               "sample": f"gates 2..{m + 1} of {wl['desc']} from its basis state ({m} gates, {dt:.1f} s; dense C oracle, OpenMP)"}

    line = {"metric": METRIC, "value": r["value"], "unit": "gates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_step"], "higher_is_better": True, "scaling": wl["scaling"],
            "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic (seeded QV/QFT generator, circuits/gen.py)",
            "config": {"workload": wl["desc"], "n_qubits": n, "gates": int(len(gates)), "chunk_bits": c,
                       "precision": args.precision, "parallelism": f"state sharded over {world} GPU(s)",
                       "l2": "state >= 4 GiB per GPU >> 126 MB L2 (no flush needed)",
                       "step": "sv_reset(basis; deferred: the first section clears the shard and runs only the tile holding the basis amplitude) + sv_apply_circuit (pass+plan+upload+sections+exchanges) + sv_probabilities(10 qubits)",
                       "path": ("unblocked per-gate baseline (SV_UNBLOCKED)" if APPLY_FLAGS & 1 else "cache-blocked") +
                               (", NCCL send/recv exchange" if APPLY_FLAGS & 4 else "")},
            "amp_updates_per_s": r["value"] * (1 << n),
            "sections_per_step": st["sections"] / args.steps, "exchanges_per_step": st["exchanges"] / args.steps,
            "exchange_bytes_per_rank_per_step": st["bytes_sent"] / args.steps,
            "exchange_ms_per_step": st["exchange_ms"] / args.steps,
            "host_pass_ms": st["pass_ms"],
            "roofline": roof, "nvlink": nvl, "cpu_baseline": cpu, "e2e": r["e2e"],
            "section_kernels": {"generated": int(st["jit_launches"]), "interpreted": int(st["interp_launches"]),
                                "compiled_total": int(st["jit_compiled"]),
                                "compile_ms_total": round(st["jit_compile_ms"], 1)},
            "gpu_launches": int(st["kernel_launches"]), "clocks": clocks}
    if sub:
        line["workloads"] = sub
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="qv33")
    ap.add_argument("--chunk-bits", type=int, default=0, help="0: the workload's measured best (DESIGN.md)")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--unblocked", action="store_true",
                    help="the paper's per-gate baseline (SV_UNBLOCKED): one pass per gate, exchanges per global gate")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the QFT30 (HBM-bound) sub-workload of the line")
    ap.add_argument("--nccl", action="store_true", help="cross-GPU exchange by NCCL send/recv (SV_EXCHANGE_NCCL)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-target-s", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # contract: W >= 3
    global APPLY_FLAGS
    APPLY_FLAGS = (sv_flags_unblocked() if args.unblocked else 0) | (4 if args.nccl else 0)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
