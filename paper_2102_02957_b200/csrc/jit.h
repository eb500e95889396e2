// jit.h — run-time specialised section kernels (host C++; NVRTC + CUDA library API).
//
// The interpreter kernel (section.cu) walks a section's program from __constant__ memory; every
// op pays a dispatch and the register file is reshuffled at each dispatch merge point.  Here the
// same program (compile.cpp, already checked by the emulator and the parity tests) is printed as
// straight-line CUDA — slots, maps and coefficient offsets become immediates, the program's ints
// are baked into the module's constant bank — and compiled for sm_100a with NVRTC.  Kernels are
// cached by the program's structure (its ints; coefficient values stay run-time data, passed as
// a kernel parameter), so a circuit with the same shape reuses them.  Mode (environment SV_JIT):
//   "sync"  (default) compile on first use, then launch the generated kernel;
//   "async" launch the interpreter while a background thread compiles;
//   "0"     interpreter only.
// Compiled cubins are also kept on disk (SV_JIT_CACHE=<dir>, default $HOME/.cache/sv_jit, "0"
// disables), keyed by the source and the embedded headers, so later processes skip NVRTC.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

#include "compile.h"

namespace sv {

struct JitCounters {
  uint64_t compiled = 0;   // kernels built by NVRTC
  uint64_t hits = 0;       // launches that found their kernel ready
  uint64_t fallbacks = 0;  // launches that ran the interpreter (mode async / 0, or no NVRTC)
  double compile_ms = 0;   // host time spent in NVRTC + module load
};

// Launch one section with its generated kernel.  Returns false if the caller must run the
// interpreter instead (mode, compile pending or NVRTC unavailable); *err is the launch status.
// split_a / split_b: restrict the launch to half / a quarter of the tiles (kernels.cuh launch_section).
// coef_host: the launch's coefficients (fp64 complex) on the host, passed as a kernel parameter.
// coef_dev: the same coefficients on the device in the state's precision (used when they exceed
// the kernel-parameter space).
bool jit_launch_section(bool dbl, void* sv, const int* prog_host, const double* coef_host, const Launch& L,
                        const void* coef_dev, const void* aux_dev, cudaStream_t st, cudaError_t* err,
                        int split_a = 0, int split_b = 0, int64_t vidx = -1, int64_t only_tile = -1);
// vidx != -1: the launch does not read the state; its input is the basis state whose single
// amplitude (1) sits at shard offset vidx (-2: on another GPU, all zeros here).
// only_tile >= 0: launch the one tile with that block index (plain kernels only).

// Make sure every launch of the program has its kernel: mode sync compiles the missing ones in
// parallel now, mode async queues them.
// virt_first: the first launch reads a deferred basis state (jit_launch_section vidx).
void jit_prepare(const Program& prog, bool dbl, bool virt_first = false);
// Whether the generated kernel of this launch can generate its input (a deferred basis state).
bool jit_virtual_input_ok(const Launch& L, bool dbl);
// Process-wide mode: 0 off, 1 sync, 2 async, -1 query; returns the previous mode.
int jit_set_mode(int mode);
// Block until background compiles have finished (mode async).
void jit_wait();
JitCounters jit_counters();
// Generated source of one launch (tests / debugging).
std::string jit_source(const int* prog_host, const Launch& L, bool dbl);
// Host only: generate + NVRTC-compile one launch (no module load); optionally dump
// <dump_dir>/section_<index>.cu / .cubin.
Status jit_compile_only(const int* prog_host, const Launch& L, bool dbl, const char* dump_dir, int index, double* ms);

}  // namespace sv
