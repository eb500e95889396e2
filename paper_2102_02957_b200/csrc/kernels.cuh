// kernels.cuh — launch interfaces of the sm_100a kernels (host-callable wrappers).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sv {

// K1: one launch per section.  Copies the section's program (int_count ints at prog_dev) and
// coefficients (coef_count complex numbers in amp dtype at coef_dev) into __constant__ memory on
// `st`, then launches 2^n_out CTAs.  dbl selects fp64 (double2 amplitudes) vs fp32 (float2).
// split_a / split_b: 0, or (1 << 16) | (value << 8) | index into the section's out bits: the
// launch covers only the tiles whose out bit has that value (pipelined exchange + section)
cudaError_t launch_section(bool dbl, void* sv, const int* prog_dev, size_t int_count, const void* coef_dev,
                           size_t coef_count, const void* aux_dev, int T, int n_out, int n_phases, int flags,
                           int n_sets, cudaStream_t st, int split_a = 0, int split_b = 0);

// K2: per-gate baseline, one pass over the shard per gate.  q0/q1 are memory bits;
// diag codes follow program.h (rank bits pre-folded to constants).
struct GateArgs {
  int type;       // SV_OP_U1 / U2 / DIAG / SWAP(=7)
  int q0, q1;
  double m[32];   // complex coefficients (fp64; converted in the wrapper for fp32)
};
cudaError_t launch_gate(bool dbl, void* sv, int nL, const GateArgs& g, cudaStream_t st);

// write the real value re at local offset off (one amplitude)
cudaError_t launch_set_amp(bool dbl, void* sv, int64_t off, double re, cudaStream_t st);
// K6: |k>: zero the shard and write 1 at local offset `off` if owned.
cudaError_t launch_set_basis(bool dbl, void* sv, int nL, int64_t off, cudaStream_t st);

// K5: reductions.  Partial arrays are device scratch of the sizes returned by *_scratch.
size_t norm_scratch_doubles();
cudaError_t launch_norm(bool dbl, const void* sv, int nL, double* scratch, double* out_dev, cudaStream_t st);
// histogram of |a|^2 over `nq` local memory bits (bin bit i <- memory bit qbits[i]); out has 2^nq doubles
size_t marginal_scratch_doubles(int nq);
cudaError_t launch_marginal(bool dbl, const void* sv, int nL, const int* qbits, int nq, double* scratch,
                            double* out_dev, cudaStream_t st);
// sums of |a|^2 over consecutive blocks of 2^B amplitudes
cudaError_t launch_block_sums(bool dbl, const void* sv, int nL, int B, double* out_dev, cudaStream_t st);
// resolve shots: for each of n_blocks work items (block id, first shot, shot count), CTA-scan the
// block and binary-search each residual u; writes local offsets.
cudaError_t launch_sample_resolve(bool dbl, const void* sv, int B, const int64_t* items, int n_items,
                                  const double* resid, uint64_t* out_off, cudaStream_t st);

// K7: out[i] = sv[offs[i]] if offs[i] != ~0 else 0.
cudaError_t launch_gather(bool dbl, const void* sv, const uint64_t* offs, size_t cnt, void* out, cudaStream_t st);

// Exchange: pack (stage[i] = sv[x_i]) or unpack (sv[x_i] = stage[i]) elements first .. first +
// count - 1 of a block, x_i = (first + i) with bit val[k] inserted at pos[k]; stage may be a peer's
// buffer mapped over NVLink.  max_blocks caps the grid (0: a full grid).
// shard_amps: the shard's amplitude count (a checked build, SV_CHECK=1, traps on indices beyond it).
cudaError_t launch_pack_bits(bool dbl, bool pack, void* sv, void* stage, uint64_t first, uint64_t count, int nins,
                             const int* pos, const int* val, uint64_t shard_amps, cudaStream_t st,
                             unsigned max_blocks = 0);
// the same pack (sv -> stage) / unpack (stage -> sv) as copy-engine 2-D copies when the block's
// runs are >= min_run elements (kernels.cu); cudaErrorNotSupported otherwise; *copies = copies issued
cudaError_t copy_bits_ce(bool pack, void* sv, void* stage, uint64_t first, uint64_t count, int nins, const int* pos,
                         const int* val, size_t amp, uint64_t min_run, cudaStream_t st, int* copies);
// state rows -> the same rows of another (peer) state with other inserted-bit values (kernels.cu)
cudaError_t copy_bits_ce_xx(void* src, const int* vsrc, void* dst, const int* vdst, uint64_t first, uint64_t count,
                            int nins, const int* pos, size_t amp, uint64_t min_run, cudaStream_t st, int* copies,
                            bool dry);

}  // namespace sv
