/*
 * sv.h — C ABI of the B200 cache-blocked state-vector library (libsv.so).
 *
 * The operation: apply a circuit of 1-/2-qubit unitaries, diagonal gates and swaps to an
 * n-qubit state vector of 2^n complex amplitudes (§II-A), with the state
 * split into chunks and the top log2(G) qubits indexing GPUs, using the
 * cache-blocking transpiler of §IV-A (Listing 3) so every gate runs inside one
 * chunk-sized tile and data crosses GPUs only at chunk_swaps.
 *
 * Conventions
 *   - Qubit k <-> bit k of the amplitude index, zero-based, little-endian.
 *   - Amplitudes are complex interleaved (re, im): 16 B (SV_FP64) or 8 B (SV_FP32) each.
 *   - Gate matrices are always fp64, complex interleaved, ROW-major, and are rounded to
 *     nearest to fp32 on upload for SV_FP32.  U2 sub-index s = bit(q0) + 2*bit(q1), so
 *     CNOT(control c, target t) = U2(q0 = t, q1 = c, Eq. 2 matrix).
 *   - Diagonality is declared by kind (SV_D1 / SV_D2), never detected.
 *   - Every getter speaks LOGICAL qubits / indices; the library tracks the permutation the
 *     blocking pass leaves behind (order is restored only on request).
 *
 * Ownership: the caller owns every input array and host output buffer (sizes given by the
 * caller).  The library copies gates before returning and never retains caller pointers,
 * except ext_dev_buf in sv_create_dist, which must outlive the handle.  Arrays the library
 * returns (sv_block_circuit, sv_plan_circuit) are freed with sv_free.
 *
 * Errors: every int-returning call returns SV_OK (0) or a negative SV_E* code; the message is
 * available from sv_last_error(handle) (thread-local when handle == NULL).  No C++ exception
 * crosses the ABI.  Handles are not thread-safe.  With world > 1 every call on a handle is
 * collective: all ranks call it in the same order with the same arguments.
 *
 * Preconditions: 1 <= chunk_bits <= n - log2(world); world is a power of two; n <= 40.
 */
#ifndef SV_H
#define SV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sv_state* sv_handle;

typedef enum { SV_FP32 = 0, SV_FP64 = 1 } sv_precision;

/* Gate / token kinds.  1-5 are input gates; 6-9 appear only in library output
 * (sv_block_circuit: 6-8; sv_plan_circuit: 6-9). */
enum {
  SV_U1 = 1,         /* 2x2 unitary on q0 (m[0..7]) — u3 of Eq. 1 arrives as this */
  SV_U2 = 2,         /* 4x4 unitary on (q0, q1) (m[0..31]) — CNOT of Eq. 2        */
  SV_D1 = 3,         /* diag(d0, d1) on q0 (m[0..3]) — u1                             */
  SV_D2 = 4,         /* diag(d0..d3) on (q0, q1) (m[0..7]) — controlled phase         */
  SV_SWAP = 5,       /* swap of q0 and q1, no payload                                        */
  SV_CHUNK_SWAP = 6, /* chunk_swap(sq0 = q0 < sq1 = q1) inserted by the pass  */
  SV_BEGIN = 7,      /* begin_blocking                                               */
  SV_END = 8,        /* end_blocking                                                 */
  SV_EXCHANGE = 9    /* plan only: physically swap local memory bit q0 with rank bit q1      */
};

typedef struct {
  int32_t kind, q0, q1, pad; /* pad: ignored on input; sv_block_circuit writes the input index */
  double m[32];
} sv_gate;

/* Flags for sv_apply_circuit / sv_block_circuit / sv_plan_circuit. */
#define SV_UNBLOCKED     (1u << 0) /* per-gate baseline: one HBM pass per gate, no pass  */
#define SV_RESTORE_ORDER (1u << 1) /* append swaps returning the paper-physical order to logical */
#define SV_EXCHANGE_NCCL (1u << 2) /* cross-GPU exchange by NCCL send/recv through a staging ring */
                                   /* instead of copy-engine peer copies (CUDA IPC)              */
#define SV_ABSORB_SWAPS  (1u << 5) /* the pass absorbs user SWAP gates as relabels of pi (the  */
                                   /* paper's bit reordering) instead of   */
                                   /* treating them as 2-qubit gates; sections that would hold  */
                                   /* only absorbed swaps are not emitted                       */
#define SV_FREE_LAYOUT   (1u << 3) /* sv_plan_circuit / sv_compile_circuit: plan as sv_apply_   */
                                   /* circuit does right after sv_reset (the state is a basis   */
                                   /* state, so the planner chooses the initial memory layout; */
                                   /* sigma0 is ignored).  sv_apply_circuit decides this itself */

/* Error codes. */
#define SV_OK           0
#define SV_EINVAL      -1 /* bad qubit, duplicate qubit, bad chunk_bits / world / argument  */
#define SV_ECAPACITY   -2 /* state does not fit device (or host) memory                      */
#define SV_EINFEASIBLE -3 /* non-diagonal 2-qubit gate with chunk_bits < 2; or a    */
                          /* per-gate (unblocked) non-diagonal gate on a global qubit          */
#define SV_EMALFORMED  -4 /* malformed record / marker sequence                               */
#define SV_ECUDA       -5 /* CUDA runtime failure                                              */
#define SV_ENCCL       -6 /* NCCL failure or NCCL library not loadable; a collective that did  */
                          /* not complete within SV_COMM_TIMEOUT_S (default 600 s; the        */
                          /* communicator is then aborted) or reported an asynchronous error   */
#define SV_EUNAVAILABLE -7 /* optional run-time component missing (NVRTC for sv_jit_compile_*) */

typedef struct sv_stats {
  uint64_t circuits;          /* sv_apply_circuit calls                                       */
  uint64_t gates;             /* input gates applied                                          */
  uint64_t sections;          /* blocked sections executed (one HBM pass each)         */
  uint64_t chunk_swaps;       /* chunk_swap tokens from the pass (all virtual relabels)       */
  uint64_t exchanges;         /* physical cross-GPU bit exchanges (local bit <-> rank bit)    */
  uint64_t exchange_batches;  /* exchange steps (each one grouped all-to-all in a subcube)    */
  uint64_t bytes_sent;        /* amplitude bytes this rank moved to peers                     */
  uint64_t kernel_launches;   /* library kernels launched                                     */
  double pass_ms;             /* host time in the blocking pass + planning (last call)        */
  double apply_ms;            /* host wall time of the last sv_apply_circuit                   */
  /* device-side accounting (filled when timing is enabled with sv_set_timing) */
  uint64_t timed_sections;    /* section launches timed with CUDA events                       */
  double section_ms;          /* summed event time of those section launches                   */
  double exchange_ms;         /* summed event time of cross-GPU exchange steps                 */
  double gate_ms;             /* summed event time of per-gate (unblocked) launches            */
  double section_bytes;       /* algorithmic HBM bytes of the timed sections (2 x shard each)  */
  double section_flops;       /* algorithmic flops of the timed sections (DESIGN "Roofline")   */
  uint64_t compactions;       /* standalone memory-bit swap passes (tile coalescing fallback)  */
  uint64_t store_swaps;       /* memory-bit swaps fused into section stores (free)            */
  /* run-time specialised section kernels (NVRTC, environment SV_JIT=sync|async|0) */
  uint64_t jit_launches;      /* section launches that ran a generated kernel                  */
  uint64_t interp_launches;   /* section launches that ran the program interpreter             */
  uint64_t jit_compiled;      /* kernels compiled by this process so far (cache misses)        */
  double jit_compile_ms;      /* host time spent compiling them (process total)                */
  /* the timed sections whose input is generated in-kernel (the first section after sv_reset:
   * write-only, 1 x shard bytes); also counted in timed_sections / section_ms / section_bytes */
  uint64_t timed_input_sections;
  double input_section_ms;
  double input_section_bytes;
  double input_section_flops;
} sv_stats_t;

/* ---- lifetime ------------------------------------------------------------------------- */
/* One GPU (the caller's current CUDA device), state |0..0>, memory allocated by the library. */
int sv_create(int n_qubits, int chunk_bits, sv_precision prec, sv_handle* out);
/* One rank of a world of `world` GPUs (one process per GPU, current device).  nccl_unique_id:
 * 128 bytes from sv_nccl_unique_id on rank 0, broadcast by the caller (required if world>1).
 * ext_dev_buf (nullable): device buffer of >= ext_bytes = 2^(n-log2 world) * amp bytes that
 * holds this rank's shard; cuda_stream (nullable): stream all work is issued on (default: a
 * library-created stream).  Rank r holds the amplitudes whose top log2(world) memory bits = r
 * (contiguous placement). */
int sv_create_dist(int n_qubits, int chunk_bits, sv_precision prec, int rank, int world,
                   const void* nccl_unique_id, void* ext_dev_buf, size_t ext_bytes,
                   void* cuda_stream, sv_handle* out);
/* Release the handle: its shard (unless ext_dev_buf), stream (unless the caller's), communicator
 * and peer mappings; waits for the handle's queued work first.  NULL is a no-op.  Always SV_OK. */
int sv_destroy(sv_handle h);
/* Write ncclGetUniqueId() into out (128 bytes): the bootstrap of P:137-143's process grid. */
int sv_nccl_unique_id(void* out128);

/* ---- in-process virtual world (testing the multi-GPU path on one device) ----------------
 * The paper distributes 2^(n - log2 G)-amplitude shards over G processes and
 * exchanges them only at chunk_swaps on global qubits.  A virtual world runs the
 * same G ranks inside ONE process on the caller's current device: sv_world_create(G) makes the
 * world, sv_create_local(..., w, r, ...) creates rank r's handle (its shard on the current device,
 * cuda_stream nullable as in sv_create_dist).  Each rank's handle must be driven by its own host
 * thread, every rank calling the same collective sequence as under NCCL; exchanges run the same
 * plans and peer copies (copy engines, pack kernels for short rows), barriers are CUDA events
 * passed through a host barrier (no device-side waiting), reductions are summed on the host in
 * rank order, send/recv are
 * device-to-device copies.  A rank that does not reach a collective within SV_COMM_TIMEOUT_S
 * seconds (default 600) makes the others fail with SV_ENCCL.  The world is reference counted:
 * sv_world_destroy may be called right after the last sv_create_local.  Errors: SV_EINVAL
 * (world not a power of two <= 64, bad rank), as sv_create_dist otherwise. */
typedef struct sv_world_s* sv_world;
int sv_world_create(int world, sv_world* out);
int sv_world_destroy(sv_world w);
int sv_create_local(int n_qubits, int chunk_bits, sv_precision prec, sv_world w, int rank, void* cuda_stream,
                    sv_handle* out);

/* ---- evolution ------------------------------------------------------------------------ */
/* |k> for LOGICAL basis index k; resets the tracked permutations to identity. */
int sv_reset(sv_handle h, uint64_t basis_index);
/* Apply n_gates input records (kinds SV_U1..SV_SWAP, logical qubits) in order.  Default:
 * blocked (Listing 3 pass, then one section kernel per section and exchanges only for
 * global qubits).  Returns after all work is enqueued on the handle's stream. */
int sv_apply_circuit(sv_handle h, const sv_gate* gates, size_t n_gates, uint32_t flags);
/* Block until the handle's stream is idle (with world > 1: polling the communicator for
 * asynchronous errors, SV_ENCCL after SV_COMM_TIMEOUT_S seconds). */
int sv_synchronize(sv_handle h);

/* ---- readout (all collective; results on every rank) --------------------------------- */
/* host_out[i] = amplitude of LOGICAL index logical_idx[i] (cnt complex values, amp dtype): the
 * paper's output state read through the tracked permutation (DESIGN R7).
 * SV_EINVAL for an index >= 2^n or null pointers. */
int sv_get_amplitudes(sv_handle h, const uint64_t* logical_idx, size_t cnt, void* host_out);
/* Full state in LOGICAL order into host_out (2^n complex, amp dtype); written on rank 0 only. */
int sv_get_state(sv_handle h, void* host_out);
/* *out = sum_x |a_x|^2 (unitarity check, north_star).  SV_EINVAL if out is NULL. */
int sv_norm(sv_handle h, double* out);
/* Marginal probabilities over LOGICAL qubits Q (qubits[0] -> bit 0 of the output index),
 * host_out has 2^nq doubles, nq <= 24.  p[y] = sum_{x : x|Q = y} |a_x|^2 (DESIGN R17). */
int sv_probabilities(sv_handle h, const int32_t* qubits, int nq, double* host_out);
/* shots samples of LOGICAL basis indices from |a|^2 into host_out; u_s = (splitmix64(seed ^ s)
 * >> 11) * 2^-53 is inverted through the CDF in memory order (DESIGN R16). */
int sv_sample(sv_handle h, size_t shots, uint64_t seed, uint64_t* host_out);
/* logical_to_physical[q] = paper-physical position of logical qubit q: the permutation pi the
 * blocking pass leaves behind ("the order of qubits is changed").  Host only, no sync.
 * SV_EINVAL if an argument is NULL; the caller's array has n entries. */
int sv_get_permutation(sv_handle h, int32_t* logical_to_physical);
/* Cumulative counters since creation / the last sv_stats_reset (synchronizes when timing).
 * sv_stats is SURVEY §8(b)'s name; sv_stats_get the same call.  Counts what the blocking pass and
 * the executor did (sections = the paper's blocked passes over the chunks, P:383, P:386-394;
 * chunk_swaps; exchanges / bytes_sent).  Errors: SV_EINVAL (null argument),
 * SV_ECUDA (reading the timing events). */
int sv_stats(sv_handle h, struct sv_stats* out);
int sv_stats_get(sv_handle h, struct sv_stats* out);
int sv_stats_reset(sv_handle h);
/* enable != 0: bracket every section / exchange / per-gate launch with CUDA events on the
 * handle's stream and accumulate device times into sv_stats (small overhead per launch). */
int sv_set_timing(sv_handle h, int enable);
const char* sv_last_error(sv_handle h);

/* ---- host-memory tier (NEXT-4) -------------------------
 * The state lives in pinned host memory (2^n amplitudes) and the GPU caches 2^device_bits-
 * amplitude chunks: every blocked section is one streaming pass of all chunks through the current
 * device (H2D, section kernel, D2H overlapped); the top n - device_bits qubits index chunks like
 * rank bits index GPUs, so an exchange with them is a bit permutation of the host array.  For
 * states beyond HBM (PCIe-bound: expect ~2 x state bytes / PCIe bandwidth per section).
 * Requires 4 <= device_bits < n <= 40, 1 <= chunk_bits <= device_bits.  State |0..0> after
 * create.  Blocked path only (flags SV_UNBLOCKED / SV_EXCHANGE_NCCL: SV_EINVAL).  Outputs: the
 * full state in logical order (2^n amplitudes of the precision), the norm, marginals as
 * sv_probabilities.  Errors: sv_host_last_error. */
typedef struct sv_host_state* sv_host_handle;
int sv_host_create(int n_qubits, int chunk_bits, sv_precision prec, int device_bits, sv_host_handle* out);
int sv_host_destroy(sv_host_handle h);
int sv_host_reset(sv_host_handle h, uint64_t basis_index);
int sv_host_apply_circuit(sv_host_handle h, const sv_gate* gates, size_t n_gates, uint32_t flags);
int sv_host_get_state(sv_host_handle h, void* host_out);
int sv_host_norm(sv_host_handle h, double* out);
int sv_host_probabilities(sv_host_handle h, const int32_t* qubits, int nq, double* host_out);
const char* sv_host_last_error(sv_host_handle h);

/* ---- host-only (no GPU needed; used for parity of the pass and the plan) -------------- */
/* The cache-blocking pass (Listing 3, DESIGN R2-R6) on logical gates.  *out receives the
 * token stream (SV_CHUNK_SWAP / SV_BEGIN / SV_END and gates on physical qubits, pad = input
 * index); pi_final[q] = physical position of logical q.  pi0 nullable (= identity). */
int sv_block_circuit(const sv_gate* gates, size_t n_gates, int n, int chunk_bits,
                     const int32_t* pi0, uint32_t flags, sv_gate** out, size_t* n_out,
                     int32_t* pi_final);
/* The executor's plan for a world of 2^world_log2 GPUs: SV_EXCHANGE records (q0 = local
 * memory bit, q1 = rank memory bit >= n - world_log2), and BEGIN ... END sections whose gates
 * act on MEMORY bits.  pi0/sigma0 nullable (= identity); pi_final / sigma_final receive the
 * logical->physical and physical->memory maps after the circuit. */
int sv_plan_circuit(const sv_gate* gates, size_t n_gates, int n, int chunk_bits, int world_log2,
                    const int32_t* pi0, const int32_t* sigma0, uint32_t flags, sv_gate** out,
                    size_t* n_out, int32_t* pi_final, int32_t* sigma_final);
/* The section programs sv_apply_circuit would launch for rank `rank` of 2^world_log2 GPUs, for
 * testing the section compiler without a GPU.  *steps: n_steps records of 12 int64:
 *   {1, int_off, int_count, coef_off, coef_count, T, n_out, flags, aux_off, aux_count}  a launch
 *   {3, m1, m2, 0, ...}                                            a memory-bit swap pass
 *   {0, m, b, batch, 0, ...}                                       an exchange pair
 *   {2, kind, q0, q1, gate index, 0, ...}                          a per-gate launch
 * *ints / *coefs / *aux: the programs (program.h layout), fp64 complex coefficients (constant
 * bank) and fp64 complex DIAGSET factor tables (global memory).  pi_final /
 * sigma_final as in sv_plan_circuit.  All outputs are freed with sv_free. */
/* Host only (no GPU): generate the run-time specialised kernel of every section launch that
 * sv_compile_circuit returns (same arguments) and compile it for sm_100a with NVRTC, as
 * sv_apply_circuit does on first use (SV_JIT, jit.h).  *n_kernels / *compile_ms report the work;
 * dump_dir (nullable) receives section_<i>.cu and section_<i>.cubin.  SV_EUNAVAILABLE if NVRTC
 * cannot be loaded. */
int sv_jit_compile_circuit(const sv_gate* gates, size_t n_gates, int n, int chunk_bits, int world_log2, int rank,
                           sv_precision prec, uint32_t flags, const char* dump_dir, int* n_kernels,
                           double* compile_ms);
/* Process-wide section-kernel mode: 0 = program interpreter only, 1 = run-time specialised
 * kernels compiled on first use (default; in parallel for all sections of a circuit), 2 = same,
 * compiled in the background while the interpreter runs.  -1 queries.  The environment variable
 * SV_JIT=0|sync|async sets the initial mode.  Returns the previous mode. */
int sv_jit_mode(int mode);
/* Block until background (mode 2) compiles have finished. */
int sv_jit_wait(void);
int sv_compile_circuit(const sv_gate* gates, size_t n_gates, int n, int chunk_bits, int world_log2,
                       int rank, sv_precision prec, const int32_t* pi0, const int32_t* sigma0,
                       uint32_t flags, int64_t** steps, size_t* n_steps,
                       int32_t** ints, size_t* n_ints, double** coefs, size_t* n_coefs,
                       double** aux, size_t* n_aux, int32_t* pi_final, int32_t* sigma_final);
void sv_free(void* p);
/* ABI version (for the binding's check). */
int sv_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SV_H */
