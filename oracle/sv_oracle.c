/*
 * sv_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct dense state-vector simulator, written from the
 * paper (/root/reference/PAPER.md, cited "P:line") and the DESIGN.md readings.  It
 * applies the gates of a circuit one at a time to a dense 2^n complex128 array, in
 * input order, with no chunks, no blocking and no reordering: the plain definition
 * of U_circuit |psi0> that the cache-blocked GPU path must reproduce (DESIGN.md
 * "Oracle").  It shares no code, header, table or constant with
 * paper_2102_02957_b200/ and must only be loaded by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs.
 *
 * Conventions (R1, R11, R12):
 *   - qubit k <-> bit k of the amplitude index, zero-based;
 *   - amplitudes are interleaved (re, im) doubles;
 *   - gate records: int32 kind, q0, q1, pad; double m[32], complex interleaved,
 *     ROW-major; 2-qubit sub-index s = bit(q0) + 2*bit(q1) (Eq. 2 with q1 = control).
 *
 * Parallelism: OpenMP over the independent pair / group loop only ("the
 * changes can be computed in parallel"); each group is touched by exactly one
 * iteration, so the result does not depend on the thread count.
 */
#include <complex.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

enum { OR_U1 = 1, OR_U2 = 2, OR_D1 = 3, OR_D2 = 4, OR_SWAP = 5, OR_CHUNK_SWAP = 6, OR_BEGIN = 7, OR_END = 8 };

typedef struct {
  int32_t kind, q0, q1, pad;
  double m[32];
} or_gate;

static inline cplx ld(const double *a, uint64_t i) { return a[2 * i] + I * a[2 * i + 1]; }
static inline void st(double *a, uint64_t i, cplx v) {
  a[2 * i] = creal(v);
  a[2 * i + 1] = cimag(v);
}
static inline cplx mat(const double *m, int idx) { return m[2 * idx] + I * m[2 * idx + 1]; }

/* Pair addressing of Listing 2: i1 = i & mask; i0 = ((i - i1) << 1) + i1; i1 = i0 + 2^k.
 * Returned as a function so the tests can check it against the worked pair (0011, 0111). */
void or_pair_address(uint64_t i, int k, uint64_t *i0, uint64_t *i1) {
  uint64_t add = 1ull << k, mask = add - 1;
  uint64_t lo = i & mask;
  uint64_t a = ((i - lo) << 1) + lo;
  *i0 = a;
  *i1 = a + add;
}

/* O2: a 2x2 matrix on qubit k.  a'_{i0} = m00 a_{i0} + m01 a_{i1}; a'_{i1} = m10 a_{i0} + m11 a_{i1}
 * (P:252-253), with m ROW-major (m[0]=m00, m[1]=m01, m[2]=m10, m[3]=m11). */
void or_apply_1q(double *a, int n, int k, const double *m) {
  cplx m00 = mat(m, 0), m01 = mat(m, 1), m10 = mat(m, 2), m11 = mat(m, 3);
  int64_t half = (int64_t)1 << (n - 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < half; i++) {
    uint64_t i0, i1;
    or_pair_address((uint64_t)i, k, &i0, &i1);
    cplx q0 = ld(a, i0), q1 = ld(a, i1);
    st(a, i0, m00 * q0 + m01 * q1);
    st(a, i1, m10 * q0 + m11 * q1);
  }
}

/* Insert a zero bit at position p of x (bits >= p move up by one). */
static inline uint64_t insert_zero(uint64_t x, int p) {
  uint64_t lo = x & ((1ull << p) - 1);
  return ((x - lo) << 1) | lo;
}

/* O3: a 4x4 matrix M on (q0, q1): every group of 4 indices that differ only in bits q0, q1,
 * ordered by s = bit(q0) + 2*bit(q1), is replaced by M v (Eq. 2 convention P:96-107). */
void or_apply_2q(double *a, int n, int q0, int q1, const double *m) {
  int lo = q0 < q1 ? q0 : q1, hi = q0 < q1 ? q1 : q0;
  int64_t quarter = (int64_t)1 << (n - 2);
  cplx M[16];
  for (int i = 0; i < 16; i++) M[i] = mat(m, i);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < quarter; i++) {
    uint64_t base = insert_zero(insert_zero((uint64_t)i, lo), hi);
    uint64_t idx[4];
    cplx v[4], w[4];
    for (int s = 0; s < 4; s++) {
      idx[s] = base | ((uint64_t)(s & 1) << q0) | ((uint64_t)(s >> 1) << q1);
      v[s] = ld(a, idx[s]);
    }
    for (int r = 0; r < 4; r++) {
      w[r] = 0;
      for (int c = 0; c < 4; c++) w[r] += M[4 * r + c] * v[c];
    }
    for (int s = 0; s < 4; s++) st(a, idx[s], w[s]);
  }
}

/* Diagonal gates: a_x <- d[s(x)] a_x for every x, no pairing. */
void or_apply_d1(double *a, int n, int q, const double *d) {
  cplx d0 = mat(d, 0), d1 = mat(d, 1);
  int64_t N = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t x = 0; x < N; x++) st(a, (uint64_t)x, ((x >> q) & 1 ? d1 : d0) * ld(a, (uint64_t)x));
}

void or_apply_d2(double *a, int n, int q0, int q1, const double *d) {
  cplx dd[4];
  for (int s = 0; s < 4; s++) dd[s] = mat(d, s);
  int64_t N = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t x = 0; x < N; x++) {
    int s = (int)(((x >> q0) & 1) + 2 * ((x >> q1) & 1));
    st(a, (uint64_t)x, dd[s] * ld(a, (uint64_t)x));
  }
}

/* SWAP(q0, q1) exchanges the s=1 and s=2 amplitudes of each group; chunk_swap has the same
 * semantics ("As in the case of the usual swap gate"). */
void or_apply_swap(double *a, int n, int q0, int q1) {
  int64_t N = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t x = 0; x < N; x++) {
    uint64_t b0 = ((uint64_t)x >> q0) & 1, b1 = ((uint64_t)x >> q1) & 1;
    if (b0 == 1 && b1 == 0) {
      uint64_t y = ((uint64_t)x & ~(1ull << q0)) | (1ull << q1);
      double t0 = a[2 * x], t1 = a[2 * x + 1];
      a[2 * x] = a[2 * y];
      a[2 * x + 1] = a[2 * y + 1];
      a[2 * y] = t0;
      a[2 * y + 1] = t1;
    }
  }
}

/* Apply records in order.  Markers BEGIN/END are no-ops and CHUNK_SWAP is a SWAP, so a blocked
 * circuit (Listing 3 output) can be executed densely too.  Returns 0, or -1 on a bad record. */
int or_apply_circuit(double *a, int n, const or_gate *g, int64_t count) {
  for (int64_t i = 0; i < count; i++) {
    const or_gate *r = &g[i];
    int one = (r->kind == OR_U1 || r->kind == OR_D1);
    int two = (r->kind == OR_U2 || r->kind == OR_D2 || r->kind == OR_SWAP || r->kind == OR_CHUNK_SWAP);
    if (one && (r->q0 < 0 || r->q0 >= n)) return -1;
    if (two && (r->q0 < 0 || r->q0 >= n || r->q1 < 0 || r->q1 >= n || r->q0 == r->q1)) return -1;
    switch (r->kind) {
      case OR_U1: or_apply_1q(a, n, r->q0, r->m); break;
      case OR_U2: or_apply_2q(a, n, r->q0, r->q1, r->m); break;
      case OR_D1: or_apply_d1(a, n, r->q0, r->m); break;
      case OR_D2: or_apply_d2(a, n, r->q0, r->q1, r->m); break;
      case OR_SWAP:
      case OR_CHUNK_SWAP: or_apply_swap(a, n, r->q0, r->q1); break;
      case OR_BEGIN:
      case OR_END: break;
      default: return -1;
    }
  }
  return 0;
}

/* |k>: amplitude k = 1, all others 0 (dense analog). */
void or_init_basis(double *a, int n, uint64_t k) {
  memset(a, 0, sizeof(double) * 2 * ((size_t)1 << n));
  a[2 * k] = 1.0;
}

/* Un-permute (DESIGN R7): a_logical[x] = a_phys[sum_q bit_q(x) 2^{pi(q)}]. */
void or_unpermute(const double *phys, int n, const int32_t *pi, double *logical) {
  int64_t N = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t x = 0; x < N; x++) {
    uint64_t y = 0;
    for (int q = 0; q < n; q++) y |= (((uint64_t)x >> q) & 1) << pi[q];
    logical[2 * x] = phys[2 * y];
    logical[2 * x + 1] = phys[2 * y + 1];
  }
}

/* sum_x |a_x|^2, summed in index order by one thread (plainness over speed). */
double or_norm2(const double *a, int n) {
  int64_t N = (int64_t)1 << n;
  double s = 0.0;
  for (int64_t x = 0; x < N; x++) s += a[2 * x] * a[2 * x] + a[2 * x + 1] * a[2 * x + 1];
  return s;
}

/* DESIGN R17: p[y] = sum over x whose bits at Q equal y (Q[0] -> bit 0 of y) of |a_x|^2. */
void or_marginal(const double *a, int n, const int32_t *Q, int nq, double *p) {
  int64_t N = (int64_t)1 << n;
  memset(p, 0, sizeof(double) * ((size_t)1 << nq));
  for (int64_t x = 0; x < N; x++) {
    uint64_t y = 0;
    for (int i = 0; i < nq; i++) y |= (((uint64_t)x >> Q[i]) & 1) << i;
    p[y] += a[2 * x] * a[2 * x] + a[2 * x + 1] * a[2 * x + 1];
  }
}

/* DESIGN R16 sampling: for each uniform u (given by the caller), the first logical index x whose
 * running sum of |a|^2 (in index order) exceeds u.  us must be sorted ascending; a u beyond the
 * total mass maps to the last index with nonzero probability. */
void or_sample_sorted(const double *a, int n, const double *us, int64_t shots, uint64_t *out) {
  int64_t N = (int64_t)1 << n;
  double cum = 0.0;
  int64_t s = 0, last_nz = 0;
  for (int64_t x = 0; x < N && s < shots; x++) {
    double p = a[2 * x] * a[2 * x] + a[2 * x + 1] * a[2 * x + 1];
    if (p > 0) last_nz = x;
    cum += p;
    while (s < shots && us[s] < cum) out[s++] = (uint64_t)x;
  }
  while (s < shots) out[s++] = (uint64_t)last_nz;
}
