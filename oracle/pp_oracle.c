/*
 * pp_oracle.c -- plain, slow, obviously-correct CPU oracle for the PP-GNN
 * mini-batch loading hot path of arXiv 2504.13266 ("Graph Learning at Scale:
 * Characterizing and Optimizing Pre-Propagation GNNs", MLSys'25).
 *
 * THIS IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * path (paper_2504_13266_b200/, libppload.so) never links, imports or calls
 * anything in oracle/, and this file shares no code, header, table or
 * constant generator with the CUDA path.
 *
 * Every function cites the passage it follows.  "PAPER.md:L" is a line of the
 * paper's LaTeX source; "SPEC.md:L" a line of the desk-scale spec derived from
 * it; "§8(c) Ox" a row of the oracle table in SURVEY.md (the readings of the
 * paper adopted where the paper is silent are listed in DESIGN.md §3).
 *
 * Pins (what this oracle is checked against, see tests/test_oracle_*.py):
 *   philox        -- Random123 known-answer vectors (golden file) and, on a
 *                    B200, cuRAND's curand_Philox4x32_10 over 10^6 random
 *                    (ctr, key) pairs (tests/test_gpu_curand_pins.py).
 *   unit keys     -- the O5 word layout against cuRAND for seeds with both
 *                    halves nonzero and u >= 2^32 (same test file).
 *   unit keys /
 *   permutation   -- bijection, chi^2 uniformity over the 24 perms of n=4,
 *                    CR(c=1) == RR, chunk contiguity, numpy lexsort brute force.
 *   slicing       -- exactly-once coverage, SPEC size example [2,2,1].
 *   gather        -- per-row memcmp, identity prefix, integer column sums.
 *   casts         -- numpy/torch CPU conversions over large bit-pattern sweeps
 *                    plus hand-derived special values.
 *   propagation   -- dense fp64 matrix power (numpy), ring/complete/edgeless
 *                    closed forms, sqrt(d~) fixed point, SPEC worked values.
 *   generators    -- range/normality properties; the generator words against
 *                    cuRAND's Philox on the O11 counter layout (same test file).
 * Nothing here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PPO_OK 0
#define PPO_ERR 1

/* dtype codes used by this oracle's own API (not the product header). */
#define PPO_F32 0
#define PPO_BF16 1
#define PPO_F16 2

/* ------------------------------------------------------------------------ */
/* O4: Philox4x32-10 (Salmon et al., SC'11; Random123).  The paper names no   */
/* RNG; the north star fixes "a counter-based Philox stream".  Constants are  */
/* the published Philox4x32 multipliers and Weyl key increments.             */
/* ------------------------------------------------------------------------ */
void ppo_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { /* key schedule: bump before rounds 2..10 */
      k0 += W0;
      k1 += W1;
    }
    uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* O5: 64-bit sort key of shuffle unit u for epoch seed `seed`.
 * ctr = (u_lo, u_hi, 0, 0), key = (seed_lo, seed_hi), key64 = (y0<<32)|y1. */
uint64_t ppo_unit_key(uint64_t seed, uint64_t u) {
  uint32_t ctr[4] = {(uint32_t)u, (uint32_t)(u >> 32), 0u, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t y[4];
  ppo_philox4x32_10(ctr, key, y);
  return ((uint64_t)y[0] << 32) | (uint64_t)y[1];
}

void ppo_unit_keys(uint64_t seed, int64_t U, uint64_t* keys) {
  for (int64_t u = 0; u < U; ++u) keys[u] = ppo_unit_key(seed, (uint64_t)u);
}

/* Batch forms for the pin tests (loops over the functions above, no arithmetic of their own). */
void ppo_philox_batch(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
  for (int64_t i = 0; i < n; ++i) ppo_philox4x32_10(ctr + 4 * i, key + 2 * i, out + 4 * i);
}

void ppo_unit_key_batch(uint64_t seed, const uint64_t* u, int64_t n, uint64_t* keys) {
  for (int64_t i = 0; i < n; ++i) keys[i] = ppo_unit_key(seed, u[i]);
}

typedef struct {
  uint64_t key;
  int64_t unit;
} ppo_keyed_unit;

static int ppo_cmp_keyed(const void* a, const void* b) {
  const ppo_keyed_unit* x = (const ppo_keyed_unit*)a;
  const ppo_keyed_unit* y = (const ppo_keyed_unit*)b;
  if (x->key < y->key) return -1;
  if (x->key > y->key) return 1;
  if (x->unit < y->unit) return -1; /* O6 tie-break: smaller unit id first */
  if (x->unit > y->unit) return 1;
  return 0;
}

/* O6: pi = units sorted ascending by (key64, u).  SGD-RR draws "a uniformly
 * random permutation ... deterministic given seed". */
int ppo_unit_permutation(uint64_t seed, int64_t U, int64_t* pi) {
  if (U < 0) return PPO_ERR;
  if (U == 0) return PPO_OK;
  ppo_keyed_unit* tmp = (ppo_keyed_unit*)malloc((size_t)U * sizeof(ppo_keyed_unit));
  if (!tmp) return PPO_ERR;
  for (int64_t u = 0; u < U; ++u) {
    tmp[u].key = ppo_unit_key(seed, (uint64_t)u);
    tmp[u].unit = u;
  }
  qsort(tmp, (size_t)U, sizeof(ppo_keyed_unit), ppo_cmp_keyed);
  for (int64_t i = 0; i < U; ++i) pi[i] = tmp[i].unit;
  free(tmp);
  return PPO_OK;
}

/* O7: chunk expansion.  "reshuffle training data indices at the chunk level,
 * with each chunk comprising contiguous node features".
 * Chunk u covers positions [u*c, min(u*c+c, N)); order = concat over the
 * permuted chunks, ascending inside a chunk.  c = 1 is SGD-RR. */
int ppo_epoch_order(uint64_t seed, int64_t N, int64_t c, int64_t* order) {
  if (N < 0 || c < 1 || (N > 0 && c > N)) return PPO_ERR;
  if (N == 0) return PPO_OK;
  int64_t U = (N + c - 1) / c;
  int64_t* pi = (int64_t*)malloc((size_t)U * sizeof(int64_t));
  if (!pi) return PPO_ERR;
  if (ppo_unit_permutation(seed, U, pi) != PPO_OK) {
    free(pi);
    return PPO_ERR;
  }
  int64_t p = 0;
  for (int64_t i = 0; i < U; ++i) {
    int64_t begin = pi[i] * c;
    int64_t end = begin + c;
    if (end > N) end = N;
    for (int64_t v = begin; v < end; ++v) order[p++] = v;
  }
  free(pi);
  return (p == N) ? PPO_OK : PPO_ERR;
}

/* O8: with a node set S, positions index S: order'[p] = S[order[p]]
 * ("PP data proportional to the labelled nodes"). */
void ppo_apply_node_set(const int64_t* S, int64_t N, int64_t* order) {
  for (int64_t p = 0; p < N; ++p) order[p] = S[order[p]];
}

/* O9: batch slicing.  Rank r of W at step t takes
 * positions [t*W*B + r*B, min(t*W*B + (r+1)*B, N)).  drop_last keeps only
 * full steps.  Returns the number of steps in an epoch. */
int64_t ppo_num_steps(int64_t N, int64_t B, int32_t W, int32_t drop_last) {
  int64_t per = B * (int64_t)W;
  if (drop_last) return N / per;
  return (N + per - 1) / per;
}

void ppo_batch_range(int64_t N, int64_t B, int32_t W, int64_t t, int32_t r,
                     int64_t* start, int64_t* end) {
  int64_t s = t * (int64_t)W * B + (int64_t)r * B;
  int64_t e = s + B;
  if (s > N) s = N;
  if (e > N) e = N;
  *start = s;
  *end = e;
}

/* ------------------------------------------------------------------------ */
/* O10: round-to-nearest-even casts (north star: "fp32->bf16/fp16 cast fused", */
/* "including the round-to-nearest-even cast").  NaN -> 0x7FFF.   */
/* ------------------------------------------------------------------------ */
uint16_t ppo_f32_to_bf16(uint32_t x) {
  if ((x & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FFFu; /* any NaN */
  /* keep the top 16 bits, rounding the dropped 16 to nearest, ties to even */
  uint32_t lsb = (x >> 16) & 1u;
  uint32_t rounded = x + 0x7FFFu + lsb;
  return (uint16_t)(rounded >> 16);
}

/* IEEE-754 binary32 -> binary16, round to nearest, ties to even.
 * Overflow -> +-Inf, subnormal results kept (no flush), -0 kept. */
uint16_t ppo_f32_to_f16(uint32_t x) {
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t ax = x & 0x7FFFFFFFu;
  if (ax > 0x7F800000u) return 0x7FFFu;                     /* NaN */
  if (ax >= 0x477FF000u) return (uint16_t)(sign | 0x7C00u); /* >= 65520 or Inf -> Inf */
  if (ax >= 0x38800000u) {
    /* normal half: rebias exponent (127 -> 15) and drop 13 mantissa bits */
    uint32_t a = ax - (112u << 23);
    uint32_t lsb = (a >> 13) & 1u;
    uint32_t r = (a + 0x0FFFu + lsb) >> 13; /* carry may bump the exponent */
    return (uint16_t)(sign | r);
  }
  /* |x| < 2^-14: the result is a half subnormal (or zero), value m * 2^-24 */
  uint32_t e = ax >> 23;
  if (e < 102u) return (uint16_t)sign; /* |x| < 2^-25: rounds to zero */
  /* |x| = mant * 2^(e-150) with the implicit bit; in units of 2^-24 that is
   * mant * 2^(e-126), i.e. mant >> (126-e), shift in [14, 24] */
  uint32_t mant = (ax & 0x7FFFFFu) | 0x800000u;
  uint32_t shift = 126u - e;
  uint32_t q = mant >> shift;
  uint32_t rem = mant & ((1u << shift) - 1u);
  uint32_t half = 1u << (shift - 1u);
  if (rem > half || (rem == half && (q & 1u))) q += 1u;
  return (uint16_t)(sign | q);
}

void ppo_cast_bf16_array(const uint32_t* in, int64_t n, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = ppo_f32_to_bf16(in[i]);
}
void ppo_cast_f16_array(const uint32_t* in, int64_t n, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = ppo_f32_to_f16(in[i]);
}

/* O10: gather + cast.  out[j,k,f] = cast(X_k[rows[j], f]) with
 * elem(k, v, f) = X[k*hop_stride + v*row_stride + f] (any layout).
 * Batch assembly "copies the scattered node features" of the batch
 * (PAPER.md:259); out is [nrows, H, F] contiguous.  nthreads > 1 runs the
 * same loop under `omp parallel for` over batch rows (cpu_baseline only). */
int ppo_gather_cast(const void* X, int32_t in_dtype, int64_t hop_stride, int64_t row_stride,
                    int32_t H, int32_t F, const int64_t* rows, int64_t nrows,
                    int32_t out_dtype, void* out, int32_t nthreads) {
  if (in_dtype == PPO_F32) {
    const uint32_t* src = (const uint32_t*)X;
    if (out_dtype == PPO_F32) {
      uint32_t* dst = (uint32_t*)out;
#pragma omp parallel for num_threads(nthreads) schedule(static)
      for (int64_t j = 0; j < nrows; ++j)
        for (int32_t k = 0; k < H; ++k)
          for (int32_t f = 0; f < F; ++f)
            dst[(j * H + k) * F + f] = src[k * hop_stride + rows[j] * row_stride + f];
      return PPO_OK;
    }
    if (out_dtype == PPO_BF16 || out_dtype == PPO_F16) {
      uint16_t* dst = (uint16_t*)out;
      int to_bf16 = (out_dtype == PPO_BF16);
#pragma omp parallel for num_threads(nthreads) schedule(static)
      for (int64_t j = 0; j < nrows; ++j)
        for (int32_t k = 0; k < H; ++k)
          for (int32_t f = 0; f < F; ++f) {
            uint32_t x = src[k * hop_stride + rows[j] * row_stride + f];
            dst[(j * H + k) * F + f] = to_bf16 ? ppo_f32_to_bf16(x) : ppo_f32_to_f16(x);
          }
      return PPO_OK;
    }
    return PPO_ERR;
  }
  if ((in_dtype == PPO_BF16 || in_dtype == PPO_F16) && out_dtype == in_dtype) {
    /* 16-bit store, same 16-bit output: a bit copy */
    const uint16_t* src = (const uint16_t*)X;
    uint16_t* dst = (uint16_t*)out;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t j = 0; j < nrows; ++j)
      for (int32_t k = 0; k < H; ++k)
        for (int32_t f = 0; f < F; ++f)
          dst[(j * H + k) * F + f] = src[k * hop_stride + rows[j] * row_stride + f];
    return PPO_OK;
  }
  return PPO_ERR;
}

/* Labels and node ids of a batch (SPEC.md:242-246 Batch contents). */
void ppo_gather_labels(const int32_t* labels, const int64_t* rows, int64_t nrows, int32_t* out) {
  for (int64_t j = 0; j < nrows; ++j) out[j] = labels[rows[j]];
}

/* ------------------------------------------------------------------------ */
/* A0 (precondition, not on the timed path): Eq. (2) propagation.             */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t a, b;
} ppo_edge;

static int ppo_cmp_edge(const void* x, const void* y) {
  const ppo_edge* p = (const ppo_edge*)x;
  const ppo_edge* q = (const ppo_edge*)y;
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  if (p->b != q->b) return p->b < q->b ? -1 : 1;
  return 0;
}

/* O1: graph -> CSR of A~ = I + A ("A~ = I + A is the adjacency
 * matrix with self-loops").  Readings: input self loops dropped, duplicate
 * edges merged, edges symmetrised (undirected), then the diagonal added, so
 * A~ has exactly one 1 on every diagonal entry.  Columns ascending per row.
 * Two calls: first with col_idx == NULL to get the nnz count into *nnz_out. */
int ppo_build_csr(int64_t n, const int64_t* src, const int64_t* dst, int64_t m,
                  int64_t* row_ptr, int64_t* col_idx, int64_t* nnz_out) {
  if (n < 0 || m < 0) return PPO_ERR;
  int64_t cap = 2 * m + n;
  ppo_edge* e = (ppo_edge*)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(ppo_edge));
  if (!e) return PPO_ERR;
  int64_t ne = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) {
      free(e);
      return PPO_ERR;
    }
    if (src[i] == dst[i]) continue; /* drop input self loops */
    e[ne].a = src[i]; e[ne].b = dst[i]; ++ne;
    e[ne].a = dst[i]; e[ne].b = src[i]; ++ne; /* symmetrise */
  }
  for (int64_t i = 0; i < n; ++i) { /* add I */
    e[ne].a = i; e[ne].b = i; ++ne;
  }
  qsort(e, (size_t)ne, sizeof(ppo_edge), ppo_cmp_edge);
  int64_t nnz = 0;
  for (int64_t i = 0; i < ne; ++i) { /* dedup */
    if (nnz > 0 && e[nnz - 1].a == e[i].a && e[nnz - 1].b == e[i].b) continue;
    e[nnz++] = e[i];
  }
  *nnz_out = nnz;
  if (col_idx != NULL) {
    for (int64_t i = 0; i <= n; ++i) row_ptr[i] = 0;
    for (int64_t i = 0; i < nnz; ++i) row_ptr[e[i].a + 1] += 1;
    for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
    for (int64_t i = 0; i < nnz; ++i) col_idx[i] = e[i].b;
  }
  free(e);
  return PPO_OK;
}

/* O2: w_ij = 1/sqrt(d~_i d~_j) with d~_i = row length of A~ (neighbours + 1),
 * i.e. B = D~^{-1/2} A~ D~^{-1/2}. */
void ppo_operator_values(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, double* val) {
  for (int64_t i = 0; i < n; ++i) {
    double di = (double)(row_ptr[i + 1] - row_ptr[i]);
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      int64_t j = col_idx[p];
      double dj = (double)(row_ptr[j + 1] - row_ptr[j]);
      val[p] = 1.0 / sqrt(di * dj);
    }
  }
}

/* O3: one SpMM, Y = B X (Eq. (2), "multiplying the operators
 * with the node feature matrix").  fp64 accumulation in ascending column
 * order, fp32 store.  X, Y are [n, F] row-major fp32. */
void ppo_spmm(int64_t n, int32_t F, const int64_t* row_ptr, const int64_t* col_idx,
              const double* val, const float* X, float* Y) {
  for (int64_t i = 0; i < n; ++i)
    for (int32_t f = 0; f < F; ++f) {
      double acc = 0.0;
      for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
        acc += val[p] * (double)X[col_idx[p] * (int64_t)F + f];
      Y[i * (int64_t)F + f] = (float)acc;
    }
}

/* Eq. (2): S = {X, BX, ..., B^K X}.  hops is [K+1, n, F] (hop-major);
 * hops[0] is a bit copy of X and hop k is computed from the fp32 hop k-1. */
void ppo_propagate(int64_t n, int32_t F, const int64_t* row_ptr, const int64_t* col_idx,
                   const double* val, const float* X, int32_t K, float* hops) {
  int64_t nf = n * (int64_t)F;
  memcpy(hops, X, (size_t)nf * sizeof(float));
  for (int32_t k = 1; k <= K; ++k)
    ppo_spmm(n, F, row_ptr, col_idx, val, hops + (int64_t)(k - 1) * nf, hops + (int64_t)k * nf);
}

/* ------------------------------------------------------------------------ */
/* O11: synthetic inputs; values are a pure function of     */
/* (data_seed, k, v, f) so any row of a TB-scale store can be regenerated.    */
/* ------------------------------------------------------------------------ */

/* word (f & 3) of Philox(ctr=(v_lo, v_hi, (k<<16)|(f>>2), 0x50504746), key=seed) */
static uint32_t ppo_gen_word(uint64_t seed, int64_t k, int64_t v, int64_t f) {
  uint32_t ctr[4] = {(uint32_t)(uint64_t)v, (uint32_t)((uint64_t)v >> 32),
                     (uint32_t)(((uint64_t)k << 16) | ((uint64_t)f >> 2)), 0x50504746u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t y[4];
  ppo_philox4x32_10(ctr, key, y);
  return y[f & 3];
}

/* G: random sign, random 23-bit mantissa, exponent field 120..135 */
uint32_t ppo_gen_f32_bits(uint64_t seed, int64_t k, int64_t v, int64_t f) {
  uint32_t w = ppo_gen_word(seed, k, v, f);
  return (w & 0x807FFFFFu) | ((120u + ((w >> 23) & 15u)) << 23);
}

/* G16: random sign, random 10-bit mantissa, exponent field 8..23 */
uint16_t ppo_gen_f16_bits(uint64_t seed, int64_t k, int64_t v, int64_t f) {
  uint32_t w = ppo_gen_word(seed, k, v, f);
  return (uint16_t)((w & 0x83FFu) | ((8u + ((w >> 10) & 15u)) << 10));
}

/* Rows `rows[0..nrows)` of the synthetic store, written node-major
 * [nrows, H, F] (dtype PPO_F32 -> G, PPO_F16 -> G16). */
int ppo_gen_rows(uint64_t seed, int32_t dtype, int32_t H, int32_t F, const int64_t* rows,
                 int64_t nrows, void* out, int32_t nthreads) {
  if (dtype == PPO_F32) {
    uint32_t* o = (uint32_t*)out;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t j = 0; j < nrows; ++j)
      for (int32_t k = 0; k < H; ++k)
        for (int32_t f = 0; f < F; ++f)
          o[(j * H + k) * F + f] = ppo_gen_f32_bits(seed, k, rows[j], f);
    return PPO_OK;
  }
  if (dtype == PPO_F16) {
    uint16_t* o = (uint16_t*)out;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t j = 0; j < nrows; ++j)
      for (int32_t k = 0; k < H; ++k)
        for (int32_t f = 0; f < F; ++f)
          o[(j * H + k) * F + f] = ppo_gen_f16_bits(seed, k, rows[j], f);
    return PPO_OK;
  }
  return PPO_ERR;
}

/* Config-1 graph: edge draw i uses
 * (y0, y1) = Philox(ctr=(i_lo, i_hi, 0, 0x45444745), key=seed); a = y0 mod n,
 * b = y1 mod n; loops and already-drawn undirected pairs are skipped; stops
 * at m distinct edges.  Duplicate check is a plain linear-probing set. */
int ppo_gen_graph(uint64_t seed, int64_t n, int64_t m, int64_t* src, int64_t* dst) {
  if (n < 2 || m < 0 || m > n * (n - 1) / 2) return PPO_ERR;
  int64_t cap = 1;
  while (cap < 4 * m + 16) cap <<= 1;
  uint64_t* set = (uint64_t*)malloc((size_t)cap * sizeof(uint64_t));
  if (!set) return PPO_ERR;
  for (int64_t i = 0; i < cap; ++i) set[i] = UINT64_MAX;
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  int64_t got = 0;
  for (uint64_t i = 0; got < m; ++i) {
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0u, 0x45444745u};
    uint32_t y[4];
    ppo_philox4x32_10(ctr, key, y);
    int64_t a = (int64_t)(y[0] % (uint64_t)n);
    int64_t b = (int64_t)(y[1] % (uint64_t)n);
    if (a == b) continue;
    int64_t lo = a < b ? a : b, hi = a < b ? b : a;
    uint64_t code = (uint64_t)lo * (uint64_t)n + (uint64_t)hi;
    uint64_t h = (code * 0x9E3779B97F4A7C15ull) & (uint64_t)(cap - 1);
    int dup = 0;
    while (set[h] != UINT64_MAX) {
      if (set[h] == code) { dup = 1; break; }
      h = (h + 1) & (uint64_t)(cap - 1);
    }
    if (dup) continue;
    set[h] = code;
    src[got] = a;
    dst[got] = b;
    ++got;
  }
  free(set);
  return PPO_OK;
}
