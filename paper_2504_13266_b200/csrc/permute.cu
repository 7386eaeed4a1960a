// Epoch permutation kernels (K1/K2 of §2.3).
//
// pi = argsort of the units' 64-bit Philox keys, ties broken by unit id
// (SGD-RR: a uniformly random permutation every epoch; chunk
// reshuffling permutes chunk ids the same way).
//
// B200 design: an MSD bucket sort that never stores the keys.
//   1. k_hist     -- key(u) recomputed from the counter-based stream; top
//                    `bits` bits pick one of 2^bits buckets (mean ~20 units).
//   2. k_scan_*   -- exclusive scan of the bucket counts (3 kernels).
//   3. k_scatter  -- key(u) recomputed again, unit id appended to its bucket
//                    (arbitrary order inside a bucket: atomics).
//   4. k_bucket_rank -- one warp per bucket: keys recomputed, each unit's
//                    final rank inside the bucket counted with warp shuffles
//                    over (key, id) pairs, unit written to pi[offset + rank].
//                    The result is unique, so the atomics' order never shows.
// HBM traffic ~12 B/unit (tmp write + read, pi write) plus the counts; the
// Philox work is ALU, tiny next to the gather.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.h"
#include "philox.cuh"

namespace ppl {

int sort_bucket_bits(uint64_t U, int delta) {
  int bits = 0;
  // largest bits with U / 2^bits >= ~20 (mean bucket between 14 and 28 units)
  while (bits < 24 && (U >> (bits + 1)) >= 20) ++bits;
  if ((U >> bits) >= 28 && bits < 24) ++bits;
  bits += delta;
  if (bits < 0) bits = 0;
  if (bits > 24) bits = 24;
  return bits;
}

__device__ __forceinline__ uint32_t bucket_of(uint64_t key, int bits) {
  return bits == 0 ? 0u : static_cast<uint32_t>(key >> (64 - bits));
}

__global__ void k_hist(uint64_t seed, uint32_t U, int bits, uint32_t* __restrict__ counts) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
    atomicAdd(&counts[bucket_of(unit_sort_key(seed, u), bits)], 1u);
  }
}

// --- block-wide exclusive scan of kScanTile = 4 x 1024 values -------------------
constexpr int kScanThreads = 1024;

__device__ __forceinline__ uint32_t block_exclusive_scan4(uint32_t v[4], uint32_t* smem_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t s0 = v[0], s1 = s0 + v[1], s2 = s1 + v[2], s3 = s2 + v[3];
  uint32_t incl = s3;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) smem_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = smem_warp[lane];  // 32 warps
    uint32_t wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += y;
    }
    smem_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) smem_warp[32] = wi;
  }
  __syncthreads();
  const uint32_t base = smem_warp[warp] + incl - s3;
  total = smem_warp[32];
  v[0] = base;
  v[1] = base + s0;
  v[2] = base + s1;
  v[3] = base + s2;
  return base;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* __restrict__ in, uint32_t n,
                                                              uint32_t* __restrict__ blocksums) {
  __shared__ uint32_t red[32];
  const uint32_t i0 = blockIdx.x * kScanTile + threadIdx.x * 4;
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) s += (i0 + q < n) ? in[i0 + q] : 0u;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t w = red[threadIdx.x];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) w += __shfl_xor_sync(0xffffffffu, w, d);
    if (threadIdx.x == 0) blocksums[blockIdx.x] = w;
  }
}

// one block: exclusive scan of blocksums[0..nblk) in place
__global__ void __launch_bounds__(kScanThreads) k_scan_top(uint32_t* __restrict__ blocksums, uint32_t nblk) {
  __shared__ uint32_t sw[33];
  uint32_t carry = 0;
  for (uint32_t base = 0; base < nblk; base += kScanTile) {
    uint32_t v[4];
    const uint32_t i0 = base + threadIdx.x * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = (i0 + q < nblk) ? blocksums[i0 + q] : 0u;
    uint32_t total;
    block_exclusive_scan4(v, sw, total);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + q < nblk) blocksums[i0 + q] = v[q] + carry;
    carry += total;
    __syncthreads();
  }
}

// counts[i] <- exclusive prefix (in place), cursor[i] <- same (i < n - 1)
__global__ void __launch_bounds__(kScanThreads) k_scan_down(uint32_t* __restrict__ counts, uint32_t n,
                                                            const uint32_t* __restrict__ blocksums,
                                                            uint32_t* __restrict__ cursor) {
  __shared__ uint32_t sw[33];
  const uint32_t i0 = blockIdx.x * kScanTile + threadIdx.x * 4;
  uint32_t v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = (i0 + q < n) ? counts[i0 + q] : 0u;
  uint32_t total;
  block_exclusive_scan4(v, sw, total);
  const uint32_t off = blocksums[blockIdx.x];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (i0 + q < n) {
      counts[i0 + q] = v[q] + off;
      if (cursor != nullptr && i0 + q + 1 < n) cursor[i0 + q] = v[q] + off;
    }
  }
}

// Four units per thread per trip so four returning atomics are in flight.
constexpr int kScatterIlp = 4;

__global__ void k_scatter(uint64_t seed, uint32_t U, int bits, uint32_t* __restrict__ cursor,
                          uint32_t* __restrict__ tmp) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t u0 = blockIdx.x * blockDim.x + threadIdx.x; u0 < U; u0 += stride * kScatterIlp) {
    uint32_t slot[kScatterIlp];
#pragma unroll
    for (int q = 0; q < kScatterIlp; ++q) {
      const uint32_t u = u0 + q * stride;
      if (u < U) slot[q] = atomicAdd(&cursor[bucket_of(unit_sort_key(seed, u), bits)], 1u);
    }
#pragma unroll
    for (int q = 0; q < kScatterIlp; ++q) {
      const uint32_t u = u0 + q * stride;
      if (u < U) tmp[slot[q]] = u;
    }
  }
}

// One warp per bucket.  Lane l holds unit i = ibase + l; its rank is the
// number of (key, id) pairs in the bucket that compare below its own, counted
// by broadcasting candidates with __shfl_sync.  Buckets of <= 32 units (all
// but ~0.3 %) compare only the 32 key bits below the bucket prefix, falling
// back to the full (key, id) order when two of them tie; larger buckets use
// tiles of 32 x 32 with full compares.
__global__ void __launch_bounds__(256) k_bucket_rank(uint64_t seed, const uint32_t* __restrict__ offsets,
                                                     uint32_t nb, int bits, uint32_t k32_mask,
                                                     const uint32_t* __restrict__ tmp,
                                                     uint32_t* __restrict__ pi) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  // Software pipeline over this warp's buckets (several per warp when the grid is capped, as
  // for the prefetched permutation): the offsets of the bucket after next and the unit ids of
  // the next bucket are loaded while the current one is ranked.
  const uint32_t first = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  auto load_range = [&](uint32_t b, uint32_t& beg_, uint32_t& n_) {
    beg_ = 0;
    n_ = 0;
    if (b < nb) {
      beg_ = offsets[b];
      n_ = offsets[b + 1] - beg_;
    }
  };
  uint32_t beg_cur, n_cur, beg_nxt, n_nxt;
  load_range(first, beg_cur, n_cur);
  load_range(first + nwarps, beg_nxt, n_nxt);
  uint32_t ui_cur = (lane < static_cast<int>(n_cur) && n_cur <= 32) ? tmp[beg_cur + lane] : 0xffffffffu;
  for (uint32_t bucket = first; bucket < nb; bucket += nwarps) {
  const uint32_t beg = beg_cur, n = n_cur, ui_pre = ui_cur;
  ui_cur = (lane < static_cast<int>(n_nxt) && n_nxt <= 32) ? tmp[beg_nxt + lane] : 0xffffffffu;
  beg_cur = beg_nxt;
  n_cur = n_nxt;
  load_range(bucket + 2 * nwarps, beg_nxt, n_nxt);
  if (n <= 32) {
    const bool vi = lane < static_cast<int>(n);
    const uint32_t ui = ui_pre;
    const uint64_t ki = vi ? unit_sort_key(seed, ui) : ~0ull;
    const uint32_t k32 = static_cast<uint32_t>((ki << bits) >> 32) & k32_mask;  // bits below the bucket prefix
    uint32_t rank = 0, eq = 0;
#pragma unroll 4
    for (uint32_t s = 0; s < n; ++s) {
      const uint32_t kk = __shfl_sync(0xffffffffu, k32, s);
      rank += kk < k32;
      eq += kk == k32;
    }
    if (__any_sync(0xffffffffu, vi && eq > 1)) {  // a 32-bit tie: full (key, id) order
      rank = 0;
      for (uint32_t s = 0; s < n; ++s) {
        const uint64_t kk = __shfl_sync(0xffffffffu, ki, s);
        const uint32_t uu = __shfl_sync(0xffffffffu, ui, s);
        rank += (kk < ki) | ((kk == ki) & (uu < ui));
      }
    }
    if (vi) pi[beg + rank] = ui;
    continue;
  }
  for (uint32_t ibase = 0; ibase < n; ibase += 32) {
    const bool vi = ibase + lane < n;
    const uint32_t ui = vi ? tmp[beg + ibase + lane] : 0xffffffffu;
    const uint64_t ki = vi ? unit_sort_key(seed, ui) : ~0ull;
    uint32_t rank = 0;
    for (uint32_t jbase = 0; jbase < n; jbase += 32) {
      uint32_t uj;
      uint64_t kj;
      if (jbase == ibase) {
        uj = ui;
        kj = ki;
      } else {
        const bool vj = jbase + lane < n;
        uj = vj ? tmp[beg + jbase + lane] : 0xffffffffu;
        kj = vj ? unit_sort_key(seed, uj) : ~0ull;
      }
      const uint32_t m = min(32u, n - jbase);
      for (uint32_t s = 0; s < m; ++s) {
        const uint64_t kk = __shfl_sync(0xffffffffu, kj, s);
        const uint32_t uu = __shfl_sync(0xffffffffu, uj, s);
        rank += (kk < ki) | ((kk == ki) & (uu < ui));
      }
    }
    if (vi) pi[beg + rank] = ui;
  }
  }  // bucket loop
}

// K2: small unit counts (chunk reshuffling: U = ceil(N / c), e.g. 299 chunks of
// 8192 products rows) -- one CTA computes every key into shared memory and
// bitonic-sorts the (key, id) pairs; padding sorts last.  Also records where
// the ragged chunk U-1 landed (needed by the chunk expansion).
constexpr uint32_t kCtaSortMax = 4096;
constexpr int kCtaSortThreads = 1024;

__global__ void __launch_bounds__(kCtaSortThreads) k_cta_sort(uint64_t seed, uint32_t U, uint32_t P,
                                                              uint32_t* __restrict__ pi,
                                                              uint32_t* __restrict__ ragged) {
  extern __shared__ uint64_t smem_keys[];
  uint32_t* ids = reinterpret_cast<uint32_t*>(smem_keys + P);
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
    smem_keys[i] = i < U ? unit_sort_key(seed, i) : ~0ull;
    ids[i] = i < U ? i : 0xffffffffu;
  }
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const uint64_t ka = smem_keys[i], kb = smem_keys[l];
          const uint32_t ia = ids[i], ib = ids[l];
          const bool a_gt_b = (ka > kb) || (ka == kb && ia > ib);
          if (a_gt_b == ((i & k) == 0)) {
            smem_keys[i] = kb;
            smem_keys[l] = ka;
            ids[i] = ib;
            ids[l] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < U; i += blockDim.x) {
    pi[i] = ids[i];
    if (ragged != nullptr && ids[i] == U - 1) *ragged = i;
  }
}

// Local shuffle: local row lr -> global node lr * W + r, in place.
__global__ void k_local_to_global(uint32_t* __restrict__ order, int64_t n, uint32_t W, uint32_t r) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    order[p] = order[p] * W + r;
}

cudaError_t launch_local_to_global(uint32_t* order, int64_t n, int32_t W, int32_t r, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_local_to_global<<<std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(order, n, W, r);
  return cudaGetLastError();
}

// Position of the ragged (last) chunk U-1 inside pi.
__global__ void k_find_ragged(const uint32_t* __restrict__ pi, uint32_t U, uint32_t* __restrict__ ragged) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < U; i += gridDim.x * blockDim.x)
    if (pi[i] == U - 1) *ragged = i;
}

// ---- two-level radix path (4096 < U <= 2^23): no global atomics -------------
// Level 1: CTA tiles of kL1Tile units histogram the top b1 key bits in shared
// memory; a digit-major scan of the per-tile counts gives every tile its own
// output offsets, so the scatter needs only shared-memory atomics.  Level 2:
// one CTA per level-1 bucket (~1-2 K units) reloads its units, counting-sorts
// them in shared memory by the next b2 bits into sub-buckets of ~8, and ranks
// each unit inside its sub-bucket by full (key, id).  The order produced by
// the atomics never shows: every rank is unique.
constexpr uint32_t kL1Tile = 8192;
constexpr int kL1Threads = 512;
constexpr int kL2Threads = 256;
constexpr uint32_t kL2Cap = 2048;         // units of one level-1 bucket held in shared memory
constexpr uint32_t kTwoLevelMaxU = 1u << 22;  // b1 <= 12 keeps the mean bucket <= 1024 (cap = mean + 32 sigma)

struct TwoLevel {
  int b1, b2;
  uint32_t ntiles;
};
static TwoLevel two_level_shape(uint32_t U) {
  TwoLevel t{};
  int b1 = 1;
  while (b1 < 12 && (U >> b1) > 1024) ++b1;  // mean level-1 bucket <= 1024 units
  const uint32_t mean = U >> b1;
  int b2 = 0;
  while (b2 < 10 && (mean >> (b2 + 1)) >= 8) ++b2;  // sub-buckets of ~8-16 units
  t.b1 = b1;
  t.b2 = b2;
  t.ntiles = (U + kL1Tile - 1) / kL1Tile;
  return t;
}

size_t two_level_hist_entries(uint64_t U) {
  if (U <= kCtaSortMax || U > kTwoLevelMaxU) return 0;
  const TwoLevel t = two_level_shape(static_cast<uint32_t>(U));
  return (static_cast<size_t>(1) << t.b1) * t.ntiles + 1;
}

__global__ void __launch_bounds__(kL1Threads) k_l1_hist(uint64_t seed, uint32_t U, int b1, uint32_t ntiles,
                                                         uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t s_hist[];
  const uint32_t nd = 1u << b1;
  for (uint32_t d = threadIdx.x; d < nd; d += blockDim.x) s_hist[d] = 0;
  __syncthreads();
  const uint32_t u0 = blockIdx.x * kL1Tile;
  for (uint32_t u = u0 + threadIdx.x; u < min(U, u0 + kL1Tile); u += blockDim.x)
    atomicAdd(&s_hist[static_cast<uint32_t>(unit_sort_key(seed, u) >> (64 - b1))], 1u);
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < nd; d += blockDim.x) hist[d * ntiles + blockIdx.x] = s_hist[d];
}

__global__ void __launch_bounds__(kL1Threads) k_l1_scatter(uint64_t seed, uint32_t U, int b1, uint32_t ntiles,
                                                            const uint32_t* __restrict__ offs,
                                                            uint32_t* __restrict__ tmp) {
  extern __shared__ uint32_t s_cur[];
  const uint32_t nd = 1u << b1;
  for (uint32_t d = threadIdx.x; d < nd; d += blockDim.x) s_cur[d] = offs[d * ntiles + blockIdx.x];
  __syncthreads();
  const uint32_t u0 = blockIdx.x * kL1Tile;
  for (uint32_t u = u0 + threadIdx.x; u < min(U, u0 + kL1Tile); u += blockDim.x) {
    const uint32_t slot = atomicAdd(&s_cur[static_cast<uint32_t>(unit_sort_key(seed, u) >> (64 - b1))], 1u);
    tmp[slot] = u;
  }
}

// One CTA per level-1 bucket.  Buckets larger than kL2Cap (a > 40-sigma event
// for the chosen means) fall back to a warp ranking straight from global memory.
__global__ void __launch_bounds__(kL2Threads) k_l2_sort(uint64_t seed, int b1, int b2, uint32_t ntiles, uint32_t U,
                                                         uint32_t cap,
                                                         const uint32_t* __restrict__ offs,
                                                         const uint32_t* __restrict__ tmp, uint32_t* __restrict__ pi) {
  __shared__ uint64_t s_key[kL2Cap];
  __shared__ uint32_t s_u[kL2Cap];
  __shared__ uint16_t s_perm[kL2Cap];
  __shared__ uint32_t s_cnt[1025], s_off[1025];
  const uint32_t d = blockIdx.x, nd = 1u << b1;
  const uint32_t beg = offs[d * ntiles];
  const uint32_t end = d + 1 < nd ? offs[(d + 1) * ntiles] : U;
  const uint32_t n = end - beg;
  if (n == 0) return;
  if (n > cap) {  // generic fallback: warp 0 ranks by full (key, id), tiles of 32 x 32
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    for (uint32_t ibase = 0; ibase < n; ibase += 32) {
      const bool vi = ibase + lane < n;
      const uint32_t ui = vi ? tmp[beg + ibase + lane] : 0xffffffffu;
      const uint64_t ki = vi ? unit_sort_key(seed, ui) : ~0ull;
      uint32_t rank = 0;
      for (uint32_t jbase = 0; jbase < n; jbase += 32) {
        const bool vj = jbase + lane < n;
        const uint32_t uj = vj ? tmp[beg + jbase + lane] : 0xffffffffu;
        const uint64_t kj = vj ? unit_sort_key(seed, uj) : ~0ull;
        const uint32_t m = min(32u, n - jbase);
        for (uint32_t s = 0; s < m; ++s) {
          const uint64_t kk = __shfl_sync(0xffffffffu, kj, s);
          const uint32_t uu = __shfl_sync(0xffffffffu, uj, s);
          rank += (kk < ki) | ((kk == ki) & (uu < ui));
        }
      }
      if (vi) pi[beg + rank] = ui;
    }
    return;
  }
  const uint32_t ns = 1u << b2;
  for (uint32_t s = threadIdx.x; s <= ns; s += blockDim.x) s_cnt[s] = 0;
  __syncthreads();
  const int shift = 64 - b1 - b2;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t u = tmp[beg + i];
    const uint64_t key = unit_sort_key(seed, u);
    s_key[i] = key;
    s_u[i] = u;
    atomicAdd(&s_cnt[b2 ? static_cast<uint32_t>((key << b1) >> (64 - b2)) : 0u], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan of <= 1024 sub-bucket counts
    uint32_t acc = 0;
    for (uint32_t s = 0; s < ns; ++s) {
      s_off[s] = acc;
      acc += s_cnt[s];
      s_cnt[s] = s_off[s];  // reuse as scatter cursor
    }
    s_off[ns] = acc;
  }
  __syncthreads();
  (void)shift;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t sb = b2 ? static_cast<uint32_t>((s_key[i] << b1) >> (64 - b2)) : 0u;
    s_perm[atomicAdd(&s_cnt[sb], 1u)] = static_cast<uint16_t>(i);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t ki = s_key[i];
    const uint32_t ui = s_u[i];
    const uint32_t sb = b2 ? static_cast<uint32_t>((ki << b1) >> (64 - b2)) : 0u;
    const uint32_t lo = s_off[sb], hi = s_off[sb + 1];
    uint32_t rank = 0;
    for (uint32_t p = lo; p < hi; ++p) {
      const uint32_t j = s_perm[p];
      const uint64_t kj = s_key[j];
      rank += (kj < ki) | ((kj == ki) & (s_u[j] < ui));
    }
    pi[beg + lo + rank] = ui;
  }
}

static cudaError_t launch_two_level(uint64_t seed, uint32_t U, const SortScratch& s, uint32_t* pi,
                                    cudaStream_t st) {
  const TwoLevel t = two_level_shape(U);
  const uint32_t nd = 1u << t.b1;
  const uint32_t n = nd * t.ntiles + 1;  // hist[n-1] = 0 -> offs[n-1] = U
  cudaError_t e = cudaMemsetAsync(s.hist + (n - 1), 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  k_l1_hist<<<t.ntiles, kL1Threads, nd * 4, st>>>(seed, U, t.b1, t.ntiles, s.hist);
  const uint32_t nblk = (n + kScanTile - 1) / kScanTile;
  k_scan_reduce<<<nblk, kScanThreads, 0, st>>>(s.hist, n, s.blocksums);
  k_scan_top<<<1, kScanThreads, 0, st>>>(s.blocksums, nblk);
  k_scan_down<<<nblk, kScanThreads, 0, st>>>(s.hist, n, s.blocksums, nullptr);
  k_l1_scatter<<<t.ntiles, kL1Threads, nd * 4, st>>>(seed, U, t.b1, t.ntiles, s.hist, s.tmp);
  k_l2_sort<<<nd, kL2Threads, 0, st>>>(seed, t.b1, t.b2, t.ntiles, U, std::min(kL2Cap, s.l2_cap), s.hist, s.tmp,
                                       pi);
  return cudaGetLastError();
}

cudaError_t launch_unit_permutation(uint64_t seed, uint32_t U, int bits, bool allow_cta, const SortScratch& s, uint32_t* pi,
                                    uint32_t* ragged, cudaStream_t st) {
  if (U == 0) return cudaSuccess;
  if (U <= kCtaSortMax && allow_cta) {
    uint32_t P = 1;
    while (P < U) P <<= 1;
    k_cta_sort<<<1, kCtaSortThreads, P * 12, st>>>(seed, U, P, pi, ragged);
    return cudaGetLastError();
  }
  if (allow_cta && s.two_level && s.hist != nullptr && two_level_hist_entries(U) != 0 &&
      two_level_hist_entries(U) <= s.hist_cap) {
    cudaError_t e = launch_two_level(seed, U, s, pi, st);
    if (e == cudaSuccess && ragged != nullptr)
      k_find_ragged<<<std::min<uint32_t>((U + 255) / 256, 148u * 8u), 256, 0, st>>>(pi, U, ragged);
    return e == cudaSuccess ? cudaGetLastError() : e;
  }
  const uint32_t nb = 1u << bits;
  const uint32_t n = nb + 1;  // counts[nb] = 0 -> offsets[nb] = U
  cudaError_t e = cudaMemsetAsync(s.counts, 0, sizeof(uint32_t) * n, st);
  if (e != cudaSuccess) return e;
  const int threads = 256;
  // s.grid_cap > 0 (prefetch on the side stream): confine the grid-stride kernels to
  // fewer CTAs so they leave most SMs to the concurrently running gathers
  const uint32_t cap = s.grid_cap > 0 ? static_cast<uint32_t>(s.grid_cap) : 148u * 16u;
  const uint32_t unit_blocks = std::min<uint32_t>((U + threads - 1) / threads, cap);
  k_hist<<<unit_blocks, threads, 0, st>>>(seed, U, bits, s.counts);
  const uint32_t nblk = (n + kScanTile - 1) / kScanTile;
  k_scan_reduce<<<nblk, kScanThreads, 0, st>>>(s.counts, n, s.blocksums);
  k_scan_top<<<1, kScanThreads, 0, st>>>(s.blocksums, nblk);
  k_scan_down<<<nblk, kScanThreads, 0, st>>>(s.counts, n, s.blocksums, s.cursor);
  k_scatter<<<unit_blocks, threads, 0, st>>>(seed, U, bits, s.cursor, s.tmp);
  const uint64_t rank_blocks = (static_cast<uint64_t>(nb) * 32 + 255) / 256;
  k_bucket_rank<<<static_cast<uint32_t>(std::min<uint64_t>(rank_blocks, s.grid_cap > 0 ? cap : rank_blocks)), 256,
                  0, st>>>(seed, s.counts, nb, bits, s.k32_mask, s.tmp, pi);
  if (ragged != nullptr) k_find_ragged<<<std::min<uint32_t>((U + 255) / 256, 148u * 8u), 256, 0, st>>>(pi, U, ragged);
  return cudaGetLastError();
}

// order = concat over i of [pi_i * c, min(pi_i * c + c, N)) (oracle step O7).
// Chunks before the ragged one start at i*c, the ragged chunk (length ls)
// sits at r*c, chunks after it start at i*c - (c - ls).
__global__ void k_chunk_expand(const uint32_t* __restrict__ pi, uint64_t N, uint64_t c, uint64_t ls,
                               const uint32_t* __restrict__ ragged, uint32_t* __restrict__ order) {
  // ragged = position of chunk U-1 in pi (written by the permutation launch)
  const uint64_t r = *ragged;
  const uint64_t rag_begin = r * c;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < N;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t i, off;
    if (p < rag_begin) {
      i = p / c;
      off = p - i * c;
    } else if (p < rag_begin + ls) {
      i = r;
      off = p - rag_begin;
    } else {
      const uint64_t q = p - rag_begin - ls;
      const uint64_t qi = q / c;
      i = r + 1 + qi;
      off = q - qi * c;
    }
    order[p] = static_cast<uint32_t>(static_cast<uint64_t>(pi[i]) * c + off);
  }
}

cudaError_t launch_chunk_expand(const uint32_t* pi, uint32_t U, uint64_t N, uint64_t c, const uint32_t* ragged,
                                uint32_t* order, cudaStream_t st) {
  if (N == 0) return cudaSuccess;
  const uint64_t ls = N - static_cast<uint64_t>(U - 1) * c;
  const uint64_t blocks = std::min<uint64_t>((N + 255) / 256, 148ull * 16ull);
  k_chunk_expand<<<static_cast<uint32_t>(blocks), 256, 0, st>>>(pi, N, c, ls, ragged, order);
  return cudaGetLastError();
}

}  // namespace ppl
