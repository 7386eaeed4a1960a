// Eq. (2) pre-propagation on the GPU (the step before the
// hot path): X_k = B X_{k-1}, k = 1..K, with B = D~^{-1/2} (I + A) D~^{-1/2}
// given as a CSR of A~ = I + A.
//
// Arithmetic is the oracle's definition (oracle O2/O3), so results are bit
// identical, not merely within tolerance:
//   w_ij = 1 / sqrt(d~_i * d~_j) in fp64 (d~ = row length; IEEE sqrt and div),
//   acc  = sum over the row's nonzeros in ascending column order of w_ij * x_j,
//          each product and each sum rounded separately in fp64 (no FMA),
//   X_k[i, f] = fp32(acc) (round to nearest even).
// B200 design: one warp per row, lanes across features (coalesced 128-byte
// reads of each neighbour row, up to 4 features per lane), the row's
// (column, weight) pairs broadcast from lane-parallel loads with shuffles.
// HBM-bound: per nonzero F*4 bytes of neighbour features (+ 16 B of CSR),
// per row F*4 bytes written; fp64 work (2 F per nonzero) is far below the
// B200's fp64 rate.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace ppl {

__global__ void k_operator_values(int64_t n, const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col,
                                  double* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < n;
       i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    const double di = static_cast<double>(e - b);
    for (int64_t p = b + lane; p < e; p += 32) {
      const int64_t j = col[p];
      const double dj = static_cast<double>(row_ptr[j + 1] - row_ptr[j]);
      val[p] = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(di, dj)));
    }
  }
}

// y[i, :] = B x[i, :] for one hop; FQ = features per lane (F <= 32 * FQ).
template <int FQ>
__global__ void __launch_bounds__(256) k_spmm_rows(int64_t n, int32_t F, const int64_t* __restrict__ row_ptr,
                                                   const int64_t* __restrict__ col, const double* __restrict__ val,
                                                   const float* __restrict__ x, float* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < n;
       i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    double acc[FQ];
#pragma unroll
    for (int q = 0; q < FQ; ++q) acc[q] = 0.0;
    for (int64_t p0 = b; p0 < e; p0 += 32) {
      const int m = static_cast<int>(min(static_cast<int64_t>(32), e - p0));
      const int64_t jl = lane < m ? col[p0 + lane] : 0;
      const double wl = lane < m ? val[p0 + lane] : 0.0;
      // One neighbour row at a time, ascending column order.  Measured: batching
      // 2, 4 or 8 rows per warp before accumulating costs registers/occupancy and
      // was slower (r1f); 40 resident warps per SM already keep ~20 KB in flight.
      for (int s = 0; s < m; ++s) {
        const int64_t j = __shfl_sync(0xffffffffu, jl, s);
        const double w = __shfl_sync(0xffffffffu, wl, s);
        const float* xr = x + j * F;
#pragma unroll
        for (int q = 0; q < FQ; ++q) {
          const int f = lane + 32 * q;
          if (f < F) acc[q] = __dadd_rn(acc[q], __dmul_rn(w, static_cast<double>(__ldg(xr + f))));
        }
      }
    }
    float* yr = y + i * F;
#pragma unroll
    for (int q = 0; q < FQ; ++q) {
      const int f = lane + 32 * q;
      if (f < F) yr[f] = __double2float_rn(acc[q]);
    }
  }
}

// Vector variant (F % 4 == 0): lane l owns features 4l..4l+3 (+ 128 + 4l.. for
// FV = 2), so a neighbour row is one 16-byte load per lane instead of up to four
// 4-byte loads, and kAhead neighbour rows are loaded before any is accumulated
// (their addresses do not depend on the sums).  The additions still run in
// ascending column order per output element: bit-identical to k_spmm_rows.
template <int FV, int kAhead>
__global__ void __launch_bounds__(256, (FV == 1 && kAhead == 4) ? 4 : 1) k_spmm_rows_v4(int64_t n, int32_t F, const int64_t* __restrict__ row_ptr,
                                                      const int64_t* __restrict__ col, const double* __restrict__ val,
                                                      const float* __restrict__ x, float* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int nv = F >> 2;  // float4 per row
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < n;
       i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    double acc[FV][4];
#pragma unroll
    for (int q = 0; q < FV; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[q][c] = 0.0;
    // (column, weight) of the next 32 nonzeros are loaded while this chunk's rows are summed
    int64_t jn = b + lane < e ? col[b + lane] : 0;
    double wn = b + lane < e ? val[b + lane] : 0.0;
    for (int64_t p0 = b; p0 < e; p0 += 32) {
      const int m = static_cast<int>(min(static_cast<int64_t>(32), e - p0));
      const int64_t jl = jn;
      const double wl = wn;
      if (p0 + 32 < e) {
        jn = p0 + 32 + lane < e ? col[p0 + 32 + lane] : 0;
        wn = p0 + 32 + lane < e ? val[p0 + 32 + lane] : 0.0;
      }
      for (int s0 = 0; s0 < m; s0 += kAhead) {
        float4 xv[kAhead][FV];
        double w[kAhead];
#pragma unroll
        for (int u = 0; u < kAhead; ++u) {
          const int s = s0 + u < m ? s0 + u : m - 1;
          const int64_t j = __shfl_sync(0xffffffffu, jl, s);
          w[u] = __shfl_sync(0xffffffffu, wl, s);
          const float4* xr = reinterpret_cast<const float4*>(x + j * F);
#pragma unroll
          for (int q = 0; q < FV; ++q) {
            const int v = lane + 32 * q;
            xv[u][q] = (s0 + u < m && v < nv) ? __ldg(xr + v) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < kAhead; ++u) {
          if (s0 + u >= m) break;
#pragma unroll
          for (int q = 0; q < FV; ++q) {
            acc[q][0] = __dadd_rn(acc[q][0], __dmul_rn(w[u], static_cast<double>(xv[u][q].x)));
            acc[q][1] = __dadd_rn(acc[q][1], __dmul_rn(w[u], static_cast<double>(xv[u][q].y)));
            acc[q][2] = __dadd_rn(acc[q][2], __dmul_rn(w[u], static_cast<double>(xv[u][q].z)));
            acc[q][3] = __dadd_rn(acc[q][3], __dmul_rn(w[u], static_cast<double>(xv[u][q].w)));
          }
        }
      }
    }
    float4* yr = reinterpret_cast<float4*>(y + i * F);
#pragma unroll
    for (int q = 0; q < FV; ++q) {
      const int v = lane + 32 * q;
      if (v < nv)
        yr[v] = make_float4(__double2float_rn(acc[q][0]), __double2float_rn(acc[q][1]), __double2float_rn(acc[q][2]),
                            __double2float_rn(acc[q][3]));
    }
  }
}

// ---- propagation into a (sharded) loader store: pp_propagate_store ----------
// Hop slot k of this rank's node-major records = B (hop slot k-1 of all rows).
// Neighbour j lives on owner j mod W at local row j div W, in that owner's HBM
// store, its pinned spill (UVA) or a peer's store over NVLink.  The weight
// w_ij = 1/sqrt(d~_i d~_j) is computed per nonzero from the global degree
// array (same IEEE fp64 operations as k_operator_values, so the result is
// bit-identical to the hop-major kernels and the oracle); d~ is tiny and
// L2-resident at products size, so this replaces an 8-B/nonzero weight read.
__device__ __forceinline__ const uint8_t* shard_record(const ShardView* sh, uint32_t W, uint32_t j, int64_t rs) {
  const uint32_t o = j % W, l = j / W;
  const ShardView& s = sh[o];
  return static_cast<int64_t>(l) < s.n_hbm ? s.hbm + static_cast<int64_t>(l) * rs
                                           : s.spill + (static_cast<int64_t>(l) - s.n_hbm) * rs;
}

__device__ __forceinline__ void store_x16(uint8_t* p, int x_dtype, float a, float b) {
  uint32_t v;
  if (x_dtype == 1) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    v = *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __half2 h = __floats2half2_rn(a, b);
    v = *reinterpret_cast<const uint32_t*>(&h);
  }
  *reinterpret_cast<uint32_t*>(p) = v;
}

// Vector variant: F % 4 == 0, lane l owns float4 slots l (+ 32 for FV = 2).
template <int FV>
__global__ void __launch_bounds__(256, FV == 1 ? 4 : 1) k_spmm_store_v4(const StorePropArgs a) {
  __shared__ ShardView s_sh[kMaxWorld];
  if (threadIdx.x < a.W) s_sh[threadIdx.x] = a.shards[threadIdx.x];
  __syncthreads();
  constexpr int kAhead = 4;
  const int lane = threadIdx.x & 31;
  const int nv = a.F >> 2;
  const uint32_t W = static_cast<uint32_t>(a.W);
  const int64_t in_off = static_cast<int64_t>(a.k - 1) * a.F * 4, out_off = static_cast<int64_t>(a.k) * a.F * 4;
  for (int64_t lr = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; lr < a.local_rows;
       lr += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = a.row_ptr[lr], e = a.row_ptr[lr + 1];
    const double di = static_cast<double>(e - b);
    double acc[FV][4];
#pragma unroll
    for (int q = 0; q < FV; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[q][c] = 0.0;
    // this lane's nonzero of the next 32: source hop vector and weight
    const uint8_t* srcn = nullptr;
    double wn = 0.0;
    if (b + lane < e) {
      const uint32_t j = static_cast<uint32_t>(a.col[b + lane]);
      srcn = shard_record(s_sh, W, j, a.rec_stride) + in_off;
      wn = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(di, static_cast<double>(a.deg[j]))));
    }
    for (int64_t p0 = b; p0 < e; p0 += 32) {
      const int m = static_cast<int>(min(static_cast<int64_t>(32), e - p0));
      const uint8_t* srcl = srcn;
      const double wl = wn;
      if (p0 + 32 + lane < e) {
        const uint32_t j = static_cast<uint32_t>(a.col[p0 + 32 + lane]);
        srcn = shard_record(s_sh, W, j, a.rec_stride) + in_off;
        wn = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(di, static_cast<double>(a.deg[j]))));
      }
      for (int s0 = 0; s0 < m; s0 += kAhead) {
        float4 xv[kAhead][FV];
        double w[kAhead];
#pragma unroll
        for (int u = 0; u < kAhead; ++u) {
          const int s = s0 + u < m ? s0 + u : m - 1;
          const float4* xr = reinterpret_cast<const float4*>(
              __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(srcl), s));
          w[u] = __shfl_sync(0xffffffffu, wl, s);
#pragma unroll
          for (int q = 0; q < FV; ++q) {
            const int v = lane + 32 * q;
            xv[u][q] = (s0 + u < m && v < nv) ? __ldcg(xr + v) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < kAhead; ++u) {
          if (s0 + u >= m) break;
#pragma unroll
          for (int q = 0; q < FV; ++q) {
            acc[q][0] = __dadd_rn(acc[q][0], __dmul_rn(w[u], static_cast<double>(xv[u][q].x)));
            acc[q][1] = __dadd_rn(acc[q][1], __dmul_rn(w[u], static_cast<double>(xv[u][q].y)));
            acc[q][2] = __dadd_rn(acc[q][2], __dmul_rn(w[u], static_cast<double>(xv[u][q].z)));
            acc[q][3] = __dadd_rn(acc[q][3], __dmul_rn(w[u], static_cast<double>(xv[u][q].w)));
          }
        }
      }
    }
    const ShardView& me = s_sh[a.rank];
    uint8_t* rec = const_cast<uint8_t*>(lr < me.n_hbm ? me.hbm + lr * a.rec_stride : me.spill + (lr - me.n_hbm) * a.rec_stride);
    float4* yr = reinterpret_cast<float4*>(rec + out_off);
    uint8_t* xr = (a.xstore != nullptr && lr < me.n_hbm) ? a.xstore + lr * a.xrec_stride + static_cast<int64_t>(a.k) * a.F * 2
                                                         : nullptr;
#pragma unroll
    for (int q = 0; q < FV; ++q) {
      const int v = lane + 32 * q;
      if (v < nv) {
        const float4 y = make_float4(__double2float_rn(acc[q][0]), __double2float_rn(acc[q][1]),
                                     __double2float_rn(acc[q][2]), __double2float_rn(acc[q][3]));
        yr[v] = y;
        if (xr != nullptr) {
          store_x16(xr + v * 8, a.x_dtype, y.x, y.y);
          store_x16(xr + v * 8 + 4, a.x_dtype, y.z, y.w);
        }
      }
    }
  }
}

// Per-element variant (any F <= 32 * FQ): lane l owns features l + 32 q.
template <int FQ>
__global__ void __launch_bounds__(256) k_spmm_store(const StorePropArgs a) {
  __shared__ ShardView s_sh[kMaxWorld];
  if (threadIdx.x < a.W) s_sh[threadIdx.x] = a.shards[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t W = static_cast<uint32_t>(a.W);
  const int F = a.F;
  const int64_t in_off = static_cast<int64_t>(a.k - 1) * F * 4, out_off = static_cast<int64_t>(a.k) * F * 4;
  for (int64_t lr = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; lr < a.local_rows;
       lr += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = a.row_ptr[lr], e = a.row_ptr[lr + 1];
    const double di = static_cast<double>(e - b);
    double acc[FQ];
#pragma unroll
    for (int q = 0; q < FQ; ++q) acc[q] = 0.0;
    for (int64_t p0 = b; p0 < e; p0 += 32) {
      const int m = static_cast<int>(min(static_cast<int64_t>(32), e - p0));
      const uint8_t* srcl = nullptr;
      double wl = 0.0;
      if (lane < m) {
        const uint32_t j = static_cast<uint32_t>(a.col[p0 + lane]);
        srcl = shard_record(s_sh, W, j, a.rec_stride) + in_off;
        wl = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(di, static_cast<double>(a.deg[j]))));
      }
      for (int s = 0; s < m; ++s) {
        const float* xr = reinterpret_cast<const float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(srcl), s));
        const double w = __shfl_sync(0xffffffffu, wl, s);
#pragma unroll
        for (int q = 0; q < FQ; ++q) {
          const int f = lane + 32 * q;
          if (f < F) acc[q] = __dadd_rn(acc[q], __dmul_rn(w, static_cast<double>(__ldcg(xr + f))));
        }
      }
    }
    const ShardView& me = s_sh[a.rank];
    uint8_t* rec = const_cast<uint8_t*>(lr < me.n_hbm ? me.hbm + lr * a.rec_stride : me.spill + (lr - me.n_hbm) * a.rec_stride);
    float* yr = reinterpret_cast<float*>(rec + out_off);
    uint8_t* xr = (a.xstore != nullptr && lr < me.n_hbm) ? a.xstore + lr * a.xrec_stride + static_cast<int64_t>(a.k) * F * 2
                                                         : nullptr;
#pragma unroll
    for (int q = 0; q < FQ; ++q) {
      const int f = lane + 32 * q;
      if (f < F) {
        const float y = __double2float_rn(acc[q]);
        yr[f] = y;
        if (xr != nullptr) {
          if (a.x_dtype == 1) {
            const __nv_bfloat16 h = __float2bfloat16_rn(y);
            *reinterpret_cast<__nv_bfloat16*>(xr + 2 * f) = h;
          } else {
            const __half h = __float2half_rn(y);
            *reinterpret_cast<__half*>(xr + 2 * f) = h;
          }
        }
      }
    }
  }
}

// ---- L2-sliced propagation ----------------------------------------------------------------------
// The neighbour reads of a hop are random rows of X_{k-1}: a products-sized hop reads ~50 GB of
// 400-byte rows (126 M nonzeros) while X_{k-1} itself is 0.98 GB, so the row-per-warp kernels above
// fetch most of it from DRAM again and again (ncu r1final: 64.9 GB of DRAM reads per hop).  The L2
// allocates 128-byte lines, so a feature window of the node-major records (32 B of every 1600-B
// record) would still occupy a whole line per row (313 MB at products size, more than the 126 MB
// L2; measured r2: 185 GB of DRAM reads per hop).  So a hop first writes X_{k-1} window-major into a
// scratch Xt[w][row][8 fp32] (k_slot_to_windows: one read of the slot, one write), then runs one
// pass per 32-byte window: pass w gathers only Xt[w] -- rows x 32 B = 78 MB of fully used lines,
// L2-resident after its first touch -- so DRAM carries X_{k-1} about twice plus the int32 column
// ids and row pointers once per pass.  One thread per output row walks the row's nonzeros in
// ascending column order with the window's features in fp64 registers: every output element is the
// same sequence of separately rounded products and sums as before (bit-identical to the oracle, O3).
// The weight 1/sqrt(d~_i d~_j) is recomputed per nonzero and pass (fp64 IEEE, as k_operator_values).
constexpr int kWinBytes = 32;  // window pitch in xt: one L2 sector; 4 rows of a window share a 128-B line

// Window width in bytes: 32 (default) or 16 (PPLOAD_SPMM_WINDOW=16: half the footprint, twice the passes).
static int spmm_window() {
  const char* e = getenv("PPLOAD_SPMM_WINDOW");
  return (e && atoi(e) == 16) ? 16 : 32;
}

// Xt[w][r] (kWinBytes each, window w = bytes [32w, 32w + 32) of the slot) from slot bytes
// [0, slot_bytes) of row r of `src` (rows < n_hbm at hbm + r * pitch + off, else spill).
__global__ void k_slot_to_windows(const uint8_t* __restrict__ hbm, const uint8_t* __restrict__ spill, int64_t n_hbm,
                                  int64_t rows, int64_t pitch, int64_t off, int32_t slot_bytes,
                                  uint8_t* __restrict__ xt, int win) {
  const int nwin = (slot_bytes + win - 1) / win;
  const int vpr = slot_bytes / 16;  // float4 per row
  // thread t -> (block of 64 rows, float4 v of the slot, row within the block): the slot's
  // float4s of 64 rows are read by one CTA back to back (their lines stay in L2), and each
  // window's 64 rows x 32 B are written contiguously
  const int64_t total = (rows + 63) / 64 * 64 * vpr;  // whole 64-row blocks (the tail block is partial)
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t blk = t / (64 * vpr);
    const int64_t rem = t - blk * 64 * vpr;
    const int v = static_cast<int>(rem / 64);
    const int64_t r = blk * 64 + (rem - static_cast<int64_t>(v) * 64);
    if (r >= rows) continue;
    const uint8_t* rec = r < n_hbm ? hbm + r * pitch : spill + (r - n_hbm) * pitch;
    const float4 x = __ldcs(reinterpret_cast<const float4*>(rec + off) + v);
    const int w = v / (win / 16), c = v % (win / 16);
    reinterpret_cast<float4*>(xt + (static_cast<int64_t>(w) * rows + r) * win)[c] = x;
    (void)nwin;
  }
}

// One pass: window `win` (nv float4 <= 2) of every output row.  Input: the compact window Xt[win]
// (pitch kWinBytes).  Output: out rows (< out.n_hbm in out.hbm, else out.spill) at pitch out_pitch,
// bytes out_off.. of the row; the owner's exchange copy (16-bit) at x_off when a.xstore is set.
// L2 eviction policies: the window being gathered stays (evict_last); the per-pass streams of
// column ids and weights, which would otherwise push it out of the L2, go first (evict_first).
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t ld_u32_hint(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_f64_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ void ld_window(const void* p, int nv, float4& a, float4& b, uint64_t pol) {
  if (nv > 1) {  // the whole 32-byte window in one 256-bit load (LDG.256)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p), "l"(pol));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
                 : "l"(p), "l"(pol));
    b = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__global__ void __launch_bounds__(256) k_spmm_sliced(const StorePropArgs a, const double* __restrict__ wv,
                                                     const uint8_t* __restrict__ xt_win, int win, int nv, ShardView out,
                                                     int64_t out_pitch, int64_t out_off, int64_t x_off) {
  constexpr int kU = 4;  // nonzeros loaded ahead of their accumulation
  const uint64_t keep = l2_policy_last(), stream = l2_policy_first();
  for (int64_t lr = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; lr < a.local_rows;
       lr += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = a.row_ptr[lr], e = a.row_ptr[lr + 1];
    double acc[2][4];
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[v][c] = 0.0;
    for (int64_t p0 = b; p0 < e; p0 += kU) {
      const int m = static_cast<int>(min(static_cast<int64_t>(kU), e - p0));
      uint32_t j[kU];
      double wu[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        j[u] = u < m ? ld_u32_hint(a.col32 + p0 + u, stream) : 0u;
        wu[u] = u < m ? ld_f64_hint(wv + p0 + u, stream) : 0.0;
      }
      float4 xv[kU][2];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (u < m) {
          ld_window(xt_win + static_cast<int64_t>(j[u]) * win, nv, xv[u][0], xv[u][1], keep);
        } else {
          xv[u][0] = xv[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (u >= m) break;
        const double w = wu[u];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          acc[v][0] = __dadd_rn(acc[v][0], __dmul_rn(w, static_cast<double>(xv[u][v].x)));
          acc[v][1] = __dadd_rn(acc[v][1], __dmul_rn(w, static_cast<double>(xv[u][v].y)));
          acc[v][2] = __dadd_rn(acc[v][2], __dmul_rn(w, static_cast<double>(xv[u][v].z)));
          acc[v][3] = __dadd_rn(acc[v][3], __dmul_rn(w, static_cast<double>(xv[u][v].w)));
        }
      }
    }
    uint8_t* rec = const_cast<uint8_t*>(lr < out.n_hbm ? out.hbm + lr * out_pitch : out.spill + (lr - out.n_hbm) * out_pitch);
    float4* yr = reinterpret_cast<float4*>(rec + out_off);
    uint8_t* xr = (a.xstore != nullptr && lr < out.n_hbm) ? a.xstore + lr * a.xrec_stride + x_off : nullptr;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      if (v >= nv) break;
      const float4 o = make_float4(__double2float_rn(acc[v][0]), __double2float_rn(acc[v][1]),
                                   __double2float_rn(acc[v][2]), __double2float_rn(acc[v][3]));
      yr[v] = o;
      if (xr != nullptr) {
        store_x16(xr + v * 8, a.x_dtype, o.x, o.y);
        store_x16(xr + v * 8 + 4, a.x_dtype, o.z, o.w);
      }
    }
  }
}

// w[p] = 1 / sqrt(d~_i d~_j) for every nonzero p of row i (column j): the oracle's O2 values (IEEE
// fp64 multiply, sqrt, divide), computed once per call and streamed by every pass.
__global__ void k_weights_from_deg(int64_t rows, const int64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col32,
                                   const int32_t* __restrict__ deg, double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < rows;
       i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    const double di = static_cast<double>(e - b);
    for (int64_t p = b + lane; p < e; p += 32)
      w[p] = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(di, static_cast<double>(deg[col32[p]]))));
  }
}

// Opt-in (PPLOAD_SPMM=sliced): measured slower than the row kernels on B200 at products size
// (r2, profiles/r2/propagation_sliced.md: 23.5 ms vs 12.1 ms per hop).  A window read by every SM
// is also cached in the reading die's L2 half, so a 78 MB window does not stay resident (54 % of
// its sectors missed), and 16-byte windows (39 MB, 96 % hits) double the per-pass column / weight
// streams instead (111 GB of DRAM reads per hop vs 65 GB for the row kernel).
bool spmm_use_sliced(int64_t rows, int32_t F) {
  (void)rows;
  const char* e = getenv("PPLOAD_SPMM");
  return e && !strcmp(e, "sliced") && F % 4 == 0;
}

int64_t spmm_sliced_scratch_bytes(int64_t rows, int32_t F, int64_t nnz) {
  // window-major slot copy + int32 column ids + fp64 weights
  return ((static_cast<int64_t>(F) * 4 + kWinBytes - 1) / kWinBytes) * rows * kWinBytes + nnz * 12 + 256;
}

// One hop through the window-major scratch: transpose slot (in) -> xt, then one pass per window.
// scratch: [weights fp64 nnz][xt] (spmm_sliced_scratch_bytes); weights computed here when fresh_w.
static cudaError_t run_sliced(const StorePropArgs& a, ShardView in, int64_t in_pitch, int64_t in_off, ShardView out,
                              int64_t out_pitch, int64_t out_off, int64_t x_off, uint8_t* scratch, int64_t nnz,
                              bool fresh_w, cudaStream_t st) {
  const int32_t slot_bytes = a.F * 4;
  const int64_t rows = a.local_rows;
  const int win = spmm_window();
  double* wv = reinterpret_cast<double*>(scratch);
  uint8_t* xt = scratch + (nnz * 8 + 255) / 256 * 256;
  if (fresh_w) {
    const int64_t blocks = std::min<int64_t>((rows * 32 + 255) / 256, 148ll * 16);
    k_weights_from_deg<<<static_cast<uint32_t>(blocks), 256, 0, st>>>(rows, a.row_ptr, a.col32, a.deg, wv);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  {
    const int64_t total = (rows + 63) / 64 * 64 * (slot_bytes / 16);
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148ll * 16);
    k_slot_to_windows<<<static_cast<uint32_t>(blocks), 256, 0, st>>>(in.hbm, in.spill, in.n_hbm, rows, in_pitch, in_off,
                                                                      slot_bytes, xt, win);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const int nwin = (slot_bytes + win - 1) / win;
  const int64_t blocks = std::min<int64_t>((rows + 255) / 256, 148ll * 8);
  for (int w = 0; w < nwin; ++w) {
    const int nv = std::min(win, slot_bytes - w * win) / 16;
    k_spmm_sliced<<<static_cast<uint32_t>(blocks), 256, 0, st>>>(a, wv, xt + static_cast<int64_t>(w) * rows * win, win,
                                                                  nv, out, out_pitch, out_off + w * win,
                                                                  x_off + w * (win / 2));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

__global__ void k_col_to_u32(const int64_t* __restrict__ col, int64_t nnz, uint32_t* __restrict__ col32) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    col32[p] = static_cast<uint32_t>(col[p]);
}

cudaError_t launch_col_to_u32(const int64_t* col, int64_t nnz, uint32_t* col32, cudaStream_t st) {
  if (nnz <= 0) return cudaSuccess;
  k_col_to_u32<<<148 * 16, 256, 0, st>>>(col, nnz, col32);
  return cudaGetLastError();
}

__global__ void k_row_lengths(const int64_t* __restrict__ row_ptr, int64_t n, int32_t* __restrict__ deg) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    deg[i] = static_cast<int32_t>(row_ptr[i + 1] - row_ptr[i]);
}

cudaError_t launch_row_lengths(const int64_t* row_ptr, int64_t n, int32_t* deg, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_row_lengths<<<148 * 8, 256, 0, st>>>(row_ptr, n, deg);
  return cudaGetLastError();
}

cudaError_t launch_spmm_sliced_rows(int64_t n, int32_t F, const int64_t* row_ptr, const uint32_t* col32,
                                   const int32_t* deg, const float* x, float* y, uint8_t* scratch, int64_t nnz,
                                   bool fresh_w, cudaStream_t st) {
  if (n <= 0 || F <= 0) return cudaSuccess;
  if (F % 4 != 0 || reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(y) % 16)
    return cudaErrorInvalidValue;
  StorePropArgs a{};
  a.local_rows = n;
  a.F = F;
  a.row_ptr = row_ptr;
  a.deg = deg;
  a.col32 = col32;
  const int64_t pitch = static_cast<int64_t>(F) * 4;
  const ShardView in{reinterpret_cast<const uint8_t*>(x), nullptr, n};
  const ShardView out{reinterpret_cast<const uint8_t*>(y), nullptr, n};
  return run_sliced(a, in, pitch, 0, out, pitch, 0, 0, scratch, nnz, fresh_w, st);
}

cudaError_t launch_spmm_store_sliced(const StorePropArgs& a, uint8_t* scratch, int64_t nnz, cudaStream_t st) {
  if (a.local_rows <= 0) return cudaSuccess;
  if (a.W != 1 || a.col32 == nullptr || a.F % 4 != 0 || a.rec_stride % 16 != 0) return cudaErrorInvalidValue;
  const ShardView me = a.shards[a.rank];
  const int64_t slot = static_cast<int64_t>(a.F) * 4;
  return run_sliced(a, me, a.rec_stride, (a.k - 1) * slot, me, a.rec_stride, a.k * slot,
                    static_cast<int64_t>(a.k) * a.F * 2, scratch, nnz, true, st);
}

cudaError_t launch_spmm_store(const StorePropArgs& a, cudaStream_t st) {
  if (a.local_rows <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((a.local_rows * 32 + 255) / 256, 148ll * 64);
  const uint32_t g = static_cast<uint32_t>(blocks);
  const bool vec = a.F % 4 == 0 && a.rec_stride % 16 == 0 && !(getenv("PPLOAD_SPMM") && !strcmp(getenv("PPLOAD_SPMM"), "scalar"));
  if (vec && a.F <= 128) k_spmm_store_v4<1><<<g, 256, 0, st>>>(a);
  else if (vec && a.F <= 256) k_spmm_store_v4<2><<<g, 256, 0, st>>>(a);
  else if (a.F <= 32) k_spmm_store<1><<<g, 256, 0, st>>>(a);
  else if (a.F <= 64) k_spmm_store<2><<<g, 256, 0, st>>>(a);
  else if (a.F <= 128) k_spmm_store<4><<<g, 256, 0, st>>>(a);
  else if (a.F <= 256) k_spmm_store<8><<<g, 256, 0, st>>>(a);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_operator_values(int64_t n, const int64_t* row_ptr, const int64_t* col, double* val,
                                   cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_operator_values<<<148 * 16, 256, 0, st>>>(n, row_ptr, col, val);
  return cudaGetLastError();
}

cudaError_t launch_spmm(int64_t n, int32_t F, const int64_t* row_ptr, const int64_t* col, const double* val,
                        const float* x, float* y, cudaStream_t st) {
  if (n <= 0 || F <= 0) return cudaSuccess;
  const int64_t warps = n;
  const int64_t blocks = std::min<int64_t>((warps * 32 + 255) / 256, 148ll * 64);
  const bool vec = F % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0 &&
                   !(getenv("PPLOAD_SPMM") && !strcmp(getenv("PPLOAD_SPMM"), "scalar"));
  const int ahead = getenv("PPLOAD_SPMM_AHEAD") ? atoi(getenv("PPLOAD_SPMM_AHEAD")) : 4;  // r1m: 8 is slower (registers)
  const uint32_t g = static_cast<uint32_t>(blocks);
  if (vec && F <= 128 && ahead == 4) k_spmm_rows_v4<1, 4><<<g, 256, 0, st>>>(n, F, row_ptr, col, val, x, y);
  else if (vec && F <= 128) k_spmm_rows_v4<1, 8><<<g, 256, 0, st>>>(n, F, row_ptr, col, val, x, y);
  else if (vec && F <= 256) k_spmm_rows_v4<2, 4><<<g, 256, 0, st>>>(n, F, row_ptr, col, val, x, y);
  else if (F <= 32) k_spmm_rows<1><<<static_cast<uint32_t>(blocks), 256, 0, st>>>(n, F, row_ptr, col, val, x, y);
  else if (F <= 64) k_spmm_rows<2><<<static_cast<uint32_t>(blocks), 256, 0, st>>>(n, F, row_ptr, col, val, x, y);
  else if (F <= 128) k_spmm_rows<4><<<static_cast<uint32_t>(blocks), 256, 0, st>>>(n, F, row_ptr, col, val, x, y);
  else if (F <= 256) k_spmm_rows<8><<<static_cast<uint32_t>(blocks), 256, 0, st>>>(n, F, row_ptr, col, val, x, y);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace ppl
