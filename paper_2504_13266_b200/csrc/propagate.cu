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

// ---- wave-synchronous propagation (k_spmm_wave) ---------------------------------------------------
// The row kernels above are bound by DRAM misses at products size: X_{k-1} (0.98 GB) is ~8x the L2,
// every nonzero reads a random 400-B row, and 93 % of those rows miss (64.7 GB of DRAM reads per hop
// for 50.5 GB of neighbour rows, profiles/r2/propagation_sliced.md).  Here the whole GPU works on one
// *wave* of output rows at a time -- R rows per CTA, their fp64 partial sums resident in shared
// memory -- and sweeps the column ids in C ascending windows of n / C ids, so at any moment all SMs
// read neighbour rows from the same window of X_{k-1}: a row j that several rows of the wave need is
// fetched from DRAM about once per wave instead of once per nonzero (S = grid * R rows per wave;
// X row j has S d / n readers per wave).  Each output row's neighbours are still summed in ascending
// column order (windows ascend; columns ascend inside a window) with the same separately rounded fp64
// products and sums as k_spmm_rows_v4 / k_spmm_store_v4, and the weights are the same IEEE
// expressions, so the result is bit-identical to them and to the oracle (O2/O3).
// Work split: a warp takes 4 rows of its CTA; lanes 8q..8q+7 read the next 8 column ids of row q,
// a ballot selects those inside the window, and the selected (row, column) entries are processed in
// order, 4 neighbour rows in flight per warp, lane l owning features 4l..4l+3; a row saturating its 8
// slots gets another round.  Between windows the CTAs keep loosely in step (a counter: before window
// g a CTA waits, boundedly, until every CTA has finished window g - lag); the counter only shapes the
// L2 working set -- no CTA reads another's results -- so the bounded wait cannot deadlock.

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wave_store16(uint8_t* p, int x_dtype, float4 y) {
  store_x16(p, x_dtype, y.x, y.y);
  store_x16(p + 4, x_dtype, y.z, y.w);
}

template <int kWaveThreads, int kWaveAhead>
__global__ void __launch_bounds__(kWaveThreads, 1) k_spmm_wave(const WaveArgs a) {
  constexpr int kWaveWarps = kWaveThreads / 32;
  extern __shared__ __align__(16) uint8_t wsm[];
  const int R = a.R, nv = a.nv;
  double2* s_st = reinterpret_cast<double2*>(wsm);  // [R][2][nv]: features (4l, 4l+1), (4l+2, 4l+3) of lane l
  int64_t* s_pos = reinterpret_cast<int64_t*>(s_st + static_cast<int64_t>(R) * 2 * nv);  // next nonzero
  int64_t* s_end = s_pos + R;
  double* s_di = reinterpret_cast<double*>(s_end + R);  // d~_i
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane >> 3, sl = lane & 7;
  const bool on = lane < nv;
  const int64_t S = static_cast<int64_t>(gridDim.x) * R;
  const int64_t nwaves = (a.n + S - 1) / S;
  for (int64_t wave = 0; wave < nwaves; ++wave) {
    const int64_t row0 = wave * S + static_cast<int64_t>(blockIdx.x) * R;
    const int rows = static_cast<int>(max(static_cast<int64_t>(0), min(static_cast<int64_t>(R), a.n - row0)));
    for (int r = tid; r < rows; r += kWaveThreads) {
      const int64_t b = a.row_ptr[row0 + r], e = a.row_ptr[row0 + r + 1];
      s_pos[r] = b;
      s_end[r] = e;
      s_di[r] = static_cast<double>(e - b);
    }
    for (int i = tid; i < rows * 2 * nv; i += kWaveThreads) s_st[i] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int c = 0; c < a.C; ++c) {
      const int64_t g = wave * a.C + c;
      if (a.lag > 0 && g >= a.lag) {
        if (tid == 0) {
          const unsigned target = gridDim.x * static_cast<unsigned>(g - a.lag + 1);
          for (int it = 0; it < a.spin && ld_relaxed_u32(a.sync) < target; ++it) __nanosleep(128);
        }
        __syncthreads();
      }
      const int64_t jend = c == a.C - 1 ? INT64_MAX : (c + 1) * a.win;
      for (int r0 = warp * 4; r0 < rows; r0 += kWaveWarps * 4) {
        unsigned active = 0xfu;
        while (active) {
          const int r = r0 + q;
          const bool mine = r < rows && ((active >> q) & 1u);
          int64_t j = 0;
          double wl = 0.0;
          bool in = false;
          if (mine) {
            const int64_t p = s_pos[r] + sl;
            if (p < s_end[r]) {
              j = a.col[p];
              in = j < jend;
              if (in)
                wl = a.val != nullptr ? a.val[p]
                                      : __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(s_di[r], static_cast<double>(a.deg[j]))));
            }
          }
          const unsigned mask = __ballot_sync(0xffffffffu, in);  // also orders the s_pos reads before the update
          unsigned sat = 0;  // rows whose 8 slots were all inside the window: they may have more
#pragma unroll
          for (int t = 0; t < 4; ++t) sat |= (((mask >> (8 * t)) & 0xffu) == 0xffu ? 1u : 0u) << t;
          if (sl == 0 && mine) s_pos[r] += __popc((mask >> (8 * q)) & 0xffu);
          unsigned mm = mask;
          int cur = -1;
          double2 lo = make_double2(0.0, 0.0), hi = lo;
          while (mm) {
            float4 xv[kWaveAhead];
            double w[kWaveAhead];
            int rq[kWaveAhead];
#pragma unroll
            for (int u = 0; u < kWaveAhead; ++u) {
              rq[u] = -1;
              w[u] = 0.0;
              xv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (mm) {  // warp-uniform
                const int L = __ffs(mm) - 1;
                mm &= mm - 1;
                const int64_t jj = __shfl_sync(0xffffffffu, j, L);
                w[u] = __shfl_sync(0xffffffffu, wl, L);
                rq[u] = L >> 3;
                if (on) xv[u] = __ldcg(reinterpret_cast<const float4*>(a.src + jj * a.src_stride) + lane);
              }
            }
#pragma unroll
            for (int u = 0; u < kWaveAhead; ++u) {
              if (rq[u] < 0) break;
              if (rq[u] != cur) {
                double2* st = s_st + static_cast<int64_t>(r0 + rq[u]) * 2 * nv + lane;
                if (cur >= 0 && on) {
                  double2* so = s_st + static_cast<int64_t>(r0 + cur) * 2 * nv + lane;
                  so[0] = lo;
                  so[nv] = hi;
                }
                cur = rq[u];
                if (on) {
                  lo = st[0];
                  hi = st[nv];
                }
              }
              lo.x = __dadd_rn(lo.x, __dmul_rn(w[u], static_cast<double>(xv[u].x)));
              lo.y = __dadd_rn(lo.y, __dmul_rn(w[u], static_cast<double>(xv[u].y)));
              hi.x = __dadd_rn(hi.x, __dmul_rn(w[u], static_cast<double>(xv[u].z)));
              hi.y = __dadd_rn(hi.y, __dmul_rn(w[u], static_cast<double>(xv[u].w)));
            }
          }
          if (cur >= 0 && on) {
            double2* so = s_st + static_cast<int64_t>(r0 + cur) * 2 * nv + lane;
            so[0] = lo;
            so[nv] = hi;
          }
          __syncwarp();
          active = sat;
        }
      }
      __syncthreads();
      if (a.lag > 0 && tid == 0) atomicAdd(a.sync, 1u);
    }
    // the wave's rows are complete: one RNE rounding to fp32 (+ the optional 16-bit copy)
    for (int r = warp; r < rows; r += kWaveWarps) {
      if (on) {
        const double2* st = s_st + static_cast<int64_t>(r) * 2 * nv + lane;
        const double2 lo = st[0], hi = st[nv];
        const float4 y = make_float4(__double2float_rn(lo.x), __double2float_rn(lo.y), __double2float_rn(hi.x),
                                     __double2float_rn(hi.y));
        reinterpret_cast<float4*>(a.dst + (row0 + r) * a.dst_stride)[lane] = y;
        if (a.xdst != nullptr) wave_store16(a.xdst + (row0 + r) * a.x_stride + lane * 8, a.x_dtype, y);
      }
    }
    __syncthreads();
  }
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

// ---- row kernel with the neighbour rows staged by cp.async (k_spmm_rows_cp) -------------------------
// k_spmm_rows_v4 / k_spmm_store_v4 keep 4 neighbour rows in flight per warp in registers (32 warps
// per SM: ~51 KB), and at products size they are bound by that memory-level parallelism against
// random 400-B rows that miss L2 93 % of the time (5.4 TB/s of DRAM reads).  Here each warp streams
// the nonzeros of its rows through a private ring of kSlots row buffers in shared memory, filled by
// cp.async (LDGSTS, 16 B per lane, no register destination), so kSlots rows per warp -- 512 per SM
// at 32 warps x 16 slots -- are in flight.  The ring runs across row boundaries: the nonzeros of a
// warp's rows form one stream, issued kSlots ahead of the one being summed.  Lane l copies and later
// reads only its own 16 bytes of each slot, so cp.async.wait_group orders everything (no barrier).
// Summation per output row: ascending column order, separately rounded fp64 products and sums -- the
// same arithmetic as the other row kernels, bit-identical to them and to the oracle (O2/O3).
struct CpCursor {  // a position in the warp's stream of nonzeros
  int64_t i, p, e;  // row, next nonzero, row end
};

// kBulk: one cp.async.bulk per neighbour row (the whole 16-B-multiple row, issued by lane 0, completing
// on a per-slot mbarrier) instead of 16 B per lane -- one request per row for the L2.
template <int kThreads, int kSlots, bool kBulk>
__global__ void __launch_bounds__(kThreads, 1) k_spmm_rows_cp(const WaveArgs a) {
  extern __shared__ __align__(16) uint8_t csm[];
  constexpr int kWarps = kThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nv = a.nv;
  const bool on = lane < nv;
  const int64_t row_bytes = static_cast<int64_t>(nv) * 16;
  uint8_t* ring = csm + static_cast<int64_t>(warp) * kSlots * row_bytes + lane * 16;
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const uint32_t ring0_s = ring_s - lane * 16;
  uint64_t* bars = reinterpret_cast<uint64_t*>(csm + static_cast<int64_t>(kWarps) * kSlots * row_bytes) + warp * kSlots;
  const uint32_t bars_s = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
  static_assert(kSlots <= 64, "one parity bit per slot");
  uint64_t phase = 0;  // kBulk: parity bit per slot
  if constexpr (kBulk) {
    if (lane == 0)
      for (int s = 0; s < kSlots; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars_s + 8 * s) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * kWarps;
  const int64_t first = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  if (first >= a.n) return;
  // issue cursor: 32 column ids at a time, lane-parallel
  CpCursor is{first, a.row_ptr[first], a.row_ptr[first + 1]};
  int64_t ichunk = is.p;
  int64_t jl = is.p + lane < is.e ? a.col[is.p + lane] : 0;
  // consume cursor: 32 (column, weight) pairs at a time
  CpCursor cs{first, 0, 0};
  double di = 0.0;
  int64_t cchunk = 0;
  double wl = 0.0;
  auto load_weights = [&]() {
    const int64_t p = cchunk + lane;
    wl = 0.0;
    if (p < cs.e) {
      if (a.val != nullptr) {
        wl = a.val[p];
      } else {
        const int64_t j = a.col[p];
        wl = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(di, static_cast<double>(a.deg[j]))));
      }
    }
  };
  auto put_row = [&](int64_t i, double2 lo, double2 hi) {  // one RNE rounding to fp32 (+ the 16-bit copy)
    if (on) {
      const float4 y = make_float4(__double2float_rn(lo.x), __double2float_rn(lo.y), __double2float_rn(hi.x),
                                   __double2float_rn(hi.y));
      reinterpret_cast<float4*>(a.dst + i * a.dst_stride)[lane] = y;
      if (a.xdst != nullptr) wave_store16(a.xdst + i * a.x_stride + lane * 8, a.x_dtype, y);
    }
  };
  // move the consume cursor onto the next row that has nonzeros (rows without any get zeros)
  auto seek_row = [&]() -> bool {
    for (; cs.i < a.n; cs.i += wstride) {
      cs.p = a.row_ptr[cs.i];
      cs.e = a.row_ptr[cs.i + 1];
      if (cs.p < cs.e) {
        di = static_cast<double>(cs.e - cs.p);
        cchunk = cs.p;
        load_weights();
        return true;
      }
      put_row(cs.i, make_double2(0.0, 0.0), make_double2(0.0, 0.0));
    }
    return false;
  };
  // advance the issue cursor to the next nonzero of the stream (next row when this one is done)
  auto issue = [&](int slot) {
    while (is.p >= is.e && is.i < a.n) {  // empty rows are skipped (every row has its diagonal, but be safe)
      is.i += wstride;
      if (is.i >= a.n) break;
      is.p = a.row_ptr[is.i];
      is.e = a.row_ptr[is.i + 1];
      ichunk = is.p;
      jl = is.p + lane < is.e ? a.col[is.p + lane] : 0;
    }
    if (is.i < a.n) {
      if (is.p - ichunk == 32) {
        ichunk = is.p;
        jl = is.p + lane < is.e ? a.col[is.p + lane] : 0;
      }
      const int64_t j = __shfl_sync(0xffffffffu, jl, static_cast<int>(is.p - ichunk));
      if constexpr (kBulk) {
        if (lane == 0) {
          const uint32_t bar = bars_s + 8 * slot;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the slot's generic reads before the copy
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                       "r"(static_cast<uint32_t>(row_bytes))
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  ring0_s + slot * static_cast<uint32_t>(row_bytes)),
              "l"(a.src + j * a.src_stride), "r"(static_cast<uint32_t>(row_bytes)), "r"(bar)
              : "memory");
        }
      } else if (on) {
        const uint8_t* src = a.src + j * a.src_stride + lane * 16;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ring_s + slot * static_cast<uint32_t>(row_bytes)),
                     "l"(src)
                     : "memory");
      }
      ++is.p;
    }
    if constexpr (!kBulk) asm volatile("cp.async.commit_group;" ::: "memory");  // possibly empty: one group per slot
  };
#pragma unroll 1
  for (int s = 0; s < kSlots; ++s) issue(s);
  double2 lo = make_double2(0.0, 0.0), hi = lo;
  int slot = 0;
  bool more = seek_row();
  while (more) {
    if constexpr (kBulk) {  // the oldest slot has landed
      const uint32_t bar = bars_s + 8 * slot, par = static_cast<uint32_t>(phase >> slot) & 1u;
      uint32_t done = 0;
      do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(par)
            : "memory");
      } while (!done);
      phase ^= 1ull << slot;
    } else {
      asm volatile("cp.async.wait_group %0;" ::"n"(kSlots - 1) : "memory");
    }
    if (cs.p - cchunk == 32) {
      cchunk = cs.p;
      load_weights();
    }
    const double w = __shfl_sync(0xffffffffu, wl, static_cast<int>(cs.p - cchunk));
    if (on) {
      const float4 x = *reinterpret_cast<const float4*>(ring + slot * row_bytes);
      lo.x = __dadd_rn(lo.x, __dmul_rn(w, static_cast<double>(x.x)));
      lo.y = __dadd_rn(lo.y, __dmul_rn(w, static_cast<double>(x.y)));
      hi.x = __dadd_rn(hi.x, __dmul_rn(w, static_cast<double>(x.z)));
      hi.y = __dadd_rn(hi.y, __dmul_rn(w, static_cast<double>(x.w)));
    }
    __syncwarp();
    issue(slot);  // refill the slot just summed (its smem read is complete: the sums above used it)
    slot = slot + 1 == kSlots ? 0 : slot + 1;
    if (++cs.p == cs.e) {
      put_row(cs.i, lo, hi);
      lo = make_double2(0.0, 0.0);
      hi = lo;
      cs.i += wstride;
      more = seek_row();
    }
  }
  if constexpr (!kBulk) asm volatile("cp.async.wait_all;" ::: "memory");
  // kBulk: every issued copy was waited for (the issue cursor ends with the consume cursor)
}

// Opt-in (PPLOAD_SPMM=cp): measured slower than k_spmm_rows_v4 / k_spmm_store_v4 (16.0 vs 12.1 ms per
// products hop, profiles/r2/propagation_sliced.md): the per-lane 16-byte LDGSTS requests reach L2 as
// 25 sector requests per 400-B row instead of a warp LDG.128's 13, for the same DRAM bytes.
bool spmm_use_cp() {
  const char* e = getenv("PPLOAD_SPMM");
  return e && !strcmp(e, "cp");
}

cudaError_t launch_spmm_rows_cp(WaveArgs a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  int dev = 0, sms = 0, smem_max = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  a.nv = a.F / 4;
  const int row_bytes = a.nv * 16;
  const int variant = env_int("PPLOAD_CP_VARIANT", 0);
  struct V {
    void (*k)(WaveArgs);
    int threads, slots;
  };
  const V vs[] = {{k_spmm_rows_cp<1024, 16, false>, 1024, 16}, {k_spmm_rows_cp<1024, 8, false>, 1024, 8},
                  {k_spmm_rows_cp<512, 32, false>, 512, 32},  {k_spmm_rows_cp<1024, 12, false>, 1024, 12},
                  {k_spmm_rows_cp<1024, 12, true>, 1024, 12},  {k_spmm_rows_cp<1024, 8, true>, 1024, 8},
                  {k_spmm_rows_cp<512, 24, true>, 512, 24},    {k_spmm_rows_cp<256, 48, true>, 256, 48}};
  V v = vs[variant >= 0 && variant < 8 ? variant : 0];
  auto bytes = [&](const V& x) { return static_cast<int64_t>(x.threads / 32) * x.slots * (row_bytes + 8); };
  if (bytes(v) > smem_max) v = variant >= 4 ? vs[5] : vs[3];
  if (bytes(v) > smem_max) v = vs[1];
  const size_t smem = static_cast<size_t>(bytes(v));
  const int64_t grid = std::min<int64_t>(sms, (a.n + v.threads / 32 - 1) / (v.threads / 32));
  e = cudaFuncSetAttribute(v.k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  v.k<<<static_cast<uint32_t>(grid), v.threads, smem, st>>>(a);
  return cudaGetLastError();
}

bool spmm_wave_eligible(int32_t F, const void* src, int64_t src_stride, const void* dst, int64_t dst_stride) {
  return F % 4 == 0 && F <= 128 && reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(dst) % 16 == 0 && src_stride % 16 == 0 && dst_stride % 16 == 0;
}

// Opt-in (PPLOAD_SPMM=wave): measured 3-4x slower than the row kernels at products size although it
// cuts the DRAM reads by 30 % (r2 second session, profiles/r2/propagation_sliced.md): each warp's
// (window, group) step is a chain of dependent round trips -- cursor, column ids, weights, neighbour
// rows, partial sums -- for ~13 nonzeros, where the row kernel streams a row's nonzeros with its
// column ids prefetched; the 30 % fewer bytes do not pay for the lost memory-level parallelism.
bool spmm_use_wave(int64_t n, int32_t F) {
  (void)n;
  (void)F;
  const char* e = getenv("PPLOAD_SPMM");
  return e && !strcmp(e, "wave");
}

size_t spmm_wave_smem(int32_t F, int32_t R) { return static_cast<size_t>(R) * (static_cast<size_t>(F) * 8 + 24); }

cudaError_t launch_spmm_wave(WaveArgs a, unsigned* sync, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  int dev = 0, sms = 0, smem_max = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  a.nv = a.F / 4;
  const int per_row = a.F * 8 + 24;
  a.R = std::max(1, std::min(smem_max / per_row, env_int("PPLOAD_WAVE_ROWS", 1 << 30)));
  const int64_t grid = std::min<int64_t>(sms, (a.n + a.R - 1) / a.R);
  a.C = std::max(1, env_int("PPLOAD_WAVE_WINDOWS", 32));
  a.lag = std::max(0, env_int("PPLOAD_WAVE_LAG", 2));
  a.spin = env_int("PPLOAD_WAVE_SPIN", 20000);
  a.win = (a.ncols + a.C - 1) / a.C;
  a.sync = sync;
  const size_t smem = spmm_wave_smem(a.F, a.R);
  const int variant = env_int("PPLOAD_WAVE_VARIANT", 0);
  void (*kern)(WaveArgs) = variant == 1 ? k_spmm_wave<1024, 4> : variant == 2 ? k_spmm_wave<512, 4> : k_spmm_wave<512, 8>;
  const int threads = variant == 1 ? 1024 : 512;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess && a.lag > 0) e = cudaMemsetAsync(sync, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  kern<<<static_cast<uint32_t>(grid), threads, smem, st>>>(a);
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
