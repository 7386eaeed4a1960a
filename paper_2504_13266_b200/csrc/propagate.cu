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
