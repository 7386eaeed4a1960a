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
