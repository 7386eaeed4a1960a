// gather4 alone: how fast can one SM pull random rows into shared memory with
// cp.async.bulk.tensor.2d.tile::gather4, as a function of box width, stages in flight and
// issuing warps -- with no MMA, conversion or epilogue behind it (DESIGN §11 / §17: the fused
// linear's A side sits at ~22 GB/s of gather4 bytes per SM). For comparison the same rows
// by LDG.128 (register staged, all loads of a warp in flight).
//
// Store: R rows of P bytes (products-shaped (node, hop) rows: 9.8 M x 400 B fp32, 3.9 GB > L2),
// row ids uniformly random (a fixed table), each CTA walks its own slice of the table.
// Output: one JSON line per configuration.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_rate gather4_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W;\n}\n" ::"r"(sa(b)),
      "r"(ph)
      : "memory");
}

// stages of 128 rows x box bytes; warps 0..nw-1 each issue 32 / nw gather4 per stage (lane 0);
// launched with max(nw, 4) warps
__global__ void __launch_bounds__(512, 1)
    k_gather4(const __grid_constant__ CUtensorMap map, const int32_t* __restrict__ rows, int64_t per_cta, int box_bytes,
              int stages, int nw, int nl, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < stages) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[threadIdx.x])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int32_t* my = rows + blockIdx.x * per_cta;
  const int64_t tiles = per_cta / 128;
  const int stage_bytes = 128 * box_bytes;
  const uint64_t mp = reinterpret_cast<uint64_t>(&map);
  auto issue = [&](int64_t t, int s) {
    if (warp < nw && lane < nl) {  // nl issuing lanes per warp, 32 / (nw nl) gather4 each
      if (warp == 0 && lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(stage_bytes)
                     : "memory");
      const int32_t* r = my + t * 128;
      const int per = 32 / (nw * nl), g0 = (warp * nl + lane) * per;
      for (int g = g0; g < g0 + per; ++g)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sa(sm + s * stage_bytes + g * 4 * box_bytes)),
            "l"(mp), "r"(0), "r"(r[4 * g]), "r"(r[4 * g + 1]), "r"(r[4 * g + 2]), "r"(r[4 * g + 3]), "r"(sa(&full[s]))
            : "memory");
    }
  };
  for (int s = 0; s < stages && s < tiles; ++s) issue(s, s);
  unsigned long long acc = 0;
  for (int64_t t = 0; t < tiles; ++t) {
    const int s = static_cast<int>(t % stages);
    bar_wait(&full[s], static_cast<uint32_t>((t / stages) & 1));
    acc += sm[s * stage_bytes + threadIdx.x];  // touch the data
    __syncthreads();                            // every thread is done with stage s
    if (t + stages < tiles) issue(t + stages, s);
  }
  if (acc == 0xffffffffffffULL) *sink = acc;
}

// the same rows by LDG.128: each warp takes rows, lane = 16-B piece, `inflight` rows per warp in flight
__global__ void __launch_bounds__(256) k_ldg(const uint8_t* __restrict__ base, const int32_t* __restrict__ rows,
                                             int64_t per_cta, int row_bytes, unsigned long long* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* my = rows + blockIdx.x * per_cta;
  const int pieces = row_bytes / 16;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int64_t i = warp * 8; i < per_cta; i += 8 * 8) {
    uint4 x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t r = my[i + u];
      x[u] = lane < pieces ? __ldg(reinterpret_cast<const uint4*>(base + r * row_bytes) + lane) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc.x ^= x[u].x ^ x[u].w;
  }
  if (acc.x == 0x12345678u) *sink = acc.x;
}

int main() {
  const int F = 100, P = F * 4;                    // products (node, hop) rows: 400 B
  const int64_t R = 2449029LL * 4;                 // 9.8 M rows, 3.9 GB
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint8_t* d_store;
  CK(cudaMalloc(&d_store, R * P));
  CK(cudaMemset(d_store, 1, R * P));
  const int64_t per_cta = 128 * 1024;              // 1024 tiles per CTA
  const int64_t nrows = per_cta * sms;
  std::vector<int32_t> h(nrows);
  uint64_t x = 0x9E3779B97F4A7C15ULL;
  for (auto& v : h) {
    x ^= x << 13, x ^= x >> 7, x ^= x << 17;
    v = static_cast<int32_t>(x % R);
  }
  int32_t* d_rows;
  CK(cudaMalloc(&d_rows, nrows * 4));
  CK(cudaMemcpy(d_rows, h.data(), nrows * 4, cudaMemcpyHostToDevice));
  unsigned long long* d_sink;
  CK(cudaMalloc(&d_sink, 8));
  CK(cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto encode = [&](CUtensorMap* m, int box) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(F), static_cast<cuuint64_t>(R)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(P)};
    const cuuint32_t bx[2] = {static_cast<cuuint32_t>(box), 1};
    const cuuint32_t es[2] = {1, 1};
    return cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, d_store, dims, strides, bx, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  const int boxes[3] = {32, 64, 128};
  for (int box : boxes) {
    CUtensorMap m;
    if (!encode(&m, box)) {
      printf("{\"kernel\": \"gather4\", \"box_elems\": %d, \"error\": \"encode\"}\n", box);
      continue;
    }
    const int bb = box * 4;
    const int cfgs[][2] = {{1, 1}, {4, 1}, {8, 1}, {16, 1}, {1, 4}, {1, 8}, {4, 2}, {4, 4}, {4, 8}};  // warps, lanes
    for (auto& c : cfgs)
      for (int stages : {2, 4}) {
        const int nw = c[0], nl = c[1];
        if (stages * 128 * bb > 200 * 1024) continue;
        const int thr = 32 * (nw < 4 ? 4 : nw);
        k_gather4<<<sms, thr, stages * 128 * bb>>>(m, d_rows, per_cta, bb, stages, nw, nl, d_sink);
        CK(cudaEventRecord(a));
        k_gather4<<<sms, thr, stages * 128 * bb>>>(m, d_rows, per_cta, bb, stages, nw, nl, d_sink);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double useful = static_cast<double>(nrows) * (box >= F ? P : bb);  // bytes of record data moved
        const double moved = static_cast<double>(nrows) * bb;
        printf("{\"kernel\": \"gather4\", \"box_elems\": %d, \"issuing_warps\": %d, \"issuing_lanes\": %d, \"stages\": %d, \"in_flight_KB\": %d, "
               "\"ms\": %.3f, \"smem_GBs\": %.1f, \"record_GBs\": %.1f, \"per_sm_GBs\": %.2f}\n",
               box, nw, nl, stages, stages * 128 * bb / 1024, ms, moved / ms / 1e6, useful / ms / 1e6, moved / ms / 1e6 / sms);
        fflush(stdout);
      }
  }
  for (int blocks_per_sm : {1, 2, 4}) {
    const int grid = sms * blocks_per_sm;
    const int64_t pc = nrows / grid;
    k_ldg<<<grid, 256>>>(d_store, d_rows, pc, P, d_sink);
    CK(cudaEventRecord(a));
    k_ldg<<<grid, 256>>>(d_store, d_rows, pc, P, d_sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double bytes = static_cast<double>(pc) * grid * P;
    printf("{\"kernel\": \"ldg128\", \"ctas_per_sm\": %d, \"rows_in_flight_per_warp\": 8, \"ms\": %.3f, \"record_GBs\": %.1f, "
           "\"per_sm_GBs\": %.2f}\n",
           blocks_per_sm, ms, bytes / ms / 1e6, bytes / ms / 1e6 / sms);
    fflush(stdout);
  }
  return 0;
}
