// Microbenchmark: HBM3e streaming bandwidth on B200 for different read:write
// mixes, to put the gather's roofline (2 bytes read per byte written for
// fp32 -> bf16 batches; the fused linear writes 2.56 bytes per byte read)
// next to the 1:1 copy figure of MEASURED_PEAKS.json.
// R read streams and Wr write streams of 16-byte vectors, fully coalesced,
// 4 independent iterations per thread in flight, buffers far larger than L2.
// Prints one JSON line per (mix, CTAs per SM): best of 10 launches, CUDA events.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_mix hbm_mix.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint4 ld_nc(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// n vectors per stream; stream s of the input starts at in + s*n, of the output at out + s*n.
template <int R, int Wr>
__global__ void __launch_bounds__(256) k_mix(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t n,
                                             uint32_t* __restrict__ sink) {
  constexpr int U = 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n; i0 += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = make_uint4(static_cast<uint32_t>(i0), 1, 2, 3);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        if (i < n) {
          const uint4 x = ld_nc(in + r * n + i);
          v[u].x ^= x.x;
          v[u].y ^= x.y;
          v[u].z ^= x.z;
          v[u].w ^= x.w;
        }
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
#pragma unroll
        for (int w = 0; w < Wr; ++w) out[w * n + i] = make_uint4(v[u].x + w, v[u].y, v[u].z, v[u].w);
        if (Wr == 0) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
      }
    }
  }
  if (Wr == 0 && acc == 0x12345678u) sink[0] = acc;
}

template <typename F>
static float best_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

template <int R, int Wr>
static void run(const char* name, const uint4* in, uint4* out, int64_t total_vec, uint32_t* sink, int grid,
                int per_sm) {
  // the same total traffic (in + out streams) for every mix
  const int64_t n = total_vec / (R + Wr);
  const float ms = best_ms([&] { k_mix<R, Wr><<<grid, 256>>>(in, out, n, sink); });
  printf("{\"mix\": \"%s\", \"read_streams\": %d, \"write_streams\": %d, \"ctas_per_sm\": %d, \"GBs\": %.1f}\n", name,
         R, Wr, per_sm, static_cast<double>(n) * 16 * (R + Wr) / ms / 1e6);
}

int main() {
  const int64_t bytes = int64_t(6) << 30;  // 6 GiB per buffer
  uint4 *in, *out;
  uint32_t* sink;
  if (cudaMalloc(&in, bytes) != cudaSuccess || cudaMalloc(&out, bytes) != cudaSuccess ||
      cudaMalloc(&sink, 4) != cudaSuccess) {
    fprintf(stderr, "alloc failed\n");
    return 1;
  }
  cudaMemset(in, 1, bytes);
  cudaMemset(out, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t tv = bytes / 16;  // traffic budget: 6 GiB moved per launch
  for (int per_sm : {4, 8}) {
    const int g = sms * per_sm;
    run<1, 0>("read only", in, out, tv, sink, g, per_sm);
    run<0, 1>("write only", in, out, tv, sink, g, per_sm);
    run<1, 1>("1:1 copy", in, out, tv, sink, g, per_sm);
    run<2, 1>("2:1 (gather fp32->bf16)", in, out, tv, sink, g, per_sm);
    run<4, 1>("4:1", in, out, tv, sink, g, per_sm);
    run<2, 5>("2:5 (fused linear ~1:2.56)", in, out, tv, sink, g, per_sm);
    run<1, 2>("1:2", in, out, tv, sink, g, per_sm);
  }
  fflush(stdout);
  return 0;
}
