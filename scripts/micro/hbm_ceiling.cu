// Microbenchmark: the HBM3e streaming ceiling of this B200 by read:write mix, with enough bytes in
// flight to saturate it (r1's hbm_mix.cu kept 4 x 16 B per thread in flight and measured below what
// the chunk-reshuffle gather itself reaches).  R read streams and Wr write streams; each CTA streams
// one contiguous block of every stream (the access shape of chunk reads); per thread U 32-byte
// loads (LDG.256) per read stream in flight before any store; buffers far larger than L2.
// Sweeps CTAs per SM x U and prints one JSON line per (mix, config) plus the best per mix.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_ceiling hbm_ceiling.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

struct V8 {
  uint32_t x[8];
};

__device__ __forceinline__ V8 ld256(const V8* p) {
  V8 v;
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.x[0]), "=r"(v.x[1]), "=r"(v.x[2]), "=r"(v.x[3]), "=r"(v.x[4]), "=r"(v.x[5]), "=r"(v.x[6]),
                 "=r"(v.x[7])
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st256(V8* p, const V8& v) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.x[0]), "r"(v.x[1]), "r"(v.x[2]),
               "r"(v.x[3]), "r"(v.x[4]), "r"(v.x[5]), "r"(v.x[6]), "r"(v.x[7])
               : "memory");
}

// n 32-byte vectors per stream; CTA b owns [b*per, (b+1)*per) of every stream.
template <int R, int Wr, int U>
__global__ void __launch_bounds__(256) k_stream(const V8* __restrict__ in, V8* __restrict__ out, int64_t n,
                                                uint32_t* __restrict__ sink) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  uint32_t acc = 0;
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += U * blockDim.x) {
    V8 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) v[u].x[k] = static_cast<uint32_t>(i0) + k;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      V8 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * static_cast<int64_t>(blockDim.x);
        if (i < hi) x[u] = ld256(in + r * n + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) v[u].x[k] ^= x[u].x[k];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * static_cast<int64_t>(blockDim.x);
      if (i < hi) {
#pragma unroll
        for (int w = 0; w < Wr; ++w) st256(out + w * n + i, v[u]);
        if (Wr == 0)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc ^= v[u].x[k];
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
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

template <int R, int Wr, int U>
static double run1(const char* name, const V8* in, V8* out, int64_t total_vec, uint32_t* sink, int sms, int per_sm) {
  const int64_t n = total_vec / (R + Wr);  // the same total traffic for every mix
  const float ms = best_ms([&] { k_stream<R, Wr, U><<<sms * per_sm, 256>>>(in, out, n, sink); });
  const double gbs = static_cast<double>(n) * 32 * (R + Wr) / ms / 1e6;
  printf("{\"mix\": \"%s\", \"read_streams\": %d, \"write_streams\": %d, \"ctas_per_sm\": %d, \"vec32_in_flight\": %d, "
         "\"GBs\": %.1f}\n",
         name, R, Wr, per_sm, U * R, gbs);
  return gbs;
}

template <int R, int Wr>
static void run(const char* name, const V8* in, V8* out, int64_t tv, uint32_t* sink, int sms) {
  double best = 0;
  for (int per_sm : {2, 4, 8}) {
    double g = run1<R, Wr, 2>(name, in, out, tv, sink, sms, per_sm);
    best = g > best ? g : best;
    g = run1<R, Wr, 4>(name, in, out, tv, sink, sms, per_sm);
    best = g > best ? g : best;
  }
  printf("{\"mix\": \"%s\", \"best_GBs\": %.1f}\n", name, best);
  fflush(stdout);
}

int main() {
  const int64_t bytes = int64_t(8) << 30;  // 8 GiB per buffer
  V8 *in, *out;
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
  const int64_t tv = bytes / 32;  // traffic per launch: 8 GiB
  run<1, 0>("read only", in, out, tv, sink, sms);
  run<0, 1>("write only", in, out, tv, sink, sms);
  run<1, 1>("1:1 copy", in, out, tv, sink, sms);
  run<2, 1>("2:1 (gather fp32->bf16)", in, out, tv, sink, sms);
  run<4, 1>("4:1", in, out, tv, sink, sms);
  run<2, 5>("2:5 (fused linear ~1:2.56)", in, out, tv, sink, sms);
  return 0;
}
