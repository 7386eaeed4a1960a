// Microbenchmark: TMEM -> register drain rate on sm_100a (experiment for the
// fused-linear epilogue).  One CTA per SM allocates all 512
// TMEM columns; `nw` drain warps (warp w reads lane quadrant w % 4, column
// group w / 4) repeatedly read the 128 x 512 fp32 accumulator with
// tcgen05.ld.32x32b.x32 and consume the values in one of several ways.
// Prints TMEM bytes read per SM clock for each variant.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_drain tmem_drain.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define LD32(taddr, v)                                                                                            \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                               \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),           \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),     \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),   \
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])    \
      : "r"(taddr))

#define LD16(taddr, v)                                                                                          \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
               "[%16];"                                                                                         \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), \
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),        \
                 "=r"(v[15])                                                                                    \
               : "r"(taddr))

#define WAIT_LD() asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory")

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t bf16x2(uint32_t lo, uint32_t hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<const uint32_t*>(&h);
}

// variant: 0 x32 wait each + xor; 1 two x32 per wait + xor; 2 x16 wait each + xor;
// 3 x32 wait each + cvt + st.shared; 4 software-pipelined x32 + xor;
// 5 software-pipelined x32 + cvt + st.shared; 6 four x32 per wait + xor
template <int V>
__global__ void __launch_bounds__(512, 1) k_drain(int nw, int reps, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) uint8_t stage[8][32 * 128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  uint32_t acc = 0;
  long long t0 = clock64();
  if (warp < nw) {
    const int e = warp & 3, g = warp >> 2, groups = nw / 4;
    const int cols = 512 / groups;
    const uint32_t base = tmem + (static_cast<uint32_t>(e * 32) << 16) + g * cols;
    uint8_t* my = stage[warp & 7] + lane * 128;
    for (int r = 0; r < reps; ++r) {
      if (V == 0 || V == 3) {
        for (int c = 0; c < cols; c += 32) {
          uint32_t v[32];
          LD32(base + c, v);
          WAIT_LD();
          if (V == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= v[j];
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              acc ^= v[j],
              *reinterpret_cast<uint4*>(my + (((j + (c & 32 ? 4 : 0)) ^ (lane & 7)) << 4)) =
                  make_uint4(bf16x2(v[8 * j], v[8 * j + 1]), bf16x2(v[8 * j + 2], v[8 * j + 3]),
                             bf16x2(v[8 * j + 4], v[8 * j + 5]), bf16x2(v[8 * j + 6], v[8 * j + 7]));
          }
        }
      } else if (V == 1) {
        for (int c = 0; c < cols; c += 64) {
          uint32_t v[32], w[32];
          LD32(base + c, v);
          LD32(base + c + 32, w);
          WAIT_LD();
#pragma unroll
          for (int j = 0; j < 32; ++j) acc ^= v[j] + w[j];
        }
      } else if (V == 6) {
        for (int c = 0; c < cols; c += 128) {
          uint32_t v[32], w[32], x[32], y[32];
          LD32(base + c, v);
          LD32(base + c + 32, w);
          LD32(base + c + 64, x);
          LD32(base + c + 96, y);
          WAIT_LD();
#pragma unroll
          for (int j = 0; j < 32; ++j) acc ^= (v[j] + w[j]) ^ (x[j] + y[j]);
        }
      } else if (V == 2) {
        for (int c = 0; c < cols; c += 16) {
          uint32_t v[16];
          LD16(base + c, v);
          WAIT_LD();
#pragma unroll
          for (int j = 0; j < 16; ++j) acc ^= v[j];
        }
      } else if (V == 4 || V == 5) {
        uint32_t v[32], w[32];
        LD32(base, v);
        WAIT_LD();
        for (int c = 0; c < cols; c += 64) {
          if (c + 32 < cols) LD32(base + c + 32, w);
          if (V == 4) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= v[j];
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(my + ((j ^ (lane & 7)) << 4)) =
                  make_uint4(bf16x2(v[8 * j], v[8 * j + 1]), bf16x2(v[8 * j + 2], v[8 * j + 3]),
                             bf16x2(v[8 * j + 4], v[8 * j + 5]), bf16x2(v[8 * j + 6], v[8 * j + 7]));
          }
          WAIT_LD();
          if (c + 64 < cols) LD32(base + c + 64, v);
          if (V == 4) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= w[j];
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(my + (((j + 4) ^ (lane & 7)) << 4)) =
                  make_uint4(bf16x2(w[8 * j], w[8 * j + 1]), bf16x2(w[8 * j + 2], w[8 * j + 3]),
                             bf16x2(w[8 * j + 4], w[8 * j + 5]), bf16x2(w[8 * j + 6], w[8 * j + 7]));
          }
          WAIT_LD();
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  if (acc == 0x12345678u) sink[threadIdx.x] = acc + stage[warp % 8][lane];
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int V>
void run(const char* name, int nw, int sms) {
  unsigned long long* d_cyc;
  uint32_t* d_sink;
  cudaMalloc(&d_cyc, sms * sizeof(unsigned long long));
  cudaMalloc(&d_sink, 1024 * 4);
  const int reps = 200;
  const int threads = (nw < 4 ? 4 : nw) * 32;
  k_drain<V><<<sms, threads>>>(nw, 2, d_cyc, d_sink);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_drain<V><<<sms, threads>>>(nw, reps, d_cyc, d_sink);
  cudaEventRecord(b);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[256];
  cudaMemcpy(h, d_cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  const double bytes = 128.0 * 512 * 4 * reps;  // per SM
  printf("{\"variant\": \"%s\", \"warps\": %d, \"err\": \"%s\", \"cycles\": %.0f, \"B_per_clk_per_sm\": %.1f, "
         "\"ms\": %.3f, \"TBs_chip\": %.2f}\n",
         name, nw, cudaGetErrorString(err), mean, bytes / mean, ms, bytes * sms / (ms * 1e-3) / 1e12);
  cudaFree(d_cyc);
  cudaFree(d_sink);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int nw : {4, 8, 16}) {
    run<0>("x32_wait_each_xor", nw, sms);
    run<1>("x32x2_per_wait_xor", nw, sms);
    run<6>("x32x4_per_wait_xor", nw, sms);
    run<2>("x16_wait_each_xor", nw, sms);
    run<3>("x32_wait_each_cvt_sts", nw, sms);
    run<4>("x32_pipelined_xor", nw, sms);
    run<5>("x32_pipelined_cvt_sts", nw, sms);
  }
  return 0;
}
