// TEST INFRASTRUCTURE (like oracle/): an independent, library implementation of Philox4x32-10 --
// cuRAND's own device routine curand_Philox4x32_10 (curand_philox4x32_x.h) -- that pins the
// oracle's Philox (O4), its unit-key word layout (O5) and the generator words (O11) on a B200
// (pins of the Philox row).  Shares nothing with the product library.
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include <cstdint>

__global__ void k_curand_philox(const uint4* __restrict__ ctr, const uint2* __restrict__ key, int64_t n,
                                uint4* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = curand_Philox4x32_10(ctr[i], key[i]);
}

// ctr: host [n][4] u32, key: host [n][2] u32 -> out: host [n][4] u32.  Returns a cudaError_t code.
extern "C" int cp_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
  if (n <= 0) return 0;
  uint4 *d_ctr = nullptr, *d_out = nullptr;
  uint2* d_key = nullptr;
  cudaError_t e = cudaMalloc(&d_ctr, n * 16);
  if (e == cudaSuccess) e = cudaMalloc(&d_key, n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, n * 16);
  if (e == cudaSuccess) e = cudaMemcpy(d_ctr, ctr, n * 16, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_key, key, n * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const int64_t blocks = (n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16;
    k_curand_philox<<<static_cast<unsigned>(blocks), 256>>>(d_ctr, d_key, n, d_out);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d_out, n * 16, cudaMemcpyDeviceToHost);
  cudaFree(d_ctr);
  cudaFree(d_key);
  cudaFree(d_out);
  return static_cast<int>(e);
}
