/* Per-batch C-ABI benchmark: one pp_next_batch call (one launch) per batch from C,
 * i.e. what a native trainer linking libppload.so sees without Python in the loop.
 * ogbn-products-shaped store (N = 2,449,029, F = 100, K = 3, fp32 -> bf16, B = 8192),
 * synthetic values (pp_fill_synthetic), next epoch's order prefetched.
 * Prints one JSON line.  Usage: pp_bench_c [epochs] [batches_per_call] */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../include/pp_loader.h"

#define CK(x)                                                                          \
  do {                                                                                 \
    int _s = (int)(x);                                                                 \
    if (_s != 0) {                                                                     \
      fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, _s, pp_last_error()); \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

int main(int argc, char** argv) {
  const int epochs = argc > 1 ? atoi(argv[1]) : 10;
  const int k = argc > 2 ? atoi(argv[2]) : 1;
  const int64_t N = 2449029;
  const int H = 4, F = 100, B = 8192;
  pp_loader_desc d = {0};
  d.hops.num_nodes = N;
  d.hops.num_hops = H;
  d.hops.feat_dim = F;
  d.hops.dtype = PP_F32;
  d.batch_size = B;
  d.out_dtype = PP_BF16;
  d.world_size = 1;
  d.peers = PP_PEERS_NONE;
  pp_loader* L = NULL;
  CK(pp_loader_create(&d, &L));
  CK(pp_fill_synthetic(L, 2504));
  pp_loader_info info;
  CK(pp_loader_query(L, &info));
  const int64_t steps = info.steps_per_epoch;
  const size_t slot = (size_t)B * H * F * 2;
  void* ring = NULL;
  CK(cudaMalloc(&ring, slot * steps));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(pp_set_stream(L, st));
  int32_t rows[512];
  int32_t done_n;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int e = 0; e < 3 + epochs; ++e) {
    if (e == 3) CK(cudaEventRecord(a, st));
    CK(pp_epoch_permute(L, 250413266ull + e, 1, st));
    CK(pp_epoch_prefetch(L, 250413266ull + e + 1, 1));
    for (int64_t t = 0; t < steps;) {
      if (k == 1) {
        CK(pp_next_batch(L, (char*)ring + t * slot, NULL, NULL, rows, st));
        t += 1;
      } else {
        CK(pp_next_batches(L, k, (char*)ring + t * slot, (int64_t)slot, NULL, NULL, rows, &done_n, st));
        t += done_n;
      }
    }
  }
  CK(cudaEventRecord(b, st));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double per_epoch_ms = ms / epochs;
  const double gbs = (double)N * (1600 + 800 + 4) / (per_epoch_ms * 1e-3) / 1e9;
  printf("{\"tool\": \"pp_bench_c\", \"batches_per_call\": %d, \"epochs\": %d, \"ms_per_epoch\": %.4f, "
         "\"nodes_per_s\": %.4e, \"algorithmic_GBs_incl_permute\": %.1f}\n",
         k, epochs, per_epoch_ms, N / (per_epoch_ms * 1e-3), gbs);
  cudaFree(ring);
  pp_loader_destroy(L);
  return 0;
}
