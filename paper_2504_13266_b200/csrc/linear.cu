// Fused batch assembly + first dense layer on the 5th-generation tensor cores
// (the consumer the paper's double-buffer pipeline feeds).
//
// Z[j, k, :] = cast_bf16(X_k[v_j, :]) @ W_k,  k = 0..H-1
// i.e. SIGN's per-hop linear transformation ("learns R+1 weight matrices for
// each hop"; Eq. (3) H = l(S_1..S_K)) applied
// to the batch the loader assembles, without the batch ever landing in HBM.
//
// B200 design (one persistent CTA per SM, 12 warps, 1 CTA/SM by shared memory):
//   * CTA (k, q): hop k = blockIdx % H; it keeps W_k^T resident in shared memory
//     (K-major, 128-byte swizzle, zero-padded to K = 128) and walks M-tiles of
//     128 batch rows q, q + Q, ...
//   * warps 0-3 (producers): thread r resolves batch row r (order -> node set ->
//     record), loads its hop-k fp32 vector with 128-bit loads, converts with
//     cvt.rn.bf16x2.f32 (the loader's RNE cast) and writes the 128 x 128 bf16 A
//     tile straight into the UMMA K-major SWIZZLE_128B layout (two stages),
//     then fence.proxy.async + mbarrier arrive.
//   * warp 4 (one elected lane): tcgen05.mma.cta_group::1.kind::f16, M = 128,
//     N = 256, K = 16 x 8 steps per accumulator; accumulators in TMEM (two
//     256-column fp32 buffers = all 512 columns); tcgen05.commit -> mbarriers.
//   * warps 8-11 (epilogue): tcgen05.ld 32x32b.x32 (each warp its 32-lane
//     quadrant), fp32 -> bf16 (or fp32), 128-bit stores of Z rows.
// HBM per batch row: H*F*4 read + H*D*s_z written (products, D = 512, bf16 Z:
// 1600 + 4096 B) instead of 1600 + 800 (gather) + 800 + 4096 (GEMM) unfused.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace ppl {

namespace {

constexpr int kLinThreads = 384;   // 12 warps
constexpr int kTileM = 128;        // batch rows per tile (UMMA M)
constexpr int kUmmaN = 256;        // columns per accumulator (UMMA N)
constexpr int kKPad = 128;         // F zero-padded to two 64-element K blocks
constexpr int kABytes = kTileM * kKPad * 2;  // 32 KB per A stage
constexpr int kStages = 2;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint4 ldg16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t bf16x2(uint32_t lo, uint32_t hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Byte offset of 16-byte chunk c (0..7) of row r inside a K-major SWIZZLE_128B
// block whose rows are 128 B (64 bf16): 8-row atoms of 1024 B, chunk index
// XOR-ed with the row's position in its atom.
__device__ __forceinline__ uint32_t sw128(uint32_t r, uint32_t c) { return r * 128u + ((c ^ (r & 7u)) << 4); }

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: start >> 4 (bits 0-13),
// LBO unused, SBO = 1024 B between 8-row atoms (bits 32-45), version 1 (bit
// 46), layout 2 = SWIZZLE_128B (bits 61-63).
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  return static_cast<uint64_t>((smem_addr(p) >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

// Instruction descriptor, kind::f16: D = F32 (bits 4-5 = 1), A = B = BF16 (bits
// 7-9, 10-12 = 1), both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kUmmaN >> 3) << 17) |
                            (static_cast<uint32_t>(kTileM >> 4) << 24);

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}

#define PPL_TMEM_LD32(taddr, v)                                                                                   \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                               \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),           \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),     \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),   \
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])    \
      : "r"(taddr))

}  // namespace

__global__ void __launch_bounds__(kLinThreads, 1) k_gather_linear(const LinearArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int D = a.D;
  uint8_t* w_s = smem;                                // [2 kb][D rows][128 B]
  uint8_t* a_s = smem + 2 * D * 128;                  // [kStages][2 kb][128 rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(a_s + kStages * kABytes);
  uint64_t* a_full = bars;                            // [kStages], 128 producer arrivals
  uint64_t* a_empty = bars + kStages;                 // [kStages], MMA commit
  uint64_t* t_full = bars + 2 * kStages;              // [2], MMA commit
  uint64_t* t_empty = bars + 2 * kStages + 2;         // [2], 128 epilogue arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.H, F = a.F;
  const int k = blockIdx.x % H;                       // this CTA's hop
  const int q = blockIdx.x / H, Q = gridDim.x / H;
  const int nh = D / kUmmaN;                          // accumulators per tile (1 or 2)

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      bar_init(&a_full[s], 128);
      bar_init(&a_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      bar_init(&t_full[h], 1);
      bar_init(&t_empty[h], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {  // TMEM: 512 fp32 columns x 128 lanes (two 256-column accumulators)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // W_k^T into shared memory: B operand row n = output column d, K index = f
  // (zero for f >= F).  Consecutive threads take consecutive d: coalesced reads.
  const __nv_bfloat16* wk = reinterpret_cast<const __nv_bfloat16*>(a.W) + static_cast<int64_t>(k) * F * D;
  for (int idx = threadIdx.x; idx < D * 16; idx += kLinThreads) {
    const int d = idx % D, c = idx / D, kb = c >> 3, cc = c & 7;
    uint16_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int f = kb * 64 + cc * 8 + j;
      v[j] = f < F ? __bfloat16_as_ushort(wk[static_cast<int64_t>(f) * D + d]) : 0;
    }
    const uint4 y = make_uint4(v[0] | (uint32_t(v[1]) << 16), v[2] | (uint32_t(v[3]) << 16),
                               v[4] | (uint32_t(v[5]) << 16), v[6] | (uint32_t(v[7]) << 16));
    *reinterpret_cast<uint4*>(w_s + kb * D * 128 + sw128(d, cc)) = y;
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t tiles_per_step = (a.B + kTileM - 1) / kTileM;
  const int64_t total = tiles_per_step * a.nsteps;
  // tile t -> (step, first row, rows); the same sequence in every role
  auto tile_rows = [&](int64_t t, int64_t& step, int& r0, int64_t& pos) -> int {
    step = t / tiles_per_step;
    r0 = static_cast<int>(t - step * tiles_per_step) * kTileM;
    pos = a.first_pos + step * a.step_stride;
    const int64_t nrows = min(static_cast<int64_t>(a.B), a.N - pos);
    return static_cast<int>(min(static_cast<int64_t>(kTileM), nrows - r0));
  };

  if (warp < 4) {
    // ---------------- producers: gather + cast into the swizzled A tile
    const int r = threadIdx.x;  // 0..127
    int i = 0;
    for (int64_t t = q; t < total; t += Q) {
      int64_t step, pos;
      int r0;
      const int rows = tile_rows(t, step, r0, pos);
      if (rows <= 0) continue;
      const int s = i & 1;
      bar_wait(&a_empty[s], ((i >> 1) & 1) ^ 1);
      uint8_t* at = a_s + s * kABytes;
      const uint8_t* src = nullptr;
      if (r < rows) {
        uint64_t v = a.order[pos + r0 + r];
        if (a.node_set != nullptr) v = static_cast<uint64_t>(a.node_set[v]);
        src = a.store + static_cast<int64_t>(v) * a.rec_stride + static_cast<int64_t>(k) * F * 4;
      }
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        uint4 x[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {  // 16 x 4 fp32 = this K block's 64 elements
          const int f = kb * 64 + j * 4;
          x[j] = (src != nullptr && f < F) ? ldg16(src + f * 4) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const uint4 y = make_uint4(bf16x2(x[2 * cc].x, x[2 * cc].y), bf16x2(x[2 * cc].z, x[2 * cc].w),
                                     bf16x2(x[2 * cc + 1].x, x[2 * cc + 1].y), bf16x2(x[2 * cc + 1].z, x[2 * cc + 1].w));
          *reinterpret_cast<uint4*>(at + kb * (kTileM * 128) + sw128(r, cc)) = y;
        }
      }
      fence_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
      bar_arrive(&a_full[s]);
      ++i;
    }
  } else if (warp == 4) {
    // ---------------- MMA issuer (one lane)
    if (lane == 0) {
      int i = 0;
      for (int64_t t = q; t < total; t += Q) {
        int64_t step, pos;
        int r0;
        if (tile_rows(t, step, r0, pos) <= 0) continue;
        const int s = i & 1;
        bar_wait(&a_full[s], (i >> 1) & 1);
        tc_fence_after();
        const uint8_t* at = a_s + s * kABytes;
        for (int h = 0; h < nh; ++h) {
          bar_wait(&t_empty[h], (i & 1) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < kKPad / 16; ++ks) {
            const int kb = ks >> 2, j = ks & 3;
            const uint64_t ad = sw128_desc(at + kb * (kTileM * 128)) + 2 * j;  // +32 B per 16-element step
            const uint64_t bd = sw128_desc(w_s + kb * D * 128 + h * kUmmaN * 128) + 2 * j;
            umma(tmem + h * kUmmaN, ad, bd, ks > 0 ? 1u : 0u);
          }
          umma_commit(&t_full[h]);
        }
        umma_commit(&a_empty[s]);  // the A stage is free once these MMAs have read it
        ++i;
      }
    }
    __syncwarp();
  } else if (warp >= 8) {
    // ---------------- epilogue: TMEM -> registers -> Z
    const int e = warp & 3;  // TMEM lane quadrant of this warp
    const int row = e * 32 + lane;
    int i = 0;
    for (int64_t t = q; t < total; t += Q) {
      int64_t step, pos;
      int r0;
      const int rows = tile_rows(t, step, r0, pos);
      if (rows <= 0) continue;
      for (int h = 0; h < nh; ++h) {
        bar_wait(&t_full[h], i & 1);
        tc_fence_after();
        uint8_t* zrow = a.Z + step * a.z_stride +
                        ((static_cast<int64_t>(r0 + row) * H + k) * D + h * kUmmaN) * a.z_elem;
#pragma unroll 1
        for (int c0 = 0; c0 < kUmmaN; c0 += 32) {
          uint32_t v[32];
          PPL_TMEM_LD32(tmem + (static_cast<uint32_t>(e * 32) << 16) + h * kUmmaN + c0, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (row < rows) {
            if (a.z_elem == 2) {
              uint4* dst = reinterpret_cast<uint4*>(zrow + c0 * 2);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                dst[j] = make_uint4(bf16x2(v[8 * j], v[8 * j + 1]), bf16x2(v[8 * j + 2], v[8 * j + 3]),
                                    bf16x2(v[8 * j + 4], v[8 * j + 5]), bf16x2(v[8 * j + 6], v[8 * j + 7]));
            } else {
              uint4* dst = reinterpret_cast<uint4*>(zrow + c0 * 4);
#pragma unroll
              for (int j = 0; j < 8; ++j) dst[j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
          }
        }
        tc_fence_before();
        bar_arrive(&t_empty[h]);
      }
      ++i;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

size_t linear_smem_bytes(int D) { return 1024 + 2 * static_cast<size_t>(D) * 128 + kStages * kABytes + 128; }

bool linear_supported(int H, int F, int D, int num_sms) {
  return F >= 1 && F <= kKPad && F % 4 == 0 && (D == 256 || D == 512) && H >= 1 && H <= num_sms;
}

cudaError_t launch_gather_linear(const LinearArgs& a, cudaStream_t st) {
  if (!linear_supported(a.H, a.F, a.D, a.num_sms)) return cudaErrorInvalidValue;
  const size_t smem = linear_smem_bytes(a.D);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_gather_linear, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(linear_smem_bytes(512)));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = (a.num_sms / a.H) * a.H;
  k_gather_linear<<<grid, kLinThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace ppl
