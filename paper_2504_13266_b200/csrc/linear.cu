// Fused batch assembly + first dense layer on the 5th-generation tensor cores
// (the consumer the paper's double-buffer pipeline feeds).
//
// Z[j, k, :] = cast_bf16(X_k[v_j, :]) @ W_k,  k = 0..H-1
// i.e. SIGN's per-hop linear transformation ("learns R+1 weight matrices for
// each hop"; Eq. (3) H = l(S_1..S_K)) applied
// to the batch the loader assembles, without the batch ever landing in HBM.
//
// B200 design (one persistent CTA per SM, 12 warps, 1 CTA/SM by shared memory):
//   * CTA (k, q): hop k = blockIdx % H; it keeps W_k resident in shared memory,
//     loaded by TMA straight from the caller's [F][D] tensor as the MN-major
//     SWIZZLE_128B B operand (64-column boxes of 128 K rows, rows >= F zero-filled
//     by the TMA out-of-bounds fill), and walks M-tiles of 128 batch rows q, q + Q, ...
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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "internal.h"

namespace ppl {

namespace {

#ifndef PPL_LIN_EPIWARPS
#define PPL_LIN_EPIWARPS 4
#endif
// Warp roles.  4 epilogue warps: 0-7 producers, 8 MMA, 9-11 idle, 12-15 epilogue.
// 8 epilogue warps: 0-7 producers, 8-15 epilogue (two per TMEM lane quadrant, each
// draining half of the columns), 16 MMA -- 17 warps, so ptxas still gets 120 registers.
constexpr int kEpiWarps = PPL_LIN_EPIWARPS;
constexpr int kLinThreads = (kEpiWarps == 8 ? 17 : 16) * 32;
constexpr int kProducerWarps = 8;
constexpr int kProducerThreads = kProducerWarps * 32;
constexpr int kMmaWarp = kEpiWarps == 8 ? 16 : 8;
constexpr int kEpiWarp0 = kEpiWarps == 8 ? 8 : 12;  // epilogue warp w: lane quadrant w % 4, column group (w - kEpiWarp0) / 4
constexpr int kEpiGroups = kEpiWarps / 4;
static_assert(kEpiWarps == 4 || kEpiWarps == 8, "4 or 8 epilogue warps");
constexpr int kTileM = 128;        // batch rows per tile (UMMA M)
constexpr int kUmmaN = 256;        // columns per accumulator (UMMA N)
constexpr int kKPad = 128;         // F zero-padded to two 64-element K blocks
constexpr int kABytes = kTileM * kKPad * 2;  // 32 KB per A stage
#ifndef PPL_LIN_STAGES
#define PPL_LIN_STAGES 2
#endif
#ifndef PPL_LIN_EPIBUFS
#define PPL_LIN_EPIBUFS 2
#endif
constexpr int kStages = PPL_LIN_STAGES;  // A-tile stages
constexpr int kStageBytes = 32 * 128;  // epilogue staging: 32 rows x 128 B, 16-byte chunks XOR-swizzled by row
constexpr int kEpiBufs = PPL_LIN_EPIBUFS;  // staging buffers per epilogue warp
#ifndef PPL_LIN_GROUP
#define PPL_LIN_GROUP 1
#endif
constexpr int kEpiGroup = PPL_LIN_GROUP;   // slices staged per fence + TMA issue round
static_assert(kEpiBufs % kEpiGroup == 0 && kEpiBufs / kEpiGroup >= 1, "staging buffers per group");
#ifndef PPL_LIN_PFDIST
#define PPL_LIN_PFDIST 1
#endif
constexpr int kPf = PPL_LIN_PFDIST;  // L2 prefetch distance of the producers, in tiles
constexpr int kWBox = kKPad * 128;  // one TMA box of W_k: 128 K rows x 64 columns (128 B)

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

__device__ __forceinline__ uint4 lds16(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr)
               : "memory");
  return r;
}
__device__ __forceinline__ void sts16(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
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

// B operand, MN-major SWIZZLE_128B: canonical ((8,n),(8,k)):((1,LBO),(8,SBO)) in
// 16-byte units -- 64 consecutive columns per 128-byte row, one row per K index,
// LBO = 16 KB between 64-column boxes, SBO = 1024 B between 8-row K groups.
__device__ __forceinline__ uint64_t sw128_mn_desc(const void* p) {
  return static_cast<uint64_t>((smem_addr(p) >> 4) & 0x3FFFu) | (static_cast<uint64_t>(kWBox >> 4) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor, kind::f16: D = F32 (bits 4-5 = 1), A = B = BF16 (bits
// 7-9, 10-12 = 1), A K-major, B MN-major (bit 16), N >> 3 at bits 17-22, M >> 4
// at bits 24-28.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                            (static_cast<uint32_t>(kUmmaN >> 3) << 17) | (static_cast<uint32_t>(kTileM >> 4) << 24);

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

// Experiment probe (LinearArgs::ts, PPLOAD_DEBUG_TS): %globaltimer at named
// points of CTA 0's first kDbgTiles tiles, kDbgSlots per tile.
constexpr int kDbgTiles = 24, kDbgSlots = 14;
// after the tile slots: per CTA {entry, W copy issued, prologue done, exit}
__device__ __forceinline__ void dbg_cta(const LinearArgs& a, int slot) {
  if (a.ts == nullptr || threadIdx.x != 0) return;
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  a.ts[kDbgTiles * kDbgSlots + 4 * blockIdx.x + slot] = t;
}
__device__ __forceinline__ void dbg_ts(const LinearArgs& a, int tile, int slot, int) {
  if (tile >= kDbgTiles) return;
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  a.ts[tile * kDbgSlots + slot] = t;
}

}  // namespace

__global__ void __launch_bounds__(kLinThreads, 1)
    k_gather_linear(const LinearArgs a, const __grid_constant__ CUtensorMap zmap,
                    const __grid_constant__ CUtensorMap wmap) {
  extern __shared__ uint8_t smem_raw[];
  // consecutive fused launches of one epoch are independent: let the next one's CTAs
  // take SMs as soon as this grid's CTAs leave them (see launch_gather_linear)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  dbg_cta(a, 0);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int D = a.D;
  uint8_t* w_s = smem;                                // [D / 64 boxes][128 K rows][128 B]
  uint8_t* a_s = smem + (D / 64) * kWBox;            // [kStages][2 kb][128 rows][128 B]
  uint8_t* z_s = a_s + kStages * kABytes;             // [epilogue warps][kEpiBufs][32 rows][128 B] staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(z_s + kEpiWarps * kEpiBufs * kStageBytes);
  uint64_t* a_full = bars;                            // [kStages], kProducerThreads arrivals
  uint64_t* a_empty = bars + kStages;                 // [kStages], MMA commit
  uint64_t* t_full = bars + 2 * kStages;              // [2], MMA commit
  uint64_t* t_empty = bars + 2 * kStages + 2;         // [2], 128 epilogue arrivals
  uint64_t* w_full = bars + 2 * kStages + 4;          // W image landed (bulk copy)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 5);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.H, F = a.F;
  const int k = blockIdx.x % H;                       // this CTA's hop
  const int q = blockIdx.x / H, Q = gridDim.x / H;
  const int nh = D / kUmmaN;                          // accumulators per tile (1 or 2)
  const int nks = (F + 15) / 16;                      // K steps: columns past F are zero, only whole 16-steps past it are skipped

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      bar_init(&a_full[s], kProducerThreads);
      bar_init(&a_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      bar_init(&t_full[h], 1);
      // arrivals: every epilogue thread whose column group overlaps accumulator h
      uint32_t cnt = 0;
      for (int g = 0; g < kEpiGroups; ++g) {
        const int lo = g * D / kEpiGroups, hi = (g + 1) * D / kEpiGroups;
        if (lo < (h + 1) * kUmmaN && hi > h * kUmmaN) cnt += 128;
      }
      bar_init(&t_empty[h], cnt > 0 ? cnt : 1);
    }
    bar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {  // TMEM: 512 fp32 columns x 128 lanes (two 256-column accumulators)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // W_k into shared memory: D / 64 TMA boxes straight from the caller's tensor
  // (MN-major B operand; K rows >= F are zero-filled out of bounds), completed on
  // w_full; only the MMA issuer waits for it, so the producers start gathering at once.
  if (threadIdx.x == 0) {
    const uint32_t nbox = static_cast<uint32_t>(D / 64);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(w_full)),
                 "r"(nbox * kWBox)
                 : "memory");
    const uint64_t wmap_addr = reinterpret_cast<uint64_t>(&wmap);
    for (uint32_t b = 0; b < nbox; ++b)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(smem_addr(w_s + b * kWBox)),
          "l"(wmap_addr), "r"(static_cast<int>(b * 64)), "r"(0), "r"(k), "r"(smem_addr(w_full))
          : "memory");
  }
  dbg_cta(a, 1);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  dbg_cta(a, 2);

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

  if (warp < kProducerWarps) {
    // ---------------- producers: gather + cast into the swizzled A tile.
    // Warp w owns tile rows 16w..16w+15; for each row the 32 lanes load the
    // row's hop-k vector as consecutive 16-byte pieces (one coalesced request
    // per row, lane l = fp32 elements 4l..4l+3, zero past F); all 16 rows are
    // in flight before any is converted.  Even lanes then pair with their odd
    // neighbour to form one 16-byte chunk of 8 bf16 = K elements 8c..8c+7.
    const int rbase = warp * 16;
    auto next_tile = [&](int64_t t) -> int64_t {  // first non-empty tile at or after t
      for (; t < total; t += Q) {
        int64_t st_, ps_;
        int r_;
        if (tile_rows(t, st_, r_, ps_) > 0) return t;
      }
      return total;
    };
    // Lane layout: half-warp hw = lane / 16 takes row 2 it + hw of iteration it,
    // lane c = lane % 16 the K chunk 8c..8c+7 (two 16-byte fp32 loads -> one
    // 16-byte bf16 store), so no shuffles are needed to pair elements.
    const int hw = lane >> 4, c = lane & 15;
    // order[] entry of tile row rbase + lane (lanes < 16), kNoRow past the batch.
    // Fetched one tile ahead: under the Z write stream an order[] read costs a
    // DRAM round trip, which would otherwise precede every tile's data loads.
    constexpr uint32_t kNoRow = 0xffffffffu;
    auto fetch_index = [&](int64_t t) -> uint32_t {
      if (t >= total) return kNoRow;
      int64_t step, pos;
      int r0;
      const int rows = tile_rows(t, step, r0, pos);
      uint32_t v = kNoRow;
      if (lane < 16 && rbase + lane < rows)
        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(a.order + pos + r0 + rbase + lane));
      return v;
    };
    auto load_tile = [&](uint32_t idx, uint4(&x)[16]) {
      const uint8_t* my_src = nullptr;  // lane j < 16 resolves row rbase + j
      if (idx != kNoRow) {
        uint64_t v = idx;
        if (a.node_set != nullptr) v = static_cast<uint64_t>(a.node_set[v]);
        my_src = a.store + static_cast<int64_t>(v) * a.rec_stride + static_cast<int64_t>(k) * F * 4;
      }
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const uint8_t* src = reinterpret_cast<const uint8_t*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_src), 2 * it + hw));
        const bool on = src != nullptr && !(a.debug & 1);
        // K block 0: elements 4c..4c+3, K block 1: 64+4c..64+4c+3 (each load 256 contiguous bytes per half-warp)
        x[2 * it] = (on && 4 * c < F) ? ldg16(src + c * 16) : make_uint4(0, 0, 0, 0);
        x[2 * it + 1] = (on && 64 + 4 * c < F) ? ldg16(src + 256 + c * 16) : make_uint4(0, 0, 0, 0);
      }
    };
    const bool dbg_lane = a.ts != nullptr && blockIdx.x == 0 && warp == 0 && lane == 0;
    auto store_tile = [&](int i, const uint4(&x)[16]) {
      const int s = i % kStages;
      if (dbg_lane) dbg_ts(a, i, 0, 0);
      bar_wait(&a_empty[s], ((i / kStages) & 1) ^ 1);
      if (dbg_lane) dbg_ts(a, i, 1, 0);
      uint8_t* at = a_s + s * kABytes;
#pragma unroll
      for (int it = 0; it < ((a.debug & 8) ? 0 : 8); ++it) {
        const uint4 x0 = x[2 * it], x1 = x[2 * it + 1];
        const int r = rbase + 2 * it + hw;
        // 4 bf16 = 8 bytes: half (c & 1) of 16-byte chunk c >> 1, in K block 0 and K block 1
        const uint32_t off = sw128(r, c >> 1) + (c & 1) * 8;
        *reinterpret_cast<uint2*>(at + off) = make_uint2(bf16x2(x0.x, x0.y), bf16x2(x0.z, x0.w));
        *reinterpret_cast<uint2*>(at + kTileM * 128 + off) = make_uint2(bf16x2(x1.x, x1.y), bf16x2(x1.z, x1.w));
      }
      fence_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
      bar_arrive(&a_full[s]);
      if (dbg_lane) dbg_ts(a, i, 2, 0);
    };
    // The next tile's rows are pulled into L2 with one bulk prefetch per row
    // (no registers, no shared memory) while this tile's loads are in flight,
    // so its own loads are L2 hits; order[] entries are fetched two tiles ahead.
    auto prefetch_rows = [&](uint32_t idx) {
      if (idx == kNoRow || (a.debug & 1)) return;
      uint64_t v = idx;
      if (a.node_set != nullptr) v = static_cast<uint64_t>(a.node_set[v]);
      const uint8_t* p = a.store + static_cast<int64_t>(v) * a.rec_stride + static_cast<int64_t>(k) * F * 4;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(F * 4) : "memory");
    };
    uint4 x[16];
    int i = 0;
    // tiles t[0] (loading now), t[1..kPf]; idx[d] = this lane's order[] entry of t[d].
    // Rows of t[kPf] are prefetched into L2 while t[0] is loaded (kPf tiles ahead).
    int64_t tq[kPf + 1];
    uint32_t idx[kPf + 1];
    tq[0] = next_tile(q);
#pragma unroll
    for (int d = 1; d <= kPf; ++d) tq[d] = tq[d - 1] < total ? next_tile(tq[d - 1] + Q) : total;
#pragma unroll
    for (int d = 0; d <= kPf; ++d) idx[d] = fetch_index(tq[d]);
#pragma unroll
    for (int d = 1; d < kPf; ++d)
      if (a.l2_prefetch) prefetch_rows(idx[d]);  // the first kPf - 1 tiles ahead
    while (tq[0] < total) {
      const int64_t tn = tq[kPf] < total ? next_tile(tq[kPf] + Q) : total;
      load_tile(idx[0], x);
      if (a.l2_prefetch) prefetch_rows(idx[kPf]);
#pragma unroll
      for (int d = 0; d < kPf; ++d) {
        idx[d] = idx[d + 1];
        tq[d] = tq[d + 1];
      }
      tq[kPf] = tn;
      idx[kPf] = fetch_index(tn);  // in flight together with this tile's data loads
      store_tile(i++, x);
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer (one lane)
    if (lane == 0) {
      bar_wait(w_full, 0);
      int i = 0;
      for (int64_t t = q; t < total; t += Q) {
        int64_t step, pos;
        int r0;
        if (tile_rows(t, step, r0, pos) <= 0) continue;
        const int s = i % kStages;
        const bool dbg_lane = a.ts != nullptr && blockIdx.x == 0;
        bar_wait(&a_full[s], (i / kStages) & 1);
        tc_fence_after();
        if (dbg_lane) dbg_ts(a, i, 3, 0);
        const uint8_t* at = a_s + s * kABytes;
        for (int h = 0; h < nh; ++h) {
          bar_wait(&t_empty[h], (i & 1) ^ 1);
          tc_fence_after();
          if (dbg_lane) dbg_ts(a, i, 4 + 2 * h, 0);
#pragma unroll
          for (int ks = 0; ks < ((a.debug & 64) ? 0 : nks); ++ks) {
            const int kb = ks >> 2, j = ks & 3;
            const uint64_t ad = sw128_desc(at + kb * (kTileM * 128)) + 2 * j;  // +32 B per 16-element step
            const uint64_t bd = sw128_mn_desc(w_s + h * (kUmmaN / 64) * kWBox + ks * 2048);  // 16 K rows per step
            umma(tmem + h * kUmmaN, ad, bd, ks > 0 ? 1u : 0u);
          }
          umma_commit(&t_full[h]);
          if (dbg_lane) dbg_ts(a, i, 5 + 2 * h, 0);
        }
        umma_commit(&a_empty[s]);  // the A stage is free once these MMAs have read it
        ++i;
      }
    }
    __syncwarp();
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue: TMEM -> registers -> swizzled shared staging -> TMA store.
    // One warp per TMEM lane quadrant (warp % 4); lane l holds row 32e + l
    // after tcgen05.ld.  Each 128-byte slice of the warp's 32 rows (64 bf16 /
    // 32 fp32 columns) is staged with 16-byte chunks XOR-swizzled by row (the
    // TMA SWIZZLE_128B pattern, conflict-free) and written to Z by one
    // cp.async.bulk.tensor store (box 32 rows x 128 B); two staging buffers
    // per warp so the next slice is converted while the previous one drains.
    // A warp whose 32 rows run past the batch (the ragged last step) or a Z
    // without a tensor map writes the staged rows with 16-byte stores instead.
    const int e = warp & 3;                          // TMEM lane quadrant
    const int grp = (warp - kEpiWarp0) >> 2;         // column group
    uint8_t* sbuf = z_s + (warp - kEpiWarp0) * kEpiBufs * kStageBytes;
    const bool dbg_lane = a.ts != nullptr && blockIdx.x == 0 && warp == kEpiWarp0 && lane == 0;
    const int cols_per_slice = 128 / a.z_elem;
    const uint64_t zmap_addr = reinterpret_cast<uint64_t>(&zmap);
    int i = 0, slice = 0;
    for (int64_t t = q; t < total; t += Q) {
      int64_t step, pos;
      int r0;
      const int rows = tile_rows(t, step, r0, pos);
      if (rows <= 0) continue;
      const bool tma_rows = a.z_tma && e * 32 + 32 <= rows;
      for (int h = 0; h < nh; ++h) {
        // this warp's columns of accumulator h: [c_lo, c_hi)
        const int c_lo = max(grp * D / kEpiGroups, h * kUmmaN) - h * kUmmaN;
        const int c_hi = min((grp + 1) * D / kEpiGroups, (h + 1) * kUmmaN) - h * kUmmaN;
        if (c_lo >= c_hi) continue;
        bar_wait(&t_full[h], i & 1);
        tc_fence_after();
        if (dbg_lane) dbg_ts(a, i, 12 + h, 0);
        // Software-pipelined: the next slice's tcgen05.ld is issued right after this
        // slice is staged, so its TMEM latency overlaps the fence + TMA store issue.
        const uint32_t trow = tmem + (static_cast<uint32_t>(e * 32) << 16) + h * kUmmaN;
        const int c_end = (a.debug & 4) ? c_lo : c_hi;
        uint32_t v[64];
        auto ld_slice = [&](int c0) {
          PPL_TMEM_LD32(trow + c0, v);
          if (a.z_elem == 2) PPL_TMEM_LD32(trow + c0 + 32, (v + 32));
        };
        if (c_lo < c_end) ld_slice(c_lo);
        // kEpiGroup slices are staged per fence.proxy.async + TMA issue round (the fence waits
        // for the staging stores to land, so grouping amortises that wait); one bulk group per round
#pragma unroll 1
        for (int g0 = c_lo; g0 < c_end; g0 += cols_per_slice * kEpiGroup) {
          // the bulk stores issued from these buffers kEpiBufs / kEpiGroup rounds ago must have read them
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kEpiBufs / kEpiGroup - 1) : "memory");
          __syncwarp();
          uint8_t* sbs[kEpiGroup];
          int ng = 0;
#pragma unroll
          for (int g = 0; g < kEpiGroup; ++g) {
            const int c0 = g0 + g * cols_per_slice;
            if (c0 >= c_end) break;
            uint8_t* sb = sbuf + (slice % kEpiBufs) * kStageBytes;
            ++slice;
            sbs[g] = sb;
            ++ng;
            uint8_t* my = sb + lane * 128;
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (a.z_elem == 2) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<uint4*>(my + ((j ^ (lane & 7)) << 4)) =
                    make_uint4(bf16x2(v[8 * j], v[8 * j + 1]), bf16x2(v[8 * j + 2], v[8 * j + 3]),
                               bf16x2(v[8 * j + 4], v[8 * j + 5]), bf16x2(v[8 * j + 6], v[8 * j + 7]));
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<uint4*>(my + ((j ^ (lane & 7)) << 4)) =
                    make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
            if (c0 + cols_per_slice < c_end) ld_slice(c0 + cols_per_slice);
            if ((a.debug & 2) || tma_rows) continue;
            __syncwarp();
#pragma unroll
            for (int it = 0; it < 8; ++it) {  // 4 rows x 128 contiguous bytes per instruction
              const int rr = it * 4 + (lane >> 3), ch = lane & 7;
              const uint4 y = *reinterpret_cast<const uint4*>(sb + rr * 128 + ((ch ^ (rr & 7)) << 4));
              if (e * 32 + rr < rows) {
                uint8_t* d = a.Z + step * a.z_stride +
                             ((static_cast<int64_t>(r0 + e * 32 + rr) * H + k) * D + h * kUmmaN + c0) * a.z_elem +
                             ch * 16;
                *reinterpret_cast<uint4*>(d) = y;
              }
            }
            __syncwarp();
          }
          if ((a.debug & 2) || !tma_rows) continue;
          fence_async_smem();  // generic-proxy staging writes -> visible to the bulk-copy engine
          __syncwarp();
          if (lane == 0) {
            for (int g = 0; g < ng; ++g)
              asm volatile(
                  "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                      zmap_addr),
                  "r"(h * kUmmaN + g0 + g * cols_per_slice), "r"(k), "r"(r0 + e * 32), "r"(static_cast<int>(step)),
                  "r"(smem_addr(sbs[g]))
                  : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        if (dbg_lane) dbg_ts(a, i, 8 + 2 * h, 0);
        tc_fence_before();
        bar_arrive(&t_empty[h]);  // every tcgen05.ld of this accumulator has completed (wait::ld)
        if (dbg_lane) dbg_ts(a, i, 9 + 2 * h, 0);
      }
      ++i;
    }
    // Z writes done before exit.  (Waiting only for the staging reads, .read, and letting the writes
    // drain after exit measured the same -- r2 second session, profiles/r2/s2f_linear_exit_wait_ab.jsonl.)
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  dbg_cta(a, 3);
}

size_t linear_smem_bytes(int D) {
  return 1024 + static_cast<size_t>(D / 64) * kWBox + kStages * kABytes + kEpiWarps * kEpiBufs * kStageBytes + 128;
}

bool linear_supported(int H, int F, int D, int num_sms) {
  return F >= 1 && F <= kKPad && F % 4 == 0 && (D == 256 || D == 512) && H >= 1 && H <= num_sms;
}

namespace {
// Z as a 4-D TMA tensor {column d, hop k, batch row j, step s} with byte strides
// {s_z, D s_z, H D s_z, z_stride}; box = 32 rows x 128 bytes of one hop, 128-byte
// swizzle (the epilogue's staging layout).  False when the driver entry point
// is unavailable or the encode is rejected (the kernel then uses 16-byte stores).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return encode;
}

bool encode_z_map(const LinearArgs& a, CUtensorMap* m) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (encode == nullptr) return false;
  const cuuint64_t z = static_cast<cuuint64_t>(a.z_elem);
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(a.D), static_cast<cuuint64_t>(a.H),
                              static_cast<cuuint64_t>(a.B), static_cast<cuuint64_t>(a.nsteps)};
  cuuint64_t strides[3] = {a.D * z, a.H * a.D * z,
                           static_cast<cuuint64_t>(a.nsteps > 1 ? a.z_stride : a.B * a.H * a.D * z)};
  if (a.debug & 256) {  // experiment only: hop-major Z [step][hop][row][d] (breaks the output contract)
    strides[0] = a.B * a.D * z;
    strides[1] = a.D * z;
  }
  const cuuint32_t box[4] = {static_cast<cuuint32_t>(128 / a.z_elem), 1, 32, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode(m, a.z_elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.Z, dims,
                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// W as a 3-D TMA tensor {column d, row f, hop k} (bf16, byte strides {2 D, 2 F D}),
// box = 64 columns x 128 rows of one hop, 128-byte swizzle: each box lands as one
// MN-major SWIZZLE_128B block of the B operand; rows f >= F are filled with zeros.
bool encode_w_map(const LinearArgs& a, CUtensorMap* m) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (encode == nullptr) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(a.D), static_cast<cuuint64_t>(a.F), static_cast<cuuint64_t>(a.H)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(a.D) * 2, static_cast<cuuint64_t>(a.F) * a.D * 2};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(kKPad), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.W), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

cudaError_t launch_gather_linear(const LinearArgs& a_in, bool pdl, cudaStream_t st) {
  if (!linear_supported(a_in.H, a_in.F, a_in.D, a_in.num_sms)) return cudaErrorInvalidValue;
  const size_t smem = linear_smem_bytes(a_in.D);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_gather_linear, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(linear_smem_bytes(512)));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  LinearArgs a = a_in;
  alignas(64) CUtensorMap zmap{};
  a.z_tma = (a.debug & 128) ? 0 : (encode_z_map(a, &zmap) ? 1 : 0);
  alignas(64) CUtensorMap wmap{};
  if (!encode_w_map(a, &wmap)) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.num_sms / a.H) * a.H);
  cfg.blockDim = dim3(kLinThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute lattr[1];
  lattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  lattr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = lattr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_gather_linear, a, zmap, wmap);
}


// ==== K-chunked variant: any F (% 4 fp32, % 8 16-bit), spilled / sharded stores ================
// The F <= 128 kernel above keeps all of W_k resident; with F = 768 (MAG240M) or 1024 (IGB-large)
// W_k is 0.75-1 MB, so here the reduction dimension is walked in chunks of 64: per 128-row M-tile
// and chunk, a 16 KB A chunk (128 rows x 64 elements, K-major SWIZZLE_128B) is filled -- by TMA
// tile::gather4 straight from the store (16-bit records), by gather4 of fp32 halves converted in
// place (fp32 records), or by register-staged producers (spilled / sharded stores) -- and a loader
// warp brings the matching 64 x D slice of W_k by TMA (D / 64 boxes of 64 x 64, MN-major
// SWIZZLE_128B; rows >= F zero-filled).  2 W stages (W_k kept resident when it fits them), the same
// TMEM accumulators and TMA-store epilogue as above.  Otherwise W_k is re-read from L2 for every
// tile (it is the same for all of a CTA's tiles), F x D x 2 bytes per 128 rows.
//   A operand = the batch the loader would produce: fp32 records cast with cvt.rn to bf16 / f16,
//   16-bit records copied; W (and the MMA's input kind) in that same 16-bit type.
//   Rows resolve through the shard views (owner v mod W, HBM / pinned spill / peer HBM), so spilled
//   and sharded stores work; peer rows are read as store records (not the exchange copy).
namespace {
constexpr int kKcChunk = 64;                     // K elements per chunk (one 128-B swizzle row of bf16)
// Shared memory at D = 512 (224 KB): 2 W stages of a whole 64-row chunk (128 KB) + 4 slots of 16 KB
// (A stages; with fp32 records gathered by TMA, 2 slot pairs: fp32 halves converted in place) + the
// epilogue staging (32 KB).  Experiment layout (debug bit 2048): 3 half-chunk W stages (96 KB) +
// 6 slots.  CTA pairs (kPair): 4 W stages of half a chunk's columns (32 KB each).
constexpr int kKcASlots = 8;   // max 16 KB A / staging slots
constexpr int kKcWStages = 4;  // max W stages of one 32-row half chunk (D / 64 boxes of 32 x 64)
constexpr int kKcABytes = kTileM * 128;          // 16 KB: 128 rows x 64 bf16
constexpr int kKcWBox = (kKcChunk / 2) * 128;    // 4 KB: 32 K rows x 64 columns (one half chunk)
constexpr int kKcLoaderWarp = 9;
constexpr int kKcRelayWarp = 10;  // pair mode, fp32 TMA path: forwards converted chunks to the leader

// MN-major SW128 B descriptor; lbo = bytes between 64-column blocks (the K rows of a stage x 128 B)
__device__ __forceinline__ uint64_t kc_w_desc(const void* p, uint32_t lbo) {
  return static_cast<uint64_t>((smem_addr(p) >> 4) & 0x3FFFu) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t kc_idesc(int out_dtype) {
  const uint32_t fmt = out_dtype == 2 ? 0u : 1u;  // kind::f16 operand format: 0 = F16, 1 = BF16
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 16) | (static_cast<uint32_t>(kUmmaN >> 3) << 17) |
         (static_cast<uint32_t>(kTileM >> 4) << 24);
}
__device__ __forceinline__ void umma_i(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ uint32_t f16x2(uint32_t lo, uint32_t hi) {
  const __half2 h = __floats2half2_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<const uint32_t*>(&h);
}

// ---- CTA-pair (cta_group::2) helpers: the leader (cluster rank 0) issues the M = 256 MMAs over both
// CTAs' shared memory; the peer's producers and epilogue signal the leader's barriers remotely.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same object in the leader CTA (rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_addr(p)));
  return r;
}
__device__ __forceinline__ void bar_arrive_remote(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
// Accumulator-empty arrival on the leader's barrier: the TMEM reads it publishes are ordered by
// tcgen05.wait::ld + tcgen05.fence::before_thread_sync (and the leader's fence::after_thread_sync), not
// by memory semantics, so the default arrive (CUTLASS's remote ClusterBarrier arrive): .release.cluster
// compiles to MEMBAR.ALL.GPU, which also waited for the epilogue lane's outstanding Z bulk stores
// (r2 second session: 5.7 % of the pair kernel's samples at that MEMBAR)
__device__ __forceinline__ void bar_arrive_remote_tmem(uint32_t caddr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
// relaxed: the arrival only posts the byte count the TMA's complete_tx will retire (the data is
// ordered by the async proxy), so no release fence -- with .release every A / W stage posted a
// MEMBAR on the issuing lane's path (r2 second session, profiles/r2/kc_issue/s2h_*)
__device__ __forceinline__ void bar_expect_tx_remote(uint32_t caddr, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(caddr), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void bar_wait_cluster(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, "
        "p;\n}"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma_i2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the barrier at this offset in both CTAs of the pair once the leader's MMAs so far complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_addr(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
// Slot and phase of a counter walking a ring of n barrier-guarded slots -- no 64-bit division on the
// single-lane issue paths (the MMA and TMA issuers are instruction-bound, not just barrier-bound).
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  int n;
  __device__ explicit Ring(int n_) : n(n_) {}
  __device__ __forceinline__ void next() {
    if (++s == n) {
      s = 0;
      ph ^= 1u;
    }
  }
};

// MMA issue / commit for the K-chunked kernel.  kElect: executed by the whole (converged) warp, one
// lane elected inside the instruction sequence -- the operands are warp-uniform, so they live in
// uniform registers and no per-instruction waterfall loop is needed; otherwise by one lane.
#define PPL_KC_MMA(CG, ELECT)                                                                         \
  asm volatile("{\n .reg .pred e, p;\n" ELECT "setp.ne.b32 p, %4, 0;\n"                            \
               " @e tcgen05.mma.cta_group::" CG ".kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d), \
               "l"(a), "l"(b), "r"(idesc), "r"(accumulate)                                           \
               : "memory")
template <bool kPair, bool kElect>
__device__ __forceinline__ void kc_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  if constexpr (kPair && kElect)
    PPL_KC_MMA("2", " elect.sync _|e, 0xffffffff;\n");
  else if constexpr (kPair)
    PPL_KC_MMA("2", " setp.eq.u32 e, 0, 0;\n");
  else if constexpr (kElect)
    PPL_KC_MMA("1", " elect.sync _|e, 0xffffffff;\n");
  else
    PPL_KC_MMA("1", " setp.eq.u32 e, 0, 0;\n");
}
#undef PPL_KC_MMA
// The four K = 16 steps of one 64-element chunk into one accumulator in one asm block, one lane
// elected: A advances 32 B (+2 in the descriptor's 16-byte address field) and B 16 K rows (2 KB,
// +128) per step; only the first step may start a fresh accumulation.
#define PPL_KC_MMA4(CG)                                                                                 \
  asm volatile(                                                                                         \
      "{\n .reg .pred e, p;\n .reg .b64 a1, a2, a3, b1, b2, b3;\n"                                       \
      " elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"                                          \
      " add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"                                 \
      " add.s64 b1, %2, 128;\n add.s64 b2, %2, 256;\n add.s64 b3, %2, 384;\n"                           \
      " @e tcgen05.mma.cta_group::" CG ".kind::f16 [%0], %1, %2, %3, p;\n"                               \
      " @e tcgen05.mma.cta_group::" CG ".kind::f16 [%0], a1, b1, %3, 1;\n"                               \
      " @e tcgen05.mma.cta_group::" CG ".kind::f16 [%0], a2, b2, %3, 1;\n"                               \
      " @e tcgen05.mma.cta_group::" CG ".kind::f16 [%0], a3, b3, %3, 1;\n}" ::"r"(tmem_d),                \
      "l"(a0), "l"(b0), "r"(idesc), "r"(accumulate)                                                     \
      : "memory")
template <bool kPair>
__device__ __forceinline__ void kc_mma4(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint32_t idesc,
                                        uint32_t accumulate) {
  if constexpr (kPair)
    PPL_KC_MMA4("2");
  else
    PPL_KC_MMA4("1");
}
#undef PPL_KC_MMA4

template <bool kPair, bool kElect>
__device__ __forceinline__ void kc_commit(uint64_t* bar) {
  if constexpr (kPair && kElect)
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e tcgen05.commit.cta_group::2.mbarrier::arrive::one"
        ".shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(smem_addr(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  else if constexpr (kPair)
    umma_commit_pair(bar);
  else if constexpr (kElect)
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e tcgen05.commit.cta_group::1.mbarrier::arrive::one"
        ".shared::cluster.b64 [%0];\n}" ::"r"(smem_addr(bar))
        : "memory");
  else
    umma_commit(bar);
}

// TMA loads whose completion goes to the leader's barrier in pair mode (.cta_group::2: the barrier
// may sit in either CTA of the pair; the data lands in the issuing CTA's shared memory)
template <bool kPair>
__device__ __forceinline__ void tma_gather4(uint32_t dst, uint64_t map, int col, int r0, int r1, int r2, int r3,
                                            uint32_t bar) {
  if constexpr (kPair)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
}
template <bool kPair>
__device__ __forceinline__ void tma_load3(uint32_t dst, uint64_t map, int c0, int c1, int c2, uint32_t bar) {
  if constexpr (kPair)
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
}  // namespace

// kPair: CTA pairs (clusters of 2, cta_group::2).  A pair takes 256-row tiles, each CTA gathering its
// own 128 rows into its A stages and loading half of each accumulator's W columns (128 of 256); the
// leader issues M = 256 x N = 256 MMAs that read both CTAs' shared memory, and each CTA's TMEM holds
// its 128 rows of the accumulators.  Half the W bytes per row and per CTA stage, so twice the stages.
template <bool kPair>
__global__ void __launch_bounds__(kLinThreads, 1)
    k_gather_linear_kc(const LinearArgs a, const __grid_constant__ CUtensorMap zmap,
                       const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap) {
  extern __shared__ uint8_t smem_raw[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int D = a.D;
  // Default: whole-chunk W stages (2 x 64 KB at D = 512) and 4 slots (fp32 gathers: 2 A stages + 2
  // staging halves).  Experiment bit 2048: 3 half-chunk W stages + 6 slots (measured slower in
  // interleaved A/B runs: IGB-large rows 26 vs 20 ms, MAG240M rows 24 vs 16 ms, r2x).
  const bool six = !kPair && (a.debug & 2048) != 0;
  constexpr int npeer = kPair ? 2 : 1;
  constexpr int bpa = kUmmaN / 64 / npeer;                // 64-column W blocks per accumulator in this CTA
  const int wsplit = six ? 2 : 1;                         // W stages per chunk
  const int wrows = kKcChunk / wsplit;                    // K rows per W stage
  const int wbrows = six ? 32 : 64;                       // K rows per W TMA box (must match encode_w_map_kc)
  const int w_stage_bytes = (D / npeer / 64) * wrows * 128;
  // Pairs: a W stage is half a chunk's columns (32 KB at D = 512), so 2 W stages leave room for 8 A
  // slots (4 fp32 chunk pairs in flight); experiment bit 65536: the first pair layout, 4 W stages + 4
  // slots (A ring 2 deep on the fp32 path: 1.3x slower than single CTAs at IGB-large rows)
  // experiment bit 131072: 3 W stages + 6 slots
  const int pair_ws = !kPair ? 2 : (a.debug & 65536) ? 4 : (a.debug & 131072) ? 3 : 2;
  const int nws = six ? 3 : pair_ws;                      // W stages
  const int nas = six ? 6 : (kPair ? 12 - 2 * pair_ws : 4);  // A / staging slots (pairs: 192 KB in all)
  uint8_t* w_s = smem;                                    // [nws][D / 64 blocks][wrows K rows][128 B]
  uint8_t* a_s = w_s + nws * w_stage_bytes;               // [nas][128 rows][128 B]
  uint8_t* z_s = w_s + 4 * ((512 / 64) * kKcWBox) + 4 * kKcABytes;  // epilogue staging (fixed offset)
  uint64_t* bars = reinterpret_cast<uint64_t*>(z_s + kEpiWarps * kEpiBufs * kStageBytes);
  uint64_t* a_full = bars;                                // [kKcASlots]
  uint64_t* a_empty = a_full + kKcASlots;                 // [kKcASlots]
  uint64_t* w_full = a_empty + kKcASlots;                 // [kKcWStages]
  uint64_t* w_empty = w_full + kKcWStages;                // [kKcWStages]
  uint64_t* t_full = w_empty + kKcWStages;                // [2]
  uint64_t* t_empty = t_full + 2;                         // [2]
  uint64_t* stg_full = t_empty + 2;                       // [kKcASlots] fp32 staging halves (tma_f32)
  uint64_t* stg_empty = stg_full + kKcASlots;             // [kKcASlots]
  uint64_t* fin = stg_empty + kKcASlots;                  // pair mode: the leader's MMAs all complete
  uint64_t* a_conv = fin + 1;                             // [kKcASlots] pair mode, fp32 TMA path: converted
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_conv + kKcASlots);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.H, F = a.F;
  const uint32_t cr = kPair ? cluster_rank() : 0u;       // rank in the pair (0 = leader)
  const int pid = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  int k = pid % H;  // hop of the current unit: fixed per CTA, or per (tile, hop) unit with a.units
  const int q = pid / H, Q = (kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x)) / H;
  constexpr int kTM = kTileM * npeer;                     // rows per tile (the pair's)
  // barrier signals that go to the leader in pair mode
  auto arrive_leader = [&](uint64_t* b) {
    if constexpr (kPair)
      bar_arrive_remote(leader_addr(b));
    else
      bar_arrive(b);
  };
  auto expect_leader = [&](uint64_t* b, uint32_t tx) {
    if constexpr (kPair)
      bar_expect_tx_remote(leader_addr(b), tx);
    else
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(tx) : "memory");
  };
  // A stage written by this thread's generic stores (converters, register producers), after its
  // fence.proxy.async: single CTAs arrive per thread (a local arrival is cheap); pairs arrive once
  // per warp on the leader's barrier, since every remote release arrival costs a MEMBAR
  auto arrive_a = [&](uint64_t* b) {
    if constexpr (kPair) {
      __syncwarp();
      if ((threadIdx.x & 31) == 0) bar_arrive_remote(leader_addr(b));
    } else {
      bar_arrive(b);
    }
  };
  auto tma_bar = [&](uint64_t* b) -> uint32_t { return kPair ? leader_addr(b) : smem_addr(b); };
  auto wait_leader = [&](uint64_t* b, uint32_t parity) {  // a barrier the peer CTA also signals
    if constexpr (kPair)
      bar_wait_cluster(b, parity);
    else
      bar_wait(b, parity);
  };
  const int nh = D / kUmmaN;
  const int nch = (F + kKcChunk - 1) / kKcChunk;
  // every W chunk of hop k fits the W stages (F <= 128): load W_k once and keep it
  const bool wres = nch * (kKcChunk / (six ? 32 : 64)) <= nws && !six;
  const int s_in = a.in_dtype == 0 ? 4 : 2;
  // A stages: one per slot (16-bit TMA gathers, register producers); fp32 TMA gathers use the slots in
  // pairs: chunk u's two 32-element fp32 halves (128 rows x 128 B, SW128) land in slots 2p and 2p + 1
  // (p = u mod nas / 2) and are converted in place -- the bf16 / f16 A chunk overwrites half 0 in slot
  // 2p, which the MMA then reads; slot 2p + 1 is free again as soon as it is converted
  const int na = a.tma_f32 ? nas / 2 : nas;
  const int a_slot_step = a.tma_f32 ? 2 : 1;  // A chunk of ring position s at slot s * a_slot_step

  if (threadIdx.x == 0) {
    for (int s = 0; s < kKcASlots; ++s) {
      // arrivals: TMA gathers (16-bit) one arrive + the bytes; fp32 converters 128; register producers 256
      // pair mode: converted chunks reach the leader through one relay arrival per CTA, register
      // producers arrive once per warp
      bar_init(&a_full[s], (a.tma_a ? 1 : a.tma_f32 ? (kPair ? 1 : 128) : kProducerThreads / (kPair ? 32 : 1)) * npeer);
      bar_init(&a_empty[s], 1);
      bar_init(&a_conv[s], 128);
    }
    for (int s = 0; s < kKcASlots; ++s) {
      bar_init(&stg_full[s], 1);
      bar_init(&stg_empty[s], 128);
    }
    for (int s = 0; s < kKcWStages; ++s) {  // (only the first nws are used)
      bar_init(&w_full[s], npeer);
      bar_init(&w_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      bar_init(&t_full[h], 1);
      uint32_t cnt = 0;
      for (int g = 0; g < kEpiGroups; ++g) {
        const int lo = g * D / kEpiGroups, hi = (g + 1) * D / kEpiGroups;
        if (lo < (h + 1) * kUmmaN && hi > h * kUmmaN) cnt += 128;
      }
      // pair mode: one (remote, release) arrival per epilogue warp instead of per thread
      bar_init(&t_empty[h], cnt > 0 ? (kPair ? cnt / 32 : cnt) * npeer : 1);
    }
    bar_init(fin, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (kPair)
    cluster_sync_all();  // the peer signals the leader's barriers: both initialised first
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t tiles_per_step = (a.B + kTM - 1) / kTM;
  const int64_t total = tiles_per_step * a.nsteps;
  auto tile_rows = [&](int64_t t, int64_t& step, int& r0, int64_t& pos) -> int {
    step = t / tiles_per_step;
    r0 = static_cast<int>(t - step * tiles_per_step) * kTM;
    pos = a.first_pos + step * a.step_stride;
    const int64_t nrows = min(static_cast<int64_t>(a.B), a.N - pos);
    return static_cast<int>(min(static_cast<int64_t>(kTM), nrows - r0));
  };
  // this CTA's rows of tile t (its 128-row half in pair mode; may be empty for the peer)
  auto tile_rows_cta = [&](int64_t t, int64_t& step, int& r0, int64_t& pos) -> int {
    const int rows = tile_rows(t, step, r0, pos);
    if constexpr (!kPair) return rows;
    r0 += static_cast<int>(cr) * kTileM;
    return max(0, min(kTileM, rows - static_cast<int>(cr) * kTileM));
  };
  auto next_tile = [&](int64_t t) -> int64_t {
    for (; t < total; t += Q) {
      int64_t st_, ps_;
      int r_;
      if (tile_rows(t, st_, r_, ps_) > 0) return t;
    }
    return total;
  };
  // Work units.  Default: CTA (pair) pid is pinned to hop pid % H and walks tiles q, q + Q, ... (W_k
  // may stay resident).  a.units (W streamed per tile anyway, TMA A paths): units u = tile * H + hop
  // dealt round-robin over every CTA (pair) of the grid, so the grid is not rounded down to a multiple
  // of H and the last wave is shared by all hops.  Every role walks the same unit sequence.
  const int64_t ustride = a.units ? (kPair ? static_cast<int64_t>(gridDim.x >> 1) : static_cast<int64_t>(gridDim.x)) : Q;
  const int64_t nunits = a.units ? total * H : total;
  const int64_t ufirst = a.units ? pid : q;
  auto unit_tile = [&](int64_t u) -> int64_t { return a.units ? u / H : u; };
  auto next_unit = [&](int64_t u) -> int64_t {
    for (; u < nunits; u += ustride) {
      int64_t st_, ps_;
      int r_;
      if (tile_rows(unit_tile(u), st_, r_, ps_) > 0) return u;
    }
    return nunits;
  };
  auto set_unit = [&](int64_t u) -> int64_t {  // this unit's tile; sets k
    if (a.units) k = static_cast<int>(u % H);
    return unit_tile(u);
  };

  const int gw = a.tma_a >= 2 ? 8 : 4;  // warps issuing gather4 (tma_a = 2: all eight producer warps)
  if ((a.tma_a || a.tma_f32) && warp < gw) {
    // ---------------- 16-bit records, F % 64 == 0, every row in HBM: the A chunks are the records'
    // bytes as they are, so TMA fetches them straight into the SW128 A tile: per chunk, 32
    // cp.async.bulk.tensor tile::gather4 (4 rows x 128 B each) on a 2-D map of the store
    // [rows][record elements] -- no register staging, all of a chunk's 16 KB in flight at once.
    // Warp w (0..3) resolves rows 32w..32w+31 of the tile (order -> node set) and its lane 0 issues
    // their 8 gather4s; warp 0 also posts the stage's expected bytes.
    __shared__ int32_t s_rows[kTileM];
    const uint64_t amap_addr = reinterpret_cast<uint64_t>(&amap);
    Ring ra(na);
    // L2 prefetch (a.l2_prefetch, PPLOAD_LINEAR_PREFETCH=1; off by default): after issuing unit u, every
    // lane pulls its row of the next unit into L2 (one cp.async.bulk.prefetch of the hop's F * s_in
    // bytes). Measured: products 1-2 % faster, MAG240M / IGB-large rows 3 % / 27 % slower (s3k_ab.jsonl)
    const int jrow = warp * (kTileM / gw) + lane;
    const bool jown = lane < kTileM / gw;
    for (int64_t u = next_unit(ufirst); u < nunits;) {
      const int64_t un = next_unit(u + ustride);
      const int64_t t = set_unit(u);
      int64_t step, pos;
      int r0;
      const int rows = tile_rows_cta(t, step, r0, pos);
      __syncwarp();
      if (jown) {
        int64_t v = 0;  // rows past the batch gather record 0; the epilogue never stores them
        if (jrow < rows) {
          v = a.order[pos + r0 + jrow];
          if (a.node_set != nullptr) v = a.node_set[v];
        }
        s_rows[jrow] = static_cast<int32_t>(a.hop_rows ? v * H + k : v);
      }
      __syncwarp();
      for (int ch = 0; ch < nch; ++ch) {
        if (a.tma_f32 == 3) {  // fp32 records, 64 < F <= 128, pairs: one 512-byte box per (node, hop) row
          if (lane == 0) {     // covers both chunks: 32 gather4 into slots 2p .. 2p + 3 (p even) at chunk 0
            const int p = ra.s;
            const uint32_t ph = ra.ph;
            ra.next();
            if ((ch & 1) == 0) {  // chunks ch, ch + 1 (nch even)
              bar_wait(&a_empty[p], ph ^ 1u);
              bar_wait(&stg_empty[2 * p + 1], ph ^ 1u);
              bar_wait(&a_empty[p + 1], ph ^ 1u);
              bar_wait(&stg_empty[2 * p + 3], ph ^ 1u);
              if (warp == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&stg_full[2 * p])),
                             "r"(4 * kKcABytes)
                             : "memory");
              uint8_t* dst = a_s + 2 * p * kKcABytes;
              for (int g = warp * (32 / gw); g < (warp + 1) * (32 / gw); ++g)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_addr(dst + g * 2048)),
                    "l"(amap_addr), "r"((a.hop_rows ? 0 : k * F) + ch * kKcChunk), "r"(s_rows[4 * g]),
                    "r"(s_rows[4 * g + 1]), "r"(s_rows[4 * g + 2]), "r"(s_rows[4 * g + 3]), "r"(smem_addr(&stg_full[2 * p]))
                    : "memory");
            }
          }
          continue;
        }
        if (a.tma_f32 == 2) {  // fp32 records, wide boxes: the whole 64-element chunk (4 rows x 256 B per
          if (lane == 0) {     // gather4, unswizzled) into slots 2p, 2p + 1 as 128 rows of 256 B
            const int p = ra.s;
            bar_wait(&a_empty[p], ra.ph ^ 1u);
            bar_wait(&stg_empty[2 * p + 1], ra.ph ^ 1u);
            ra.next();
            if (warp == 0)
              asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&stg_full[2 * p])),
                           "r"(2 * kKcABytes)
                           : "memory");
            const int col = (a.hop_rows ? 0 : k * F) + ch * kKcChunk;
            uint8_t* dst = a_s + 2 * p * kKcABytes;
            for (int g = warp * (32 / gw); g < (warp + 1) * (32 / gw); ++g)
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_addr(dst + g * 1024)),
                  "l"(amap_addr), "r"(col), "r"(s_rows[4 * g]), "r"(s_rows[4 * g + 1]), "r"(s_rows[4 * g + 2]),
                  "r"(s_rows[4 * g + 3]), "r"(smem_addr(&stg_full[2 * p]))
                  : "memory");
          }
          continue;
        }
        if (a.tma_f32) {  // fp32 records: two 32-element halves into slots 2p, 2p + 1, converted by warps 4-7
          if (lane == 0) {
            const int p = ra.s;
            bar_wait(&a_empty[p], ra.ph ^ 1u);               // slot 2p: the MMA is done with A(u - na)
            bar_wait(&stg_empty[2 * p + 1], ra.ph ^ 1u);     // slot 2p + 1: converted
            ra.next();
            for (int hh = 0; hh < 2; ++hh) {
              const int sl = 2 * p + hh;
              if (warp == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&stg_full[sl])),
                             "r"(kKcABytes)
                             : "memory");
              const int col = (a.hop_rows ? 0 : k * F) + ch * kKcChunk + hh * 32;
              uint8_t* dst = a_s + sl * kKcABytes;
              for (int g = warp * (32 / gw); g < (warp + 1) * (32 / gw); ++g)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_addr(dst + g * 512)),
                    "l"(amap_addr), "r"(col), "r"(s_rows[4 * g]), "r"(s_rows[4 * g + 1]), "r"(s_rows[4 * g + 2]),
                    "r"(s_rows[4 * g + 3]), "r"(smem_addr(&stg_full[sl]))
                    : "memory");
            }
          }
          continue;
        }
        if (lane == 0) {
          const int s = ra.s;
          bar_wait(&a_empty[s], ra.ph ^ 1u);
          ra.next();
          if (warp == 0) expect_leader(&a_full[s], kKcABytes);
          const int col = k * F + ch * kKcChunk;
          uint8_t* dst = a_s + s * kKcABytes;
          const uint32_t fb = tma_bar(&a_full[s]);
          for (int g = warp * (32 / gw); g < (warp + 1) * (32 / gw); ++g)
            tma_gather4<kPair>(smem_addr(dst + g * 512), amap_addr, col, s_rows[4 * g], s_rows[4 * g + 1],
                               s_rows[4 * g + 2], s_rows[4 * g + 3], fb);
        }
      }
      if (a.l2_prefetch && jown && un < nunits) {
        int64_t stn, psn;
        int r0n;
        const int rowsn = tile_rows_cta(unit_tile(un), stn, r0n, psn);
        if (jrow < rowsn) {
          int64_t v = a.order[psn + r0n + jrow];
          if (a.node_set != nullptr) v = a.node_set[v];
          const int kn = a.units ? static_cast<int>(un % H) : k;
          const uint8_t* pr = a.shards[0].hbm + v * a.rec_stride + static_cast<int64_t>(kn) * F * s_in;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pr), "r"(F * s_in) : "memory");
        }
      }
      u = un;
    }
    __syncwarp();
  } else if (a.tma_f32 && warp < kProducerWarps) {
    // ---------------- fp32 records gathered by TMA: warps 4-7 convert chunk u's staged halves (SW128
    // fp32, 32 per row) into the SW128 bf16 / f16 A chunk in slot 2p, in place: thread (row r, 16-B A
    // chunk j of the half) reads staged chunks 2j, 2j+1 (8 fp32), converts with cvt.rn, writes one
    // 16-byte A chunk.  The four threads of a row are consecutive lanes of one warp, so a __syncwarp
    // between the reads and the writes of half 0 orders every read of a row before the writes into it.
    const int tid = threadIdx.x - 128;
    const uint32_t a_base = smem_addr(a_s);
    Ring ra(na);
    for (int64_t u = next_unit(ufirst); u < nunits; u = next_unit(u + ustride)) {
      for (int ch = 0; ch < nch; ++ch, ra.next()) {
        const int p = ra.s;
        const uint32_t at = a_base + 2 * p * kKcABytes;
        if (a.tma_f32 == 3) {
          // one tile's rows staged at chunk 0 (p even): staged row r = 512 B (128 fp32, zero past F) at
          // 2p * 16 KB + 512 r, i.e. rows 32i..32i+31 in slot 2p + i. A chunk 0 goes to slot 2p, chunk 1
          // to slot 2p + 2 (where the MMA reads ring positions p and p + 1), so only staged rows 0-31 and
          // 64-95 are overwritten: those are read into registers first, the four converter warps meet at
          // a named barrier, then they are written; rows 32-63 and 96-127 (slots 2p + 1, 2p + 3, never
          // written) are converted straight from shared memory
          if (ch & 1) continue;
          bar_wait(&stg_full[2 * p], ra.ph);
          const uint32_t a1 = at + 2 * kKcABytes;
          auto cvt_store = [&](int r, int j8, uint4 x0, uint4 x1) {
            const int e0 = ch * kKcChunk + 8 * j8;
            if (e0 >= F) x0 = make_uint4(0, 0, 0, 0);
            if (e0 + 4 >= F) x1 = make_uint4(0, 0, 0, 0);
            const uint4 y = a.out_dtype == 2
                                ? make_uint4(f16x2(x0.x, x0.y), f16x2(x0.z, x0.w), f16x2(x1.x, x1.y), f16x2(x1.z, x1.w))
                                : make_uint4(bf16x2(x0.x, x0.y), bf16x2(x0.z, x0.w), bf16x2(x1.x, x1.y),
                                             bf16x2(x1.z, x1.w));
            sts16(((j8 >> 3) ? a1 : at) + sw128(r, j8 & 7), y);
          };
          uint4 x[8][2];
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int item = tid + 128 * it;  // (row index 0..63, 32-byte group j8 of 16)
            const int ri = item >> 4, j8 = item & 15;
            const int r = ri < 32 ? ri : ri + 32;
            const uint32_t src = at + r * 512 + j8 * 32;
            x[it][0] = lds16(src);
            x[it][1] = lds16(src + 16);
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int item = tid + 128 * it;
            const int ri = item >> 4, j8 = item & 15;
            cvt_store(ri < 32 ? ri : ri + 32, j8, x[it][0], x[it][1]);
          }
#pragma unroll 2
          for (int it = 0; it < 8; ++it) {
            const int item = tid + 128 * it;
            const int ri = item >> 4, j8 = item & 15;
            const int r = ri < 32 ? ri + 32 : ri + 64;
            const uint32_t src = at + r * 512 + j8 * 32;
            cvt_store(r, j8, lds16(src), lds16(src + 16));
          }
          bar_arrive(&stg_empty[2 * p + 1]);
          bar_arrive(&stg_empty[2 * p + 3]);
          fence_async_smem();
          if constexpr (kPair) {
            bar_arrive(&a_conv[p]);
            bar_arrive(&a_conv[p + 1]);
          } else {
            bar_arrive(&a_full[p]);
            bar_arrive(&a_full[p + 1]);
          }
          continue;
        }
        if (a.tma_f32 == 2) {
          // wide boxes: staging row r = 256 B (64 fp32) at 2p * 16 KB + 256 r; the A chunk (rows of 128 B,
          // SW128) overwrites staging rows 0-63, which other warps' threads read -- so every thread reads
          // all of its items first, the four converter warps meet at a named barrier, then write
          bar_wait(&stg_full[2 * p], ra.ph);
          uint4 x[4][2][2];
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int item = tid + 128 * it;
            const int r = item >> 2, j = item & 3;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const uint32_t src = at + r * 256 + hh * 128 + j * 32;
              x[it][hh][0] = lds16(src);
              x[it][hh][1] = lds16(src + 16);
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int item = tid + 128 * it;
            const int r = item >> 2, j = item & 3;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              uint4 x0 = x[it][hh][0], x1 = x[it][hh][1];
              const int e0 = ch * kKcChunk + hh * 32 + 8 * j;
              if (e0 >= F) x0 = make_uint4(0, 0, 0, 0);
              if (e0 + 4 >= F) x1 = make_uint4(0, 0, 0, 0);
              const uint4 y = a.out_dtype == 2
                                  ? make_uint4(f16x2(x0.x, x0.y), f16x2(x0.z, x0.w), f16x2(x1.x, x1.y), f16x2(x1.z, x1.w))
                                  : make_uint4(bf16x2(x0.x, x0.y), bf16x2(x0.z, x0.w), bf16x2(x1.x, x1.y),
                                               bf16x2(x1.z, x1.w));
              sts16(at + sw128(r, hh * 4 + j), y);
            }
          }
          bar_arrive(&stg_empty[2 * p + 1]);  // slot 2p + 1 read out (before the barrier); 2p holds A(u)
          fence_async_smem();
          if constexpr (kPair)
            bar_arrive(&a_conv[p]);
          else
            bar_arrive(&a_full[p]);
          continue;
        }
        for (int hh = 0; hh < 2; ++hh) {
          const int sl = 2 * p + hh;
          bar_wait(&stg_full[sl], ra.ph);
          const uint32_t sh = a_base + sl * kKcABytes;
          uint4 x[4][2];
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int item = tid + 128 * it;
            const int r = item >> 2, j = item & 3;
            x[it][0] = lds16(sh + r * 128 + (((2 * j) ^ (r & 7)) << 4));
            x[it][1] = lds16(sh + r * 128 + (((2 * j + 1) ^ (r & 7)) << 4));
          }
          __syncwarp();
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int item = tid + 128 * it;
            const int r = item >> 2, j = item & 3;
            uint4 x0 = x[it][0], x1 = x[it][1];
            // F % 64 != 0: elements past F belong to the next hop (or are the map's zero fill); the
            // K padding must be zero (F % 4 == 0, so a 16-byte group is all in or all out)
            const int e0 = ch * kKcChunk + hh * 32 + 8 * j;
            if (e0 >= F) x0 = make_uint4(0, 0, 0, 0);
            if (e0 + 4 >= F) x1 = make_uint4(0, 0, 0, 0);
            const uint4 y = a.out_dtype == 2
                                ? make_uint4(f16x2(x0.x, x0.y), f16x2(x0.z, x0.w), f16x2(x1.x, x1.y), f16x2(x1.z, x1.w))
                                : make_uint4(bf16x2(x0.x, x0.y), bf16x2(x0.z, x0.w), bf16x2(x1.x, x1.y),
                                             bf16x2(x1.z, x1.w));
            sts16(at + sw128(r, hh * 4 + j), y);
          }
          if (hh == 1) bar_arrive(&stg_empty[sl]);  // slot 2p + 1 read out; slot 2p now holds A(u)
        }
        fence_async_smem();
        if constexpr (kPair)
          bar_arrive(&a_conv[p]);  // the relay warp forwards it to the leader
        else
          bar_arrive(&a_full[p]);
      }
    }
  } else if (a.tma_a && warp < kProducerWarps) {  // warps 4-7
    // (idle in the TMA-gather mode)
  } else if (warp < kProducerWarps) {
    // ---------------- producers: warp w owns rows 16w..16w+15 of every tile.  Lanes 0-15 resolve
    // the 16 row pointers once per tile; per chunk, fp32 records: half-warp per row (lane c loads
    // elements 4c..4c+3 of the chunk, 16 B), 8 iterations; 16-bit records: quarter-warp per row
    // (lane c8 loads elements 8 c8..8 c8+7), 4 iterations.  The next chunk's loads are issued before
    // the current chunk is converted and stored.
    const int rbase = warp * 16;
    constexpr uint32_t kNoRow = 0xffffffffu;
    auto fetch_index = [&](int64_t t) -> uint32_t {
      if (t >= total) return kNoRow;
      int64_t step, pos;
      int r0;
      const int rows = tile_rows_cta(t, step, r0, pos);
      uint32_t v = kNoRow;
      if (lane < 16 && rbase + lane < rows)
        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(a.order + pos + r0 + rbase + lane));
      return v;
    };
    auto resolve = [&](uint32_t idx) -> const uint8_t* {  // this lane's row record (hop k), or null
      if (idx == kNoRow) return nullptr;
      uint64_t v = idx;
      if (a.node_set != nullptr) v = static_cast<uint64_t>(a.node_set[v]);
      const uint64_t W = static_cast<uint64_t>(a.world);
      const ShardView sh = a.shards[W > 1 ? v % W : 0];
      const int64_t l = static_cast<int64_t>(W > 1 ? v / W : v);
      const uint8_t* rec = l < sh.n_hbm ? sh.hbm + l * a.rec_stride : sh.spill + (l - sh.n_hbm) * a.rec_stride;
      return rec + static_cast<int64_t>(k) * F * s_in;
    };
    const bool f32 = s_in == 4;
    const int hw = lane >> 4, c16 = lane & 15;  // fp32 records
    const int qw = lane >> 3, c8 = lane & 7;    // 16-bit records
    auto load_chunk = [&](const uint8_t* my_src, int ch, uint4 (&x)[8]) {
      if (f32) {
        const int e = ch * kKcChunk + 4 * c16;  // first element of this lane's 16 B
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const uint8_t* src =
              reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_src), 2 * it + hw));
          x[it] = (src != nullptr && e < F && !(a.debug & 1)) ? ldg16(src + static_cast<int64_t>(e) * 4)
                                                             : make_uint4(0, 0, 0, 0);
        }
      } else {
        const int e = ch * kKcChunk + 8 * c8;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const uint8_t* src =
              reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_src), 4 * it + qw));
          x[it] = (src != nullptr && e < F && !(a.debug & 1)) ? ldg16(src + static_cast<int64_t>(e) * 2)
                                                             : make_uint4(0, 0, 0, 0);
        }
      }
    };
    Ring ra(na);
    auto store_chunk = [&](const uint4 (&x)[8]) {
      const int s = ra.s;
      bar_wait(&a_empty[s], ra.ph ^ 1u);
      ra.next();
      uint8_t* at = a_s + s * kKcABytes;
      if (f32) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int r = rbase + 2 * it + hw;
          const uint32_t off = sw128(r, c16 >> 1) + (c16 & 1) * 8;
          const uint4 v = x[it];
          *reinterpret_cast<uint2*>(at + off) =
              a.out_dtype == 2 ? make_uint2(f16x2(v.x, v.y), f16x2(v.z, v.w)) : make_uint2(bf16x2(v.x, v.y), bf16x2(v.z, v.w));
        }
      } else {
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int r = rbase + 4 * it + qw;
          *reinterpret_cast<uint4*>(at + sw128(r, c8)) = x[it];
        }
      }
      fence_async_smem();
      arrive_a(&a_full[s]);
    };
    // Register-staged loads keep only two chunks (64 KB per SM) in flight, less than HBM latency
    // needs, so each lane also pulls its row's chunk pf chunks ahead into L2 with one bulk prefetch
    // (no registers): the loads then hit L2.  Crossing into the next tile uses its rows.
    const int pf = a.l2_prefetch > 0 ? a.l2_prefetch : 0;
    const int chunk_bytes = kKcChunk * s_in;
    auto prefetch_chunk = [&](const uint8_t* my_src, int ch) {
      if (lane < 16 && my_src != nullptr && ch * kKcChunk < F) {
        const int bytes = min(chunk_bytes, (F - ch * kKcChunk) * s_in);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(my_src + static_cast<int64_t>(ch) * chunk_bytes),
                     "r"(bytes)
                     : "memory");
      }
    };
    // Register ring of R chunks: the loads of unit u + R - 1 are issued before unit u is converted
    // and stored, across tile boundaries.  R = 2 for fp32 records (8 x 16 B per lane and chunk),
    // R = 4 for 16-bit records (4 x 16 B): 64 registers of loads in flight either way.
    int64_t lt = next_tile(q);  // the load cursor: tile, chunk, this lane's row pointer
    int lch = 0;
    const uint8_t* lsrc = lt < total ? resolve(fetch_index(lt)) : nullptr;
    int64_t pt = lt < total ? next_tile(lt + Q) : total;  // the L2-prefetch cursor, pf units ahead
    int pch = 0;
    const uint8_t* psrc = pt < total ? resolve(fetch_index(pt)) : nullptr;
    auto load_next = [&](uint4 (&buf)[8]) -> bool {
      if (lt >= total) return false;
      load_chunk(lsrc, lch, buf);
      if (++lch == nch) {
        lch = 0;
        lt = next_tile(lt + Q);
        lsrc = lt < total ? resolve(fetch_index(lt)) : nullptr;
      }
      return true;
    };
    auto run = [&](auto ring) {
      constexpr int R = decltype(ring)::value;
      uint4 x[R][8];
      bool have[R];
#pragma unroll
      for (int j = 0; j < R - 1; ++j) have[j] = load_next(x[j]);
      have[R - 1] = false;
      for (;;) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          constexpr int dummy = 0;
          (void)dummy;
          const int jn = (j + R - 1) % R;
          have[jn] = load_next(x[jn]);
          if (pf > 0 && pt < total) {  // bulk L2 prefetch of the chunk pf units ahead of the loads
            prefetch_chunk(psrc, pch);
            if (++pch == nch) {
              pch = 0;
              pt = next_tile(pt + Q);
              psrc = pt < total ? resolve(fetch_index(pt)) : nullptr;
            }
          }
          if (!have[j]) return;
          store_chunk(x[j]);
        }
      }
    };
    if (f32)
      run(std::integral_constant<int, 2>{});
    else
      run(std::integral_constant<int, 4>{});
  } else if (warp == kKcLoaderWarp) {
    // ---------------- W loader: the same (tile, chunk) sequence; chunk ch of W_k into the next stage
    // of the ring (or, W_k resident, chunk ch into stage ch once)
    if (lane == 0) {
      const uint64_t wmap_addr = reinterpret_cast<uint64_t>(&wmap);
      const uint32_t nbox = static_cast<uint32_t>(D / npeer / 64);
      Ring rw(nws);  // W stage fills: (tile, chunk, part) in order
      for (int64_t u = next_unit(ufirst); u < nunits; u = next_unit(u + ustride)) {
        set_unit(u);
        for (int ch = 0; ch < nch; ++ch) {
          for (int wh = 0; wh < wsplit; ++wh, rw.next()) {
            const int s = rw.s;
            bar_wait(&w_empty[s], rw.ph ^ 1u);
            if (a.debug & 16) {  // experiment: no W traffic (the MMAs read stale shared memory)
              arrive_leader(&w_full[s]);
              continue;
            }
            expect_leader(&w_full[s], w_stage_bytes);
            const uint32_t fb = tma_bar(&w_full[s]);
            for (uint32_t b = 0; b < nbox; ++b) {
              // block b: columns of accumulator b / bpa; in pair mode this CTA's half of them
              const int col = static_cast<int>(b / bpa) * kUmmaN + static_cast<int>(cr) * (kUmmaN / 2) +
                              static_cast<int>(b % bpa) * 64;
              for (int sub = 0; sub < wrows / wbrows; ++sub)  // boxes stacked inside the 64-column block
                tma_load3<kPair>(smem_addr(w_s + s * w_stage_bytes + b * wrows * 128 + sub * wbrows * 128), wmap_addr,
                                 col, ch * kKcChunk + wh * wrows + sub * wbrows, k, fb);
            }
          }
        }
        if (wres) break;  // W_k resident in stages 0 .. nch - 1 for every tile
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer: per unit, 4 K-steps of 16 into each accumulator.  The whole warp runs
    // the loop and one elected lane issues (experiment bit 16384: lane 0 alone runs it); in pair mode
    // the leader issues for both CTAs.
    auto mma_role = [&](auto warpwide) {
      constexpr bool kW = decltype(warpwide)::value;
      const uint32_t idesc =
          kPair ? ((kc_idesc(a.out_dtype) & ~(0x1Fu << 24)) | (static_cast<uint32_t>(kTM >> 4) << 24)) : kc_idesc(a.out_dtype);
      Ring ra(na), rw(nws);
      int i = 0;
      for (int64_t u = next_unit(ufirst); u < nunits; u = next_unit(u + ustride), ++i) {
        for (int ch = 0; ch < nch; ++ch, ra.next()) {
          const int sa = ra.s;
          wait_leader(&a_full[sa], ra.ph);
          tc_fence_after();
          const uint8_t* at = a_s + sa * a_slot_step * kKcABytes;
          // the chunk's W in wsplit stages (whole, or K rows 0-31 and 32-63)
          for (int wh = 0; wh < wsplit; ++wh, rw.next()) {
            const int sw = wres ? ch : rw.s;
            wait_leader(&w_full[sw], wres ? 0u : rw.ph);
            tc_fence_after();
            const uint8_t* wt = w_s + sw * w_stage_bytes;
            for (int h = 0; h < nh; ++h) {
              if (ch == 0 && wh == 0) {  // accumulator h of the previous tile drained (the epilogue
                wait_leader(&t_empty[h], (i & 1) ^ 1);  // drains h = 0 first, so h = 0 MMAs overlap the h = 1 drain)
                tc_fence_after();
              }
              const int steps = (a.debug & 64) ? 0 : 4 / wsplit;
              // descriptors of the first K step; each further step of 16 advances A by 32 B and B by
              // 16 K rows (2 KB) -- added to the start-address field (bits 0-13, 16-B units)
              const uint64_t ad0 = sw128_desc(at) + 2 * (wh * (4 / wsplit));
              const uint64_t bd0 = kc_w_desc(wt + h * bpa * wrows * 128, wrows * 128);
              if (kW && steps == 4 && !(a.debug & 32768)) {  // a whole chunk: one issue block
                kc_mma4<kPair>(tmem + h * kUmmaN, ad0, bd0, idesc, (ch > 0 || wh > 0) ? 1u : 0u);
              } else {
                for (int jj = 0; jj < steps; ++jj)
                  kc_mma<kPair, kW>(tmem + h * kUmmaN, ad0 + 2 * jj, bd0 + 128 * jj, idesc,
                                    (ch > 0 || wh > 0 || jj > 0) ? 1u : 0u);
              }
              // last chunk: accumulator h is complete once its last MMAs are -- the epilogue can start
              // draining it while the other accumulator's last MMAs run
              if (ch == nch - 1 && wh == wsplit - 1) kc_commit<kPair, kW>(&t_full[h]);
            }
            if (!wres) kc_commit<kPair, kW>(&w_empty[sw]);
          }
          kc_commit<kPair, kW>(&a_empty[sa]);
        }
      }
      if constexpr (kPair) kc_commit<kPair, kW>(fin);  // both CTAs learn when every MMA (and signal) landed
    };
    if (cr == 0) {
      if (a.debug & 16384) {
        if (lane == 0) mma_role(std::false_type{});
      } else {
        mma_role(std::true_type{});
      }
    }
    __syncwarp();
  } else if (kPair && a.tma_f32 && warp == kKcRelayWarp) {
    // ---------------- pair mode, fp32 records: one lane forwards "chunk u converted" (the 128 converter
    // threads' local arrivals, acquired here; their generic stores were made visible to the async proxy
    // by fence.proxy.async before those arrivals) to the leader's a_full with a default-semantics remote
    // arrival, as CUTLASS's ClusterBarrier::arrive(cta_id) does for UMMA operands written by threads.
    // A .release.cluster arrival compiles to MEMBAR.ALL.GPU on every chunk's handoff chain: interleaved
    // A/B (r2 third session, profiles/r2/kc_products/s3y_ab.jsonl) IGB-large rows 15.0-15.3 vs 15.9-17.3 ms
    // per epoch (A side alone 10.4-11.3 vs 16.2-16.6), products 2.88-2.92 vs 2.94-3.05; experiment bit
    // 67108864 restores the release.cluster arrival
    if (lane == 0) {
      Ring ra(na);
      for (int64_t u = next_unit(ufirst); u < nunits; u = next_unit(u + ustride))
        for (int ch = 0; ch < nch; ++ch, ra.next()) {
          bar_wait(&a_conv[ra.s], ra.ph);
          if (a.debug & 67108864)
            bar_arrive_remote(leader_addr(&a_full[ra.s]));
          else
            bar_arrive_remote_tmem(leader_addr(&a_full[ra.s]));
        }
    }
    __syncwarp();
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue (as in k_gather_linear)
    const int e = warp & 3;
    const int grp = (warp - kEpiWarp0) >> 2;
    uint8_t* sbuf = z_s + (warp - kEpiWarp0) * kEpiBufs * kStageBytes;
    const int cols_per_slice = 128 / a.z_elem;
    const uint64_t zmap_addr = reinterpret_cast<uint64_t>(&zmap);
    int i = 0, slice = 0;
    for (int64_t u = next_unit(ufirst); u < nunits; u = next_unit(u + ustride), ++i) {
      const int64_t t = set_unit(u);
      int64_t step, pos;
      int r0;
      const int rows = tile_rows_cta(t, step, r0, pos);
      const bool tma_rows = a.z_tma && e * 32 + 32 <= rows;
      for (int h = 0; h < nh; ++h) {
        const int c_lo = max(grp * D / kEpiGroups, h * kUmmaN) - h * kUmmaN;
        const int c_hi = min((grp + 1) * D / kEpiGroups, (h + 1) * kUmmaN) - h * kUmmaN;
        if (c_lo >= c_hi) continue;
        bar_wait(&t_full[h], i & 1);
        tc_fence_after();
        if (a.debug & 2097152) {  // experiment: no accumulator drain at all (no TMEM loads, no Z)
          tc_fence_before();
          if constexpr (kPair) {
            __syncwarp();
            if (lane == 0) bar_arrive_remote_tmem(leader_addr(&t_empty[h]));
          } else {
            arrive_leader(&t_empty[h]);
          }
          continue;
        }
        const uint32_t trow = tmem + (static_cast<uint32_t>(e * 32) << 16) + h * kUmmaN;
        uint32_t v[64];
        auto ld_slice = [&](int c0) {
          PPL_TMEM_LD32(trow + c0, v);
          if (a.z_elem == 2) PPL_TMEM_LD32(trow + c0 + 32, (v + 32));
        };
        ld_slice(c_lo);
#pragma unroll 1
        for (int c0 = c_lo; c0 < c_hi; c0 += cols_per_slice) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kEpiBufs - 1) : "memory");
          __syncwarp();
          uint8_t* sb = sbuf + (slice % kEpiBufs) * kStageBytes;
          ++slice;
          uint8_t* my = sb + lane * 128;
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const bool more = c0 + cols_per_slice < c_hi;
          if (a.z_elem == 2 && !(a.debug & 134217728)) {
            // bf16 Z: the next slice's first 32 columns load into v[0..31] as soon as this slice's first
            // half is staged, so the TMEM load latency overlaps the second half's conversion and stores
            // (experiment bit 134217728: both loads after all eight stores)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(my + ((j ^ (lane & 7)) << 4)) =
                  make_uint4(bf16x2(v[8 * j], v[8 * j + 1]), bf16x2(v[8 * j + 2], v[8 * j + 3]),
                             bf16x2(v[8 * j + 4], v[8 * j + 5]), bf16x2(v[8 * j + 6], v[8 * j + 7]));
            if (more) PPL_TMEM_LD32(trow + c0 + cols_per_slice, v);
#pragma unroll
            for (int j = 4; j < 8; ++j)
              *reinterpret_cast<uint4*>(my + ((j ^ (lane & 7)) << 4)) =
                  make_uint4(bf16x2(v[8 * j], v[8 * j + 1]), bf16x2(v[8 * j + 2], v[8 * j + 3]),
                             bf16x2(v[8 * j + 4], v[8 * j + 5]), bf16x2(v[8 * j + 6], v[8 * j + 7]));
            if (more) PPL_TMEM_LD32(trow + c0 + cols_per_slice + 32, (v + 32));
          } else {
            if (a.z_elem == 2) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<uint4*>(my + ((j ^ (lane & 7)) << 4)) =
                    make_uint4(bf16x2(v[8 * j], v[8 * j + 1]), bf16x2(v[8 * j + 2], v[8 * j + 3]),
                               bf16x2(v[8 * j + 4], v[8 * j + 5]), bf16x2(v[8 * j + 6], v[8 * j + 7]));
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<uint4*>(my + ((j ^ (lane & 7)) << 4)) =
                    make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
            if (more) ld_slice(c0 + cols_per_slice);
          }
          __syncwarp();
          if (a.debug & 2) continue;  // experiment: no Z stores
          if (tma_rows) {
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              asm volatile(
                  "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(zmap_addr),
                  "r"(h * kUmmaN + c0), "r"(k), "r"(r0 + e * 32), "r"(static_cast<int>(step)), "r"(smem_addr(sb))
                  : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
          } else {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int rr = it * 4 + (lane >> 3), chk = lane & 7;
              const uint4 y = *reinterpret_cast<const uint4*>(sb + rr * 128 + ((chk ^ (rr & 7)) << 4));
              if (e * 32 + rr < rows) {
                uint8_t* d = a.Z + step * a.z_stride +
                             ((static_cast<int64_t>(r0 + e * 32 + rr) * H + k) * D + h * kUmmaN + c0) * a.z_elem +
                             chk * 16;
                *reinterpret_cast<uint4*>(d) = y;
              }
            }
            __syncwarp();
          }
        }
        tc_fence_before();
        if constexpr (kPair) {  // every lane's tcgen05.ld has completed (wait::ld) before the warp's arrival
          __syncwarp();
          if (lane == 0) bar_arrive_remote_tmem(leader_addr(&t_empty[h]));
        } else {
          arrive_leader(&t_empty[h]);
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // as in k_gather_linear
  }
  if constexpr (kPair) {
    // no CTA leaves while the leader's MMAs may still read the peer's shared memory or signal its barriers
    if (warp == kMmaWarp) {
      if (lane == 0) bar_wait(fin, 0);
      __syncwarp();
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == kMmaWarp) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
  } else {
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
  }
}

static size_t linear_kc_smem_bytes(int D) {
  (void)D;  // the layout is sized for D = 512 (z_s at a fixed offset)
  return 1024 + static_cast<size_t>(kKcWStages) * (512 / 64) * kKcWBox + 4 * kKcABytes + 64 +
         kEpiWarps * kEpiBufs * kStageBytes + 512;
}

bool linear_kc_supported(int H, int F, int D, int num_sms, int in_dtype, int out_dtype) {
  return F >= 4 && F % (in_dtype == 0 ? 4 : 8) == 0 && (D == 256 || D == 512) && H >= 1 && H <= num_sms && (out_dtype == 1 || out_dtype == 2);
}

namespace {
// W as {column d, row f, hop k} of the batch dtype, box 64 columns x 64 rows (one K chunk).
bool encode_w_map_kc(const LinearArgs& a, CUtensorMap* m) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (encode == nullptr) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(a.D), static_cast<cuuint64_t>(a.F), static_cast<cuuint64_t>(a.H)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(a.D) * 2, static_cast<cuuint64_t>(a.F) * a.D * 2};
  // one whole chunk per box (64 K rows), half a chunk in the half-chunk experiment layout (bit 2048)
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>((a.debug & 2048) ? kKcChunk / 2 : kKcChunk), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(m, a.out_dtype == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                const_cast<void*>(a.W), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
// The store as a 2-D map {record element, row} of 16-bit elements (row pitch = the record stride),
// box 64 elements x 1 row, 128-byte swizzle: each tile::gather4 lands 4 rows x 128 B as rows of
// the SW128 K-major A chunk.
bool encode_a_map_kc(const LinearArgs& a, CUtensorMap* m) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (encode == nullptr) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.rec_stride / 2), static_cast<cuuint64_t>(a.shards[0].n_hbm)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.rec_stride)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kKcChunk), 1};
  const cuuint32_t estr[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint8_t*>(a.shards[0].hbm), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// fp32 records: {record element, row} of fp32, box 32 elements (128 B) x 1 row, 128-byte swizzle; or
// (wide) box 64 elements (256 B) x 1 row, unswizzled: one gather4 per 4 rows of a whole chunk.
// hop_rows: the map is {hop element, (node, hop) row} with row pitch F * 4 (records unpadded: rec_stride
// == H F 4), so a chunk past F reads nothing -- the K padding is the out-of-bounds zero fill instead of
// the next hop's bytes (products' F = 100: 400 instead of 512 bytes per row and hop).
bool encode_a_map_f32_kc(const LinearArgs& a, CUtensorMap* m, bool wide, bool hop_rows, bool tile = false) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (encode == nullptr) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(hop_rows ? a.F : a.rec_stride / 4),
                              static_cast<cuuint64_t>(a.shards[0].n_hbm * (hop_rows ? a.H : 1))};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(hop_rows ? a.F * 4 : a.rec_stride)};
  const cuuint32_t box[2] = {tile ? 128u : wide ? 64u : 32u, 1};
  const cuuint32_t estr[2] = {1, 1};
  wide = wide || tile;
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint8_t*>(a.shards[0].hbm), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, wide ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                wide ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

cudaError_t launch_gather_linear_kc(const LinearArgs& a_in, bool pdl, cudaStream_t st) {
  if (!linear_kc_supported(a_in.H, a_in.F, a_in.D, a_in.num_sms, a_in.in_dtype, a_in.out_dtype))
    return cudaErrorInvalidValue;
  const size_t smem = linear_kc_smem_bytes(a_in.D);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_gather_linear_kc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(linear_kc_smem_bytes(512)));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_gather_linear_kc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(linear_kc_smem_bytes(512)));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  LinearArgs a = a_in;
  alignas(64) CUtensorMap zmap{};
  a.z_tma = encode_z_map(a, &zmap) ? 1 : 0;
  alignas(64) CUtensorMap wmap{};
  if (!encode_w_map_kc(a, &wmap)) return cudaErrorNotSupported;
  // A chunks by TMA gather4: 16-bit records (copied as they are), whole 64-element chunks inside
  // each hop (F % 64 == 0), one HBM-resident unsharded store
  alignas(64) CUtensorMap amap{};
  // Default for eligible stores; PPLOAD_LINEAR_TMA_A=0 forces the register-staged producers,
  // =2 spreads the gather4 issue over all eight producer warps (r2: one issuing lane 21.4 ms, four
  // warps 12.6 ms, register producers 14.8 ms per MAG240M-row epoch)
  const char* ta = getenv("PPLOAD_LINEAR_TMA_A");
  const int want_tma = ta ? atoi(ta) : 1;
  a.tma_a = 0;
  if (want_tma > 0 && a.in_dtype != 0 && a.F % kKcChunk == 0 && a.world == 1 &&
      a.shards[0].spill == nullptr && a.shards[0].hbm != nullptr && a.shards[0].n_hbm > 0 &&
      a.shards[0].n_hbm < (int64_t(1) << 31) && a.rec_stride % 16 == 0)
    a.tma_a = encode_a_map_kc(a, &amap) ? want_tma : 0;
  // fp32 records: gather4 into a staging ring, converted in place by four warps. Default (2): whole
  // 64-element chunks as unswizzled 256-byte boxes (half the gather4s; the converters take 2-way bank
  // conflicts); interleaved A/B at IGB-large rows 15.8-16.9 vs 16.8-18.9 ms per epoch in pairs, 18.8-20.2
  // vs 20.5-21.3 single (profiles/r2/kc_pair/s2s_ab_wide.jsonl). =1: 128-byte SW128 halves; =0: the
  // register-staged producers
  const char* tf = getenv("PPLOAD_LINEAR_TMA_F32");
  a.tma_f32 = 0;
  if (!(tf && !strcmp(tf, "0")) && a.in_dtype == 0 && a.F % 4 == 0 && a.world == 1 &&
      a.shards[0].spill == nullptr && a.shards[0].hbm != nullptr && a.shards[0].n_hbm > 0 &&
      a.shards[0].n_hbm < (int64_t(1) << 31) && a.rec_stride % 16 == 0)
  {
    const int want = tf ? atoi(tf) : 2;
    // (node, hop) rows when the records are unpadded and F % 64 != 0 (experiment bit 524288: off)
    const bool hop_rows = a.F % kKcChunk != 0 && a.rec_stride == static_cast<int64_t>(a.H) * a.F * 4 &&
                          a.shards[0].n_hbm * a.H < (int64_t(1) << 31) && (a.debug & 524288) == 0;
    a.tma_f32 = encode_a_map_f32_kc(a, &amap, want >= 2, hop_rows) ? (want >= 2 ? 2 : 1) : 0;
    a.hop_rows = a.tma_f32 && hop_rows ? 1 : 0;
  }
  // CTA pairs (cta_group::2, M = 256): the default when the A chunks come by TMA (HBM-resident,
  // unsharded stores) -- half the W bytes through each SM's shared memory; interleaved A/B at MAG240M
  // rows 13.0-13.6 vs 16.4-17.9 ms (single CTAs also drop further under the power cap), IGB-large rows
  // 18.5-18.8 vs 19.0 ms (r2 second session, profiles/r2/kc_issue/s2*_ab_pair.jsonl).
  // PPLOAD_LINEAR_PAIR=0/1 forces the choice; experiment bit 8192 flips it
  const char* pe = getenv("PPLOAD_LINEAR_PAIR");
  bool pair = pe && *pe ? !strcmp(pe, "1") : (a.tma_a || a.tma_f32);
  if (a.debug & 8192) pair = !pair;
  pair = pair && (a.num_sms / 2) >= a.H && (a.debug & 2048) == 0;
  a.pair = pair ? 1 : 0;
  // experiment bit 4194304 (fp32 records with 64 < F <= 128 in pairs, A ring of 4 chunk positions): one
  // 512-byte gather4 box per (node, hop) row stages both chunks of a tile at once -- half the gather4 row
  // requests of the 256-byte boxes. Measured no faster at the products shape (A side alone 1.65 vs
  // 1.56 ms per epoch, whole kernel equal; profiles/r2/kc_products/s3j_ab.jsonl, s3k_ab.jsonl), so off
  // Generalised to any even number of chunks (F > 64): chunk pairs (2c, 2c + 1) as one 512-byte box per row
  // (PPLOAD_LINEAR_TMA_F32=3 or the bit; the (node, hop) row map when F % 64 != 0, else the record map)
  const int nch_ = (a.F + kKcChunk - 1) / kKcChunk;
  const bool want3 = (a.debug & 4194304) != 0 || (tf && atoi(tf) == 3);
  if (pair && a.tma_f32 == 2 && a.F > kKcChunk && nch_ % 2 == 0 && want3) {
    const bool hr = a.F % kKcChunk != 0;  // the record map reads whole 128-element boxes inside the hop
    alignas(64) CUtensorMap tmap{};
    if ((!hr || (a.rec_stride == static_cast<int64_t>(a.H) * a.F * 4 &&
                 a.shards[0].n_hbm * a.H < (int64_t(1) << 31) && (a.debug & 524288) == 0)) &&
        encode_a_map_f32_kc(a, &tmap, true, hr, true)) {
      amap = tmap;
      a.tma_f32 = 3;
      a.hop_rows = hr ? 1 : 0;
    }
  }
  // (tile, hop) work units over the whole grid when W_k is streamed per tile (F > 128) and the A
  // chunks come by TMA (the register producers keep hop-pinned CTAs); experiment bit 262144: off
  const bool w_resident = (a.F + kKcChunk - 1) / kKcChunk <= 2;
  a.units = (a.tma_a || a.tma_f32) && !w_resident && (a.debug & (2048 | 262144)) == 0 ? 1 : 0;
  const int per = a.units ? (pair ? 2 : 1) : a.H * (pair ? 2 : 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.num_sms / per) * per);
  cfg.blockDim = dim3(kLinThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute lattr[2];
  lattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  lattr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  lattr[1].id = cudaLaunchAttributeClusterDimension;
  lattr[1].val.clusterDim.x = pair ? 2 : 1;
  lattr[1].val.clusterDim.y = 1;
  lattr[1].val.clusterDim.z = 1;
  cfg.attrs = lattr;
  cfg.numAttrs = 2;
  return pair ? cudaLaunchKernelEx(&cfg, k_gather_linear_kc<true>, a, zmap, wmap, amap)
              : cudaLaunchKernelEx(&cfg, k_gather_linear_kc<false>, a, zmap, wmap, amap);
}

}  // namespace ppl
