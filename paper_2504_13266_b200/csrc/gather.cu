// Batch assembly kernels (K3/K5/K6 of §2.3).
//
// out[j, k, f] = cast(X_k[v_j, f]),  v_j = S[order[p_j]]  (oracle O8-O10)
// "copy the scattered node features" of a batch into one contiguous tensor
// (PAPER.md:259), done on the GPU with the fp32 -> bf16/fp16 RNE cast fused.
//
// B200 design.
//   * The store is node-major [rows, H, F]: one node's K+1 hop vectors are one
//     contiguous record (1600 B for ogbn-products fp32), so a batch row is a
//     single streaming copy instead of H scattered ones.
//   * A CTA takes a tile of 32 batch rows.  Threads 0..31 resolve the rows
//     (order -> node set -> owner shard -> HBM or pinned-host record) once and
//     park the 32 source pointers in shared memory; all 256 threads then sweep
//     the tile's rows x (record / 32 B) vector slots flattened, so every lane
//     works even when a record is not a multiple of 32 vectors (50 for
//     products).  Loads are 128-bit, read-only, L1-no-allocate, four slots per
//     thread issued before any store (~64 KB in flight per SM).
//   * Rows past the HBM budget are read from pinned, mapped host memory with
//     the same instructions (UVA zero-copy over PCIe, K6).  Sharded loaders
//     read the owner's store through a peer pointer (NVLink loads, A5).
//   * Casts use cvt.rn.{bf16x2,f16x2}.f32 (round to nearest even).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.h"
#include "philox.cuh"

namespace ppl {

constexpr int kMaxTileRows = 128;  // small records use larger tiles (pp_loader picks tile_rows)
constexpr int kGatherThreads = 256;
constexpr int kUnroll = 4;
constexpr int kMinBlocksPerSM = 4;  // caps registers at 64 -> 32 resident warps per SM

enum { kF32 = 0, kBF16 = 1, kF16 = 2 };
enum { kModeBF16 = 0, kModeF16 = 1, kModeCopy = 2 };

__device__ __forceinline__ uint4 ld_stream(const void* p, int l2_prefetch = 0) {
  uint4 r;
  if (l2_prefetch == 2) {  // experiment knob (PPLOAD_L2_PREFETCH): 256-byte L2 prefetch hint
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  } else if (l2_prefetch == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  }
  return r;
}

__device__ __forceinline__ void st_vec(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack_f16(uint32_t lo, uint32_t hi) {
  const __half2 h = __floats2half2_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<const uint32_t*>(&h);
}

// e / d for e * d < 2^40 with M = ceil(2^40 / d)
__device__ __forceinline__ uint32_t fast_div(uint32_t e, uint64_t M) {
  return static_cast<uint32_t>((static_cast<uint64_t>(e) * M) >> 40);
}

// Tile t of a launch -> (step, first row j0, rows, first order position); rows <= 0: empty.
struct TileCursor {
  int64_t step, pos;
  int j0, rows;
};
__device__ __forceinline__ TileCursor tile_cursor(const GatherArgs& a, int64_t tile, int64_t tiles_per_step,
                                                  int64_t total_tiles, int tile_rows) {
  TileCursor c{0, 0, 0, 0};
  if (tile >= total_tiles) return c;
  c.step = tile / tiles_per_step;
  c.j0 = static_cast<int>(tile - c.step * tiles_per_step) * tile_rows;
  const int64_t step_pos = a.first_pos + c.step * a.step_stride;
  const int64_t nrows_step = min(static_cast<int64_t>(a.B), a.N - step_pos);
  c.rows = static_cast<int>(min(static_cast<int64_t>(tile_rows), nrows_step - c.j0));
  c.pos = step_pos + c.j0;
  return c;
}

// This thread's order[] entry of tile t (threads < rows), loaded a tile ahead of its use.
__device__ __forceinline__ uint32_t prefetch_order(const GatherArgs& a, int64_t tile, int64_t tiles_per_step,
                                                   int64_t total_tiles, int tile_rows) {
  const TileCursor c = tile_cursor(a, tile, tiles_per_step, total_tiles, tile_rows);
  return (c.rows > 0 && static_cast<int>(threadIdx.x) < c.rows) ? a.order[c.pos + threadIdx.x] : 0u;
}

// Resolve the tile's rows (threads 0..rows-1): source record pointer into
// shared memory, labels / node ids out.
// PF: `ord` is this row's order[] entry, fetched a tile ahead; otherwise it is loaded here.
template <bool SHARDED, bool PF>
__device__ __forceinline__ void resolve_rows(const GatherArgs& a, int64_t step, int64_t step_pos, int j0, int rows,
                                             uint32_t ord, const uint8_t** s_src) {
  if (threadIdx.x < rows) {
    uint64_t v = PF ? ord : a.order[step_pos + j0 + threadIdx.x];
    if (a.node_set != nullptr) v = static_cast<uint64_t>(a.node_set[v]);
    int owner = 0;
    uint64_t lr = v;
    if (SHARDED) {
      owner = static_cast<int>(v % static_cast<uint64_t>(a.W));
      lr = v / static_cast<uint64_t>(a.W);
    }
    const ShardView sh = a.shards[owner];
    const int64_t l = static_cast<int64_t>(lr);
    if (SHARDED && sh.xhbm != nullptr && l < sh.n_hbm)  // peer row, already cast: bit 0 marks it
      s_src[threadIdx.x] = sh.xhbm + l * a.xrec_stride + 1;
    else
      s_src[threadIdx.x] = l < sh.n_hbm ? sh.hbm + l * a.rec_stride : sh.spill + (l - sh.n_hbm) * a.rec_stride;
    const int64_t oj = step * a.B + j0 + threadIdx.x;
    const uint64_t id = a.out_ids != nullptr ? static_cast<uint64_t>(a.out_ids[v]) : v;
    if (a.out_labels != nullptr) a.out_labels[oj] = a.labels[id];
    if (a.out_nodes != nullptr) a.out_nodes[oj] = static_cast<int64_t>(id);
  }
}

// Vector path: MODE bf16/f16 reads 32 B (8 fp32) and writes 16 B; copy mode
// moves 16 B.  vpr = vector slots per row.
// PF: fetch the next tile's order[] entries one tile ahead (used with the larger tiles of
// small records, where the order -> record round trip would dominate; for records >= 1 KB
// the extra registers cost more than they save, r1z).
template <int MODE, bool SHARDED, bool PF>
__global__ void __launch_bounds__(kGatherThreads, kMinBlocksPerSM)
    k_gather_vec(const GatherArgs a, uint32_t vpr, uint64_t vpr_M, int64_t row_out_bytes) {
  __shared__ const uint8_t* s_src[2][kMaxTileRows];
  // Programmatic dependent launch: the next batch's gather may start as soon as
  // every CTA of this one is running (batches are independent; see launch_gather).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int kInBytes = (MODE == kModeCopy) ? 16 : 32;
  const int kTileRows = a.tile_rows;
  const int64_t tiles_per_step = (a.B + kTileRows - 1) / kTileRows;
  const int64_t total_tiles = tiles_per_step * a.nsteps;
  int buf = 0;
  // order[] entries of this CTA's next tile are loaded one tile ahead, so the order ->
  // record dependency costs no extra memory round trip per tile (matters for small records)
  uint32_t ord = PF ? prefetch_order(a, blockIdx.x, tiles_per_step, total_tiles, kTileRows) : 0u;
  for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    const int64_t step = tile / tiles_per_step;
    const int j0 = static_cast<int>(tile - step * tiles_per_step) * kTileRows;
    const int64_t step_pos = a.first_pos + step * a.step_stride;
    const int64_t nrows_step = min(static_cast<int64_t>(a.B), a.N - step_pos);
    const int rows = static_cast<int>(min(static_cast<int64_t>(kTileRows), nrows_step - j0));
    const uint32_t my_ord = ord;
    if (PF) ord = prefetch_order(a, tile + gridDim.x, tiles_per_step, total_tiles, kTileRows);
    if (rows <= 0) continue;  // block-uniform; buf is not toggled
    resolve_rows<SHARDED, PF>(a, step, step_pos, j0, rows, my_ord, s_src[buf]);
    __syncthreads();
    uint8_t* out_tile = a.out + step * a.out_stride + static_cast<int64_t>(j0) * row_out_bytes;
    const uint32_t nvec = static_cast<uint32_t>(rows) * vpr;
    for (uint32_t e0 = threadIdx.x; e0 < nvec; e0 += kGatherThreads * kUnroll) {
      uint4 x0[kUnroll], x1[kUnroll];
      bool pre[kUnroll];  // slot of a peer's exchange copy: 16 bytes already in the batch dtype
#pragma unroll
      for (int q = 0; q < kUnroll; ++q) {
        const uint32_t e = e0 + q * kGatherThreads;
        pre[q] = false;
        if (e < nvec) {
          const uint32_t r = fast_div(e, vpr_M);
          const uint32_t c = e - r * vpr;
          const uint8_t* row = s_src[buf][r];
          if (SHARDED && MODE != kModeCopy && (reinterpret_cast<uintptr_t>(row) & 1u)) {
            pre[q] = true;
            x0[q] = ld_stream(row - 1 + static_cast<int64_t>(c) * 16, a.l2_prefetch);
          } else {
            const uint8_t* src = row + static_cast<int64_t>(c) * kInBytes;
            x0[q] = ld_stream(src, a.l2_prefetch);
            if (MODE != kModeCopy) x1[q] = ld_stream(src + 16, a.l2_prefetch);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kUnroll; ++q) {
        const uint32_t e = e0 + q * kGatherThreads;
        if (e < nvec) {
          const uint32_t r = fast_div(e, vpr_M);
          const uint32_t c = e - r * vpr;
          uint8_t* dst = out_tile + static_cast<int64_t>(r) * row_out_bytes + static_cast<int64_t>(c) * 16;
          uint4 y;
          if (SHARDED && pre[q]) {
            y = x0[q];
          } else if (MODE == kModeBF16) {
            y = make_uint4(pack_bf16(x0[q].x, x0[q].y), pack_bf16(x0[q].z, x0[q].w), pack_bf16(x1[q].x, x1[q].y),
                           pack_bf16(x1[q].z, x1[q].w));
          } else if (MODE == kModeF16) {
            y = make_uint4(pack_f16(x0[q].x, x0[q].y), pack_f16(x0[q].z, x0[q].w), pack_f16(x1[q].x, x1[q].y),
                           pack_f16(x1[q].z, x1[q].w));
          } else {
            y = x0[q];
          }
          st_vec(dst, y);
        }
      }
    }
    buf ^= 1;
  }
}

// Scalar fallback for records whose size / alignment rule out the vector
// path.  Same tile structure, one element per slot.
template <bool SHARDED>
__global__ void __launch_bounds__(kGatherThreads, kMinBlocksPerSM)
    k_gather_scalar(const GatherArgs a, uint32_t HF, uint64_t HF_M) {
  __shared__ const uint8_t* s_src[2][kMaxTileRows];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int kTileRows = a.tile_rows;
  const int s_in = a.in_dtype == kF32 ? 4 : 2;
  const int s_out = a.out_dtype == kF32 ? 4 : 2;
  const int64_t row_out_bytes = static_cast<int64_t>(HF) * s_out;
  const int64_t tiles_per_step = (a.B + kTileRows - 1) / kTileRows;
  const int64_t total_tiles = tiles_per_step * a.nsteps;
  int buf = 0;
  for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    const int64_t step = tile / tiles_per_step;
    const int j0 = static_cast<int>(tile - step * tiles_per_step) * kTileRows;
    const int64_t step_pos = a.first_pos + step * a.step_stride;
    const int64_t nrows_step = min(static_cast<int64_t>(a.B), a.N - step_pos);
    const int rows = static_cast<int>(min(static_cast<int64_t>(kTileRows), nrows_step - j0));
    if (rows <= 0) continue;
    resolve_rows<SHARDED, false>(a, step, step_pos, j0, rows, 0u, s_src[buf]);
    __syncthreads();
    uint8_t* out_tile = a.out + step * a.out_stride + static_cast<int64_t>(j0) * row_out_bytes;
    const uint32_t nel = static_cast<uint32_t>(rows) * HF;
    for (uint32_t e = threadIdx.x; e < nel; e += kGatherThreads) {
      const uint32_t r = fast_div(e, HF_M);
      const uint32_t i = e - r * HF;
      const uint8_t* row = s_src[buf][r];
      uint8_t* dst = out_tile + static_cast<int64_t>(r) * row_out_bytes + static_cast<int64_t>(i) * s_out;
      if (SHARDED && (reinterpret_cast<uintptr_t>(row) & 1u)) {
        // a peer's exchange copy (bit 0 tags it, see resolve_rows): elements already in the batch dtype
        *reinterpret_cast<uint16_t*>(dst) =
            __ldg(reinterpret_cast<const unsigned short*>(row - 1 + static_cast<int64_t>(i) * 2));
        continue;
      }
      const uint8_t* src = row + static_cast<int64_t>(i) * s_in;
      if (s_in == 4) {
        const uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(src));
        if (a.out_dtype == kBF16) {
          const __nv_bfloat16 h = __float2bfloat16_rn(__uint_as_float(x));
          *reinterpret_cast<__nv_bfloat16*>(dst) = h;
        } else if (a.out_dtype == kF16) {
          const __half h = __float2half_rn(__uint_as_float(x));
          *reinterpret_cast<__half*>(dst) = h;
        } else {
          *reinterpret_cast<uint32_t*>(dst) = x;
        }
      } else {
        *reinterpret_cast<uint16_t*>(dst) = __ldg(reinterpret_cast<const unsigned short*>(src));
      }
    }
    buf ^= 1;
  }
}

// ---- K4: bulk-copy (TMA engine) variant --------------------------------------
// Whole node records are moved global -> shared by cp.async.bulk (one bulk copy
// per batch row, issued by the lane that resolved the row), tracked by an
// mbarrier per stage; all warps then convert shared -> registers -> 128-bit
// global stores.  kStages tiles of rows are in flight per CTA, so the number
// of outstanding bytes no longer depends on registers and the copy engine
// issues large requests (this is the path for pinned-host (PCIe) and peer
// (NVLink) sources, where request size and depth matter most).
constexpr int kTmaStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int MODE, bool SHARDED>
__global__ void __launch_bounds__(kGatherThreads, 2)
    k_gather_tma(const GatherArgs a, uint32_t vpr, uint64_t vpr_M, int64_t row_out_bytes, int32_t rec_in,
                 int32_t tr) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kTmaStages];
  __shared__ uint8_t s_pre[kTmaStages][32];  // row holds a peer's exchange copy (already cast)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int kInBytes = (MODE == kModeCopy) ? 16 : 32;
  const int64_t tiles_per_step = (a.B + tr - 1) / tr;
  const int64_t total_tiles = tiles_per_step * a.nsteps;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // tile k of this CTA -> (step, first row, rows); rows <= 0 marks an empty tile
  auto tile_of = [&](int64_t k, int64_t& step, int& j0, int64_t& step_pos) -> int {
    const int64_t tile = blockIdx.x + k * gridDim.x;
    if (tile >= total_tiles) return -1;
    step = tile / tiles_per_step;
    j0 = static_cast<int>(tile - step * tiles_per_step) * tr;
    step_pos = a.first_pos + step * a.step_stride;
    const int64_t nrows_step = min(static_cast<int64_t>(a.B), a.N - step_pos);
    return static_cast<int>(min(static_cast<int64_t>(tr), nrows_step - j0));
  };
  const int64_t stage_bytes = static_cast<int64_t>(tr) * rec_in;
  // warp 0: resolve the rows of tile k and start their bulk copies into stage s
  auto issue = [&](int64_t k) {
    int64_t step, step_pos;
    int j0;
    const int rows = tile_of(k, step, j0, step_pos);
    if (rows <= 0) return;
    const int s = static_cast<int>(k % kTmaStages);
    uint8_t* stage = smem + s * stage_bytes;
    // rows <= 16 <= 32: lane j resolves row j, the warp sums the bytes for expect_tx
    const int j = lane;
    const uint8_t* src = nullptr;
    uint32_t bytes = 0;
    uint64_t v = 0;
    if (j < rows) {
      const int64_t p = step_pos + j0 + j;
      v = a.order[p];
      if (a.node_set != nullptr) v = static_cast<uint64_t>(a.node_set[v]);
      int owner = 0;
      uint64_t lr = v;
      if (SHARDED) {
        owner = static_cast<int>(v % static_cast<uint64_t>(a.W));
        lr = v / static_cast<uint64_t>(a.W);
      }
      const ShardView sh = a.shards[owner];
      const int64_t l = static_cast<int64_t>(lr);
      const bool pre = SHARDED && MODE != kModeCopy && sh.xhbm != nullptr && l < sh.n_hbm;
      src = pre ? sh.xhbm + l * a.xrec_stride
                : (l < sh.n_hbm ? sh.hbm + l * a.rec_stride : sh.spill + (l - sh.n_hbm) * a.rec_stride);
      bytes = static_cast<uint32_t>(pre ? rec_in / 2 : rec_in);
      s_pre[s][j] = pre ? 1 : 0;
    }
    const uint32_t total_bytes = __reduce_add_sync(0xffffffffu, bytes);
    if (lane == 0) mbar_arrive_expect_tx(&full[s], total_bytes);
    __syncwarp();
    if (j < rows) {
      bulk_g2s(stage + static_cast<int64_t>(j) * rec_in, src, bytes, &full[s]);
      const int64_t oj = step * a.B + j0 + j;
      const uint64_t id = a.out_ids != nullptr ? static_cast<uint64_t>(a.out_ids[v]) : v;
      if (a.out_labels != nullptr) a.out_labels[oj] = a.labels[id];
      if (a.out_nodes != nullptr) a.out_nodes[oj] = static_cast<int64_t>(id);
    }
  };
  if (warp == 0)
    for (int k = 0; k < kTmaStages; ++k) issue(k);
  uint32_t phase = 0;  // bit s = parity of stage s
  for (int64_t k = 0;; ++k) {
    int64_t step, step_pos;
    int j0;
    const int rows = tile_of(k, step, j0, step_pos);
    if (rows == -1) break;
    const int s = static_cast<int>(k % kTmaStages);
    if (rows > 0) {
      mbar_wait(&full[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      const uint8_t* stage = smem + s * stage_bytes;
      uint8_t* out_tile = a.out + step * a.out_stride + static_cast<int64_t>(j0) * row_out_bytes;
      const uint32_t nvec = static_cast<uint32_t>(rows) * vpr;
      for (uint32_t e = threadIdx.x; e < nvec; e += kGatherThreads) {
        const uint32_t r = fast_div(e, vpr_M);
        const uint32_t c = e - r * vpr;
        const uint4* src = reinterpret_cast<const uint4*>(stage + static_cast<int64_t>(r) * rec_in + c * kInBytes);
        uint4 y;
        if (SHARDED && MODE != kModeCopy && s_pre[s][r]) {
          y = reinterpret_cast<const uint4*>(stage + static_cast<int64_t>(r) * rec_in)[c];
        } else if (MODE == kModeBF16) {
          const uint4 x0 = src[0], x1 = src[1];
          y = make_uint4(pack_bf16(x0.x, x0.y), pack_bf16(x0.z, x0.w), pack_bf16(x1.x, x1.y), pack_bf16(x1.z, x1.w));
        } else if (MODE == kModeF16) {
          const uint4 x0 = src[0], x1 = src[1];
          y = make_uint4(pack_f16(x0.x, x0.y), pack_f16(x0.z, x0.w), pack_f16(x1.x, x1.y), pack_f16(x1.z, x1.w));
        } else {
          y = src[0];
        }
        st_vec(out_tile + static_cast<int64_t>(r) * row_out_bytes + static_cast<int64_t>(c) * 16, y);
      }
    }
    __syncthreads();  // every warp is done reading stage s
    if (warp == 0) issue(k + kTmaStages);
  }
}

// rows per stage for the bulk-copy path (0: record too large for it)
static int tma_rows_per_stage(int64_t rec_in) {
  if (rec_in % 16 != 0 || rec_in * kTmaStages > 96 * 1024) return 0;
  int64_t tr = (24 * 1024) / rec_in;
  if (tr < 1) tr = 1;
  if (tr > 16) tr = 16;
  return static_cast<int>(tr);
}

// Exchange copy: one thread per 16-byte output vector (8 elements).
template <int MODE>
__global__ void k_cast_records(const uint8_t* __restrict__ src, int64_t rows, int64_t rec_stride, uint32_t vpr,
                               uint8_t* __restrict__ dst, int64_t xrec_stride) {
  const int64_t total = rows * vpr;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / vpr, c = i - r * vpr;
    const uint8_t* p = src + r * rec_stride + c * 32;
    const uint4 x0 = ld_stream(p), x1 = ld_stream(p + 16);
    uint4 y;
    if (MODE == kModeBF16)
      y = make_uint4(pack_bf16(x0.x, x0.y), pack_bf16(x0.z, x0.w), pack_bf16(x1.x, x1.y), pack_bf16(x1.z, x1.w));
    else
      y = make_uint4(pack_f16(x0.x, x0.y), pack_f16(x0.z, x0.w), pack_f16(x1.x, x1.y), pack_f16(x1.z, x1.w));
    st_vec(dst + r * xrec_stride + c * 16, y);
  }
}

cudaError_t launch_cast_records(const uint8_t* src, int64_t rows, int64_t rec_stride, int32_t HF, int32_t out_dtype,
                                uint8_t* dst, int64_t xrec_stride, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (HF % 8 != 0 || (out_dtype != kBF16 && out_dtype != kF16)) return cudaErrorInvalidValue;
  const uint32_t vpr = static_cast<uint32_t>(HF / 8);
  const int64_t total = rows * vpr;
  const int blocks = static_cast<int>(total / 256 + 1 < 148 * 16 ? total / 256 + 1 : 148 * 16);
  if (out_dtype == kBF16)
    k_cast_records<kModeBF16><<<blocks, 256, 0, st>>>(src, rows, rec_stride, vpr, dst, xrec_stride);
  else
    k_cast_records<kModeF16><<<blocks, 256, 0, st>>>(src, rows, rec_stride, vpr, dst, xrec_stride);
  return cudaGetLastError();
}

bool gather_vector_ok(int32_t HF, int32_t in_dtype, int32_t out_dtype, int64_t rec_stride) {
  const int s_in = in_dtype == kF32 ? 4 : 2;
  const int s_out = out_dtype == kF32 ? 4 : 2;
  const int64_t in_row = static_cast<int64_t>(HF) * s_in, out_row = static_cast<int64_t>(HF) * s_out;
  if (rec_stride % 16 != 0 || out_row % 16 != 0) return false;
  if (s_in == s_out) return in_row % 16 == 0;
  return in_row % 32 == 0;  // fp32 -> 16-bit: 8 elements per slot
}

template <typename Kern, typename... Args>
static cudaError_t launch_ex(Kern kern, uint32_t grid, bool pdl, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGatherThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

bool gather_tma_ok(int32_t HF, int32_t in_dtype) {
  return tma_rows_per_stage(static_cast<int64_t>(HF) * (in_dtype == kF32 ? 4 : 2)) > 0;
}

template <int MODE, bool SH>
static cudaError_t launch_tma(const GatherArgs& a, bool pdl, int grid_per_sm, cudaStream_t st, uint32_t vpr,
                              uint64_t M, int64_t row_out_bytes) {
  const int32_t rec_in = a.HF * (a.in_dtype == kF32 ? 4 : 2);
  const int tr = tma_rows_per_stage(rec_in);
  if (tr == 0) return cudaErrorInvalidValue;
  const size_t smem = static_cast<size_t>(kTmaStages) * tr * rec_in;
  static bool attr_set = false;  // per (MODE, SH) instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gather_tma<MODE, SH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         96 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int64_t tiles = ((a.B + tr - 1) / tr) * static_cast<int64_t>(a.nsteps);
  int64_t cap = static_cast<int64_t>(a.num_sms) * grid_per_sm;
  if (a.max_ctas > 0 && a.max_ctas < cap) cap = a.max_ctas;
  const uint32_t grid = static_cast<uint32_t>(tiles < cap ? tiles : cap);
  return launch_ex(k_gather_tma<MODE, SH>, grid, pdl, smem, st, a, vpr, M, row_out_bytes, rec_in, tr);
}

cudaError_t launch_gather(const GatherArgs& a, int path, bool pdl, int grid_per_sm, cudaStream_t st) {
  if (a.tile_rows < 1 || a.tile_rows > kMaxTileRows) return cudaErrorInvalidValue;
  const int64_t tiles = ((a.B + a.tile_rows - 1) / a.tile_rows) * static_cast<int64_t>(a.nsteps);
  if (tiles <= 0) return cudaSuccess;
  int64_t cap = static_cast<int64_t>(a.num_sms) * grid_per_sm;
  if (a.max_ctas > 0 && a.max_ctas < cap) cap = a.max_ctas;
  const uint32_t grid = static_cast<uint32_t>(tiles < cap ? tiles : cap);
  const bool sharded = a.W > 1;
  const int s_out = a.out_dtype == kF32 ? 4 : 2;
  if (path == kPathTma) {
    const int mode = (a.in_dtype == a.out_dtype) ? kModeCopy : (a.out_dtype == kBF16 ? kModeBF16 : kModeF16);
    const int64_t row_out_bytes = static_cast<int64_t>(a.HF) * s_out;
    const uint32_t vpr = static_cast<uint32_t>(row_out_bytes / 16);
    const uint64_t M = ((1ull << 40) + vpr - 1) / vpr;
#define PPL_GT(MODE, SH) return launch_tma<MODE, SH>(a, pdl, 2, st, vpr, M, row_out_bytes)
    if (mode == kModeBF16) { if (sharded) PPL_GT(kModeBF16, true); else PPL_GT(kModeBF16, false); }
    else if (mode == kModeF16) { if (sharded) PPL_GT(kModeF16, true); else PPL_GT(kModeF16, false); }
    else { if (sharded) PPL_GT(kModeCopy, true); else PPL_GT(kModeCopy, false); }
#undef PPL_GT
  }
  if (path == kPathVector) {
    const int mode = (a.in_dtype == a.out_dtype) ? kModeCopy : (a.out_dtype == kBF16 ? kModeBF16 : kModeF16);
    const int64_t row_out_bytes = static_cast<int64_t>(a.HF) * s_out;
    const uint32_t vpr = static_cast<uint32_t>(row_out_bytes / 16);
    const uint64_t M = ((1ull << 40) + vpr - 1) / vpr;
    if (static_cast<uint64_t>(kMaxTileRows) * vpr * vpr >= (1ull << 40)) return cudaErrorInvalidValue;
#define PPL_GV(MODE, SH)                                                                                 \
  return a.tile_rows > 32 ? launch_ex(k_gather_vec<MODE, SH, true>, grid, pdl, 0, st, a, vpr, M, row_out_bytes) \
                          : launch_ex(k_gather_vec<MODE, SH, false>, grid, pdl, 0, st, a, vpr, M, row_out_bytes)
    if (mode == kModeBF16) { if (sharded) PPL_GV(kModeBF16, true); else PPL_GV(kModeBF16, false); }
    else if (mode == kModeF16) { if (sharded) PPL_GV(kModeF16, true); else PPL_GV(kModeF16, false); }
    else { if (sharded) PPL_GV(kModeCopy, true); else PPL_GV(kModeCopy, false); }
#undef PPL_GV
  }
  const uint32_t HF = static_cast<uint32_t>(a.HF);
  if (static_cast<uint64_t>(kMaxTileRows) * HF * HF >= (1ull << 40)) return cudaErrorInvalidValue;
  const uint64_t M = ((1ull << 40) + HF - 1) / HF;
  if (sharded) return launch_ex(k_gather_scalar<true>, grid, pdl, 0, st, a, HF, M);
  return launch_ex(k_gather_scalar<false>, grid, pdl, 0, st, a, HF, M);
}

// ---- DMA-staged assembly (chunk reshuffling over host-resident rows) -----------
// The batch's records were DMA'd by the copy engines, in batch order, into a device
// staging area (one cudaMemcpyAsync per run of consecutive rows); this kernel casts
// staging record j into out row j and writes node ids / labels from the order.
template <int MODE>
__global__ void k_stage_cast(const uint8_t* __restrict__ stage, int64_t rec_stride, int32_t rows, uint32_t vpr,
                             int64_t row_out_bytes, uint8_t* __restrict__ out, const uint32_t* __restrict__ order,
                             const int64_t* __restrict__ node_set, const int32_t* __restrict__ labels,
                             int32_t* __restrict__ out_labels, int64_t* __restrict__ out_nodes) {
  constexpr int kInBytes = (MODE == kModeCopy) ? 16 : 32;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t j = tid; j < rows; j += nthr) {
    const uint64_t o = order[j];
    const int64_t id = node_set != nullptr ? node_set[o] : static_cast<int64_t>(o);
    if (out_nodes) out_nodes[j] = id;
    if (out_labels) out_labels[j] = labels[id];
  }
  const int64_t total = static_cast<int64_t>(rows) * vpr;
  for (int64_t e = tid; e < total; e += nthr) {
    const int64_t r = e / vpr, c = e - r * vpr;
    const uint8_t* src = stage + r * rec_stride + c * kInBytes;
    const uint4 x0 = ld_stream(src);
    uint4 y = x0;
    if (MODE != kModeCopy) {
      const uint4 x1 = ld_stream(src + 16);
      y = MODE == kModeBF16 ? make_uint4(pack_bf16(x0.x, x0.y), pack_bf16(x0.z, x0.w), pack_bf16(x1.x, x1.y),
                                         pack_bf16(x1.z, x1.w))
                            : make_uint4(pack_f16(x0.x, x0.y), pack_f16(x0.z, x0.w), pack_f16(x1.x, x1.y),
                                         pack_f16(x1.z, x1.w));
    }
    st_vec(out + r * row_out_bytes + c * 16, y);
  }
}

// Scalar variant (records that rule out 16-byte vectors).
__global__ void k_stage_cast_scalar(const uint8_t* __restrict__ stage, int64_t rec_stride, int32_t rows, int32_t HF,
                                    int32_t in_dtype, int32_t out_dtype, uint8_t* __restrict__ out,
                                    const uint32_t* __restrict__ order, const int64_t* __restrict__ node_set,
                                    const int32_t* __restrict__ labels, int32_t* __restrict__ out_labels,
                                    int64_t* __restrict__ out_nodes) {
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t j = tid; j < rows; j += nthr) {
    const uint64_t o = order[j];
    const int64_t id = node_set != nullptr ? node_set[o] : static_cast<int64_t>(o);
    if (out_nodes) out_nodes[j] = id;
    if (out_labels) out_labels[j] = labels[id];
  }
  const int s_in = in_dtype == kF32 ? 4 : 2, s_out = out_dtype == kF32 ? 4 : 2;
  const int64_t total = static_cast<int64_t>(rows) * HF;
  for (int64_t e = tid; e < total; e += nthr) {
    const int64_t r = e / HF, i = e - r * HF;
    const uint8_t* src = stage + r * rec_stride + i * s_in;
    uint8_t* dst = out + (r * HF + i) * s_out;
    if (s_in == 4) {
      const uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(src));
      if (out_dtype == kBF16)
        *reinterpret_cast<__nv_bfloat16*>(dst) = __float2bfloat16_rn(__uint_as_float(x));
      else if (out_dtype == kF16)
        *reinterpret_cast<__half*>(dst) = __float2half_rn(__uint_as_float(x));
      else
        *reinterpret_cast<uint32_t*>(dst) = x;
    } else {
      *reinterpret_cast<uint16_t*>(dst) = __ldg(reinterpret_cast<const unsigned short*>(src));
    }
  }
}

cudaError_t launch_stage_cast(const uint8_t* stage, int64_t rec_stride, int32_t rows, int32_t HF, int32_t in_dtype,
                              int32_t out_dtype, bool vec, uint8_t* out, const uint32_t* order,
                              const int64_t* node_set, const int32_t* labels, int32_t* out_labels, int64_t* out_nodes,
                              cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int s_out = out_dtype == kF32 ? 4 : 2;
  const int64_t row_out_bytes = static_cast<int64_t>(HF) * s_out;
  if (vec) {
    const uint32_t vpr = static_cast<uint32_t>(row_out_bytes / 16);
    const int64_t total = static_cast<int64_t>(rows) * vpr;
    const uint32_t grid = static_cast<uint32_t>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    const int mode = (in_dtype == out_dtype) ? kModeCopy : (out_dtype == kBF16 ? kModeBF16 : kModeF16);
    if (mode == kModeBF16)
      k_stage_cast<kModeBF16><<<grid, 256, 0, st>>>(stage, rec_stride, rows, vpr, row_out_bytes, out, order, node_set,
                                                      labels, out_labels, out_nodes);
    else if (mode == kModeF16)
      k_stage_cast<kModeF16><<<grid, 256, 0, st>>>(stage, rec_stride, rows, vpr, row_out_bytes, out, order, node_set,
                                                     labels, out_labels, out_nodes);
    else
      k_stage_cast<kModeCopy><<<grid, 256, 0, st>>>(stage, rec_stride, rows, vpr, row_out_bytes, out, order, node_set,
                                                      labels, out_labels, out_nodes);
  } else {
    const int64_t total = static_cast<int64_t>(rows) * HF;
    const uint32_t grid = static_cast<uint32_t>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    k_stage_cast_scalar<<<grid, 256, 0, st>>>(stage, rec_stride, rows, HF, in_dtype, out_dtype, out, order, node_set,
                                              labels, out_labels, out_nodes);
  }
  return cudaGetLastError();
}

// ---- K10: synthetic fill (SURVEY.md §8(d) generators G / G16) ----------------
__global__ void k_fill_synthetic(uint8_t* __restrict__ base, int64_t row0, int64_t nrows, int64_t rec_stride,
                                 int32_t H, int32_t F, int32_t dtype, uint64_t seed, int32_t W, int32_t rank,
                                 const int64_t* __restrict__ ids) {
  const int32_t F4 = (F + 3) / 4;
  const int64_t total = nrows * H * F4;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = t / (static_cast<int64_t>(H) * F4);
    const int32_t rem = static_cast<int32_t>(t - row * H * F4);
    const int32_t k = rem / F4;
    const int32_t f4 = rem - k * F4;
    const uint64_t x = static_cast<uint64_t>(row0 + row) * W + rank;  // row space index of this record
    const uint64_t v = ids != nullptr ? static_cast<uint64_t>(ids[x]) : x;  // global node id
    const uint4 w4 = synth_block(seed, v, static_cast<uint32_t>(k), static_cast<uint32_t>(f4));
    const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
    uint8_t* rec = base + row * rec_stride;
    for (int q = 0; q < 4; ++q) {
      const int32_t f = f4 * 4 + q;
      if (f >= F) break;
      if (dtype == kF32) {
        const uint32_t bits = (w[q] & 0x807FFFFFu) | ((120u + ((w[q] >> 23) & 15u)) << 23);
        reinterpret_cast<uint32_t*>(rec)[static_cast<int64_t>(k) * F + f] = bits;
      } else {
        const uint16_t h = static_cast<uint16_t>((w[q] & 0x83FFu) | ((8u + ((w[q] >> 10) & 15u)) << 10));
        reinterpret_cast<uint16_t*>(rec)[static_cast<int64_t>(k) * F + f] = h;
      }
    }
  }
}

cudaError_t launch_fill_synthetic(uint8_t* base, int64_t row0, int64_t nrows, int64_t rec_stride, int32_t H,
                                  int32_t F, int32_t dtype, uint64_t data_seed, int32_t W, int32_t rank,
                                  const int64_t* ids, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  k_fill_synthetic<<<148 * 16, 256, 0, st>>>(base, row0, nrows, rec_stride, H, F, dtype, data_seed, W, rank, ids);
  return cudaGetLastError();
}

// Compact store from a device source: record r = the H hop vectors of node ids[r*W + rank]
// (element strides hop_stride / row_stride of the source), elem = 2 or 4 bytes.
__global__ void k_pack_rows(const uint8_t* __restrict__ src, int64_t hop_stride, int64_t row_stride, int32_t elem,
                            int32_t H, int32_t F, const int64_t* __restrict__ ids, int64_t nrows, int32_t W,
                            int32_t rank, uint8_t* __restrict__ dst, int64_t rec_stride) {
  const int64_t total = nrows * H * F;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / (static_cast<int64_t>(H) * F);
    const int32_t kf = static_cast<int32_t>(t - r * H * F);
    const int32_t k = kf / F, f = kf - k * F;
    const int64_t v = ids[r * W + rank];
    const int64_t e = k * hop_stride + v * row_stride + f;
    uint8_t* d = dst + r * rec_stride + static_cast<int64_t>(kf) * elem;
    if (elem == 4)
      *reinterpret_cast<uint32_t*>(d) = reinterpret_cast<const uint32_t*>(src)[e];
    else
      *reinterpret_cast<uint16_t*>(d) = reinterpret_cast<const uint16_t*>(src)[e];
  }
}

cudaError_t launch_pack_rows(const void* src, int64_t hop_stride, int64_t row_stride, int32_t elem, int32_t H,
                             int32_t F, const int64_t* ids, int64_t nrows, int32_t W, int32_t rank, uint8_t* dst,
                             int64_t rec_stride, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  k_pack_rows<<<148 * 16, 256, 0, st>>>(static_cast<const uint8_t*>(src), hop_stride, row_stride, elem, H, F, ids,
                                        nrows, W, rank, dst, rec_stride);
  return cudaGetLastError();
}

__global__ void k_order_to_nodes(const uint32_t* __restrict__ order, const int64_t* __restrict__ node_set,
                                 int64_t N, int64_t* __restrict__ dst) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < N;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t i = order[p];
    dst[p] = node_set != nullptr ? node_set[i] : static_cast<int64_t>(i);
  }
}

cudaError_t launch_order_to_nodes(const uint32_t* order, const int64_t* node_set, int64_t N, int64_t* dst,
                                  cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  k_order_to_nodes<<<148 * 8, 256, 0, st>>>(order, node_set, N, dst);
  return cudaGetLastError();
}

}  // namespace ppl
