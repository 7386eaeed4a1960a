// C-ABI implementation of libppload.so (include/pp_loader.h).
//
// Owns: the node-major hop store (HBM part + pinned/mapped host spill), the
// uploaded node set and labels, the epoch order and sort scratch, the loader
// stream and its events, and peer store mappings.  All compute is in the
// kernels of permute.cu / gather.cu; this file validates, allocates, lays out
// and enqueues.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/pp_loader.h"
#include "internal.h"

using namespace ppl;

namespace {

thread_local std::string g_last_error;

pp_status fail(pp_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

int elem_bytes(pp_dtype d) { return d == PP_F32 ? 4 : 2; }
bool valid_dtype(int d) { return d == PP_F32 || d == PP_BF16 || d == PP_F16; }

// NVTX range around each public call (nsys / ncu timelines show the loader's host-side phases; the
// header-only NVTX API costs a few ns when no tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DevGuard {
  int prev = -1;
  bool ok = true;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DevGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

struct pp_loader {
  pp_loader_desc desc{};
  int dev = 0;
  int32_t W = 1, rank = 0, H = 0, F = 0, HF = 0;
  pp_dtype in_dtype = PP_F32, out_dtype = PP_BF16;
  int64_t N_total = 0, N = 0, B = 0, local_rows = 0, n_hbm = 0, n_spill = 0;
  int64_t rec_in = 0, rec_stride = 0, rec_out = 0, steps = 0;
  bool vector_path = true;

  uint8_t* d_store = nullptr;
  bool borrowed = false;        // d_store is the caller's buffer (desc.borrow_device_data)
  uint8_t* h_spill = nullptr;
  uint8_t* d_spill = nullptr;  // device alias of h_spill
  int spill_fd = -1;           // PP_PEERS_IPC spill: memfd shared with the peers (h_spill = its mapping)
  size_t spill_bytes = 0;
  struct PeerSpill {
    void* p;
    size_t bytes;
  };
  std::vector<PeerSpill> peer_spills;  // peers' spill files mapped + registered here
  uint8_t* d_xstore = nullptr;  // exchange copy: HBM rows cast to out_dtype, read by the peers (W > 1)
  int64_t xrec_stride = 0;      // its pitch (same on every rank; 0 when the dtype pair has no cast)
  int64_t* d_node_set = nullptr;
  int32_t* d_labels = nullptr;
  bool has_labels = false;

  uint32_t* d_orders[2] = {nullptr, nullptr};  // current epoch + prefetched next epoch (allocated at first prefetch)
  int cur = 0;
  uint32_t* d_order = nullptr;                  // == d_orders[cur]
  uint32_t* d_pi = nullptr;
  int64_t pi_cap = 0;
  int64_t tmp_cap = 0;  // units SortScratch::tmp holds (allocated for the largest U seen)
  SortScratch sort{};
  int sort_bits_max = 0;
  int sort_bits_delta = 0;

  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaStream_t pstream = nullptr;  // side stream for pp_epoch_prefetch
  cudaEvent_t ev_pref = nullptr, ev_pref_in = nullptr;
  bool pref_pending = false;
  uint64_t pref_seed = 0;
  int64_t pref_chunk = 0;

  // launch tuning (defaults; PPLOAD_TILE_ROWS / PPLOAD_PDL / PPLOAD_GRID_PER_SM override)
  int num_sms = 148;
  int tile_rows = 32;  // 16 vs 32 measured: 32 is ~1.4 % faster at k = 8 (profiles/r1i_exp_l2hint.jsonl)
  bool pdl = true;
  int grid_per_sm = 4;
  int gather_mode = 0;           // 0 auto, 1 ldg (register-staged), 2 tma (bulk copy); PPLOAD_GATHER
  bool tma_ok = false;
  int l2_prefetch = 0;           // load hint experiment (PPLOAD_L2_PREFETCH)
  // CTA cap for the prefetched permutation (PPLOAD_PREFETCH_CTAS; 0 = full grid).
  // Measured on products (profiles/r1j_exp_prefetch.jsonl): full grid 1.002 ms/epoch,
  // 148-296 CTAs 0.972 ms, 64 CTAs 1.11-1.15 ms (the sort then outlasts the epoch).
  int prefetch_ctas = 148;  // r1zz: 148 >= 296 > 444 once k_bucket_rank pipelines its loads
  int max_ctas = 0;  // pp_set_grid_limit: cap on the gather grid (0 = the full persistent grid)
  // previous op on the loader stream (programmatic dependent launch is only used
  // between consecutive launches of the same kind within one epoch)
  enum { kLastNone = 0, kLastGather = 1, kLastLinear = 2 };
  int last_kernel = kLastNone;
  // Byte ranges written by the launches of the current programmatic-dependent-launch chain (hulls):
  // chained launches may run concurrently, so a launch whose outputs overlap them is not chained.
  struct Span {
    uintptr_t lo = 0, hi = 0;
    bool overlaps(const Span& o) const { return lo < hi && o.lo < o.hi && lo < o.hi && o.lo < hi; }
    void join(const Span& o) {
      if (o.lo >= o.hi) return;
      if (lo >= hi) { *this = o; return; }
      lo = std::min(lo, o.lo);
      hi = std::max(hi, o.hi);
    }
  };
  Span chain[3];  // out (or Z), labels, node ids

  ShardView shards[kMaxWorld]{};
  bool linked = false;
  std::vector<void*> ipc_opened;
  // collective (seed, chunk) check of pp_epoch_permute (PP_PEERS_IPC): word[seq & 1] =
  // (seq << 32) | hash, in device memory every peer maps
  uint64_t* d_flags = nullptr;
  const uint64_t* peer_flags[kMaxWorld]{};
  uint32_t coll_seq = 0;
  cudaStream_t cstream = nullptr;  // host <-> flag-word copies (never waits on other streams)
  // all-to-all exchange (PP_PEERS_NCCL, or PP_PEERS_LOOPBACK with PPLOAD_EXCHANGE=a2a)
  bool a2a = false;
  void* nccl = nullptr;              // ncclComm_t
  int64_t* d_nccl_scratch = nullptr;  // int64[2] for the argument check
  uint32_t* d_counts = nullptr;      // [steps][W][W] of the current epoch
  uint32_t* h_counts = nullptr;      // pinned host copy
  int64_t counts_cap = 0;
  uint32_t* d_send_rows = nullptr;
  uint32_t* d_recv_src = nullptr;
  uint8_t* d_sendbuf = nullptr;
  uint8_t* d_recvbuf = nullptr;
  int64_t pdl_launches = 0;
  uint32_t* d_col32 = nullptr;  // int32 column ids for the L2-sliced propagation (pp_propagate_store)
  int64_t col32_cap = 0;
  uint8_t* d_xt = nullptr;      // its window-major copy of the input hop slot
  void* d_wave_sync = nullptr;  // window counter of the wave-synchronous propagation
  int64_t xt_cap = 0;
  int64_t scratch_bytes = 0;  // HBM of order / sort / exchange buffers allocated so far

  // storage tier (hops.where == PP_MEM_FILES): no store; steps are read from the hop files
  FileTier* files = nullptr;
  std::vector<uint32_t> h_order;      // host copy of the current epoch's order
  std::vector<int64_t> h_node_set;    // host copy of the node set (empty: identity)
  // compact store (desc.store_set_only): records are node-set positions, not node ids
  bool compact = false;
  // DMA-staged assembly for host-resident rows under chunk reshuffling (the paper's chunk
  // transfer): runs of consecutive rows are moved by the copy engines
  int dma_mode = 0;              // PPLOAD_SPILL_PATH: 0 auto (chunk >= dma_min_chunk), 1 always, 2 never
  int64_t dma_min_chunk = 64;    // PPLOAD_DMA_MIN_CHUNK
  bool dma_epoch = false;        // the current epoch uses it
  uint32_t* h_order_pin = nullptr;  // pinned host copy of the order (run planning)
  uint8_t* d_stage = nullptr;       // [B] records, batch order
  uint64_t epoch_id = 0;              // bumped by every permute / seek (invalidates staged steps)

  bool permuted = false, poisoned = false;
  bool local = false;         // current epoch from pp_epoch_permute_local
  int64_t steps_global = 0;   // steps of a global-permutation epoch
  uint64_t seed = 0;
  int64_t chunk = 1, cursor = 0;
};

namespace {

pp_status cuda_fail(pp_loader* L, cudaError_t e, const char* what) {
  if (L) L->poisoned = true;
  return fail(PP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define PPL_CUDA(L, call)                                  \
  do {                                                     \
    cudaError_t _e = (call);                               \
    if (_e != cudaSuccess) return cuda_fail((L), _e, #call); \
  } while (0)

void release(pp_loader* L) {
  if (!L) return;
  if (L->stream) cudaStreamSynchronize(L->stream);
  if (L->files) file_tier_close(L->files);
  if (L->h_order_pin) cudaFreeHost(L->h_order_pin);
  cudaFree(L->d_stage);
  for (void* p : L->ipc_opened) cudaIpcCloseMemHandle(p);
  for (const auto& ps : L->peer_spills) {
    cudaHostUnregister(ps.p);
    munmap(ps.p, ps.bytes);
  }
  if (L->nccl) nccl_comm_destroy(L->nccl, L->poisoned);
  cudaFree(L->d_nccl_scratch);
  cudaFree(L->d_counts);
  if (L->h_counts) cudaFreeHost(L->h_counts);
  cudaFree(L->d_send_rows);
  cudaFree(L->d_recv_src);
  cudaFree(L->d_sendbuf);
  cudaFree(L->d_recvbuf);
  cudaFree(L->d_flags);
  cudaFree(L->d_col32);
  cudaFree(L->d_xt);
  cudaFree(L->d_wave_sync);
  if (L->cstream) cudaStreamDestroy(L->cstream);
  if (!L->borrowed) cudaFree(L->d_store);
  cudaFree(L->d_xstore);
  if (L->spill_fd >= 0) {
    cudaHostUnregister(L->h_spill);
    munmap(L->h_spill, L->spill_bytes);
    close(L->spill_fd);
  } else if (L->h_spill) {
    cudaFreeHost(L->h_spill);
  }
  cudaFree(L->d_node_set);
  cudaFree(L->d_labels);
  if (L->pstream) cudaStreamSynchronize(L->pstream);
  cudaFree(L->d_orders[0]);
  cudaFree(L->d_orders[1]);
  cudaFree(L->d_pi);
  cudaFree(L->sort.counts);
  cudaFree(L->sort.cursor);
  cudaFree(L->sort.blocksums);
  cudaFree(L->sort.tmp);
  cudaFree(L->sort.ragged);
  cudaFree(L->sort.hist);
  if (L->ev_in) cudaEventDestroy(L->ev_in);
  if (L->ev_out) cudaEventDestroy(L->ev_out);
  if (L->ev_pref) cudaEventDestroy(L->ev_pref);
  if (L->ev_pref_in) cudaEventDestroy(L->ev_pref_in);
  if (L->pstream) cudaStreamDestroy(L->pstream);
  if (L->own_stream && L->stream) cudaStreamDestroy(L->stream);
  delete L;
}

// Copy rows [row0, row0 + n) of this rank's slice (global rows v = lr*W + r)
// of every hop into dst (record pitch rec_stride), strided 2-D copies.
cudaError_t copy_in(const pp_loader* L, const pp_hop_desc& h, int64_t row0, int64_t n, uint8_t* dst) {
  const int s = elem_bytes(h.dtype);
  const uint8_t* src = static_cast<const uint8_t*>(h.data);
  const size_t spitch = static_cast<size_t>(h.row_stride) * L->W * s;
  const int64_t kMaxRows = 1 << 22;
  for (int32_t k = 0; k < L->H; ++k) {
    for (int64_t a = 0; a < n; a += kMaxRows) {
      const int64_t m = std::min(kMaxRows, n - a);
      const int64_t lr = row0 + a;
      const int64_t v = lr * L->W + L->rank;
      const uint8_t* s0 = src + (static_cast<int64_t>(k) * h.hop_stride + v * h.row_stride) * s;
      uint8_t* d0 = dst + a * L->rec_stride + static_cast<int64_t>(k) * L->F * s;
      cudaError_t e = cudaMemcpy2D(d0, L->rec_stride, s0, spitch, static_cast<size_t>(L->F) * s, m, cudaMemcpyDefault);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

// Compact store (store_set_only): record lr of rank r holds node S[lr*W + r] of the
// node set S.  Device sources are packed by a kernel; host sources row by row on the
// host, into the pinned spill directly or through a pinned staging buffer.
cudaError_t copy_in_compact(const pp_loader* L, const pp_hop_desc& h, const int64_t* S_host, int64_t row0, int64_t n,
                            uint8_t* dst, bool dst_is_host) {
  const int s = elem_bytes(h.dtype);
  if (n <= 0) return cudaSuccess;
  if (h.where == PP_MEM_DEVICE) {
    cudaError_t e = launch_pack_rows(h.data, h.hop_stride, h.row_stride, s, L->H, L->F, L->d_node_set + row0 * L->W, n,
                                     L->W, L->rank, dst_is_host ? L->d_spill + (dst - L->h_spill) : dst,
                                     L->rec_stride, nullptr);
    return e == cudaSuccess ? cudaDeviceSynchronize() : e;
  }
  const uint8_t* src = static_cast<const uint8_t*>(h.data);
  const size_t rb = static_cast<size_t>(L->F) * s;
  auto pack = [&](uint8_t* out, int64_t r0, int64_t m) {
    for (int64_t r = 0; r < m; ++r) {
      const int64_t v = S_host[(row0 + r0 + r) * L->W + L->rank];
      for (int32_t k = 0; k < L->H; ++k)
        memcpy(out + r * L->rec_stride + static_cast<size_t>(k) * rb,
               src + (static_cast<int64_t>(k) * h.hop_stride + v * h.row_stride) * s, rb);
    }
  };
  if (dst_is_host) {
    pack(dst, 0, n);
    return cudaSuccess;
  }
  const int64_t chunk = std::max<int64_t>(1, (int64_t(64) << 20) / L->rec_stride);
  uint8_t* stage = nullptr;
  if (cudaHostAlloc(&stage, static_cast<size_t>(std::min(chunk, n) * L->rec_stride), cudaHostAllocDefault) != cudaSuccess)
    return cudaErrorMemoryAllocation;
  cudaError_t e = cudaSuccess;
  for (int64_t a = 0; a < n && e == cudaSuccess; a += chunk) {
    const int64_t m = std::min(chunk, n - a);
    pack(stage, a, m);
    e = cudaMemcpy(dst + a * L->rec_stride, stage, static_cast<size_t>(m * L->rec_stride), cudaMemcpyHostToDevice);
  }
  cudaFreeHost(stage);
  return e;
}

// The prefetched permutation runs at the lowest stream priority so the block
// scheduler serves the current epoch's gathers first.
int prefetch_priority() {
  int least = 0, greatest = 0;
  if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return 0;
  return least;
}

// Spill of an IPC-sharded loader: an anonymous shared-memory file (memfd), mapped MAP_SHARED here
// and registered with CUDA (pinned, mapped); the peers open it through /proc/<pid>/fd/<fd>, map and
// register it too (pp_import_peer_stores), so any rank reads any owner's spilled rows zero-copy
// (host placement of data beyond GPU memory).
bool alloc_shared_spill(pp_loader* L, size_t bytes, std::string* err) {
  const int fd = memfd_create("ppload-spill", MFD_CLOEXEC);
  if (fd < 0) {
    *err = std::string("memfd_create: ") + strerror(errno);
    return false;
  }
  void* p = MAP_FAILED;
  if (ftruncate(fd, static_cast<off_t>(bytes)) == 0)
    p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (p == MAP_FAILED) {
    *err = std::string("ftruncate / mmap of ") + std::to_string(bytes) + " bytes: " + strerror(errno);
    close(fd);
    return false;
  }
  const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    *err = std::string("cudaHostRegister: ") + cudaGetErrorString(e);
    munmap(p, bytes);
    close(fd);
    return false;
  }
  L->h_spill = static_cast<uint8_t*>(p);
  L->spill_fd = fd;
  L->spill_bytes = bytes;
  return true;
}

bool fast_div_ok(int64_t d) { return d > 0 && static_cast<uint64_t>(128) * d * d < (uint64_t(1) << 40); }

pp_status validate(const pp_loader_desc* d) {
  if (!d) return fail(PP_ERR_INVALID, "desc is NULL");
  const pp_hop_desc& h = d->hops;
  if (h.num_nodes < 1 || h.num_nodes >= (int64_t(1) << 32))
    return fail(PP_ERR_INVALID, "num_nodes must be in [1, 2^32), got %lld", (long long)h.num_nodes);
  if (h.num_hops < 1 || h.feat_dim < 1) return fail(PP_ERR_INVALID, "num_hops and feat_dim must be >= 1");
  if (static_cast<int64_t>(h.num_hops) * h.feat_dim >= (int64_t(1) << 24))
    return fail(PP_ERR_INVALID, "H*F too large");
  if (!valid_dtype(h.dtype) || !valid_dtype(d->out_dtype)) return fail(PP_ERR_INVALID, "unknown dtype");
  if (h.where != PP_MEM_HOST && h.where != PP_MEM_DEVICE && h.where != PP_MEM_FILES)
    return fail(PP_ERR_INVALID, "unknown memory kind");
  const bool files = h.where == PP_MEM_FILES;
  if (files && !h.data) return fail(PP_ERR_INVALID, "PP_MEM_FILES needs the array of H hop file paths");
  if (files && d->peers != PP_PEERS_NONE) return fail(PP_ERR_INVALID, "file loaders take peers = PP_PEERS_NONE");
  if (d->store_set_only && (!d->node_set || files))
    return fail(PP_ERR_INVALID, "store_set_only needs a node_set and an in-memory source");
  const bool cast = h.dtype == PP_F32 && (d->out_dtype == PP_BF16 || d->out_dtype == PP_F16);
  if (!cast && h.dtype != d->out_dtype)
    return fail(PP_ERR_INVALID, "unsupported dtype pair (store %d -> out %d)", h.dtype, d->out_dtype);
  if (h.data && !files) {
    if (h.row_stride < h.feat_dim || h.hop_stride < 0)
      return fail(PP_ERR_INVALID, "row_stride must be >= feat_dim and hop_stride >= 0");
  }
  if (d->batch_size < 1) return fail(PP_ERR_INVALID, "batch_size must be >= 1");
  if (d->world_size < 1 || d->world_size > kMaxWorld)
    return fail(PP_ERR_INVALID, "world_size must be in [1, %d]", kMaxWorld);
  if (d->rank < 0 || d->rank >= d->world_size) return fail(PP_ERR_INVALID, "rank out of range");
  if (d->peers != PP_PEERS_NONE && d->peers != PP_PEERS_IPC && d->peers != PP_PEERS_LOOPBACK &&
      d->peers != PP_PEERS_NCCL)
    return fail(PP_ERR_INVALID, "unknown peers mode");
  if (!files && d->world_size == 1 && d->peers != PP_PEERS_NONE && d->peers != PP_PEERS_NCCL)
    return fail(PP_ERR_INVALID, "world_size == 1 takes peers = PP_PEERS_NONE (or PP_PEERS_NCCL)");
  if (!files && d->world_size > 1 && d->peers == PP_PEERS_NONE)
    return fail(PP_ERR_INVALID, "world_size > 1 needs peers = IPC, LOOPBACK or NCCL");
  if (d->peers == PP_PEERS_NCCL && !d->nccl_unique_id)
    return fail(PP_ERR_INVALID, "PP_PEERS_NCCL needs nccl_unique_id (pp_nccl_unique_id, broadcast by the caller)");
  if (d->node_set) {
    if (d->num_set < 1 || d->num_set >= (int64_t(1) << 32)) return fail(PP_ERR_INVALID, "num_set out of range");
    for (int64_t i = 0; i < d->num_set; ++i)
      if (d->node_set[i] < 0 || d->node_set[i] >= h.num_nodes)
        return fail(PP_ERR_INVALID, "node_set[%lld] = %lld out of range", (long long)i, (long long)d->node_set[i]);
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || d->device < 0 || d->device >= ndev)
    return fail(PP_ERR_INVALID, "device %d not available", d->device);
  return PP_OK;
}

// Rewrite the exchange copy from the HBM rows of the store (after any store write).
cudaError_t refresh_exchange_copy(pp_loader* L) {
  if (!L->d_xstore) return cudaSuccess;
  cudaError_t e = launch_cast_records(L->d_store, L->n_hbm, L->rec_stride, L->HF, L->out_dtype, L->d_xstore,
                                      L->xrec_stride, L->stream ? L->stream : 0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L->stream ? L->stream : 0);
  return e;
}

pp_status ensure_sort_scratch(pp_loader* L, uint32_t U, int bits) {
  const size_t hist_need = L->sort.two_level ? two_level_hist_entries(U) : 0;
  const bool grow_tmp = static_cast<int64_t>(U) > L->tmp_cap;
  if (grow_tmp || bits > L->sort_bits_max || !L->sort.counts || hist_need > L->sort.hist_cap) {
    // work on either stream may still use the scratch being replaced
    if (L->stream) cudaStreamSynchronize(L->stream);
    if (L->pstream) cudaStreamSynchronize(L->pstream);
  }
  if (grow_tmp) {  // unit ids grouped by bucket: U entries (U = N for SGD-RR, ceil(N / c) with chunks)
    cudaFree(L->sort.tmp);
    L->sort.tmp = nullptr;
    L->scratch_bytes -= L->tmp_cap * 4;
    L->tmp_cap = 0;
    if (cudaMalloc(&L->sort.tmp, static_cast<size_t>(U) * 4) != cudaSuccess)
      return fail(PP_ERR_OOM, "sort scratch allocation failed (%u units)", U);
    L->tmp_cap = U;
    L->scratch_bytes += L->tmp_cap * 4;
  }
  if (bits > L->sort_bits_max || !L->sort.counts || hist_need > L->sort.hist_cap) {
    const int nbits = std::max(bits, L->sort_bits_max);
    const size_t hist_cap = std::max(hist_need, L->sort.hist_cap);
    cudaFree(L->sort.counts);
    cudaFree(L->sort.cursor);
    cudaFree(L->sort.blocksums);
    cudaFree(L->sort.hist);
    L->sort.counts = L->sort.cursor = L->sort.blocksums = L->sort.hist = nullptr;
    L->sort.hist_cap = 0;
    const size_t nb = size_t(1) << nbits;
    const size_t nblk = (std::max(nb + 1, hist_cap) + kScanTile - 1) / kScanTile;  // scans of either path
    if (cudaMalloc(&L->sort.counts, (nb + 1) * 4) != cudaSuccess || cudaMalloc(&L->sort.cursor, nb * 4) != cudaSuccess ||
        cudaMalloc(&L->sort.blocksums, nblk * 4) != cudaSuccess ||
        (hist_cap > 0 && cudaMalloc(&L->sort.hist, hist_cap * 4) != cudaSuccess))
      return fail(PP_ERR_OOM, "sort scratch allocation failed (2^%d buckets)", nbits);
    L->sort_bits_max = nbits;
    L->sort.hist_cap = hist_cap;
  }
  return PP_OK;
}

}  // namespace

extern "C" {

int32_t pp_abi_version(void) { return PP_ABI_VERSION; }

const char* pp_last_error(void) { return g_last_error.c_str(); }

pp_status pp_propagate(int64_t n, int32_t F, const int64_t* row_ptr, const int64_t* col_idx, const float* X,
                       int32_t K, float* hops, void* stream) {
  NvtxRange nvtx_range("pp_propagate");
  if (n < 1 || F < 1 || F > 256 || K < 0) return fail(PP_ERR_INVALID, "need n >= 1, 1 <= F <= 256, K >= 0");
  if (!row_ptr || !col_idx || !X || !hops) return fail(PP_ERR_INVALID, "NULL pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t nnz = 0;
  cudaError_t e = cudaMemcpyAsync(&nnz, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(PP_ERR_CUDA, "reading row_ptr[n]: %s", cudaGetErrorString(e));
  if (nnz < n) return fail(PP_ERR_INVALID, "row_ptr[n] = %lld < n: every row needs its diagonal entry", (long long)nnz);
  const size_t plane = static_cast<size_t>(n) * F * sizeof(float);
  e = cudaMemcpyAsync(hops, X, plane, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return fail(PP_ERR_CUDA, "hop 0 copy: %s", cudaGetErrorString(e));
  if (K == 0) return PP_OK;
  double* val = nullptr;
  // stream-ordered scratch from a library-private pool (per device) that keeps its memory
  // between calls; the device's default pool and its release threshold are left alone
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail(PP_ERR_CUDA, "cudaGetDevice failed");
  {
    static std::mutex pools_mu;
    std::lock_guard<std::mutex> lk(pools_mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      cudaMemPool_t pool = nullptr;
      if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return fail(PP_ERR_CUDA, "cudaMemPoolCreate failed");
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[dev] = pool;
    }
  }
  if (spmm_use_sliced(n, F) && n < (int64_t(1) << 32) && reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(hops) % 16 == 0) {
    // L2-sliced passes (propagate.cu): int32 columns + degrees, weights recomputed per nonzero
    uint32_t* col32 = nullptr;
    int32_t* deg = nullptr;
    uint8_t* xt = nullptr;
    if (cudaMallocFromPoolAsync(reinterpret_cast<void**>(&col32), static_cast<size_t>(nnz) * 4, pools[dev], st) !=
            cudaSuccess ||
        cudaMallocFromPoolAsync(reinterpret_cast<void**>(&deg), static_cast<size_t>(n) * 4, pools[dev], st) !=
            cudaSuccess ||
        cudaMallocFromPoolAsync(reinterpret_cast<void**>(&xt),
                                static_cast<size_t>(spmm_sliced_scratch_bytes(n, F, nnz)), pools[dev], st) != cudaSuccess)
      return fail(PP_ERR_OOM, "propagation scratch (%lld nonzeros)", (long long)nnz);
    e = launch_col_to_u32(col_idx, nnz, col32, st);
    if (e == cudaSuccess) e = launch_row_lengths(row_ptr, n, deg, st);
    for (int32_t k = 1; k <= K && e == cudaSuccess; ++k)
      e = launch_spmm_sliced_rows(n, F, row_ptr, col32, deg, hops + (k - 1) * (plane / sizeof(float)),
                                  hops + k * (plane / sizeof(float)), xt, nnz, k == 1, st);
    cudaFreeAsync(col32, st);
    cudaFreeAsync(deg, st);
    cudaFreeAsync(xt, st);
    if (e != cudaSuccess) return fail(PP_ERR_CUDA, "propagation: %s", cudaGetErrorString(e));
    return PP_OK;
  }
  if (cudaMallocFromPoolAsync(reinterpret_cast<void**>(&val), static_cast<size_t>(nnz) * sizeof(double), pools[dev],
                              st) != cudaSuccess)
    return fail(PP_ERR_OOM, "operator values (%lld nonzeros)", (long long)nnz);
  // wave-synchronous kernel (propagate.cu) for large graphs: the same arithmetic, a fraction of
  // the DRAM traffic; it needs a 4-byte window counter
  unsigned* wave_sync = nullptr;
  const bool eligible = spmm_wave_eligible(F, X, int64_t(F) * 4, hops, int64_t(F) * 4);
  const bool cp = eligible && spmm_use_cp();
  const bool wave = !cp && eligible && spmm_use_wave(n, F) &&
                    cudaMallocFromPoolAsync(reinterpret_cast<void**>(&wave_sync), 256, pools[dev], st) == cudaSuccess;
  e = launch_operator_values(n, row_ptr, col_idx, val, st);
  for (int32_t k = 1; k <= K && e == cudaSuccess; ++k) {
    const float* x = hops + (k - 1) * (plane / sizeof(float));
    float* y = hops + k * (plane / sizeof(float));
    if (wave || cp) {
      WaveArgs a;
      a.n = a.ncols = n;
      a.F = F;
      a.row_ptr = row_ptr;
      a.col = col_idx;
      a.val = val;
      a.src = reinterpret_cast<const uint8_t*>(x);
      a.dst = reinterpret_cast<uint8_t*>(y);
      a.src_stride = a.dst_stride = int64_t(F) * 4;
      e = cp ? launch_spmm_rows_cp(a, st) : launch_spmm_wave(a, wave_sync, st);
    } else {
      e = launch_spmm(n, F, row_ptr, col_idx, val, x, y, st);
    }
  }
  if (wave_sync) cudaFreeAsync(wave_sync, st);
  cudaFreeAsync(val, st);
  if (e != cudaSuccess) return fail(PP_ERR_CUDA, "propagation: %s", cudaGetErrorString(e));
  return PP_OK;
}

int64_t pp_footprint_bytes(int64_t num_nodes, int32_t feat_dim, int32_t elem_bytes_, int32_t num_ops,
                           int32_t num_hops_R) {
  if (num_nodes < 0 || feat_dim < 0 || elem_bytes_ < 0 || num_ops < 0 || num_hops_R < 0) return -1;
  return num_nodes * feat_dim * elem_bytes_ * static_cast<int64_t>(num_ops) * (num_hops_R + 1);
}

pp_status pp_loader_create(const pp_loader_desc* desc, pp_loader** out) {
  NvtxRange nvtx_range("pp_loader_create");
  if (!out) return fail(PP_ERR_INVALID, "out is NULL");
  *out = nullptr;
  pp_status st = validate(desc);
  if (st != PP_OK) return st;
  DevGuard g(desc->device);
  if (!g.ok) return fail(PP_ERR_CUDA, "cudaSetDevice(%d) failed", desc->device);

  pp_loader* L = new (std::nothrow) pp_loader();
  if (!L) return fail(PP_ERR_OOM, "host allocation failed");
  L->desc = *desc;
  L->desc.node_set = nullptr;
  L->desc.labels = nullptr;
  L->desc.hops.data = nullptr;
  L->dev = desc->device;
  L->W = desc->world_size;
  L->rank = desc->rank;
  L->H = desc->hops.num_hops;
  L->F = desc->hops.feat_dim;
  L->HF = L->H * L->F;
  L->in_dtype = desc->hops.dtype;
  L->out_dtype = desc->out_dtype;
  L->N_total = desc->hops.num_nodes;
  L->N = desc->node_set ? desc->num_set : L->N_total;
  L->B = desc->batch_size;
  const int64_t per_step = L->B * L->W;
  L->steps = desc->drop_last ? L->N / per_step : (L->N + per_step - 1) / per_step;
  L->steps_global = L->steps;
  L->compact = desc->store_set_only != 0;
  // row space of the store: node ids 0..N_total-1, or node-set positions 0..N-1 (compact)
  const int64_t R = L->compact ? L->N : L->N_total;
  L->local_rows = (R - L->rank + L->W - 1) / L->W;
  L->rec_in = static_cast<int64_t>(L->HF) * elem_bytes(L->in_dtype);
  L->rec_stride = (L->rec_in + 15) / 16 * 16;
  // experiment knob: record pitch rounded up to a power of two >= 16 bytes (e.g. 128: whole L2 lines)
  if (const char* e = getenv("PPLOAD_REC_ALIGN")) {
    const int64_t al = atoll(e);
    if (al >= 16 && (al & (al - 1)) == 0) L->rec_stride = (L->rec_in + al - 1) / al * al;
  }
  L->rec_out = static_cast<int64_t>(L->HF) * elem_bytes(L->out_dtype);
  L->vector_path = gather_vector_ok(L->HF, L->in_dtype, L->out_dtype, L->rec_stride);
  // the gather kernels divide slot indices by a 2^40 reciprocal: tile (<= 128 rows) x slots per row
  // x divisor must stay below 2^40 (vector path: vpr = rec_out / 16 slots; scalar: H*F elements)
  if (!fast_div_ok(L->vector_path ? L->rec_out / 16 : L->HF)) {
    release(L);
    return fail(PP_ERR_INVALID, "record of H*F = %d elements too large for the %s gather path", L->HF,
                L->vector_path ? "vector" : "scalar");
  }

  auto bail = [&](pp_status s) {
    release(L);
    return s;
  };
  cudaError_t e_x = cudaSuccess;
  const bool files = desc->hops.where == PP_MEM_FILES;
  if (files) {
    std::string err;
    L->files = file_tier_open(static_cast<const char* const*>(desc->hops.data), L->H, L->N_total, L->F,
                              elem_bytes(L->in_dtype), L->B, L->dev, &err);
    if (!L->files) return bail(fail(PP_ERR_INVALID, "storage tier: %s", err.c_str()));
    L->h_order.resize(L->N);
    if (desc->node_set) L->h_node_set.assign(desc->node_set, desc->node_set + L->N);
  }

  if (desc->node_set) {  // before the store upload (the compact store is packed through it)
    if (cudaMalloc(&L->d_node_set, L->N * 8) != cudaSuccess) return bail(fail(PP_ERR_OOM, "node_set allocation"));
    if (cudaMemcpy(L->d_node_set, desc->node_set, L->N * 8, cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(PP_ERR_CUDA, "node_set upload"));
  }
  // ---- placement: HBM budget, remainder spills to pinned mapped host memory.  The automatic
  // budget leaves 2 GiB plus what this loader allocates next: labels, the epoch order and the sort
  // scratch for U = N units (a prefetched second order is allocated at the first pp_epoch_prefetch).
  const int64_t scratch = L->N * 4 * 2 + (int64_t(1) << 26) + (desc->labels ? L->N_total * 4 : 0);
  int64_t budget = desc->hbm_budget_bytes;
  if (budget == 0) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return bail(fail(PP_ERR_CUDA, "cudaMemGetInfo failed"));
    budget = static_cast<int64_t>(fr) - (int64_t(2) << 30) - scratch;
    if (budget < 0) budget = 0;
  }
  L->n_hbm = files ? 0 : budget < 0 ? 0 : std::min<int64_t>(L->local_rows, budget / L->rec_stride);
  if (desc->borrow_device_data && desc->hbm_budget_bytes == 0) L->n_hbm = L->local_rows;  // nothing to allocate
  if (files) L->local_rows = 0;
  L->n_spill = L->local_rows - L->n_hbm;

  if (desc->borrow_device_data) {
    // the caller's node-major device tensor IS the store (no copy; it must outlive the loader)
    if (desc->hops.where != PP_MEM_DEVICE || !desc->hops.data || L->W != 1 || L->compact || files ||
        desc->hops.hop_stride != L->F || desc->hops.row_stride != L->HF || L->rec_stride != L->rec_in ||
        reinterpret_cast<uintptr_t>(desc->hops.data) % 16 != 0 || L->n_hbm != L->local_rows)
      return bail(fail(PP_ERR_INVALID,
                       "borrow_device_data needs a 16-B aligned node-major device tensor [N][H][F] with H*F*elem a "
                       "16-B multiple, W == 1, no node-set compaction, and no HBM budget below the store"));
    L->d_store = static_cast<uint8_t*>(const_cast<void*>(desc->hops.data));
    L->borrowed = true;
  }
  if (!L->borrowed && L->n_hbm > 0 && cudaMalloc(&L->d_store, static_cast<size_t>(L->n_hbm * L->rec_stride)) != cudaSuccess)
    return bail(fail(PP_ERR_OOM, "cudaMalloc of the %lld-byte HBM store failed", (long long)(L->n_hbm * L->rec_stride)));
  if (L->n_spill > 0) {
    const size_t bytes = static_cast<size_t>(L->n_spill * L->rec_stride);
    if (L->W > 1 && desc->peers == PP_PEERS_IPC) {
      std::string err;
      if (!alloc_shared_spill(L, bytes, &err)) return bail(fail(PP_ERR_OOM, "shared spill: %s", err.c_str()));
    } else {
      if (cudaHostAlloc(&L->h_spill, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
        return bail(fail(PP_ERR_OOM, "pinned spill allocation of %lld bytes failed", (long long)bytes));
      L->spill_bytes = bytes;
    }
    if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&L->d_spill), L->h_spill, 0) != cudaSuccess)
      return bail(fail(PP_ERR_CUDA, "cudaHostGetDevicePointer failed"));
  }
  if (desc->hops.data && !files && L->compact) {
    cudaError_t e = copy_in_compact(L, desc->hops, desc->node_set, 0, L->n_hbm, L->d_store, false);
    if (e == cudaSuccess && L->n_spill > 0)
      e = copy_in_compact(L, desc->hops, desc->node_set, L->n_hbm, L->n_spill, L->h_spill, true);
    if (e != cudaSuccess) return bail(fail(PP_ERR_CUDA, "store upload failed: %s", cudaGetErrorString(e)));
  } else if (desc->hops.data && !files && !L->borrowed) {
    cudaError_t e = copy_in(L, desc->hops, 0, L->n_hbm, L->d_store);
    if (e == cudaSuccess && L->n_spill > 0) e = copy_in(L, desc->hops, L->n_hbm, L->n_spill, L->h_spill);
    if (e != cudaSuccess) return bail(fail(PP_ERR_CUDA, "store upload failed: %s", cudaGetErrorString(e)));
  }
  // The uploads above run on the legacy stream (cudaMemcpy2D may return before a device-source or
  // staged copy lands); the exchange copy below reads d_store on the non-blocking loader stream.
  if (desc->hops.data && !files && !L->borrowed && cudaDeviceSynchronize() != cudaSuccess)
    return bail(fail(PP_ERR_CUDA, "store upload sync failed"));
  // ---- labels, order, sort scratch
  if (desc->labels) {
    L->has_labels = true;
    if (cudaMalloc(&L->d_labels, L->N_total * 4) != cudaSuccess) return bail(fail(PP_ERR_OOM, "labels allocation"));
    if (cudaMemcpy(L->d_labels, desc->labels, L->N_total * 4, cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(PP_ERR_CUDA, "labels upload"));
  }
  if (cudaMalloc(&L->d_orders[0], L->N * 4) != cudaSuccess || cudaMalloc(&L->sort.ragged, 4) != cudaSuccess)
    return bail(fail(PP_ERR_OOM, "order allocation"));
  L->scratch_bytes += L->N * 4;
  L->d_order = L->d_orders[0];
  if (cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(PP_ERR_CUDA, "stream creation"));
  L->own_stream = true;
  if (cudaEventCreateWithFlags(&L->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_out, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_pref, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_pref_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithPriority(&L->pstream, cudaStreamNonBlocking, prefetch_priority()) != cudaSuccess)
    return bail(fail(PP_ERR_CUDA, "event creation"));
  cudaDeviceGetAttribute(&L->num_sms, cudaDevAttrMultiProcessorCount, L->dev);
  // rows per gather tile: 32 for records >= 1 KB (measured best, r1i); small records get up to 128
  // rows so a tile still carries ~32 KB of loads per order round trip (r1z sweep)
  while (L->tile_rows < 128 && L->tile_rows * L->rec_in < 32768) L->tile_rows *= 2;
  if (const char* e = getenv("PPLOAD_TILE_ROWS")) L->tile_rows = std::max(1, std::min(128, atoi(e)));
  if (const char* e = getenv("PPLOAD_PDL")) L->pdl = atoi(e) != 0;
  if (const char* e = getenv("PPLOAD_GRID_PER_SM")) L->grid_per_sm = std::max(1, atoi(e));
  if (const char* e = getenv("PPLOAD_DEBUG_TIE_BITS")) {  // test knob: keep only the top n sub-key bits
    const int n = std::max(1, std::min(32, atoi(e)));
    L->sort.k32_mask = n == 32 ? 0xffffffffu : ~((1u << (32 - n)) - 1u);
  }
  if (const char* e = getenv("PPLOAD_DEBUG_L2CAP")) L->sort.l2_cap = static_cast<uint32_t>(std::max(1, atoi(e)));
  if (const char* e = getenv("PPLOAD_PERMUTE")) L->sort.two_level = !strcmp(e, "two_level");
  if (const char* e = getenv("PPLOAD_L2_PREFETCH")) L->l2_prefetch = std::max(0, std::min(2, atoi(e)));
  if (const char* e = getenv("PPLOAD_PREFETCH_CTAS")) L->prefetch_ctas = std::max(0, atoi(e));
  if (const char* e = getenv("PPLOAD_GATHER")) L->gather_mode = !strcmp(e, "ldg") ? 1 : !strcmp(e, "tma") ? 2 : 0;
  if (const char* e = getenv("PPLOAD_SPILL_PATH")) L->dma_mode = !strcmp(e, "dma") ? 1 : !strcmp(e, "kernel") ? 2 : 0;
  if (const char* e = getenv("PPLOAD_DMA_MIN_CHUNK")) L->dma_min_chunk = std::max<long long>(1, atoll(e));
  if (L->n_spill > 0 && desc->node_set && L->h_node_set.empty())  // run planning of the DMA path
    L->h_node_set.assign(desc->node_set, desc->node_set + L->N);
  L->tma_ok = L->vector_path && gather_tma_ok(L->HF, L->in_dtype);
  L->shards[L->rank] = ShardView{L->d_store, L->d_spill, L->n_hbm};
  L->linked = (L->W == 1) || files;
  // ---- all-to-all exchange (NCCL baseline; loopback emulation with PPLOAD_EXCHANGE=a2a)
  const char* xenv = getenv("PPLOAD_EXCHANGE");
  L->a2a = !files && (desc->peers == PP_PEERS_NCCL ||
                      (desc->peers == PP_PEERS_LOOPBACK && xenv && !strcmp(xenv, "a2a")));
  // ---- exchange copy for the peers (see pp_loader.h): only if it fits after everything else
  if (L->W > 1 && !L->a2a && L->in_dtype == PP_F32 && L->out_dtype != PP_F32 && L->vector_path) {
    L->xrec_stride = (L->rec_out + 15) / 16 * 16;
    const char* env = getenv("PPLOAD_EXCHANGE_CAST");
    size_t fr = 0, tot = 0;
    const size_t xbytes = static_cast<size_t>(L->n_hbm) * L->xrec_stride;
    if (L->n_hbm > 0 && !(env && !strcmp(env, "0")) && cudaMemGetInfo(&fr, &tot) == cudaSuccess &&
        fr > xbytes + (size_t(1) << 30)) {
      if (cudaMalloc(&L->d_xstore, xbytes) != cudaSuccess) return bail(fail(PP_ERR_OOM, "exchange copy allocation"));
      if (desc->hops.data && (e_x = refresh_exchange_copy(L)) != cudaSuccess)
        return bail(fail(PP_ERR_CUDA, "exchange copy: %s", cudaGetErrorString(e_x)));
    }
  }
  // ---- collective argument check: flag words the peers map (PP_PEERS_IPC)
  if (L->W > 1 && desc->peers == PP_PEERS_IPC) {
    if (cudaMalloc(&L->d_flags, 64) != cudaSuccess || cudaMemset(L->d_flags, 0, 64) != cudaSuccess ||
        cudaStreamCreateWithFlags(&L->cstream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(PP_ERR_CUDA, "collective flag words"));
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(PP_ERR_CUDA, "create sync"));
  if (desc->peers == PP_PEERS_NCCL && !files) {  // collective: every rank's create joins here
    if (cudaMalloc(&L->d_nccl_scratch, 16) != cudaSuccess) return bail(fail(PP_ERR_OOM, "NCCL scratch"));
    std::string err;
    L->nccl = nccl_comm_create(desc->nccl_unique_id, L->W, L->rank, &err);
    if (!L->nccl) return bail(fail(PP_ERR_NCCL, "%s", err.c_str()));
    L->linked = true;
  }
  L->desc.nccl_unique_id = nullptr;
  *out = L;
  return PP_OK;
}

pp_status pp_loader_destroy(pp_loader* L) {
  if (!L) return PP_OK;
  DevGuard g(L->dev);
  release(L);
  return PP_OK;
}

pp_status pp_propagate_store(pp_loader* L, int32_t k, const int64_t* row_ptr, const int64_t* col_idx,
                             const int32_t* deg, void* stream) {
  NvtxRange nvtx_range("pp_propagate_store");
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (L->poisoned) return fail(PP_ERR_CUDA, "loader is poisoned by an earlier CUDA error");
  if (!row_ptr || !col_idx || !deg) return fail(PP_ERR_INVALID, "NULL CSR / degree pointer");
  if (L->in_dtype != PP_F32 || L->files || L->compact)
    return fail(PP_ERR_INVALID, "pp_propagate_store needs an fp32 store of every node (not compact)");
  if (k < 1 || k >= L->H) return fail(PP_ERR_INVALID, "hop slot k = %d must be in [1, H-1 = %d]", k, L->H - 1);
  if (L->F > 256) return fail(PP_ERR_INVALID, "F = %d > 256", L->F);
  if (!L->linked) return fail(PP_ERR_STATE, "sharded loader not linked to its peers yet");
  if (L->W > 1 && L->desc.peers == PP_PEERS_NCCL)
    return fail(PP_ERR_INVALID, "pp_propagate_store reads the peers' stores: needs PP_PEERS_IPC or LOOPBACK");
  DevGuard g(L->dev);
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  if (user != L->stream) {  // order after this loader's gathers (they read the store) ...
    PPL_CUDA(L, cudaEventRecord(L->ev_in, L->stream));
    PPL_CUDA(L, cudaStreamWaitEvent(user, L->ev_in, 0));
  }
  StorePropArgs a{};
  a.local_rows = L->local_rows;
  a.F = L->F;
  a.k = k;
  a.W = L->W;
  a.rank = L->rank;
  a.row_ptr = row_ptr;
  a.col = col_idx;
  a.deg = deg;
  for (int i = 0; i < kMaxWorld; ++i) a.shards[i] = L->shards[i];
  a.rec_stride = L->rec_stride;
  a.xstore = L->d_xstore;
  a.xrec_stride = L->xrec_stride;
  a.x_dtype = L->out_dtype == PP_F16 ? 2 : 1;
  bool sliced = false;
  int64_t nnz_sliced = 0;
  if (L->W == 1 && spmm_use_sliced(L->N_total, L->F) && L->F % 4 == 0 && L->rec_stride % 16 == 0) {
    // the L2-sliced kernel: int32 column ids (converted per call; the CSR may change) and a
    // window-major copy of the input slot, both loader-owned scratch kept between calls
    int64_t nnz = 0;
    PPL_CUDA(L, cudaMemcpyAsync(&nnz, row_ptr + L->local_rows, 8, cudaMemcpyDeviceToHost, user));
    PPL_CUDA(L, cudaStreamSynchronize(user));
    const int64_t xt_bytes = spmm_sliced_scratch_bytes(L->local_rows, L->F, nnz);
    if (nnz > L->col32_cap || xt_bytes > L->xt_cap) {
      cudaFree(L->d_col32);
      cudaFree(L->d_xt);
      L->d_col32 = nullptr;
      L->d_xt = nullptr;
      L->scratch_bytes -= L->col32_cap * 4 + L->xt_cap;
      L->col32_cap = L->xt_cap = 0;
      if (cudaMalloc(&L->d_col32, static_cast<size_t>(nnz) * 4) == cudaSuccess &&
          cudaMalloc(&L->d_xt, static_cast<size_t>(xt_bytes)) == cudaSuccess) {
        L->col32_cap = nnz;
        L->xt_cap = xt_bytes;
        L->scratch_bytes += nnz * 4 + xt_bytes;
      } else {  // no room: the row kernels read the int64 ids and the records directly
        cudaFree(L->d_col32);
        L->d_col32 = nullptr;
        cudaGetLastError();
      }
    }
    if (L->d_col32 && L->d_xt) {
      PPL_CUDA(L, launch_col_to_u32(col_idx, nnz, L->d_col32, user));
      a.col32 = L->d_col32;
      sliced = true;
      nnz_sliced = nnz;
    }
  }
  const ShardView& me = L->shards[L->rank];
  const bool cp = spmm_use_cp();
  if (!sliced && L->W == 1 && me.n_hbm == L->local_rows && (cp || spmm_use_wave(L->local_rows, L->F)) &&
      spmm_wave_eligible(L->F, me.hbm, L->rec_stride, me.hbm, L->rec_stride)) {
    // wave-synchronous or cp.async-staged row kernel (propagate.cu): slot k of every record from slot k - 1
    if (!cp && !L->d_wave_sync) {
      if (cudaMalloc(&L->d_wave_sync, 256) != cudaSuccess) {
        cudaGetLastError();
        return fail(PP_ERR_OOM, "propagation counter (256 B)");
      }
      L->scratch_bytes += 256;
    }
    WaveArgs w;
    w.n = w.ncols = L->local_rows;
    w.F = L->F;
    w.row_ptr = row_ptr;
    w.col = col_idx;
    w.deg = deg;
    w.src = me.hbm + static_cast<int64_t>(k - 1) * L->F * 4;
    w.dst = const_cast<uint8_t*>(me.hbm) + static_cast<int64_t>(k) * L->F * 4;
    w.src_stride = w.dst_stride = L->rec_stride;
    if (L->d_xstore) {
      w.xdst = L->d_xstore + static_cast<int64_t>(k) * L->F * 2;
      w.x_stride = L->xrec_stride;
      w.x_dtype = a.x_dtype;
    }
    PPL_CUDA(L, cp ? launch_spmm_rows_cp(w, user) : launch_spmm_wave(w, static_cast<unsigned*>(L->d_wave_sync), user));
  } else {
    PPL_CUDA(L, sliced ? launch_spmm_store_sliced(a, L->d_xt, nnz_sliced, user) : launch_spmm_store(a, user));
  }
  if (user != L->stream) {  // ... and later loader work after this hop
    PPL_CUDA(L, cudaEventRecord(L->ev_out, user));
    PPL_CUDA(L, cudaStreamWaitEvent(L->stream, L->ev_out, 0));
  }
  L->last_kernel = pp_loader::kLastNone;
  return PP_OK;
}

pp_status pp_set_stream(pp_loader* L, void* stream) {
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (L->poisoned) return fail(PP_ERR_CUDA, "loader is poisoned by an earlier CUDA error");
  DevGuard g(L->dev);
  PPL_CUDA(L, cudaStreamSynchronize(L->stream));
  if (L->own_stream) cudaStreamDestroy(L->stream);
  L->stream = static_cast<cudaStream_t>(stream);
  L->own_stream = false;
  L->last_kernel = pp_loader::kLastNone;
  return PP_OK;
}

pp_status pp_set_grid_limit(pp_loader* L, int32_t max_ctas) {
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (max_ctas < 0) return fail(PP_ERR_INVALID, "max_ctas must be >= 0");
  L->max_ctas = max_ctas;
  return PP_OK;
}

pp_status pp_debug_set_sort_bits_delta(pp_loader* L, int32_t delta) {
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  L->sort_bits_delta = delta;
  return PP_OK;
}

// order[0..n) = the epoch order of n positions for (seed, chunk) (oracle O5-O7).
static pp_status enqueue_order(pp_loader* L, uint64_t seed, int64_t chunk, uint32_t* order, cudaStream_t st,
                               int64_t n) {
  const uint32_t U = static_cast<uint32_t>((n + chunk - 1) / chunk);
  const int bits = sort_bucket_bits(U, L->sort_bits_delta);
  pp_status ps = ensure_sort_scratch(L, U, bits);
  if (ps != PP_OK) return ps;
  if (chunk == 1) {
    PPL_CUDA(L, launch_unit_permutation(seed, U, bits, L->sort_bits_delta == 0, L->sort, order, nullptr, st));
  } else {
    if (L->pi_cap < U) {
      cudaStreamSynchronize(L->stream);  // either stream may still read the old buffer
      cudaStreamSynchronize(L->pstream);
      cudaFree(L->d_pi);
      L->d_pi = nullptr;
      L->scratch_bytes -= L->pi_cap * 4;
      L->pi_cap = 0;
      if (cudaMalloc(&L->d_pi, static_cast<size_t>(U) * 4) != cudaSuccess) return fail(PP_ERR_OOM, "pi allocation");
      L->pi_cap = U;
      L->scratch_bytes += L->pi_cap * 4;
    }
    PPL_CUDA(L, launch_unit_permutation(seed, U, bits, L->sort_bits_delta == 0, L->sort, L->d_pi, L->sort.ragged, st));
    PPL_CUDA(L, launch_chunk_expand(L->d_pi, U, static_cast<uint64_t>(n), static_cast<uint64_t>(chunk),
                                    L->sort.ragged, order, st));
  }
  return PP_OK;
}

// SURVEY.md §8(f)-4, the paper's "locality-aware" placement taken
// literally: each rank shuffles only the rows it owns, so every batch is read
// from local HBM and no exchange is needed at any W.  Local position lr maps
// to global node lr * W + rank.  Not collective; ranks may use different seeds.
pp_status pp_epoch_permute_local(pp_loader* L, uint64_t seed, int64_t chunk, void* stream) {
  NvtxRange nvtx_range("pp_epoch_permute_local");
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (L->poisoned) return fail(PP_ERR_CUDA, "loader is poisoned by an earlier CUDA error");
  if (L->d_node_set) return fail(PP_ERR_INVALID, "local shuffling is defined without a node set");
  if (L->files) return fail(PP_ERR_INVALID, "file loaders have no local shard to shuffle");
  if (chunk < 1 || chunk > L->local_rows)
    return fail(PP_ERR_INVALID, "chunk must be in [1, local_rows=%lld]", (long long)L->local_rows);
  DevGuard g(L->dev);
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  if (user != L->stream) {
    PPL_CUDA(L, cudaEventRecord(L->ev_in, user));
    PPL_CUDA(L, cudaStreamWaitEvent(L->stream, L->ev_in, 0));
  }
  if (L->pref_pending) {  // a pending (global) prefetch shares the scratch: order after it, discard it
    PPL_CUDA(L, cudaStreamWaitEvent(L->stream, L->ev_pref, 0));
    L->pref_pending = false;
  }
  pp_status ps = enqueue_order(L, seed, chunk, L->d_order, L->stream, L->local_rows);
  if (ps != PP_OK) return ps;
  if (L->W > 1) PPL_CUDA(L, launch_local_to_global(L->d_order, L->local_rows, L->W, L->rank, L->stream));
  if (user != L->stream) {
    PPL_CUDA(L, cudaEventRecord(L->ev_out, L->stream));
    PPL_CUDA(L, cudaStreamWaitEvent(user, L->ev_out, 0));
  }
  L->local = true;
  L->dma_epoch = false;
  L->steps = L->desc.drop_last ? L->local_rows / L->B : (L->local_rows + L->B - 1) / L->B;
  L->last_kernel = pp_loader::kLastNone;
  L->permuted = true;
  L->seed = seed;
  L->chunk = chunk;
  L->cursor = 0;
  return PP_OK;
}

// 32-bit digest of an epoch's collective arguments (splitmix64 finaliser over seed and chunk).
static uint32_t epoch_arg_hash(uint64_t seed, int64_t chunk) {
  uint64_t z = seed ^ (static_cast<uint64_t>(chunk) * 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<uint32_t>(z ^ (z >> 32));
}

// pp_epoch_permute is collective: every rank must pass the same (seed, chunk), or the ranks' slices
// of "the" global permutation would overlap and leave gaps.  NCCL: all-reduce of the digest.  IPC:
// each rank posts (seq << 32 | digest) into word seq & 1 of its flag words and reads every peer's
// same word until it carries seq (a peer is at most one epoch ahead, and then writes the other
// word).  Loopback shards share one caller, which drives them all.
static pp_status check_epoch_args(pp_loader* L, uint64_t seed, int64_t chunk) {
  const uint32_t h = epoch_arg_hash(seed, chunk);
  if (L->nccl) {
    bool same = false;
    std::string err;
    if (!nccl_same_everywhere(L->nccl, h, L->d_nccl_scratch, L->stream, &same, &err)) {
      L->poisoned = true;
      return fail(PP_ERR_NCCL, "epoch argument check: %s", err.c_str());
    }
    return same ? PP_OK : fail(PP_ERR_INVALID, "pp_epoch_permute arguments (seed, chunk) differ across ranks");
  }
  if (L->W == 1 || L->desc.peers != PP_PEERS_IPC || !L->d_flags) return PP_OK;
  if (!L->linked) return fail(PP_ERR_STATE, "sharded loader: peers not linked yet");
  const uint32_t seq = ++L->coll_seq;
  const int slot = static_cast<int>(seq & 1u);
  uint64_t word = (static_cast<uint64_t>(seq) << 32) | h;
  PPL_CUDA(L, cudaMemcpyAsync(L->d_flags + slot, &word, 8, cudaMemcpyHostToDevice, L->cstream));
  PPL_CUDA(L, cudaStreamSynchronize(L->cstream));
  double limit_s = 300.0;
  if (const char* e = getenv("PPLOAD_COLLECTIVE_TIMEOUT_S")) limit_s = atof(e);
  const auto t0 = std::chrono::steady_clock::now();
  int bad = -1;
  for (int o = 0; o < L->W; ++o) {
    if (o == L->rank) continue;
    for (int polls = 0;; ++polls) {
      uint64_t w = 0;
      PPL_CUDA(L, cudaMemcpyAsync(&w, L->peer_flags[o] + slot, 8, cudaMemcpyDeviceToHost, L->cstream));
      PPL_CUDA(L, cudaStreamSynchronize(L->cstream));
      if (static_cast<uint32_t>(w >> 32) == seq) {
        if (static_cast<uint32_t>(w) != h && bad < 0) bad = o;
        break;
      }
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit_s) {
        // this epoch did not happen: retract the posted word so a later attempt is not matched against it
        const uint64_t zero = 0;
        PPL_CUDA(L, cudaMemcpyAsync(L->d_flags + slot, &zero, 8, cudaMemcpyHostToDevice, L->cstream));
        PPL_CUDA(L, cudaStreamSynchronize(L->cstream));
        --L->coll_seq;
        return fail(PP_ERR_STATE, "rank %d did not reach pp_epoch_permute #%u within %.0f s", o, seq, limit_s);
      }
      if (polls > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  if (bad >= 0)
    return fail(PP_ERR_INVALID, "pp_epoch_permute arguments (seed, chunk) differ across ranks (rank %d vs rank %d)",
                L->rank, bad);
  return PP_OK;
}

// All-to-all epochs: n[t][d][o] for every step of the epoch, on the host (sizes every send / recv).
static pp_status build_a2a_counts(pp_loader* L) {
  const int64_t need = L->steps_global * L->W * L->W;
  if (need > L->counts_cap) {
    cudaFree(L->d_counts);
    if (L->h_counts) cudaFreeHost(L->h_counts);
    L->d_counts = nullptr;
    L->h_counts = nullptr;
    L->scratch_bytes -= L->counts_cap * 4;
    L->counts_cap = 0;
    if (cudaMalloc(&L->d_counts, need * 4) != cudaSuccess ||
        cudaHostAlloc(&L->h_counts, need * 4, cudaHostAllocDefault) != cudaSuccess)
      return fail(PP_ERR_OOM, "exchange count table");
    L->counts_cap = need;
    L->scratch_bytes += need * 4;
  }
  PPL_CUDA(L, launch_a2a_counts(L->d_order, L->compact ? nullptr : L->d_node_set, L->N, L->steps_global,
                                static_cast<int32_t>(L->B), L->W, L->d_counts, L->stream));
  PPL_CUDA(L, cudaMemcpyAsync(L->h_counts, L->d_counts, need * 4, cudaMemcpyDeviceToHost, L->stream));
  PPL_CUDA(L, cudaStreamSynchronize(L->stream));
  return PP_OK;
}

pp_status pp_epoch_permute(pp_loader* L, uint64_t seed, int64_t chunk, void* stream) {
  NvtxRange nvtx_range("pp_epoch_permute");
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (L->poisoned) return fail(PP_ERR_CUDA, "loader is poisoned by an earlier CUDA error");
  if (chunk < 1 || chunk > L->N) return fail(PP_ERR_INVALID, "chunk must be in [1, N=%lld]", (long long)L->N);
  DevGuard g(L->dev);
  {
    const pp_status cs = check_epoch_args(L, seed, chunk);
    if (cs != PP_OK) return cs;
  }
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  if (user != L->stream) {
    PPL_CUDA(L, cudaEventRecord(L->ev_in, user));
    PPL_CUDA(L, cudaStreamWaitEvent(L->stream, L->ev_in, 0));
  }
  if (L->pref_pending) {
    // the prefetch shares the sort scratch: order after it either way
    PPL_CUDA(L, cudaStreamWaitEvent(L->stream, L->ev_pref, 0));
    L->pref_pending = false;
    if (L->pref_seed == seed && L->pref_chunk == chunk) {
      L->cur ^= 1;  // the prefetched order becomes current
      L->d_order = L->d_orders[L->cur];
    } else {
      pp_status ps = enqueue_order(L, seed, chunk, L->d_order, L->stream, L->N);
      if (ps != PP_OK) return ps;
    }
  } else {
    pp_status ps = enqueue_order(L, seed, chunk, L->d_order, L->stream, L->N);
    if (ps != PP_OK) return ps;
  }
  if (user != L->stream) {
    PPL_CUDA(L, cudaEventRecord(L->ev_out, L->stream));
    PPL_CUDA(L, cudaStreamWaitEvent(user, L->ev_out, 0));
  }
  if (L->files) {  // the I/O planner needs the order on the host
    file_tier_reset(L->files);
    PPL_CUDA(L, cudaMemcpyAsync(L->h_order.data(), L->d_order, L->N * 4, cudaMemcpyDeviceToHost, L->stream));
    PPL_CUDA(L, cudaStreamSynchronize(L->stream));
    ++L->epoch_id;
    std::string err;
    if (!file_tier_set_epoch(L->files, L->epoch_id, L->h_order.data(), L->h_node_set.empty() ? nullptr : L->h_node_set.data(),
                             L->N, L->W, L->rank, L->steps_global, &err)) {
      L->poisoned = true;
      return fail(PP_ERR_OOM, "storage tier: %s", err.c_str());
    }
  }
  L->dma_epoch = L->W == 1 && L->n_spill > 0 && !L->files &&
                 (L->dma_mode == 1 || (L->dma_mode == 0 && chunk >= L->dma_min_chunk));
  if (L->dma_epoch) {  // the run planner needs the order on the host
    if (!L->h_order_pin && cudaHostAlloc(&L->h_order_pin, L->N * 4, cudaHostAllocDefault) != cudaSuccess)
      return fail(PP_ERR_OOM, "pinned order copy");
    if (!L->d_stage && cudaMalloc(&L->d_stage, static_cast<size_t>(L->B * L->rec_stride)) != cudaSuccess)
      return fail(PP_ERR_OOM, "DMA staging");
    PPL_CUDA(L, cudaMemcpyAsync(L->h_order_pin, L->d_order, L->N * 4, cudaMemcpyDeviceToHost, L->stream));
    PPL_CUDA(L, cudaStreamSynchronize(L->stream));
  }
  if (L->a2a) {
    const pp_status cs = build_a2a_counts(L);
    if (cs != PP_OK) return cs;
  }
  L->local = false;
  L->steps = L->steps_global;
  L->last_kernel = pp_loader::kLastNone;
  L->permuted = true;
  L->seed = seed;
  L->chunk = chunk;
  L->cursor = 0;
  return PP_OK;
}

pp_status pp_epoch_prefetch(pp_loader* L, uint64_t seed, int64_t chunk) {
  NvtxRange nvtx_range("pp_epoch_prefetch");
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (L->poisoned) return fail(PP_ERR_CUDA, "loader is poisoned by an earlier CUDA error");
  if (chunk < 1 || chunk > L->N) return fail(PP_ERR_INVALID, "chunk must be in [1, N=%lld]", (long long)L->N);
  DevGuard g(L->dev);
  if (L->pref_pending) PPL_CUDA(L, cudaStreamWaitEvent(L->pstream, L->ev_pref, 0));
  if (!L->d_orders[L->cur ^ 1]) {  // the second order buffer: allocated at the first prefetch
    if (cudaMalloc(&L->d_orders[L->cur ^ 1], L->N * 4) != cudaSuccess)
      return fail(PP_ERR_OOM, "prefetch order buffer (%lld bytes)", (long long)(L->N * 4));
    L->scratch_bytes += L->N * 4;
  }
  // WAR on the spare order buffer (read by the previous epoch's batches) and on
  // the sort scratch (used by work already enqueued on the loader stream)
  PPL_CUDA(L, cudaEventRecord(L->ev_pref_in, L->stream));
  PPL_CUDA(L, cudaStreamWaitEvent(L->pstream, L->ev_pref_in, 0));
  L->sort.grid_cap = L->prefetch_ctas;  // leave most SMs to the gathers it overlaps
  pp_status ps = enqueue_order(L, seed, chunk, L->d_orders[L->cur ^ 1], L->pstream, L->N);
  L->sort.grid_cap = 0;
  if (ps != PP_OK) return ps;
  PPL_CUDA(L, cudaEventRecord(L->ev_pref, L->pstream));
  L->pref_pending = true;
  L->pref_seed = seed;
  L->pref_chunk = chunk;
  return PP_OK;
}

// How a call orders itself against the consumer: a consumer stream (the call waits for the
// work enqueued on it so far and makes its later work wait for the batch), or explicit
// events (wait for `wait_ev` before writing `out`, record `ready_ev` when it is written).
struct Handoff {
  bool events = false;
  cudaStream_t cons = nullptr;
  cudaEvent_t wait_ev = nullptr, ready_ev = nullptr;
};

// The output slots of one next_steps call: step i goes to out + i*stride (labels / node
// ids + i*B), rows[i] receives its row count.
struct StepOut {
  uint8_t* out;
  int64_t stride;
  int32_t* labels;
  int64_t* nodes;
  int32_t* rows;
  bool vec;      // 16-byte aligned slots and a vector-path record: the vector kernels apply
  bool aligned;  // 16-byte aligned slots (out and its pitch)
};

// Storage tier: each step's rows are read from the hop files, then assembled on the GPU.
static pp_status enqueue_file_steps(pp_loader* L, int64_t nsteps, const StepOut& o) {
  for (int64_t i = 0; i < nsteps; ++i) {
    std::string err;
    cudaError_t e = file_tier_step(L->files, L->cursor + i, L->in_dtype, L->out_dtype, L->d_labels, o.out + i * o.stride,
                                   o.labels ? o.labels + i * L->B : nullptr, o.nodes ? o.nodes + i * L->B : nullptr,
                                   o.aligned, L->stream, &o.rows[i], &err);
    if (e == cudaErrorUnknown) {
      L->poisoned = true;
      return fail(PP_ERR_CUDA, "storage tier: %s", err.c_str());
    }
    if (e != cudaSuccess) return cuda_fail(L, e, "storage tier step");
  }
  L->last_kernel = pp_loader::kLastNone;
  return PP_OK;
}

// Chunk reshuffling over host-resident rows: one copy-engine DMA per run of consecutive
// records (pinned spill -> staging, or HBM -> staging), then a cast of the staged batch.
static pp_status enqueue_dma_steps(pp_loader* L, int64_t nsteps, const StepOut& o) {
  for (int64_t i = 0; i < nsteps; ++i) {
    const int64_t p0 = (L->cursor + i) * L->B;
    const int32_t nr = static_cast<int32_t>(std::max<int64_t>(0, std::min<int64_t>(L->B, L->N - p0)));
    auto row_of = [&](int32_t j) -> int64_t {
      const uint32_t v = L->h_order_pin[p0 + j];
      return (L->compact || L->h_node_set.empty()) ? static_cast<int64_t>(v) : L->h_node_set[v];
    };
    auto src_of = [&](int64_t r) -> const uint8_t* {
      return r < L->n_hbm ? L->d_store + r * L->rec_stride : L->h_spill + (r - L->n_hbm) * L->rec_stride;
    };
    for (int32_t j = 0; j < nr;) {
      const int64_t r0 = row_of(j);
      int32_t e = j + 1;
      while (e < nr && row_of(e) == r0 + (e - j) && ((r0 + (e - j) < L->n_hbm) == (r0 < L->n_hbm))) ++e;
      PPL_CUDA(L, cudaMemcpyAsync(L->d_stage + static_cast<int64_t>(j) * L->rec_stride, src_of(r0),
                                  static_cast<size_t>(e - j) * L->rec_stride, cudaMemcpyDefault, L->stream));
      j = e;
    }
    PPL_CUDA(L, launch_stage_cast(L->d_stage, L->rec_stride, nr, L->HF, L->in_dtype, L->out_dtype, o.vec,
                                  o.out + i * o.stride, L->d_order + p0, L->d_node_set, L->d_labels,
                                  o.labels ? o.labels + i * L->B : nullptr, o.nodes ? o.nodes + i * L->B : nullptr,
                                  L->stream));
    o.rows[i] = nr;
  }
  L->last_kernel = pp_loader::kLastNone;
  return PP_OK;
}

// Whether the next launch of `kind` may be chained to the previous one by programmatic dependent
// launch (only after a launch of the same kind, and only if its output spans do not overlap any
// span written by the chain so far); updates the chain's hulls.
static bool chain_pdl(pp_loader* L, int kind, const pp_loader::Span (&spans)[3]) {
  bool pdl = L->pdl && L->last_kernel == kind;
  for (int i = 0; i < 3 && pdl; ++i) pdl = !L->chain[i].overlaps(spans[i]);
  for (int i = 0; i < 3; ++i) {
    if (!pdl) L->chain[i] = pp_loader::Span{};
    L->chain[i].join(spans[i]);
  }
  return pdl;
}

// HBM / zero-copy host / peer rows: the gather kernels, all nsteps in one launch.
static pp_status enqueue_gather_steps(pp_loader* L, int64_t nsteps, const StepOut& o, bool pdl_ok) {
  GatherArgs a{};
  a.order = L->d_order;
  a.node_set = L->compact ? nullptr : L->d_node_set;  // compact: rows are node-set positions
  a.out_ids = L->compact ? L->d_node_set : nullptr;
  a.labels = L->d_labels;
  // global epoch: step t of rank r = positions [tWB + rB, ...) of the shared order;
  // local epoch: step t = positions [tB, ...) of this rank's own order
  a.N = L->local ? L->local_rows : L->N;
  a.first_pos = L->local ? L->cursor * L->B : L->cursor * L->B * L->W + static_cast<int64_t>(L->rank) * L->B;
  a.step_stride = L->local ? L->B : L->B * L->W;
  a.B = static_cast<int32_t>(L->B);
  a.nsteps = static_cast<int32_t>(nsteps);
  a.out = o.out;
  a.out_stride = o.stride;
  a.out_labels = o.labels;
  a.out_nodes = o.nodes;
  a.W = L->W;
  for (int i = 0; i < kMaxWorld; ++i) a.shards[i] = L->shards[i];
  a.rec_stride = L->rec_stride;
  a.xrec_stride = L->xrec_stride;
  a.HF = L->HF;
  a.in_dtype = L->in_dtype;
  a.out_dtype = L->out_dtype;
  a.tile_rows = L->tile_rows;
  a.num_sms = L->num_sms;
  a.l2_prefetch = L->l2_prefetch;
  a.max_ctas = L->max_ctas;
  int path = o.vec ? kPathVector : kPathScalar;
  // auto: register-staged loads for HBM-resident stores (96 % of copy bandwidth measured);
  // bulk copies when rows come over PCIe (2x the zero-copy LDG rate measured) or NVLink
  const bool remote = L->n_spill > 0 || L->desc.peers == PP_PEERS_IPC;
  if (o.vec && L->tma_ok && (L->gather_mode == 2 || (L->gather_mode == 0 && remote))) path = kPathTma;
  // Programmatic dependent launch only right after another gather of this epoch: batches of
  // one epoch are independent, and the first gather after a permute or an event wait is
  // fully serialised, so every gather sees a complete order.  A launch that rewrites memory an
  // earlier launch of the chain writes (a reused slot) is serialised too (chain_pdl).
  const auto span = [](const void* p, int64_t bytes) {
    pp_loader::Span sp;
    sp.lo = reinterpret_cast<uintptr_t>(p);
    sp.hi = p ? sp.lo + static_cast<uintptr_t>(bytes) : sp.lo;
    return sp;
  };
  const pp_loader::Span spans[3] = {span(o.out, (nsteps - 1) * o.stride + L->B * L->rec_out),
                                    span(o.labels, nsteps * L->B * 4), span(o.nodes, nsteps * L->B * 8)};
  const bool pdl = chain_pdl(L, pp_loader::kLastGather, spans);
  PPL_CUDA(L, launch_gather(a, path, pdl, L->grid_per_sm, L->stream));
  L->pdl_launches += pdl ? 1 : 0;
  // the next gather may overlap this one unless an event record follows it (pdl_ok false)
  L->last_kernel = pdl_ok ? pp_loader::kLastGather : pp_loader::kLastNone;
  for (int64_t i = 0; i < nsteps; ++i) {
    const int64_t s0 = a.first_pos + i * a.step_stride;
    o.rows[i] = static_cast<int32_t>(std::max<int64_t>(0, std::min<int64_t>(L->B, a.N - s0)));
  }
  return PP_OK;
}

// All-to-all steps (SURVEY.md §8(e) NCCL baseline, exchange.cu): per step, a stable compaction of
// every slice by owner (k_a2a_index), the pack of this rank's rows for every destination with the
// loader's gather kernel (cast fused), ncclSend / ncclRecv of the segments (sizes from the epoch's
// count table), and the unpack into batch order.  Loopback shards (PPLOAD_EXCHANGE=a2a) run each
// owner's index + pack inside this call, writing straight into this rank's receive buffer.
static pp_status enqueue_a2a_steps(pp_loader* L, int64_t nsteps, const StepOut& o) {
  const int W = L->W, r = L->rank;
  const int64_t B = L->B;
  if (!L->d_recvbuf) {
    const int64_t send_rows = L->nccl ? W * B : B;
    if (cudaMalloc(&L->d_recv_src, B * 4) != cudaSuccess || cudaMalloc(&L->d_send_rows, send_rows * 4) != cudaSuccess ||
        cudaMalloc(&L->d_recvbuf, B * L->rec_out) != cudaSuccess ||
        (L->nccl && cudaMalloc(&L->d_sendbuf, send_rows * L->rec_out) != cudaSuccess))
      return fail(PP_ERR_OOM, "all-to-all exchange buffers");
    L->scratch_bytes += B * 4 + send_rows * 4 + B * L->rec_out + (L->nccl ? send_rows * L->rec_out : 0);
  }
  const bool unpack_vec = o.aligned && L->rec_out % 16 == 0;
  for (int64_t i = 0; i < nsteps; ++i) {
    const int64_t t = L->cursor + i;
    const uint32_t* n = L->h_counts + t * W * W;  // n[d * W + o]
    A2AIndexArgs a{};
    a.order = L->d_order;
    a.node_set = L->compact ? nullptr : L->d_node_set;
    a.out_ids = L->compact ? L->d_node_set : nullptr;
    a.labels = L->d_labels;
    a.N = L->N;
    a.step_pos0 = t * W * B;
    a.B = static_cast<int32_t>(B);
    a.W = W;
    a.send_rows = L->d_send_rows;
    a.recv_src = L->d_recv_src;
    a.out_labels = o.labels ? o.labels + i * B : nullptr;
    a.out_nodes = o.nodes ? o.nodes + i * B : nullptr;
    int32_t rows = 0;
    for (int q = 0; q < W; ++q) {
      a.recv_off[q] = rows;
      rows += static_cast<int32_t>(n[r * W + q]);
    }
    // the pack: the loader's gather over a list of local rows of one owner (W = 1 view of its shard)
    auto pack = [&](int owner, int64_t count, uint8_t* dst) -> pp_status {
      GatherArgs g{};
      g.order = L->d_send_rows;
      g.N = count;
      g.B = static_cast<int32_t>(count);
      g.nsteps = 1;
      g.out = dst;
      g.W = 1;
      g.shards[0] = ShardView{L->shards[owner].hbm, L->shards[owner].spill, L->shards[owner].n_hbm, nullptr};
      g.rec_stride = L->rec_stride;
      g.HF = L->HF;
      g.in_dtype = L->in_dtype;
      g.out_dtype = L->out_dtype;
      g.tile_rows = L->tile_rows;
      g.num_sms = L->num_sms;
      g.max_ctas = L->max_ctas;
      if (count > 0)
        PPL_CUDA(L, launch_gather(g, L->vector_path ? kPathVector : kPathScalar, false, L->grid_per_sm, L->stream));
      return PP_OK;
    };
    if (L->nccl) {
      int64_t send_off[kMaxWorld], send_bytes[kMaxWorld], recv_off[kMaxWorld], recv_bytes[kMaxWorld];
      int32_t total = 0;
      for (int d = 0; d < W; ++d) {
        a.send_off[d] = total;
        send_off[d] = static_cast<int64_t>(total) * L->rec_out;
        send_bytes[d] = static_cast<int64_t>(n[d * W + r]) * L->rec_out;
        total += static_cast<int32_t>(n[d * W + r]);
        recv_off[d] = static_cast<int64_t>(a.recv_off[d]) * L->rec_out;
        recv_bytes[d] = static_cast<int64_t>(n[r * W + d]) * L->rec_out;
      }
      a.self = r;
      a.slice_lo = 0;
      a.slice_hi = W;
      a.recv_rank = r;
      PPL_CUDA(L, launch_a2a_index(a, L->stream));
      pp_status ps = pack(r, total, L->d_sendbuf);
      if (ps != PP_OK) return ps;
      std::string err;
      if (!nccl_exchange(L->nccl, W, L->d_sendbuf, send_off, send_bytes, L->d_recvbuf, recv_off, recv_bytes, L->stream,
                         &err)) {
        L->poisoned = true;
        return fail(PP_ERR_NCCL, "%s", err.c_str());
      }
    } else {  // loopback emulation: owner q packs its rows of slice r into the receive buffer
      for (int q = 0; q < W; ++q) {
        a.self = q;
        a.slice_lo = r;
        a.slice_hi = r + 1;
        a.recv_rank = q == 0 ? r : -1;
        for (int d = 0; d < W; ++d) a.send_off[d] = 0;
        PPL_CUDA(L, launch_a2a_index(a, L->stream));
        pp_status ps = pack(q, n[r * W + q], L->d_recvbuf + static_cast<int64_t>(a.recv_off[q]) * L->rec_out);
        if (ps != PP_OK) return ps;
      }
    }
    PPL_CUDA(L, launch_a2a_unpack(L->d_recvbuf, L->d_recv_src, rows, L->rec_out, o.out + i * o.stride, unpack_vec,
                                  L->stream));
    o.rows[i] = rows;
  }
  L->last_kernel = pp_loader::kLastNone;
  return PP_OK;
}

static pp_status next_steps(pp_loader* L, int32_t n, void* out, int64_t out_stride, int32_t* out_labels,
                            int64_t* out_nodes, int32_t* rows, int32_t* n_done, const Handoff& ho) {
  NvtxRange nvtx_range("pp_next_batches");
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (L->poisoned) return fail(PP_ERR_CUDA, "loader is poisoned by an earlier CUDA error");
  if (!rows || n < 1) return fail(PP_ERR_INVALID, "rows is NULL or n < 1");
  if (!L->permuted) return fail(PP_ERR_STATE, "pp_next_batch before pp_epoch_permute");
  if (!L->linked && !L->local) return fail(PP_ERR_STATE, "sharded loader: peers not linked yet");
  if (out_labels && !L->has_labels) return fail(PP_ERR_INVALID, "out_labels given but the loader has no labels");
  if (L->cursor >= L->steps) {
    rows[0] = 0;
    if (n_done) *n_done = 0;
    return PP_END_OF_EPOCH;
  }
  if (!out) return fail(PP_ERR_INVALID, "out is NULL");
  const int64_t nsteps = std::min<int64_t>(n, L->steps - L->cursor);
  if (nsteps > 1 && out_stride < L->B * L->rec_out)
    return fail(PP_ERR_INVALID, "out_stride_bytes %lld < one batch (%lld)", (long long)out_stride,
                (long long)(L->B * L->rec_out));
  const bool aligned = (reinterpret_cast<uintptr_t>(out) % 16 == 0) && (out_stride % 16 == 0);
  if (!(L->vector_path && aligned) && !L->files && !L->dma_epoch && !fast_div_ok(L->HF))
    return fail(PP_ERR_INVALID, "records of H*F = %d elements need a 16-byte aligned out / out_stride", L->HF);
  DevGuard g(L->dev);
  // ---- consumer -> loader (WAR on `out`)
  const bool handoff = !ho.events && ho.cons != L->stream;
  if (handoff) {  // the consumer stream's work so far
    PPL_CUDA(L, cudaEventRecord(L->ev_in, ho.cons));
    PPL_CUDA(L, cudaStreamWaitEvent(L->stream, L->ev_in, 0));
    L->last_kernel = pp_loader::kLastNone;
  }
  if (ho.events && ho.wait_ev) {  // the consumer's last use of `out`
    PPL_CUDA(L, cudaStreamWaitEvent(L->stream, ho.wait_ev, 0));
    L->last_kernel = pp_loader::kLastNone;
  }
  // ---- the steps
  StepOut o{static_cast<uint8_t*>(out), out_stride, out_labels, out_nodes, rows, L->vector_path && aligned, aligned};
  const bool signals = handoff || (ho.events && ho.ready_ev);  // an event record follows the steps
  pp_status st = L->files ? enqueue_file_steps(L, nsteps, o)
                 : L->dma_epoch ? enqueue_dma_steps(L, nsteps, o)
                 : (L->a2a && !L->local) ? enqueue_a2a_steps(L, nsteps, o)
                                         : enqueue_gather_steps(L, nsteps, o, !signals);
  if (st != PP_OK) return st;
  // ---- loader -> consumer (RAW on `out`)
  if (handoff) {
    PPL_CUDA(L, cudaEventRecord(L->ev_out, L->stream));
    PPL_CUDA(L, cudaStreamWaitEvent(ho.cons, L->ev_out, 0));
  }
  if (ho.events && ho.ready_ev) PPL_CUDA(L, cudaEventRecord(ho.ready_ev, L->stream));
  L->cursor += nsteps;
  if (n_done) *n_done = static_cast<int32_t>(nsteps);
  return PP_OK;
}

pp_status pp_next_batch(pp_loader* L, void* out, int32_t* out_labels, int64_t* out_nodes, int32_t* rows,
                        void* consumer_stream) {
  Handoff ho;
  ho.cons = static_cast<cudaStream_t>(consumer_stream);
  return next_steps(L, 1, out, 0, out_labels, out_nodes, rows, nullptr, ho);
}

pp_status pp_next_batches(pp_loader* L, int32_t n, void* out, int64_t out_stride_bytes, int32_t* out_labels,
                          int64_t* out_nodes, int32_t* rows, int32_t* n_done, void* consumer_stream) {
  Handoff ho;
  ho.cons = static_cast<cudaStream_t>(consumer_stream);
  return next_steps(L, n, out, out_stride_bytes, out_labels, out_nodes, rows, n_done, ho);
}

pp_status pp_next_batches_ev(pp_loader* L, int32_t n, void* out, int64_t out_stride_bytes, int32_t* out_labels,
                             int64_t* out_nodes, int32_t* rows, int32_t* n_done, void* wait_event,
                             void* ready_event) {
  Handoff ho;
  ho.events = true;
  ho.wait_ev = static_cast<cudaEvent_t>(wait_event);
  ho.ready_ev = static_cast<cudaEvent_t>(ready_event);
  return next_steps(L, n, out, out_stride_bytes, out_labels, out_nodes, rows, n_done, ho);
}

pp_status pp_next_batches_linear(pp_loader* L, int32_t n, const void* W, int32_t D, void* Z, pp_dtype z_dtype,
                                 int64_t z_stride_bytes, int32_t* rows, int32_t* n_done, void* consumer_stream) {
  NvtxRange nvtx_range("pp_next_batches_linear");
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (L->poisoned) return fail(PP_ERR_CUDA, "loader is poisoned by an earlier CUDA error");
  if (!rows || n < 1 || !W || !Z) return fail(PP_ERR_INVALID, "NULL argument or n < 1");
  if (L->files) return fail(PP_ERR_INVALID, "fused linear needs an in-memory store (not the storage tier)");
  if (L->out_dtype == PP_F32) return fail(PP_ERR_INVALID, "fused linear needs a 16-bit batch dtype (bf16 / f16)");
  // the K-chunked kernel for every shape, dtype and placement; the round-1 kernel with W_k resident in
  // shared memory (fp32 -> bf16 unsharded HBM stores, F <= 128) only on request (PPLOAD_LINEAR=res):
  // at the products shape the K-chunked CTA pairs measured 2.99-3.00 vs 3.13 ms per epoch (interleaved
  // A/B medians, profiles/r2/kc_pair/s3a_ab_products.jsonl, s3c_ab_products.jsonl)
  const char* kc_env = getenv("PPLOAD_LINEAR");
  const bool resident = L->in_dtype == PP_F32 && L->out_dtype == PP_BF16 && L->n_spill == 0 && L->W == 1 &&
                        linear_supported(L->H, L->F, D, L->num_sms) && kc_env && !strcmp(kc_env, "res");
  if (!resident && !linear_kc_supported(L->H, L->F, D, L->num_sms, L->in_dtype, L->out_dtype))
    return fail(PP_ERR_INVALID, "fused linear supports F %% 4 == 0 (fp32 records) or F %% 8 == 0 (16-bit records) and D in {256, 512} "
                "(F=%d, D=%d)", L->F, D);
  if (z_dtype != PP_BF16 && z_dtype != PP_F32) return fail(PP_ERR_INVALID, "z_dtype must be PP_BF16 or PP_F32");
  if (reinterpret_cast<uintptr_t>(W) % 16 || reinterpret_cast<uintptr_t>(Z) % 16 || z_stride_bytes % 16)
    return fail(PP_ERR_INVALID, "W, Z and z_stride_bytes must be 16-byte aligned");
  const int z_elem = z_dtype == PP_F32 ? 4 : 2;
  if (n > 1 && z_stride_bytes < L->B * L->H * static_cast<int64_t>(D) * z_elem)
    return fail(PP_ERR_INVALID, "z_stride_bytes smaller than one step");
  if (!L->permuted) return fail(PP_ERR_STATE, "pp_next_batches_linear before pp_epoch_permute");
  if (!L->linked && !L->local) return fail(PP_ERR_STATE, "sharded loader: peers not linked yet");
  if (L->cursor >= L->steps) {
    rows[0] = 0;
    if (n_done) *n_done = 0;
    return PP_END_OF_EPOCH;
  }
  const int64_t nsteps = std::min<int64_t>(n, L->steps - L->cursor);
  DevGuard g(L->dev);
  cudaStream_t cons = static_cast<cudaStream_t>(consumer_stream);
  const bool handoff = cons != L->stream;
  if (handoff) {
    PPL_CUDA(L, cudaEventRecord(L->ev_in, cons));
    PPL_CUDA(L, cudaStreamWaitEvent(L->stream, L->ev_in, 0));
  }
  LinearArgs a{};
  a.order = L->d_order;
  a.node_set = L->compact ? nullptr : L->d_node_set;
  a.store = L->d_store;
  a.rec_stride = L->rec_stride;
  // step t of this rank: positions [tWB + rB, ...) of the global order, or [tB, ...) of a local epoch
  a.N = L->local ? L->local_rows : L->N;
  a.first_pos = L->local ? L->cursor * L->B : L->cursor * L->B * L->W + static_cast<int64_t>(L->rank) * L->B;
  a.step_stride = L->local ? L->B : L->B * L->W;
  a.B = static_cast<int32_t>(L->B);
  a.nsteps = static_cast<int32_t>(nsteps);
  a.W = W;
  a.H = L->H;
  a.F = L->F;
  a.D = D;
  a.Z = static_cast<uint8_t*>(Z);
  a.z_stride = z_stride_bytes;
  a.z_elem = z_elem;
  a.num_sms = L->num_sms;
  a.in_dtype = L->in_dtype;
  a.out_dtype = L->out_dtype;
  a.world = L->W;
  for (int i = 0; i < kMaxWorld; ++i) a.shards[i] = ShardView{L->shards[i].hbm, L->shards[i].spill, L->shards[i].n_hbm};
  if (const char* e = getenv("PPLOAD_DEBUG_LINEAR")) a.debug = atoi(e);
  a.l2_prefetch = resident ? 1 : 0;  // resident kernel: next tile's rows; K-chunked: off (r2 sweep: no gain)
  if (const char* e = getenv("PPLOAD_LINEAR_PREFETCH")) a.l2_prefetch = atoi(e);
  static uint64_t* dbg_ts = nullptr;  // experiment probe: timestamps of CTA 0 (PPLOAD_DEBUG_TS=1)
  const bool want_ts = resident && getenv("PPLOAD_DEBUG_TS") != nullptr;
  if (want_ts && !dbg_ts) PPL_CUDA(L, cudaMalloc(&dbg_ts, (24 * 14 + 4 * 1024) * 8));
  if (want_ts) {
    PPL_CUDA(L, cudaMemsetAsync(dbg_ts, 0, (24 * 14 + 4 * 1024) * 8, L->stream));
    a.ts = dbg_ts;
  }
  pp_loader::Span zspans[3];
  zspans[0].lo = reinterpret_cast<uintptr_t>(Z);
  zspans[0].hi = zspans[0].lo + static_cast<uintptr_t>((nsteps - 1) * z_stride_bytes + L->B * L->H * D * z_elem);
  const bool pdl = !handoff && chain_pdl(L, pp_loader::kLastLinear, zspans);
  PPL_CUDA(L, resident ? launch_gather_linear(a, pdl, L->stream) : launch_gather_linear_kc(a, pdl, L->stream));
  L->pdl_launches += pdl ? 1 : 0;
  if (want_ts) {
    static uint64_t h[24 * 14 + 4 * 1024];
    PPL_CUDA(L, cudaMemcpyAsync(h, dbg_ts, sizeof(h), cudaMemcpyDeviceToHost, L->stream));
    PPL_CUDA(L, cudaStreamSynchronize(L->stream));
    const uint64_t t0 = h[0];
    for (int t = 0; t < 24; ++t) {
      fprintf(stderr, "ts tile %2d:", t);
      for (int s = 0; s < 14; ++s)
        fprintf(stderr, " %7.2f", h[t * 14 + s] ? (double)(int64_t)(h[t * 14 + s] - t0) / 1e3 : -1.0);
      fprintf(stderr, "\n");
    }
    // per-CTA entry / prologue done / exit, relative to the earliest entry
    const int nb = (L->num_sms / L->H) * L->H;
    uint64_t e0 = UINT64_MAX;
    for (int b = 0; b < nb; ++b) e0 = std::min(e0, h[24 * 14 + 4 * b]);
    double mx[4] = {0, 0, 0, 0}, sm[4] = {0, 0, 0, 0};
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < 4; ++j) {
        const double v = (double)(int64_t)(h[24 * 14 + 4 * b + j] - e0) / 1e3;
        mx[j] = std::max(mx[j], v);
        sm[j] += v / nb;
      }
    fprintf(stderr, "cta us (mean/max): entry %.2f/%.2f w_staged %.2f/%.2f prologue_done %.2f/%.2f exit %.2f/%.2f\n",
            sm[0], mx[0], sm[1], mx[1], sm[2], mx[2], sm[3], mx[3]);
  }
  L->last_kernel = handoff ? pp_loader::kLastNone : pp_loader::kLastLinear;
  if (handoff) {
    PPL_CUDA(L, cudaEventRecord(L->ev_out, L->stream));
    PPL_CUDA(L, cudaStreamWaitEvent(cons, L->ev_out, 0));
  }
  for (int64_t i = 0; i < nsteps; ++i)
    rows[i] = static_cast<int32_t>(std::max<int64_t>(0, std::min<int64_t>(L->B, a.N - (a.first_pos + i * a.step_stride))));
  L->cursor += nsteps;
  if (n_done) *n_done = static_cast<int32_t>(nsteps);
  return PP_OK;
}

pp_status pp_seek(pp_loader* L, int64_t step) {
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (!L->permuted) return fail(PP_ERR_STATE, "pp_seek before pp_epoch_permute");
  if (step < 0 || step > L->steps) return fail(PP_ERR_INVALID, "step out of range");
  if (L->files && step != L->cursor) file_tier_reset(L->files);  // staged next step no longer follows
  L->cursor = step;
  return PP_OK;
}

pp_status pp_loader_query(const pp_loader* L, pp_loader_info* info) {
  if (!L || !info) return fail(PP_ERR_INVALID, "NULL argument");
  info->num_positions = L->N;
  info->num_nodes_total = L->N_total;
  info->local_rows = L->local_rows;
  info->rows_hbm = L->n_hbm;
  info->rows_spill = L->n_spill;
  info->record_bytes_in = L->rec_in;
  info->record_stride = L->rec_stride;
  info->record_bytes_out = L->rec_out;
  info->steps_per_epoch = L->steps;
  info->cursor = L->cursor;
  info->permuted = L->permuted ? 1 : 0;
  info->gather_path = L->vector_path ? 0 : 1;
  info->local_epoch = L->local ? 1 : 0;
  info->epoch_positions = L->local ? L->local_rows : L->N;
  info->exchange_cast = L->d_xstore != nullptr ? 1 : 0;
  info->storage_mode = L->files ? (file_tier_direct(L->files) ? 1 : 2) : 0;
  info->storage_bytes_read = L->files ? file_tier_bytes_read(L->files) : 0;
  info->pdl_launches = L->pdl_launches;
  info->all_to_all = L->a2a ? 1 : 0;
  info->spill_shared = L->spill_fd >= 0 ? 1 : 0;
  info->hbm_store_bytes = L->borrowed ? 0 : L->n_hbm * L->rec_stride;
  info->hbm_exchange_bytes = L->d_xstore ? L->n_hbm * L->xrec_stride : 0;
  info->hbm_scratch_bytes = L->scratch_bytes;
  info->host_spill_bytes = static_cast<int64_t>(L->spill_bytes);
  return PP_OK;
}

pp_status pp_fill_synthetic(pp_loader* L, uint64_t data_seed) {
  NvtxRange nvtx_range("pp_fill_synthetic");
  if (!L) return fail(PP_ERR_INVALID, "loader is NULL");
  if (L->poisoned) return fail(PP_ERR_CUDA, "loader is poisoned by an earlier CUDA error");
  if (L->in_dtype == PP_BF16) return fail(PP_ERR_INVALID, "no synthetic generator for bf16 stores");
  if (L->files) return fail(PP_ERR_INVALID, "file loaders have no store to fill");
  DevGuard g(L->dev);
  const int64_t* ids = L->compact ? L->d_node_set : nullptr;
  PPL_CUDA(L, launch_fill_synthetic(L->d_store, 0, L->n_hbm, L->rec_stride, L->H, L->F, L->in_dtype, data_seed, L->W,
                                    L->rank, ids, L->stream));
  PPL_CUDA(L, launch_fill_synthetic(L->d_spill, L->n_hbm, L->n_spill, L->rec_stride, L->H, L->F, L->in_dtype,
                                    data_seed, L->W, L->rank, ids, L->stream));
  PPL_CUDA(L, cudaStreamSynchronize(L->stream));
  PPL_CUDA(L, refresh_exchange_copy(L));
  return PP_OK;
}

pp_status pp_get_order(pp_loader* L, int64_t* dst_host) {
  if (!L || !dst_host) return fail(PP_ERR_INVALID, "NULL argument");
  if (L->poisoned) return fail(PP_ERR_CUDA, "loader is poisoned by an earlier CUDA error");
  if (!L->permuted) return fail(PP_ERR_STATE, "pp_get_order before pp_epoch_permute");
  DevGuard g(L->dev);
  int64_t* tmp = nullptr;
  const int64_t n = L->local ? L->local_rows : L->N;
  if (cudaMalloc(&tmp, n * 8) != cudaSuccess) return fail(PP_ERR_OOM, "order staging allocation");
  cudaError_t e = launch_order_to_nodes(L->d_order, L->d_node_set, n, tmp, L->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dst_host, tmp, n * 8, cudaMemcpyDeviceToHost, L->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L->stream);
  cudaFree(tmp);
  if (e != cudaSuccess) return cuda_fail(L, e, "pp_get_order");
  return PP_OK;
}

pp_status pp_read_store(pp_loader* L, int64_t row0, int64_t n, void* dst_host) {
  if (!L || !dst_host) return fail(PP_ERR_INVALID, "NULL argument");
  if (row0 < 0 || n < 0 || row0 + n > L->local_rows) return fail(PP_ERR_INVALID, "row range out of bounds");
  if (L->files) return fail(PP_ERR_INVALID, "file loaders have no store");
  DevGuard g(L->dev);
  PPL_CUDA(L, cudaStreamSynchronize(L->stream));
  uint8_t* dst = static_cast<uint8_t*>(dst_host);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lr = row0 + i;
    const uint8_t* src = lr < L->n_hbm ? L->d_store + lr * L->rec_stride : L->h_spill + (lr - L->n_hbm) * L->rec_stride;
    PPL_CUDA(L, cudaMemcpy(dst + i * L->rec_in, src, L->rec_in, cudaMemcpyDefault));
  }
  return PP_OK;
}

// Exported handle (PP_IPC_HANDLE_BYTES = 256):
//   [0, 64)    CUDA IPC handle of the HBM store (zeros if every row spills)
//   [64, 128)  CUDA IPC handle of the exchange copy (zeros if none)
//   [128, 192) CUDA IPC handle of the collective flag words
//   [192, 256) HandleTail: rows in HBM, the shared spill file (owner pid + descriptor, bytes)
struct HandleTail {
  uint32_t magic;  // 'PPH6'
  int32_t pid;
  int32_t spill_fd;  // -1: no spill
  int32_t pad;
  int64_t n_hbm;
  int64_t spill_bytes;
};
static_assert(sizeof(HandleTail) <= 64, "handle tail");
constexpr uint32_t kHandleMagic = 0x36485050u;  // "PPH6"

pp_status pp_export_store(pp_loader* L, void* handle_out) {
  if (!L || !handle_out) return fail(PP_ERR_INVALID, "NULL argument");
  if (L->desc.peers != PP_PEERS_IPC) return fail(PP_ERR_INVALID, "pp_export_store needs PP_PEERS_IPC");
  DevGuard g(L->dev);
  static_assert(sizeof(cudaIpcMemHandle_t) == 64 && PP_IPC_HANDLE_BYTES == 256, "IPC handle layout");
  uint8_t* o = static_cast<uint8_t*>(handle_out);
  memset(o, 0, PP_IPC_HANDLE_BYTES);
  cudaIpcMemHandle_t h;
  if (L->d_store) {
    PPL_CUDA(L, cudaIpcGetMemHandle(&h, L->d_store));
    memcpy(o, &h, 64);
  }
  if (L->d_xstore) {
    PPL_CUDA(L, cudaIpcGetMemHandle(&h, L->d_xstore));
    memcpy(o + 64, &h, 64);
  }
  if (L->d_flags) {
    PPL_CUDA(L, cudaIpcGetMemHandle(&h, L->d_flags));
    memcpy(o + 128, &h, 64);
  }
  HandleTail t{kHandleMagic, static_cast<int32_t>(getpid()), L->spill_fd, 0, L->n_hbm,
               static_cast<int64_t>(L->spill_fd >= 0 ? L->spill_bytes : 0)};
  memcpy(o + 192, &t, sizeof(t));
  return PP_OK;
}

static bool nonzero(const uint8_t* p, int n) {
  for (int i = 0; i < n; ++i)
    if (p[i]) return true;
  return false;
}

pp_status pp_import_peer_stores(pp_loader* L, const void* handles) {
  NvtxRange nvtx_range("pp_import_peer_stores");
  if (!L || !handles) return fail(PP_ERR_INVALID, "NULL argument");
  if (L->desc.peers != PP_PEERS_IPC) return fail(PP_ERR_INVALID, "pp_import_peer_stores needs PP_PEERS_IPC");
  if (L->linked) return fail(PP_ERR_STATE, "peers already imported");
  DevGuard g(L->dev);
  const int64_t R = L->compact ? L->N : L->N_total;
  for (int o = 0; o < L->W; ++o) {
    if (o == L->rank) continue;
    const uint8_t* rec = static_cast<const uint8_t*>(handles) + PP_IPC_HANDLE_BYTES * o;
    HandleTail t;
    memcpy(&t, rec + 192, sizeof(t));
    if (t.magic != kHandleMagic) return fail(PP_ERR_INVALID, "handle %d is not a pp_export_store handle (ABI 6)", o);
    const int64_t rows_o = (R - o + L->W - 1) / L->W;
    if (t.n_hbm < 0 || t.n_hbm > rows_o || (t.n_hbm < rows_o && t.spill_bytes < (rows_o - t.n_hbm) * L->rec_stride))
      return fail(PP_ERR_INVALID, "handle %d: inconsistent placement (%lld of %lld rows in HBM)", o, (long long)t.n_hbm,
                  (long long)rows_o);
    cudaIpcMemHandle_t h;
    void* p = nullptr;
    if (nonzero(rec, 64)) {
      memcpy(&h, rec, 64);
      PPL_CUDA(L, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      L->ipc_opened.push_back(p);
    }
    void* x = nullptr;
    if (nonzero(rec + 64, 64) && L->xrec_stride > 0) {  // the owner keeps an exchange copy: read remote rows from it
      memcpy(&h, rec + 64, 64);
      PPL_CUDA(L, cudaIpcOpenMemHandle(&x, h, cudaIpcMemLazyEnablePeerAccess));
      L->ipc_opened.push_back(x);
    }
    if (nonzero(rec + 128, 64)) {
      void* f = nullptr;
      memcpy(&h, rec + 128, 64);
      PPL_CUDA(L, cudaIpcOpenMemHandle(&f, h, cudaIpcMemLazyEnablePeerAccess));
      L->ipc_opened.push_back(f);
      L->peer_flags[o] = static_cast<const uint64_t*>(f);
    }
    uint8_t* spill_dev = nullptr;
    if (t.spill_bytes > 0) {  // the owner's spilled rows: map its shared spill file and register it here
      char path[64];
      snprintf(path, sizeof(path), "/proc/%d/fd/%d", t.pid, t.spill_fd);
      const int fd = open(path, O_RDWR | O_CLOEXEC);
      if (fd < 0) return fail(PP_ERR_INVALID, "rank %d's spill (%s): %s", o, path, strerror(errno));
      void* m = mmap(nullptr, static_cast<size_t>(t.spill_bytes), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      close(fd);
      if (m == MAP_FAILED) return fail(PP_ERR_OOM, "mmap of rank %d's spill: %s", o, strerror(errno));
      if (cudaHostRegister(m, static_cast<size_t>(t.spill_bytes), cudaHostRegisterMapped | cudaHostRegisterPortable) !=
          cudaSuccess) {
        munmap(m, static_cast<size_t>(t.spill_bytes));
        return fail(PP_ERR_OOM, "cudaHostRegister of rank %d's spill failed", o);
      }
      L->peer_spills.push_back({m, static_cast<size_t>(t.spill_bytes)});
      PPL_CUDA(L, cudaHostGetDevicePointer(reinterpret_cast<void**>(&spill_dev), m, 0));
    }
    L->shards[o] = ShardView{static_cast<const uint8_t*>(p), spill_dev, t.n_hbm, static_cast<const uint8_t*>(x)};
  }
  L->linked = true;
  return PP_OK;
}

pp_status pp_nccl_unique_id(void* out) {
  if (!out) return fail(PP_ERR_INVALID, "NULL argument");
  std::string err;
  if (!nccl_unique_id(out, &err)) return fail(PP_ERR_NCCL, "%s", err.c_str());
  return PP_OK;
}

pp_status pp_link_loopback(pp_loader* const* Ls, int32_t W) {
  if (!Ls || W < 2 || W > kMaxWorld) return fail(PP_ERR_INVALID, "need 2..%d loaders", kMaxWorld);
  for (int r = 0; r < W; ++r) {
    const pp_loader* L = Ls[r];
    if (!L) return fail(PP_ERR_INVALID, "loader %d is NULL", r);
    if (L->desc.peers != PP_PEERS_LOOPBACK || L->W != W || L->rank != r)
      return fail(PP_ERR_INVALID, "loader %d: not a loopback rank %d of %d", r, r, W);
    if (L->dev != Ls[0]->dev || L->H != Ls[0]->H || L->F != Ls[0]->F || L->in_dtype != Ls[0]->in_dtype ||
        L->N_total != Ls[0]->N_total || L->rec_stride != Ls[0]->rec_stride ||
        L->out_dtype != Ls[0]->out_dtype || L->xrec_stride != Ls[0]->xrec_stride || L->compact != Ls[0]->compact ||
        L->N != Ls[0]->N)
      return fail(PP_ERR_INVALID, "loader %d: store shape differs from rank 0", r);
  }
  for (int r = 0; r < W; ++r) {
    for (int o = 0; o < W; ++o)
      Ls[r]->shards[o] = ShardView{Ls[o]->d_store, Ls[o]->d_spill, Ls[o]->n_hbm, o == r ? nullptr : Ls[o]->d_xstore};
    Ls[r]->linked = true;
  }
  return PP_OK;
}

}  // extern "C"
