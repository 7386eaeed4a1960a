// Internal interfaces between the C-ABI host code (pp_loader.cu) and the
// sm_100a kernels (permute.cu, gather.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace ppl {

constexpr int kMaxWorld = 8;

// Where the rows owned by one rank live: local row lr < n_hbm at
// hbm + lr * rec_stride, otherwise at spill + (lr - n_hbm) * rec_stride
// (spill = device alias of pinned, mapped host memory: UVA zero-copy).
// xhbm: the owner's exchange copy (rows < n_hbm already cast to the batch
// dtype, pitch GatherArgs::xrec_stride) that a peer reads instead of the fp32
// record; null for the reader's own shard or when the owner has none.
struct ShardView {
  const uint8_t* hbm;
  const uint8_t* spill;
  int64_t n_hbm;
  const uint8_t* xhbm = nullptr;
};

// ---- permutation (permute.cu) ------------------------------------------------
struct SortScratch {
  uint32_t* counts;     // [nb + 1]  bucket histogram, then exclusive offsets
  uint32_t* cursor;     // [nb]      scatter cursors
  uint32_t* blocksums;  // [ceil((nb+1)/kScanTile)]
  uint32_t* tmp;        // [U]       unit ids grouped by bucket
  uint32_t* ragged;     // [1]       position of the ragged chunk in pi
  uint32_t k32_mask = 0xffffffffu;  // test knob: compare fewer sub-key bits (forces the tie path)
  uint32_t* hist = nullptr;  // two-level path: per-tile digit counts, then offsets
  size_t hist_cap = 0;       // entries allocated in hist
  uint32_t l2_cap = 0xffffffffu;  // test knob (PPLOAD_DEBUG_L2CAP): smaller level-2 capacity forces the fallback
  // Two-level radix path (PPLOAD_PERMUTE=two_level): no global atomics, but measured
  // slower than the bucket sort on products (124 vs 111 us, and it interferes more
  // with overlapped gathers, profiles/r1g_*), so off by default.
  bool two_level = false;
  int grid_cap = 0;  // CTAs for the bucket-sort kernels (0: full grid); set for the prefetch stream
};
// Entries of SortScratch::hist the two-level path needs for U units (0: path not used).
size_t two_level_hist_entries(uint64_t U);
constexpr int kScanTile = 4096;

// Buckets used for U units: 2^bits with U / 2^bits in ~[14, 28).
int sort_bucket_bits(uint64_t U, int delta);

// pi[0..U) = units sorted by (Philox key, unit id); if ragged != null also
// *ragged = position of unit U-1 in pi.  U <= 4096 (and bits >= 0): one-CTA
// bitonic sort; otherwise the bucket sort.  All on `st`.
cudaError_t launch_unit_permutation(uint64_t seed, uint32_t U, int bits, bool allow_cta, const SortScratch& s, uint32_t* pi,
                                    uint32_t* ragged, cudaStream_t st);

// order[p], p in [0, N): chunk expansion of pi (chunk c, U = ceil(N / c)).
cudaError_t launch_chunk_expand(const uint32_t* pi, uint32_t U, uint64_t N, uint64_t c, const uint32_t* ragged,
                                uint32_t* order, cudaStream_t st);

// Local shuffle (pp_epoch_permute_local): order[p] <- order[p] * W + r.
cudaError_t launch_local_to_global(uint32_t* order, int64_t n, int32_t W, int32_t r, cudaStream_t st);

// ---- batch assembly (gather.cu) ----------------------------------------------
struct GatherArgs {
  const uint32_t* order;    // positions -> index into node set (or node id)
  const int64_t* node_set;  // row resolution: store row space index x -> node_set[x]; null: x itself
  const int64_t* out_ids;   // compact store: output node ids / labels via out_ids[x] (rows are node-set
                            // positions); null: the resolved row id is the node id
  const int32_t* labels;    // may be null
  int64_t N;                // positions in an epoch
  int64_t first_pos;        // first position of this rank in the first step
  int64_t step_stride;      // W * B
  int32_t B;
  int32_t nsteps;
  uint8_t* out;
  int64_t out_stride;       // bytes between step slots
  int32_t* out_labels;      // [nsteps * B] or null
  int64_t* out_nodes;       // [nsteps * B] or null
  int32_t W;
  ShardView shards[kMaxWorld];
  int64_t rec_stride;       // store pitch (bytes)
  int64_t xrec_stride;      // exchange-copy pitch (bytes), see ShardView::xhbm
  int32_t HF;               // elements per record
  int32_t in_dtype, out_dtype;  // pp_dtype codes
  int32_t tile_rows;        // batch rows per CTA tile (1..32)
  int32_t num_sms;
  int32_t l2_prefetch;      // 0 none, 1 L2::128B, 2 L2::256B load hint (PPLOAD_L2_PREFETCH)
  int32_t max_ctas = 0;     // > 0: cap on the grid (pp_set_grid_limit: leave SMs to an overlapped consumer)
};

// One launch assembling a.nsteps steps.  pdl: launch with programmatic stream
// serialization (may overlap the previous gather on the stream; only valid
// when the previous kernel on `st` is a gather of the same epoch).
// grid_per_sm caps the persistent grid at num_sms * grid_per_sm CTAs.
enum { kPathVector = 0, kPathScalar = 1, kPathTma = 2 };
cudaError_t launch_gather(const GatherArgs& a, int path, bool pdl, int grid_per_sm, cudaStream_t st);
bool gather_vector_ok(int32_t HF, int32_t in_dtype, int32_t out_dtype, int64_t rec_stride);
bool gather_tma_ok(int32_t HF, int32_t in_dtype);  // record fits the bulk-copy stages

// ---- fused gather + per-hop linear on tcgen05 (linear.cu) --------------------
struct LinearArgs {
  const uint32_t* order;
  const int64_t* node_set;
  const uint8_t* store;     // HBM store, node-major fp32 records
  int64_t rec_stride;
  int64_t N, first_pos, step_stride;
  int32_t B, nsteps;
  const void* W;            // bf16 [H][F][D], read by TMA (MN-major B operand)
  int32_t H, F, D;
  uint8_t* Z;               // [nsteps][B][H][D] of z_elem bytes
  int64_t z_stride;         // bytes between step slots
  int32_t z_elem;           // 2 (bf16) or 4 (fp32)
  int32_t num_sms;
  int32_t debug;            // experiment knob (PPLOAD_DEBUG_LINEAR), bits: 1 skip loads, 2 skip Z stores,
                            // 4 skip the drain, 8 skip A-tile stores,
                            // 64 skip MMAs, 128 no TMA stores (16-byte stores instead), 256 hop-major Z (timing only)
  int32_t l2_prefetch;      // 1: bulk L2 prefetch of the next tile's rows (PPLOAD_LINEAR_PREFETCH, default 1)
  int32_t z_tma;            // set by launch_gather_linear: Z tensor map encoded, epilogue uses TMA stores
  uint64_t* ts;             // experiment probe (PPLOAD_DEBUG_TS): per-tile timestamps of CTA 0, or null
  // K-chunked kernel (any F % 8 == 0; any store dtype; spilled / sharded stores)
  int32_t in_dtype = 0, out_dtype = 1;  // store dtype; A operand = W dtype = out_dtype (bf16 / f16)
  int32_t world = 1;                    // owners: row v on shards[v % world] at local row v / world
  ShardView shards[kMaxWorld];
  int32_t tma_a = 0;                    // set by launch_gather_linear_kc: A chunks by TMA tile::gather4
  int32_t tma_f32 = 0;                  // set by launch_gather_linear_kc: fp32 records by gather4 into staging
  int32_t hop_rows = 0;                 // set by launch_gather_linear_kc: the fp32 A map is [rows x H][F] (hop k of
                                        // node v = map row v H + k; K padding zero-filled out of bounds)
  int32_t pair = 0;                     // set by launch_gather_linear_kc: CTA pairs (cta_group::2, M = 256)
  int32_t units = 0;                    // set by launch_gather_linear_kc: (tile, hop) units over the whole grid
};
bool linear_supported(int H, int F, int D, int num_sms);
// The K-chunked kernel: F % 8 == 0, D in {256, 512}, 16-bit batch dtype.
bool linear_kc_supported(int H, int F, int D, int num_sms, int in_dtype, int out_dtype);
cudaError_t launch_gather_linear_kc(const LinearArgs& a, bool pdl, cudaStream_t st);
// Encodes the Z and W tensor maps and launches the fused kernel on `st`.
// pdl: programmatic dependent launch (only right after another fused launch of this
// epoch on `st`: launches are independent, so the next grid's CTAs may start on SMs
// the previous grid's finished CTAs have left).
cudaError_t launch_gather_linear(const LinearArgs& a, bool pdl, cudaStream_t st);

// ---- Eq. (2) propagation (propagate.cu) --------------------------------------
cudaError_t launch_operator_values(int64_t n, const int64_t* row_ptr, const int64_t* col, double* val,
                                   cudaStream_t st);
cudaError_t launch_spmm(int64_t n, int32_t F, const int64_t* row_ptr, const int64_t* col, const double* val,
                        const float* x, float* y, cudaStream_t st);
// Propagation into the loader's node-major fp32 store (pp_propagate_store).
struct StorePropArgs {
  int64_t local_rows;       // rows of this rank (CSR rows, local order)
  int32_t F, k;             // features; hop slot written (reads slot k-1)
  int32_t W, rank;
  const int64_t* row_ptr;   // [local_rows + 1]
  const int64_t* col;       // global column ids
  const int32_t* deg;       // [N_total] d~ (row lengths of I + A)
  ShardView shards[kMaxWorld];  // fp32 stores of every owner (shards[rank] = own)
  int64_t rec_stride;
  uint8_t* xstore;          // own exchange copy or null: slot k rewritten with the cast
  int64_t xrec_stride;
  int32_t x_dtype;          // 1 bf16, 2 f16
  const uint32_t* col32 = nullptr;  // int32 copy of col (the L2-sliced kernel), or null
};
cudaError_t launch_spmm_store(const StorePropArgs& a, cudaStream_t st);
// col32[p] = col[p] (nnz entries; ids < 2^32), for the L2-sliced kernels.
cudaError_t launch_col_to_u32(const int64_t* col, int64_t nnz, uint32_t* col32, cudaStream_t st);
// deg[i] = row_ptr[i+1] - row_ptr[i] (hop-major propagation through the sliced kernel).
cudaError_t launch_row_lengths(const int64_t* row_ptr, int64_t n, int32_t* deg, cudaStream_t st);
// L2-sliced propagation (propagate.cu): a hop through a scratch of spmm_sliced_scratch_bytes
// (fp64 weights per nonzero + a window-major copy of the input slot).  Hop-major: y = B x over n
// rows of F fp32; fresh_w: compute the weights (else reuse the scratch's from the previous hop).
cudaError_t launch_spmm_sliced_rows(int64_t n, int32_t F, const int64_t* row_ptr, const uint32_t* col32,
                                   const int32_t* deg, const float* x, float* y, uint8_t* scratch, int64_t nnz,
                                   bool fresh_w, cudaStream_t st);
// Into a W = 1 loader store (slot a.k from slot a.k - 1; a.col32 required).
cudaError_t launch_spmm_store_sliced(const StorePropArgs& a, uint8_t* scratch, int64_t nnz, cudaStream_t st);
int64_t spmm_sliced_scratch_bytes(int64_t rows, int32_t F, int64_t nnz);
// Wave-synchronous propagation (propagate.cu, k_spmm_wave): W = 1, F % 4 == 0, F <= 128, every
// row in HBM.  y row i (dst + i * dst_stride, fp32) = sum over the CSR row of w_ij * x row j
// (src + j * src_stride); weights val[p] or, with val == null, 1/sqrt(d~_i deg[j]).
struct WaveArgs {
  int64_t n = 0, ncols = 0;  // output rows; column-id range (windows split [0, ncols))
  int32_t F = 0, nv = 0;     // nv = F / 4 (set by the launcher)
  const int64_t* row_ptr = nullptr;
  const int64_t* col = nullptr;
  const double* val = nullptr;
  const int32_t* deg = nullptr;
  const uint8_t* src = nullptr;
  int64_t src_stride = 0;    // bytes
  uint8_t* dst = nullptr;
  int64_t dst_stride = 0;
  uint8_t* xdst = nullptr;   // optional 16-bit copy of the output rows (exchange copy slot)
  int64_t x_stride = 0;
  int32_t x_dtype = 1;       // 1 bf16, 2 f16
  // set by launch_spmm_wave
  int32_t R = 0, C = 0, lag = 0, spin = 0;
  int64_t win = 0;
  unsigned* sync = nullptr;
};
bool spmm_wave_eligible(int32_t F, const void* src, int64_t src_stride, const void* dst, int64_t dst_stride);
bool spmm_use_wave(int64_t n, int32_t F);
// sync: 4 bytes of device scratch (zeroed here, stream-ordered).
cudaError_t launch_spmm_wave(WaveArgs a, unsigned* sync, cudaStream_t st);
// Row kernel with the neighbour rows staged in shared memory by cp.async (same WaveArgs; W = 1,
// F % 4 == 0, F <= 128, every row in HBM); PPLOAD_SPMM=cp selects it.
bool spmm_use_cp();
cudaError_t launch_spmm_rows_cp(WaveArgs a, cudaStream_t st);
bool spmm_use_sliced(int64_t rows, int32_t F);

// ---- DMA-staged assembly (gather.cu): out row j = cast(stage record j) ----------
// order: the step's order entries (positions -> node-set index or node id), for ids / labels.
cudaError_t launch_stage_cast(const uint8_t* stage, int64_t rec_stride, int32_t rows, int32_t HF, int32_t in_dtype,
                              int32_t out_dtype, bool vec, uint8_t* out, const uint32_t* order,
                              const int64_t* node_set, const int32_t* labels, int32_t* out_labels, int64_t* out_nodes,
                              cudaStream_t st);

// ---- exchange copy (gather.cu) ----------------------------------------------
// dst[r] = cast(src[r]) for rows [0, rows): fp32 records (pitch rec_stride) ->
// 16-bit records (pitch xrec_stride), the gather's RNE cast.  HF % 8 == 0.
cudaError_t launch_cast_records(const uint8_t* src, int64_t rows, int64_t rec_stride, int32_t HF, int32_t out_dtype,
                                uint8_t* dst, int64_t xrec_stride, cudaStream_t st);

// ---- synthetic fill (gather.cu) ---------------------------------------------
// ids (compact store): record x holds node ids[x] (x = row0 + row, times W plus rank); null: node x.
cudaError_t launch_fill_synthetic(uint8_t* base, int64_t row0, int64_t nrows, int64_t rec_stride, int32_t H,
                                  int32_t F, int32_t dtype, uint64_t data_seed, int32_t W, int32_t rank,
                                  const int64_t* ids, cudaStream_t st);
// Compact store upload from a device source (see k_pack_rows).
cudaError_t launch_pack_rows(const void* src, int64_t hop_stride, int64_t row_stride, int32_t elem, int32_t H,
                             int32_t F, const int64_t* ids, int64_t nrows, int32_t W, int32_t rank, uint8_t* dst,
                             int64_t rec_stride, cudaStream_t st);

// ---- storage tier (storage.cu) ----------------------------------------------
struct FileTier;
FileTier* file_tier_open(const char* const* paths, int H, int64_t N_total, int F, int s_in, int64_t B, int dev,
                         std::string* err);
void file_tier_close(FileTier* T);
bool file_tier_direct(const FileTier* T);
int64_t file_tier_bytes_read(const FileTier* T);
void file_tier_reset(FileTier* T);  // drop staged steps (waits for their reads)
// New epoch: host order (N positions -> node-set index or node id), optional host
// node set, slicing (B from open, W, rank) and step count; grows the staging
// for the epoch's largest step.  The arrays must live until the next call.
bool file_tier_set_epoch(FileTier* T, uint64_t epoch, const uint32_t* order, const int64_t* node_set, int64_t N,
                         int32_t W, int32_t rank, int64_t steps, std::string* err);
// Assemble `step` into out on st (waits for its reads; keeps the next steps staging).
cudaError_t file_tier_step(FileTier* T, int64_t step, int32_t in_dtype, int32_t out_dtype, const int32_t* labels,
                           uint8_t* out, int32_t* out_labels, int64_t* out_nodes, bool out_vec, cudaStream_t st,
                           int32_t* rows, std::string* err);

// ---- all-to-all exchange (exchange.cu): the NCCL baseline of SURVEY.md §8(e) ----------------
// n[t][d][o] (u32 [steps][W][W]): positions of slice d of step t whose row owner o holds.
cudaError_t launch_a2a_counts(const uint32_t* order, const int64_t* node_set, int64_t N, int64_t steps, int32_t B,
                              int32_t W, uint32_t* table, cudaStream_t st);
struct A2AIndexArgs {
  const uint32_t* order;
  const int64_t* node_set;  // row-space resolution as in GatherArgs (null for compact stores)
  const int64_t* out_ids;   // compact stores: node ids / labels via out_ids[x]
  const int32_t* labels;
  int64_t N;                // positions of the epoch
  int64_t step_pos0;        // first position of the step (t * W * B)
  int32_t B, W;
  int32_t self;             // owner whose local rows go to send_rows
  int32_t slice_lo, slice_hi;  // destination slices handled (one CTA each)
  int32_t recv_rank;        // slice whose receive index / ids / labels are written (-1: none)
  int32_t send_off[kMaxWorld];  // row offset of segment d in send_rows
  int32_t recv_off[kMaxWorld];  // row offset of owner o's rows in the receive buffer
  uint32_t* send_rows;      // local rows of `self`, by destination segment, slice order
  uint32_t* recv_src;       // [B]: receive-buffer row of slice position j
  int32_t* out_labels;      // [B] or null
  int64_t* out_nodes;       // [B] or null
};
cudaError_t launch_a2a_index(const A2AIndexArgs& a, cudaStream_t st);
cudaError_t launch_a2a_unpack(const uint8_t* recv, const uint32_t* recv_src, int32_t rows, int64_t rec_out,
                              uint8_t* out, bool vec, cudaStream_t st);
// NCCL, loaded with dlopen on first use.
bool nccl_unique_id(void* out128, std::string* err);
void* nccl_comm_create(const void* id128, int W, int rank, std::string* err);
void nccl_comm_destroy(void* comm, bool abort);
bool nccl_check_async(void* comm, std::string* err);
bool nccl_exchange(void* comm, int W, const uint8_t* send, const int64_t* send_off, const int64_t* send_bytes,
                   uint8_t* recv, const int64_t* recv_off, const int64_t* recv_bytes, cudaStream_t st,
                   std::string* err);
bool nccl_same_everywhere(void* comm, int64_t h, int64_t* buf, cudaStream_t st, bool* same, std::string* err);

// order (u32 positions) -> global node ids (int64), for pp_get_order.
cudaError_t launch_order_to_nodes(const uint32_t* order, const int64_t* node_set, int64_t N, int64_t* dst,
                                  cudaStream_t st);

}  // namespace ppl
