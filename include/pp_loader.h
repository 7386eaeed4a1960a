/*
 * pp_loader.h -- C ABI of libppload.so, a B200-native (sm_100a) mini-batch
 * loader for pre-propagation GNNs (PP-GNNs), the hot path that arXiv
 * 2504.13266 ("Graph Learning at Scale: Characterizing and Optimizing
 * Pre-Propagation GNNs") optimises.
 *
 * What the library computes (PAPER.md line numbers are lines of the paper's
 * LaTeX source; "Ox" are the oracle steps of SURVEY.md §8(c)):
 *   - Input: the K+1 pre-propagated hop matrices X_k = B^k X, k = 0..K, with
 *     B = D~^{-1/2}(I+A)D~^{-1/2} (Eq. (2)), each
 *     [N_total, F], plus an optional training-node set and labels.
 *   - pp_epoch_permute: the per-epoch shuffle.  chunk = 1 is SGD-RR, a fresh
 *     uniform row permutation; chunk = c > 1 is the paper's
 *     chunk reshuffling, "reshuffle training data indices at the chunk level,
 *     with each chunk comprising contiguous node features".
 *     The permutation is the argsort of 64-bit Philox4x32-10 keys (O4-O7).
 *   - pp_next_batch: batch assembly, "copy the scattered node features into"
 *     one contiguous batch, done on the GPU: out[j,k,f] =
 *     cast(X_k[v_j, f]) with the fp32 -> bf16/fp16 round-to-nearest-even cast
 *     fused in (O9, O10).  Asynchronous on a loader stream with an event
 *     handoff to the consumer stream: the paper's double-buffer prefetch on
 *     separate streams when the caller alternates two
 *     output buffers.
 *   - Rows beyond the HBM budget live in pinned, mapped host memory and are
 *     read zero-copy over PCIe (host placement).
 *   - W > 1: nodes are sharded round-robin over W GPUs (owner(v) = v mod W,
 *     local row v div W; "distributing data across multiple GPUs",
 *     PAPER.md:285) and each rank reads the rows of its batch from the
 *     owners' HBM by peer (NVLink) loads.
 *
 * Conventions for every entry point:
 *   - Every call returns pp_status; no C++ exception crosses the ABI.
 *   - PP_ERR_INVALID: bad arguments, no side effects.  pp_last_error() has a
 *     message (thread-local, valid until the next failing call on the thread).
 *   - PP_ERR_CUDA / PP_ERR_NCCL are sticky: the handle is poisoned and only
 *     pp_loader_destroy is valid afterwards.
 *   - One handle is used by one host thread at a time.
 *   - "stream" arguments are cudaStream_t values passed as void*; NULL is the
 *     legacy default stream.
 *   - Tracing: every call opens an NVTX range named after it (nsys / ncu
 *     timelines; no cost beyond a few ns without a tool attached).
 */
#ifndef PP_LOADER_H
#define PP_LOADER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_ABI_VERSION 6

/* Bytes of one rank's exported store handle (pp_export_store). */
#define PP_IPC_HANDLE_BYTES 256

/* Bytes of an NCCL unique id (pp_nccl_unique_id, pp_loader_desc.nccl_unique_id). */
#define PP_NCCL_ID_BYTES 128

typedef struct pp_loader pp_loader; /* opaque handle */

typedef enum {
  PP_OK = 0,
  PP_ERR_INVALID = 1,   /* bad argument; no side effects */
  PP_ERR_OOM = 2,       /* device or pinned-host allocation failed */
  PP_ERR_CUDA = 3,      /* CUDA runtime error; handle poisoned */
  PP_ERR_NCCL = 4,      /* NCCL failure (PP_PEERS_NCCL); handle poisoned */
  PP_ERR_STATE = 5,     /* call out of order (e.g. next_batch before any permute) */
  PP_END_OF_EPOCH = 6   /* cursor exhausted; *rows = 0, nothing enqueued */
} pp_status;

typedef enum { PP_F32 = 0, PP_BF16 = 1, PP_F16 = 2 } pp_dtype;
/* PP_MEM_FILES: the storage tier (see pp_hop_desc). */
typedef enum { PP_MEM_HOST = 0, PP_MEM_DEVICE = 1, PP_MEM_FILES = 2 } pp_mem;

/* How the W ranks of a sharded loader reach each other's stores. */
typedef enum {
  PP_PEERS_NONE = 0,     /* W == 1 */
  PP_PEERS_IPC = 1,      /* one process per GPU; handles exchanged with
                            pp_export_store / pp_import_peer_stores */
  PP_PEERS_LOOPBACK = 2, /* W shards in ONE process on ONE device, linked with
                            pp_link_loopback (tests the sharded path on 1 GPU) */
  PP_PEERS_NCCL = 3      /* one process per GPU; every step's rows are exchanged by an
                            NCCL all-to-all (ncclSend / ncclRecv):
                            each owner packs the rows it holds for every rank (cast
                            fused), the receiver unpacks them into batch order.  Needs
                            desc.nccl_unique_id.  Also valid with W == 1 (a
                            self-exchange through NCCL). */
} pp_peers;

/* The K+1 hop matrices X_0..X_K.
 *   elem(k, v, f) = data[k*hop_stride + v*row_stride + f]   (element units)
 *   hop-major [H][N][F]: hop_stride = N*F, row_stride = F
 *   node-major [N][H][F]: hop_stride = F,   row_stride = H*F
 * Requirements: row_stride >= F.  data == NULL: allocate the store only
 * (fill it with pp_fill_synthetic).  For W > 1, data (if given) covers all
 * N rows; rank r copies only the rows it owns (v mod W == r).
 *
 * where == PP_MEM_FILES (storage tier; "Direct Storage
 * Access"): data is a `const char* const*` array of H file
 * paths, hop k's file holding X_k as raw little-endian [N_total][F] of dtype
 * (no header; "we split input features of different hops into separate
 * files"); hop_stride / row_stride are ignored.  No store is
 * built: every step's rows are read from the files (one read per run of
 * consecutive node ids and hop -- a chunk with chunk reshuffling
 * -- O_DIRECT unless the file system refuses it or PPLOAD_IO_DIRECT=0) into a
 * pinned staging slot by a pool of I/O threads, DMA'd to the GPU and cast into
 * `out` there; the next step is read while the GPU consumes the current one.
 * The files must stay unchanged while the loader lives.  W > 1 is allowed with
 * peers == PP_PEERS_NONE: each rank reads its own slice of the global epoch
 * from the shared files.  Not available for file loaders: a store (so no
 * pp_fill_synthetic / pp_read_store / pp_propagate_store / fused linear /
 * peer linking), pp_epoch_permute_local, hbm_budget_bytes. */
typedef struct {
  const void* data;
  pp_mem where;        /* memory space of data */
  int64_t num_nodes;   /* N_total rows per hop matrix (>= 1, < 2^32) */
  int32_t num_hops;    /* H = K + 1 (>= 1) */
  int32_t feat_dim;    /* F (>= 1) */
  int64_t hop_stride;  /* elements */
  int64_t row_stride;  /* elements */
  pp_dtype dtype;      /* PP_F32, PP_F16 or PP_BF16 */
} pp_hop_desc;

typedef struct {
  pp_hop_desc hops;
  const int64_t* node_set;  /* host, num_set ids in [0, N_total) (training nodes,
                               PAPER.md:365); NULL => all rows 0..N_total-1 */
  int64_t num_set;          /* ignored when node_set == NULL */
  const int32_t* labels;    /* host, length N_total; NULL => no labels */
  int32_t batch_size;       /* B rows per rank per step (>= 1) */
  pp_dtype out_dtype;       /* PP_BF16 / PP_F16 (RNE cast from PP_F32), or
                               == hops.dtype (bit copy) */
  int32_t drop_last;        /* 0: keep the ragged last step; 1: drop it */
  int64_t hbm_budget_bytes; /* bytes of HBM for this rank's store; rows
                               beyond it spill to pinned mapped host memory.
                               0 => (free HBM - 2 GiB reserve - this
                               loader's own scratch); < 0 => all rows in host
                               memory (the paper's host placement).  W > 1 with
                               PP_PEERS_IPC: the spill is an anonymous
                               shared-memory file (memfd) that the peers map
                               and register too, so every
                               rank reads another's spilled rows zero-copy.
                               Host-resident rows are read zero-copy by the
                               gather kernel; under chunk reshuffling
                               (chunk >= 64, PPLOAD_DMA_MIN_CHUNK) each step's
                               runs of consecutive records are moved by the
                               copy engines instead (one cudaMemcpyAsync per
                               run) and cast on the GPU
                               (PPLOAD_SPILL_PATH=dma|kernel forces a path). */
  int32_t world_size;       /* W >= 1 */
  int32_t rank;             /* 0 <= r < W */
  pp_peers peers;           /* W == 1: PP_PEERS_NONE (or PP_PEERS_NCCL); W > 1:
                               IPC, LOOPBACK or NCCL (file loaders: always
                               PP_PEERS_NONE, any W) */
  int32_t device;           /* CUDA device ordinal */
  int32_t store_set_only;   /* 1: the store holds only the node_set rows ("the input
                               data size after preprocessing is proportional to the
                               number of labeled nodes"): record i is
                               node node_set[i]; sharding (W > 1) is over node-set
                               positions (owner i mod W).  Needs node_set and an
                               in-memory source; batches are identical to the full
                               store's.  Not with pp_propagate_store (which needs
                               every node).  0: every node has a record. */
  int32_t borrow_device_data; /* 1: hops.data is a device tensor already in the
                               store layout (node-major [N][H][F], hop_stride = F,
                               row_stride = H*F, H*F*elem a 16-B multiple,
                               16-B aligned): the loader uses it in place instead
                               of copying it (no second copy of GPU-resident hop
                               features).  The caller keeps it alive until
                               pp_loader_destroy; pp_fill_synthetic and
                               pp_propagate_store write into it.  Needs W == 1,
                               no store_set_only and the whole store in HBM,
                               else PP_ERR_INVALID.  0: copy (default). */
  const void* nccl_unique_id; /* PP_PEERS_NCCL: PP_NCCL_ID_BYTES from pp_nccl_unique_id on one
                               rank, broadcast by the caller (e.g. torch.distributed); NULL
                               otherwise.  Read during pp_loader_create only. */
} pp_loader_desc;

/* Read-only facts about a loader (pp_loader_query). */
typedef struct {
  int64_t num_positions;    /* N: |node_set| or N_total */
  int64_t num_nodes_total;  /* N_total */
  int64_t local_rows;       /* records owned by this rank (node ids, or node-set positions
                               with store_set_only) */
  int64_t rows_hbm;         /* of which in HBM */
  int64_t rows_spill;       /* of which in pinned host memory (UVA) */
  int64_t record_bytes_in;  /* H*F*s_in: bytes of one node record in the store */
  int64_t record_stride;    /* store pitch between records (>= record_bytes_in, 16-B multiple) */
  int64_t record_bytes_out; /* H*F*s_out: bytes of one output row */
  int64_t steps_per_epoch;  /* ceil(N / (W*B)), or floor with drop_last */
  int64_t cursor;           /* next step index */
  int32_t permuted;         /* 1 after the first pp_epoch_permute */
  int32_t gather_path;      /* 0 = vector (16-B) path, 1 = scalar fallback */
  int32_t local_epoch;      /* 1 if the current epoch came from pp_epoch_permute_local */
  int64_t epoch_positions;  /* positions of the current epoch (N, or local_rows when local) */
  int32_t exchange_cast;    /* 1: this rank keeps a cast exchange copy of its HBM rows that the
                               peers read instead of the fp32 records (W > 1, see below) */
  int32_t storage_mode;     /* 0: no file tier; 1: file tier with O_DIRECT reads; 2: buffered reads */
  int64_t storage_bytes_read; /* bytes read from the hop files so far (aligned extents included) */
  /* ABI 6 */
  int64_t pdl_launches;     /* batch launches chained to the previous one by programmatic dependent
                               launch so far (a launch rewriting a slot the chain writes is not) */
  int32_t all_to_all;       /* 1: steps are exchanged by the all-to-all path (PP_PEERS_NCCL, or
                               PP_PEERS_LOOPBACK with PPLOAD_EXCHANGE=a2a) */
  int32_t spill_shared;     /* 1: the spill is a shared-memory file the peers map (PP_PEERS_IPC) */
  int64_t hbm_store_bytes;  /* memory plan: HBM part of the store (0 if borrowed) */
  int64_t hbm_exchange_bytes; /* exchange copy (cast rows for the peers) */
  int64_t hbm_scratch_bytes;  /* order buffers, sort scratch, exchange buffers allocated so far */
  int64_t host_spill_bytes;   /* pinned host spill */
} pp_loader_info;

/* Create a loader.  Copies the hop data into a library-owned, node-major store
 * [local_rows, H, F] (HBM part + optional pinned-host spill; only the node
 * set's records with store_set_only; no store but the opened hop files with
 * PP_MEM_FILES), uploads node_set / labels, and creates the loader stream.
 * Synchronous.  *out is NULL on error.
 * Errors: PP_ERR_INVALID (null/out-of-range fields, node_set id out of range,
 * unsupported dtype pair, IPC sharding with spill, unreadable / short hop
 * files, store_set_only without a node set), PP_ERR_OOM, PP_ERR_CUDA. */
pp_status pp_loader_create(const pp_loader_desc* desc, pp_loader** out);

/* Release everything the handle owns (store, spill, order, streams, peer
 * mappings).  Waits for the handle's outstanding work.  NULL is a no-op. */
pp_status pp_loader_destroy(pp_loader* L);

/* Start an epoch: compute order[] on the device from (seed, chunk) and reset
 * the cursor to step 0.  1 <= chunk <= N (chunk = 1: SGD-RR; chunk = c:
 * chunk reshuffling).  Runs on the loader stream after all work
 * enqueued on `stream` so far; later pp_next_batch calls are ordered after it.
 * Collective for W > 1: every rank passes the same (seed, chunk).  With
 * PP_PEERS_IPC each rank posts a hash of (seed, chunk) with a sequence number
 * into its IPC-mapped flag word and reads every peer's (blocking until all
 * ranks have called, PPLOAD_COLLECTIVE_TIMEOUT_S, default 300 s); with
 * PP_PEERS_NCCL the hash is all-reduced.  Differing arguments return
 * PP_ERR_INVALID on every rank and leave the previous epoch in place.
 * PP_PEERS_NCCL also derives the epoch's per-step send / receive counts from
 * the order here (one [steps][W][W] table, copied to the host).
 * Errors: PP_ERR_INVALID (chunk out of range, arguments differ across ranks),
 * PP_ERR_STATE (peers did not arrive in time), PP_ERR_CUDA, PP_ERR_NCCL. */
pp_status pp_epoch_permute(pp_loader* L, uint64_t seed, int64_t chunk, void* stream);

/* Locality-aware alternative for sharded loaders ("data
 * loader fetching data in a locality-aware manner"): this rank
 * shuffles only the local_rows nodes it owns (local row lr = global node
 * lr*W + rank), with the same Philox argsort and chunk rules over local
 * positions, and its batches are slices [tB, min((t+1)B, local_rows)) of that
 * order -- every row comes from local HBM, no peer traffic.  Not collective;
 * results depend on W (each rank sees only its shard).  Requires no node set.
 * steps_per_epoch (pp_loader_query) becomes ceil(local_rows / B) until the
 * next pp_epoch_permute.  Errors: PP_ERR_INVALID (chunk, node set), PP_ERR_CUDA. */
pp_status pp_epoch_permute_local(pp_loader* L, uint64_t seed, int64_t chunk, void* stream);

/* Compute the order of a FUTURE epoch now, on a library side stream, so that
 * it overlaps the current epoch's batches (the per-epoch shuffle runs "at the
 * start of each epoch"; prefetching it is the double-buffer idea
 * of PAPER.md:262 applied to the order).  The next pp_epoch_permute with the
 * same (seed, chunk) only switches to the prefetched order; a permute with
 * other arguments discards it.  At most one prefetch is pending (a second call
 * replaces the first).  Errors: PP_ERR_INVALID (chunk), PP_ERR_CUDA. */
pp_status pp_epoch_prefetch(pp_loader* L, uint64_t seed, int64_t chunk);

/* Assemble this rank's batch of the current step into `out` and advance the
 * cursor.  out: device, [B][H][F] of out_dtype, contiguous, caller-owned,
 * 16-byte aligned for the vector path.  out_labels: device int32 [B] or NULL
 * (must be NULL if the loader has no labels).  out_nodes: device int64 [B] or
 * NULL (global node ids).  *rows receives the rows written (< B only in the
 * last step; may be 0 on high ranks of the last step for W > 1).
 * Stream semantics: `out` is written after all work enqueued on
 * consumer_stream before this call, and is valid for work enqueued on
 * consumer_stream after it.  This orders the batch simply but cannot overlap
 * it with the consumer: the call both waits for and is waited on by the same
 * point of consumer_stream.  For the paper's double buffer (PAPER.md:262-263:
 * batch t+1 assembled while the consumer works on batch t) use
 * pp_next_batches_ev with per-buffer events.
 * When consumer_stream is the loader stream (pp_set_stream), consecutive
 * batches of one epoch may execute concurrently (programmatic dependent
 * launch); the library only chains a launch whose out / labels / node-id
 * ranges do not overlap those of the launches it would run beside, so a
 * reused slot serialises instead of racing.
 * Errors: PP_ERR_STATE (no permute yet), PP_END_OF_EPOCH (*rows = 0),
 * PP_ERR_INVALID, PP_ERR_CUDA. */
pp_status pp_next_batch(pp_loader* L, void* out, int32_t* out_labels, int64_t* out_nodes,
                        int32_t* rows, void* consumer_stream);

/* Assemble the next n steps in ONE launch: step i goes to
 * out + i*out_stride_bytes (and labels/nodes + i*B elements when non-NULL);
 * rows[i] receives its row count.  Stops early at the end of the epoch
 * (*n_done < n).  Same semantics as n calls of pp_next_batch; a k-slot ring
 * of prefetched batches.  Errors as pp_next_batch (PP_END_OF_EPOCH only if
 * no step remains). */
pp_status pp_next_batches(pp_loader* L, int32_t n, void* out, int64_t out_stride_bytes,
                          int32_t* out_labels, int64_t* out_nodes, int32_t* rows,
                          int32_t* n_done, void* consumer_stream);

/* pp_next_batches with explicit events instead of a consumer stream -- the
 * double buffer.  wait_event (cudaEvent_t or NULL): the
 * assembly waits for it before writing `out` (record it on the consumer's stream
 * after the consumer's last use of these slots).  ready_event (cudaEvent_t or
 * NULL): recorded on the loader stream once the slots are written; the consumer
 * waits for it before reading them.  With two buffers A/B the loop is
 *   next(A, wait=NULL, ready=rA)
 *   for t: next(other, wait=free[other], ready=r[other]);  consumer: wait r[cur],
 *          step(cur), record free[cur]
 * so batch t+1 is assembled while step t runs.  Other semantics (cursor, rows,
 * n_done, errors) as pp_next_batches. */
pp_status pp_next_batches_ev(pp_loader* L, int32_t n, void* out, int64_t out_stride_bytes, int32_t* out_labels,
                             int64_t* out_nodes, int32_t* rows, int32_t* n_done, void* wait_event,
                             void* ready_event);

/* Consumer fusion: assemble the next n steps AND apply
 * SIGN's per-hop linear layer ("learns R+1 weight matrices for each hop",
 * PAPER.md:184-185) in one tensor-core kernel:
 *   Z[j, k, :] = bf16_rne(X_k[v_j, :]) @ W_k      (fp32 accumulation)
 * The batch itself is never written to memory.
 * X_k is the batch the loader would produce: fp32 records cast to the batch
 * dtype (bf16 / f16, RNE), 16-bit records as they are.
 *   W: device [H][F][D] row-major in the batch dtype (W_k = W[k] is F x D),
 *      16-B aligned.
 *   D: 256 or 512.  F % 4 == 0 for fp32 records, F % 8 == 0 for 16-bit ones;
 *      any placement (HBM, spilled, sharded W > 1, compact store).  Every
 *      call takes the K-chunked kernel (PPLOAD_LINEAR=res selects the round-1
 *      W-resident kernel for fp32 -> bf16 HBM stores with F <= 128, W == 1),
 *      which runs as CTA pairs (tcgen05 cta_group::2, clusters of two) when the A
 *      chunks come by TMA (an unsharded, HBM-resident store; PPLOAD_LINEAR_PAIR
 *      = 0 / 1 forces single CTAs / pairs).  Results are identical either way
 *      up to fp32 accumulation order.
 *   Z: device [n][B][H][D] of z_dtype (PP_BF16: RNE from fp32, or PP_F32),
 *      slot pitch z_stride_bytes (>= B*H*D*elem when n > 1), 16-B aligned.
 * W is read by TMA at every launch (nothing is cached across calls), so it may
 * change between calls (an optimizer step).
 * Cursor, rows[], n_done and stream semantics as pp_next_batches; in
 * particular, calls issued back to back with consumer_stream == the loader
 * stream may overlap (programmatic dependent launch), so give each such call
 * its own Z slots or put the work that consumes / rewrites them between calls.
 * Errors: PP_ERR_INVALID (unsupported loader or shapes), PP_ERR_STATE,
 * PP_END_OF_EPOCH, PP_ERR_CUDA. */
pp_status pp_next_batches_linear(pp_loader* L, int32_t n, const void* W, int32_t D, void* Z, pp_dtype z_dtype,
                                 int64_t z_stride_bytes, int32_t* rows, int32_t* n_done, void* consumer_stream);

/* Pre-propagation on the GPU (Eq. (2)):
 * hops[k] = B hops[k-1] for k = 1..K, hops[0] = X, with the SGC/SIGN/HOGA
 * operator B = D~^{-1/2} (I + A) D~^{-1/2}.
 *   row_ptr: device int64 [n+1], col_idx: device int64 [nnz] -- CSR of
 *            A~ = I + A: symmetric, exactly one diagonal entry per row,
 *            columns ascending within a row (d~_i = row length).
 *   X:    device fp32 [n][F] row-major; hops: device fp32 [K+1][n][F].
 * Arithmetic: w_ij = 1/sqrt(d~_i d~_j) in fp64, row sums in ascending column
 * order in fp64 with separately rounded products and sums, one RNE rounding
 * to fp32 per output (bit-identical to the CPU reference definition).
 * Enqueued on `stream`; temporary fp64 weights (8 B per nonzero) are
 * allocated stream-ordered.  Reads row_ptr[n] synchronously.
 * Errors: PP_ERR_INVALID (n < 1, F not in [1, 256], K < 0, NULL pointers),
 * PP_ERR_OOM, PP_ERR_CUDA. */
pp_status pp_propagate(int64_t n, int32_t F, const int64_t* row_ptr, const int64_t* col_idx, const float* X,
                       int32_t K, float* hops, void* stream);

/* Pre-propagation INTO the loader's store, one hop per call (SURVEY.md
 * §8(f)-2, the multi-GPU 1D-partitioned SpMM; Eq. (2), PAPER.md:158-167,
 * operator PAPER.md:182): for every node i this rank owns (local row lr,
 * global id i = lr*W + rank)
 *   store[lr][k][:] = sum_{j in row i, ascending j} w_ij * X_{k-1}[j][:],
 *   w_ij = 1/sqrt(d~_i d~_j),
 * where X_{k-1}[j] is hop slot k-1 of node j's record in its OWNER's store
 * (owner j mod W, local row j div W): local HBM, the pinned spill, or a peer's
 * HBM over NVLink (PP_PEERS_IPC / PP_PEERS_LOOPBACK, after linking).  Same
 * arithmetic as pp_propagate: bit-identical to the CPU reference definition.
 * So hop 0 (X) given at create -- e.g. hop_stride = 0 with data = X broadcasts
 * X into every slot -- plus K calls k = 1..K turn the store into the
 * pre-propagated input without a hop-major copy of the K+1 matrices.  When the
 * rank keeps an exchange copy (pp_loader_info.exchange_cast) its slot k is
 * rewritten with the cast in the same kernel.
 *   k:       hop slot to write, 1 <= k < H (slot k-1 is read).
 *   row_ptr: device int64 [local_rows + 1], col_idx: device int64 [nnz]:
 *            the CSR rows of A~ = I + A for this rank's nodes in local-row
 *            order, GLOBAL column ids ascending within a row, each row
 *            holding its diagonal entry.
 *   deg:     device int32 [N_total]: d~_j (row length of A~) of every node;
 *            deg[i] must equal the length of i's row here.
 * Requires an fp32 store, F <= 256.  Enqueued on `stream`, ordered after the
 * loader's earlier work, and the loader's later work is ordered after it.
 * W > 1: hop k reads every owner's slot k-1, so all ranks must have finished
 * hop k-1 first (the caller synchronises `stream` and barriers between hops;
 * loopback shards sharing one `stream` are ordered by it).
 * Errors: PP_ERR_INVALID (k, dtype, F, NULL pointers), PP_ERR_STATE (not
 * linked), PP_ERR_CUDA. */
pp_status pp_propagate_store(pp_loader* L, int32_t k, const int64_t* row_ptr, const int64_t* col_idx,
                             const int32_t* deg, void* stream);

/* Move the cursor to step t (0 <= t <= steps_per_epoch): resume support.
 * (seed, chunk, cursor) is the loader's whole epoch state. */
pp_status pp_seek(pp_loader* L, int64_t step);

/* Use `stream` as the loader stream (default: a library-created non-blocking
 * stream).  When consumer_stream == loader stream, no events are recorded. */
pp_status pp_set_stream(pp_loader* L, void* stream);

/* Cap the batch-assembly grid at max_ctas CTAs (0: the full persistent grid,
 * default).  A loader whose batches overlap a consumer on the same GPU (the
 * double buffer, pp_next_batches_ev) otherwise takes every SM while it runs;
 * a PCIe-bound (host-resident) gather needs only a few CTAs to keep the link
 * busy.  Applies to later pp_next_batch / pp_next_batches(_ev) calls.
 * Errors: PP_ERR_INVALID (max_ctas < 0). */
pp_status pp_set_grid_limit(pp_loader* L, int32_t max_ctas);

pp_status pp_loader_query(const pp_loader* L, pp_loader_info* info);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char* pp_last_error(void);

int32_t pp_abi_version(void);

/* Bytes of the expanded PP-GNN input: N * F * elem_bytes * num_ops * (R + 1)
 * ("the input feature size is expanded to K(R+1) times"). */
int64_t pp_footprint_bytes(int64_t num_nodes, int32_t feat_dim, int32_t elem_bytes,
                           int32_t num_ops, int32_t num_hops_R);

/* ---- multi-GPU plumbing (W > 1) ------------------------------------------ */

/* Exchange copy (W > 1, fp32 store -> 16-bit batches).  Each rank keeps, next
 * to its fp32 shard, a copy of its HBM rows already cast to the batch dtype
 * (the same RNE cast as the gather, written at create and by
 * pp_fill_synthetic).  Peers read a remote row from that copy, so NVLink
 * carries H*F*s_out bytes per remote row -- the cast-before-transfer traffic
 * of an owner-side push -- while local rows are still read
 * in fp32 and cast inside the gather.  It costs s_out/s_in of the shard in
 * HBM; a rank that cannot fit it (or runs with PPLOAD_EXCHANGE_CAST=0) simply
 * exports none and its peers pull its fp32 records.  Batches are bit-identical
 * either way (pp_loader_info.exchange_cast reports the choice).
 *
 * PP_PEERS_IPC: write this rank's handle (PP_IPC_HANDLE_BYTES opaque bytes:
 * the store and, if present, the exchange copy) to handle_out; the caller
 * all-gathers the W handles (e.g. torch.distributed) and passes them,
 * rank-ordered, to pp_import_peer_stores on every rank. */
pp_status pp_export_store(pp_loader* L, void* handle_out);
/* The handle carries: the store's and the exchange copy's CUDA IPC handles, the
 * IPC handle of the rank's collective flag words (pp_epoch_permute), the number
 * of HBM rows, and -- when the rank spills -- the process id and descriptor of
 * its shared spill file, which every peer maps and registers at import (so the
 * importing ranks must run on the same host, as CUDA IPC already requires). */
pp_status pp_import_peer_stores(pp_loader* L, const void* handles /* W*PP_IPC_HANDLE_BYTES bytes */);

/* PP_PEERS_LOOPBACK: link W handles of one process (same device), rank-ordered. */
pp_status pp_link_loopback(pp_loader* const* loaders, int32_t world_size);

/* PP_PEERS_NCCL: write a fresh NCCL unique id (PP_NCCL_ID_BYTES) to out; one rank
 * calls it and broadcasts the bytes.  libnccl.so.2 is loaded on first use (the
 * copy already in the process, else PPLOAD_NCCL_LIB, else the system one).
 * Errors: PP_ERR_INVALID (NULL), PP_ERR_NCCL (library missing / failure). */
pp_status pp_nccl_unique_id(void* out);

/* ---- test / bench only ---------------------------------------------------- */

/* Fill this rank's store in place with the §8(d) generator (G for F32, G16
 * for F16): elem(k, v, f) is a pure function of (data_seed, k, v, f), v the
 * GLOBAL node id.  Synchronous. */
pp_status pp_fill_synthetic(pp_loader* L, uint64_t data_seed);

/* Copy the current epoch's order as global node ids (int64, N entries, after
 * node-set mapping) to host memory.  Synchronous.  PP_ERR_STATE before the
 * first permute. */
pp_status pp_get_order(pp_loader* L, int64_t* dst_host);

/* Copy store rows [row0, row0+n) of this rank (local row ids, node-major
 * records of record_bytes_in each) to host memory.  Synchronous. */
pp_status pp_read_store(pp_loader* L, int64_t row0, int64_t n, void* dst_host);

/* Test knob: shift the permutation's bucket count by `delta` bits (negative
 * = fewer, larger buckets) so the large-bucket path is exercised. */
pp_status pp_debug_set_sort_bits_delta(pp_loader* L, int32_t delta);

#ifdef __cplusplus
}
#endif
#endif /* PP_LOADER_H */
