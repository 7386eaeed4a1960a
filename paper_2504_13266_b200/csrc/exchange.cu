// All-to-all exchange of batch rows over NCCL (the "NCCL (baseline)"
// variant, K9 of §2.3): "distributing data across multiple GPUs", owner(v) = v mod W.
//
// Every rank holds the same global order, so the rows owner o must send to rank d at step t, and
// their count n[t][d][o], follow from the order alone -- no count exchange:
//   1. k_a2a_counts (once per epoch): n[t][d][o] for every step, slice and owner (order pass,
//      warp-aggregated atomics); copied to the host, which sizes every send / receive with it.
//   2. k_a2a_index (per step, one CTA per destination slice d): a stable compaction of the slice's
//      positions by owner.  The sending rank writes the local rows it owns, slice by slice, into
//      send_rows (segment d at send_off[d]); for its own slice it writes, per position, where the
//      row will land in the receive buffer (recv_off[o] + rank within owner o) plus ids / labels.
//   3. pack: the loader's own gather kernel over send_rows (local HBM rows, cast fused), so the
//      link carries H*F*s_out bytes per row -- cast before the transfer.
//   4. ncclGroupStart; ncclSend(segment d) / ncclRecv(segment o) for every peer incl. self;
//      ncclGroupEnd -- on the loader stream.
//   5. k_a2a_unpack: out[j] = recv[recv_src[j]] (16-byte vectors).
// Batches are identical to the peer-read design and to the oracle (O9/O10): the exchange only
// moves already-cast rows.  PP_PEERS_LOOPBACK with PPLOAD_EXCHANGE=a2a runs steps 1-3 and 5 for
// every owner inside one process (each owner's pack writes straight into the receiver's buffer),
// so the index / pack / unpack logic is tested on one GPU without NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "internal.h"

namespace ppl {

__device__ __forceinline__ uint64_t row_space_index(const uint32_t* order, const int64_t* node_set, int64_t p) {
  uint64_t x = order[p];
  if (node_set != nullptr) x = static_cast<uint64_t>(node_set[x]);
  return x;
}

// n[t][d][o]: positions of slice d of step t whose row is owned by o.  One position per thread;
// lanes with the same (t, d, o) key add once (the order visits few distinct keys per warp).
__global__ void k_a2a_counts(const uint32_t* __restrict__ order, const int64_t* __restrict__ node_set, int64_t N,
                             int64_t steps, int32_t B, int32_t W, uint32_t* __restrict__ table) {
  const int64_t WB = static_cast<int64_t>(W) * B;
  const int64_t end = steps * WB < N ? steps * WB : N;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < end; base += stride) {
    const int64_t p = base + threadIdx.x;
    const bool valid = p < end;
    uint32_t key = 0xffffffffu;
    if (valid) {
      const uint64_t x = row_space_index(order, node_set, p);
      const int64_t t = p / WB;
      const int32_t d = static_cast<int32_t>((p - t * WB) / B);
      const int32_t o = static_cast<int32_t>(x % static_cast<uint64_t>(W));
      key = static_cast<uint32_t>((t * W + d) * W + o);
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    if (valid && static_cast<int>(threadIdx.x & 31) == leader) atomicAdd(&table[key], __popc(peers));
  }
}

cudaError_t launch_a2a_counts(const uint32_t* order, const int64_t* node_set, int64_t N, int64_t steps, int32_t B,
                              int32_t W, uint32_t* table, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(table, 0, static_cast<size_t>(steps) * W * W * 4, st);
  if (e != cudaSuccess || N <= 0) return e;
  const int64_t blocks = (N + 255) / 256 < 148 * 16 ? (N + 255) / 256 : 148 * 16;
  k_a2a_counts<<<static_cast<unsigned>(blocks), 256, 0, st>>>(order, node_set, N, steps, B, W, table);
  return cudaGetLastError();
}

constexpr int kIndexThreads = 1024;

// One CTA per destination slice d in [a.slice_lo, a.slice_hi).  Stable compaction by owner: the
// rank of position j among the slice's positions owned by o is the number of such positions before
// it (warp ballots + a per-owner scan over the 32 warps, carried across 1024-position rounds).
__global__ void __launch_bounds__(kIndexThreads) k_a2a_index(const A2AIndexArgs a) {
  __shared__ uint32_t s_tot[kIndexThreads / 32][kMaxWorld];
  __shared__ uint32_t s_run[kMaxWorld];
  const int d = a.slice_lo + static_cast<int>(blockIdx.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pos0 = a.step_pos0 + static_cast<int64_t>(d) * a.B;
  const int64_t nd64 = a.N - pos0 < a.B ? a.N - pos0 : a.B;
  const int32_t nd = nd64 > 0 ? static_cast<int32_t>(nd64) : 0;
  if (threadIdx.x < kMaxWorld) s_run[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  for (int32_t j0 = 0; j0 < nd; j0 += kIndexThreads) {
    const int32_t j = j0 + static_cast<int32_t>(threadIdx.x);
    const bool valid = j < nd;
    uint64_t x = 0;
    int o = -1;
    if (valid) {
      x = row_space_index(a.order, a.node_set, pos0 + j);
      o = static_cast<int>(x % static_cast<uint64_t>(a.W));
    }
    uint32_t mine = 0;
    for (int q = 0; q < a.W; ++q) {
      const uint32_t m = __ballot_sync(0xffffffffu, o == q);
      if (lane == 0) s_tot[warp][q] = __popc(m);
      if (o == q) mine = __popc(m & lt);
    }
    __syncthreads();
    if (valid) {
      uint32_t rank = s_run[o] + mine;
      for (int w = 0; w < warp; ++w) rank += s_tot[w][o];
      if (o == a.self) a.send_rows[a.send_off[d] + rank] = static_cast<uint32_t>(x / static_cast<uint64_t>(a.W));
      if (d == a.recv_rank) {
        a.recv_src[j] = static_cast<uint32_t>(a.recv_off[o] + rank);
        const uint64_t id = a.out_ids != nullptr ? static_cast<uint64_t>(a.out_ids[x]) : x;
        if (a.out_labels != nullptr) a.out_labels[j] = a.labels[id];
        if (a.out_nodes != nullptr) a.out_nodes[j] = static_cast<int64_t>(id);
      }
    }
    __syncthreads();
    if (threadIdx.x < static_cast<unsigned>(a.W)) {
      uint32_t s = 0;
      for (int w = 0; w < kIndexThreads / 32; ++w) s += s_tot[w][threadIdx.x];
      s_run[threadIdx.x] += s;
    }
    __syncthreads();
  }
}

cudaError_t launch_a2a_index(const A2AIndexArgs& a, cudaStream_t st) {
  if (a.slice_hi <= a.slice_lo) return cudaSuccess;
  k_a2a_index<<<a.slice_hi - a.slice_lo, kIndexThreads, 0, st>>>(a);
  return cudaGetLastError();
}

// out row j (rec_out bytes) = recv row recv_src[j]; 16-byte vectors when both sides allow it.
__global__ void k_a2a_unpack(const uint8_t* __restrict__ recv, const uint32_t* __restrict__ recv_src, int32_t rows,
                             int64_t rec_out, uint8_t* __restrict__ out, bool vec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vec) {
    const int64_t vpr = rec_out / 16;
    for (int64_t e = tid; e < rows * vpr; e += stride) {
      const int64_t j = e / vpr, c = e - j * vpr;
      reinterpret_cast<uint4*>(out + j * rec_out)[c] =
          reinterpret_cast<const uint4*>(recv + static_cast<int64_t>(recv_src[j]) * rec_out)[c];
    }
  } else {
    const int64_t hpr = rec_out / 2;
    for (int64_t e = tid; e < rows * hpr; e += stride) {
      const int64_t j = e / hpr, c = e - j * hpr;
      reinterpret_cast<uint16_t*>(out + j * rec_out)[c] =
          reinterpret_cast<const uint16_t*>(recv + static_cast<int64_t>(recv_src[j]) * rec_out)[c];
    }
  }
}

cudaError_t launch_a2a_unpack(const uint8_t* recv, const uint32_t* recv_src, int32_t rows, int64_t rec_out,
                              uint8_t* out, bool vec, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int64_t units = static_cast<int64_t>(rows) * (vec ? rec_out / 16 : rec_out / 2);
  const int64_t blocks = (units + 255) / 256 < 148 * 8 ? (units + 255) / 256 : 148 * 8;
  k_a2a_unpack<<<static_cast<unsigned>(blocks), 256, 0, st>>>(recv, recv_src, rows, rec_out, out, vec);
  return cudaGetLastError();
}

// ---- NCCL, loaded at run time (only loaders with PP_PEERS_NCCL need it) -------------------------
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the copy already in the process (e.g. loaded by torch) first, then PPLOAD_NCCL_LIB, then the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && getenv("PPLOAD_NCCL_LIB")) h = dlopen(getenv("PPLOAD_NCCL_LIB"), RTLD_NOW);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) {
      api.err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return;
    }
#define PPL_SYM(field, name)                                                  \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));          \
  if (!api.field) {                                                           \
    api.err = std::string("libnccl.so.2 lacks ") + name;                      \
    return;                                                                   \
  }
    PPL_SYM(GetUniqueId, "ncclGetUniqueId")
    PPL_SYM(CommInitRank, "ncclCommInitRank")
    PPL_SYM(CommDestroy, "ncclCommDestroy")
    PPL_SYM(CommAbort, "ncclCommAbort")
    PPL_SYM(CommGetAsyncError, "ncclCommGetAsyncError")
    PPL_SYM(Send, "ncclSend")
    PPL_SYM(Recv, "ncclRecv")
    PPL_SYM(GroupStart, "ncclGroupStart")
    PPL_SYM(GroupEnd, "ncclGroupEnd")
    PPL_SYM(AllReduce, "ncclAllReduce")
    PPL_SYM(GetErrorString, "ncclGetErrorString")
#undef PPL_SYM
    api.ok = true;
  });
  return api;
}

static std::string nccl_err(const NcclApi& api, ncclResult_t r, const char* what) {
  return std::string(what) + ": " + (api.GetErrorString ? api.GetErrorString(r) : "nccl error");
}

bool nccl_unique_id(void* out128, std::string* err) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  NcclApi& api = nccl_api();
  if (!api.ok) {
    *err = api.err;
    return false;
  }
  ncclUniqueId id;
  const ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) {
    *err = nccl_err(api, r, "ncclGetUniqueId");
    return false;
  }
  memcpy(out128, &id, sizeof(id));
  return true;
}

void* nccl_comm_create(const void* id128, int W, int rank, std::string* err) {
  NcclApi& api = nccl_api();
  if (!api.ok) {
    *err = api.err;
    return nullptr;
  }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t comm = nullptr;
  const ncclResult_t r = api.CommInitRank(&comm, W, id, rank);
  if (r != ncclSuccess) {
    *err = nccl_err(api, r, "ncclCommInitRank");
    return nullptr;
  }
  return comm;
}

void nccl_comm_destroy(void* comm, bool abort) {
  if (!comm) return;
  NcclApi& api = nccl_api();
  if (!api.ok) return;
  if (abort)
    api.CommAbort(static_cast<ncclComm_t>(comm));
  else
    api.CommDestroy(static_cast<ncclComm_t>(comm));
}

// Poll the communicator's asynchronous error state (NCCL reports transport failures there).
bool nccl_check_async(void* comm, std::string* err) {
  NcclApi& api = nccl_api();
  ncclResult_t st = ncclSuccess;
  const ncclResult_t r = api.CommGetAsyncError(static_cast<ncclComm_t>(comm), &st);
  if (r != ncclSuccess || (st != ncclSuccess && st != ncclInProgress)) {
    *err = nccl_err(api, r != ncclSuccess ? r : st, "NCCL asynchronous error");
    return false;
  }
  return true;
}

// One step's exchange: segment q of `send` to rank q, segment q of `recv` from rank q (bytes).
bool nccl_exchange(void* comm, int W, const uint8_t* send, const int64_t* send_off, const int64_t* send_bytes,
                   uint8_t* recv, const int64_t* recv_off, const int64_t* recv_bytes, cudaStream_t st,
                   std::string* err) {
  NcclApi& api = nccl_api();
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = api.GroupStart();
  for (int q = 0; q < W && r == ncclSuccess; ++q) {
    if (send_bytes[q] > 0) r = api.Send(send + send_off[q], static_cast<size_t>(send_bytes[q]), ncclUint8, q, c, st);
    if (r == ncclSuccess && recv_bytes[q] > 0)
      r = api.Recv(recv + recv_off[q], static_cast<size_t>(recv_bytes[q]), ncclUint8, q, c, st);
  }
  const ncclResult_t r2 = api.GroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess) {
    *err = nccl_err(api, r != ncclSuccess ? r : r2, "ncclSend/ncclRecv group");
    return false;
  }
  return nccl_check_async(comm, err);
}

// Collective check of an epoch's arguments: max over ranks of (h, -h) (int64) == (h, -h) on every
// rank iff all ranks passed the same hash.  `buf`: device int64[2].  Synchronous.
bool nccl_same_everywhere(void* comm, int64_t h, int64_t* buf, cudaStream_t st, bool* same, std::string* err) {
  NcclApi& api = nccl_api();
  int64_t hv[2] = {h, -h};
  cudaError_t ce = cudaMemcpyAsync(buf, hv, 16, cudaMemcpyHostToDevice, st);
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return false;
  }
  const ncclResult_t r = api.AllReduce(buf, buf, 2, ncclInt64, ncclMax, static_cast<ncclComm_t>(comm), st);
  if (r != ncclSuccess) {
    *err = nccl_err(api, r, "ncclAllReduce");
    return false;
  }
  int64_t got[2];
  ce = cudaMemcpyAsync(got, buf, 16, cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return false;
  }
  *same = got[0] == h && got[1] == -h;
  return nccl_check_async(comm, err);
}

}  // namespace ppl
