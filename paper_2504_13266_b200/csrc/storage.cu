// Storage tier (the paper's "Direct Storage Access",
// PAPER.md:272-279, and its storage placement): hop features
// that exceed host memory stay in files -- one file per hop, "we split input
// features of different hops into separate files, enabling parallel storage
// access requests" -- and each step's rows are read from
// storage, then assembled into the batch on the GPU.
//
// Per step (positions [p0, p0 + rows) of the epoch order):
//   1. plan: node ids v_j, maximal runs of consecutive ids (one run per chunk
//      with chunk reshuffling: "reading chunks from the storage system is
//      significantly more efficient compared to reading individual node
//      features"), each run's byte range widened to the
//      direct-I/O alignment;
//   2. read: every (hop file, run) cut into <= 1 MiB pieces, spread over a
//      pool of I/O threads (pread into a pinned staging slot), O_DIRECT so
//      storage -- not the page cache -- is measured (the DMA-through-a-bounce-
//      buffer data path GDS itself uses without nvidia-fs);
//   3. H2D: one DMA of the slot on the loader stream;
//   4. assemble: k_assemble_staged casts each staged row into out[j][k][:]
//      (the gather's RNE cast), plus labels / node ids.
// PPLOAD_IO_DEPTH (default 4) staging slots: while the GPU consumes step t,
// the I/O threads already read steps t+1 .. t+3 (the paper's double-buffer
// prefetch, made deeper so the device queue stays full).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

namespace ppl {

namespace {

constexpr int64_t kAlign = 4096;  // direct-I/O alignment (offset, size, buffer)

enum { kF32 = 0, kBF16 = 1, kF16 = 2 };

__device__ __forceinline__ uint16_t cast16(float x, int out_dtype) {
  if (out_dtype == kBF16) {
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    return *reinterpret_cast<const uint16_t*>(&h);
  }
  const __half h = __float2half_rn(x);
  return *reinterpret_cast<const uint16_t*>(&h);
}

// out[j][k][f] = cast(stage[k * region + row_src[j] + f * s_in]).
// Vector form: 4 elements per thread-op (16-B fp32 loads -> 8-B 16-bit stores,
// or 16-B copies of 16-bit / fp32 data); VEC requires F % 4 == 0 and 16-byte
// aligned staged rows (F * s_in % 16 == 0).
template <bool VEC>
__global__ void __launch_bounds__(256) k_assemble_staged(const uint8_t* __restrict__ stage, int64_t region,
                                                         const int64_t* __restrict__ row_src,
                                                         const int64_t* __restrict__ nodes, int32_t rows, int32_t H,
                                                         int32_t F, int32_t in_dtype, int32_t out_dtype,
                                                         uint8_t* __restrict__ out, const int32_t* __restrict__ labels,
                                                         int32_t* __restrict__ out_labels, int64_t* __restrict__ out_nodes) {
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t j = tid; j < rows; j += nthr) {
    if (out_nodes) out_nodes[j] = nodes[j];
    if (out_labels) out_labels[j] = labels[nodes[j]];
  }
  const int s_in = in_dtype == kF32 ? 4 : 2, s_out = out_dtype == kF32 ? 4 : 2;
  const bool cast = in_dtype == kF32 && out_dtype != kF32;
  const int per = VEC ? 4 : 1;
  const int units = F / per;
  const int64_t total = static_cast<int64_t>(rows) * H * units;
  for (int64_t i = tid; i < total; i += nthr) {
    const int u = static_cast<int>(i % units);
    const int64_t jk = i / units;
    const int k = static_cast<int>(jk % H);
    const int64_t j = jk / H;
    const uint8_t* src = stage + k * region + row_src[j] + static_cast<int64_t>(u) * per * s_in;
    uint8_t* dst = out + (jk * F + static_cast<int64_t>(u) * per) * s_out;
    if (VEC) {
      if (cast) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(src));
        uint2 y;
        y.x = static_cast<uint32_t>(cast16(x.x, out_dtype)) | (static_cast<uint32_t>(cast16(x.y, out_dtype)) << 16);
        y.y = static_cast<uint32_t>(cast16(x.z, out_dtype)) | (static_cast<uint32_t>(cast16(x.w, out_dtype)) << 16);
        *reinterpret_cast<uint2*>(dst) = y;
      } else if (s_in == 4) {
        *reinterpret_cast<uint4*>(dst) = __ldg(reinterpret_cast<const uint4*>(src));
      } else {
        *reinterpret_cast<uint2*>(dst) = __ldg(reinterpret_cast<const uint2*>(src));
      }
    } else {
      if (cast) {
        *reinterpret_cast<uint16_t*>(dst) = cast16(__ldg(reinterpret_cast<const float*>(src)), out_dtype);
      } else if (s_in == 4) {
        *reinterpret_cast<uint32_t*>(dst) = __ldg(reinterpret_cast<const uint32_t*>(src));
      } else {
        *reinterpret_cast<uint16_t*>(dst) = __ldg(reinterpret_cast<const uint16_t*>(src));
      }
    }
  }
}

struct Piece {
  int hop;
  int64_t file_off, bytes, stage_off;
};

struct Run {
  int64_t file_off;  // aligned file offset of the read
  int64_t bytes;     // aligned length
  int64_t stage_off; // offset inside a hop region (aligned)
};

// One staging slot: pinned host [meta | hop 0 region | hop 1 region | ...],
// and its device twin.  meta = row_src[B] int64 + nodes[B] int64.
struct Slot {
  uint8_t* h = nullptr;
  uint8_t* d = nullptr;
  cudaEvent_t ev_h2d = nullptr;  // the H2D out of h has completed
  bool h2d_pending = false;      // written by the caller thread before the next plan job is submitted
  int64_t step = -1;             // step staged (or being staged) in it; -1: none
  uint64_t epoch = 0;
  int32_t rows = 0;
  int64_t region_used = 0;
  std::vector<Run> runs;
  std::vector<Piece> pieces;
  std::mutex mu;
  std::condition_variable cv;
  int jobs_left = 0;  // plan job + piece jobs still running
  std::string err;
};

}  // namespace

struct FileTier {
  int dev = 0;
  int H = 0, F = 0;
  int64_t N_total = 0, B = 0;
  int s_in = 4;
  int64_t rb = 0;  // bytes of one row in a hop file
  std::vector<int> fds;
  bool direct = true;
  int64_t meta_bytes = 0, region_cap = 0;
  std::vector<std::unique_ptr<Slot>> slots;  // PPLOAD_IO_DEPTH steps staged ahead (default 4)
  int nthreads = 16;                         // PPLOAD_IO_THREADS
  int64_t piece_bytes = int64_t(1) << 20;    // PPLOAD_IO_PIECE
  // current epoch (set_epoch): positions -> node ids, slicing
  uint64_t epoch = 0;
  const uint32_t* order = nullptr;
  const int64_t* node_set = nullptr;
  int64_t N = 0, steps = 0;
  int32_t W = 1, rank = 0;
  std::vector<std::thread> workers;
  std::mutex qmu;
  std::condition_variable qcv;
  std::deque<std::function<void()>> queue;
  bool stop = false;
  std::atomic<int64_t> bytes_read{0};

  ~FileTier() {
    for (auto& s : slots) wait_reads(*s);
    {
      std::lock_guard<std::mutex> lk(qmu);
      stop = true;
    }
    qcv.notify_all();
    for (auto& t : workers) t.join();
    for (int fd : fds)
      if (fd >= 0) close(fd);
    for (auto& s : slots) {
      if (s->h) cudaFreeHost(s->h);
      if (s->d) cudaFree(s->d);
      if (s->ev_h2d) cudaEventDestroy(s->ev_h2d);
    }
  }

  void worker() {
    cudaSetDevice(dev);
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(qmu);
        qcv.wait(lk, [&] { return stop || !queue.empty(); });
        if (stop && queue.empty()) return;
        job = std::move(queue.front());
        queue.pop_front();
      }
      job();
    }
  }

  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(qmu);
      queue.push_back(std::move(f));
    }
    qcv.notify_one();
  }

  bool alloc_slots(int64_t cap, std::string* err) {
    for (auto& s : slots) {
      if (s->h) cudaFreeHost(s->h);
      if (s->d) cudaFree(s->d);
      s->h = nullptr;
      s->d = nullptr;
    }
    region_cap = cap;
    const size_t bytes = static_cast<size_t>(meta_bytes + H * region_cap);
    for (auto& s : slots) {
      if (cudaHostAlloc(&s->h, bytes, cudaHostAllocPortable) != cudaSuccess || cudaMalloc(&s->d, bytes) != cudaSuccess) {
        *err = "staging allocation of " + std::to_string(bytes) + " bytes failed";
        return false;
      }
    }
    return true;
  }

  std::string wait_reads(Slot& s) {
    std::unique_lock<std::mutex> lk(s.mu);
    s.cv.wait(lk, [&] { return s.jobs_left == 0; });
    return s.err;
  }

  // rows of `step` and the node id of its j-th row
  int32_t step_rows(int64_t step) const {
    const int64_t p0 = step * B * W + static_cast<int64_t>(rank) * B;
    return static_cast<int32_t>(std::max<int64_t>(0, std::min<int64_t>(B, N - p0)));
  }
  int64_t node_at(int64_t step, int32_t j) const {
    const uint32_t o = order[step * B * W + static_cast<int64_t>(rank) * B + j];
    return node_set ? node_set[o] : static_cast<int64_t>(o);
  }

  // Runs of consecutive node ids of `step`, each widened to the direct-I/O
  // alignment; fills row_src / nodes when given; returns the staged bytes per hop.
  int64_t plan(int64_t step, std::vector<Run>* runs, int64_t* row_src, int64_t* nodes) const {
    const int32_t rows = step_rows(step);
    int64_t off = 0;
    int64_t v_prev = -2;
    int64_t b0 = 0, a0 = 0, j0 = 0;
    auto close_run = [&](int32_t j_end, int64_t v_last) {
      const int64_t b1 = v_last * rb + rb;
      const int64_t a1 = (b1 + kAlign - 1) / kAlign * kAlign;
      if (runs) runs->push_back(Run{a0, a1 - a0, off});
      if (row_src)
        for (int32_t i = static_cast<int32_t>(j0); i < j_end; ++i) row_src[i] = off + (b0 - a0) + (i - j0) * rb;
      off += a1 - a0;
    };
    for (int32_t j = 0; j < rows; ++j) {
      const int64_t v = node_at(step, j);
      if (nodes) nodes[j] = v;
      if (j > 0 && v == v_prev + 1) {
        v_prev = v;
        continue;
      }
      if (j > 0) close_run(j, v_prev);
      b0 = v * rb;
      a0 = b0 / kAlign * kAlign;
      j0 = j;
      v_prev = v;
    }
    if (rows > 0) close_run(rows, v_prev);
    return off;
  }

  // Stage `step` of the current epoch into its slot (step mod depth): a plan job
  // (waits for the slot's previous DMA, writes meta, cuts pieces) then piece jobs.
  void dispatch(int64_t step) {
    Slot& s = *slots[step % static_cast<int64_t>(slots.size())];
    wait_reads(s);
    s.step = step;
    s.epoch = epoch;
    s.err.clear();
    {
      std::lock_guard<std::mutex> lk(s.mu);
      s.jobs_left = 1;
    }
    Slot* sp = &s;
    const bool pending = s.h2d_pending;
    s.h2d_pending = false;
    submit([this, sp, step, pending] {
      std::string e;
      if (pending && cudaEventSynchronize(sp->ev_h2d) != cudaSuccess) e = "staging event wait failed";
      int njobs = 0;
      int64_t np_ = 0;
      if (e.empty()) {
        sp->runs.clear();
        sp->rows = step_rows(step);
        int64_t* row_src = reinterpret_cast<int64_t*>(sp->h);
        sp->region_used = plan(step, &sp->runs, row_src, row_src + B);
        // pieces: every (hop file, run), long runs cut into <= piece_bytes requests so that
        // all I/O threads (and the device's queue) stay busy even with a few large chunks
        sp->pieces.clear();
        for (int k = 0; k < H; ++k)
          for (const Run& run : sp->runs)
            for (int64_t o = 0; o < run.bytes; o += piece_bytes)
              sp->pieces.push_back(Piece{k, run.file_off + o, std::min(piece_bytes, run.bytes - o), run.stage_off + o});
        np_ = static_cast<int64_t>(sp->pieces.size());
        njobs = static_cast<int>(std::min<int64_t>(nthreads, np_));
      }
      {
        std::lock_guard<std::mutex> lk(sp->mu);
        sp->jobs_left += njobs;
      }
      for (int jb = 0; jb < njobs; ++jb) {
        // interleaved: job jb takes pieces jb, jb + njobs, ... (spreads hops and offsets)
        submit([this, sp, jb, njobs, np_] {
          std::string err;
          int64_t got_total = 0;
          for (int64_t i = jb; i < np_ && err.empty(); i += njobs) {
            const Piece& pc = sp->pieces[i];
            uint8_t* region = sp->h + meta_bytes + pc.hop * region_cap;
            int64_t done = 0;
            while (done < pc.bytes) {
              const ssize_t got = pread(fds[pc.hop], region + pc.stage_off + done, pc.bytes - done, pc.file_off + done);
              if (got < 0) {
                if (errno == EINTR) continue;
                err = std::string("pread: ") + strerror(errno);
                break;
              }
              if (got == 0) break;  // end of file inside the last aligned block
              done += got;
            }
            got_total += done;
          }
          bytes_read += got_total;
          std::lock_guard<std::mutex> lk(sp->mu);
          if (!err.empty() && sp->err.empty()) sp->err = err;
          if (--sp->jobs_left == 0) sp->cv.notify_all();
        });
      }
      std::lock_guard<std::mutex> lk(sp->mu);
      if (!e.empty() && sp->err.empty()) sp->err = e;
      if (--sp->jobs_left == 0) sp->cv.notify_all();
    });
  }

  bool staged(int64_t step) const {
    const Slot& s = *slots[step % static_cast<int64_t>(slots.size())];
    return s.step == step && s.epoch == epoch;
  }

  void reset() {
    for (auto& s : slots) {
      wait_reads(*s);
      s->err.clear();
      s->step = -1;
    }
  }
};

FileTier* file_tier_open(const char* const* paths, int H, int64_t N_total, int F, int s_in, int64_t B, int dev,
                         std::string* err) {
  FileTier* T = new FileTier();
  T->dev = dev;
  T->H = H;
  T->F = F;
  T->N_total = N_total;
  T->B = B;
  T->s_in = s_in;
  T->rb = static_cast<int64_t>(F) * s_in;
  const char* e = getenv("PPLOAD_IO_DIRECT");
  T->direct = !(e && !strcmp(e, "0"));
  if (const char* t = getenv("PPLOAD_IO_THREADS")) T->nthreads = std::max(1, atoi(t));
  if (const char* t = getenv("PPLOAD_IO_PIECE")) T->piece_bytes = std::max<int64_t>(kAlign, atoll(t) / kAlign * kAlign);
  int depth = 4;
  if (const char* t = getenv("PPLOAD_IO_DEPTH")) depth = std::max(2, std::min(64, atoi(t)));
  for (int i = 0; i < depth; ++i) T->slots.emplace_back(new Slot());
  for (int k = 0; k < H; ++k) {
    if (!paths[k]) {
      *err = "hop file path " + std::to_string(k) + " is NULL";
      delete T;
      return nullptr;
    }
    int fd = T->direct ? open(paths[k], O_RDONLY | O_DIRECT) : -1;
    if (fd < 0 && T->direct && k == 0) T->direct = false;  // no direct I/O here (e.g. tmpfs): buffered reads
    if (fd < 0) fd = open(paths[k], O_RDONLY);
    if (fd < 0) {
      *err = std::string("open(") + paths[k] + "): " + strerror(errno);
      delete T;
      return nullptr;
    }
    T->fds.push_back(fd);
    struct stat st;
    if (fstat(fd, &st) != 0 || st.st_size < N_total * T->rb) {
      *err = std::string(paths[k]) + ": file holds fewer than N_total * F elements";
      delete T;
      return nullptr;
    }
    // Headerless raw [N_total][F] only: a file with the PPGF container header (magic, version,
    // data offset, per-chunk padding) would be misread row by row, so it is refused.
    char magic[4] = {0, 0, 0, 0};
    const int fd_probe = open(paths[k], O_RDONLY);  // buffered: O_DIRECT reads need aligned buffers
    const bool ppgf = fd_probe >= 0 && pread(fd_probe, magic, 4, 0) == 4 && !memcmp(magic, "PPGF", 4);
    if (fd_probe >= 0) close(fd_probe);
    if (ppgf) {
      *err = std::string(paths[k]) + ": PPGF container files are not supported (raw [N_total][F] hop files only)";
      delete T;
      return nullptr;
    }
  }
  if (!T->direct) {
    for (int k = 0; k < H; ++k) {  // all files the same way
      close(T->fds[k]);
      T->fds[k] = open(paths[k], O_RDONLY);
      posix_fadvise(T->fds[k], 0, 0, POSIX_FADV_RANDOM);
    }
  }
  T->meta_bytes = (16 * B + kAlign - 1) / kAlign * kAlign;
  for (auto& s : T->slots)
    if (cudaEventCreateWithFlags(&s->ev_h2d, cudaEventDisableTiming) != cudaSuccess) {
      *err = "event creation failed";
      delete T;
      return nullptr;
    }
  // a chunk-reshuffled step needs about B rows plus two aligned blocks per chunk (grown per epoch)
  if (!T->alloc_slots((B * T->rb + kAlign - 1) / kAlign * kAlign + 16 * kAlign, err)) {
    delete T;
    return nullptr;
  }
  for (int i = 0; i < T->nthreads; ++i) T->workers.emplace_back([T] { T->worker(); });
  return T;
}

void file_tier_close(FileTier* T) { delete T; }
bool file_tier_direct(const FileTier* T) { return T->direct; }
int64_t file_tier_bytes_read(const FileTier* T) { return T->bytes_read.load(); }
void file_tier_reset(FileTier* T) { T->reset(); }

bool file_tier_set_epoch(FileTier* T, uint64_t epoch, const uint32_t* order, const int64_t* node_set, int64_t N,
                         int32_t W, int32_t rank, int64_t steps, std::string* err) {
  T->reset();
  T->epoch = epoch;
  T->order = order;
  T->node_set = node_set;
  T->N = N;
  T->W = W;
  T->rank = rank;
  T->steps = steps;
  int64_t need = 0;  // the epoch's largest staged step per hop
  for (int64_t t = 0; t < steps; ++t) need = std::max(need, T->plan(t, nullptr, nullptr, nullptr));
  if (need > T->region_cap) {
    for (auto& s : T->slots)
      if (s->h2d_pending) {
        cudaEventSynchronize(s->ev_h2d);
        s->h2d_pending = false;
      }
    if (cudaDeviceSynchronize() != cudaSuccess) {  // device slots may still be read by kernels
      *err = "device sync before staging growth failed";
      return false;
    }
    if (!T->alloc_slots(need, err)) return false;
  }
  return true;
}

cudaError_t file_tier_step(FileTier* T, int64_t step, int32_t in_dtype, int32_t out_dtype, const int32_t* labels,
                           uint8_t* out, int32_t* out_labels, int64_t* out_nodes, bool out_vec, cudaStream_t st,
                           int32_t* rows, std::string* err) {
  const int64_t depth = static_cast<int64_t>(T->slots.size());
  if (!T->staged(step)) T->dispatch(step);
  for (int64_t d = step + 1; d < std::min(step + depth, T->steps); ++d)  // keep the window full
    if (!T->staged(d)) T->dispatch(d);
  Slot& cur = *T->slots[step % depth];
  const std::string re = T->wait_reads(cur);
  if (!re.empty()) {
    *err = re;
    cur.step = -1;
    return cudaErrorUnknown;
  }
  *rows = cur.rows;
  if (cur.rows > 0) {
    // meta + the used part of every hop region (one DMA each)
    cudaError_t e = cudaMemcpyAsync(cur.d, cur.h, 16 * T->B, cudaMemcpyHostToDevice, st);
    for (int k = 0; k < T->H && e == cudaSuccess; ++k) {
      const int64_t o = T->meta_bytes + k * T->region_cap;
      e = cudaMemcpyAsync(cur.d + o, cur.h + o, cur.region_used, cudaMemcpyHostToDevice, st);
    }
    if (e == cudaSuccess) e = cudaEventRecord(cur.ev_h2d, st);
    if (e != cudaSuccess) return e;
    cur.h2d_pending = true;
    // 4-element vectors need F % 4 == 0 and a 16-B aligned `out` / slot pitch (out_vec)
    const bool vec = out_vec && T->F % 4 == 0 && T->rb % 16 == 0;
    const int64_t units = static_cast<int64_t>(cur.rows) * T->H * (vec ? T->F / 4 : T->F);
    const uint32_t grid = static_cast<uint32_t>(std::min<int64_t>((units + 255) / 256, 148 * 16));
    const int64_t* row_src = reinterpret_cast<const int64_t*>(cur.d);
    const int64_t* nodes = row_src + T->B;
    if (vec)
      k_assemble_staged<true><<<grid, 256, 0, st>>>(cur.d + T->meta_bytes, T->region_cap, row_src, nodes, cur.rows,
                                                    T->H, T->F, in_dtype, out_dtype, out, labels, out_labels, out_nodes);
    else
      k_assemble_staged<false><<<grid, 256, 0, st>>>(cur.d + T->meta_bytes, T->region_cap, row_src, nodes, cur.rows,
                                                     T->H, T->F, in_dtype, out_dtype, out, labels, out_labels, out_nodes);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  cur.step = -1;  // consumed; the slot takes step + depth next
  if (step + depth < T->steps) T->dispatch(step + depth);
  return cudaSuccess;
}

}  // namespace ppl
