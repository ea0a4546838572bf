// bmg_api.cpp -- host runtime behind the C ABI (include/bandmatch_gpu.h).
//
// Owns, per CUDA device context:
//   * the HBM descriptor arena (DeviceArena semantics, engine.cpp:18-40) on a
//     stream-ordered memory pool, fed by asynchronous H2D copies on a copy
//     stream (pinned sources go straight to the copy engine, pageable ones
//     through a double-buffered pinned staging ring);
//   * the per-row scratch (codes + bucket tables of every resident image,
//     recomputed per row because codes are relative to the row mean,
//     engine.cpp:446-465);
//   * the match scratch and a device-resident result log that rows append to
//     without host synchronisation; execute_plan reads it back once.
// No exception crosses the ABI: every entry point returns a bmg_status.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <emmintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

#include "../../include/bandmatch_gpu.h"
#include "bmg_internal.h"

namespace bmg {

uint64_t seed_for(uint64_t root, std::string_view stage);
bool valid_hash_params(const bmg_hash_params& p);
void make_planes(uint64_t seed, const bmg_hash_params& p, float* coarse, float* fine);

namespace {

struct Failure {
  int status;
  std::string msg;
};

[[noreturn]] void fail(int status, std::string msg) { throw Failure{status, std::move(msg)}; }

#define BMG_CUDA(x)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      fail(e_ == cudaErrorMemoryAllocation ? BMG_OUT_OF_MEMORY : BMG_CUDA_ERROR,        \
           std::string(#x) + ": " + cudaGetErrorString(e_));                           \
  } while (0)

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return BMG_OK;
  } catch (const Failure& e) {
    g_last_error = e.msg;
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return BMG_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BMG_CUDA_ERROR;
  }
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t n) {
    if (n <= cap) return;
    if (p) {
      BMG_CUDA(cudaDeviceSynchronize());
      cudaFree(p);
      p = nullptr;
      cap = 0;
    }
    n = align_up(std::max<size_t>(n, 256), 1 << 20);
    BMG_CUDA(cudaMalloc(&p, n));
    cap = n;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Pinned, device-mapped host buffer: kernels write results straight into host
// memory over PCIe as rows finish, so reading them back needs no D2H copy.
struct HostMapped {
  void* h = nullptr;
  void* d = nullptr;
  size_t cap = 0;
  void ensure(size_t n) {
    if (n <= cap) return;
    if (h) {
      BMG_CUDA(cudaDeviceSynchronize());
      cudaFreeHost(h);
      h = d = nullptr;
      cap = 0;
    }
    n = align_up(std::max<size_t>(n, 4096), 1 << 20);
    BMG_CUDA(cudaHostAlloc(&h, n, cudaHostAllocMapped | cudaHostAllocPortable));
    BMG_CUDA(cudaHostGetDevicePointer(&d, h, 0));
    cap = n;
  }
  template <typename T>
  T* host() const { return static_cast<T*>(h); }
  template <typename T>
  T* dev() const { return static_cast<T*>(d); }
  void release() {
    if (h) cudaFreeHost(h);
    h = d = nullptr;
    cap = 0;
  }
};

// Pinned host ring for small metadata uploads (tables of pointers, work
// lists): a slice stays valid until the ring wraps, and a wrap synchronises
// the streams that could still be reading it.
struct PinnedRing {
  char* base = nullptr;
  size_t cap = 0, head = 0;
  void init(size_t n) {
    // mapped: the row streams' meta_kernel reads slices straight from here
    BMG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&base), n, cudaHostAllocMapped | cudaHostAllocPortable));
    cap = n;
  }
  template <typename T>
  T* alloc(size_t count, cudaStream_t a, cudaStream_t b) {
    size_t bytes = align_up(std::max<size_t>(count * sizeof(T), 16), 256);
    if (bytes > cap) fail(BMG_OUT_OF_MEMORY, "metadata exceeds the pinned staging ring");
    if (head + bytes > cap) {
      (void)a;
      (void)b;
      BMG_CUDA(cudaDeviceSynchronize());  // every stream that may read the ring
      head = 0;
    }
    T* out = reinterpret_cast<T*>(base + head);
    head += bytes;
    return out;
  }
  void release() {
    if (base) cudaFreeHost(base);
    base = nullptr;
  }
};

// Fork-join pool of host threads for the staging copies: pageable
// descriptors memcpy'd into pinned slots, feature files read and
// de-interleaved into them (one thread of the caller plus workers).
class HostPool {
 public:
  explicit HostPool(int threads) {
    for (int i = 1; i < threads; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (std::thread& t : workers_) t.join();
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  // fn(i) for i in [0, n) on the workers and the caller; returns when all ran
  template <typename F>
  void run(int n, F&& fn) {
    std::function<void(int)> job(std::forward<F>(fn));
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &job;
      n_ = n;
      next_.store(0);
      pending_ = n;
      ++gen_;
    }
    cv_.notify_all();
    work(&job, n);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void work(const std::function<void(int)>* job, int n) {
    for (int i; (i = next_.fetch_add(1)) < n;) {
      (*job)(i);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      int n;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_); });
        if (stop_) return;
        seen = gen_;
        job = job_;
        n = n_;
      }
      work(job, n);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, pending_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

int host_threads() {
  if (const char* v = getenv("BMG_HOST_THREADS")) return std::max(1, atoi(v));
  const unsigned hc = std::thread::hardware_concurrency();
  return static_cast<int>(std::clamp(hc > 2 ? hc - 2 : 1u, 1u, 16u));
}

// Where an image's descriptors come from: a host array (pinned or pageable)
// or a feature file (features.cpp:199-249 layout), read when it uploads.
struct Source {
  const float* desc = nullptr;
  const char* path = nullptr;
  uint64_t count = 0;
};

struct ArenaImage {
  float* d = nullptr;         // [n][128] descriptors, then proj [n][proj_stride], dnorm [n], tile statistics
  float* proj = nullptr;
  float* dnorm = nullptr;
  void* tsum = nullptr;       // row-mean tile statistics (ImgDev::tsum / trng / tlow)
  void* trng = nullptr;
  uint32_t* tlow = nullptr;
  uint64_t n = 0;
  cudaEvent_t ev = nullptr;  // recorded on the projection stream once the image is usable
  uint64_t seq = 0;          // upload order
  int pstream = 0;           // projection stream that records `ev`
  uint64_t reproj = 0;       // execute_plan call that last re-projected it (BMG_EXEC_REPROJECT)
};

// A row's view of one image (descriptors, their projections and norms).
struct RowImage {
  const float* desc;
  uint64_t n;
  float* proj;
  float* dnorm;
  void* tsum = nullptr;
  void* trng = nullptr;
  uint32_t* tlow = nullptr;
};

// the image block after the descriptors: projections, norms, tile statistics
size_t image_extra_bytes(uint64_t n, int proj_stride) {
  return align_up(proj_bytes(n, proj_stride), 16) + tile_stats_bytes(n);
}

// Process-wide pool of pinned host buffers that execution results own (the
// row regions of the result log are DMA'd straight into them; freeing the
// result returns the buffer).
class PinnedPool {
 public:
  static void* acquire(size_t bytes, size_t* got) {
    std::lock_guard<std::mutex> g(mu());
    auto& f = free_list();
    auto it = f.lower_bound(bytes);
    if (it != f.end()) {
      void* p = it->second;
      *got = it->first;
      f.erase(it);
      return p;
    }
    const size_t n = align_up(std::max<size_t>(bytes, 1), 1 << 20);
    void* p = nullptr;
    if (cudaHostAlloc(&p, n, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
      cudaGetLastError();
      fail(BMG_OUT_OF_MEMORY, "pinned result buffer allocation failed");
    }
    *got = n;
    return p;
  }
  static void release(void* p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> g(mu());
    free_list().emplace(bytes, p);
  }

 private:
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::multimap<size_t, void*>& free_list() {
    static auto* f = new std::multimap<size_t, void*>();  // leaked at exit on purpose
    return *f;
  }
};

struct Timer {
  std::string cls;
  cudaEvent_t a, b;
};

struct RowLayout {
  size_t coarse_off, fine_off, offsets_off, cursor_off, slots_off, bfine_off;
};

// What the codes/tables kernels of the current row need to be (re)issued.
struct RowState {
  int n_imgs = 0;
  size_t n_tiles = 0;
  uint32_t fix_cap = 0;
  uint64_t total_desc = 0;
  size_t codes_bytes = 0, offsets_begin = 0, offsets_bytes = 0;
};

}  // namespace

}  // namespace bmg

namespace bmg {
namespace {
// Everything one block row needs on the device while it is in flight.
// bmg_execute_plan alternates two slots so row r+1 (its own stream, scratch
// and match buffers) overlaps row r; the single-row entry points use slot 0.
struct RowSlot {
  cudaStream_t s_comp = nullptr;  // the stream of the row the slot holds (home or a priority stream)
  cudaStream_t home = nullptr;    // the slot's own stream (single-row entry points, rows past the levels)
  cudaEvent_t done = nullptr;     // recorded after the slot's last row
  RowState rs;
  float* cur_mean = nullptr;
  // exact parallel row mean: F96 tile sums + state (kernels.cu K1)
  DevBuf d_mean_sums, d_mean_state;
  bool last_mean_chain_only = false;
  std::vector<uint64_t> row_ids;
  std::unordered_map<uint64_t, int> row_slot;
  std::vector<ImgDev> row_imgs;
  bool row_valid = false;
  DevBuf d_imgs, d_tiles, d_scratch, d_mean, d_acc, d_fix, d_fixcnt, d_diag, d_mproj;
  // match state
  DevBuf d_work, d_dense, d_dense_off, d_pair_count, d_nq;
  MetaBatch meta{};  // pending metadata copies / zero fills for s_comp
  void release() {
    for (DevBuf* b : {&d_imgs, &d_tiles, &d_scratch, &d_mean, &d_acc, &d_fix, &d_fixcnt, &d_diag, &d_mproj, &d_work,
                      &d_dense, &d_dense_off, &d_pair_count, &d_nq, &d_mean_sums, &d_mean_state})
      b->release();
    if (home) cudaStreamDestroy(home);
    if (done) cudaEventDestroy(done);
    home = s_comp = nullptr;
    done = nullptr;
  }
};
// One VLAD batch in flight (bmg_encode_vlad alternates two): device
// buffers and mapped host tables, kept by the context across calls
// (grow-only, like the row slots).
struct VladSlot {
  DevBuf desc, assign, fix, fixcnt, acc, members, member_off, dmeta;
  HostMapped meta, out;
  cudaEvent_t done = nullptr;
  std::vector<uint64_t> imgs;  // caller indices of the batch
  void release() {
    for (DevBuf* b : {&desc, &assign, &fix, &fixcnt, &acc, &members, &member_off, &dmeta}) b->release();
    meta.release();
    out.release();
    if (done) cudaEventDestroy(done);
    done = nullptr;
    imgs.clear();
  }
};
}  // namespace
}  // namespace bmg

struct bmg_context {
  int device = 0;
  bmg_hash_params hp{};
  bmg::HashDev hd{};
  uint64_t seed = 0;
  bmg::DevBuf planes_t, planes, plane_norm, tc_b, tc_fexp;
  // arena (DeviceArena, engine.hpp:20-44)
  uint64_t capacity = 0, occupancy = 0, peak = 0, uploads = 0, evictions = 0, units_uploaded = 0;
  std::map<uint64_t, bmg::ArenaImage> resident;
  cudaStream_t s_copy = nullptr;
  std::vector<cudaStream_t> s_prio;  // row streams by priority: row r of a call runs on s_prio[r]
  static constexpr int kProjStreams = 4;
  cudaStream_t s_proj[kProjStreams] = {};  // per-image projections, right behind each upload
  int proj_rr = 0;
  cudaEvent_t ev_copied = nullptr;
  uint64_t exec_serial = 0;        // execute_plan calls so far (re-projection epochs)
  bmg::RowSlot slot[2];
  bmg::VladSlot vlad[2];
  int cur = 0;
  bmg::RowSlot& S() { return slot[cur]; }
  bool mean_chain_only = false;  // test hook: the literal sequential chain
  cudaMemPool_t pool = nullptr;
  cudaEvent_t ev_uploaded = nullptr;
  bool pending_upload = false;
  // projection-ready events the current row's codes must wait for (set by
  // bmg_execute_plan: the row's mean only needs the copies)
  std::vector<cudaEvent_t> proj_waits;
  // pinned staging slots for pageable / file sources: slot k is refilled
  // (by the host pool) once the DMA that last read it has finished
  static constexpr int kStageSlots = 4;
  char* stage[kStageSlots] = {};
  cudaEvent_t stage_ev[kStageSlots] = {};
  int stage_i = 0;
  size_t stage_bytes = 0;
  std::unique_ptr<bmg::HostPool> host;
  bmg::PinnedRing ring;
  // result log (compacted per row into its own region of d_res) and the
  // per-pair [begin, end) ranges, written by the scan kernels straight into
  // mapped pinned host memory
  bmg::HostMapped res_ranges, res_log;
  bmg::DevBuf d_res;
  // temporaries for the stateless entry points
  bmg::DevBuf d_tmp_desc, d_tmp_codes;
  bmg::DevBuf d_rp;  // BMG_EXEC_REPROJECT: image table + tile list
  // instrumentation
  uint64_t launches = 0;
  bool profiling = false;
  std::vector<bmg::Timer> timers;
  std::vector<cudaEvent_t> free_events;
  uint32_t test_flags = 0;  // bmg_set_test_flags
  // BMG_TIMELINE diagnostics: labelled events recorded by the row body
  std::vector<std::pair<std::string, cudaEvent_t>>* marks = nullptr;
};

struct bmg_result {
  std::vector<uint64_t> pair_ids;  // (query image, train image) per pair, sorted by IdPair
  std::vector<uint64_t> ranges;    // [begin, end) of each pair's matches in `log` (entries)
  int32_t* log = nullptr;          // pinned: (query_idx, train_idx) int32 pairs
  size_t log_bytes = 0;
  uint64_t n_matches = 0;
  uint64_t counters[6] = {0, 0, 0, 0, 0, 0};
  std::vector<uint64_t> iterations;  // 3 per iteration
  // per plan row: host ms at which its pairs were handed to on_pair, device
  // ms at which its last kernel / copy finished, both since the call's first
  // device operation was issued; -1 when not recorded
  std::vector<double> row_handoff_ms, row_done_ms;
  double wall_s = 0.0;
  double device_ms = 0.0;
  ~bmg_result() { bmg::PinnedPool::release(log, log_bytes); }
};

namespace bmg {
namespace {

using Ctx = bmg_context;

cudaEvent_t take_event(Ctx& c) {
  if (!c.free_events.empty()) {
    cudaEvent_t e = c.free_events.back();
    c.free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  BMG_CUDA(cudaEventCreate(&e));
  return e;
}

struct Timed {
  Ctx& c;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  const char* cls;
  Timed(Ctx& ctx, const char* k, cudaStream_t st) : c(ctx), s(st), cls(k) {
    if (c.profiling) {
      a = take_event(c);
      b = take_event(c);
      cudaEventRecord(a, s);
    }
  }
  ~Timed() {
    if (a) {
      cudaEventRecord(b, s);
      c.timers.push_back({cls, a, b});
    }
  }
};

void set_device(Ctx& c) { BMG_CUDA(cudaSetDevice(c.device)); }

void check_launch();

void meta_flush(Ctx& c) {
  RowSlot& S = c.S();
  if (!S.meta.n) return;
  launch_meta(S.meta, S.s_comp);
  S.meta.n = 0;
  ++c.launches;
  check_launch();
}

// queue a small copy (src may be mapped pinned host memory) or, with
// src == nullptr, a zero fill on the current row stream
void meta_add(Ctx& c, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  RowSlot& S = c.S();
  if (S.meta.n == kMetaOps) meta_flush(c);
  S.meta.op[S.meta.n++] = MetaOp{dst, src, bytes};
}

void check_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(BMG_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
}

int padded_words(int fw) {
  int p = 1;
  while (p < fw) p <<= 1;
  return p;
}

int bit_width(uint32_t v) {
  int b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

// ---- arena ----------------------------------------------------------------

HostPool& host_pool(Ctx& c) {
  if (!c.host) c.host = std::make_unique<HostPool>(host_threads());
  return *c.host;
}

// the next staging slot, once the DMA that last read it has finished
char* next_slot(Ctx& c, int* i) {
  *i = c.stage_i;
  c.stage_i = (c.stage_i + 1) % bmg_context::kStageSlots;
  BMG_CUDA(cudaEventSynchronize(c.stage_ev[*i]));
  return c.stage[*i];
}

void slot_dma(Ctx& c, int i, void* dst, size_t bytes) {
  BMG_CUDA(cudaMemcpyAsync(dst, c.stage[i], bytes, cudaMemcpyHostToDevice, c.s_copy));
  BMG_CUDA(cudaEventRecord(c.stage_ev[i], c.s_copy));
}

// Copy into a pinned staging slot with streaming (non-temporal) stores: the
// slot is only read by the copy engine, so a plain memcpy's read-for-
// ownership of every destination line is wasted host-memory traffic (the
// staging competes with the DMA for it).  dst 16-byte aligned.
void stream_copy(char* dst, const char* src, size_t n, bool fence = true) {
  static const bool plain = [] {
    const char* v = getenv("BMG_STAGE_MEMCPY");  // A/B switch
    return v && v[0] == '1';
  }();
  if (plain || (reinterpret_cast<uintptr_t>(dst) & 15u)) {
    std::memcpy(dst, src, n);
    return;
  }
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c2);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  if (i < n) std::memcpy(dst + i, src + i, n - i);
  if (fence) _mm_sfence();  // the stores are visible before the DMA is issued
}

void stage_h2d(Ctx& c, void* dst, const void* src, size_t bytes) {
  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, src) == cudaSuccess &&
                      attr.type == cudaMemoryTypeHost;
  cudaGetLastError();
  if (pinned || bytes == 0) {
    if (bytes) BMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.s_copy));
    return;
  }
  // pageable (a std::vector FeatureSet): the host pool copies each slot-
  // sized chunk into a pinned slot in parallel while the copy engine DMAs
  // the previous slots
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  HostPool& pool = host_pool(c);
  for (size_t off = 0; off < bytes; off += c.stage_bytes) {
    const size_t sz = std::min(c.stage_bytes, bytes - off);
    int i;
    char* slot = next_slot(c, &i);
    const int parts = static_cast<int>(std::min<size_t>(pool.size(), (sz + (256u << 10) - 1) >> 18));
    const size_t per = ((sz + parts - 1) / parts + 63) & ~static_cast<size_t>(63);
    pool.run(parts, [&](int k) {
      const size_t a = k * per, n = a < sz ? std::min(per, sz - a) : 0;
      if (n) stream_copy(slot + a, s + off + a, n);
    });
    slot_dma(c, i, d + off, sz);
  }
}

// A feature file's descriptors straight into HBM: the header is checked like
// read_features (features.cpp:222-236) and must agree with the planned
// count; the 528-byte records are read by the host pool with pread and
// de-interleaved into pinned slots, each DMA'd while the next fills.
constexpr size_t kFeatHeader = 24, kFeatRecord = (4 + kDim) * sizeof(float);
constexpr uint64_t kFeatBlock = 256;  // records per pread (~132 KiB): 32 reads per 8k image

// Opens a feature file for streaming: the header is checked like
// read_features (features.cpp:222-236) and must agree with the planned
// count, and the body must hold every record.  Returns the descriptor.
int open_feature_file(const char* path, uint64_t count) {
  uint64_t id = 0, n = 0;
  if (const int rc = bmg_read_features_header(path, &id, &n); rc != BMG_OK) fail(rc, bmg_last_error());
  if (n != count)
    fail(BMG_INVALID_ARGUMENT, std::string(path) + ": holds " + std::to_string(n) + " features, planned " +
                                   std::to_string(count));
  const int fd = open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) fail(BMG_FORMAT_ERROR, std::string("cannot open ") + path + " for reading");
  struct stat st{};
  if (fstat(fd, &st) != 0) {
    close(fd);
    fail(BMG_FORMAT_ERROR, std::string("cannot stat ") + path);
  }
  const uint64_t body =
      static_cast<uint64_t>(st.st_size) > kFeatHeader ? static_cast<uint64_t>(st.st_size) - kFeatHeader : 0;
  if (body < count * kFeatRecord) {
    close(fd);
    fail(BMG_TRUNCATED_FILE, std::string("unexpected end of file while reading ") +
                                 (body % kFeatRecord < 16 ? "keypoint" : "descriptor"));
  }
  return fd;
}

// Records [r0, r0 + m) of an open feature file, de-interleaved into dst
// (streaming stores; the caller fences).  Returns false on a short read.
bool read_feature_block(int fd, uint64_t r0, uint64_t m, float* dst) {
  thread_local std::vector<unsigned char> buf;
  buf.resize(kFeatBlock * kFeatRecord);
  const off_t off = static_cast<off_t>(kFeatHeader + r0 * kFeatRecord);
  size_t have = 0;
  while (have < m * kFeatRecord) {
    const ssize_t got = pread(fd, buf.data() + have, m * kFeatRecord - have, off + static_cast<off_t>(have));
    if (got <= 0) break;
    have += static_cast<size_t>(got);
  }
  const uint64_t full = have / kFeatRecord;
  for (uint64_t k = 0; k < full; ++k)
    stream_copy(reinterpret_cast<char*>(dst + k * kDim),
                reinterpret_cast<const char*>(buf.data() + k * kFeatRecord + 16), kDim * sizeof(float), false);
  return have >= m * kFeatRecord;
}

// A feature file's descriptors straight into HBM: the 528-byte records are
// read by the host pool with pread and de-interleaved into pinned slots,
// each DMA'd while the next fills.
void stage_file(Ctx& c, void* dst, const char* path, uint64_t count) {
  const int fd = open_feature_file(path, count);
  struct FdGuard {
    int fd;
    ~FdGuard() { close(fd); }
  } guard{fd};
  HostPool& pool = host_pool(c);
  const uint64_t per_slot = c.stage_bytes / (kDim * sizeof(float));
  char* d = static_cast<char*>(dst);
  for (uint64_t r0 = 0; r0 < count; r0 += per_slot) {
    const uint64_t nr = std::min(per_slot, count - r0);
    int i;
    float* slot = reinterpret_cast<float*>(next_slot(c, &i));
    const int blocks = static_cast<int>((nr + kFeatBlock - 1) / kFeatBlock);
    std::atomic<bool> short_read{false};
    pool.run(blocks, [&](int b) {
      const uint64_t b0 = b * kFeatBlock, m = std::min(kFeatBlock, nr - b0);
      if (!read_feature_block(fd, r0 + b0, m, slot + b0 * kDim)) short_read.store(true);
      _mm_sfence();
    });
    if (short_read.load()) fail(BMG_TRUNCATED_FILE, "unexpected end of file while reading descriptor");
    slot_dma(c, i, d + r0 * kDim * sizeof(float), nr * kDim * sizeof(float));
  }
}

void stage_source(Ctx& c, void* dst, const Source& src) {
  if (src.path)
    stage_file(c, dst, src.path, src.count);
  else
    stage_h2d(c, dst, src.desc, src.count * kDim * sizeof(float));
}

// DeviceArena::upload bookkeeping (engine.cpp:18-25): capacity check and
// counters.  bmg_execute_plan runs it in the plan's order; the physical
// allocation (arena_alloc) may happen in another order.
void arena_account_upload(Ctx& c, uint64_t id, bool has_data, uint64_t n) {
  if (c.occupancy + n > c.capacity)
    fail(BMG_CAPACITY_EXCEEDED, "uploading image " + std::to_string(id) + " (" + std::to_string(n) +
                                    " units) would raise occupancy to " +
                                    std::to_string(c.occupancy + n) + " of " +
                                    std::to_string(c.capacity));
  if (n && !has_data) fail(BMG_INVALID_ARGUMENT, "null descriptor pointer");
  c.occupancy += n;
  c.peak = std::max(c.peak, c.occupancy);
  ++c.uploads;
  c.units_uploaded += n;
}

// the stream-ordered allocation of an image's HBM block (descriptors, then
// its projections and norms); the copy is issued separately (arena_copy)
ArenaImage& arena_alloc(Ctx& c, uint64_t id, uint64_t n) {
  ArenaImage im;
  im.n = n;
  const size_t bytes = n * 512 + image_extra_bytes(n, c.hd.proj_stride);
  BMG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&im.d), std::max<size_t>(bytes, 512), c.pool, c.s_copy));
  im.proj = im.d + n * kDim;
  im.dnorm = im.proj + n * c.hd.proj_stride;
  const size_t nt = (n + kCodesTile - 1) / kCodesTile;
  char* ts = reinterpret_cast<char*>(im.d) + n * 512 + align_up(proj_bytes(n, c.hd.proj_stride), 16);
  im.tsum = ts;
  im.trng = ts + nt * kDim * 16;
  im.tlow = reinterpret_cast<uint32_t*>(ts + nt * kDim * 48);
  return c.resident.emplace(id, im).first->second;
}

ArenaImage& arena_reserve(Ctx& c, uint64_t id, const float* desc, uint64_t n) {
  arena_account_upload(c, id, desc != nullptr, n);
  return arena_alloc(c, id, n);
}

uint64_t g_upload_seq = 0;

ImgDev proj_view(const ArenaImage& a) {
  ImgDev v{};
  v.desc = a.d;
  v.proj = a.proj;
  v.dnorm = a.dnorm;
  v.tsum = a.tsum;
  v.trng = a.trng;
  v.tlow = a.tlow;
  v.n = static_cast<uint32_t>(a.n);
  return v;
}

// The H2D of a reserved image on the copy stream; the projection stream then
// computes its mean-independent projections (K2 project_kernel) while the
// next images upload, and records the image's ready event.
// after an image's H2D is on the copy stream: its projections (and the
// row-mean tile statistics) right behind it on a projection stream
void arena_after_copy(Ctx& c, ArenaImage& im) {
  BMG_CUDA(cudaEventRecord(c.ev_copied, c.s_copy));
  im.pstream = c.proj_rr;
  c.proj_rr = (c.proj_rr + 1) % bmg_context::kProjStreams;
  cudaStream_t ps = c.s_proj[im.pstream];
  BMG_CUDA(cudaStreamWaitEvent(ps, c.ev_copied, 0));
  if (im.n) {
    Timed t(c, "project", ps);
    launch_project(c.hd, proj_view(im), ps);
    ++c.launches;
    check_launch();
  }
  if (!im.ev) im.ev = take_event(c);
  BMG_CUDA(cudaEventRecord(im.ev, ps));
  im.seq = ++g_upload_seq;
  c.pending_upload = true;
}

void arena_copy(Ctx& c, ArenaImage& im, const Source& src) {
  stage_source(c, im.d, src);
  arena_after_copy(c, im);
}

// A row's missing images in order: pinned arrays go straight to the copy
// engine and files through stage_file, one image at a time; consecutive
// pageable arrays that fit one staging slot together are memcpy'd into it
// by one fork-join of the host pool (one wake-up per slot, not per image),
// then DMA'd image by image, each followed by its projections.
void arena_copy_many(Ctx& c, const std::vector<std::pair<ArenaImage*, const Source*>>& imgs,
                     const std::function<void(size_t)>& after) {
  auto is_file = [&](const Source& src) { return src.path != nullptr && src.count > 0; };
  auto pageable = [&](const Source& src) {
    if (src.path || !src.desc || src.count == 0) return false;
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, src.desc) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return !pinned;
  };
  static const bool batch_off = [] {
    const char* v = getenv("BMG_STAGE_BATCH");  // A/B switch: 0 = one image per fork-join
    return v && v[0] == '0';
  }();
  size_t k = 0;
  while (k < imgs.size()) {
    const Source& s0 = *imgs[k].second;
    const size_t b0 = s0.count * kDim * sizeof(float);
    const bool files = is_file(s0);
    if (batch_off || !(files || pageable(s0)) || b0 > c.stage_bytes) {
      arena_copy(c, *imgs[k].first, s0);
      after(k++);
      continue;
    }
    // pack images [k, e) of the same kind into one slot
    size_t e = k + 1, used = b0;
    while (e < imgs.size()) {
      const Source& se = *imgs[e].second;
      const size_t be = align_up(se.count * kDim * sizeof(float), 256);
      if ((files ? !is_file(se) : !pageable(se)) || align_up(used, 256) + be > c.stage_bytes) break;
      used = align_up(used, 256) + be;
      ++e;
    }
    // files: headers checked and opened in order before any read
    std::vector<int> fds;
    struct FdsGuard {
      std::vector<int>& v;
      ~FdsGuard() {
        for (int fd : v) close(fd);
      }
    } fds_guard{fds};
    if (files)
      for (size_t j = k; j < e; ++j) fds.push_back(open_feature_file(imgs[j].second->path, imgs[j].second->count));
    int si;
    char* slot = next_slot(c, &si);
    std::vector<size_t> off(e - k);
    size_t o = 0;
    for (size_t j = k; j < e; ++j) {
      o = align_up(o, 256);
      off[j - k] = o;
      o += imgs[j].second->count * kDim * sizeof(float);
    }
    // tasks: 256 KiB of a pageable array, or kFeatBlock records of a file
    const size_t kPart = files ? kFeatBlock * kDim * sizeof(float) : (256u << 10);
    std::vector<std::pair<size_t, size_t>> parts;  // (image in batch, byte offset)
    for (size_t j = k; j < e; ++j) {
      const size_t bj = imgs[j].second->count * kDim * sizeof(float);
      for (size_t a = 0; a < bj; a += kPart) parts.emplace_back(j - k, a);
    }
    HostPool& pool = host_pool(c);
    std::atomic<bool> short_read{false};
    pool.run(static_cast<int>(parts.size()), [&](int q) {
      const auto [j, a] = parts[q];
      const Source& src = *imgs[k + j].second;
      const size_t bj = src.count * kDim * sizeof(float);
      if (files) {
        const uint64_t r0 = a / (kDim * sizeof(float)), m = std::min<uint64_t>(kFeatBlock, src.count - r0);
        if (!read_feature_block(fds[j], r0, m, reinterpret_cast<float*>(slot + off[j] + a))) short_read.store(true);
        _mm_sfence();
      } else {
        stream_copy(slot + off[j] + a, reinterpret_cast<const char*>(src.desc) + a, std::min(kPart, bj - a));
      }
    });
    if (short_read.load()) fail(BMG_TRUNCATED_FILE, "unexpected end of file while reading descriptor");
    for (size_t j = k; j < e; ++j) {
      BMG_CUDA(cudaMemcpyAsync(imgs[j].first->d, slot + off[j - k], imgs[j].second->count * kDim * sizeof(float),
                               cudaMemcpyHostToDevice, c.s_copy));
      if (j + 1 == e) BMG_CUDA(cudaEventRecord(c.stage_ev[si], c.s_copy));
      arena_after_copy(c, *imgs[j].first);
      after(j);
    }
    k = e;
  }
}

void arena_upload(Ctx& c, uint64_t id, const float* desc, uint64_t n) {
  if (c.resident.count(id)) return;  // engine.cpp:19
  arena_copy(c, arena_reserve(c, id, desc, n), Source{desc, nullptr, n});
}

// stream-ordered free of a resident image after every kernel already queued
// on the compute streams that may read it (the current slot's, and the other
// slot's row still in flight)
void arena_free(Ctx& c, uint64_t id) {
  const auto it = c.resident.find(id);
  if (it == c.resident.end()) fail(BMG_INVALID_ARGUMENT, "freeing image " + std::to_string(id) + ": not allocated");
  RowSlot& S = c.S();
  RowSlot& O = c.slot[c.cur ^ 1];
  if (O.s_comp) {
    cudaEvent_t e = take_event(c);
    BMG_CUDA(cudaEventRecord(e, O.s_comp));
    BMG_CUDA(cudaStreamWaitEvent(S.s_comp, e, 0));
    c.free_events.push_back(e);
  }
  BMG_CUDA(cudaFreeAsync(it->second.d, S.s_comp));
  if (it->second.ev) c.free_events.push_back(it->second.ev);
  c.resident.erase(it);
  if (S.row_slot.count(id)) S.row_valid = false;
  if (O.row_slot.count(id)) O.row_valid = false;
}

// DeviceArena::evict bookkeeping (engine.cpp:34-40)
void arena_account_evict(Ctx& c, uint64_t n) {
  c.occupancy -= n;
  ++c.evictions;
}

void arena_evict(Ctx& c, uint64_t id) {
  const auto it = c.resident.find(id);
  if (it == c.resident.end())
    fail(BMG_NOT_RESIDENT, "cannot evict image " + std::to_string(id) + ": not resident");
  arena_account_evict(c, it->second.n);
  arena_free(c, id);
}

void join_uploads(Ctx& c) {
  if (!c.pending_upload) return;
  for (cudaStream_t ps : c.s_proj) {
    BMG_CUDA(cudaEventRecord(c.ev_uploaded, ps));
    BMG_CUDA(cudaStreamWaitEvent(c.S().s_comp, c.ev_uploaded, 0));
  }
  c.pending_upload = false;
}

// ---- row body -------------------------------------------------------------

// Codes (+ FP64 fixups) and bucket tables for the current row views, centred
// on `d_mean`.
void enqueue_codes_tables(Ctx& c, const float* d_mean) {
  const RowState& rs = c.S().rs;
  if (rs.n_tiles == 0) {
    meta_flush(c);
    return;
  }
  cudaStream_t s = c.S().s_comp;
  const HashDev& h = c.hd;
  char* base = c.S().d_scratch.as<char>();
  const int plane_chunks = (h.n_planes + kPlaneChunk - 1) / kPlaneChunk;
  meta_add(c, base + rs.offsets_begin, nullptr, rs.offsets_bytes);
  if (plane_chunks > 1) meta_add(c, base, nullptr, rs.codes_bytes);
  meta_add(c, c.S().d_fixcnt.p, nullptr, sizeof(uint32_t) * (1 + rs.n_imgs));
  meta_flush(c);
  const ImgDev* d_imgs = c.S().d_imgs.as<ImgDev>();
  const uint32_t* d_tile_img = c.S().d_tiles.as<uint32_t>();
  const uint32_t* d_tile_start = d_tile_img + rs.n_tiles;
  unsigned long long* diag = c.S().d_diag.as<unsigned long long>();
  {
    Timed t(c, "codes", s);
    c.S().d_mproj.ensure(sizeof(float) * (h.n_planes + 1));
    launch_codes(h, d_imgs, d_tile_img, d_tile_start, static_cast<int>(rs.n_tiles), d_mean,
                 c.S().d_mproj.as<float>(), c.S().d_fix.as<Fixup>(), c.S().d_fixcnt.as<uint32_t>(), rs.fix_cap, s);
    c.launches += 2;
    check_launch();
  }
  {
    Timed t(c, "fixup", s);
    launch_codes_fixup(h, d_imgs, rs.n_imgs, d_mean, c.S().d_fix.as<Fixup>(), c.S().d_fixcnt.as<uint32_t>(),
                       rs.fix_cap, diag, s);
    c.launches += 2;
    check_launch();
  }
  {
    Timed t(c, "tables", s);
    c.launches += launch_tables(h, d_imgs, d_tile_img, d_tile_start, static_cast<int>(rs.n_tiles), rs.n_imgs, s);
    check_launch();
  }
}

// Lays out codes + tables for `descs` (device pointers, counts) in the row
// scratch, computes the mean (unless given) and launches codes, fixup and
// bucket-table kernels on the compute stream.
void prepare_row_views(Ctx& c, const std::vector<RowImage>& descs, const float* mean_host,
                       const float* mean_dev, bool compute_mean) {
  const HashDev& h = c.hd;
  const int n_imgs = static_cast<int>(descs.size());
  const int L = h.tables;
  const size_t NB = static_cast<size_t>(h.n_buckets);
  size_t off = 0, total_desc = 0, n_tiles = 0;
  std::vector<RowLayout> lay(n_imgs);
  // codes (coarse + fine) of all images first, then all bucket offsets, so
  // each group is one contiguous memset
  for (int i = 0; i < n_imgs; ++i) {
    const uint64_t n = descs[i].n;
    if (n >= (1ull << 31)) fail(BMG_UNSUPPORTED, "images with >= 2^31 descriptors");
    lay[i].coarse_off = off;
    off = align_up(off + n * L * 4, 256);
    lay[i].fine_off = off;
    off = align_up(off + align_up(n, 2) * h.fwp * 8, 256);
    total_desc += n;
    n_tiles += (n + kCodesTile - 1) / kCodesTile;
  }
  const size_t codes_end = off;
  for (int i = 0; i < n_imgs; ++i) {
    lay[i].offsets_off = off;
    off = align_up(off + L * (NB + 1) * 4, 256);
  }
  const size_t offsets_end = off;
  for (int i = 0; i < n_imgs; ++i) {
    lay[i].cursor_off = off;
    off = align_up(off + L * NB * 4, 256);
    const uint64_t ns = slot_stride(descs[i].n, h.n_buckets, h.bucket_pad);
    lay[i].slots_off = off;
    off = align_up(off + ns * L * 4, 256);
    lay[i].bfine_off = off;
    off = align_up(off + ns * L * h.fwp * 8, 256);
  }
  c.S().d_scratch.ensure(off);
  char* base = c.S().d_scratch.as<char>();
  c.S().row_imgs.assign(n_imgs, ImgDev{});
  for (int i = 0; i < n_imgs; ++i) {
    ImgDev& im = c.S().row_imgs[i];
    im.desc = descs[i].desc;
    im.proj = descs[i].proj;
    im.dnorm = descs[i].dnorm;
    im.tsum = descs[i].tsum;
    im.trng = descs[i].trng;
    im.tlow = descs[i].tlow;
    im.n = static_cast<uint32_t>(descs[i].n);
    im.coarse = reinterpret_cast<uint32_t*>(base + lay[i].coarse_off);
    im.fine = reinterpret_cast<uint64_t*>(base + lay[i].fine_off);
    im.offsets = reinterpret_cast<uint32_t*>(base + lay[i].offsets_off);
    im.cursor = reinterpret_cast<uint32_t*>(base + lay[i].cursor_off);
    im.slots = reinterpret_cast<uint32_t*>(base + lay[i].slots_off);
    im.bfine = reinterpret_cast<uint64_t*>(base + lay[i].bfine_off);
    im.overflow = 0;
    im.ns = slot_stride(im.n, h.n_buckets, h.bucket_pad);
  }
  // metadata
  ImgDev* h_imgs = c.ring.alloc<ImgDev>(std::max(n_imgs, 1), c.S().s_comp, c.s_copy);
  std::memcpy(h_imgs, c.S().row_imgs.data(), sizeof(ImgDev) * n_imgs);
  uint32_t* h_tiles = c.ring.alloc<uint32_t>(2 * std::max<size_t>(n_tiles, 1), c.S().s_comp, c.s_copy);
  {
    size_t t = 0;
    for (int i = 0; i < n_imgs; ++i)
      for (uint64_t s = 0; s < descs[i].n; s += kCodesTile) {
        h_tiles[t] = static_cast<uint32_t>(i);
        h_tiles[n_tiles + t] = static_cast<uint32_t>(s);
        ++t;
      }
  }
  c.S().d_imgs.ensure(sizeof(ImgDev) * std::max(n_imgs, 1));
  c.S().d_tiles.ensure(sizeof(uint32_t) * 2 * std::max<size_t>(n_tiles, 1));
  c.S().d_mean.ensure(sizeof(float) * kDim);
  c.S().d_acc.ensure(sizeof(double) * kDim);
  const uint32_t fix_cap = static_cast<uint32_t>(std::max<size_t>(65536, total_desc / 4));
  c.S().d_fix.ensure(sizeof(Fixup) * fix_cap);
  c.S().d_fixcnt.ensure(sizeof(uint32_t) * (1 + std::max(n_imgs, 1)));
  c.S().d_diag.ensure(sizeof(unsigned long long) * 4);
  cudaStream_t s = c.S().s_comp;
  (void)s;
  meta_add(c, c.S().d_imgs.p, h_imgs, sizeof(ImgDev) * n_imgs);
  meta_add(c, c.S().d_tiles.p, h_tiles, sizeof(uint32_t) * 2 * n_tiles);
  meta_add(c, c.S().d_diag.p, nullptr, sizeof(unsigned long long) * 4);
  RowState& rs = c.S().rs;
  rs.n_imgs = n_imgs;
  rs.n_tiles = n_tiles;
  rs.fix_cap = fix_cap;
  rs.total_desc = total_desc;
  rs.codes_bytes = codes_end;
  rs.offsets_begin = codes_end;
  rs.offsets_bytes = offsets_end - codes_end;
  join_uploads(c);

  const ImgDev* d_imgs = c.S().d_imgs.as<ImgDev>();
  float* d_mean = c.S().d_mean.as<float>();
  c.S().cur_mean = d_mean;
  if (mean_dev) {
    meta_add(c, d_mean, mean_dev, sizeof(float) * kDim);
  } else if (mean_host) {
    float* hm = c.ring.alloc<float>(kDim, c.S().s_comp, c.s_copy);
    std::memcpy(hm, mean_host, sizeof(float) * kDim);
    meta_add(c, d_mean, hm, sizeof(float) * kDim);
  } else if (compute_mean) {
    // exact row mean (engine.cpp:446-461): F96 reconstruction of the FP64
    // chain, the chain itself only as fallback (rows over 2^23 descriptors
    // exceed the F96 headroom and take the chain directly)
    const bool chain_only = c.mean_chain_only || total_desc > (1ull << 23) || n_tiles == 0;
    c.S().last_mean_chain_only = chain_only;
    c.S().d_mean_sums.ensure(mean_scratch_bytes(std::max<size_t>(n_tiles, 1)));
    c.S().d_mean_state.ensure(sizeof(MeanState));
    meta_add(c, c.S().d_mean_state.p, nullptr, sizeof(MeanState));
    meta_flush(c);
    // the tile statistics come with the images' projections (tensor-core
    // K2): the mean waits for those, then only resolves
    const bool resident = project_writes_tile_stats(c.hd);
    if (resident) {
      for (cudaEvent_t e : c.proj_waits) BMG_CUDA(cudaStreamWaitEvent(s, e, 0));
      c.proj_waits.clear();
    }
    Timed t(c, "mean", s);
    c.launches += launch_row_mean(d_imgs, n_imgs, c.S().d_tiles.as<uint32_t>(),
                                  c.S().d_tiles.as<uint32_t>() + n_tiles, static_cast<int>(n_tiles),
                                  total_desc, c.S().d_mean_sums.p, c.S().d_mean_state.as<MeanState>(), d_mean,
                                  c.S().d_acc.as<double>(), chain_only, resident, s);
    check_launch();
  }
  if (c.marks) {
    cudaEvent_t e;
    BMG_CUDA(cudaEventCreate(&e));
    BMG_CUDA(cudaEventRecord(e, s));
    c.marks->emplace_back("  mean done", e);
  }
  for (cudaEvent_t e : c.proj_waits) BMG_CUDA(cudaStreamWaitEvent(s, e, 0));
  c.proj_waits.clear();
  enqueue_codes_tables(c, d_mean);
}

void prepare_row(Ctx& c, const uint64_t* ids, uint64_t n, const float* mean_host) {
  std::vector<RowImage> descs;
  descs.reserve(n);
  c.S().row_ids.assign(ids, ids + n);
  c.S().row_slot.clear();
  for (uint64_t i = 0; i < n; ++i) {
    if (i && ids[i] <= ids[i - 1])
      fail(BMG_INVALID_ARGUMENT, "needed image ids must be strictly ascending");
    const auto it = c.resident.find(ids[i]);
    if (it == c.resident.end())
      fail(BMG_NOT_RESIDENT, "row needs image " + std::to_string(ids[i]) + " which is not resident");
    descs.push_back(RowImage{it->second.d, it->second.n, it->second.proj, it->second.dnorm, it->second.tsum,
                             it->second.trng, it->second.tlow});
    c.S().row_slot[ids[i]] = static_cast<int>(i);
  }
  c.S().row_valid = false;
  prepare_row_views(c, descs, mean_host, nullptr, true);
  c.S().row_valid = true;
}

// ---- matching ---------------------------------------------------------------



void check_match_params(const Ctx& c, const bmg_match_params& mp) {
  if (mp.k_nearest < 1) fail(BMG_INVALID_ARGUMENT, "k_nearest must be >= 1");
  if (mp.k_nearest > 32) fail(BMG_UNSUPPORTED, "k_nearest > 32 is not supported by the GPU matcher");
  (void)c;
}

// Enqueues match + scan + compact for (query slot, train slot) pairs of the
// current row views.  Pair i's matches land in d_res at the [begin, end)
// written to out_off[2i], out_off[2i+1]; the launch packs them from `base`.
void enqueue_match(Ctx& c, const std::vector<std::pair<int, int>>& slot_pairs,
                   const bmg_match_params& mp, uint64_t* out_off, int32_t* d_res, uint64_t base) {
  check_match_params(c, mp);
  const int n_pairs = static_cast<int>(slot_pairs.size());
  if (n_pairs == 0) return;
  const HashDev& h = c.hd;
  int chunk = match_queries_per_cta(h.fwp, mp.k_nearest);
  if (h.tables > 32) fail(BMG_UNSUPPORTED, "more than 32 hash tables is not supported by the GPU matcher");
  const int idx_bits = 32 - bit_width(static_cast<uint32_t>(h.fine_bits));
  std::vector<int> order(n_pairs);
  for (int p = 0; p < n_pairs; ++p) order[p] = p;
  // CTAs of pairs sharing a train image run back to back (L2 reuse of its
  // descriptors during the re-rank gathers)
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return slot_pairs[x].second < slot_pairs[y].second; });
  uint64_t total_q = 0;
  for (int p = 0; p < n_pairs; ++p) {
    const ImgDev& t = c.S().row_imgs[slot_pairs[p].second];
    if (t.n > (1u << idx_bits) - 1u) fail(BMG_UNSUPPORTED, "train image too large for the key packing");
    total_q += c.S().row_imgs[slot_pairs[p].first].n;
  }
  // few pairs (e.g. a single pair): smaller query ranges so the grid still
  // covers every SM twice (down to one query per warp)
  {
    const uint64_t want = 2ull * static_cast<uint64_t>(device_sm_count());
    if ((total_q + chunk - 1) / chunk < want)
      chunk = static_cast<int>(std::max<uint64_t>(32, (total_q + want - 1) / want + 31) / 32 * 32);
    chunk = std::min(chunk, match_queries_per_cta(h.fwp, mp.k_nearest));
  }
  size_t n_work = 0;
  for (int p = 0; p < n_pairs; ++p) n_work += (c.S().row_imgs[slot_pairs[p].first].n + chunk - 1) / chunk;
  PairWork* h_work = c.ring.alloc<PairWork>(std::max<size_t>(n_work, 1), c.S().s_comp, c.s_copy);
  uint64_t* h_dense_off = c.ring.alloc<uint64_t>(n_pairs, c.S().s_comp, c.s_copy);
  uint32_t* h_nq = c.ring.alloc<uint32_t>(n_pairs, c.S().s_comp, c.s_copy);
  uint64_t dense_total = 0;
  for (int p = 0; p < n_pairs; ++p) {
    h_dense_off[p] = dense_total;
    h_nq[p] = c.S().row_imgs[slot_pairs[p].first].n;
    dense_total += h_nq[p];
  }
  size_t w = 0;
  for (int oi = 0; oi < n_pairs; ++oi) {
    const int p = order[oi];
    const uint32_t nq = h_nq[p];
    for (uint32_t q0 = 0; q0 < nq; q0 += chunk) {
      PairWork& pw = h_work[w++];
      pw.q_img = static_cast<uint32_t>(slot_pairs[p].first);
      pw.t_img = static_cast<uint32_t>(slot_pairs[p].second);
      pw.q_begin = q0;
      pw.q_end = std::min<uint32_t>(nq, q0 + chunk);
      pw.pair = static_cast<uint32_t>(p);
    }
  }
  c.S().d_work.ensure(sizeof(PairWork) * std::max<size_t>(n_work, 1));
  c.S().d_dense_off.ensure(sizeof(uint64_t) * n_pairs);
  c.S().d_nq.ensure(sizeof(uint32_t) * n_pairs);
  c.S().d_pair_count.ensure(sizeof(uint32_t) * n_pairs);
  c.S().d_dense.ensure(sizeof(int32_t) * std::max<uint64_t>(dense_total, 1));
  cudaStream_t s = c.S().s_comp;
  meta_add(c, c.S().d_work.p, h_work, sizeof(PairWork) * n_work);
  meta_add(c, c.S().d_dense_off.p, h_dense_off, sizeof(uint64_t) * n_pairs);
  meta_add(c, c.S().d_nq.p, h_nq, sizeof(uint32_t) * n_pairs);
  meta_add(c, c.S().d_pair_count.p, nullptr, sizeof(uint32_t) * n_pairs);
  meta_flush(c);
  MatchLaunch a{};
  a.imgs = c.S().d_imgs.as<ImgDev>();
  a.work = c.S().d_work.as<PairWork>();
  a.dense_off = c.S().d_dense_off.as<uint64_t>();
  a.dense = c.S().d_dense.as<int32_t>();
  a.pair_count = c.S().d_pair_count.as<uint32_t>();
  a.exact_queries = c.S().d_diag.as<unsigned long long>() + 1;
  a.tables = h.tables;
  a.n_buckets = h.n_buckets;
  a.k = mp.k_nearest;
  a.idx_bits = idx_bits;
  a.ratio = mp.ratio;
  a.test_flags = c.test_flags;
  if (n_work) {
    Timed t(c, "match", s);
    launch_match(a, h.fwp, static_cast<int>(n_work), s);
    ++c.launches;
    check_launch();
  }
  {
    Timed t(c, "compact", s);
    launch_scan_counts(c.S().d_pair_count.as<uint32_t>(), n_pairs, out_off, base, s);
    launch_compact(c.S().d_dense.as<int32_t>(), c.S().d_dense_off.as<uint64_t>(), c.S().d_nq.as<uint32_t>(),
                   out_off, n_pairs, d_res, s);
    c.launches += 2;
    check_launch();
  }
}

HashDev build_hash(Ctx& c, const bmg_hash_params& p, const float* coarse, const float* fine) {
  HashDev h{};
  h.tables = p.tables;
  h.coarse_bits = p.coarse_bits;
  h.fine_bits = p.fine_bits;
  h.n_planes = p.tables * p.coarse_bits + p.fine_bits;
  h.fw = (p.fine_bits + 63) / 64;
  h.fwp = padded_words(h.fw);
  h.n_buckets = 1 << p.coarse_bits;
  h.n_planes_pad = static_cast<int>(align_up(h.n_planes, kPlaneChunk));
  h.proj_stride = static_cast<int>(align_up(h.n_planes, 4));
  h.bucket_pad = kBucketPad;
  const int np = h.n_planes, npp = h.n_planes_pad;
  std::vector<float> planes(static_cast<size_t>(np) * kDim), planes_t(static_cast<size_t>(npp) * kDim, 0.f),
      norm(npp, 0.f);
  const size_t nc = static_cast<size_t>(p.tables) * p.coarse_bits * kDim;
  std::memcpy(planes.data(), coarse, nc * sizeof(float));
  std::memcpy(planes.data() + nc, fine, static_cast<size_t>(p.fine_bits) * kDim * sizeof(float));
  for (int q = 0; q < np; ++q) {
    double ss = 0.0;
    for (int d = 0; d < kDim; ++d) {
      const float v = planes[static_cast<size_t>(q) * kDim + d];
      planes_t[static_cast<size_t>(d) * npp + q] = v;
      ss += static_cast<double>(v) * v;
    }
    // ||p||_2 rounded up (the certificate needs an upper bound)
    norm[q] = static_cast<float>(std::sqrt(ss) * (1.0 + 1e-6)) ;
  }
  c.planes.ensure(planes.size() * sizeof(float));
  c.planes_t.ensure(planes_t.size() * sizeof(float));
  c.plane_norm.ensure(norm.size() * sizeof(float));
  BMG_CUDA(cudaMemcpy(c.planes.p, planes.data(), planes.size() * sizeof(float), cudaMemcpyHostToDevice));
  BMG_CUDA(cudaMemcpy(c.planes_t.p, planes_t.data(), planes_t.size() * sizeof(float), cudaMemcpyHostToDevice));
  BMG_CUDA(cudaMemcpy(c.plane_norm.p, norm.data(), norm.size() * sizeof(float), cudaMemcpyHostToDevice));
  h.planes = c.planes.as<float>();
  h.planes_t = c.planes_t.as<float>();
  h.plane_norm = c.plane_norm.as<float>();
  // tensor-core K2 operand: each plane scaled by its own power of two and
  // rounded to a 22-bit integer, split into balanced base-256 digits, laid
  // out K-major with the 128-byte swizzle (kernels.cu project_tc_kernel)
  h.tc_npad = static_cast<int>(align_up(np, 16));
  if (h.tc_npad <= 96) {
    h.tc_pass0 = h.tc_npad;
  } else if (h.tc_npad <= 192) {
    h.tc_pass0 = static_cast<int>(align_up((h.tc_npad + 1) / 2, 16));
  }
  if (h.tc_npad <= 192) {
    const int npad = h.tc_npad;
    std::vector<int8_t> img(static_cast<size_t>(3) * npad * 128, 0);
    std::vector<int> fexp(npad, 0);
    for (int q = 0; q < np; ++q) {
      float mx = 0.f;
      for (int d = 0; d < kDim; ++d) mx = std::max(mx, std::fabs(planes[static_cast<size_t>(q) * kDim + d]));
      int f = 0;
      if (mx > 0.f) std::frexp(mx, &f);
      fexp[q] = f;
      for (int d = 0; d < kDim; ++d) {
        int x = static_cast<int>(std::nearbyint(std::ldexp(static_cast<double>(planes[static_cast<size_t>(q) * kDim + d]), 22 - f)));
        const int d0 = static_cast<int8_t>(x & 0xff);
        x = (x - d0) >> 8;
        const int d1 = static_cast<int8_t>(x & 0xff);
        const int d2 = (x - d1) >> 8;
        const size_t off = static_cast<size_t>(q >> 3) * 1024 + static_cast<size_t>(q & 7) * 128 +
                           static_cast<size_t>(((d >> 4) ^ (q & 7)) * 16 + (d & 15));
        img[off] = static_cast<int8_t>(d0);
        img[static_cast<size_t>(npad) * 128 + off] = static_cast<int8_t>(d1);
        img[static_cast<size_t>(2) * npad * 128 + off] = static_cast<int8_t>(d2);
      }
    }
    c.tc_b.ensure(img.size());
    c.tc_fexp.ensure(fexp.size() * sizeof(int));
    BMG_CUDA(cudaMemcpy(c.tc_b.p, img.data(), img.size(), cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(c.tc_fexp.p, fexp.data(), fexp.size() * sizeof(int), cudaMemcpyHostToDevice));
    h.tc_b = c.tc_b.as<signed char>();
    h.tc_fexp = c.tc_fexp.as<int>();
  }
  return h;
}

void copy_codes_out(Ctx& c, const ImgDev& im, uint32_t* coarse_out, uint64_t* fine_out) {
  const HashDev& h = c.hd;
  const size_t n = im.n;
  if (coarse_out && n)
    BMG_CUDA(cudaMemcpyAsync(coarse_out, im.coarse, n * h.tables * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, c.S().s_comp));
  if (fine_out && n) {
    if (h.fw == h.fwp) {
      BMG_CUDA(cudaMemcpyAsync(fine_out, im.fine, n * h.fw * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                               c.S().s_comp));
    } else {
      BMG_CUDA(cudaMemcpy2DAsync(fine_out, h.fw * sizeof(uint64_t), im.fine, h.fwp * sizeof(uint64_t),
                                 h.fw * sizeof(uint64_t), n, cudaMemcpyDeviceToHost, c.S().s_comp));
    }
  }
  BMG_CUDA(cudaStreamSynchronize(c.S().s_comp));
}

// capacity: matches the device log must hold (0: the caller compacts into
// its own buffer)
void reset_results(Ctx& c, uint64_t n_pairs, uint64_t capacity, bool host_mirror = true) {
  c.res_ranges.ensure(sizeof(uint64_t) * 2 * std::max<uint64_t>(n_pairs, 1));  // [begin, end) per pair
  if (host_mirror) c.res_log.ensure(sizeof(int32_t) * 2 * std::max<uint64_t>(capacity, 1));
  if (capacity) c.d_res.ensure(sizeof(int32_t) * 2 * capacity);
}

// Hands each block row's matches to the caller's on_pair callback (the
// VerifyPool::push hand-off, engine.cpp:478-479) from a collector thread as
// soon as the row's log region is in host memory, while later rows still
// run on the GPU.  Rows are handed over in the order they were issued; pairs
// of a row in plan (block) order.  The executor joins the thread before it
// returns, so every callback has run by then.
class Collector {
 public:
  struct Row {
    cudaEvent_t done;  // recorded after the row's last copy / compaction
    uint64_t plan_row, pb, pe;
  };
  Collector(int device, const bmg_plan* plan, const bmg_execute_options* opts, const int32_t* log,
            const uint64_t* ranges, std::chrono::steady_clock::time_point t0, bmg_result* res)
      : device_(device), plan_(plan), opts_(opts), log_(log), ranges_(ranges), t0_(t0), res_(res) {
    th_ = std::thread([this] { run(); });
  }
  ~Collector() { finish(); }
  void push(const Row& r) {
    std::lock_guard<std::mutex> g(mu_);
    q_.push_back(r);
    cv_.notify_one();
  }
  // no more rows: wait until every queued row has been handed over
  void finish() {
    {
      std::lock_guard<std::mutex> g(mu_);
      if (closed_) return;
      closed_ = true;
    }
    cv_.notify_one();
    th_.join();
  }
  std::vector<cudaEvent_t> events;  // owned by the executor's event pool

 private:
  void run() {
    cudaSetDevice(device_);
    for (;;) {
      Row r;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return closed_ || !q_.empty(); });
        if (q_.empty()) return;
        r = q_.front();
        q_.pop_front();
      }
      if (cudaEventSynchronize(r.done) != cudaSuccess) {
        cudaGetLastError();
        continue;  // the executor reports the failure
      }
      res_->row_handoff_ms[r.plan_row] =
          1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
      for (uint64_t p = r.pb; p < r.pe; ++p) {
        const uint64_t b = ranges_[2 * p], e = ranges_[2 * p + 1];
        opts_->on_pair(opts_->on_pair_user, plan_->pairs[2 * p], plan_->pairs[2 * p + 1], log_ + 2 * b, e - b);
      }
    }
  }
  int device_;
  const bmg_plan* plan_;
  const bmg_execute_options* opts_;
  const int32_t* log_;
  const uint64_t* ranges_;
  std::chrono::steady_clock::time_point t0_;
  bmg_result* res_;
  std::thread th_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Row> q_;
  bool closed_ = false;
};

// After the compute stream drained: DMA the log entries [0, end) into the
// pinned host mirror and return it.
const int32_t* fetch_log(Ctx& c, uint64_t end) {
  if (end)
    BMG_CUDA(cudaMemcpy(c.res_log.host<int32_t>(), c.d_res.p, sizeof(int32_t) * 2 * end,
                        cudaMemcpyDeviceToHost));
  return c.res_log.host<int32_t>();
}

}  // namespace
}  // namespace bmg

namespace bmg {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace bmg

using namespace bmg;

extern "C" {

const char* bmg_status_name(int status) {
  switch (status) {
    case BMG_OK: return "Ok";
    case BMG_INVALID_ARGUMENT: return "InvalidArgument";
    case BMG_HASH_MISMATCH: return "HashMismatch";
    case BMG_CAPACITY_EXCEEDED: return "CapacityExceeded";
    case BMG_NOT_RESIDENT: return "NotResident";
    case BMG_CUDA_ERROR: return "CudaError";
    case BMG_OUT_OF_MEMORY: return "OutOfMemory";
    case BMG_UNSUPPORTED: return "Unsupported";
    case BMG_INVALID_SCENE: return "InvalidScene";
    case BMG_FORMAT_ERROR: return "FormatError";
    case BMG_TRUNCATED_FILE: return "TruncatedFile";
    case BMG_TOO_FEW_DESCRIPTORS: return "TooFewDescriptors";
    default: return "Unknown";
  }
}

const char* bmg_last_error(void) { return g_last_error.c_str(); }
int bmg_abi_version(void) { return BMG_ABI_VERSION; }

uint64_t bmg_seed_for(uint64_t root, const char* stage) { return seed_for(root, stage ? stage : ""); }

int bmg_make_hash_functions(uint64_t seed, const bmg_hash_params* params, float* coarse_out,
                            float* fine_out) {
  return guarded([&] {
    if (!params || !valid_hash_params(*params))
      fail(BMG_INVALID_ARGUMENT, "hash params out of range (tables>=1, coarse_bits in [1,32], fine_bits>=1)");
    make_planes(seed, *params, coarse_out, fine_out);
  });
}

int bmg_create(const bmg_config* cfg, bmg_context** out) {
  return guarded([&] {
    if (!cfg || !out) fail(BMG_INVALID_ARGUMENT, "null argument");
    if (!valid_hash_params(cfg->hash))
      fail(BMG_INVALID_ARGUMENT, "hash params out of range (tables>=1, coarse_bits in [1,32], fine_bits>=1)");
    if (cfg->hash.fine_bits > 1024)
      fail(BMG_UNSUPPORTED, "fine_bits > 1024 (config.cpp:116-122 range) is not supported on the GPU path");
    if (cfg->hash.coarse_bits > 16)
      fail(BMG_UNSUPPORTED, "coarse_bits > 16 (>65536 buckets per table) is not supported on the GPU path");
    if (!cfg->coarse_planes || !cfg->fine_planes) fail(BMG_INVALID_ARGUMENT, "null hash planes");
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
      cudaGetLastError();
      fail(BMG_CUDA_ERROR, "no CUDA device available: the B200 matcher has no CPU fallback");
    }
    if (cfg->device < 0 || cfg->device >= n_dev) fail(BMG_INVALID_ARGUMENT, "bad device ordinal");
    auto c = std::make_unique<bmg_context>();
    c->device = cfg->device;
    set_device(*c);
    c->hp = cfg->hash;
    c->seed = cfg->function_seed;
    c->capacity = cfg->capacity_units;
    BMG_CUDA(cudaStreamCreateWithFlags(&c->s_copy, cudaStreamNonBlocking));
    // both row slots share one priority (which of two overlapping rows is on
    // the critical path depends on the plan); projections get the higher one
    int prio_lo = 0, prio_hi = 0;
    BMG_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    for (RowSlot& sl : c->slot) {
      BMG_CUDA(cudaStreamCreateWithPriority(&sl.home, cudaStreamNonBlocking, prio_lo));
      sl.s_comp = sl.home;
      BMG_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    }
    // earlier rows of a plan get higher priority (two rows overlap: the
    // earlier one gates its slot's next row); rows past the levels alternate
    // between the two equal-priority home streams
    for (int pr = prio_hi; pr < prio_lo; ++pr) {
      cudaStream_t st;
      BMG_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, pr));
      c->s_prio.push_back(st);
    }
    // projections feed the next rows' codes: highest priority too
    for (cudaStream_t& ps : c->s_proj) BMG_CUDA(cudaStreamCreateWithPriority(&ps, cudaStreamNonBlocking, prio_hi));
    BMG_CUDA(cudaEventCreateWithFlags(&c->ev_uploaded, cudaEventDisableTiming));
    BMG_CUDA(cudaEventCreateWithFlags(&c->ev_copied, cudaEventDisableTiming));

    BMG_CUDA(cudaDeviceGetDefaultMemPool(&c->pool, c->device));
    uint64_t thresh = ~0ull;
    BMG_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    // never make an upload wait for the compute stream that freed the memory
    // it would reuse (the DeviceArena's capacity accounting is logical; the
    // physical pool may grow so the next row's H2D overlaps this row's work)
    int no = 0;
    BMG_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowInternalDependencies, &no));
    c->stage_bytes = 16u << 20;
    for (int i = 0; i < bmg_context::kStageSlots; ++i) {
      BMG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&c->stage[i]), c->stage_bytes));
      BMG_CUDA(cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming));
      BMG_CUDA(cudaEventRecord(c->stage_ev[i], c->s_copy));
    }
    c->ring.init(64u << 20);
    c->hd = build_hash(*c, cfg->hash, cfg->coarse_planes, cfg->fine_planes);
    *out = c.release();
  });
}

int bmg_destroy(bmg_context* c) {
  if (!c) return BMG_OK;
  return guarded([&] {
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto& [id, im] : c->resident) {
      cudaFree(im.d);
      if (im.ev) cudaEventDestroy(im.ev);
      im.ev = nullptr;
    }
    c->resident.clear();
    for (DevBuf* b : {&c->planes_t, &c->planes, &c->plane_norm, &c->tc_b, &c->tc_fexp, &c->d_tmp_desc, &c->d_tmp_codes, &c->d_rp})
      b->release();
    for (RowSlot& sl : c->slot) sl.release();
    for (VladSlot& v : c->vlad) v.release();
    c->res_ranges.release();
    c->res_log.release();
    c->d_res.release();
    c->host.reset();
    for (int i = 0; i < bmg_context::kStageSlots; ++i) {
      if (c->stage[i]) cudaFreeHost(c->stage[i]);
      if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
    }
    c->ring.release();
    for (auto& t : c->timers) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    for (cudaEvent_t e : c->free_events) cudaEventDestroy(e);
    if (c->ev_uploaded) cudaEventDestroy(c->ev_uploaded);
    if (c->ev_copied) cudaEventDestroy(c->ev_copied);
    if (c->s_copy) cudaStreamDestroy(c->s_copy);
    for (cudaStream_t ps : c->s_proj)
      if (ps) cudaStreamDestroy(ps);
    for (cudaStream_t ps : c->s_prio) cudaStreamDestroy(ps);
    delete c;
  });
}

int bmg_synchronize(bmg_context* c) {
  return guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null context");
    set_device(*c);
    BMG_CUDA(cudaStreamSynchronize(c->s_copy));
    for (cudaStream_t ps : c->s_proj) BMG_CUDA(cudaStreamSynchronize(ps));
    for (RowSlot& sl : c->slot) BMG_CUDA(cudaStreamSynchronize(sl.s_comp));
    for (cudaStream_t ps : c->s_prio) BMG_CUDA(cudaStreamSynchronize(ps));
  });
}

int bmg_upload(bmg_context* c, uint64_t id, const float* desc, uint64_t count) {
  return guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null context");
    set_device(*c);
    arena_upload(*c, id, desc, count);
  });
}

int bmg_evict(bmg_context* c, uint64_t id) {
  return guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null context");
    set_device(*c);
    arena_evict(*c, id);
  });
}

int bmg_is_resident(bmg_context* c, uint64_t id) { return c && c->resident.count(id) ? 1 : 0; }

int bmg_arena_stats_get(bmg_context* c, bmg_arena_stats* o) {
  return guarded([&] {
    if (!c || !o) fail(BMG_INVALID_ARGUMENT, "null argument");
    o->capacity = c->capacity;
    o->occupancy = c->occupancy;
    o->peak_occupancy = c->peak;
    o->uploads = c->uploads;
    o->evictions = c->evictions;
    o->units_uploaded = c->units_uploaded;
    o->resident_count = c->resident.size();
  });
}

int bmg_row(bmg_context* c, const uint64_t* needed, uint64_t n, const float* mean) {
  return guarded([&] {
    if (!c || (n && !needed)) fail(BMG_INVALID_ARGUMENT, "null argument");
    set_device(*c);
    prepare_row(*c, needed, n, mean);
  });
}

int bmg_row_mean(bmg_context* c, float* mean_out) {
  return guarded([&] {
    if (!c || !mean_out) fail(BMG_INVALID_ARGUMENT, "null argument");
    if (!c->S().row_valid) fail(BMG_INVALID_ARGUMENT, "no row has been prepared");
    set_device(*c);
    BMG_CUDA(cudaMemcpyAsync(mean_out, c->S().cur_mean, sizeof(float) * kDim, cudaMemcpyDeviceToHost, c->S().s_comp));
    BMG_CUDA(cudaStreamSynchronize(c->S().s_comp));
  });
}

int bmg_codes(bmg_context* c, uint64_t id, uint32_t* coarse_out, uint64_t* fine_out) {
  return guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null context");
    if (!c->S().row_valid) fail(BMG_INVALID_ARGUMENT, "no row has been prepared");
    const auto it = c->S().row_slot.find(id);
    if (it == c->S().row_slot.end()) fail(BMG_INVALID_ARGUMENT, "image " + std::to_string(id) + " is not in the current row");
    set_device(*c);
    copy_codes_out(*c, c->S().row_imgs[it->second], coarse_out, fine_out);
  });
}

int bmg_match(bmg_context* c, const uint64_t* qids, const uint64_t* tids, uint64_t n_pairs,
              const bmg_match_params* mp, uint64_t* offsets_out, int32_t* matches_out,
              uint64_t capacity) {
  return guarded([&] {
    if (!c || !mp || !offsets_out || (n_pairs && (!qids || !tids)))
      fail(BMG_INVALID_ARGUMENT, "null argument");
    check_match_params(*c, *mp);
    if (!c->S().row_valid) fail(BMG_INVALID_ARGUMENT, "no row has been prepared");
    set_device(*c);
    std::vector<std::pair<int, int>> sp;
    uint64_t max_matches = 0;
    for (uint64_t p = 0; p < n_pairs; ++p) {
      const auto qi = c->S().row_slot.find(qids[p]);
      const auto ti = c->S().row_slot.find(tids[p]);
      if (qi == c->S().row_slot.end() || ti == c->S().row_slot.end())
        fail(BMG_INVALID_ARGUMENT, "pair image not in the current row");
      sp.emplace_back(qi->second, ti->second);
      max_matches += c->S().row_imgs[qi->second].n;
    }
    reset_results(*c, n_pairs, max_matches);
    enqueue_match(*c, sp, *mp, c->res_ranges.dev<uint64_t>(), c->d_res.as<int32_t>(), 0);
    if (n_pairs == 0) {
      offsets_out[0] = 0;
      return;
    }
    BMG_CUDA(cudaStreamSynchronize(c->S().s_comp));
    const uint64_t* ranges = c->res_ranges.host<uint64_t>();
    // one pass, so the pairs' ranges are contiguous from 0
    offsets_out[0] = 0;
    for (uint64_t p = 0; p < n_pairs; ++p) offsets_out[p + 1] = ranges[2 * p + 1];
    const uint64_t total = offsets_out[n_pairs];
    if (total > capacity) fail(BMG_INVALID_ARGUMENT, "match output capacity too small");
    if (total) {
      if (!matches_out) fail(BMG_INVALID_ARGUMENT, "null match output");
      std::memcpy(matches_out, fetch_log(*c, total), sizeof(int32_t) * 2 * total);
    }
  });
}

int bmg_compute_codes(bmg_context* c, const float* desc, uint64_t count, const float* mean,
                      uint32_t* coarse_out, uint64_t* fine_out) {
  return guarded([&] {
    if (!c || !mean || (count && (!desc || !coarse_out || !fine_out)))
      fail(BMG_INVALID_ARGUMENT, "null argument");
    set_device(*c);
    c->S().row_valid = false;
    c->d_tmp_desc.ensure(std::max<uint64_t>(count, 1) * 512 + proj_bytes(count, c->hd.proj_stride) + 16);
    BMG_CUDA(cudaStreamSynchronize(c->s_copy));
    for (cudaStream_t ps : c->s_proj) BMG_CUDA(cudaStreamSynchronize(ps));
    ArenaImage tmp;
    tmp.d = c->d_tmp_desc.as<float>();
    tmp.n = count;
    tmp.proj = tmp.d + count * kDim;
    tmp.dnorm = tmp.proj + count * c->hd.proj_stride;
    arena_copy(*c, tmp, Source{desc, nullptr, count});
    c->free_events.push_back(tmp.ev);
    std::vector<RowImage> one{RowImage{tmp.d, count, tmp.proj, tmp.dnorm}};
    prepare_row_views(*c, one, mean, nullptr, false);
    copy_codes_out(*c, c->S().row_imgs[0], coarse_out, fine_out);
  });
}

int bmg_match_pair(bmg_context* c, const float* qdesc, const bmg_code_set* qc, const float* tdesc,
                   const bmg_code_set* tc, const bmg_match_params* mp, int32_t* matches_out,
                   uint64_t* n_out) {
  return guarded([&] {
    if (!c || !qc || !tc || !mp || !n_out) fail(BMG_INVALID_ARGUMENT, "null argument");
    *n_out = 0;
    // hashmatch.cpp:105-113
    if (qc->function_seed != tc->function_seed)
      fail(BMG_HASH_MISMATCH, "code sets built from different hash function seeds");
    if (qc->params.tables != tc->params.tables || qc->params.coarse_bits != tc->params.coarse_bits ||
        qc->params.fine_bits != tc->params.fine_bits)
      fail(BMG_HASH_MISMATCH, "code sets built with different hash parameters");
    if (mp->k_nearest < 1) fail(BMG_INVALID_ARGUMENT, "k_nearest must be >= 1");
    check_match_params(*c, *mp);
    if (qc->count == 0 || tc->count == 0) return;  // :118
    if (qc->params.tables != c->hp.tables || qc->params.coarse_bits != c->hp.coarse_bits ||
        qc->params.fine_bits != c->hp.fine_bits)
      fail(BMG_HASH_MISMATCH, "code sets built with parameters other than this context's");
    if (!qdesc || !tdesc || !qc->coarse || !qc->fine || !tc->coarse || !tc->fine || !matches_out)
      fail(BMG_INVALID_ARGUMENT, "null data pointer");
    set_device(*c);
    c->S().row_valid = false;
    const HashDev& h = c->hd;
    const uint64_t nq = qc->count, nt = tc->count;
    // descriptors
    c->d_tmp_desc.ensure((nq + nt) * 512);
    BMG_CUDA(cudaStreamSynchronize(c->s_copy));
    BMG_CUDA(cudaStreamSynchronize(c->S().s_comp));
    float* dq = c->d_tmp_desc.as<float>();
    float* dt = dq + nq * kDim;
    stage_h2d(*c, dq, qdesc, nq * 512);
    stage_h2d(*c, dt, tdesc, nt * 512);
    c->pending_upload = true;
    // lay out two images (no codes computed: the given codes are uploaded)
    std::vector<std::pair<const float*, uint64_t>> two{{dq, nq}, {dt, nt}};
    // reuse the row layout, but skip the projection kernels: upload codes into place
    c->S().row_imgs.clear();
    {
      // layout only
      const int L = h.tables;
      const size_t NB = h.n_buckets;
      size_t off = 0;
      size_t co[2], fo[2], oo[2], cu[2], so[2], bo[2];
      for (int i = 0; i < 2; ++i) {
        co[i] = off; off = align_up(off + two[i].second * L * 4, 256);
        fo[i] = off; off = align_up(off + align_up(two[i].second, 2) * h.fwp * 8, 256);
      }
      for (int i = 0; i < 2; ++i) { oo[i] = off; off = align_up(off + L * (NB + 1) * 4, 256); }
      const size_t off_begin = oo[0], off_end = off;
      for (int i = 0; i < 2; ++i) {
        cu[i] = off; off = align_up(off + L * NB * 4, 256);
        const uint64_t ns = slot_stride(two[i].second, h.n_buckets, h.bucket_pad);
        so[i] = off; off = align_up(off + ns * L * 4, 256);
        bo[i] = off; off = align_up(off + ns * L * h.fwp * 8, 256);
      }
      c->S().d_scratch.ensure(off);
      char* base = c->S().d_scratch.as<char>();
      const bmg_code_set* sets[2] = {qc, tc};
      for (int i = 0; i < 2; ++i) {
        ImgDev im{};
        im.desc = two[i].first;
        im.n = static_cast<uint32_t>(two[i].second);
        im.coarse = reinterpret_cast<uint32_t*>(base + co[i]);
        im.fine = reinterpret_cast<uint64_t*>(base + fo[i]);
        im.offsets = reinterpret_cast<uint32_t*>(base + oo[i]);
        im.cursor = reinterpret_cast<uint32_t*>(base + cu[i]);
        im.slots = reinterpret_cast<uint32_t*>(base + so[i]);
        im.bfine = reinterpret_cast<uint64_t*>(base + bo[i]);
        im.ns = slot_stride(im.n, h.n_buckets, h.bucket_pad);
        c->S().row_imgs.push_back(im);
        const uint64_t n = two[i].second;
        for (uint64_t j = 0; j < n * L; ++j)
          if (sets[i]->coarse[j] >= static_cast<uint32_t>(h.n_buckets))
            fail(BMG_INVALID_ARGUMENT, "bucket id out of range for coarse_bits");
        uint32_t* hc = c->ring.alloc<uint32_t>(n * L, c->S().s_comp, c->s_copy);
        std::memcpy(hc, sets[i]->coarse, n * L * 4);
        meta_add(*c, im.coarse, hc, n * L * 4);
        uint64_t* hf = c->ring.alloc<uint64_t>(n * h.fwp, c->S().s_comp, c->s_copy);
        std::memset(hf, 0, n * h.fwp * 8);
        for (uint64_t j = 0; j < n; ++j)
          std::memcpy(hf + j * h.fwp, sets[i]->fine + j * h.fw, h.fw * 8);
        meta_add(*c, im.fine, hf, n * h.fwp * 8);
      }
      meta_add(*c, base + off_begin, nullptr, off_end - off_begin);
      ImgDev* hi = c->ring.alloc<ImgDev>(2, c->S().s_comp, c->s_copy);
      std::memcpy(hi, c->S().row_imgs.data(), sizeof(ImgDev) * 2);
      c->S().d_imgs.ensure(sizeof(ImgDev) * 2);
      meta_add(*c, c->S().d_imgs.p, hi, sizeof(ImgDev) * 2);
      // tables for the train image only (slot 1)
      const size_t n_tiles = (nt + kCodesTile - 1) / kCodesTile;
      uint32_t* ht = c->ring.alloc<uint32_t>(2 * n_tiles, c->S().s_comp, c->s_copy);
      for (size_t t = 0; t < n_tiles; ++t) {
        ht[t] = 1;
        ht[n_tiles + t] = static_cast<uint32_t>(t * kCodesTile);
      }
      c->S().d_tiles.ensure(sizeof(uint32_t) * 2 * n_tiles);
      meta_add(*c, c->S().d_tiles.p, ht, sizeof(uint32_t) * 2 * n_tiles);
      c->S().d_diag.ensure(sizeof(unsigned long long) * 4);
      meta_add(*c, c->S().d_diag.p, nullptr, sizeof(unsigned long long) * 4);
      meta_flush(*c);
      join_uploads(*c);
      // a 2-image table: the tile list covers image 1 only (the global-atomic
      // path); the fused shared-memory path builds both images' tables
      c->launches += launch_tables(h, c->S().d_imgs.as<ImgDev>(), c->S().d_tiles.as<uint32_t>(),
                                   c->S().d_tiles.as<uint32_t>() + n_tiles, static_cast<int>(n_tiles), 2,
                                   c->S().s_comp);
      check_launch();
    }
    std::vector<std::pair<int, int>> sp{{0, 1}};
    reset_results(*c, 1, nq);
    enqueue_match(*c, sp, *mp, c->res_ranges.dev<uint64_t>(), c->d_res.as<int32_t>(), 0);
    BMG_CUDA(cudaStreamSynchronize(c->S().s_comp));
    const uint64_t* offs = c->res_ranges.host<uint64_t>();
    const uint64_t total = offs[1] - offs[0];
    if (total)
      std::memcpy(matches_out, fetch_log(*c, offs[1]) + 2 * offs[0], sizeof(int32_t) * 2 * total);
    *n_out = total;
  });
}

namespace bmg {
namespace {
void execute_plan_impl(Ctx* c, const bmg_plan* plan, const std::unordered_map<uint64_t, Source>& fmap,
                       const bmg_execute_options* opts, bmg_result** out,
                       std::chrono::steady_clock::time_point t0);
}  // namespace
}  // namespace bmg

int bmg_execute_plan(bmg_context* c, const bmg_plan* plan, const bmg_feature_view* features,
                     uint64_t n_features, const bmg_execute_options* opts, bmg_result** out) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    if (!c || !plan || !opts || !out || (n_features && !features))
      fail(BMG_INVALID_ARGUMENT, "null argument");
    std::unordered_map<uint64_t, Source> fmap;
    for (uint64_t i = 0; i < n_features; ++i)
      fmap[features[i].image_id] = Source{features[i].descriptors, nullptr, features[i].count};
    execute_plan_impl(c, plan, fmap, opts, out, t0);
  });
}

int bmg_execute_plan_files(bmg_context* c, const bmg_plan* plan, const bmg_feature_file* files,
                           uint64_t n_files, const bmg_execute_options* opts, bmg_result** out) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    if (!c || !plan || !opts || !out || (n_files && !files)) fail(BMG_INVALID_ARGUMENT, "null argument");
    std::unordered_map<uint64_t, Source> fmap;
    for (uint64_t i = 0; i < n_files; ++i) {
      if (!files[i].path) fail(BMG_INVALID_ARGUMENT, "null feature file path");
      fmap[files[i].image_id] = Source{nullptr, files[i].path, files[i].count};
    }
    execute_plan_impl(c, plan, fmap, opts, out, t0);
  });
}

}  // extern "C"

namespace bmg {
namespace {
void execute_plan_impl(Ctx* c, const bmg_plan* plan, const std::unordered_map<uint64_t, Source>& fmap,
                       const bmg_execute_options* opts, bmg_result** out,
                       std::chrono::steady_clock::time_point t0) {
  {
    *out = nullptr;
    check_match_params(*c, opts->match);
    set_device(*c);
    auto features_of = [&](uint64_t id) -> const Source& {
      const auto it = fmap.find(id);
      if (it == fmap.end())
        fail(BMG_INVALID_ARGUMENT, "plan references image " + std::to_string(id) + " with no features");
      return it->second;
    };
    uint64_t total_rows = 0;
    for (uint64_t i = 0; i < plan->n_iterations; ++i) total_rows += plan->rows_per_iteration[i];
    if (total_rows != plan->n_rows) fail(BMG_INVALID_ARGUMENT, "rows_per_iteration does not sum to n_rows");
    const uint64_t n_pairs = plan->n_rows ? plan->row_pair_offsets[plan->n_rows] : 0;
    // row r's matches are packed into its own region [row_base[r], row_base[r+1])
    // of the result log (capacity: one match per query of each pair)
    std::vector<uint64_t> row_base(plan->n_rows + 1, 0);
    for (uint64_t r = 0; r < plan->n_rows; ++r) {
      uint64_t cap = 0;
      for (uint64_t p = plan->row_pair_offsets[r]; p < plan->row_pair_offsets[r + 1]; ++p) {
        const uint64_t a = plan->pairs[2 * p], b = plan->pairs[2 * p + 1];
        if (a >= b) fail(BMG_INVALID_ARGUMENT, "plan pairs must be (lower id, higher id)");
        cap += features_of(a).count;
      }
      row_base[r + 1] = row_base[r] + cap;
    }
    const uint64_t total_cap = row_base[plan->n_rows];
    auto res = std::make_unique<bmg_result>();
    // BMG_LOG_ZC=1 (A/B switch): every row compacts straight into pinned
    // host memory; default: only the call's last row does
    static const bool log_zc_all = [] {
      const char* v = getenv("BMG_LOG_ZC");
      return v && v[0] == '1';
    }();
    reset_results(*c, n_pairs, log_zc_all ? 0 : total_cap, false);
    res->log = static_cast<int32_t*>(PinnedPool::acquire(8 * std::max<uint64_t>(total_cap, 1), &res->log_bytes));
    uint64_t* d_off = c->res_ranges.dev<uint64_t>();
    int32_t* d_log = log_zc_all ? nullptr : c->d_res.as<int32_t>();
    int32_t* h_log = nullptr;
    BMG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_log), res->log, 0));
    res->row_handoff_ms.assign(plan->n_rows, -1.0);
    res->row_done_ms.assign(plan->n_rows, -1.0);
    std::vector<std::pair<uint64_t, cudaEvent_t>> row_done;  // (plan row, event)
    c->cur = 0;
    cudaEvent_t span0 = take_event(*c), span1 = take_event(*c);
    BMG_CUDA(cudaEventRecord(span0, c->slot[0].s_comp));
    // host origin of the row hand-off times: the moment span0 was issued to
    // the (idle) stream, so host and device times share an origin to within
    // the launch latency
    const auto t_span0 = std::chrono::steady_clock::now();
    BMG_CUDA(cudaStreamWaitEvent(c->s_copy, span0, 0));
    for (cudaStream_t ps : c->s_proj) BMG_CUDA(cudaStreamWaitEvent(ps, span0, 0));
    BMG_CUDA(cudaStreamWaitEvent(c->slot[1].s_comp, span0, 0));
    if ((opts->flags & BMG_EXEC_REPROJECT) && !c->resident.empty()) {
      // recompute the projections of every resident image inside this call
      // (one batched launch on slot 0; slot 1 waits for it)
      std::vector<ImgDev> v;
      for (const auto& kv : c->resident)
        if (kv.second.n) v.push_back(proj_view(kv.second));
      size_t n_tiles = 0;
      for (const ImgDev& im : v) n_tiles += (im.n + kCodesTile - 1) / kCodesTile;
      if (n_tiles) {
        ImgDev* hi = c->ring.alloc<ImgDev>(v.size(), c->slot[0].s_comp, c->s_copy);
        std::memcpy(hi, v.data(), sizeof(ImgDev) * v.size());
        uint32_t* ht = c->ring.alloc<uint32_t>(2 * n_tiles, c->slot[0].s_comp, c->s_copy);
        size_t t = 0;
        for (size_t i = 0; i < v.size(); ++i)
          for (uint32_t s0 = 0; s0 < v[i].n; s0 += kCodesTile, ++t) {
            ht[t] = static_cast<uint32_t>(i);
            ht[n_tiles + t] = s0;
          }
        const size_t ib = align_up(sizeof(ImgDev) * v.size(), 256);
        c->d_rp.ensure(ib + sizeof(uint32_t) * 2 * n_tiles);
        char* base = c->d_rp.as<char>();
        meta_add(*c, base, hi, sizeof(ImgDev) * v.size());
        meta_add(*c, base + ib, ht, sizeof(uint32_t) * 2 * n_tiles);
        meta_flush(*c);
        const uint32_t* dt = reinterpret_cast<const uint32_t*>(base + ib);
        {
          Timed tm(*c, "project", c->slot[0].s_comp);
          launch_project_tiles(c->hd, reinterpret_cast<const ImgDev*>(base), dt, dt + n_tiles,
                               static_cast<int>(n_tiles), c->slot[0].s_comp);
        }
        ++c->launches;
        check_launch();
        cudaEvent_t e = take_event(*c);
        BMG_CUDA(cudaEventRecord(e, c->slot[0].s_comp));
        BMG_CUDA(cudaStreamWaitEvent(c->slot[1].s_comp, e, 0));
        c->free_events.push_back(e);
      }
    }
    for (RowSlot& sl : c->slot) BMG_CUDA(cudaEventRecord(sl.done, sl.home));
    const bool retain = (opts->flags & BMG_EXEC_RETAIN) != 0;
    struct ChainHook {
      Ctx& c;
      ~ChainHook() {
        // failing part-way: queued D2H copies and zero-copy compactions may
        // still target the result's pinned log, which returns to the pool
        // when the result is destroyed right after this -- drain them first
        if (std::uncaught_exceptions() > 0) cudaDeviceSynchronize();
        c.mean_chain_only = false;
        c.cur = 0;
        for (RowSlot& sl : c.slot) {
          if (sl.s_comp != sl.home) cudaStreamWaitEvent(sl.home, sl.done, 0);
          sl.s_comp = sl.home;
        }
      }
    } chain_hook{*c};
    // declared after the hook: on an error it is joined (and its queued rows
    // drained) after the hook has synchronised the device
    std::unique_ptr<Collector> collector;
    if (opts->on_pair)
      collector = std::make_unique<Collector>(c->device, plan, opts, res->log, c->res_ranges.host<uint64_t>(),
                                              t_span0, res.get());
    for (RowSlot& sl : c->slot) BMG_CUDA(cudaEventRecord(sl.done, sl.home));
    c->mean_chain_only = (opts->flags & BMG_EXEC_MEAN_CHAIN) != 0;
    uint64_t row = 0;
    std::vector<uint64_t> missing;
    // BMG_TIMELINE=1: per-row event timeline on stderr (diagnostics)
    static const bool timeline = [] {
      const char* v = getenv("BMG_TIMELINE");
      return v && v[0] == '1';
    }();
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    auto mark = [&](const std::string& what, cudaStream_t st) {
      if (!timeline) return;
      cudaEvent_t e = take_event(*c);
      BMG_CUDA(cudaEventRecord(e, st));
      const double host_ms = 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      marks.emplace_back(what + " (host issue " + std::to_string(host_ms) + " ms)", e);
    };
    if (timeline) c->marks = &marks;
    uint64_t xrow = 0;  // rows issued so far (stream priority, slot)
    bool prio_late = false;
    for (uint64_t k = 0; k < plan->row_needed_offsets[plan->n_rows] && !prio_late; ++k)
      prio_late = !c->resident.count(plan->needed_ids[k]);
    if (const char* v = getenv("BMG_PRIO_LATE")) prio_late = v[0] == '1';  // A/B override
    for (uint64_t it = 0; it < plan->n_iterations; ++it) {
      const uint64_t row0 = row, nr = plan->rows_per_iteration[it];
      row += nr;
      const uint64_t up0 = c->uploads, units0 = c->units_uploaded;
      // ---- the arena in the reference's order (engine.cpp:438-444, 491-494):
      // capacity errors, counters and hooks exactly as the reference raises
      // them; the device work below may run the rows in another order
      std::unordered_set<uint64_t> logical;
      for (const auto& kv : c->resident) logical.insert(kv.first);
      std::unordered_map<uint64_t, uint64_t> evict_row;  // id -> plan row evicting it
      bool in_order = (opts->flags & BMG_EXEC_SERIAL) != 0;
      for (uint64_t r = row0; r < row0 + nr; ++r) {
        for (uint64_t k = plan->row_needed_offsets[r]; k < plan->row_needed_offsets[r + 1]; ++k) {
          const uint64_t id = plan->needed_ids[k];
          // needed again after its eviction in this iteration: the reference
          // re-uploads it (counted below); physically it never left HBM, and
          // only a later eviction (if any) frees it.  Rows then run in plan
          // order.
          if (evict_row.erase(id)) in_order = true;
          if (logical.count(id)) continue;
          const Source& fv = features_of(id);
          arena_account_upload(*c, id, fv.desc || fv.path, fv.count);
          if (opts->on_upload) opts->on_upload(opts->hook_user, id, fv.count);
          logical.insert(id);
        }
        for (uint64_t k = plan->row_evict_offsets[r]; !retain && k < plan->row_evict_offsets[r + 1]; ++k) {
          const uint64_t id = plan->evict_ids[k];
          if (!logical.count(id))
            fail(BMG_NOT_RESIDENT, "cannot evict image " + std::to_string(id) + ": not resident");
          const auto f = c->resident.find(id);
          arena_account_evict(*c, f != c->resident.end() ? f->second.n : features_of(id).count);
          if (opts->on_evict) opts->on_evict(opts->hook_user, id);
          logical.erase(id);
          evict_row[id] = r;
        }
      }
      // ---- device order: a row can only start once every image it needs
      // (its whole needed set: the row mean covers it) is in HBM, so the
      // first row's uploads are exposed.  Rows of an iteration are
      // independent: run first the row with the fewest bytes to upload, then
      // greedily the row with the fewest bytes still missing (for band plans
      // the reverse of the plan order).  Frees of images an earlier-run row
      // evicts wait until the last row that needs them has run.
      std::vector<uint64_t> order(nr);
      for (uint64_t i = 0; i < nr; ++i) order[i] = row0 + i;
      if (!in_order && nr > 1) {
        std::unordered_set<uint64_t> have;
        for (const auto& kv : c->resident) have.insert(kv.first);
        std::vector<char> done(nr, 0);
        for (uint64_t e = 0; e < nr; ++e) {
          uint64_t best = nr, best_units = ~0ull;
          for (uint64_t i = 0; i < nr; ++i) {
            if (done[i]) continue;
            uint64_t units = 0;
            for (uint64_t k = plan->row_needed_offsets[row0 + i]; k < plan->row_needed_offsets[row0 + i + 1]; ++k)
              if (!have.count(plan->needed_ids[k])) units += features_of(plan->needed_ids[k]).count + 1;
            if (units < best_units) best = i, best_units = units;  // ties: plan order
          }
          done[best] = 1;
          order[e] = row0 + best;
          for (uint64_t k = plan->row_needed_offsets[row0 + best]; k < plan->row_needed_offsets[row0 + best + 1]; ++k)
            have.insert(plan->needed_ids[k]);
        }
      }
      // position of each row in `order`, the last position needing each
      // image, when each evicted image can be freed, and the HBM peak (units)
      std::unordered_map<uint64_t, uint64_t> last_need;
      std::vector<std::vector<uint64_t>> frees;
      auto schedule = [&]() -> uint64_t {
        std::unordered_map<uint64_t, uint64_t> pos_of;
        last_need.clear();
        frees.assign(nr, {});
        for (uint64_t e = 0; e < nr; ++e) {
          pos_of[order[e]] = e;
          for (uint64_t k = plan->row_needed_offsets[order[e]]; k < plan->row_needed_offsets[order[e] + 1]; ++k)
            last_need[plan->needed_ids[k]] = e;
        }
        for (const auto& [id, r] : evict_row) {
          uint64_t e = pos_of[r];
          const auto f = last_need.find(id);
          if (f != last_need.end()) e = std::max(e, f->second);
          frees[e].push_back(id);
        }
        for (auto& v : frees) std::sort(v.begin(), v.end());
        std::unordered_set<uint64_t> have;
        uint64_t units = 0, peak = 0;
        for (const auto& kv : c->resident) have.insert(kv.first), units += kv.second.n;
        for (uint64_t e = 0; e < nr; ++e) {
          for (uint64_t k = plan->row_needed_offsets[order[e]]; k < plan->row_needed_offsets[order[e] + 1]; ++k)
            if (have.insert(plan->needed_ids[k]).second) units += features_of(plan->needed_ids[k]).count;
          peak = std::max(peak, units);
          for (uint64_t id : frees[e]) units -= features_of(id).count, have.erase(id);
        }
        return peak;
      };
      const uint64_t peak = schedule();
      if (peak > c->capacity && !std::is_sorted(order.begin(), order.end())) {
        // deferred frees would hold more than the arena's capacity: allowed
        // while the overshoot fits comfortably in free HBM, else plan order
        size_t free_b = 0, total_b = 0;
        BMG_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const uint64_t unit_b = 512 + sizeof(float) * (c->hd.proj_stride + 1);
        if ((peak - c->capacity) * unit_b > free_b / 2) {
          for (uint64_t i = 0; i < nr; ++i) order[i] = row0 + i;
          schedule();
        }
      }
      uint64_t it_pairs = 0;
      for (uint64_t e = 0; e < nr; ++e, ++xrow) {
        const uint64_t r = order[e];
        c->cur = (opts->flags & BMG_EXEC_SERIAL) ? 0 : static_cast<int>(xrow & 1);
        RowSlot& S = c->S();
        if (!(opts->flags & BMG_EXEC_SERIAL)) {
          // a call that uploads: the last rows get the highest priorities
          // (the last row's work after the last upload is the end-to-end
          // tail; its prep must not queue behind the previous row's match);
          // all images resident: earlier rows first (a row gates its slot's
          // next row)
          const uint64_t rank = prio_late ? total_rows - 1 - xrow : xrow;
          cudaStream_t st = rank < c->s_prio.size() ? c->s_prio[rank] : S.home;
          if (st != S.s_comp) BMG_CUDA(cudaStreamWaitEvent(st, S.done, 0));
          S.s_comp = st;
        }
        const uint64_t nb = plan->row_needed_offsets[r], ne = plan->row_needed_offsets[r + 1];
        const uint64_t* needed = plan->needed_ids + nb;
        // the row's missing images, copied in descending order of the last
        // row that needs them, so later rows can start before this row's
        // other images have arrived
        missing.clear();
        for (uint64_t k = nb; k < ne; ++k) {
          const uint64_t id = plan->needed_ids[k];
          if (!c->resident.count(id)) {
            arena_alloc(*c, id, features_of(id).count);
            missing.push_back(id);
          }
        }
        std::stable_sort(missing.begin(), missing.end(),
                         [&](uint64_t x, uint64_t y) { return last_need[x] > last_need[y]; });
        {
          std::vector<std::pair<ArenaImage*, const Source*>> mv;
          mv.reserve(missing.size());
          for (uint64_t id : missing) mv.emplace_back(&c->resident.at(id), &features_of(id));
          arena_copy_many(*c, mv, [&](size_t k) {
            if (timeline && k % 25 == 24) mark("row " + std::to_string(r) + " upload " + std::to_string(k + 1), c->s_copy);
          });
        }
        if (!missing.empty()) mark("row " + std::to_string(r) + " uploads done", c->s_copy);
        // the row's mean waits only for the copies (the copy stream is in
        // order: an event after this row's copies covers every earlier one);
        // its codes wait, per projection stream, for the last image of the
        // row that stream projected (its events are in stream order)
        {
          cudaEvent_t e = take_event(*c);
          BMG_CUDA(cudaEventRecord(e, c->s_copy));
          BMG_CUDA(cudaStreamWaitEvent(S.s_comp, e, 0));
          c->free_events.push_back(e);
        }
        const ArenaImage* last[bmg_context::kProjStreams] = {};
        for (uint64_t k = 0; k < ne - nb; ++k) {
          const auto f = c->resident.find(needed[k]);
          if (f == c->resident.end() || !f->second.ev) continue;
          const ArenaImage*& l = last[f->second.pstream];
          if (!l || f->second.seq > l->seq) l = &f->second;
        }
        c->proj_waits.clear();
        for (const ArenaImage* l : last)
          if (l) c->proj_waits.push_back(l->ev);
        c->pending_upload = false;
        mark("row " + std::to_string(r) + " start", S.s_comp);
        prepare_row(*c, needed, ne - nb, nullptr);
        mark("row " + std::to_string(r) + " codes+tables done", S.s_comp);
        const uint64_t pb = plan->row_pair_offsets[r], pe = plan->row_pair_offsets[r + 1];
        std::vector<std::pair<int, int>> sp;
        sp.reserve(pe - pb);
        for (uint64_t p = pb; p < pe; ++p) {
          const auto qa = S.row_slot.find(plan->pairs[2 * p]);
          const auto tb = S.row_slot.find(plan->pairs[2 * p + 1]);
          if (qa == S.row_slot.end() || tb == S.row_slot.end())
            fail(BMG_INVALID_ARGUMENT, "block pair image missing from the row's resident set");
          sp.emplace_back(qa->second, tb->second);
        }
        // a row's log region goes to the result's pinned buffer by DMA while
        // later rows compute; the call's last row, whose transfer nothing
        // hides, compacts straight into pinned host memory over PCIe (only
        // its matches cross, not its capacity-sized region)
        const bool log_dma = !log_zc_all && (it + 1 < plan->n_iterations || e + 1 < nr);
        enqueue_match(*c, sp, opts->match, d_off + 2 * pb, log_dma ? d_log : h_log, row_base[r]);
        mark("row " + std::to_string(r) + " match done", S.s_comp);
        if (log_dma && row_base[r + 1] > row_base[r])
          BMG_CUDA(cudaMemcpyAsync(res->log + 2 * row_base[r], d_log + 2 * row_base[r],
                                   8 * (row_base[r + 1] - row_base[r]), cudaMemcpyDeviceToHost, S.s_comp));
        it_pairs += pe - pb;
        {
          cudaEvent_t ev = take_event(*c);
          BMG_CUDA(cudaEventRecord(ev, S.s_comp));
          row_done.emplace_back(r, ev);
          if (collector) collector->push({ev, r, pb, pe});
        }
        for (uint64_t id : frees[e]) arena_free(*c, id);
        BMG_CUDA(cudaEventRecord(S.done, S.s_comp));
      }
      res->iterations.push_back(it_pairs);
      res->iterations.push_back(c->uploads - up0);
      res->iterations.push_back(c->units_uploaded - units0);
    }
    // join both slots' last rows into slot 0's home stream for the span end
    for (RowSlot& sl : c->slot) {
      BMG_CUDA(cudaStreamWaitEvent(c->slot[0].home, sl.done, 0));
      sl.s_comp = sl.home;
    }
    BMG_CUDA(cudaStreamWaitEvent(c->slot[1].home, c->slot[1].done, 0));
    BMG_CUDA(cudaEventRecord(span1, c->slot[0].home));
    BMG_CUDA(cudaStreamSynchronize(c->slot[0].home));
    for (auto& [what, e] : marks) {
      float ms = 0.f;
      BMG_CUDA(cudaEventSynchronize(e));
      BMG_CUDA(cudaEventElapsedTime(&ms, span0, e));
      fprintf(stderr, "[bmg timeline] %8.3f ms  %s\n", ms, what.c_str());
      c->free_events.push_back(e);
    }
    c->marks = nullptr;
    if (timeline)
      for (int k = 0; k < 2; ++k)
        if (c->slot[k].d_mean_state.p) {
          MeanState st{};
          BMG_CUDA(cudaMemcpy(&st, c->slot[k].d_mean_state.p, sizeof(st), cudaMemcpyDeviceToHost));
          fprintf(stderr, "[bmg timeline] slot %d mean: bad %u need_chain %u rounds %u events %u\n", k, st.bad,
                  st.need_chain, st.rounds, st.events);
        }
    if (collector) collector->finish();
    for (auto& [r, ev] : row_done) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, span0, ev) == cudaSuccess) res->row_done_ms[r] = ms;
      cudaGetLastError();
      c->free_events.push_back(ev);
    }
    // per-pair [begin, end) ranges are in mapped host memory; the matches
    // are already in the result's pinned log
    const uint64_t* ranges = c->res_ranges.host<uint64_t>();
    // results keyed and sorted by IdPair (engine.cpp:419, 506-512); a pair
    // planned twice keeps its last match list, like the reference's map
    std::map<std::pair<uint64_t, uint64_t>, uint64_t> last;
    for (uint64_t p = 0; p < n_pairs; ++p) last[{plan->pairs[2 * p], plan->pairs[2 * p + 1]}] = p;
    res->pair_ids.reserve(2 * last.size());
    res->ranges.reserve(2 * last.size());
    uint64_t total = 0;
    for (const auto& [key, p] : last) {
      res->pair_ids.push_back(key.first);
      res->pair_ids.push_back(key.second);
      const uint64_t b = ranges[2 * p], e = ranges[2 * p + 1];
      res->ranges.push_back(b);
      res->ranges.push_back(e);
      total += e - b;
    }
    res->n_matches = total;
    res->counters[0] = n_pairs;
    res->counters[1] = total;
    res->counters[2] = c->uploads;
    res->counters[3] = c->evictions;
    res->counters[4] = c->units_uploaded;
    res->counters[5] = c->peak;
    res->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    {
      float ms = 0.f;
      BMG_CUDA(cudaEventSynchronize(span1));
      BMG_CUDA(cudaEventElapsedTime(&ms, span0, span1));
      res->device_ms = ms;
      c->free_events.push_back(span0);
      c->free_events.push_back(span1);
    }
    *out = res.release();
  }
}
}  // namespace
}  // namespace bmg

extern "C" {

uint64_t bmg_result_pair_count(const bmg_result* r) { return r ? r->pair_ids.size() / 2 : 0; }
uint64_t bmg_result_match_count(const bmg_result* r) { return r ? r->n_matches : 0; }

int bmg_result_copy(const bmg_result* r, uint64_t* pair_ids, uint64_t* offsets, int32_t* matches) {
  return guarded([&] {
    if (!r) fail(BMG_INVALID_ARGUMENT, "null result");
    const size_t np = r->pair_ids.size() / 2;
    if (pair_ids && np) std::memcpy(pair_ids, r->pair_ids.data(), sizeof(uint64_t) * 2 * np);
    uint64_t o = 0;
    if (offsets) offsets[0] = 0;
    for (size_t p = 0; p < np; ++p) {
      const uint64_t b = r->ranges[2 * p], e = r->ranges[2 * p + 1];
      if (matches && e > b) std::memcpy(matches + 2 * o, r->log + 2 * b, sizeof(int32_t) * 2 * (e - b));
      o += e - b;
      if (offsets) offsets[p + 1] = o;
    }
  });
}

int bmg_result_view(const bmg_result* r, const uint64_t** pair_ids, const uint64_t** ranges,
                    const int32_t** log) {
  return guarded([&] {
    if (!r || !pair_ids || !ranges || !log) fail(BMG_INVALID_ARGUMENT, "null argument");
    *pair_ids = r->pair_ids.data();
    *ranges = r->ranges.data();
    *log = r->log;
  });
}

int bmg_result_write_matches(const bmg_result* r, const char* path) {
  if (!r) {
    bmg::set_last_error("null result");
    return BMG_INVALID_ARGUMENT;
  }
  return bmg_write_matches_binary(path, r->pair_ids.size() / 2, r->pair_ids.data(), r->ranges.data(), r->log,
                                  nullptr);
}

int bmg_result_metrics(const bmg_result* r, uint64_t counters_out[6], double* wall_s_out) {
  return guarded([&] {
    if (!r) fail(BMG_INVALID_ARGUMENT, "null result");
    if (counters_out) std::memcpy(counters_out, r->counters, sizeof(r->counters));
    if (wall_s_out) *wall_s_out = r->wall_s;
  });
}

uint64_t bmg_result_iteration_count(const bmg_result* r) { return r ? r->iterations.size() / 3 : 0; }

int bmg_result_iteration(const bmg_result* r, uint64_t i, uint64_t out3[3]) {
  return guarded([&] {
    if (!r || !out3 || i >= r->iterations.size() / 3) fail(BMG_INVALID_ARGUMENT, "bad iteration index");
    std::memcpy(out3, r->iterations.data() + 3 * i, sizeof(uint64_t) * 3);
  });
}

int bmg_result_device_ms(const bmg_result* r, double* ms_out) {
  return guarded([&] {
    if (!r || !ms_out) fail(BMG_INVALID_ARGUMENT, "null argument");
    *ms_out = r->device_ms;
  });
}

int bmg_result_row_timing(const bmg_result* r, uint64_t row, double out[2]) {
  return guarded([&] {
    if (!r || !out || row >= r->row_done_ms.size()) fail(BMG_INVALID_ARGUMENT, "bad row index");
    out[0] = r->row_handoff_ms[row];
    out[1] = r->row_done_ms[row];
  });
}

void bmg_result_free(bmg_result* r) { delete r; }

uint64_t bmg_launch_count(bmg_context* c) { return c ? c->launches : 0; }

// ---- retrieval: encode_vlad (retrieval.cpp:160-205) -----------------------
// Images are encoded in batches of up to 256 MiB of descriptors on
// the two row slots' home streams: batch b+1's uploads (pinned sources
// straight to the copy engine, pageable ones through the staging slots)
// overlap batch b's kernels; each batch's vectors are written by V3 into
// mapped pinned memory and copied to the caller's arrays once it completes.
namespace bmg {
namespace {
size_t vlad_batch_bytes() {  // BMG_VLAD_BATCH_BYTES: test hook (multi-batch paths)
  if (const char* e = std::getenv("BMG_VLAD_BATCH_BYTES")) return std::max<size_t>(std::strtoull(e, nullptr, 10), 1);
  return size_t(256) << 20;
}
}  // namespace
}  // namespace bmg

int bmg_encode_vlad(bmg_context* c, const float* centroids, int k_words, const bmg_feature_view* images,
                    uint64_t n_images, float* values_out, uint8_t* degenerate_out) {
  using namespace bmg;
  // the two batch slots persist in the context (no per-call allocation);
  // on any exit their last batches are waited for
  auto cleanup = [&] {
    if (!c) return;
    for (VladSlot& v : c->vlad) {
      if (v.done) cudaEventSynchronize(v.done);
      v.imgs.clear();
    }
  };
  const int rc = guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null argument");
    VladSlot* vs = c->vlad;
    for (int k = 0; k < 2; ++k) vs[k].imgs.clear();
    if (k_words < 1) fail(BMG_INVALID_ARGUMENT, "codebook has no words");  // retrieval.cpp:161
    if (k_words > kVladMaxWords)
      fail(BMG_UNSUPPORTED, "codebooks of more than " + std::to_string(kVladMaxWords) +
                                " words are not supported by the GPU VLAD encoder");
    if (!centroids || (n_images && (!images || !values_out || !degenerate_out)))
      fail(BMG_INVALID_ARGUMENT, "null argument");
    for (uint64_t i = 0; i < n_images; ++i)
      if (images[i].count && !images[i].descriptors) fail(BMG_INVALID_ARGUMENT, "null descriptors");
    set_device(*c);
    const size_t dim = static_cast<size_t>(k_words) * kDim;
    DevBuf d_cent;
    d_cent.ensure(dim * sizeof(float));
    BMG_CUDA(cudaMemcpy(d_cent.p, centroids, dim * sizeof(float), cudaMemcpyHostToDevice));
    auto drain = [&](VladSlot& v) {
      if (v.imgs.empty()) return;
      BMG_CUDA(cudaEventSynchronize(v.done));
      const float* vals = v.out.host<float>();
      const uint8_t* deg = reinterpret_cast<const uint8_t*>(vals + v.imgs.size() * dim);
      for (size_t j = 0; j < v.imgs.size(); ++j) {
        std::memcpy(values_out + v.imgs[j] * dim, vals + j * dim, dim * sizeof(float));
        degenerate_out[v.imgs[j]] = deg[j];
      }
      v.imgs.clear();
    };
    for (int k = 0; k < 2; ++k)
      if (!vs[k].done) BMG_CUDA(cudaEventCreateWithFlags(&vs[k].done, cudaEventDisableTiming));
    int si = 0;
    const size_t batch_bytes = vlad_batch_bytes();
    for (uint64_t i0 = 0; i0 < n_images;) {
      // the batch: images [i0, i1)
      uint64_t i1 = i0, desc_total = 0, tiles = 0;
      while (i1 < n_images && (i1 == i0 || (desc_total + images[i1].count) * kDim * sizeof(float) <= batch_bytes)) {
        desc_total += images[i1].count;
        tiles += (images[i1].count + kVladTile - 1) / kVladTile;
        ++i1;
      }
      const uint64_t nb = i1 - i0;
      VladSlot& v = vs[si];
      RowSlot& rs = c->slot[si];
      si ^= 1;
      drain(v);  // the slot's previous batch (its buffers are reused below)
      v.desc.ensure(std::max<uint64_t>(desc_total, 1) * kDim * sizeof(float));
      v.assign.ensure(std::max<uint64_t>(desc_total, 1) * sizeof(int32_t));
      v.fix.ensure(std::max<uint64_t>(desc_total, 1) * sizeof(uint2));
      v.fixcnt.ensure(16);
      v.acc.ensure(nb * dim * sizeof(double));
      v.members.ensure(std::max<uint64_t>(desc_total, 1) * sizeof(uint32_t));
      v.member_off.ensure(nb * (k_words + 1) * sizeof(uint32_t));
      const size_t meta_bytes = align_up(nb * sizeof(VladImg) + 2 * std::max<uint64_t>(tiles, 1) * sizeof(uint32_t), 16);
      v.meta.ensure(meta_bytes);
      v.dmeta.ensure(meta_bytes);
      v.out.ensure(nb * dim * sizeof(float) + nb);
      VladImg* mi = v.meta.host<VladImg>();
      uint32_t* t_img = reinterpret_cast<uint32_t*>(mi + nb);
      uint32_t* t_start = t_img + std::max<uint64_t>(tiles, 1);
      float* dd = v.desc.as<float>();
      uint64_t off = 0, t = 0;
      for (uint64_t j = 0; j < nb; ++j) {
        const bmg_feature_view& f = images[i0 + j];
        if (f.count > 0xffffffffull) fail(BMG_UNSUPPORTED, "image too large for the VLAD encoder");
        mi[j].desc = dd + off * kDim;
        mi[j].n = static_cast<uint32_t>(f.count);
        mi[j].pad_ = 0;
        mi[j].assign_off = off;
        for (uint64_t r = 0; r < f.count; r += kVladTile) {
          t_img[t] = static_cast<uint32_t>(j);
          t_start[t] = static_cast<uint32_t>(r);
          ++t;
        }
        stage_h2d(*c, dd + off * kDim, f.descriptors, f.count * kDim * sizeof(float));
        off += f.count;
        v.imgs.push_back(i0 + j);
      }
      cudaEvent_t copied = take_event(*c);
      BMG_CUDA(cudaEventRecord(copied, c->s_copy));
      BMG_CUDA(cudaStreamWaitEvent(rs.home, copied, 0));
      c->free_events.push_back(copied);
      // image / tile tables into device memory by a kernel (reading them
      // over PCIe from every CTA would stall it; a memcpy would queue
      // behind the bulk uploads on the copy engine)
      MetaBatch mb{};
      mb.op[0] = MetaOp{v.dmeta.p, v.meta.dev<void>(), meta_bytes};
      mb.op[1] = MetaOp{v.fixcnt.p, nullptr, 16};
      mb.n = 2;
      launch_meta(mb, rs.home);
      VladBatch b{};
      b.imgs = v.dmeta.as<VladImg>();
      b.tile_img = reinterpret_cast<const uint32_t*>(b.imgs + nb);
      b.tile_start = b.tile_img + std::max<uint64_t>(tiles, 1);
      b.centroids = d_cent.as<float>();
      b.k_words = k_words;
      b.assign = v.assign.as<int32_t>();
      b.fix = v.fix.as<uint2>();
      b.fix_count = v.fixcnt.as<uint32_t>();
      b.fix_cap = static_cast<uint32_t>(std::max<uint64_t>(desc_total, 1));
      b.members = v.members.as<uint32_t>();
      b.member_off = v.member_off.as<uint32_t>();
      b.acc = v.acc.as<double>();
      b.values = v.out.dev<float>();
      b.degenerate = reinterpret_cast<uint8_t*>(b.values + nb * dim);
      {
        Timed tm(*c, "vlad", rs.home);
        launch_vlad(b, static_cast<int>(nb), static_cast<int>(tiles), rs.home);
        c->launches += tiles ? 6 : 4;
        check_launch();
      }
      BMG_CUDA(cudaEventRecord(v.done, rs.home));
      i0 = i1;
    }
    drain(vs[si]);
    drain(vs[si ^ 1]);
    // the staging slots / copy stream are idle again before d_cent goes
    BMG_CUDA(cudaStreamSynchronize(c->s_copy));
    d_cent.release();
  });
  cleanup();
  return rc;
}

int bmg_train_codebook(bmg_context* c, const float* desc, uint64_t n, int k_words, int max_iters, uint64_t seed,
                       float* centroids_out, double* sse_out, int* n_sse_out) {
  using namespace bmg;
  return guarded([&] {
    if (!c || !centroids_out || !n_sse_out) fail(BMG_INVALID_ARGUMENT, "null argument");
    // argument checks in the reference's order (retrieval.cpp:59-64)
    if (k_words < 1) fail(BMG_INVALID_ARGUMENT, "k_words must be >= 1");
    if (max_iters < 1) fail(BMG_INVALID_ARGUMENT, "max_iters must be >= 1");
    if (n < static_cast<uint64_t>(k_words))
      fail(BMG_TOO_FEW_DESCRIPTORS,
           "need at least " + std::to_string(k_words) + " descriptors, got " + std::to_string(n));
    if (k_words > kVladMaxWords)
      fail(BMG_UNSUPPORTED, "codebooks of more than " + std::to_string(kVladMaxWords) +
                                " words are not supported by the GPU k-means");
    if (n > 0xffffffffull) fail(BMG_UNSUPPORTED, "training pools of 2^32 descriptors or more");
    if (!desc) fail(BMG_INVALID_ARGUMENT, "null descriptors");
    set_device(*c);
    *n_sse_out = 0;
    const size_t K = static_cast<size_t>(k_words), dimk = K * kDim;
    // initial centroids: k distinct descriptor values in shuffled order (:69-96)
    std::vector<uint64_t> order(n);
    for (uint64_t i = 0; i < n; ++i) order[i] = i;
    std::mt19937_64 rng(seed);
    std::shuffle(order.begin(), order.end(), rng);
    std::vector<double> cent(dimk);
    size_t picked = 0;
    for (uint64_t idx : order) {
      if (picked == K) break;
      const float* d = desc + idx * kDim;
      bool duplicate = false;
      for (size_t k = 0; k < picked && !duplicate; ++k) {
        const double* cc = cent.data() + k * kDim;
        duplicate = true;
        for (int j = 0; j < kDim; ++j)
          if (static_cast<double>(d[j]) != cc[j]) {
            duplicate = false;
            break;
          }
      }
      if (duplicate) continue;
      for (int j = 0; j < kDim; ++j) cent[picked * kDim + j] = d[j];
      ++picked;
    }
    if (picked < K)
      fail(BMG_TOO_FEW_DESCRIPTORS, "fewer than " + std::to_string(k_words) + " distinct descriptor values");
    // device state: the pool as one "image", tiles of 128
    cudaStream_t s = c->slot[0].home;
    const uint64_t tiles = (n + kVladTile - 1) / kVladTile;
    DevBuf d_desc, d_cent32, d_cent64, d_zero, d_assign, d_fix, d_fixcnt, d_d2, d_members, d_moff, d_sums, d_meta;
    d_desc.ensure(n * kDim * sizeof(float));
    d_cent32.ensure(dimk * sizeof(float));
    d_cent64.ensure(dimk * sizeof(double));
    d_zero.ensure(dimk * sizeof(float));
    d_assign.ensure(n * sizeof(int32_t));
    d_fix.ensure(n * sizeof(uint2));
    d_fixcnt.ensure(16);
    d_d2.ensure(n * sizeof(double));
    d_members.ensure(n * sizeof(uint32_t));
    d_moff.ensure((K + 1) * sizeof(uint32_t));
    d_sums.ensure(dimk * sizeof(double));
    const size_t meta_bytes = align_up(sizeof(VladImg) + 2 * tiles * sizeof(uint32_t), 16);
    d_meta.ensure(meta_bytes);
    {
      std::vector<char> meta(meta_bytes, 0);
      VladImg* mi = reinterpret_cast<VladImg*>(meta.data());
      mi->desc = d_desc.as<float>();
      mi->n = static_cast<uint32_t>(n);
      mi->assign_off = 0;
      uint32_t* ti = reinterpret_cast<uint32_t*>(mi + 1);
      for (uint64_t t = 0; t < tiles; ++t) {
        ti[t] = 0;
        ti[tiles + t] = static_cast<uint32_t>(t * kVladTile);
      }
      BMG_CUDA(cudaMemcpyAsync(d_meta.p, meta.data(), meta_bytes, cudaMemcpyHostToDevice, s));
      BMG_CUDA(cudaMemsetAsync(d_zero.p, 0, dimk * sizeof(float), s));
      stage_h2d(*c, d_desc.p, desc, n * kDim * sizeof(float));
      cudaEvent_t e = take_event(*c);
      BMG_CUDA(cudaEventRecord(e, c->s_copy));
      BMG_CUDA(cudaStreamWaitEvent(s, e, 0));
      c->free_events.push_back(e);
    }
    VladBatch b{};
    b.imgs = d_meta.as<VladImg>();
    b.tile_img = reinterpret_cast<const uint32_t*>(b.imgs + 1);
    b.tile_start = b.tile_img + tiles;
    b.k_words = k_words;
    b.assign = d_assign.as<int32_t>();
    b.fix = d_fix.as<uint2>();
    b.fix_count = d_fixcnt.as<uint32_t>();
    b.fix_cap = static_cast<uint32_t>(n);
    b.members = d_members.as<uint32_t>();
    b.member_off = d_moff.as<uint32_t>();
    b.acc = d_sums.as<double>();
    b.cent64 = d_cent64.as<double>();
    b.point_d2 = d_d2.as<double>();
    std::vector<int32_t> assign(n), prev(n, -1);
    std::vector<double> d2(n), sums(dimk);
    std::vector<float> c32(dimk);
    for (int iter = 0; iter < max_iters; ++iter) {
      // ---- assignment (:99-117) on the device
      float cmax = 0.f;
      for (size_t k = 0; k < K; ++k) {
        double nn = 0.0;
        for (int j = 0; j < kDim; ++j) {
          c32[k * kDim + j] = static_cast<float>(cent[k * kDim + j]);
          nn += cent[k * kDim + j] * cent[k * kDim + j];
        }
        cmax = std::max(cmax, static_cast<float>(std::sqrt(nn)) * 1.0001f);
      }
      if (!std::isfinite(cmax)) cmax = std::numeric_limits<float>::infinity();
      BMG_CUDA(cudaMemcpyAsync(d_cent32.p, c32.data(), dimk * sizeof(float), cudaMemcpyHostToDevice, s));
      BMG_CUDA(cudaMemcpyAsync(d_cent64.p, cent.data(), dimk * sizeof(double), cudaMemcpyHostToDevice, s));
      BMG_CUDA(cudaMemsetAsync(d_fixcnt.p, 0, 16, s));
      b.centroids = d_cent32.as<float>();
      b.cnorm_max = cmax;
      {
        Timed tm(*c, "kmeans", s);
        launch_kmeans_assign(b, static_cast<int>(tiles), s);
        c->launches += 3;
        check_launch();
      }
      BMG_CUDA(cudaMemcpyAsync(assign.data(), d_assign.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      BMG_CUDA(cudaMemcpyAsync(d2.data(), d_d2.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
      BMG_CUDA(cudaStreamSynchronize(s));
      double sse = 0.0;  // in point order, as the reference
      for (uint64_t i = 0; i < n; ++i) sse += d2[i];
      if (sse_out) sse_out[iter] = sse;
      *n_sse_out = iter + 1;
      if (assign == prev) break;
      prev = assign;
      // ---- update (:121-136): FP64 sums in point order on the device
      b.centroids = d_zero.as<float>();  // the residual chains with zero centroids: plain sums
      {
        Timed tm(*c, "kmeans", s);
        launch_kmeans_sums(b, s);
        c->launches += 2;
        check_launch();
      }
      BMG_CUDA(cudaMemcpyAsync(sums.data(), d_sums.p, dimk * sizeof(double), cudaMemcpyDeviceToHost, s));
      BMG_CUDA(cudaStreamSynchronize(s));
      std::vector<uint64_t> counts(K, 0);
      for (uint64_t i = 0; i < n; ++i) ++counts[static_cast<size_t>(assign[i])];
      for (size_t k = 0; k < K; ++k) {
        if (counts[k] == 0) continue;
        const double inv = 1.0 / static_cast<double>(counts[k]);
        for (int j = 0; j < kDim; ++j) cent[k * kDim + j] = sums[k * kDim + j] * inv;
      }
      // empty clusters take the point worst served by its centroid (:137-147)
      for (size_t k = 0; k < K; ++k) {
        if (counts[k] != 0) continue;
        uint64_t far = 0;
        for (uint64_t i = 1; i < n; ++i)
          if (d2[i] > d2[far]) far = i;
        for (int j = 0; j < kDim; ++j) cent[k * kDim + j] = desc[far * kDim + j];
        d2[far] = 0.0;
      }
    }
    for (size_t i = 0; i < dimk; ++i) centroids_out[i] = static_cast<float>(cent[i]);
    BMG_CUDA(cudaStreamSynchronize(c->s_copy));
  });
}

int bmg_set_profiling(bmg_context* c, int enabled) {
  return guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null context");
    set_device(*c);
    for (cudaStream_t ps : c->s_proj) BMG_CUDA(cudaStreamSynchronize(ps));
    for (RowSlot& sl : c->slot) BMG_CUDA(cudaStreamSynchronize(sl.s_comp));
    for (auto& t : c->timers) {
      c->free_events.push_back(t.a);
      c->free_events.push_back(t.b);
    }
    c->timers.clear();
    c->profiling = enabled != 0;
  });
}

int bmg_kernel_time(bmg_context* c, const char* cls, double* total_ms, uint64_t* launches) {
  return guarded([&] {
    if (!c || !cls) fail(BMG_INVALID_ARGUMENT, "null argument");
    set_device(*c);
    for (cudaStream_t ps : c->s_proj) BMG_CUDA(cudaStreamSynchronize(ps));
    for (RowSlot& sl : c->slot) {
      BMG_CUDA(cudaStreamSynchronize(sl.s_comp));
      BMG_CUDA(cudaStreamSynchronize(sl.home));
    }
    double ms = 0.0;
    uint64_t n = 0;
    for (auto& t : c->timers) {
      if (t.cls != cls) continue;
      float x = 0.f;
      BMG_CUDA(cudaEventElapsedTime(&x, t.a, t.b));
      ms += x;
      ++n;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = n;
  });
}

int bmg_fixup_counts(bmg_context* c, uint64_t* code_bits, uint64_t* rerank_queries) {
  return guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null context");
    set_device(*c);
    unsigned long long d[4] = {0, 0, 0, 0};
    if (c->S().d_diag.p) {
      BMG_CUDA(cudaMemcpyAsync(d, c->S().d_diag.p, sizeof(d), cudaMemcpyDeviceToHost, c->S().s_comp));
      BMG_CUDA(cudaStreamSynchronize(c->S().s_comp));
    }
    if (code_bits) *code_bits = d[0];
    if (rerank_queries) *rerank_queries = d[1];
  });
}

int bmg_exact_walk_count(bmg_context* c, uint64_t* queries) {
  return guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null context");
    set_device(*c);
    unsigned long long d[4] = {0, 0, 0, 0};
    if (c->S().d_diag.p) {
      BMG_CUDA(cudaMemcpyAsync(d, c->S().d_diag.p, sizeof(d), cudaMemcpyDeviceToHost, c->S().s_comp));
      BMG_CUDA(cudaStreamSynchronize(c->S().s_comp));
    }
    if (queries) *queries = d[2];
  });
}

int bmg_set_test_flags(bmg_context* c, uint32_t flags) {
  return guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null context");
    if (flags & ~(BMG_TEST_FORCE_EXACT_WALK | BMG_TEST_FORCE_FP64_RERANK))
      fail(BMG_INVALID_ARGUMENT, "unknown test flag");
    c->test_flags = flags;
  });
}

int bmg_row_mean_info(bmg_context* c, uint32_t* rounds, int* used_chain) {
  return guarded([&] {
    if (!c) fail(BMG_INVALID_ARGUMENT, "null context");
    set_device(*c);
    MeanState st{};
    if (c->S().d_mean_state.p && !c->S().last_mean_chain_only) {
      BMG_CUDA(cudaMemcpyAsync(&st, c->S().d_mean_state.p, sizeof(st), cudaMemcpyDeviceToHost, c->S().s_comp));
      BMG_CUDA(cudaStreamSynchronize(c->S().s_comp));
    }
    if (rounds) *rounds = st.rounds;
    if (used_chain) *used_chain = (c->S().last_mean_chain_only || st.need_chain) ? 1 : 0;
  });
}

}  // extern "C"
