// ft_capi.cu -- the extern "C" boundary (include/fasttrig_b200.h).
//
// Argument validation, status codes and a thread-local error string; the
// host-pointer batch entry points (the reference's std::span -> std::vector
// API, R:proj/include/fasttrig/kernels.hpp:84-94) as a chunked H2D / K1 / D2H
// pipeline over three streams; grid sizing; the host bisection that derives
// the fast path's quadrant / pole-guard thresholds from IEEE division and
// subtraction (their compiled-in copies must match it bit for bit, see
// ft_thresholds and tests/test_capi_host.py).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <memory>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "ft_internal.h"

namespace ft {
namespace {

thread_local std::string g_err;
std::atomic<std::uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FT_OK;
  (void)cudaGetLastError();  // clear sticky-free errors
  const int code = e == cudaErrorMemoryAllocation ? FT_ERR_OOM
                   : e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? FT_ERR_NO_DEVICE
                                                                                 : FT_ERR_CUDA;
  return fail(code, std::string(where) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e));
}

// ---- thresholds (host, binary64, no contraction: see Makefile flags) ----
template <class Pred>
double first_true(double lo, double hi, Pred pred) {
  // pred is monotone false..true on [lo, hi], lo >= 0, pred(lo) false,
  // pred(hi) true.  Bisect on bit patterns (ordered like the values for >= 0).
  std::uint64_t l, h;
  std::memcpy(&l, &lo, 8);
  std::memcpy(&h, &hi, 8);
  while (h - l > 1) {
    const std::uint64_t m = l + (h - l) / 2;
    double dm;
    std::memcpy(&dm, &m, 8);
    if (pred(dm)) h = m;
    else l = m;
  }
  double r;
  std::memcpy(&r, &h, 8);
  return r;
}

struct Thresholds {
  double quad[3];
  double guard;
};

Thresholds compute_thresholds() {
  Thresholds t{};
  volatile double hp = kHalfPi;  // keep the divisions as IEEE divisions
  for (int j = 1; j <= 3; ++j) {
    t.quad[j - 1] = first_true(0.0, kTwoPi, [&](double r) { return std::floor(r / hp) >= j; });
  }
  t.guard = first_true(0.0, kHalfPi,
                       [&](double red) { return std::fabs(red - hp) < kTanPoleGuard; });
  return t;
}

const Thresholds& thresholds() {
  static const Thresholds t = compute_thresholds();
  return t;
}

// ---- device info ----
constexpr int kMaxDevices = 128;
std::mutex g_mu;
std::unordered_map<const void*, int> g_occ;  // kernel -> resident blocks/SM
int g_sms[kMaxDevices] = {0};

// The calling thread's CUDA device, or -1 (with the CUDA error in *err) when
// the runtime cannot report one.
int current_device(cudaError_t* err = nullptr) {
  int d = -1;
  const cudaError_t e = cudaGetDevice(&d);
  if (err) *err = e;
  return e == cudaSuccess ? d : -1;
}

int device_or_fail(int* dev) {
  cudaError_t e;
  *dev = current_device(&e);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  if (*dev >= kMaxDevices) return fail(FT_ERR_CUDA, "device index >= 128 is not supported");
  return FT_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15u) == 0; }

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int check_common(int dtype, unsigned mask, std::size_t n, const void* x, void* const out[3]) {
  if (dtype != FT_F32 && dtype != FT_F64) return fail(FT_ERR_INVALID_ARG, "dtype must be FT_F32 or FT_F64");
  if (mask == 0 || mask > 7) return fail(FT_ERR_INVALID_ARG, "mask must select 1..3 of sin/cos/tan");
  if (n == 0) return FT_OK;
  if (!x) return fail(FT_ERR_INVALID_ARG, "x is NULL");
  for (int j = 0; j < 3; ++j)
    if ((mask & (1u << j)) && !out[j]) return fail(FT_ERR_INVALID_ARG, "a selected output pointer is NULL");
  return FT_OK;
}

EvalArgs make_args(const void* x, std::size_t n, unsigned mask, void* const out[3],
                   std::uint8_t* seg_sc, std::uint8_t* seg_t, int steps) {
  EvalArgs a{};
  a.x = x;
  for (int j = 0; j < 3; ++j) a.out[j] = (mask & (1u << j)) ? out[j] : nullptr;
  a.seg_sc = seg_sc;
  a.seg_t = seg_t;
  a.n = n;
  a.steps = steps;
  bool ok = aligned16(x);
  for (int j = 0; j < 3; ++j) ok = ok && (a.out[j] == nullptr || aligned16(a.out[j]));
  // segment bytes are written one per element; any alignment works.
  a.vec_ok = ok ? 1 : 0;
  return a;
}

int sqrt_kind(ft_sqrt_mode m) {
  if (m.method == FT_SQRT_EXACT) return kExact;
  return m.newton_steps == 1 ? kFisr1 : m.newton_steps == 2 ? kFisr2 : kFisrN;
}

int check_mode(ft_sqrt_mode m) {
  if (m.method != FT_SQRT_EXACT && m.method != FT_SQRT_FISR)
    return fail(FT_ERR_INVALID_ARG, "sqrt mode method must be 0 (exact) or 1 (fisr)");
  return FT_OK;
}

// ---- host pipeline state (per device) ----
constexpr int kPipe = 3;
struct HostPipe {
  std::mutex mu;
  bool init = false;
  cudaStream_t st[kPipe]{};
  void* buf[kPipe][4]{};  // x, sin, cos, tan
  std::size_t cap_bytes = 0;
};
HostPipe g_pipe[kMaxDevices];

int pipe_reserve(HostPipe& p, std::size_t bytes) {
  if (!p.init) {
    for (auto& s : p.st) {
      cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_status(e, "cudaStreamCreate");
    }
    p.init = true;
  }
  if (bytes <= p.cap_bytes) return FT_OK;
  for (auto& row : p.buf)
    for (auto& b : row) {
      if (b) cudaFree(b);
      b = nullptr;
    }
  p.cap_bytes = 0;
  for (auto& row : p.buf)
    for (auto& b : row) {
      cudaError_t e = cudaMalloc(&b, bytes);
      if (e != cudaSuccess) return cuda_status(e, "cudaMalloc(host pipeline)");
    }
  p.cap_bytes = bytes;
  return FT_OK;
}

// Pageable host memory (e.g. the std::vector the reference API returns) goes
// through a pinned staging ring: parallel host memcpys into / out of pinned
// slots, overlapped with the H2D / kernel / D2H streams of other chunks.
// Bytes per array per staged chunk (16 MiB: 2 Mi f64 / 4 Mi f32 elements;
// FT_STAGE_MB overrides it for measurements).
std::size_t stage_bytes() {
  static const std::size_t b = [] {
    const char* e = std::getenv("FT_STAGE_MB");
    const long mb = e ? std::atol(e) : 16;
    return static_cast<std::size_t>(mb >= 1 && mb <= 256 ? mb : 16) << 20;
  }();
  return b;
}
struct Staging {
  void* pin[kPipe][4]{};  // x, sin, cos, tan
  cudaEvent_t done[kPipe]{};
  std::size_t cap_bytes = 0;
};
Staging g_stage[kMaxDevices];

bool host_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice ||
         at.type == cudaMemoryTypeManaged;
}

int stage_reserve(Staging& g, std::size_t bytes) {
  if (!g.done[0]) {
    for (auto& e : g.done) {
      cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      if (r != cudaSuccess) return cuda_status(r, "cudaEventCreate");
    }
  }
  if (bytes <= g.cap_bytes) return FT_OK;
  for (auto& row : g.pin)
    for (auto& b : row) {
      if (b) cudaFreeHost(b);
      b = nullptr;
    }
  g.cap_bytes = 0;
  for (auto& row : g.pin)
    for (auto& b : row) {
      cudaError_t r = cudaHostAlloc(&b, bytes, cudaHostAllocDefault);
      if (r != cudaSuccess) return cuda_status(r, "cudaHostAlloc(staging)");
    }
  g.cap_bytes = bytes;
  return FT_OK;
}

// A batch of memcpys split into ~4 MiB parts over a persistent pool of up to 16
// host threads (one core moves ~10 GB/s; the staged path needs ~32 B per
// element through memory).  The pool replaces per-chunk std::thread spawning
// (~2000 thread creations per 2^28-element call); the calling thread works on
// its own job too, and concurrent callers (one per device in host_sharded)
// share the workers.
extern "C" void ft_copy_stream(void* dst, const void* src, std::size_t n);  // ft_hostcopy.cpp
// FT_HOST_NT=0 in the environment keeps the cached memcpy (measurements).
bool stream_copies() {
  static const bool on = [] {
    const char* e = std::getenv("FT_HOST_NT");
    return !(e && e[0] == '0');
  }();
  return on;
}

struct Copy {
  void* dst;
  const void* src;
  std::size_t bytes;
};

class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }

  void run(std::vector<Copy> parts) {
    if (parts.empty()) return;
    auto job = std::make_shared<Job>();
    job->parts = std::move(parts);
    if (!th_.empty() && job->parts.size() > 1) {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(job);
      cv_.notify_all();
    }
    work(*job);
    std::unique_lock<std::mutex> lk(job->m);
    job->cv.wait(lk, [&] { return job->done.load() == job->parts.size(); });
    lk.unlock();
    std::lock_guard<std::mutex> ql(mu_);
    for (auto it = q_.begin(); it != q_.end(); ++it)
      if (*it == job) {
        q_.erase(it);
        break;
      }
  }

  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      cv_.notify_all();
    }
    for (auto& t : th_) t.join();
  }

 private:
  struct Job {
    std::vector<Copy> parts;
    std::atomic<std::size_t> next{0}, done{0};
    std::mutex m;
    std::condition_variable cv;
  };

  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned n = std::min(16u, hw ? hw : 1u);
    for (unsigned i = 1; i < n; ++i) th_.emplace_back([this] { worker(); });
  }

  static void work(Job& j) {
    std::size_t i;
    while ((i = j.next.fetch_add(1)) < j.parts.size()) {
      if (stream_copies()) ft_copy_stream(j.parts[i].dst, j.parts[i].src, j.parts[i].bytes);
      else std::memcpy(j.parts[i].dst, j.parts[i].src, j.parts[i].bytes);
      if (j.done.fetch_add(1) + 1 == j.parts.size()) {
        std::lock_guard<std::mutex> lk(j.m);
        j.cv.notify_all();
      }
    }
  }

  void worker() {
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
      if (stop_) return;
      std::shared_ptr<Job> j;
      for (auto& cand : q_)
        if (cand->next.load() < cand->parts.size()) {
          j = cand;
          break;
        }
      if (!j) {  // every queued job is fully claimed: wait for the next one
        cv_.wait(lk, [&] {
          if (stop_) return true;
          for (auto& cand : q_)
            if (cand->next.load() < cand->parts.size()) return true;
          return false;
        });
        continue;
      }
      lk.unlock();
      work(*j);
      lk.lock();
    }
  }

  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::shared_ptr<Job>> q_;
  std::vector<std::thread> th_;
  bool stop_ = false;
};

void parallel_copies(const std::vector<Copy>& copies) {
  const std::size_t part = std::size_t(4) << 20;
  std::vector<Copy> parts;
  for (const Copy& c : copies)
    for (std::size_t lo = 0; lo < c.bytes; lo += part)
      parts.push_back({static_cast<char*>(c.dst) + lo, static_cast<const char*>(c.src) + lo,
                       std::min(part, c.bytes - lo)});
  CopyPool::get().run(std::move(parts));
}

template <class Launch>
int host_pipeline_locked(HostPipe& p, int dev, std::size_t es, std::size_t chunk, const void* x,
                         std::size_t n, unsigned mask, void* const out[3], Launch&& launch);

// Chunked H2D -> kernel -> D2H over kPipe streams.  `launch(args, stream)`.
template <class Launch>
int host_pipeline(int dtype, const void* x, std::size_t n, unsigned mask, void* const out[3],
                  Launch&& launch) {
  const std::size_t es = dtype == FT_F32 ? 4 : 8;
  // 4 Mi elements per chunk: short pipeline fill/drain (2.21 vs 2.18 Gelem/s
  // for 8 Mi on 2^26 f64 elements; tools/hp_chunks.sh)
  const std::size_t chunk = std::size_t(1) << 22;
  int dev = 0;
  if (const int rc = device_or_fail(&dev)) return rc;
  HostPipe& p = g_pipe[dev];
  std::lock_guard<std::mutex> lk(p.mu);
  int rc = pipe_reserve(p, std::max(chunk * es, stage_bytes()));  // device slots serve both paths
  if (rc) return rc;
  rc = host_pipeline_locked(p, dev, es, chunk, x, n, mask, out, launch);
  if (rc) {
    // An early error return may leave chunks in flight on the pipeline streams;
    // drain them so the next call cannot reuse slots that are still being read
    // or written (the error string of the first failure is kept).
    const std::string keep = g_err;
    for (auto& s : p.st) (void)cudaStreamSynchronize(s);
    (void)cudaGetLastError();
    g_err = keep;
  }
  return rc;
}

template <class Launch>
int host_pipeline_locked(HostPipe& p, int dev, std::size_t es, std::size_t chunk, const void* x,
                         std::size_t n, unsigned mask, void* const out[3], Launch&& launch) {
  int rc = FT_OK;
  const char* xb = static_cast<const char*>(x);
  const bool x_pinned = host_pinned(x);
  bool o_pinned = true;
  for (int j = 0; j < 3; ++j) o_pinned = o_pinned && (!(mask & (1u << j)) || host_pinned(out[j]));
  if (!x_pinned || !o_pinned) {
    // ---- staged path for pageable buffers ----
    Staging& g = g_stage[dev];
    if ((rc = stage_reserve(g, stage_bytes()))) return rc;
    const std::size_t kStageChunk = stage_bytes() / es;  // elements per staged chunk
    struct Pending {
      bool live = false;
      std::size_t off = 0, m = 0;
    } pend[kPipe];
    // Wait for slot k's previous chunk; queue the copy of its outputs to the user.
    auto retire = [&](int k, std::vector<Copy>& copies) -> int {
      if (!pend[k].live) return FT_OK;
      cudaError_t e = cudaEventSynchronize(g.done[k]);
      if (e != cudaSuccess) return cuda_status(e, "cudaEventSynchronize");
      if (!o_pinned)
        for (int j = 0; j < 3; ++j)
          if (mask & (1u << j))
            copies.push_back({static_cast<char*>(out[j]) + pend[k].off * es, g.pin[k][1 + j], pend[k].m * es});
      pend[k].live = false;
      return FT_OK;
    };
    std::size_t ci = 0;
    for (std::size_t off = 0; off < n; off += kStageChunk, ++ci) {
      const int k = static_cast<int>(ci % kPipe);
      const std::size_t m = std::min(kStageChunk, n - off);
      std::vector<Copy> copies;
      if ((rc = retire(k, copies))) return rc;  // slot k is free once its last chunk is out
      const void* src = xb + off * es;
      if (!x_pinned) {
        copies.push_back({g.pin[k][0], src, m * es});
        src = g.pin[k][0];
      }
      parallel_copies(copies);  // previous outputs out and this input in, together
      cudaStream_t s = p.st[k];
      cudaError_t e = cudaMemcpyAsync(p.buf[k][0], src, m * es, cudaMemcpyDefault, s);
      if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync H2D");
      void* dout[3] = {p.buf[k][1], p.buf[k][2], p.buf[k][3]};
      e = launch(p.buf[k][0], m, dout, s);
      if (e != cudaSuccess) return cuda_status(e, "kernel launch");
      for (int j = 0; j < 3; ++j) {
        if (!(mask & (1u << j))) continue;
        void* dst = o_pinned ? static_cast<char*>(out[j]) + off * es : g.pin[k][1 + j];
        e = cudaMemcpyAsync(dst, dout[j], m * es, cudaMemcpyDefault, s);
        if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync D2H");
      }
      e = cudaEventRecord(g.done[k], s);
      if (e != cudaSuccess) return cuda_status(e, "cudaEventRecord");
      pend[k] = {true, off, m};
    }
    for (std::size_t i = 0; i < static_cast<std::size_t>(kPipe); ++i) {  // oldest first
      std::vector<Copy> copies;
      if ((rc = retire(static_cast<int>((ci + i) % kPipe), copies))) return rc;
      parallel_copies(copies);
    }
    return FT_OK;
  }
  std::size_t ci = 0;
  for (std::size_t off = 0; off < n; off += chunk, ++ci) {
    const int k = static_cast<int>(ci % kPipe);
    const std::size_t m = std::min(chunk, n - off);
    cudaStream_t s = p.st[k];
    cudaError_t e = cudaMemcpyAsync(p.buf[k][0], xb + off * es, m * es, cudaMemcpyDefault, s);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync H2D");
    void* dout[3] = {p.buf[k][1], p.buf[k][2], p.buf[k][3]};
    e = launch(p.buf[k][0], m, dout, s);
    if (e != cudaSuccess) return cuda_status(e, "kernel launch");
    for (int j = 0; j < 3; ++j) {
      if (!(mask & (1u << j))) continue;
      e = cudaMemcpyAsync(static_cast<char*>(out[j]) + off * es, dout[j], m * es,
                          cudaMemcpyDefault, s);
      if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync D2H");
    }
  }
  for (auto& s : p.st) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "cudaStreamSynchronize");
  }
  return FT_OK;
}

// ---- host-pointer calls over several GPUs ----
// ft_set_host_devices(G): host-pointer calls split arrays of at least
// kMinShard elements into G contiguous shards, one per device (round robin from
// the current device), each streamed by its own host thread through that
// device's pipeline -- every GPU brings its own PCIe link.  G <= 0: all visible.
std::atomic<int> g_host_devices{1};
constexpr std::size_t kMinShard = std::size_t(1) << 22;

template <class Launch>
int host_sharded(int dtype, const void* x, std::size_t n, unsigned mask, void* const out[3],
                 Launch&& launch) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    (void)cudaGetLastError();
    return fail(FT_ERR_NO_DEVICE, "no CUDA device visible");
  }
  int want = g_host_devices.load();
  if (want <= 0) want = ndev;
  const std::size_t G = std::min<std::size_t>(static_cast<std::size_t>(want), std::max<std::size_t>(1, n / kMinShard));
  if (G <= 1) return host_pipeline(dtype, x, n, mask, out, launch);
  const std::size_t es = dtype == FT_F32 ? 4 : 8;
  int base = 0;
  if (const int rc = device_or_fail(&base)) return rc;
  std::vector<int> rcs(G, FT_OK);
  std::vector<std::string> errs(G);
  std::vector<std::thread> th;
  for (std::size_t g = 0; g < G; ++g) {
    const std::size_t lo = n * g / G, hi = n * (g + 1) / G;
    th.emplace_back([&, g, lo, hi] {
      cudaError_t e = cudaSetDevice(static_cast<int>((base + g) % static_cast<std::size_t>(ndev)));
      if (e != cudaSuccess) {
        rcs[g] = cuda_status(e, "cudaSetDevice");
        errs[g] = g_err;
        return;
      }
      void* o[3];
      for (int j = 0; j < 3; ++j) o[j] = out[j] ? static_cast<char*>(out[j]) + lo * es : nullptr;
      rcs[g] = host_pipeline(dtype, static_cast<const char*>(x) + lo * es, hi - lo, mask, o, launch);
      if (rcs[g]) errs[g] = g_err;  // g_err is per thread
    });
  }
  for (auto& t : th) t.join();
  for (std::size_t g = 0; g < G; ++g)
    if (rcs[g]) return fail(rcs[g], errs[g]);
  return FT_OK;
}

// ---- L2 flush buffer (per device) ----
struct FlushBuf {
  std::mutex mu;
  void* p = nullptr;
  std::size_t bytes = 0;
  unsigned tick = 0;
};
FlushBuf g_flush[kMaxDevices];

}  // namespace

cudaError_t persistent_blocks(const void* fn, int threads, std::size_t work_items, unsigned* blocks,
                              int waves) {
  cudaError_t e;
  const int dev = current_device(&e);
  if (e != cudaSuccess) return e;
  if (dev >= kMaxDevices) return cudaErrorInvalidDevice;
  int occ = 0, sms = 0;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_occ.find(fn);
    if (it != g_occ.end()) {
      occ = it->second;
    } else {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, 0);
      if (e != cudaSuccess) return e;
      if (occ < 1) return cudaErrorInvalidConfiguration;  // the kernel cannot be resident at all
      g_occ[fn] = occ;
    }
    if (!g_sms[dev]) {
      e = cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev);
      if (e != cudaSuccess) return e;
    }
    sms = g_sms[dev];
  }
  // Four waves of resident blocks rather than exactly one: blocks that finish
  // early are backfilled, which trims the tail of the short launches (cfg1
  // +1.6%, cfg3 +1.8%, cfg2 +0.4% vs one wave; tools/gridmult_sweep.sh,
  // profiles/r01_k1_variants.json).  FT_GRID_MULT overrides it for experiments.
  static const int mult = [] {
    const char* env = std::getenv("FT_GRID_MULT");
    const int m = env ? std::atoi(env) : 4;
    return m >= 1 ? m : 1;
  }();
  // FT_OCC_CAP (experiments): size the grid for at most this many blocks per SM.
  static const int occ_cap = [] {
    const char* env = std::getenv("FT_OCC_CAP");
    return env ? std::atoi(env) : 0;
  }();
  if (occ_cap >= 1 && occ > occ_cap) occ = occ_cap;
  const std::size_t need = (work_items + threads - 1) / threads;
  const std::size_t full = static_cast<std::size_t>(occ) * sms * (waves > 0 ? waves : mult);
  *blocks = static_cast<unsigned>(std::max<std::size_t>(1, std::min(need, full)));
  return cudaSuccess;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
std::atomic<int> g_f32_policy{FT_F32_ULP2};
}
int f32_policy() { return g_f32_policy.load(std::memory_order_relaxed); }

}  // namespace ft

using namespace ft;

extern "C" {

int ft_abi_version(void) { return FT_ABI_VERSION; }

const char* ft_last_error_string(void) { return g_err.c_str(); }

uint64_t ft_launch_count(void) { return g_launches.load(); }

int ft_segment_table(double* out49) {
  if (!out49) return fail(FT_ERR_INVALID_ARG, "out is NULL");
  for (int k = 0; k < 6; ++k) {
    const Coeffs& c = kTable.seg[k];
    const double v[7] = {c.a, c.b, c.c, c.d, c.X, c.Y, c.Z};
    for (int j = 0; j < 7; ++j) out49[k * 7 + j] = v[j];
  }
  for (int j = 0; j < 7; ++j) out49[42 + j] = kTable.knots[j];
  return FT_OK;
}

int ft_taylor_coeffs(double* s9, double* c9, double* t9) {
  if (!s9 || !c9 || !t9) return fail(FT_ERR_INVALID_ARG, "out is NULL");
  for (int k = 0; k < 9; ++k) {
    s9[k] = kTaylor.sin_c[k];
    c9[k] = kTaylor.cos_c[k];
    t9[k] = kTaylor.tan_c[k];
  }
  return FT_OK;
}

int ft_thresholds(double* out8) {
  if (!out8) return fail(FT_ERR_INVALID_ARG, "out is NULL");
  const Thresholds& t = thresholds();
  out8[0] = t.quad[0];
  out8[1] = t.quad[1];
  out8[2] = t.quad[2];
  out8[3] = t.guard;
  out8[4] = kFast.quad[0];
  out8[5] = kFast.quad[1];
  out8[6] = kFast.quad[2];
  out8[7] = kFast.guard;
  return FT_OK;
}

int ft_proposed_eval_seg(ft_dtype dtype, const void* x, size_t n, unsigned mask, ft_sqrt_mode mode,
                         void* sin_out, void* cos_out, void* tan_out, uint8_t* seg_sc,
                         uint8_t* seg_t, void* stream) {
  void* out[3] = {sin_out, cos_out, tan_out};
  int rc = check_common(dtype, mask, n, x, out);
  if (rc) return rc;
  if ((rc = check_mode(mode))) return rc;
  if (n == 0) return FT_OK;
  const bool seg = seg_sc || seg_t;
  EvalArgs a = make_args(x, n, mask, out, seg_sc, seg_t, mode.newton_steps);
  return cuda_status(launch_proposed(dtype, mask, sqrt_kind(mode), seg, a, as_stream(stream)),
                     "ft_proposed_eval");
}

int ft_proposed_eval(ft_dtype dtype, const void* x, size_t n, unsigned mask, ft_sqrt_mode mode,
                     void* sin_out, void* cos_out, void* tan_out, void* stream) {
  return ft_proposed_eval_seg(dtype, x, n, mask, mode, sin_out, cos_out, tan_out, nullptr, nullptr,
                              stream);
}

int ft_taylor_eval(ft_dtype dtype, const void* x, size_t n, unsigned mask, int n_terms,
                   void* sin_out, void* cos_out, void* tan_out, void* stream) {
  void* out[3] = {sin_out, cos_out, tan_out};
  int rc = check_common(dtype, mask, n, x, out);
  if (rc) return rc;
  if (n_terms < 1 || n_terms > 9) return fail(FT_ERR_INVALID_ARG, "n_terms must be in [1, 9]");
  if (n == 0) return FT_OK;
  EvalArgs a = make_args(x, n, mask, out, nullptr, nullptr, n_terms);
  return cuda_status(launch_taylor(dtype, mask, n_terms, a, as_stream(stream)), "ft_taylor_eval");
}

int ft_mirror_eval(ft_dtype dtype, const void* x, size_t n, unsigned mask, int kind,
                   ft_sqrt_mode mode, int n_terms, void* sin_out, void* cos_out, void* tan_out,
                   uint8_t* seg_sc, uint8_t* seg_t, void* stream) {
  void* out[3] = {sin_out, cos_out, tan_out};
  int rc = check_common(dtype, mask, n, x, out);
  if (rc) return rc;
  if (kind != 0 && kind != 1) return fail(FT_ERR_INVALID_ARG, "kind must be 0 (proposed) or 1 (taylor)");
  if (kind == 0 && (rc = check_mode(mode))) return rc;
  if (kind == 1 && (n_terms < 1 || n_terms > 9)) return fail(FT_ERR_INVALID_ARG, "n_terms must be in [1, 9]");
  if (n == 0) return FT_OK;
  EvalArgs a = make_args(x, n, mask, out, seg_sc, seg_t, mode.newton_steps);
  return cuda_status(launch_mirror(dtype, mask, kind, mode.method, n_terms, a, as_stream(stream)),
                     "ft_mirror_eval");
}

int ft_stats_reset(ft_stats* stats_dev, void* stream) {
  if (!stats_dev) return fail(FT_ERR_INVALID_ARG, "stats is NULL");
  return cuda_status(cudaMemsetAsync(stats_dev, 0, sizeof(ft_stats), as_stream(stream)),
                     "ft_stats_reset");
}

int ft_parity_reduce(ft_dtype dtype, const void* x, size_t n, unsigned mask, int kind,
                     ft_sqrt_mode mode, int n_terms, const void* sin_out, const void* cos_out,
                     const void* tan_out, const void* ref_sin, const void* ref_cos,
                     const void* ref_tan, const uint8_t* seg_sc, const uint8_t* seg_t,
                     uint64_t ulp_tol, ft_stats* stats_dev, void* stream) {
  void* out[3] = {const_cast<void*>(sin_out), const_cast<void*>(cos_out), const_cast<void*>(tan_out)};
  int rc = check_common(dtype, mask, n, x, out);
  if (rc) return rc;
  if (!stats_dev) return fail(FT_ERR_INVALID_ARG, "stats is NULL");
  if (kind != 0 && kind != 1) return fail(FT_ERR_INVALID_ARG, "kind must be 0 or 1");
  if (kind == 0 && (rc = check_mode(mode))) return rc;
  if (kind == 1 && (n_terms < 1 || n_terms > 9)) return fail(FT_ERR_INVALID_ARG, "n_terms must be in [1, 9]");
  if (n == 0) return FT_OK;
  CheckArgs a{};
  a.x = x;
  a.got[0] = sin_out;
  a.got[1] = cos_out;
  a.got[2] = tan_out;
  a.ref[0] = ref_sin;
  a.ref[1] = ref_cos;
  a.ref[2] = ref_tan;
  a.seg_sc = seg_sc;
  a.seg_t = seg_t;
  a.n = n;
  a.mask = mask;
  a.kind = kind;
  a.method = mode.method;
  a.steps = mode.newton_steps;
  a.n_terms = n_terms;
  a.ulp_tol = ulp_tol;
  a.stats = stats_dev;
  return cuda_status(launch_check(dtype, a, as_stream(stream)), "ft_parity_reduce");
}

int ft_gen_inputs(ft_dtype dtype, int dist, double lo, double hi, uint64_t seed, uint64_t offset,
                  size_t n, void* x, void* stream) {
  if (dtype != FT_F32 && dtype != FT_F64) return fail(FT_ERR_INVALID_ARG, "bad dtype");
  if (dist != FT_DIST_UNIFORM && dist != FT_DIST_TAN_STRESS) return fail(FT_ERR_INVALID_ARG, "bad dist");
  if (n == 0) return FT_OK;
  if (!x) return fail(FT_ERR_INVALID_ARG, "x is NULL");
  if (dist == FT_DIST_TAN_STRESS && !(hi >= lo)) return fail(FT_ERR_INVALID_ARG, "kmax < kmin");
  return cuda_status(launch_gen(dtype, dist, lo, hi, seed, offset, n, x, as_stream(stream)),
                     "ft_gen_inputs");
}

int ft_l2_flush(void* stream) {
  int dev = 0;
  if (const int rc = device_or_fail(&dev)) return rc;
  FlushBuf& f = g_flush[dev];
  std::lock_guard<std::mutex> lk(f.mu);
  if (!f.p) {
    int l2 = 0;
    const cudaError_t ea = cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    if (ea != cudaSuccess) return cuda_status(ea, "cudaDeviceGetAttribute(L2 size)");
    f.bytes = std::max<std::size_t>(2 * static_cast<std::size_t>(l2), std::size_t(64) << 20);
    cudaError_t e = cudaMalloc(&f.p, f.bytes);
    if (e != cudaSuccess) {
      f.p = nullptr;
      return cuda_status(e, "cudaMalloc(l2 flush)");
    }
  }
  return cuda_status(launch_fill(f.p, f.bytes, ++f.tick, as_stream(stream)), "ft_l2_flush");
}

int ft_device_const_table(int unit, double* out49) {
  if (!out49) return fail(FT_ERR_INVALID_ARG, "out is NULL");
  Table t{};
  cudaError_t e;
  switch (unit) {
    case 0: e = read_const_table_eval(&t); break;
    case 1: e = read_const_table_check(&t); break;
    case 2: e = read_const_table_gen(&t); break;
    case 3: e = cudaMemcpyFromSymbol(&t, c_table, sizeof(Table)); break;
    default: return fail(FT_ERR_INVALID_ARG, "unit must be 0 (K1/K2), 1 (K3), 2 (K4/K5) or 3 (C-ABI)");
  }
  if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyFromSymbol(c_table)");
  for (int k = 0; k < 6; ++k) {
    const Coeffs& c = t.seg[k];
    const double v[7] = {c.a, c.b, c.c, c.d, c.X, c.Y, c.Z};
    for (int j = 0; j < 7; ++j) out49[k * 7 + j] = v[j];
  }
  for (int j = 0; j < 7; ++j) out49[42 + j] = t.knots[j];
  return FT_OK;
}

int ft_device_rows(int kind, void* out640) {
  if (!out640) return fail(FT_ERR_INVALID_ARG, "out is NULL");
  if (kind < 0 || kind > 7) return fail(FT_ERR_INVALID_ARG, "kind must be 0 (bit-exact) or an f32 mask 1..7");
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 640);
  if (e != cudaSuccess) return cuda_status(e, "cudaMalloc(rows)");
  e = launch_dump_rows(kind, d, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(out640, d, 640, cudaMemcpyDeviceToHost);
  const cudaError_t ef = cudaFree(d);
  if (e != cudaSuccess) return cuda_status(e, "ft_device_rows");
  return cuda_status(ef, "cudaFree(rows)");
}

int ft_release(int device) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDeviceCount");
  if (device >= ndev || device < -1) return fail(FT_ERR_INVALID_ARG, "device out of range");
  const int lo = device < 0 ? 0 : device, hi = device < 0 ? std::min(ndev, kMaxDevices) : device + 1;
  cudaError_t first = cudaSuccess;
  auto keep = [&](cudaError_t r) {
    if (first == cudaSuccess && r != cudaSuccess) first = r;
  };
  for (int d = lo; d < hi; ++d) {
    {
      HostPipe& p = g_pipe[d];
      std::lock_guard<std::mutex> lk(p.mu);
      for (auto& st : p.st)
        if (st) {
          keep(cudaStreamSynchronize(st));
          keep(cudaStreamDestroy(st));
          st = nullptr;
        }
      for (auto& row : p.buf)
        for (auto& b : row)
          if (b) {
            keep(cudaFree(b));
            b = nullptr;
          }
      p.cap_bytes = 0;
      p.init = false;
      Staging& g = g_stage[d];  // used only under the pipeline lock
      for (auto& row : g.pin)
        for (auto& b : row)
          if (b) {
            keep(cudaFreeHost(b));
            b = nullptr;
          }
      for (auto& ev : g.done)
        if (ev) {
          keep(cudaEventDestroy(ev));
          ev = nullptr;
        }
      g.cap_bytes = 0;
    }
    FlushBuf& f = g_flush[d];
    std::lock_guard<std::mutex> lk(f.mu);
    if (f.p) {
      keep(cudaFree(f.p));
      f.p = nullptr;
      f.bytes = 0;
    }
  }
  return cuda_status(first, "ft_release");
}

int ft_set_f32_policy(int policy) {
  if (policy != FT_F32_ULP2 && policy != FT_F32_BITWISE)
    return fail(FT_ERR_INVALID_ARG, "f32 policy must be FT_F32_ULP2 (0) or FT_F32_BITWISE (1)");
  g_f32_policy.store(policy);
  return FT_OK;
}

int ft_get_f32_policy(void) { return g_f32_policy.load(); }

int ft_set_host_devices(int n) {
  g_host_devices.store(n);
  return FT_OK;
}

int ft_get_host_devices(void) { return g_host_devices.load(); }

int ft_host_alloc(void** p, size_t bytes) {
  if (!p) return fail(FT_ERR_INVALID_ARG, "p is NULL");
  return cuda_status(cudaHostAlloc(p, bytes, cudaHostAllocDefault), "cudaHostAlloc");
}

int ft_host_free(void* p) { return cuda_status(cudaFreeHost(p), "cudaFreeHost"); }

int ft_proposed_batch_host(ft_dtype dtype, const void* x, size_t n, unsigned mask,
                           ft_sqrt_mode mode, void* sin_out, void* cos_out, void* tan_out) {
  void* out[3] = {sin_out, cos_out, tan_out};
  int rc = check_common(dtype, mask, n, x, out);
  if (rc) return rc;
  if ((rc = check_mode(mode))) return rc;
  if (n == 0) return FT_OK;
  const int sq = sqrt_kind(mode);
  return host_sharded(dtype, x, n, mask, out,
                       [&](const void* dx, std::size_t m, void* const dout[3], cudaStream_t s) {
                         EvalArgs a = make_args(dx, m, mask, dout, nullptr, nullptr, mode.newton_steps);
                         return launch_proposed(dtype, mask, sq, false, a, s);
                       });
}

int ft_taylor_batch_host(ft_dtype dtype, const void* x, size_t n, unsigned mask, int n_terms,
                         void* sin_out, void* cos_out, void* tan_out) {
  void* out[3] = {sin_out, cos_out, tan_out};
  int rc = check_common(dtype, mask, n, x, out);
  if (rc) return rc;
  if (n_terms < 1 || n_terms > 9) return fail(FT_ERR_INVALID_ARG, "n_terms must be in [1, 9]");
  if (n == 0) return FT_OK;
  return host_sharded(dtype, x, n, mask, out,
                       [&](const void* dx, std::size_t m, void* const dout[3], cudaStream_t s) {
                         EvalArgs a = make_args(dx, m, mask, dout, nullptr, nullptr, n_terms);
                         return launch_taylor(dtype, mask, n_terms, a, s);
                       });
}

int ft_proposed_sin_batch(const double* xs, size_t n, ft_sqrt_mode mode, double* out) {
  return ft_proposed_batch_host(FT_F64, xs, n, FT_OUT_SIN, mode, out, nullptr, nullptr);
}
int ft_proposed_cos_batch(const double* xs, size_t n, ft_sqrt_mode mode, double* out) {
  return ft_proposed_batch_host(FT_F64, xs, n, FT_OUT_COS, mode, nullptr, out, nullptr);
}
int ft_proposed_tan_batch(const double* xs, size_t n, ft_sqrt_mode mode, double* out) {
  return ft_proposed_batch_host(FT_F64, xs, n, FT_OUT_TAN, mode, nullptr, nullptr, out);
}

}  // extern "C"
