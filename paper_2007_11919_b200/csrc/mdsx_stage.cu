// Host <-> device staging of caller-owned PAGEABLE host arrays (the reference
// API takes numpy arrays, linalg.py:28-38 coerces them with np.asarray).
//
// A pageable cudaMemcpy runs at a few GB/s on the B200 hosts (the driver
// copies through its own small bounce buffer, serially).  mdsx_h2d instead
// splits the array over T persistent host threads; each owns two page-locked
// chunk buffers and its own stream, copies chunk i into one buffer while the
// other one's DMA is in flight, so host memcpy bandwidth (several threads) and
// PCIe DMA overlap.  Ordering: every worker stream first waits for the
// caller's stream (the destination may be memory the caller's earlier work
// still reads), and the caller's stream waits for every worker before later
// work.  The call returns when every chunk has been copied OUT of the
// caller's array (the source may be freed or overwritten afterwards); the
// DMA into dst is stream-ordered like cudaMemcpyAsync.
#include "mdsx_common.cuh"

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>

namespace mdsx {
int fail(mdsx_handle* h, int code, const std::string& msg);
int cuda_check(mdsx_handle* h, cudaError_t e, const char* what);
}  // namespace mdsx

namespace {

constexpr size_t kChunkMax = (size_t)32 << 20;   // pinned bytes per worker buffer
constexpr int kMaxThreads = 16;

struct Worker {
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t freed[2] = {nullptr, nullptr};  // DMA out of buf[b] finished
  cudaEvent_t done = nullptr;                 // last DMA of this call
  cudaStream_t st = nullptr;
  int rc = MDSX_OK;
};

// Fixed pool of host threads; run(n, f) calls f(0..n-1) on n workers and
// returns when all have finished.
struct StagePool {
  int device = 0;
  std::vector<std::thread> th;
  std::vector<Worker> w;
  std::mutex m;
  std::condition_variable cv, done_cv;
  std::function<void(int)> job;
  int gen = 0, active = 0, pending = 0;
  bool stop = false;
  cudaEvent_t ev_start = nullptr;

  explicit StagePool(int dev) : device(dev) {}

  int init(int n) {
    if ((int)th.size() >= n) return MDSX_OK;
    cudaSetDevice(device);
    if (!ev_start && cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) != cudaSuccess)
      return MDSX_CUDA;
    const int old = (int)w.size();
    w.resize(n);
    for (int i = old; i < n; ++i) {
      Worker& k = w[i];
      for (int b = 0; b < 2; ++b) {
        if (cudaHostAlloc(&k.buf[b], kChunkMax, cudaHostAllocDefault) != cudaSuccess) return MDSX_CUDA;
        if (cudaEventCreateWithFlags(&k.freed[b], cudaEventDisableTiming) != cudaSuccess)
          return MDSX_CUDA;
      }
      if (cudaEventCreateWithFlags(&k.done, cudaEventDisableTiming) != cudaSuccess) return MDSX_CUDA;
      if (cudaStreamCreateWithFlags(&k.st, cudaStreamNonBlocking) != cudaSuccess) return MDSX_CUDA;
    }
    for (int i = (int)th.size(); i < n; ++i) th.emplace_back([this, i] { loop(i); });
    return MDSX_OK;
  }

  void loop(int i) {
    cudaSetDevice(device);
    int seen = 0;
    for (;;) {
      std::function<void(int)> f;
      {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return stop || (gen != seen && i < active); });
        if (stop) return;
        seen = gen;
        f = job;
      }
      f(i);
      {
        std::lock_guard<std::mutex> lk(m);
        if (--pending == 0) done_cv.notify_all();
      }
    }
  }

  void run(int n, std::function<void(int)> f) {
    {
      std::lock_guard<std::mutex> lk(m);
      job = std::move(f);
      active = n;
      pending = n;
      ++gen;
    }
    cv.notify_all();
    std::unique_lock<std::mutex> lk(m);
    done_cv.wait(lk, [&] { return pending == 0; });
  }

  ~StagePool() {
    {
      std::lock_guard<std::mutex> lk(m);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
    for (auto& k : w) {
      for (int b = 0; b < 2; ++b) {
        if (k.buf[b]) cudaFreeHost(k.buf[b]);
        if (k.freed[b]) cudaEventDestroy(k.freed[b]);
      }
      if (k.done) cudaEventDestroy(k.done);
      if (k.st) cudaStreamDestroy(k.st);
    }
    if (ev_start) cudaEventDestroy(ev_start);
  }
};

// One pool per device for the life of the process; deliberately never
// destroyed (a static destructor would call the CUDA runtime during process
// teardown and join threads blocked on the condition variable).
std::mutex g_pools_mu;
std::vector<StagePool*>* g_pools = new std::vector<StagePool*>();

StagePool* pool_for(int device) {
  std::lock_guard<std::mutex> lk(g_pools_mu);
  for (StagePool* p : *g_pools)
    if (p->device == device) return p;
  g_pools->push_back(new StagePool(device));
  return g_pools->back();
}

}  // namespace

using namespace mdsx;

extern "C" int mdsx_h2d(mdsx_handle* h, void* dst, const void* src, int64_t bytes,
                        int32_t threads, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(h, MDSX_PARAM, "bad h2d arguments");
  if (bytes == 0) return MDSX_OK;
  int T = threads > 0 ? threads : 8;               // measured best on the B200 hosts
  const char* ec = getenv("MDSX_H2D_CHUNK_MB");
  const size_t kChunk = std::min(kChunkMax, ec ? (size_t)atoi(ec) << 20 : (size_t)8 << 20);
  const int64_t nchunks = (bytes + (int64_t)kChunk - 1) / (int64_t)kChunk;
  T = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)T, (int64_t)kMaxThreads, nchunks}));
  StagePool* pool = pool_for(h->device);
  std::lock_guard<std::mutex> run_lk(g_pools_mu);   // one staged copy per process at a time
  if (pool->init(T) != MDSX_OK) return fail(h, MDSX_CUDA, "h2d staging allocation failed");
  if (cudaEventRecord(pool->ev_start, st) != cudaSuccess)
    return fail(h, MDSX_CUDA, "h2d: event record failed");
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  pool->run(T, [&](int wi) {
    Worker& k = pool->w[wi];
    k.rc = MDSX_OK;
    cudaStreamWaitEvent(k.st, pool->ev_start, 0);
    int b = 0;
    for (int64_t c = wi; c < nchunks; c += T, b ^= 1) {
      const int64_t off = c * (int64_t)kChunk;
      const size_t len = (size_t)std::min<int64_t>((int64_t)kChunk, bytes - off);
      cudaEventSynchronize(k.freed[b]);          // previous DMA out of this buffer
      std::memcpy(k.buf[b], s + off, len);
      if (cudaMemcpyAsync(d + off, k.buf[b], len, cudaMemcpyHostToDevice, k.st) != cudaSuccess)
        k.rc = MDSX_CUDA;
      cudaEventRecord(k.freed[b], k.st);
    }
    cudaEventRecord(k.done, k.st);
  });
  for (int wi = 0; wi < T; ++wi) {
    if (pool->w[wi].rc != MDSX_OK) return fail(h, MDSX_CUDA, "h2d: cudaMemcpyAsync failed");
    cudaStreamWaitEvent(st, pool->w[wi].done, 0);
  }
  return cuda_check(h, cudaGetLastError(), "h2d");
}
