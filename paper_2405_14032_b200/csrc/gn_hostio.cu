// Host-memory transfers of the GN_MEM_HOST calls -- the reference's std::span seams hand the
// library pageable std::vector storage (solver.hpp:143-146, lifted.hpp).  A cudaMemcpy from
// or to pageable memory is staged by the driver through its own small pinned buffers, one
// CPU thread at a time; here it goes through a ring of pinned bounce buffers in chunks instead:
// the host-side copies are split over a few threads and overlap the DMA of the neighbouring
// chunk (PCIe is not idle while the CPU copies).  Caller memory that is already pinned
// (cudaHostAlloc / cudaHostRegister), or device memory, is copied directly.  Both calls return when the copy is
// complete, as the host modes require.
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "gn_internal.cuh"

namespace gnb {
namespace {

constexpr size_t kDirect = 1u << 20;      // below this: one plain cudaMemcpyAsync
constexpr int kMaxBufs = 4;

long env_long(const char* name, long dflt, long lo, long hi) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  const long x = std::strtol(v, nullptr, 10);
  return x < lo ? lo : (x > hi ? hi : x);
}
// bytes per bounce buffer and the number of buffers in rotation (GN_HOSTIO_CHUNK_MB,
// GN_HOSTIO_BUFS, GN_HOSTIO_THREADS: tuning knobs, read once).  8 MB x 4 measured 3-5% faster
// than 16 MB x 2 on every host-mode call of scripts/hostio_probe.py (two alternating sweeps;
// 4 MB, 3 buffers, 6 or 12 copy threads, 32 and 64 MB chunks all slower or equal)
size_t chunk_bytes() {
  static const size_t c = static_cast<size_t>(env_long("GN_HOSTIO_CHUNK_MB", 8, 1, 256)) << 20;
  return c;
}
int nbufs() {
  static const int n = static_cast<int>(env_long("GN_HOSTIO_BUFS", 4, 2, kMaxBufs));
  return n;
}

// A fixed pool of host threads for the bounce copies.
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    n_ = hw >= 16 ? 8 : (hw >= 4 ? hw / 2 : 1);
    n_ = static_cast<unsigned>(env_long("GN_HOSTIO_THREADS", n_, 1, 64));
    for (unsigned i = 1; i < n_; ++i) th_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // memcpy(dst, src, bytes) split over the pool (the calling thread takes part 0)
  void copy(void* dst, const void* src, size_t bytes) {
    if (n_ == 1 || bytes < (1u << 20)) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> op(op_);  // one split copy at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    part(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void part(unsigned i) {
    const size_t per = (bytes_ / n_ + 63) & ~size_t(63);
    const size_t a = std::min(bytes_, per * i), b = std::min(bytes_, per * (i + 1));
    if (b > a) std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void run(unsigned i) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      part(i);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  unsigned n_ = 1;
  std::vector<std::thread> th_;
  std::mutex mu_, op_;
  std::condition_variable cv_, done_;
  uint64_t gen_ = 0;
  unsigned pending_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
};

struct Bounce {
  std::mutex mu;  // one transfer at a time owns the buffers
  char* buf[kMaxBufs] = {};
  cudaEvent_t ev[kMaxBufs] = {};
  int device = -1;
};

CopyPool& pool() {
  static CopyPool p;
  return p;
}
Bounce& bounce_for(int dev) {
  static std::mutex mu;
  static std::vector<Bounce*> per;
  std::lock_guard<std::mutex> lk(mu);
  if (static_cast<size_t>(dev) >= per.size()) per.resize(static_cast<size_t>(dev) + 1, nullptr);
  if (!per[dev]) {
    auto* b = new Bounce();  // process lifetime (pinned memory is freed at exit)
    b->device = dev;
    for (int i = 0; i < nbufs(); ++i) {
      GN_CK(cudaHostAlloc(reinterpret_cast<void**>(&b->buf[i]), chunk_bytes(), cudaHostAllocDefault));
      GN_CK(cudaEventCreateWithFlags(&b->ev[i], cudaEventDisableTiming));
    }
    per[dev] = b;
  }
  return *per[dev];
}

// Memory the copy engine can address directly: pinned host, device or managed memory (a
// device pointer handed to a host mode by mistake is then still copied correctly).
bool direct(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type != cudaMemoryTypeUnregistered;
}

}  // namespace

void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (bytes <= kDirect || direct(src)) {
    GN_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    GN_CK(cudaStreamSynchronize(s));
    return;
  }
  int dev = 0;
  GN_CK(cudaGetDevice(&dev));
  Bounce& b = bounce_for(dev);
  std::lock_guard<std::mutex> lk(b.mu);
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  const size_t kChunk = chunk_bytes();
  const int nb = nbufs();
  bool used[kMaxBufs] = {};
  for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
    const int k = static_cast<int>(i % nb);
    const size_t n = std::min(kChunk, bytes - off);
    if (used[k]) GN_CK(cudaEventSynchronize(b.ev[k]));  // its previous DMA has read it
    pool().copy(b.buf[k], in + off, n);                  // overlaps the other buffer's DMA
    GN_CK(cudaMemcpyAsync(out + off, b.buf[k], n, cudaMemcpyHostToDevice, s));
    GN_CK(cudaEventRecord(b.ev[k], s));
    used[k] = true;
  }
  GN_CK(cudaStreamSynchronize(s));
}

void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (bytes <= kDirect || direct(dst)) {
    GN_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    GN_CK(cudaStreamSynchronize(s));
    return;
  }
  int dev = 0;
  GN_CK(cudaGetDevice(&dev));
  Bounce& b = bounce_for(dev);
  std::lock_guard<std::mutex> lk(b.mu);
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  const size_t kChunk = chunk_bytes();
  const size_t nb = static_cast<size_t>(nbufs());
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t i) {
    const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
    GN_CK(cudaMemcpyAsync(b.buf[i % nb], in + off, n, cudaMemcpyDeviceToHost, s));
    GN_CK(cudaEventRecord(b.ev[i % nb], s));
  };
  // the DMA of the next nb - 1 chunks runs while this one is copied out
  for (size_t i = 0; i + 1 < nb && i < nch; ++i) issue(i);
  for (size_t i = 0; i < nch; ++i) {
    if (i + nb - 1 < nch) issue(i + nb - 1);
    GN_CK(cudaEventSynchronize(b.ev[i % nb]));
    const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
    pool().copy(out + off, b.buf[i % nb], n);
  }
}

}  // namespace gnb
