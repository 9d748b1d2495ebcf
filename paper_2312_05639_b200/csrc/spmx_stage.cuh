// spmx_stage.cuh — host <-> device copies of PAGEABLE host memory for the host-buffer entry points.
//
// The reference's run_spmm takes std::vector-backed matrices (include/spmx/csr.hpp:10-20,
// dense.hpp:9-21): pageable memory. cudaMemcpyAsync from or to pageable memory is staged by the
// driver through one thread (13 GB/s on the B200 boxes of this pool: c2 through spmx_spmm_host
// took 52 ms from pageable buffers against 10.9 ms from pinned ones). This stager does the same
// staging with several host threads: a copy is cut into pieces, every worker owns two pinned
// slots, copies a piece into a slot and enqueues the slot's DMA on the target stream (H2D), or
// enqueues the DMA into a slot, waits for it and copies the piece out (D2H). Pinned, registered
// and managed pointers never come here (Stager::pageable): they go to the DMA engines directly.
//
// A job is done when all its pieces are ENQUEUED (H2D; the stream orders the rest) or COPIED OUT
// (D2H). Pieces of one job may be enqueued in any order: they cover disjoint ranges.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#if defined(__x86_64__) && !defined(SPMX_STAGE_PLAIN_MEMCPY)
#include <emmintrin.h>
#define SPMX_STAGE_STREAMING 1
#else
#define SPMX_STAGE_STREAMING 0
#endif

namespace spmx_stage {

// memcpy with non-temporal stores: both destinations of a staged copy (the pinned slot the DMA
// engine reads next, the caller's Y) are written once and not read by this core again, so the
// lines are not fetched for ownership first (a third less DRAM traffic per byte than memcpy,
// and the copies of several threads are bound by exactly that). SSE2: every x86-64 has it.
inline void stream_copy(void* dst, const void* src, size_t bytes) {
#if SPMX_STAGE_STREAMING
  char* d = (char*)dst;
  const char* s = (const char*)src;
  const size_t head = (size_t)(-(uintptr_t)d & 15u);
  if (bytes < 256 + head) {
    std::memcpy(d, s, bytes);
    return;
  }
  if (head) {
    std::memcpy(d, s, head);
    d += head; s += head; bytes -= head;
  }
  const size_t body = bytes & ~(size_t)63;
  for (size_t i = 0; i < body; i += 64) {
    const __m128i a = _mm_loadu_si128((const __m128i*)(s + i));
    const __m128i b = _mm_loadu_si128((const __m128i*)(s + i + 16));
    const __m128i c = _mm_loadu_si128((const __m128i*)(s + i + 32));
    const __m128i e = _mm_loadu_si128((const __m128i*)(s + i + 48));
    _mm_stream_si128((__m128i*)(d + i), a);
    _mm_stream_si128((__m128i*)(d + i + 16), b);
    _mm_stream_si128((__m128i*)(d + i + 32), c);
    _mm_stream_si128((__m128i*)(d + i + 48), e);
  }
  _mm_sfence();
  if (bytes > body) std::memcpy(d + body, s + body, bytes - body);
#else
  std::memcpy(dst, src, bytes);
#endif
}

class Stager {
 public:
  struct Job {
    std::mutex mu;
    std::condition_variable cv;
    size_t left = 0;
    std::string error;
  };
  using Ticket = std::shared_ptr<Job>;

  static constexpr size_t kPiece = 4u << 20;

  // pageable host memory: what the driver would stage on one thread
  static bool pageable(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
  }

  Stager(int device, int workers) : device_(device) {
    if (workers < 1) workers = 1;
    // slots and events are created by their worker on its first piece (pinned allocations are
    // slow: a copy of a few pieces should not pay for every worker's slots)
    slots_.resize((size_t)workers * 2, nullptr);
    events_.resize((size_t)workers * 2, nullptr);
    busy_.assign((size_t)workers * 2, 0);
    for (int w = 0; w < workers; ++w) threads_.emplace_back([this, w] { run(w); });
  }
  ~Stager() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
    release();
  }
  Stager(const Stager&) = delete;
  Stager& operator=(const Stager&) = delete;

  int workers() const { return (int)threads_.size(); }

  Ticket h2d(void* dst_dev, const void* src, size_t bytes, cudaStream_t s) { return submit(true, dst_dev, src, bytes, s); }
  Ticket d2h(void* dst, const void* src_dev, size_t bytes, cudaStream_t s) { return submit(false, dst, src_dev, bytes, s); }

  // blocks until the job is done; throws what a worker caught
  static void wait(const Ticket& t) {
    if (!t) return;
    std::unique_lock<std::mutex> lk(t->mu);
    t->cv.wait(lk, [&] { return t->left == 0; });
    if (!t->error.empty()) throw std::runtime_error(t->error);
  }
  // the same without throwing (error paths)
  static void wait_quiet(const Ticket& t) noexcept {
    if (!t) return;
    std::unique_lock<std::mutex> lk(t->mu);
    t->cv.wait(lk, [&] { return t->left == 0; });
  }

 private:
  struct Piece {
    bool up;
    char* dst;
    const char* src;
    size_t bytes;
    cudaStream_t stream;
    Ticket job;
  };

  Ticket submit(bool up, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    auto job = std::make_shared<Job>();
    const size_t n = (bytes + kPiece - 1) / kPiece;
    job->left = n;
    if (n == 0) return job;
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (size_t i = 0; i < n; ++i) {
        const size_t off = i * kPiece;
        queue_.push_back(Piece{up, (char*)dst + off, (const char*)src + off, std::min(kPiece, bytes - off), s, job});
      }
    }
    cv_.notify_all();
    return job;
  }

  void run(int w) {
    cudaSetDevice(device_);
    int turn = 0;
    for (;;) {
      Piece p;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !queue_.empty(); });
        if (queue_.empty()) return;  // stop_ and nothing left
        p = std::move(queue_.front());
        queue_.pop_front();
      }
      const size_t slot = (size_t)w * 2 + (size_t)(turn ^= 1);
      std::string err;
      auto ok = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess && err.empty()) err = std::string("host stager: ") + what + ": " + cudaGetErrorString(e);
        return e == cudaSuccess;
      };
      if (!slots_[slot]) {
        if (!ok(cudaMallocHost(&slots_[slot], kPiece), "pinned slot") ||
            !ok(cudaEventCreateWithFlags(&events_[slot], cudaEventDisableTiming), "slot event")) {
          if (slots_[slot] && !events_[slot]) { cudaFreeHost(slots_[slot]); slots_[slot] = nullptr; }
          cudaGetLastError();
        }
      }
      // the slot's previous DMA (an upload enqueued two pieces ago) must have read it
      if (busy_[slot]) {
        ok(cudaEventSynchronize(events_[slot]), "slot wait");
        busy_[slot] = 0;
      }
      if (!err.empty()) {
        // no slot: fall through to the completion below with the error recorded
      } else if (p.up) {
        stream_copy(slots_[slot], p.src, p.bytes);
        if (ok(cudaMemcpyAsync(p.dst, slots_[slot], p.bytes, cudaMemcpyHostToDevice, p.stream), "H2D") &&
            ok(cudaEventRecord(events_[slot], p.stream), "event"))
          busy_[slot] = 1;
      } else {
        if (ok(cudaMemcpyAsync(slots_[slot], p.src, p.bytes, cudaMemcpyDeviceToHost, p.stream), "D2H") &&
            ok(cudaEventRecord(events_[slot], p.stream), "event") &&
            ok(cudaEventSynchronize(events_[slot]), "D2H wait"))
          stream_copy(p.dst, slots_[slot], p.bytes);
      }
      {
        std::lock_guard<std::mutex> lk(p.job->mu);
        if (!err.empty() && p.job->error.empty()) p.job->error = err;
        --p.job->left;
      }
      p.job->cv.notify_all();
    }
  }

  void release() {
    for (void* s : slots_)
      if (s) cudaFreeHost(s);
    for (cudaEvent_t e : events_)
      if (e) cudaEventDestroy(e);
    slots_.clear();
    events_.clear();
  }

  int device_;
  std::vector<void*> slots_;
  std::vector<cudaEvent_t> events_;
  std::vector<char> busy_;  // per slot, touched by its owner only
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Piece> queue_;
  bool stop_ = false;
};

// One stager per device and direction for the whole process, shared by every context (its jobs
// are independent of each other) and never destroyed: worker threads and pinned slots outlive
// the contexts, and nothing of the CUDA runtime is torn down from a static destructor at exit.
inline Stager& shared_stager(int device, bool up, int workers) {
  static std::mutex mu;
  static std::vector<Stager*> inst;  // [2 * device + up]
  std::lock_guard<std::mutex> lk(mu);
  const size_t key = (size_t)device * 2 + (up ? 1 : 0);
  if (inst.size() <= key) inst.resize(key + 1, nullptr);
  if (!inst[key]) inst[key] = new Stager(device, workers);
  return *inst[key];
}

}  // namespace spmx_stage
