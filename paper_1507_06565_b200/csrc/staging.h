// Host-side runtime helpers for moving the caller's (usually pageable) arrays
// to the device (pgpu_create's geometry upload).
//
// The CUDA driver copies pageable memory through its own small pinned bounce
// buffer at ~11 GB/s on the B200 hosts (700 MB: 65 ms), while a pinned source
// reaches ~52 GB/s and eight host threads copy pageable -> pinned at ~70 GB/s
// (tools/h2d_probe2.py).  StagedUpload therefore fills 16 MB pinned chunks
// with a persistent worker pool while the DMA engine drains the previous
// chunk.  The chunks and the threads are created once per process and reused
// (a runtime cache).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace pgpu {

// Fixed set of worker threads running fn(0..n-1) together with the caller.
class WorkerPool {
 public:
  explicit WorkerPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this] { loop(); });
  }
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  WorkerPool(const WorkerPool&) = delete;
  WorkerPool& operator=(const WorkerPool&) = delete;

  void run(int n, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> l(mu_);
    job_ = &fn;
    njob_.store(n);
    next_.store(0);
    remaining_ = n;
    ++gen_;
    cv_.notify_all();
    l.unlock();
    work();  // the caller takes items too
    l.lock();
    done_.wait(l, [this] { return remaining_ == 0; });
    job_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= njob_) return;
      (*job_)(i);
      std::lock_guard<std::mutex> l(mu_);
      if (--remaining_ == 0) done_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return stop_ || (gen_ != seen && job_ != nullptr); });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  std::atomic<int> njob_{0};
  std::atomic<int> next_{0};
  int remaining_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Pipelined pageable -> device copy through pinned chunks.
class StagedUpload {
 public:
  static StagedUpload& get() {
    static StagedUpload s;
    return s;
  }
  // Copies `bytes` from host `src` to device `dst` on `st`; returns when the
  // copy has completed (the caller may free `src`).  Returns a cudaError_t.
  cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return cudaSuccess;
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess &&
                        (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice ||
                         at.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    const size_t kChunk = chunk_;
    if (pinned || bytes < 2 * kChunk) {
      cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
      return e != cudaSuccess ? e : cudaStreamSynchronize(st);
    }
    std::lock_guard<std::mutex> lock(mu_);
    if (!stage_[0]) {  // all slots or none: a failed allocation leaves no partial set
      void* got[kSlots] = {nullptr, nullptr, nullptr, nullptr};
      for (int k = 0; k < kSlots; ++k) {
        const cudaError_t e = cudaHostAlloc(&got[k], chunk_, cudaHostAllocPortable);
        if (e != cudaSuccess) {
          for (int j = 0; j < k; ++j) cudaFreeHost(got[j]);
          return e;
        }
      }
      for (int k = 0; k < kSlots; ++k) stage_[k] = got[k];
    }
    cudaEvent_t ev[kSlots];
    for (int k = 0; k < kSlots; ++k) {
      const cudaError_t r = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
      if (r != cudaSuccess) {
        for (int j = 0; j < k; ++j) cudaEventDestroy(ev[j]);
        return r;
      }
    }
    cudaError_t err = cudaSuccess;
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    size_t i = 0;
    for (size_t off = 0; off < bytes && err == cudaSuccess; off += kChunk, ++i) {
      const size_t n = bytes - off < kChunk ? bytes - off : kChunk;
      const int b = (int)(i % kSlots);
      if (i >= (size_t)kSlots) err = cudaEventSynchronize(ev[b]);  // slot drained
      if (err != cudaSuccess) break;
      char* stg = static_cast<char*>(stage_[b]);
      const char* from = s + off;
      pool_.run(kParts, [&](int t) {
        const size_t a = n * t / kParts, e = n * (t + 1) / kParts;
        std::memcpy(stg + a, from + a, e - a);
      });
      err = cudaMemcpyAsync(d + off, stg, n, cudaMemcpyHostToDevice, st);
      if (err == cudaSuccess) err = cudaEventRecord(ev[b], st);
    }
    for (auto& e : ev) {
      const cudaError_t r = cudaEventSynchronize(e);
      if (err == cudaSuccess) err = r;
      cudaEventDestroy(e);
    }
    return err;
  }

 private:
  StagedUpload() : pool_(kParts - 1) {
    if (const char* e = std::getenv("PGPU_STAGE_MB")) chunk_ = size_t(std::max(1, atoi(e))) << 20;
  }
  size_t chunk_ = size_t(16) << 20;  // bytes per pinned chunk (PGPU_STAGE_MB overrides)
  static constexpr int kSlots = 4;
  static constexpr int kParts = 8;
  std::mutex mu_;
  void* stage_[kSlots] = {nullptr, nullptr, nullptr, nullptr};
  WorkerPool pool_;
};

}  // namespace pgpu
