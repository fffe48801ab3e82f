// Pageable host memory <-> device for the host-buffer entry points
// (sdct_exec_host: the numpy surface and the C++ RealTensor API). A
// cudaMemcpy from pageable memory is staged by the driver on the calling
// thread, and the first write to a freshly allocated result array faults its
// pages in on that thread as well: ~27 ms for a 134 MB array on the B200
// host. Here the transfer runs in chunks through two pinned staging buffers:
// a pool of host threads copies chunk c between the caller's memory and one
// buffer while the copy engine moves chunk c-1 through the other, so the
// page faults and memcpy bandwidth of several cores overlap the PCIe DMA.
#pragma once

#include <sched.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace sdctb {

class CopyPool {
 public:
  // process-wide, never destroyed (idle workers are simply left blocked at exit)
  static CopyPool& get() {
    static CopyPool* p = new CopyPool;
    return *p;
  }
  int threads() const { return n_ + 1; }

  // memcpy split into page-aligned contiguous parts, one per pool thread plus
  // the caller's own part
  void copy(void* dst, const void* src, size_t bytes) {
    if (n_ == 0 || bytes < (4u << 20)) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> one(call_mu_);
    {
      std::lock_guard<std::mutex> l(m_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      pending_ = n_;
      ++gen_;
    }
    cv_.notify_all();
    part(static_cast<char*>(dst), static_cast<const char*>(src), bytes, n_ + 1, 0);
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [&] { return pending_ == 0; });
  }

 private:
  CopyPool() {
    cpu_set_t set;
    int cpus = static_cast<int>(std::thread::hardware_concurrency());
    if (sched_getaffinity(0, sizeof(set), &set) == 0) cpus = CPU_COUNT(&set);
    n_ = std::max(0, std::min(cpus, 16) - 1);
    for (int i = 0; i < n_; ++i) std::thread([this, i] { worker(i + 1); }).detach();
  }
  static void part(char* d, const char* s, size_t b, int parts, int idx) {
    const size_t per = ((b + parts - 1) / parts + 4095) & ~size_t(4095);
    const size_t off = per * static_cast<size_t>(idx);
    if (off < b) std::memcpy(d + off, s + off, std::min(per, b - off));
  }
  void worker(int idx) {
    unsigned long long seen = 0;
    std::unique_lock<std::mutex> l(m_);
    for (;;) {
      cv_.wait(l, [&] { return gen_ != seen; });
      seen = gen_;
      char* d = dst_;
      const char* s = src_;
      const size_t b = bytes_;
      l.unlock();
      part(d, s, b, n_ + 1, idx);
      l.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }

  int n_ = 0;
  std::mutex call_mu_, m_;
  std::condition_variable cv_, done_;
  unsigned long long gen_ = 0;
  int pending_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
};

}  // namespace sdctb
