// gs_arena.h — the executor's per-device job arena.
//
// One cudaMalloc'd slab per device, sized to the ledger capacity the
// placement engine hands out (spec.mem_bytes), sub-allocated on the host in
// 2 MiB granules — the granule the probe's mem_bytes is counted in
// (round_granule, gs_job_probe).  It replaces per-buffer cudaMallocAsync
// from the stream-ordered pool for co-located jobs: growing that pool maps
// physical memory under a driver lock every worker then waits on, and its
// chunks fragment under 2-40 GB jobs (cfg 2), so an admitted
// job could stall in the allocator for hundreds of ms.  Here an allocation
// is a best-fit search in two ordered maps under one mutex, no driver call.
//
// Memory safety: the ledger admits a task only while Σ admitted footprints
// <= capacity = the slab, and a job's buffers (+ one control granule out of
// its 8 MiB heap allowance) sum to at most its footprint.  Free SPACE is
// therefore always there; only a contiguous hole may be missing
// (fragmentation).  A job of a memory-safe policy then waits for the next
// free and retries — all of its buffers at once (all-or-nothing), so no job
// holds part of its memory while waiting, and once every other job is done
// the slab is empty and the request fits: no deadlock, and never an OOM.
// Policies without a memory check (sa, cg) get no wait: a failed request is
// the job's out-of-memory crash (sim_engine.py:342-350).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <map>
#include <mutex>
#include <vector>

namespace gsa {

constexpr int64_t kGranule = 2 << 20;

class Arena {
 public:
  Arena(int device, char *base, int64_t size) : device_(device), base_(base), size_(size), limit_(size) {
    insert(0, size);
  }
  int device() const { return device_; }
  int64_t size() const { return size_; }
  char *base() const { return base_; }
  int64_t in_use() {
    std::lock_guard<std::mutex> g(mu_);
    return used_;
  }
  // Limit the usable part of the slab to its first `limit` bytes (the
  // run's ledger capacity).  Only between runs (nothing allocated).
  bool reset(int64_t limit) {
    std::lock_guard<std::mutex> g(mu_);
    if (used_ != 0 || limit > size_) return false;
    by_off_.clear();
    by_len_.clear();
    limit_ = limit / kGranule * kGranule;
    if (limit_ > 0) insert(0, limit_);
    return true;
  }

  // Place every request (bytes, rounded up to granules) or none.  With
  // `wait`, an unplaceable request blocks until a free changes the holes
  // (and fails only if it is larger than the whole slab).  Returns false on
  // failure; *waited_ms gets the time spent blocked.
  bool alloc_all(const std::vector<int64_t> &bytes, std::vector<void *> &out, bool wait, double *waited_ms) {
    std::unique_lock<std::mutex> lk(mu_);
    int64_t total = 0;
    for (int64_t b : bytes) total += round(b);
    if (waited_ms) *waited_ms = 0;
    if (total > limit_) return false;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      if (try_place(bytes, out)) break;
      if (!wait) return false;
      const uint64_t seen = frees_;
      cv_.wait(lk, [&] { return frees_ != seen; });
    }
    if (waited_ms)
      *waited_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return true;
  }

  void free_all(const std::vector<void *> &ptrs, const std::vector<int64_t> &bytes) {
    {
      std::lock_guard<std::mutex> g(mu_);
      for (size_t i = 0; i < ptrs.size(); ++i) {
        if (!ptrs[i]) continue;
        give_back((char *)ptrs[i] - base_, round(bytes[i]));
      }
      ++frees_;
    }
    cv_.notify_all();
  }

 private:
  static int64_t round(int64_t b) { return (std::max<int64_t>(b, 1) + kGranule - 1) / kGranule * kGranule; }

  // largest request first, each into the smallest hole that holds it
  bool try_place(const std::vector<int64_t> &bytes, std::vector<void *> &out) {
    std::vector<size_t> order(bytes.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return bytes[a] > bytes[b]; });
    std::vector<std::pair<int64_t, int64_t>> taken;  // (offset, len) for rollback
    out.assign(bytes.size(), nullptr);
    for (size_t i : order) {
      const int64_t len = round(bytes[i]);
      auto it = by_len_.lower_bound(len);
      if (it == by_len_.end()) {
        for (auto &t : taken) give_back(t.first, t.second);
        out.assign(bytes.size(), nullptr);
        return false;
      }
      const int64_t hole_len = it->first, off = it->second;
      erase(off, hole_len);
      if (hole_len > len) insert(off + len, hole_len - len);
      taken.push_back({off, len});
      out[i] = base_ + off;
      used_ += len;
    }
    return true;
  }

  void give_back(int64_t off, int64_t len) {
    used_ -= len;
    // coalesce with the neighbouring holes
    auto next = by_off_.lower_bound(off);
    if (next != by_off_.end() && next->first == off + len) {
      len += next->second;
      erase(next->first, next->second);
    }
    auto prev = by_off_.lower_bound(off);
    if (prev != by_off_.begin()) {
      --prev;
      if (prev->first + prev->second == off) {
        off = prev->first;
        len += prev->second;
        erase(prev->first, prev->second);
      }
    }
    insert(off, len);
  }

  void insert(int64_t off, int64_t len) {
    by_off_[off] = len;
    by_len_.insert({len, off});
  }
  void erase(int64_t off, int64_t len) {
    by_off_.erase(off);
    auto r = by_len_.equal_range(len);
    for (auto it = r.first; it != r.second; ++it)
      if (it->second == off) {
        by_len_.erase(it);
        break;
      }
  }

  int device_;
  char *base_;
  int64_t size_, limit_;
  int64_t used_ = 0;
  uint64_t frees_ = 0;
  std::map<int64_t, int64_t> by_off_;        // hole offset -> length
  std::multimap<int64_t, int64_t> by_len_;   // hole length -> offset
  std::mutex mu_;
  std::condition_variable cv_;
};

}  // namespace gsa
