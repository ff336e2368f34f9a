// Stream-ordered pool behaviour on this driver: after growing the default
// pool once (malloc + free of one big block), how long do sub-allocations
// of job-sized buffers take?   nvcc -o /tmp/pool_probe tools/pool_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <chrono>
#include <thread>
#include <vector>
using Clock = std::chrono::steady_clock;
static double ms(Clock::time_point t) { return std::chrono::duration<double, std::milli>(Clock::now() - t).count(); }
int main(int argc, char **argv) {
  const size_t GB = 1ull << 30;
  size_t grow = (argc > 1 ? atoll(argv[1]) : 120) * GB;
  cudaSetDevice(0);
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto t = Clock::now();
  void *big = nullptr;
  cudaError_t e = cudaMallocAsync(&big, grow, st);
  cudaFreeAsync(big, st);
  cudaStreamSynchronize(st);
  printf("grow %zu GB: %.1f ms (%s)\n", grow / GB, ms(t), cudaGetErrorString(e));
  size_t sizes[] = {15 * GB, 7 * GB, 340ull << 20, 1358ull << 20, 85ull << 20, 7 * GB, 2 * GB, 128000, 4 * GB};
  for (int rep = 0; rep < 3; ++rep) {
    std::vector<void *> ps;
    for (size_t s : sizes) {
      void *p = nullptr;
      t = Clock::now();
      e = cudaMallocAsync(&p, s, st);
      printf("rep %d alloc %10zu B: %.3f ms (%s)\n", rep, s, ms(t), cudaGetErrorString(e));
      ps.push_back(p);
    }
    t = Clock::now();
    for (void *p : ps) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    printf("rep %d free+sync: %.3f ms\n", rep, ms(t));
  }
  // 8 threads, one stream each, allocating / freeing concurrently
  for (int rep = 0; rep < 3; ++rep) {
    std::vector<std::thread> th;
    std::vector<double> worst(8, 0.0);
    t = Clock::now();
    for (int w = 0; w < 8; ++w)
      th.emplace_back([&, w] {
        cudaSetDevice(0);
        cudaStream_t s2;
        cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
        for (int k = 0; k < 4; ++k) {
          void *p = nullptr;
          const size_t sz = sizes[(w + k) % 9] / 2 + 4096;
          auto t2 = Clock::now();
          cudaMallocAsync(&p, sz, s2);
          double d = ms(t2);
          if (d > worst[w]) worst[w] = d;
          cudaMemsetAsync(p, 0, 1 << 20, s2);
          cudaFreeAsync(p, s2);
          cudaStreamSynchronize(s2);
        }
        cudaStreamDestroy(s2);
      });
    for (auto &x : th) x.join();
    double wm = 0;
    for (double d : worst) wm = d > wm ? d : wm;
    printf("threads rep %d: %.1f ms total, worst alloc %.3f ms\n", rep, ms(t), wm);
  }
  uint64_t reserved = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
  printf("reserved %.1f GB\n", reserved / (double)GB);
  return 0;
}
