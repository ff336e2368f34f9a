// Green-context probe (B200): do runtime-API launches into cuGreenCtx
// streams stay on the partition's SMs, and what HBM bandwidth does a
// streaming kernel reach on 8..148 SMs, alone and next to another partition?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/green_probe.cu -lcuda -o /tmp/green_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <set>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char *s; cuGetErrorString(r_, &s); \
  printf("FAIL %s: %s\n", #x, s); exit(1); } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(r_)); exit(1); } } while (0)

__global__ void smids(int *out) {
  if (threadIdx.x == 0) { unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); out[blockIdx.x] = (int)s; }
}
__global__ void big_smem(float *out) {
  extern __shared__ float sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sm[(threadIdx.x + 1) % blockDim.x] + 100000.f / 4 * 0;
}
__global__ void copy4(const float4 *__restrict__ a, float4 *__restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  RK(cudaSetDevice(0)); RK(cudaFree(0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs %u\n", all.sm.smCount);
  unsigned ng = 0;
  CK(cuDevSmResourceSplitByCount(nullptr, &ng, &all, nullptr, 0, 8));
  std::vector<CUdevResource> g(ng); CUdevResource rem;
  CK(cuDevSmResourceSplitByCount(g.data(), &ng, &all, &rem, 0, 8));
  printf("groups %u of %u SMs, remaining %u\n", ng, g[0].sm.smCount, rem.sm.smCount);
  const long n = (2L << 30) / 16;  // 2 GiB per buffer
  float4 *a, *b, *c, *d;
  RK(cudaMalloc(&a, n * 16)); RK(cudaMalloc(&b, n * 16)); RK(cudaMalloc(&c, n * 16)); RK(cudaMalloc(&d, n * 16));
  RK(cudaMemset(a, 1, n * 16)); RK(cudaMemset(c, 1, n * 16));
  int *ids; RK(cudaMalloc(&ids, 4096 * 4));
  auto mk = [&](int first, int count, CUstream *st) {
    std::vector<CUdevResource> r(g.begin() + first, g.begin() + first + count);
    CUdevResourceDesc desc; CK(cuDevResourceGenerateDesc(&desc, r.data(), count));
    CUgreenCtx gc; CK(cuGreenCtxCreate(&gc, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxStreamCreate(st, gc, CU_STREAM_NON_BLOCKING, 0));
  };
  auto timed = [&](cudaStream_t st, const float4 *x, float4 *y, int grid) {
    cudaEvent_t e0, e1; RK(cudaEventCreate(&e0)); RK(cudaEventCreate(&e1));
    copy4<<<grid, 512, 0, st>>>(x, y, n);
    RK(cudaEventRecord(e0, st));
    for (int k = 0; k < 3; ++k) copy4<<<grid, 512, 0, st>>>(x, y, n);
    RK(cudaEventRecord(e1, st)); RK(cudaEventSynchronize(e1));
    float ms; RK(cudaEventElapsedTime(&ms, e0, e1));
    return 3 * 2.0 * n * 16 / (ms * 1e-3) / 1e9;
  };
  for (int cnt : {1, 2, 4, 8, 9, 16, 18}) {
    if (cnt > (int)ng) continue;
    CUstream st; mk(0, cnt, &st);
    smids<<<2048, 32, 0, (cudaStream_t)st>>>(ids);
    RK(cudaGetLastError()); RK(cudaStreamSynchronize((cudaStream_t)st));
    std::vector<int> h(2048); RK(cudaMemcpy(h.data(), ids, 2048 * 4, cudaMemcpyDeviceToHost));
    std::set<int> u(h.begin(), h.end());
    printf("partition %3d SMs: kernel used %3zu distinct SMs; copy %.0f GB/s\n", cnt * 8, u.size(),
           timed((cudaStream_t)st, a, b, 2 * 148));
  }
  // two disjoint partitions of 9 groups each, concurrently
  CUstream s1, s2; mk(0, ng / 2, &s1); mk(ng / 2, ng - ng / 2, &s2);
  cudaEvent_t e0, e1, f0, f1; RK(cudaEventCreate(&e0)); RK(cudaEventCreate(&e1)); RK(cudaEventCreate(&f0)); RK(cudaEventCreate(&f1));
  RK(cudaDeviceSynchronize());
  RK(cudaEventRecord(e0, (cudaStream_t)s1)); RK(cudaEventRecord(f0, (cudaStream_t)s2));
  for (int k = 0; k < 3; ++k) { copy4<<<296, 512, 0, (cudaStream_t)s1>>>(a, b, n); copy4<<<296, 512, 0, (cudaStream_t)s2>>>(c, d, n); }
  RK(cudaEventRecord(e1, (cudaStream_t)s1)); RK(cudaEventRecord(f1, (cudaStream_t)s2)); RK(cudaDeviceSynchronize());
  float m1, m2; RK(cudaEventElapsedTime(&m1, e0, e1)); RK(cudaEventElapsedTime(&m2, f0, f1));
  printf("concurrent halves: %.0f + %.0f GB/s\n", 3 * 2.0 * n * 16 / (m1 * 1e-3) / 1e9, 3 * 2.0 * n * 16 / (m2 * 1e-3) / 1e9);
  // runtime API inside a green-context stream: >48 KB dynamic smem after
  // cudaFuncSetAttribute in the primary context, stream-ordered alloc,
  // async copies, events, a high-priority green stream
  {
    int lo = 0, hi = 0;
    RK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    std::vector<CUdevResource> r(g.begin(), g.begin() + 4);
    CUdevResourceDesc desc; CK(cuDevResourceGenerateDesc(&desc, r.data(), 4));
    CUgreenCtx gc; CK(cuGreenCtxCreate(&gc, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sh; CK(cuGreenCtxStreamCreate(&sh, gc, CU_STREAM_NON_BLOCKING, hi));
    cudaStream_t st = (cudaStream_t)sh;
    RK(cudaFuncSetAttribute(big_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    float *o = nullptr;
    RK(cudaMallocAsync((void **)&o, 1 << 20, st));
    big_smem<<<64, 256, 100 * 1024, st>>>(o);
    cudaError_t le = cudaGetLastError();
    printf("big-smem launch in green stream: %s\n", cudaGetErrorString(le));
    RK(cudaMemcpyAsync(o, a, 1 << 20, cudaMemcpyDeviceToDevice, st));
    cudaEvent_t x0, x1; RK(cudaEventCreate(&x0)); RK(cudaEventCreate(&x1));
    RK(cudaEventRecord(x0, st)); copy4<<<64, 512, 0, st>>>(a, b, n); RK(cudaEventRecord(x1, st));
    RK(cudaFreeAsync(o, st));
    cudaError_t se = cudaStreamSynchronize(st);
    float ms = 0; RK(cudaEventElapsedTime(&ms, x0, x1));
    printf("green stream (hi prio %d): malloc/copy/events ok=%s, 32-SM copy %.0f GB/s\n", hi,
           se == cudaSuccess ? "yes" : cudaGetErrorString(se), 2.0 * n * 16 / (ms * 1e-3) / 1e9);
    CUcontext cc; CK(cuCtxFromGreenCtx(&cc, gc));
    printf("cuCtxFromGreenCtx ok\n");
  }
  printf("ok\n");
  return 0;
}
