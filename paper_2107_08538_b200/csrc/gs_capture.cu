// gs_capture.cu — probe capture from real CUDA host code, and lazy replay.
//
// The reference derives a task's ResourceRequest from its trace by static
// analysis (task_builder.py:258-290) and, for lazy tasks, defers every
// unbound op until the first kernel launch: lazy_alloc hands out pseudo
// addresses, kernel_launch_prepare folds the queued allocation bytes into
// the request, and once the scheduler has picked a device, replay
// materializes the queue there (lazy_runtime.py:56-195, sim_engine.py:
// 417-449).  On a B200 the CUDA driver already records exactly that queue:
// the task's host code runs once against a stream in CAPTURE mode
// (cudaStreamBeginCapture), so
//   * cudaMallocAsync returns an address reserved for the graph but backs it
//     with no memory — the pseudo address (gs_capture_malloc);
//   * copies, memsets and kernel launches are recorded, not executed — the
//     queued ops;
//   * the recorded graph holds every launch's function, grid, block and
//     dynamic shared memory and every allocation's size, so the probe is
//     computed from what the code really launches (cudaFuncGetAttributes
//     for registers / static smem, gs_request_from_launches for the
//     reference's aggregation) — kernel_launch_prepare;
//   * launching the graph on the chosen device's stream allocates, copies
//     and runs the queue in recorded order, exactly once — replay; the
//     task's frees are free nodes, so nothing outlives it.
// gs_job_capture records a catalog job's whole device-side life this way
// (the executor's capture mode); gs_capture_begin / _end wrap arbitrary
// host code issued on the returned stream.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/gs.h"
#include "../../include/gs_work.h"
#include "gs_work_internal.h"

using namespace gsw;

#define CUC(call)                                                                 \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) return err(GS_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

struct gs_task_graph {
  int device = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  gs_probe probe{};
  int32_t n_kernels = 0, n_allocs = 0;
  int64_t alloc_bytes = 0;
  // catalog jobs: where the output digest lands (pinned), -1 otherwise
  unsigned long long *host_sum = nullptr;
};

namespace {

constexpr int64_t kHeapDefault = 8 << 20;  // task_builder.py:29
constexpr int64_t kGranule = 2 << 20;

// Nodes in dependency order (Kahn; ties by creation index) — a captured
// stream is a chain, so this is the order the host code issued them.
int topo_nodes(cudaGraph_t g, std::vector<cudaGraphNode_t> &out) {
  size_t n = 0;
  CUC(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  CUC(cudaGraphGetNodes(g, nodes.data(), &n));
  std::vector<int> indeg(n, 0);
  std::vector<std::vector<int>> succ(n);
  for (size_t i = 0; i < n; ++i) {
    size_t nd = 0;
    CUC(cudaGraphNodeGetDependentNodes(nodes[i], nullptr, &nd));
    std::vector<cudaGraphNode_t> dep(nd);
    if (nd) CUC(cudaGraphNodeGetDependentNodes(nodes[i], dep.data(), &nd));
    for (cudaGraphNode_t d : dep) {
      const size_t j = std::find(nodes.begin(), nodes.end(), d) - nodes.begin();
      if (j < n) {
        succ[i].push_back((int)j);
        indeg[j]++;
      }
    }
  }
  std::vector<int> ready;
  for (size_t i = 0; i < n; ++i)
    if (!indeg[i]) ready.push_back((int)i);
  out.clear();
  while (!ready.empty()) {
    std::sort(ready.begin(), ready.end(), std::greater<int>());
    const int i = ready.back();
    ready.pop_back();
    out.push_back(nodes[i]);
    for (int j : succ[i])
      if (--indeg[j] == 0) ready.push_back(j);
  }
  if (out.size() != n) return err(GS_ERR_CUDA, "captured graph has a cycle");
  return GS_OK;
}

// kernel_launch_prepare over a recorded graph: every kernel node's launch
// shape and every allocation node's bytes (on the 2 MiB granule the
// executor allocates in), aggregated by the reference's rule.
int probe_of_graph(gs_task_graph *t, int64_t heap) {
  std::vector<cudaGraphNode_t> nodes;
  int rc = topo_nodes(t->graph, nodes);
  if (rc) return rc;
  std::vector<gs_launch_desc> launches;
  std::vector<int64_t> bytes;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    CUC(cudaGraphNodeGetType(nd, &ty));
    if (ty == cudaGraphNodeTypeKernel) {
      cudaKernelNodeParams kp;
      CUC(cudaGraphKernelNodeGetParams(nd, &kp));
      gs_launch_desc d;
      const int grid = (int)(kp.gridDim.x * kp.gridDim.y * kp.gridDim.z);
      const int block = (int)(kp.blockDim.x * kp.blockDim.y * kp.blockDim.z);
      rc = gs_launch_desc_of(kp.func, grid, block, (int32_t)kp.sharedMemBytes, &d);
      if (rc) return rc;
      launches.push_back(d);
    } else if (ty == cudaGraphNodeTypeMemAlloc) {
      cudaMemAllocNodeParams ap;
      CUC(cudaGraphMemAllocNodeGetParams(nd, &ap));
      const int64_t b = ((int64_t)ap.bytesize + kGranule - 1) / kGranule * kGranule;
      bytes.push_back(b);
      t->alloc_bytes += b;
    }
  }
  t->n_kernels = (int32_t)launches.size();
  t->n_allocs = (int32_t)bytes.size();
  if (launches.empty()) return err(GS_ERR_CONFIG, "captured task launched no kernel");
  return gs_request_from_launches(launches.data(), (int32_t)launches.size(), bytes.data(), (int32_t)bytes.size(),
                                  heap, &t->probe);
}

}  // namespace

namespace gsw {
// gs_exec.cu: the staged inputs of `j` on `device` (device copy or pinned
// host copy), or nullptr
const void *staged_input(const gs_job_desc &j, int device, size_t buf, bool *host);
}

extern "C" {

int gs_capture_begin(int32_t cuda_device, void **stream) {
  CUC(cudaSetDevice(cuda_device));
  cudaStream_t st;
  CUC(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaStreamDestroy(st);
    return err(GS_ERR_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e));
  }
  *stream = st;
  return GS_OK;
}

int gs_capture_malloc(void *stream, int64_t bytes, void **ptr) {
  if (bytes <= 0) return err(GS_ERR_CONFIG, "allocation size must be positive");
  CUC(cudaMallocAsync(ptr, (size_t)bytes, (cudaStream_t)stream));
  return GS_OK;
}

int gs_capture_free(void *stream, void *ptr) {
  CUC(cudaFreeAsync(ptr, (cudaStream_t)stream));
  return GS_OK;
}

int gs_capture_end(void *stream, int64_t heap_limit_bytes, gs_task_graph **out) {
  cudaStream_t st = (cudaStream_t)stream;
  auto *t = new gs_task_graph;
  cudaGetDevice(&t->device);
  const cudaError_t e = cudaStreamEndCapture(st, &t->graph);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) {
    delete t;
    return err(GS_ERR_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
  }
  const int rc = probe_of_graph(t, heap_limit_bytes > 0 ? heap_limit_bytes : kHeapDefault);
  if (rc) {
    cudaGraphDestroy(t->graph);
    delete t;
    return rc;
  }
  *out = t;
  return GS_OK;
}

int gs_task_graph_probe(const gs_task_graph *g, gs_probe *out, int32_t *n_kernels, int32_t *n_allocs) {
  if (!g) return err(GS_ERR_CONFIG, "null task graph");
  if (out) *out = g->probe;
  if (n_kernels) *n_kernels = g->n_kernels;
  if (n_allocs) *n_allocs = g->n_allocs;
  return GS_OK;
}

// replay: materialize the recorded queue on the capture device's `stream`
// (instantiated on first use) and wait for it.  *checksum gets a catalog
// job's output digest; *ms the graph's device time.
int gs_task_graph_run(gs_task_graph *g, void *stream, uint64_t *checksum, float *ms) {
  if (!g) return err(GS_ERR_CONFIG, "null task graph");
  CUC(cudaSetDevice(g->device));
  if (!g->exec) CUC(cudaGraphInstantiate(&g->exec, g->graph, 0));
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms) {
    CUC(cudaEventCreate(&e0));
    CUC(cudaEventCreate(&e1));
    CUC(cudaEventRecord(e0, st));
  }
  cudaError_t e = cudaGraphLaunch(g->exec, st);
  if (e == cudaSuccess && ms) e = cudaEventRecord(e1, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && ms) e = cudaEventElapsedTime(ms, e0, e1);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (e != cudaSuccess) return err(GS_ERR_CUDA, std::string("task graph replay: ") + cudaGetErrorString(e));
  if (checksum) *checksum = g->host_sum ? *g->host_sum : 0;
  return GS_OK;
}

int gs_task_graph_device(const gs_task_graph *g) { return g ? g->device : -1; }

void gs_task_graph_destroy(gs_task_graph *g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  if (g->host_sum) cudaFreeHost(g->host_sum);
  delete g;
}

// A catalog job's whole device-side life captured on `cuda_device`:
// allocations, SCR zero-fills, input copies from the job's staged inputs
// (device copy on that GPU, else the pinned host copy), its kernels, the
// output digest and its read-back, and the frees.  Jobs whose host code
// reads device results between launches (bfs: the level loop) cannot be
// captured (GS_ERR_CONFIG).
int gs_job_capture(const gs_job_desc *job, int32_t cuda_device, gs_task_graph **out) {
  int rc = validate(*job);
  if (rc) return rc;
  if (job->kind == GS_JOB_BFS) return err(GS_ERR_CONFIG, "bfs reads its frontier count on the host: not capturable");
  unsigned long long *host_sum = nullptr;
  CUC(cudaSetDevice(cuda_device));
  CUC(cudaHostAlloc((void **)&host_sum, 16, 0));
  void *sv = nullptr;
  rc = gs_capture_begin(cuda_device, &sv);
  if (rc) {
    cudaFreeHost(host_sum);
    return rc;
  }
  cudaStream_t st = (cudaStream_t)sv;
  const std::vector<Buf> bufs = job_buffers(*job);
  std::vector<void *> buf(bufs.size(), nullptr);
  unsigned long long *dsum = nullptr;
  int32_t scalar[4] = {0, 0, 0, 0};
  auto body = [&]() -> int {
    for (size_t i = 0; i < bufs.size(); ++i) CUC(cudaMallocAsync(&buf[i], bufs[i].bytes, st));
    CUC(cudaMallocAsync((void **)&dsum, 32, st));
    CUC(cudaMemsetAsync(dsum, 0, 32, st));
    for (size_t i = 0; i < bufs.size(); ++i) {
      if (bufs[i].role == IN || bufs[i].role == INOUT) {
        bool host = false;
        const void *src = staged_input(*job, cuda_device, i, &host);
        if (!src) return err(GS_ERR_CONFIG, "stage the job's inputs (gs_exec_stage) before capturing it");
        (void)host;  // (UVA: host, own-device or peer copy alike)
        CUC(cudaMemcpyAsync(buf[i], src, bufs[i].bytes, cudaMemcpyDefault, st));
      } else if (bufs[i].role == SCR) {
        CUC(cudaMemsetAsync(buf[i], 0, bufs[i].bytes, st));
      }
    }
    int out_idx = 0;
    int64_t launches = 0;
    int r = run_kernels(*job, buf, st, &out_idx, &launches, scalar, reinterpret_cast<unsigned *>(dsum + 1));
    if (r) return r;
    r = digest(buf[out_idx], bufs[out_idx].bytes, dsum, st);
    if (r) return r;
    CUC(cudaMemcpyAsync(host_sum, dsum, 8, cudaMemcpyDeviceToHost, st));
    for (void *p : buf) CUC(cudaFreeAsync(p, st));
    CUC(cudaFreeAsync(dsum, st));
    return GS_OK;
  };
  rc = body();
  gs_task_graph *t = nullptr;
  const int rc2 = gs_capture_end(sv, kHeapDefault, &t);  // always ends the capture
  if (rc || rc2) {
    gs_task_graph_destroy(t);
    cudaFreeHost(host_sum);
    return rc ? rc : rc2;
  }
  t->host_sum = host_sum;
  *out = t;
  return GS_OK;
}

}  // extern "C"
