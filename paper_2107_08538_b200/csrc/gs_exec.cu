// gs_exec.cu — the executor: real jobs under the placement engine.
//
// Replaces the reference's virtual-time runtime (sim_engine.py: worker pool
// _on_pull :286-303, probe admission _handle_probe :393-415, processor-
// sharing _Pool :191-218, release + FIFO re-drive :541-547 / :278-282) with
// wall-clock execution on B200s:
//   * W worker threads pull jobs in order (the reference's workers);
//   * each job's probe (footprint + launch shape, gs_job_probe) is decided
//     by the GPU decision kernel (gs_submit); DEFER parks the worker until a
//     release re-drives the FIFO (gs_on_release) and admits it;
//   * the job runs on its own stream of the chosen device, allocating from
//     that device's stream-ordered pool — the ledger never promises more
//     than the pool can give, so memory-safe policies cannot OOM; sa / cg
//     allocate without checks and can (a failed allocation is an "oom"
//     crash record, sim_engine.py:342-350);
//   * completion releases the task's ledger entry and re-drives the queue.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gs.h"
#include "../../include/gs_work.h"
#include "gs_arena.h"
#include "gs_cache.h"
#include "gs_work_internal.h"

using namespace gsw;

#define CUE(call)                                                                 \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) return err(GS_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

namespace {

using Clock = std::chrono::steady_clock;

static const bool g_alloc_log = getenv("GS_ALLOC_LOG") != nullptr;

double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// Staged inputs of one job: device buffers (GS_MODE_DEVICE) or pinned host
// buffers (GS_MODE_E2E), one per job buffer (nullptr for OUT/SCR).
struct Staged {
  gs_job_desc desc{};
  int device = 0;
  bool host = false;
  std::vector<void *> ptr;
  void *host_out = nullptr;  // e2e: pinned destination of the job's outputs
  int64_t host_out_bytes = 0;
};

std::mutex g_stage_mu;
std::vector<Staged> g_staged;

// Placement log of the most recent run (gs_exec_log): every decision-engine
// call in the order the single decision authority made it.
std::mutex g_log_mu;
std::vector<gs_exec_event> g_log;
std::vector<gs_spec> g_log_specs;
int32_t g_log_policy = 0, g_log_cg_ratio = 0;

void free_staged(Staged &s) {
  for (void *p : s.ptr) {
    if (!p) continue;
    if (s.host) cudaFreeHost(p);
    else cudaFree(p);
  }
  s.ptr.clear();
  if (s.host_out) cudaFreeHost(s.host_out);
  s.host_out = nullptr;
}

// Capacity of a job's pinned output area: every buffer that can hold an
// output (OUT, INOUT, and the ping-pong scratch SCR of hotspot / srad).
int64_t e2e_out_bytes(const gs_job_desc &j) {
  int64_t o = 0;
  for (const Buf &b : job_buffers(j))
    if (b.role != IN && b.role != WRK) o += b.bytes;
  return o;
}

bool same_desc(const gs_job_desc &a, const gs_job_desc &b) { return memcmp(&a, &b, sizeof(a)) == 0; }

// The staged inputs of job `d` for a run on `device`: that device's own
// copy first (device mode stages one per fleet GPU), else a pinned host copy
// (e2e), else any device's copy (pulled over NVLink by a peer copy).
const Staged *find_staged(const gs_job_desc &d, int device = -1) {
  const Staged *any = nullptr;
  for (const Staged &s : g_staged) {
    if (!same_desc(s.desc, d)) continue;
    if (s.host || s.device == device) return &s;
    if (!any) any = &s;
  }
  return any;
}

}  // namespace

namespace gsw {
// the capture path's view of the staged inputs (gs_capture.cu)
const void *staged_input(const gs_job_desc &j, int device, size_t i, bool *host) {
  std::lock_guard<std::mutex> g(g_stage_mu);
  const Staged *s = find_staged(j, device);
  if (!s || i >= s->ptr.size() || !s->ptr[i]) return nullptr;
  *host = s->host;
  return s->ptr[i];
}
}  // namespace gsw

namespace {

bool staged_on(const gs_job_desc &d, int device, bool host) {
  for (const Staged &s : g_staged)
    if (same_desc(s.desc, d) && s.host == host && (host || s.device == device)) return true;
  return false;
}

// Per-device job arenas (gs_arena.h), process-lifetime: the slab is
// allocated once and reused by every later run whose ledger capacity fits
// in it (a run limits it to its own capacity); a larger capacity replaces
// it between runs.  GS_ARENA=0 falls back to the stream-ordered pool.
std::mutex g_arena_mu;
std::map<int, gsa::Arena *> g_arenas;

static bool arena_enabled() {
  const char *e = getenv("GS_ARENA");
  return !(e && e[0] == '0');
}

static int64_t arena_idle_bytes(int device) {
  std::lock_guard<std::mutex> g(g_arena_mu);
  auto it = g_arenas.find(device);
  return it != g_arenas.end() && it->second->in_use() == 0 ? it->second->size() : 0;
}

// free an idle arena (staging or another allocator needs the memory)
void arena_drop_idle(int device) {
  std::lock_guard<std::mutex> g(g_arena_mu);
  auto it = g_arenas.find(device);
  if (it == g_arenas.end() || it->second->in_use()) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaDeviceSynchronize();
  cudaFree(it->second->base());
  delete it->second;
  g_arenas.erase(it);
  cudaSetDevice(prev);
}

// engine-internal allocations that find the device full give the idle
// arena back first (gs_cache.h)
struct ArenaOomHook {
  ArenaOomHook() { gscache::set_oom_hook(arena_drop_idle); }
} g_arena_oom_hook;

static gsa::Arena *arena_for(int device, int64_t capacity) {
  std::lock_guard<std::mutex> g(g_arena_mu);
  gsa::Arena *&a = g_arenas[device];
  capacity = capacity / gsa::kGranule * gsa::kGranule;  // whole granules
  if (a && a->size() >= capacity && a->reset(capacity)) return a;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  if (a) {
    if (a->in_use()) {
      cudaSetDevice(prev);
      return nullptr;
    }
    cudaFree(a->base());
    delete a;
    a = nullptr;
  }
  // memory the stream-ordered pool keeps (solo runs) goes back first
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
  }
  char *base = nullptr;
  const int64_t size = capacity;
  if (size > 0 && cudaMalloc((void **)&base, (size_t)size) == cudaSuccess) {
    a = new gsa::Arena(device, base, size);
  } else {
    cudaGetLastError();
  }
  cudaSetDevice(prev);
  return a;
}

int stage_one(const gs_job_desc &j, int device, int mode, Staged &out) {
  CUE(cudaSetDevice(device));
  const std::vector<Buf> bufs = job_buffers(j);
  std::vector<void *> dev(bufs.size(), nullptr);
  out.desc = j;
  out.device = device;
  out.host = mode == GS_MODE_E2E;
  out.ptr.assign(bufs.size(), nullptr);
  cudaStream_t st;
  CUE(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (size_t i = 0; i < bufs.size(); ++i)
    if (bufs[i].role == IN || bufs[i].role == INOUT) {
      if (cudaMalloc(&dev[i], bufs[i].bytes) != cudaSuccess) {
        cudaGetLastError();  // an idle job arena holds the memory: give it back and retry
        arena_drop_idle(device);
        CUE(cudaMalloc(&dev[i], bufs[i].bytes));
      }
    }
  int rc = generate_inputs(j, dev, st);
  if (rc) return rc;
  for (size_t i = 0; i < bufs.size(); ++i) {
    if (!dev[i]) continue;
    if (out.host) {
      CUE(cudaHostAlloc(&out.ptr[i], bufs[i].bytes, cudaHostAllocPortable));
      CUE(cudaMemcpyAsync(out.ptr[i], dev[i], bufs[i].bytes, cudaMemcpyDeviceToHost, st));
    } else {
      out.ptr[i] = dev[i];
      dev[i] = nullptr;
    }
  }
  if (out.host) {  // the user's pinned output buffers, allocated outside the timed region
    out.host_out_bytes = e2e_out_bytes(j);
    CUE(cudaHostAlloc(&out.host_out, out.host_out_bytes, cudaHostAllocPortable));
  }
  CUE(cudaStreamSynchronize(st));
  for (void *p : dev)
    if (p) cudaFree(p);
  cudaStreamDestroy(st);
  return GS_OK;
}

// One job, start to finish, on (device, stream).  *oom is set when the
// device pool refused an allocation.
int run_job(const gs_job_desc &j, const Staged *stg, int mode, cudaStream_t st, gs_job_record &rec, bool *oom,
            void *host_out, int64_t host_out_bytes, int32_t *host_scalar, std::atomic<int64_t> *kernel_count,
            unsigned long long *host_sum, int device, gsa::Arena *arena = nullptr, bool wait_mem = false) {
  *oom = false;
  const auto t_admit = Clock::now();
  const std::vector<Buf> bufs = job_buffers(j);
  std::vector<void *> buf(bufs.size(), nullptr);
  unsigned long long *dsum = nullptr;
  // arena requests: every buffer, then the control block (one granule of
  // the job's heap allowance)
  std::vector<int64_t> req;
  std::vector<void *> got;
  std::vector<int> slot(bufs.size(), -1);  // buffer -> arena request index
  // Read-only inputs (IN) of a job whose inputs are resident on its own
  // GPU are read in place: the job's kernels never write an IN buffer, so
  // copying 50 GB of them per cfg 1 step D2D was pure HBM traffic.  INOUT
  // buffers (modified in place) still get a private copy.
  // An INOUT buffer whose first kernel reads a separate source
  // (reads_source: hotspot T, srad J, backprop w1) gets its private buffer
  // uninitialised and the resident input as that source: 36 GB less D2D
  // copy traffic per cfg 1 step.
  // From pinned host memory (e2e) a job moves only real inputs over PCIe:
  // derived inputs (bfs's transposed CSR) are rebuilt on the device, and
  // needle copies only its score matrix's boundary (reads_source_host).
  std::vector<char> alias(bufs.size(), 0), derive(bufs.size(), 0);
  std::vector<const void *> src(bufs.size(), nullptr);
  if (stg && !stg->host && stg->device == device)
    for (size_t i = 0; i < bufs.size(); ++i) {
      alias[i] = bufs[i].role == IN && stg->ptr[i] != nullptr;
      if (bufs[i].role == INOUT && stg->ptr[i] != nullptr && reads_source(j, i)) src[i] = stg->ptr[i];
    }
  bool need_derive = false;
  if (stg && stg->host)
    for (size_t i = 0; i < bufs.size(); ++i) {
      if (derived_input(j, i)) derive[i] = need_derive = true;
      if (bufs[i].role == INOUT && stg->ptr[i] != nullptr && reads_source_host(j, i)) {
        src[i] = stg->ptr[i];
        rec.h2d_bytes += source_host_bytes(j, i);  // copied by the job's first step
      }
    }
  auto release = [&]() {
    if (arena) {
      cudaStreamSynchronize(st);
      if (!got.empty()) arena->free_all(got, req);
      got.clear();
      return;
    }
    for (size_t i = 0; i < buf.size(); ++i)
      if (buf[i] && !alias[i]) cudaFreeAsync(buf[i], st);
    if (dsum) cudaFreeAsync(dsum, st);
    cudaStreamSynchronize(st);
  };
  if (arena) {
    for (size_t i = 0; i < bufs.size(); ++i)
      if (!alias[i]) {
        slot[i] = (int)req.size();
        req.push_back(bufs[i].bytes);
      }
    req.push_back(32);
    double waited = 0;
    if (!arena->alloc_all(req, got, wait_mem, &waited)) {
      got.clear();
      *oom = true;
      return GS_OK;
    }
    for (size_t i = 0; i < bufs.size(); ++i) buf[i] = alias[i] ? stg->ptr[i] : got[slot[i]];
    dsum = (unsigned long long *)got.back();
  }
  for (size_t i = 0; i < bufs.size() && !arena; ++i) {
    if (alias[i]) {
      buf[i] = stg->ptr[i];
      continue;
    }
    const auto ta = Clock::now();
    cudaError_t e = cudaMallocAsync(&buf[i], bufs[i].bytes, st);
    if (g_alloc_log && ms_since(ta) > 5.0)
      fprintf(stderr, "[gs alloc] %.1f ms for %lld B (rc %d)\n", ms_since(ta), (long long)bufs[i].bytes, (int)e);
    if (e == cudaErrorMemoryAllocation) {
      // the pool may hold enough free memory in chunks too small for this
      // buffer: give the unused chunks back and retry once
      cudaGetLastError();
      cudaMemPool_t pool;
      const auto tt = Clock::now();
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
      e = cudaMallocAsync(&buf[i], bufs[i].bytes, st);
      if (g_alloc_log)
        fprintf(stderr, "[gs alloc] trim+retry %.1f ms for %lld B (rc %d)\n", ms_since(tt), (long long)bufs[i].bytes,
                (int)e);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      buf[i] = nullptr;
      release();
      if (e == cudaErrorMemoryAllocation) {
        *oom = true;
        return GS_OK;
      }
      return err(GS_ERR_CUDA, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    }
  }
  // 32 B of job control: [0] the output digest, [1..] the kernels' tile tickets
  if (!arena && cudaMallocAsync((void **)&dsum, 32, st) != cudaSuccess) {
    cudaGetLastError();
    dsum = nullptr;
    release();
    *oom = true;
    return GS_OK;
  }
  // from here on every return path (errors included) destroys the events
  // and gives the job's memory back
  cudaEvent_t es = nullptr, e0 = nullptr, e1 = nullptr, ed = nullptr;
  struct Cleanup {
    std::function<void()> f;
    ~Cleanup() { f(); }
  } cleanup{[&]() {
    for (cudaEvent_t ev : {es, e0, e1, ed})
      if (ev) cudaEventDestroy(ev);
    release();
  }};
  CUE(cudaEventCreate(&es));
  CUE(cudaEventCreate(&e0));
  CUE(cudaEventCreate(&e1));
  CUE(cudaEventCreate(&ed));
  CUE(cudaEventRecord(es, st));
  CUE(cudaMemsetAsync(dsum, 0, 32, st));
  // inputs in
  for (size_t i = 0; i < bufs.size(); ++i) {
    if (alias[i] || src[i] || derive[i]) continue;  // read in place / rebuilt below
    if (bufs[i].role == IN || bufs[i].role == INOUT) {
      if (stg) {
        if (stg->host) {
          CUE(cudaMemcpyAsync(buf[i], stg->ptr[i], bufs[i].bytes, cudaMemcpyHostToDevice, st));
          rec.h2d_bytes += bufs[i].bytes;
        } else if (stg->device == device) {
          CUE(cudaMemcpyAsync(buf[i], stg->ptr[i], bufs[i].bytes, cudaMemcpyDeviceToDevice, st));
        } else {
          CUE(cudaMemcpyPeerAsync(buf[i], device, stg->ptr[i], stg->device, bufs[i].bytes, st));
        }
      }
    } else if (bufs[i].role == SCR) {
      CUE(cudaMemsetAsync(buf[i], 0, bufs[i].bytes, st));
    }
  }
  if (!stg) {  // unstaged: synthesize the inputs in place
    int rc = generate_inputs(j, buf, st);
    if (rc) return rc;
  } else if (need_derive) {
    int rc = derive_inputs(j, buf, st);
    if (rc) return rc;
  }
  rec.setup_ms = ms_since(t_admit);
  CUE(cudaEventRecord(e0, st));
  int out_idx = 0;
  int64_t launches = 0;
  bool digested = false;
  int rc = run_kernels(j, buf, st, &out_idx, &launches, host_scalar, reinterpret_cast<unsigned *>(dsum + 1),
                       src.data(), &digested);
  if (rc) return rc;
  CUE(cudaEventRecord(e1, st));
  rec.n_kernels = (int32_t)launches;
  kernel_count->fetch_add(launches + (digested ? 0 : 1));
  // outputs: the primary output buffer (and every OUT buffer in e2e); its
  // digest unless the last kernel already summed it
  if (!digested) {
    rc = digest(buf[out_idx], bufs[out_idx].bytes, dsum, st);
    if (rc) return rc;
  }
  if (mode == GS_MODE_E2E) {
    if (stg && stg->host_out) {
      host_out = stg->host_out;
      host_out_bytes = stg->host_out_bytes;
    }
    int64_t off = 0;
    for (size_t i = 0; i < bufs.size(); ++i) {
      const bool is_out = bufs[i].role == OUT || (int)i == out_idx;
      if (!is_out) continue;
      if (host_out && off + bufs[i].bytes <= host_out_bytes) {
        CUE(cudaMemcpyAsync((char *)host_out + off, buf[i], bufs[i].bytes, cudaMemcpyDeviceToHost, st));
        off += bufs[i].bytes;
        rec.d2h_bytes += bufs[i].bytes;
      }
    }
  } else if (host_out && bufs[out_idx].bytes <= host_out_bytes) {
    CUE(cudaMemcpyAsync(host_out, buf[out_idx], bufs[out_idx].bytes, cudaMemcpyDeviceToHost, st));
  }
  CUE(cudaMemcpyAsync(host_sum, dsum, 8, cudaMemcpyDeviceToHost, st));
  rec.d2h_bytes += 8;
  CUE(cudaEventRecord(ed, st));
  CUE(cudaStreamSynchronize(st));
  float ms = 0;
  CUE(cudaEventElapsedTime(&ms, e0, e1));
  rec.compute_ms = ms;
  CUE(cudaEventElapsedTime(&ms, es, e0));
  rec.gen_ms = ms;
  CUE(cudaEventElapsedTime(&ms, e1, ed));
  rec.tail_ms = ms;
  rec.checksum = *host_sum + (digested ? digest_tail(bufs[out_idx].bytes) : 0ull);
  return GS_OK;
}

int64_t max_out_bytes(const gs_job_desc *jobs, int n) {
  int64_t m = 0;
  for (int i = 0; i < n; ++i) {
    int64_t o = 0;
    for (const Buf &b : job_buffers(jobs[i])) o += b.bytes;  // conservative: every buffer
    m = std::max(m, o);
  }
  return m;
}

}  // namespace

extern "C" {

int gs_exec_stage(const gs_job_desc *jobs, int32_t n_jobs, const int32_t *cuda_devices, int32_t n_devices,
                  int32_t mode) {
  std::lock_guard<std::mutex> g(g_stage_mu);
  // Identical jobs (same descriptor: a template's instances) share one
  // staged copy: device mode stages a copy on EVERY listed device (a job
  // reads its inputs from the GPU it was placed on), e2e mode one pinned
  // host copy (portable: any device's copy engine reads it).
  const bool host = mode == GS_MODE_E2E;
  for (int i = 0; i < n_jobs; ++i) {
    int rc = validate(jobs[i]);
    if (rc) return rc;
    for (int d = 0; d < (host ? 1 : n_devices); ++d) {
      if (staged_on(jobs[i], cuda_devices[d], host)) continue;
      Staged s;
      rc = stage_one(jobs[i], cuda_devices[d], mode, s);
      if (rc) {
        free_staged(s);
        return rc;
      }
      g_staged.push_back(std::move(s));
    }
  }
  return GS_OK;
}

int gs_exec_log(gs_exec_event *events, int64_t cap, int64_t *n_events, gs_spec *specs, int32_t spec_cap,
                int32_t *n_devices, int32_t *policy, int32_t *cg_ratio) {
  std::lock_guard<std::mutex> g(g_log_mu);
  if (n_events) *n_events = (int64_t)g_log.size();
  if (events && cap > 0) memcpy(events, g_log.data(), sizeof(gs_exec_event) * std::min<int64_t>(cap, g_log.size()));
  if (n_devices) *n_devices = (int32_t)g_log_specs.size();
  if (specs && spec_cap > 0)
    memcpy(specs, g_log_specs.data(), sizeof(gs_spec) * std::min<size_t>(spec_cap, g_log_specs.size()));
  if (policy) *policy = g_log_policy;
  if (cg_ratio) *cg_ratio = g_log_cg_ratio;
  return GS_OK;
}

void gs_exec_unstage(void) {
  gs_exec_drop_graphs();  // recorded graphs copy from the staged inputs
  std::lock_guard<std::mutex> g(g_stage_mu);
  for (Staged &s : g_staged) free_staged(s);
  g_staged.clear();
}

// ---- green-context SM partitions (gs_exec_set_sm_parts) -------------------
// Built once per (device, parts) and kept for the process: the device's SMs
// are split into 8-SM groups (plus the remainder group the split leaves),
// and the groups are dealt to the partitions largest-first onto the
// partition with the fewest SMs so far.  Each partition has a default- and
// a high-priority stream created in its green context; runtime-API work
// (cudaMallocAsync, copies, launches, events) issued to those streams runs
// on the partition's SMs only (measured: tools/green_probe.cu).
struct GreenPart {
  CUgreenCtx g = nullptr;
  cudaStream_t lo = nullptr, hi = nullptr;
  int sms = 0;
};
struct GreenSet {
  std::vector<GreenPart> parts;
  std::vector<char> busy;
  std::mutex mu;
  std::condition_variable cv;
  int acquire() {
    std::unique_lock<std::mutex> lk(mu);
    for (;;) {
      for (size_t i = 0; i < busy.size(); ++i)
        if (!busy[i]) {
          busy[i] = 1;
          return (int)i;
        }
      cv.wait(lk);
    }
  }
  void release(int i) {
    {
      std::lock_guard<std::mutex> g(mu);
      busy[i] = 0;
    }
    cv.notify_one();
  }
};
std::mutex g_green_mu;
std::map<std::pair<int, int>, GreenSet *> g_green;
std::atomic<int> g_sm_parts{0};
std::atomic<bool> g_capture{false};

#define CUD(call)                                                                  \
  do {                                                                             \
    CUresult r_ = (call);                                                          \
    if (r_ != CUDA_SUCCESS) {                                                      \
      const char *s_ = nullptr;                                                    \
      green_api().getErrorString(r_, &s_);                                         \
      return err(GS_ERR_CUDA, std::string(#call ": ") + (s_ ? s_ : "?"));          \
    }                                                                              \
  } while (0)

// Driver entry points, resolved through the runtime (libgs does not link
// libcuda: the library must load on hosts without a driver).
struct GreenApi {
  CUresult (*getErrorString)(CUresult, const char **) = nullptr;
  CUresult (*deviceGet)(CUdevice *, int) = nullptr;
  CUresult (*getDevResource)(CUdevice, CUdevResource *, CUdevResourceType) = nullptr;
  CUresult (*split)(CUdevResource *, unsigned *, const CUdevResource *, CUdevResource *, unsigned, unsigned) = nullptr;
  CUresult (*genDesc)(CUdevResourceDesc *, CUdevResource *, unsigned) = nullptr;
  CUresult (*create)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
  CUresult (*streamCreate)(CUstream *, CUgreenCtx, unsigned, int) = nullptr;
  bool ok = false;
};
static const GreenApi &green_api() {
  static GreenApi a = [] {
    GreenApi g;
    auto get = [](const char *name, void **fn) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        *fn = nullptr;
      return *fn != nullptr;
    };
    g.ok = get("cuGetErrorString", (void **)&g.getErrorString) && get("cuDeviceGet", (void **)&g.deviceGet) &&
           get("cuDeviceGetDevResource", (void **)&g.getDevResource) &&
           get("cuDevSmResourceSplitByCount", (void **)&g.split) &&
           get("cuDevResourceGenerateDesc", (void **)&g.genDesc) && get("cuGreenCtxCreate", (void **)&g.create) &&
           get("cuGreenCtxStreamCreate", (void **)&g.streamCreate);
    return g;
  }();
  return a;
}

static int green_for(int device, int parts, GreenSet **out) {
  std::lock_guard<std::mutex> g(g_green_mu);
  GreenSet *&gs = g_green[{device, parts}];
  if (gs) {
    *out = gs;
    return GS_OK;
  }
  CUE(cudaSetDevice(device));
  CUE(cudaFree(0));  // the driver and the primary context exist before the green ones
  const GreenApi &A = green_api();
  if (!A.ok) return err(GS_ERR_CUDA, "green-context driver entry points unavailable");
  CUdevice dev;
  CUD(A.deviceGet(&dev, device));
  CUdevResource all;
  CUD(A.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  unsigned ng = 0;
  CUD(A.split(nullptr, &ng, &all, nullptr, 0, 8));
  std::vector<CUdevResource> grp(ng + 1);
  CUdevResource rem;
  CUD(A.split(grp.data(), &ng, &all, &rem, 0, 8));
  grp.resize(ng);
  if (rem.sm.smCount > 0) grp.push_back(rem);
  if (parts < 1 || parts > (int)grp.size()) return err(GS_ERR_CONFIG, "more SM partitions than 8-SM groups");
  std::vector<int> order(grp.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return grp[a].sm.smCount > grp[b].sm.smCount; });
  std::vector<std::vector<CUdevResource>> deal(parts);
  std::vector<int> sms(parts, 0);
  for (int i : order) {
    const int p = (int)(std::min_element(sms.begin(), sms.end()) - sms.begin());
    deal[p].push_back(grp[i]);
    sms[p] += grp[i].sm.smCount;
  }
  int lo = 0, hi = 0;
  CUE(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  auto *set = new GreenSet;
  set->parts.resize(parts);
  set->busy.assign(parts, 0);
  for (int p = 0; p < parts; ++p) {
    CUdevResourceDesc desc;
    CUD(A.genDesc(&desc, deal[p].data(), (unsigned)deal[p].size()));
    GreenPart &gp = set->parts[p];
    CUD(A.create(&gp.g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream a, b;
    CUD(A.streamCreate(&a, gp.g, CU_STREAM_NON_BLOCKING, 0));
    CUD(A.streamCreate(&b, gp.g, CU_STREAM_NON_BLOCKING, hi));
    gp.lo = (cudaStream_t)a;
    gp.hi = (cudaStream_t)b;
    gp.sms = sms[p];
  }
  gs = set;
  *out = set;
  return GS_OK;
}

// The device pool jobs allocate from.  Growing a stream-ordered pool maps
// fresh physical memory (measured ~5.5 ms per GiB on B200) under a driver
// lock every worker thread then waits on, and a pool grown piecemeal by
// jobs of different sizes fragments.  So the pool never trims
// (release threshold = max) and, before a run, it is grown ONCE, as one
// chunk, to `need` bytes: the most the run can have allocated at a time.
static void prepare_pool(int device, int64_t need) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  uint64_t reserved = 0, used = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  if (need <= 0 || (int64_t)(reserved - used) >= need) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess) {
    const auto t = Clock::now();
    if (used == 0) cudaMemPoolTrimTo(pool, 0);  // start from one clean chunk
    void *p = nullptr;
    if (cudaMallocAsync(&p, (size_t)need, st) == cudaSuccess) cudaFreeAsync(p, st);
    cudaGetLastError();  // a pool that cannot grow that far still works, piecemeal
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (g_alloc_log) fprintf(stderr, "[gs alloc] pool grown to %lld B in %.1f ms\n", (long long)need, ms_since(t));
  }
  cudaSetDevice(prev);
}

void gs_exec_release_memory(void) {
  std::vector<int> devs;
  {
    std::lock_guard<std::mutex> g(g_arena_mu);
    for (auto &kv : g_arenas) devs.push_back(kv.first);
  }
  for (int d : devs) arena_drop_idle(d);
}

// Recorded task graphs of catalog jobs, kept per (job descriptor, device)
// for the process: instances of one template record the same graph, so a
// graph is recorded and instantiated once and replayed by every later
// instance (one replay at a time per cached graph; a busy template records
// another).  Replays reuse the graph-memory pool's mapped memory.
std::mutex g_graph_mu;
std::map<std::pair<std::string, int>, std::vector<gs_task_graph *>> g_graph_cache;

static std::string desc_key(const gs_job_desc &d) { return std::string((const char *)&d, sizeof d); }

static int graph_take(const gs_job_desc &j, int device, gs_task_graph **out) {
  {
    std::lock_guard<std::mutex> g(g_graph_mu);
    auto &v = g_graph_cache[{desc_key(j), device}];
    if (!v.empty()) {
      *out = v.back();
      v.pop_back();
      return GS_OK;
    }
  }
  return gs_job_capture(&j, device, out);
}

static void graph_give(const gs_job_desc &j, gs_task_graph *t) {
  if (!t) return;
  std::lock_guard<std::mutex> g(g_graph_mu);
  g_graph_cache[{desc_key(j), gs_task_graph_device(t)}].push_back(t);
}

void gs_exec_drop_graphs(void) {
  std::lock_guard<std::mutex> g(g_graph_mu);
  for (auto &kv : g_graph_cache)
    for (gs_task_graph *t : kv.second) gs_task_graph_destroy(t);
  g_graph_cache.clear();
}

int gs_exec_set_capture(int32_t on) {
  g_capture = on != 0;
  return GS_OK;
}

int gs_exec_set_sm_parts(int32_t parts) {
  if (parts < 0 || parts > 64) return err(GS_ERR_CONFIG, "sm parts must be 0..64");
  g_sm_parts = parts;
  return GS_OK;
}

int gs_exec_sm_parts_layout(int32_t cuda_device, int32_t parts, int32_t *sms_out, int32_t cap, int32_t *n_out) {
  GreenSet *set = nullptr;
  int rc = green_for(cuda_device, parts, &set);
  if (rc) return rc;
  if (n_out) *n_out = (int32_t)set->parts.size();
  for (int i = 0; i < (int)set->parts.size() && i < cap; ++i) sms_out[i] = set->parts[i].sms;
  return GS_OK;
}

int gs_exec_ledger_capacity(int32_t cuda_device, int64_t *bytes) {
  CUE(cudaSetDevice(cuda_device));
  size_t free_b = 0, total_b = 0;
  CUE(cudaMemGetInfo(&free_b, &total_b));
  // memory an earlier run left mapped in the pool is free for this run's
  // jobs: cudaMemGetInfo counts it as used
  cudaMemPool_t pool;
  CUE(cudaDeviceGetDefaultMemPool(&pool, cuda_device));
  uint64_t reserved = 0, used = 0;
  CUE(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  CUE(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  if (reserved > used) free_b += (size_t)(reserved - used);
  free_b += (size_t)arena_idle_bytes(cuda_device);  // the idle job arena is this run's to use
  uint64_t g_res = 0, g_used = 0;  // graph-memory pool (capture mode) kept after its graphs freed
  if (cudaDeviceGetGraphMemAttribute(cuda_device, cudaGraphMemAttrReservedMemCurrent, &g_res) == cudaSuccess &&
      cudaDeviceGetGraphMemAttribute(cuda_device, cudaGraphMemAttrUsedMemCurrent, &g_used) == cudaSuccess &&
      g_res > g_used)
    free_b += (size_t)(g_res - g_used);
  cudaGetLastError();
  *bytes = (int64_t)free_b - (int64_t)(6ll << 30);  // 6 GiB reserve (context, other allocators)
  return GS_OK;
}

int gs_job_run_solo(const gs_job_desc *job, int cuda_device, int mode, void *host_out, int64_t host_out_bytes,
                    gs_job_record *rec) {
  int rc = validate(*job);
  if (rc) return rc;
  CUE(cudaSetDevice(cuda_device));
  memset(rec, 0, sizeof(*rec));
  cudaStream_t st;
  CUE(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  int32_t *scalar;
  unsigned long long *hsum;
  CUE(cudaHostAlloc((void **)&scalar, 16, 0));
  CUE(cudaHostAlloc((void **)&hsum, 16, 0));
  std::atomic<int64_t> kc{0};
  const Staged *stg = nullptr;
  {
    std::lock_guard<std::mutex> g(g_stage_mu);
    stg = find_staged(*job, cuda_device);
  }
  bool oom = false;
  {
    gs_probe pr;
    if (gs_job_probe(job, &pr) == GS_OK) prepare_pool(cuda_device, pr.mem_bytes);
  }
  // an idle job arena on the device (kept by an earlier run) holds most of
  // its memory: a solo run allocates from it
  gsa::Arena *ar = nullptr;
  bool drop = false;
  {
    gs_probe pr;
    const int64_t need = gs_job_probe(job, &pr) == GS_OK ? pr.mem_bytes : INT64_MAX;
    std::lock_guard<std::mutex> g(g_arena_mu);
    auto it = g_arenas.find(cuda_device);
    if (it != g_arenas.end()) {
      if (it->second->size() >= need && it->second->reset(it->second->size())) ar = it->second;
      else drop = true;  // too small for this job: give its memory to the pool
    }
  }
  if (drop) arena_drop_idle(cuda_device);
  const auto t0 = Clock::now();
  rc = run_job(*job, stg, mode, st, *rec, &oom, host_out, host_out_bytes, scalar, &kc, hsum, cuda_device, ar, false);
  rec->end_ms = ms_since(t0);
  rec->device = cuda_device;
  rec->state = oom ? 1 : 0;
  cudaFreeHost(scalar);
  cudaFreeHost(hsum);
  cudaStreamDestroy(st);
  return rc;
}

int gs_exec_run(const gs_job_desc *jobs, int32_t n_jobs, int32_t policy, int32_t cg_ratio,
                const int32_t *cuda_devices, int32_t n_devices, int32_t workers, int32_t mode, int64_t ledger_bytes,
                gs_job_record *records, gs_exec_stats *stats) {
  return gs_exec_run_arrivals(jobs, n_jobs, nullptr, policy, cg_ratio, cuda_devices, n_devices, workers, mode,
                              ledger_bytes, records, stats);
}

int gs_exec_run_arrivals(const gs_job_desc *jobs, int32_t n_jobs, const double *arrival_ms, int32_t policy,
                         int32_t cg_ratio, const int32_t *cuda_devices, int32_t n_devices, int32_t workers,
                         int32_t mode, int64_t ledger_bytes, gs_job_record *records, gs_exec_stats *stats) {
  if (n_jobs <= 0) return GS_OK;
  const auto t_call = Clock::now();
  auto phase = [&](const char *what) {
    if (g_alloc_log) fprintf(stderr, "[gs exec] %8.1f ms %s\n", ms_since(t_call), what);
  };
  if (n_devices < 1 || n_devices > GS_MAX_DEVICES) return err(GS_ERR_CONFIG, "1..32 devices");
  if (workers < 1) return err(GS_ERR_CONFIG, "need at least one worker");
  for (int i = 0; i < n_jobs; ++i) {
    int rc = validate(jobs[i]);
    if (rc) return rc;
  }
  const bool task_level = policy == GS_POLICY_MGB_SM || policy == GS_POLICY_MGB_WARPS;
  const bool capture = g_capture.load();
  // decision engine on the first device; one ledger per device
  gs_engine *eng = nullptr;
  int rc = gs_engine_open(cuda_devices[0], &eng);
  if (rc) return err(rc, gs_last_error());
  phase("engine open");
  std::vector<gs_device *> ledgers(n_devices, nullptr);
  std::vector<gsa::Arena *> arenas(n_devices, nullptr);
  std::vector<GreenSet *> greens(n_devices, nullptr);
  const int sm_parts = g_sm_parts.load();
  if (sm_parts > 1)
    for (int d = 0; d < n_devices; ++d) {
      int rc2 = green_for(cuda_devices[d], sm_parts, &greens[d]);
      if (rc2) return rc2;
    }
  std::vector<gs_spec> specs(n_devices);
  for (int d = 0; d < n_devices; ++d) {
    const cudaDeviceProp &prop = gscache::device_props(cuda_devices[d]);
    CUE(cudaSetDevice(cuda_devices[d]));
    // keep the pool's memory (no trimming between jobs)
    cudaMemPool_t pool;
    CUE(cudaDeviceGetDefaultMemPool(&pool, cuda_devices[d]));
    uint64_t thr = UINT64_MAX;
    CUE(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    gs_spec spec;
    spec.sm_count = prop.multiProcessorCount;
    if (ledger_bytes > 0) {
      spec.mem_bytes = ledger_bytes;
    } else {  // (cudaMemGetInfo takes 5-40 ms now and then: callers that run
              // many steps pass gs_exec_ledger_capacity's value instead)
      int64_t cap = 0;
      rc = gs_exec_ledger_capacity(cuda_devices[d], &cap);
      if (rc) return rc;
      spec.mem_bytes = cap;
    }
    spec.max_warps_per_sm = prop.maxThreadsPerMultiProcessor / 32;
    spec.max_tbs_per_sm = prop.maxBlocksPerMultiProcessor;
    spec.regs_per_sm = prop.regsPerMultiprocessor;
    spec.smem_per_sm_bytes = (int64_t)prop.sharedMemPerMultiprocessor;
    rc = gs_device_create(eng, &spec, d, &ledgers[d]);
    if (rc) return err(rc, gs_last_error());
    specs[d] = spec;
    phase("ledger created");
    // at most `workers` jobs hold memory at once: the pool (or the arena)
    // needs the sum of the largest `workers` footprints, capped by the ledger
    std::vector<int64_t> foot;
    foot.reserve(n_jobs);
    for (int i = 0; i < n_jobs; ++i) {
      gs_probe pr;
      if (gs_job_probe(&jobs[i], &pr) == GS_OK) foot.push_back(pr.mem_bytes);
    }
    const size_t k = std::min(foot.size(), (size_t)std::max(workers, 1));
    std::partial_sort(foot.begin(), foot.begin() + k, foot.end(), std::greater<int64_t>());
    int64_t need = 0;
    for (size_t i = 0; i < k; ++i) need += foot[i];
    if (capture) {
      arena_drop_idle(cuda_devices[d]);  // task graphs allocate from the graph-memory pool
    } else if (arena_enabled()) {
      // the slab: what the run can hold at once, capped by the ledger (a
      // policy without a memory check then OOMs exactly when its
      // co-running jobs exceed the ledger capacity)
      arenas[d] = arena_for(cuda_devices[d], std::min<int64_t>(need, spec.mem_bytes));
      if (arenas[d]) continue;  // jobs allocate from the arena: no pool growth
    }
    // ... unless that is most of the device: one chunk that large fragments
    // under jobs of 7-42 GB (cfg 2) and, with no physical memory left to
    // grow into, an allocation that does not fit a hole stalls; such runs
    // let the pool grow and trim per allocation instead
    if (need <= spec.mem_bytes / 2) prepare_pool(cuda_devices[d], need);
  }
  gs_sched *sched = nullptr;
  phase("pool ready");
  rc = gs_sched_create(eng, ledgers.data(), n_devices, policy, cg_ratio, 1, &sched);
  if (rc) return err(rc, gs_last_error());
  phase("sched created");
  rc = gs_engine_reserve_handles(eng, n_jobs + 1);
  if (rc) return err(rc, gs_last_error());
  // Placement calls: the single decision authority serializes every
  // worker's calls under its lock.  On one GPU they go as one decision
  // launch each (~40 us; the resident ring measured the same makespan).  A
  // fleet has N x workers callers behind that lock, so runs over several GPUs
  // serve them from the resident decision warp over the host-mapped command
  // ring (~7 us per decision, tools/ring_bench.cpp).  GS_RING=0 / 1 forces
  // either; never under ncu, which serializes kernels.
  const char *ring_env = getenv("GS_RING");
  const bool use_ring = ring_env ? ring_env[0] == '1' : n_devices > 1;
  if (use_ring) {
    rc = gs_sched_ring_start(sched, n_jobs + 1, n_jobs + 1, n_jobs + 1);
    if (rc) return err(rc, gs_last_error());
  }

  memset(records, 0, sizeof(gs_job_record) * n_jobs);
  // the placement log (caller holds mu while appending: the log order is
  // the decision authority's linearization order)
  std::vector<gs_exec_event> log;
  log.reserve((size_t)n_jobs * 4 + 16);
  auto log_ev = [&](int32_t kind, int32_t handle, int32_t device, int32_t outcome, int64_t freed,
                    const gs_probe *pr) {
    gs_exec_event e;
    memset(&e, 0, sizeof e);
    e.kind = kind;
    e.handle = handle;
    e.device = device;
    e.outcome = outcome;
    e.freed = freed;
    e.t_ms = 0;
    if (pr) e.probe = *pr;
    log.push_back(e);
  };
  std::vector<int> admitted(n_jobs, -1);
  std::vector<gs_decision> drain(n_jobs + 1);
  std::mutex mu;
  std::condition_variable cv;
  std::atomic<int> next{0};
  std::atomic<int64_t> kernels{0};
  double decision_ms = 0;
  int first_err = GS_OK;
  std::string first_msg;
  // e2e outputs land in the staged jobs' pinned buffers; a per-worker
  // fallback buffer is allocated only for jobs that were not staged
  int64_t out_cap = 0;
  if (mode == GS_MODE_E2E) {
    std::lock_guard<std::mutex> g(g_stage_mu);
    for (int i = 0; i < n_jobs; ++i)
      if (!find_staged(jobs[i], -1)) out_cap = std::max(out_cap, max_out_bytes(jobs + i, 1));
  }
  const auto t0 = Clock::now();

  auto admit_drained = [&](int32_t tried, int32_t adm) {  // caller holds mu
    for (int k = 0; k < tried; ++k) {
      log_ev(GS_EV_DRAIN, drain[k].handle, drain[k].device, drain[k].outcome, 0, nullptr);
      log.back().t_ms = ms_since(t0);
      log.back().free_mem_after = drain[k].free_mem_after;
      log.back().in_use_warps_after = drain[k].in_use_warps_after;
      if (drain[k].outcome == GS_ASSIGN) admitted[drain[k].handle] = drain[k].device;
    }
    if (adm) cv.notify_all();
  };
  auto redrive = [&]() {  // caller holds mu
    int32_t tried = 0, adm = 0;
    const auto a = Clock::now();
    int r = gs_on_release(sched, drain.data(), (int32_t)drain.size(), &tried, &adm);
    decision_ms += ms_since(a);
    if (r < 0) return r;
    admit_drained(tried, adm);
    return GS_OK;
  };

  auto worker = [&](int wid) {
    // two streams per device: latency-chain jobs (bfs, lud, needle: many
    // dependent launches or a wavefront) run at high stream priority so their
    // next kernel is not queued behind co-located streaming kernels; the
    // bandwidth-bound kinds at the default.  (A three-class shortest-job-first
    // variant starved the long streaming jobs: cfg 3 turnaround 907 ms vs
    // 106 ms, cfg 1 makespan 324-414 ms vs 285 ms.)
    // streams and pinned scratch come from process-lifetime caches
    // (gs_cache.h): creating / freeing them per run stalled whole runs
    std::vector<cudaStream_t> streams(n_devices, nullptr), hi_streams(n_devices, nullptr);
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    for (int d = 0; d < n_devices; ++d) {
      cudaSetDevice(cuda_devices[d]);
      gscache::stream_get(&streams[d], 0);
      gscache::stream_get(&hi_streams[d], prio_hi);
    }
    void *host_out = nullptr;
    if (out_cap) gscache::host_alloc(&host_out, out_cap);
    int32_t *scalar = nullptr;
    unsigned long long *hsum = nullptr;
    gscache::host_alloc((void **)&scalar, 16);
    gscache::host_alloc((void **)&hsum, 16);
    for (;;) {
      const int j = next.fetch_add(1);
      if (j >= n_jobs) break;
      gs_job_record &rec = records[j];
      if (arrival_ms) {  // the job has not arrived yet: this worker waits for it
        rec.arrival_ms = arrival_ms[j];
        const double now = ms_since(t0);
        if (arrival_ms[j] > now)
          std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(arrival_ms[j] - now));
      }
      rec.pull_ms = ms_since(t0);
      gs_probe pr;
      // capture mode: the job's host code is recorded into a task graph
      // (nothing runs, nothing is allocated) and the probe is computed from
      // the recorded launches and allocations — kernel_launch_prepare
      gs_task_graph *tg = nullptr;
      if (capture && jobs[j].kind != GS_JOB_BFS) {
        const int cr = graph_take(jobs[j], cuda_devices[0], &tg);
        if (cr) {
          std::lock_guard<std::mutex> lk(mu);
          if (!first_err) {
            first_err = cr;
            first_msg = t_err;
          }
          rec.state = 2;
          continue;
        }
        gs_task_graph_probe(tg, &pr, nullptr, nullptr);
      } else {
        gs_job_probe(&jobs[j], &pr);
      }
      rec.mem_bytes = pr.mem_bytes;
      pr.handle = j;
      pr.job = j;
      if (task_level) {
        pr.level = GS_PROBE_FRESH;
      } else {  // job-granular claim with zero resources (sim_engine.py:295-302)
        gs_probe z;
        memset(&z, 0, sizeof z);
        z.handle = j;
        z.job = j;
        z.level = GS_PROBE_JOB;
        pr = z;
      }
      int dev = -1;
      {
        std::unique_lock<std::mutex> lk(mu);
        gs_decision dec;
        memset(&dec, 0, sizeof dec);
        const auto a = Clock::now();
        int r = gs_submit(sched, &pr, &dec);
        decision_ms += ms_since(a);
        log_ev(GS_EV_SUBMIT, j, r < 0 ? -1 : dec.device, r < 0 ? r : dec.outcome, 0, &pr);
        log.back().t_ms = ms_since(t0);
        log.back().free_mem_after = dec.free_mem_after;
        log.back().in_use_warps_after = dec.in_use_warps_after;
        if (r < 0) {
          if (!first_err) {
            first_err = r;
            first_msg = gs_last_error();
          }
          rec.state = 2;
          graph_give(jobs[j], tg);
          continue;
        }
        if (dec.outcome == GS_REJECTED) {
          rec.state = 2;
          rec.end_ms = ms_since(t0);
          graph_give(jobs[j], tg);
          continue;
        }
        if (dec.outcome == GS_ASSIGN) {
          dev = dec.device;
        } else {
          cv.wait(lk, [&] { return admitted[j] >= 0; });
          dev = admitted[j];
        }
      }
      rec.admit_ms = ms_since(t0);
      rec.wait_ms = rec.admit_ms - rec.pull_ms;
      rec.device = dev;
      cudaSetDevice(cuda_devices[dev]);
      const Staged *stg = nullptr;
      {
        std::lock_guard<std::mutex> g(g_stage_mu);
        stg = find_staged(jobs[j], cuda_devices[dev]);
      }
      bool oom = false;
      const bool chain = jobs[j].kind == GS_JOB_BFS || jobs[j].kind == GS_JOB_LUD || jobs[j].kind == GS_JOB_NEEDLE;
      cudaStream_t js = chain ? hi_streams[dev] : streams[dev];
      int part = -1;
      if (greens[dev]) {  // an SM partition of the device for the job's whole run
        part = greens[dev]->acquire();
        const GreenPart &gp = greens[dev]->parts[part];
        js = chain ? gp.hi : gp.lo;
        set_job_sms(gp.sms);
        rec.sm_share = gp.sms;
      }
      int r = GS_OK;
      if (tg) {
        // replay: the recorded queue materialized on the chosen device (a
        // graph is bound to the device it was recorded on: re-record there)
        if (gs_task_graph_device(tg) != cuda_devices[dev]) {
          graph_give(jobs[j], tg);
          tg = nullptr;
          r = graph_take(jobs[j], cuda_devices[dev], &tg);
        }
        float gms = 0;
        uint64_t cs = 0;
        if (!r) r = gs_task_graph_run(tg, js, &cs, &gms);
        if (!r) {
          rec.compute_ms = gms;
          rec.checksum = cs;
          int32_t nk = 0;
          gs_task_graph_probe(tg, nullptr, &nk, nullptr);
          rec.n_kernels = nk;
          kernels.fetch_add(nk);
        }
        if (!r) graph_give(jobs[j], tg);
        else gs_task_graph_destroy(tg);
        tg = nullptr;
      } else {
        // memory-safe policies wait out arena fragmentation; sa / cg OOM
        r = run_job(jobs[j], stg, mode, js, rec, &oom, host_out, out_cap, scalar, &kernels, hsum,
                    cuda_devices[dev], arenas[dev], task_level);
      }
      rec.end_ms = ms_since(t0);
      rec.state = oom ? 1 : 0;
      if (part >= 0) {
        set_job_sms(0);
        greens[dev]->release(part);
      }
      std::unique_lock<std::mutex> lk(mu);
      if (r < 0 && !first_err) {
        first_err = r;
        first_msg = t_err;
      }
      if (task_level) {
        // release_task + the FIFO re-drive in one decision launch
        int32_t tried = 0, adm = 0;
        int64_t freed = 0;
        const auto a = Clock::now();
        const int rr = gs_release_redrive(sched, dev, j, &freed, drain.data(), (int32_t)drain.size(), &tried, &adm);
        decision_ms += ms_since(a);
        log_ev(GS_EV_RELEASE, j, dev, rr, freed, nullptr);
        log.back().t_ms = ms_since(t0);
        // the re-drive runs even when the release itself fails (unknown
        // task -> GS_ERR_CONTRACT after the drain): whatever it admitted
        // must still wake its workers, and the failure must surface
        if (tried > 0) admit_drained(tried, adm);
        if (rr < 0 && !first_err) {
          first_err = rr;
          first_msg = gs_last_error();
        }
      } else {
        const auto a = Clock::now();
        gs_job_ended(sched, j);
        decision_ms += ms_since(a);
        log_ev(GS_EV_JOB_ENDED, j, dev, GS_OK, 0, nullptr);
        log.back().t_ms = ms_since(t0);
        redrive();
      }
    }
    const auto tw = Clock::now();
    for (int d = 0; d < n_devices; ++d) {
      gscache::stream_put(streams[d], cuda_devices[d], 0);
      gscache::stream_put(hi_streams[d], cuda_devices[d], prio_hi);
    }
    if (host_out) gscache::host_free(host_out, out_cap);
    gscache::host_free(scalar, 16);
    gscache::host_free(hsum, 16);
    if (g_alloc_log) fprintf(stderr, "[gs exec] worker %d teardown %.1f ms (at %.1f)\n", wid, ms_since(tw), ms_since(t_call));
  };
  phase("setup done");
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w) pool.emplace_back(worker, w);
  for (auto &t : pool) t.join();
  phase("workers joined");
  gs_sched_ring_stop(sched);  // retire the resident decision kernel before draining the devices
  for (int d = 0; d < n_devices; ++d) {
    cudaSetDevice(cuda_devices[d]);
    cudaDeviceSynchronize();
  }
  phase("devices drained");
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    for (int i = 0; i < n_jobs; ++i) {
      stats->makespan_ms = std::max(stats->makespan_ms, records[i].end_ms);
      if (records[i].state == 0) stats->completed++;
      else stats->crashed++;
      if (records[i].state == 1) stats->oom++;
      if (records[i].state == 2) stats->rejected++;
    }
    stats->kernel_launches = kernels.load();
    stats->decision_launches = gs_engine_decisions(eng);
    stats->decision_ms = decision_ms;
  }
  gs_sched_ring_stop(sched);
  gs_sched_destroy(sched);
  phase("sched destroyed");
  {
    std::lock_guard<std::mutex> g(g_log_mu);
    g_log.swap(log);
    g_log_specs = specs;
    g_log_policy = policy;
    g_log_cg_ratio = cg_ratio;
  }
  for (gs_device *d : ledgers) gs_device_destroy(d);
  phase("ledgers destroyed");
  gs_engine_close(eng);
  phase("engine closed");
  if (first_err) return err(first_err, first_msg);
  return GS_OK;
}

}  // extern "C"
