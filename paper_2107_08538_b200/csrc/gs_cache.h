// gs_cache.h — process-lifetime caches for the runtime's small buffers and
// streams.  Pinned host allocations, cudaMalloc / cudaFree and stream
// creation take driver locks and may synchronize the device; measured on
// B200, re-creating the engine, ledgers and worker scratch around every
// executor run stalled runs for 10-390 ms (profiles/exec_setup_stall_r01.txt).
// Blocks are kept by (device, bytes) and handed back zero-filled by the
// caller; streams by (device, priority).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace gscache {

// pinned, mapped + portable host memory (cudaHostAllocMapped | Portable)
cudaError_t host_alloc(void **p, size_t bytes);
void host_free(void *p, size_t bytes);
// device memory on the current device; a cudaMalloc that runs out of
// memory calls the OOM hook (the executor frees its idle job arena) and
// retries once
cudaError_t dev_alloc(void **p, size_t bytes);
void set_oom_hook(void (*hook)(int device));
void dev_free(void *p, size_t bytes, int device);
// cudaGetDeviceProperties, queried once per device
const cudaDeviceProp &device_props(int device);
// non-blocking stream on the current device at `prio` (0 = default)
cudaError_t stream_get(cudaStream_t *s, int prio);
void stream_put(cudaStream_t s, int device, int prio);

}  // namespace gscache
