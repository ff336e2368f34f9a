// gs_work_internal.h — internal interfaces between the job runners
// (gs_work.cu), the tcgen05 GEMM layers (gs_gemm.cu) and the executor
// (gs_exec.cu).  Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gs_work.h"

namespace gsw {

enum Role { IN = 0, INOUT = 1, OUT = 2, SCR = 3 };

struct Buf {
  int64_t bytes;
  int role;
};

struct Shape {
  const void *fn;
  int grid, block;
};

std::vector<Shape> gemm_launches(const gs_job_desc &j);

extern thread_local std::string t_err;
int err(int code, const std::string &m);

std::vector<Buf> job_buffers(const gs_job_desc &j);
int validate(const gs_job_desc &j);
int generate_inputs(const gs_job_desc &j, const std::vector<void *> &dst, cudaStream_t st);
int run_kernels(const gs_job_desc &j, std::vector<void *> &buf, cudaStream_t st, int *out_idx, int64_t *kernels,
                int32_t *host_scalar);
int digest(const void *p, int64_t bytes, unsigned long long *dsum, cudaStream_t st);
int64_t round_granule(int64_t b);

// Darknet-style layer stacks on tcgen05 (gs_gemm.cu)
std::vector<Buf> gemm_buffers(const gs_job_desc &j);
int gemm_validate(const gs_job_desc &j);
int gemm_generate(const gs_job_desc &j, const std::vector<void *> &dst, cudaStream_t st);
int gemm_run(const gs_job_desc &j, std::vector<void *> &buf, cudaStream_t st, int *out_idx, int64_t *launches);

}  // namespace gsw
