// gs_work_internal.h — internal interfaces between the job runners
// (gs_work.cu), the tcgen05 GEMM layers (gs_gemm.cu) and the executor
// (gs_exec.cu).  Not part of the C-ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gs_work.h"

namespace gsw {

// SMs the current job's kernels may use (grids are sized from it): the
// current device's SM count, or the job's green-context partition when the
// executor runs it on one (set_job_sms, per worker thread; 0 = the device)
int sm_count();
void set_job_sms(int n);

// IN staged input, INOUT staged input that is also an output, OUT output,
// SCR zeroed scratch, WRK uninitialized workspace (fully overwritten), PING
// uninitialized ping-pong buffer that may end up holding the output
enum Role { IN = 0, INOUT = 1, OUT = 2, SCR = 3, WRK = 4, PING = 5 };

struct Buf {
  int64_t bytes;
  int role;
};

struct Shape {
  const void *fn;
  int grid, block;
  int dsmem = 0;  // dynamic shared memory per block
};

std::vector<Shape> gemm_launches(const gs_job_desc &j);

extern thread_local std::string t_err;
int err(int code, const std::string &m);

std::vector<Buf> job_buffers(const gs_job_desc &j);
int validate(const gs_job_desc &j);
int generate_inputs(const gs_job_desc &j, const std::vector<void *> &dst, cudaStream_t st);
// tk: the job's two tile-ticket counters (zeroed before the first kernel).
// src: per buffer, a read-only copy of an INOUT buffer's input that the
// job's first kernel reads instead of the (then uninitialised) buffer, or
// null — only where reads_source() says the kernels support it.
// digested: non-null lets the job's last kernel accumulate the output digest
// (C * word sum) into tk's control word 0; *digested then says whether it did
// (the caller skips digest() and adds digest_tail to the read-back).
int run_kernels(const gs_job_desc &j, std::vector<void *> &buf, cudaStream_t st, int *out_idx, int64_t *kernels,
                int32_t *host_scalar, unsigned *tk, const void *const *src = nullptr, bool *digested = nullptr);
unsigned long long digest_tail(int64_t bytes);
bool reads_source(const gs_job_desc &j, size_t buf);
bool reads_source_host(const gs_job_desc &j, size_t buf);
int64_t source_host_bytes(const gs_job_desc &j, size_t buf);
bool derived_input(const gs_job_desc &j, size_t buf);
int derive_inputs(const gs_job_desc &j, std::vector<void *> &buf, cudaStream_t st);
int digest(const void *p, int64_t bytes, unsigned long long *dsum, cudaStream_t st);
int64_t round_granule(int64_t b);

// Darknet-style layer stacks on tcgen05 (gs_gemm.cu)
std::vector<Buf> gemm_buffers(const gs_job_desc &j);
int gemm_validate(const gs_job_desc &j);
int gemm_generate(const gs_job_desc &j, const std::vector<void *> &dst, cudaStream_t st);
int gemm_run(const gs_job_desc &j, std::vector<void *> &buf, cudaStream_t st, int *out_idx, int64_t *launches,
             unsigned *tk);
int gemm_pick_bn(int m, int n);
int conv_gemm_bf16(const void *in, int nb, int h, int w, int pitch, int log2c, int oh, int ow, int k, int stride,
                   int pad, const void *B, int64_t ldb, const float *bias, void *out, int64_t ldo, int cout,
                   int out_f32, int act, int max_ctas, cudaStream_t st, const void *res, int64_t ldr, unsigned *tk);
const void *conv_kernel_fn(int bn);
int conv_block_threads();
int make_tmap_f32(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int box_cols, int box_rows);
size_t gemm_smem_for(int bn);
int gemm_block_threads();
const void *gemm_kernel_fn(int bn);
int gemm_bf16(const void *A, int64_t lda, const void *B, int64_t ldb, const float *bias, void *out, int64_t ldo,
              int m, int n, int k, int out_f32, int act, int max_ctas, cudaStream_t st, const void *res = nullptr,
              int64_t ldr = 0, unsigned *tk = nullptr);

}  // namespace gsw
