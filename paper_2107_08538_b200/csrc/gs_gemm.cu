// gs_gemm.cu — Darknet-style layer stacks on tcgen05 (placeholder until the
// tcgen05 GEMM lands; GEMM jobs are refused with a config error).
#include "gs_work_internal.h"

namespace gsw {

std::vector<Buf> gemm_buffers(const gs_job_desc &) { return {}; }
int gemm_validate(const gs_job_desc &) { return err(GS_ERR_CONFIG, "gemm jobs are not available in this build"); }
std::vector<Shape> gemm_launches(const gs_job_desc &) { return {}; }
int gemm_generate(const gs_job_desc &, const std::vector<void *> &, cudaStream_t) { return GS_ERR_CONFIG; }
int gemm_run(const gs_job_desc &, std::vector<void *> &, cudaStream_t, int *, int64_t *) { return GS_ERR_CONFIG; }

}  // namespace gsw
