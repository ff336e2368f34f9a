/*
 * gs_work.h — workload jobs (Rodinia-class + Darknet-style) and the
 * executor that runs them under the placement engine.
 *
 * The reference models every job as a catalog entry with a footprint and a
 * duration (gpushare/data/catalog.json, sim_engine.py:191-218 `_Pool`);
 * there is no kernel code to bind.  These entry points are the B200-native
 * replacement of that simulated execution: each job
 * allocates its buffers on the device the engine chose, runs hand-written
 * sm_100a kernels on its own stream, and releases its ledger entry.
 *
 * Synthetic inputs come from a counter-based hash (gs_hash64) shared with
 * the CPU oracle (oracle/kernels_cpu.c), so both sides see identical data.
 */
#ifndef GS_WORK_H
#define GS_WORK_H

#include <stdint.h>

#include "gs.h"

#ifdef __cplusplus
extern "C" {
#endif

/* job kinds */
#define GS_JOB_BFS 0
#define GS_JOB_HOTSPOT 1
#define GS_JOB_SRAD 2
#define GS_JOB_KMEANS 3
#define GS_JOB_BACKPROP 4
#define GS_JOB_NEEDLE 5
#define GS_JOB_LUD 6
#define GS_JOB_YOLO 7      /* Darknet YOLOv3-tiny inference (bf16 im2col + tcgen05 GEMM) */
#define GS_JOB_RESNET 8    /* ResNet-50 inference (same layers: im2col + tcgen05 GEMM, fused shortcut) */
#define GS_JOB_KINDS 9

/* executor modes */
#define GS_MODE_DEVICE 0   /* inputs pre-staged in HBM, D2D into the job's buffers */
#define GS_MODE_E2E 1      /* inputs in pinned host memory: H2D in, D2H of results */

typedef struct gs_job_desc {
    int32_t kind;
    int32_t iters;        /* iterations (hotspot/srad/kmeans/backprop), forward passes (yolo/resnet) */
    int64_t n;            /* problem size: nodes / grid edge / points / inputs / matrix edge / image edge */
    int64_t m;            /* secondary size: features (kmeans), hidden (backprop), batch (yolo/resnet) */
    uint64_t seed;
} gs_job_desc;

/* Per-job outcome (SimReport.jobs rows, sim_engine.py:597-609, on a wall clock). */
typedef struct gs_job_record {
    int32_t state;        /* 0 done, 1 crashed (oom), 2 rejected */
    int32_t device;
    double arrival_ms;    /* job arrival (0 for a batch, sim_engine.py:607) */
    double pull_ms;       /* worker picked the job (>= arrival) */
    double admit_ms;      /* placement decided ASSIGN */
    double end_ms;
    double wait_ms;       /* admit - pull */
    double compute_ms;    /* Σ device time of the job's kernels (CUDA events) */
    int64_t mem_bytes;    /* probe footprint */
    int64_t h2d_bytes, d2h_bytes;
    uint64_t checksum;    /* order-independent digest of the job's outputs */
    int32_t n_kernels;
    int32_t sm_share;     /* SMs of the green-context partition the job ran on (0 = whole device) */
    /* where a job's wall time goes (diagnostics): host time from admission
     * to the inputs' launches returning, device time from the job's first
     * queued op to its first kernel (input fill / generation, including
     * waiting for an SM), and from its last kernel to the output digest's
     * readback */
    double setup_ms, gen_ms, tail_ms;
} gs_job_record;

typedef struct gs_exec_stats {
    double makespan_ms;
    int32_t completed, crashed, oom, rejected;
    int64_t kernel_launches;   /* workload kernels launched */
    int64_t decision_launches; /* placement-kernel launches */
    double decision_ms;        /* host wall time spent in placement calls */
} gs_exec_stats;

/* ---- probe capture (replaces the reference's trace-level
 * compute_resource_request, gs/task_builder.py:258-290, for real CUDA host
 * code: a launch wrapper or interceptor records each kernel launch of a task
 * and its buffers, and the probe follows the reference's aggregation) ---- */
typedef struct gs_launch_desc {
    int32_t thread_blocks;
    int32_t threads_per_block;
    int32_t regs_per_thread;
    int32_t smem_per_block;   /* static + dynamic bytes */
    double est_duration_ms;
} gs_launch_desc;
/* Descriptor of launching `fn` (a __global__ function's host stub, as
 * cudaLaunchKernel takes it) with grid x block and `dyn_smem` dynamic shared
 * memory: registers and static shared memory from cudaFuncGetAttributes
 * (queried once per kernel). */
int gs_launch_desc_of(const void *fn, int32_t grid, int32_t block, int32_t dyn_smem, gs_launch_desc *out);
/* compute_resource_request: mem = sum of the task's distinct buffers + the
 * heap limit, counted once; the widest launch is the FIRST maximum of
 * tbs * ceil(threads / 32) and gives the shape; regs / smem are maxima over
 * all launches; the duration estimate is the sum.  Pure host arithmetic (no
 * GPU needed).  GS_ERR_CONFIG for no launches or a byte overflow. */
int gs_request_from_launches(const gs_launch_desc *launches, int32_t n, const int64_t *buffer_bytes, int32_t nbuf,
                             int64_t heap_limit_bytes, gs_probe *out);
/* Probe of a catalog job: its kernels' real launch shapes through
 * gs_launch_desc_of, its buffers rounded to the executor's 2 MiB allocation
 * granule, plus the 8 MiB device heap the reference counts per task
 * (task_builder.py:264-268). */
int gs_job_probe(const gs_job_desc *job, gs_probe *out);
/* Bytes a job moves host -> device / device -> host in e2e mode: its
 * inputs less what it rebuilds on the device (bfs's transposed CSR) and,
 * for needle's score matrix, only the boundary (row 0 and the pad + column
 * 0 lead of every row); its outputs. */
int gs_job_io_bytes(const gs_job_desc *job, int64_t *in_bytes, int64_t *out_bytes);

/* Run one job to completion on `cuda_device` (isolated), for tests and the
 * solo baseline: writes outputs to host buffers when non-NULL. */
int gs_job_run_solo(const gs_job_desc *job, int cuda_device, int mode, void *host_out, int64_t host_out_bytes,
                    gs_job_record *rec);

/* Executor: run `n_jobs` jobs through `workers` worker threads on
 * `n_devices` CUDA devices under `policy` (GS_POLICY_*), like
 * metrics.run_workload -> run_sim (metrics.py:101-119, sim_engine.py:632).
 * ledger_bytes: per-device ledger capacity (0 = free HBM - reserve). */
int gs_exec_run(const gs_job_desc *jobs, int32_t n_jobs, int32_t policy, int32_t cg_ratio,
                const int32_t *cuda_devices, int32_t n_devices, int32_t workers, int32_t mode,
                int64_t ledger_bytes, gs_job_record *records, gs_exec_stats *stats);
/* Same, with per-job arrival times (ms after the run starts, non-decreasing;
 * NULL = batch arrival): a worker that pulls a job before it arrives waits
 * for it (BASELINE cfg 3's Poisson stream; the reference has batch arrival
 * only). */
/* The ledger capacity a run on `cuda_device` gets when ledger_bytes <= 0:
 * free HBM + memory the device pool holds unused - 6 GiB reserve.  Callers
 * timing many runs query it once (it calls cudaMemGetInfo, a slow driver
 * query) and pass it as ledger_bytes. */
int gs_exec_ledger_capacity(int32_t cuda_device, int64_t *bytes);
int gs_exec_run_arrivals(const gs_job_desc *jobs, int32_t n_jobs, const double *arrival_ms, int32_t policy,
                         int32_t cg_ratio, const int32_t *cuda_devices, int32_t n_devices, int32_t workers,
                         int32_t mode, int64_t ledger_bytes, gs_job_record *records, gs_exec_stats *stats);

/* Darknet layer GEMM on tcgen05 (csrc/gs_gemm.cu): D = act(A . B^T + bias)
 * with A [m x k] and B [n x k] bf16 row-major (K contiguous, k % 8 == 0),
 * bias fp32 [n] or NULL, D [m x n] bf16 or fp32 (out_f32) with row pitch ldo,
 * act 0 linear / 1 leaky-ReLU 0.1.  Device pointers; stream may be NULL. */
int gs_gemm_bf16(const void *A, int64_t lda, const void *B, int64_t ldb, const float *bias, void *out,
                 int64_t ldo, int32_t m, int32_t n, int32_t k, int32_t out_f32, int32_t act, void *stream);

/* Prepare (generate) the inputs of a job list ahead of gs_exec_run so the
 * timed region starts with inputs resident (device) or pinned (e2e). */
int gs_exec_stage(const gs_job_desc *jobs, int32_t n_jobs, const int32_t *cuda_devices, int32_t n_devices,
                  int32_t mode);
void gs_exec_unstage(void);

/* SM shares of co-located jobs (the paper's MPS
 * partitions): parts > 1 splits every device's SMs into `parts` disjoint
 * green-context partitions (cuDevSmResourceSplitByCount in 8-SM groups,
 * cuGreenCtxCreate); a job placed on a device runs on a free partition's
 * streams with its grids sized to the partition's SM count, waiting for
 * one when all are taken.  parts <= 1 (the default) runs every job on
 * ordinary streams over the whole device.  Applies to later gs_exec_run*
 * calls; *sms_out (optional) gets the partitions' SM counts on device 0
 * once they are built by a run. */
int gs_exec_set_sm_parts(int32_t parts);
/* ---- probe capture and lazy replay (csrc/gs_capture.cu) ----------------
 * A task's host code runs once against a stream in CAPTURE mode: its
 * stream-ordered allocations get addresses but no memory (the reference's
 * pseudo addresses, lazy_runtime.py:56-67), its copies / memsets / kernel
 * launches are recorded, not run (the queued ops).  Ending the capture
 * computes the task's probe from what was recorded — every kernel node's
 * grid, block and dynamic smem (+ registers / static smem from the
 * function's attributes), every allocation node's bytes on the 2 MiB
 * granule, aggregated by task_builder.py:258-290 (kernel_launch_prepare,
 * lazy_runtime.py:103-168).  Running the graph on the chosen device
 * materializes the queue there once, in recorded order (replay,
 * lazy_runtime.py:181-195).  A graph is bound to the device it was
 * recorded on. */
typedef struct gs_task_graph gs_task_graph;
int gs_capture_begin(int32_t cuda_device, void **stream);
int gs_capture_malloc(void *stream, int64_t bytes, void **ptr);   /* lazy_alloc */
int gs_capture_free(void *stream, void *ptr);
int gs_capture_end(void *stream, int64_t heap_limit_bytes, gs_task_graph **out);  /* heap <= 0: 8 MiB */
int gs_task_graph_probe(const gs_task_graph *g, gs_probe *out, int32_t *n_kernels, int32_t *n_allocs);
int gs_task_graph_run(gs_task_graph *g, void *stream, uint64_t *checksum, float *ms);
int gs_task_graph_device(const gs_task_graph *g);  /* the CUDA device it was recorded on */
void gs_task_graph_destroy(gs_task_graph *g);
/* A staged catalog job's whole device-side life (allocations, input copies,
 * kernels, output digest + read-back, frees) as a task graph.  bfs (its
 * level loop reads a count on the host) is not capturable. */
int gs_job_capture(const gs_job_desc *job, int32_t cuda_device, gs_task_graph **out);
/* Executor capture mode (on != 0): every capturable job's probe comes from
 * its recorded task graph and the job runs by replaying the graph on the
 * device it was placed on (bfs runs directly). */
int gs_exec_set_capture(int32_t on);
/* Free the task graphs capture mode recorded and keeps per (job, device)
 * (gs_exec_unstage does this too: the graphs read the staged inputs). */
void gs_exec_drop_graphs(void);

/* Give back the executor's idle per-device job arenas (the slab a run
 * allocates once, sized to its ledger capacity, and keeps for later runs;
 * csrc/gs_arena.h).  Later runs allocate a new one. */
void gs_exec_release_memory(void);
int gs_exec_sm_parts_layout(int32_t cuda_device, int32_t parts, int32_t *sms_out, int32_t cap, int32_t *n_out);

/* Measured FP32 FMA throughput of `cuda_device` in TFLOP/s (8 independent
 * FFMA chains per thread, 8 x 256-thread blocks per SM): the roofline
 * denominator of the FP32 CUDA-core kernels (lud). */
int gs_measure_fp32_peak(int32_t cuda_device, double *tflops);

/* Self-test of srad's branch-free IEEE division (gs_kernels.cuh,
 * srad_coeff_fast): n random operand pairs across and beyond its proven
 * domain against __fdiv_rn, and n random coefficient windows against
 * srad_coeff_one with ROI statistic q0sqr.  out4 = {division mismatches
 * inside the domain, in-domain pairs, coefficient mismatches where the fast
 * path claimed its proof, such windows}; both mismatch counts must be 0. */
int gs_selftest_division(int32_t cuda_device, int64_t n, uint64_t seed, float q0sqr, int64_t *out4);

/* ---- placement log of the most recent executor run ---------------------
 * Every call the run made into the decision engine, in the order the single
 * decision authority serialized them (the linearization SPEC.md:419 asks
 * for), so the run's placements can be replayed through the reference
 * Scheduler semantics (schedulers.py:89-123) and checked decision for
 * decision.  Job j's probe / task handle is j. */
#define GS_EV_SUBMIT 0     /* submit(probe): outcome + device decided */
#define GS_EV_RELEASE 1    /* DeviceState.release_task(handle) on ledger `device` (+ on_release) */
#define GS_EV_JOB_ENDED 2  /* Scheduler.job_ended(handle) (+ on_release): sa / cg */
#define GS_EV_DRAIN 3      /* one decision of the re-drive that followed (FIFO order) */
typedef struct gs_exec_event {
    int32_t kind;
    int32_t handle;
    int32_t device;      /* ledger index (-1 none) */
    int32_t outcome;     /* GS_ASSIGN / GS_DEFER / GS_REJECTED, or a status code < 0 */
    int64_t freed;       /* GS_EV_RELEASE: bytes release_task returned */
    int64_t free_mem_after;      /* submit / drain: the decision-log values */
    int64_t in_use_warps_after;  /* (schedulers.py:203-218) */
    double t_ms;         /* wall time since the run started */
    gs_probe probe;      /* GS_EV_SUBMIT: the probe as submitted */
} gs_exec_event;
/* Copies up to `cap` events of the last run (returns the full count in
 * *n_events), the per-ledger specs the run used (up to spec_cap; count in
 * *n_devices), and its policy.  Any pointer may be NULL. */
int gs_exec_log(gs_exec_event *events, int64_t cap, int64_t *n_events, gs_spec *specs, int32_t spec_cap,
                int32_t *n_devices, int32_t *policy, int32_t *cg_ratio);

#ifdef __cplusplus
}
#endif

/* ---- shared synthetic-input generator (host + device) ----------------- */
#ifdef __CUDACC__
#define GS_HD __host__ __device__ __forceinline__
#else
#define GS_HD static inline
#endif

GS_HD uint64_t gs_hash64(uint64_t seed, uint64_t i) {
    uint64_t z = seed * 0x9E3779B97F4A7C15ull + i + 0x632BE59BD9B4E019ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* uniform float in [0, 1) with 24 random bits (exactly representable) */
GS_HD float gs_unit(uint64_t seed, uint64_t i) {
    return (float)(gs_hash64(seed, i) >> 40) * (1.0f / 16777216.0f);
}

/* ---- per-workload synthetic inputs (public Rodinia algorithm inputs,
 * restated with a shared generator; PAPER.md:770-771 names Rodinia v3.1) -- */

#define GS_BFS_DEGREE 6
#define GS_KMEANS_K 5
#define GS_NW_PENALTY 10
#define GS_BP_ETA 0.3f
#define GS_BP_MOMENTUM 0.3f
#define GS_BP_TARGET 0.1f
#define GS_SRAD_LAMBDA 0.5f
#define GS_HOTSPOT_AMB 80.0f
#define GS_LUD_BS 32

/* bfs: uniform random out-degree 6 CSR, row_ptr[v] = 6 v, source 0 */
GS_HD int32_t gs_bfs_col(uint64_t seed, uint64_t e, int64_t n) {
    return (int32_t)(gs_hash64(seed, e) % (uint64_t)n);
}
/* hotspot: temperatures around 323 K, power in [0, 0.1) */
GS_HD float gs_hotspot_temp0(uint64_t seed, uint64_t i) { return 323.0f + 10.0f * gs_unit(seed, i); }
GS_HD float gs_hotspot_power(uint64_t seed, uint64_t i) { return 0.1f * gs_unit(seed ^ 0xA5A5A5A5ull, i); }
/* srad: positive image in [1, 2) (no transcendental, for exact parity) */
GS_HD float gs_srad_j0(uint64_t seed, uint64_t i) { return 1.0f + gs_unit(seed, i); }
/* kmeans: feature-major ("flipped") features in [0, 1) */
GS_HD float gs_kmeans_feature(uint64_t seed, uint64_t i) { return gs_unit(seed, i); }
/* backprop: bias input 1, inputs in [0, 1), small weights */
GS_HD float gs_bp_input(uint64_t seed, uint64_t i) { return i == 0 ? 1.0f : gs_unit(seed, i); }
GS_HD float gs_bp_w1(uint64_t seed, uint64_t i) { return (gs_unit(seed + 1, i) - 0.5f) * 2e-3f; }
GS_HD float gs_bp_w2(uint64_t seed, uint64_t j) { return (gs_unit(seed + 2, j) - 0.5f) * 0.2f; }
/* needle: residues in [1, 10] like Rodinia's rand() % 10 + 1 */
GS_HD int32_t gs_nw_seq(uint64_t seed, uint64_t i) { return (int32_t)(gs_hash64(seed, i) % 10u) + 1; }
/* lud: diagonally dominant matrix (no pivoting needed) */
GS_HD float gs_lud_a(uint64_t seed, int64_t i, int64_t j, int64_t n) {
    return gs_unit(seed, (uint64_t)(i * n + j)) + (i == j ? (float)n : 0.0f);
}

/* BLOSUM62, residue order A R N D C Q E G H I L K M F P S T W Y V B Z X * */
#define GS_BLOSUM62_INIT {                                                                  \
    { 4,-1,-2,-2, 0,-1,-1, 0,-2,-1,-1,-1,-1,-2,-1, 1, 0,-3,-2, 0,-2,-1, 0,-4},            \
    {-1, 5, 0,-2,-3, 1, 0,-2, 0,-3,-2, 2,-1,-3,-2,-1,-1,-3,-2,-3,-1, 0,-1,-4},            \
    {-2, 0, 6, 1,-3, 0, 0, 0, 1,-3,-3, 0,-2,-3,-2, 1, 0,-4,-2,-3, 3, 0,-1,-4},            \
    {-2,-2, 1, 6,-3, 0, 2,-1,-1,-3,-4,-1,-3,-3,-1, 0,-1,-4,-3,-3, 4, 1,-1,-4},            \
    { 0,-3,-3,-3, 9,-3,-4,-3,-3,-1,-1,-3,-1,-2,-3,-1,-1,-2,-2,-1,-3,-3,-2,-4},            \
    {-1, 1, 0, 0,-3, 5, 2,-2, 0,-3,-2, 1, 0,-3,-1, 0,-1,-2,-1,-2, 0, 3,-1,-4},            \
    {-1, 0, 0, 2,-4, 2, 5,-2, 0,-3,-3, 1,-2,-3,-1, 0,-1,-3,-2,-2, 1, 4,-1,-4},            \
    { 0,-2, 0,-1,-3,-2,-2, 6,-2,-4,-4,-2,-3,-3,-2, 0,-2,-2,-3,-3,-1,-2,-1,-4},            \
    {-2, 0, 1,-1,-3, 0, 0,-2, 8,-3,-3,-1,-2,-1,-2,-1,-2,-2, 2,-3, 0, 0,-1,-4},            \
    {-1,-3,-3,-3,-1,-3,-3,-4,-3, 4, 2,-3, 1, 0,-3,-2,-1,-3,-1, 3,-3,-3,-1,-4},            \
    {-1,-2,-3,-4,-1,-2,-3,-4,-3, 2, 4,-2, 2, 0,-3,-2,-1,-2,-1, 1,-4,-3,-1,-4},            \
    {-1, 2, 0,-1,-3, 1, 1,-2,-1,-3,-2, 5,-1,-3,-1, 0,-1,-3,-2,-2, 0, 1,-1,-4},            \
    {-1,-1,-2,-3,-1, 0,-2,-3,-2, 1, 2,-1, 5, 0,-2,-1,-1,-1,-1, 1,-3,-1,-1,-4},            \
    {-2,-3,-3,-3,-2,-3,-3,-3,-1, 0, 0,-3, 0, 6,-4,-2,-2, 1, 3,-1,-3,-3,-1,-4},            \
    {-1,-2,-2,-1,-3,-1,-1,-2,-2,-3,-3,-1,-2,-4, 7,-1,-1,-4,-3,-2,-2,-1,-2,-4},            \
    { 1,-1, 1, 0,-1, 0, 0, 0,-1,-2,-2, 0,-1,-2,-1, 4, 1,-3,-2,-2, 0, 0, 0,-4},            \
    { 0,-1, 0,-1,-1,-1,-1,-2,-2,-1,-1,-1,-1,-2,-1, 1, 5,-2,-2, 0,-1,-1, 0,-4},            \
    {-3,-3,-4,-4,-2,-2,-3,-2,-2,-3,-2,-3,-1, 1,-4,-3,-2,11, 2,-3,-4,-3,-2,-4},            \
    {-2,-2,-2,-3,-2,-1,-2,-3, 2,-1,-1,-2,-1, 3,-3,-2,-2, 2, 7,-1,-3,-2,-1,-4},            \
    { 0,-3,-3,-3,-1,-2,-2,-3,-3, 3, 1,-2, 1,-1,-2,-2, 0,-3,-1, 4,-3,-2,-1,-4},            \
    {-2,-1, 3, 4,-3, 0, 1,-1, 0,-3,-4, 0,-3,-3,-2, 0,-1,-4,-3,-3, 4, 1,-1,-4},            \
    {-1, 0, 0, 1,-3, 3, 4,-2, 0,-3,-3, 1,-1,-3,-1, 0,-1,-3,-2,-2, 1, 4,-1,-4},            \
    { 0,-1,-1,-1,-2,-1,-1,-1,-1,-1,-1,-1,-1,-1,-2, 0, 0,-2,-1,-1,-1,-1,-1,-4},            \
    {-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4, 1}}

/* hotspot coefficients (Rodinia hotspot constants; the cell size is fixed
 * at a 1024-grid of a 16 mm chip so larger grids stay numerically stable).
 * Computed in double on the host, identically for the GPU and the oracle. */
static inline void gs_hotspot_coeffs(float *cc, float *rx1, float *ry1, float *rz1) {
    const double t_chip = 0.0005, chip = 0.016, factor_chip = 0.5, spec_heat_si = 1.75e6, k_si = 100.0;
    const double precision = 0.001, max_pd = 3.0e6;
    const double gh = chip / 1024.0, gw = chip / 1024.0;
    const double cap = factor_chip * spec_heat_si * t_chip * gw * gh;
    const double rx = gw / (2.0 * k_si * t_chip * gh);
    const double ry = gh / (2.0 * k_si * t_chip * gw);
    const double rz = t_chip / (k_si * gh * gw);
    const double max_slope = max_pd / (factor_chip * t_chip * spec_heat_si);
    const double step = precision / max_slope;
    *cc = (float)(step / cap);
    *rx1 = (float)(1.0 / rx);
    *ry1 = (float)(1.0 / ry);
    *rz1 = (float)(1.0 / rz);
}

#endif /* GS_WORK_H */
