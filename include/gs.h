/*
 * gs.h — C-ABI of libgs: the B200-native ledger + placement engine that
 * replaces the reference's Python hot path (arXiv 2107.08538 "MGB",
 * artifact package `gpushare`, /root/reference/pkg/src/gpushare).
 *
 * Everything here is plain C: fixed-width integers, plain pointers and
 * sizes, no torch types.  The Python drop-in (paper_2107_08538_b200.gpushare)
 * binds it with ctypes; INTEGRATION.md shows that binding.
 *
 * Ownership / threading: every entry point is synchronous and linearizable
 * ("linearizable in arrival order"); calls on one engine are
 * serialized by an internal mutex.  All decisions are computed by sm_100a
 * kernels (csrc/gs_sched.cu); the host code only marshals commands.
 *
 * Status codes: 0 ok, 1 infeasible (None plan / False /
 * DEFER), 2 reject, -2 config error (ConfigError), -3 contract violation
 * (ContractViolation), -4 CUDA error, -5 out of host/device memory.
 */
#ifndef GS_H
#define GS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 1
#define GS_MAX_DEVICES 32   /* one warp lane per device in mgb-warps */

/* status codes */
#define GS_OK 0
#define GS_INFEASIBLE 1
#define GS_REJECT 2
#define GS_ERR_CONFIG (-2)
#define GS_ERR_CONTRACT (-3)
#define GS_ERR_CUDA (-4)
#define GS_ERR_NOMEM (-5)

/* decision outcomes — schedulers.py:11-13 ASSIGN / DEFER / REJECT */
#define GS_ASSIGN 0
#define GS_DEFER 1
#define GS_REJECTED 2
#define GS_NOT_TRIED 3

/* gs_probe.level flag bits */
#define GS_PROBE_JOB 1
#define GS_PROBE_FRESH 2

/* policies — schedulers.py:26-53 PolicyConfig.kind */
#define GS_POLICY_SA 0
#define GS_POLICY_CG 1
#define GS_POLICY_MGB_SM 2
#define GS_POLICY_MGB_WARPS 3

/* conservation-check violation kinds — device_model.py:220-245, in the
 * order the reference checks them */
#define GS_CHECK_OK 0
#define GS_CHECK_MEM 1
#define GS_CHECK_WARPS 2
#define GS_CHECK_SM_TBS 3
#define GS_CHECK_SM_WARPS 4
#define GS_CHECK_SM_REGS 5
#define GS_CHECK_SM_SMEM 6

/* DeviceSpec — device_model.py:22-30 (field meanings identical). */
typedef struct gs_spec {
    int64_t sm_count;
    int64_t mem_bytes;
    int64_t max_warps_per_sm;
    int64_t max_tbs_per_sm;
    int64_t regs_per_sm;
    int64_t smem_per_sm_bytes;
} gs_spec;

/* The 64-byte probe record: ResourceRequest (task_builder.py:45-55) plus
 * the interned task / job handles of ScheduleRequest (schedulers.py:56-62).
 * Task uids (sim_engine.py:168) and job ids are strings in the reference;
 * the shim interns them to int32 handles. */
typedef struct gs_probe {
    int64_t mem_bytes;
    int64_t heap_limit_bytes;
    int64_t total_warps;
    double est_duration_ms;
    int32_t thread_blocks;
    int32_t warps_per_block;
    int32_t threads_per_block;
    int32_t regs_per_thread;
    int32_t smem_per_block;
    int32_t handle;   /* task uid handle (residency row) */
    int32_t job;      /* job id handle */
    int32_t level;    /* bit 0: 1 = "job" level, 0 = "task"; bit 1 (GS_PROBE_FRESH):
                       * the caller guarantees no device holds a residency row
                       * for `handle`, so the decision skips reading it */
} gs_probe;

/* Per-device ledger header, in pinned host-mapped memory so the host reads
 * and writes the same bytes the decision kernels stage (DeviceState fields,
 * device_model.py:85-93).  Followed by four int32[sm_count] arrays, each
 * padded to a multiple of 4 entries: sm_warps, sm_tbs, sm_regs, sm_smem. */
typedef struct gs_ledger {
    int64_t free_mem;
    int64_t in_use_warps;
    int64_t version;
    int64_t held_mem;     /* Σ resident mem_bytes (check_conservation) */
    int64_t held_warps;   /* Σ resident warps */
    /* Grow epoch: bumped by every operation that can ENLARGE a device's
     * free resources (release_task, negative reservations) and by host-side
     * writes to the ledger.  A scheduler's FIFO re-drive only re-scores
     * pending probes against devices whose epoch moved since its last full
     * pass — exact, because inside and between passes resources otherwise
     * only shrink (schedulers.py:105-112 tries every pending request). */
    int64_t grow_epoch;
    int64_t reserved;     /* keeps the header 64 B (arrays 16 B aligned) */
    int32_t rr_cursor;
    int32_t sm_count;
} gs_ledger;

/* One decision (Decision, schedulers.py:65-68, plus the decision-log
 * values free_mem_after / in_use_warps_after, schedulers.py:203-218). */
typedef struct gs_decision {
    int32_t outcome;        /* GS_ASSIGN / GS_DEFER / GS_REJECTED / GS_NOT_TRIED */
    int32_t device;         /* -1 when none */
    int64_t free_mem_after;
    int64_t in_use_warps_after;
    int32_t pending_index;  /* on_release: FIFO position before the pass */
    int32_t handle;
} gs_decision;

/* A resident task's row (_Residency, device_model.py:69-77). */
typedef struct gs_residency {
    int64_t mem_bytes;
    int64_t warps;
    int64_t regs_per_block;
    int64_t smem_per_block;
    int32_t present;
    int32_t has_blocks;
    int32_t warps_per_block;
    int32_t thread_blocks;  /* Σ blocks_per_sm of the committed plan */
} gs_residency;

typedef struct gs_engine gs_engine;
typedef struct gs_device gs_device;
typedef struct gs_sched gs_sched;

/* ---- engine ---------------------------------------------------------- */
int gs_abi_version(void);
const char *gs_last_error(void);
/* Opens the engine on CUDA device `cuda_device`; fails (GS_ERR_CUDA) when
 * no GPU is present — there is no CPU fallback. */
int gs_engine_open(int cuda_device, gs_engine **out);
void gs_engine_close(gs_engine *eng);
/* Grow every device's residency table to hold handles [0, capacity). */
int gs_engine_reserve_handles(gs_engine *eng, int32_t capacity);
int32_t gs_engine_handle_capacity(gs_engine *eng);
/* Number of decision-kernel launches issued so far (evidence counter). */
int64_t gs_engine_launches(gs_engine *eng);

/* ---- device ledgers: DeviceState (device_model.py:80-245) ------------- */
int gs_device_create(gs_engine *eng, const gs_spec *spec, int32_t index, gs_device **out);
void gs_device_destroy(gs_device *dev);
/* Host pointer of the mapped ledger header; arrays follow (see gs_ledger). */
gs_ledger *gs_device_ledger(gs_device *dev);
/* which: 0 sm_warps, 1 sm_tbs, 2 sm_regs, 3 sm_smem */
int32_t *gs_device_sm_array(gs_device *dev, int32_t which);

/* try_place_blocks (device_model.py:120-139): GS_OK + plan, or
 * GS_INFEASIBLE (None).  Pure: does not mutate the ledger. */
int gs_try_place(gs_device *dev, const gs_probe *req, int32_t *blocks_per_sm,
                 int32_t *final_cursor, int64_t *version);
/* commit_placement (device_model.py:141-161): GS_ERR_CONTRACT if stale. */
int gs_commit(gs_device *dev, int32_t handle, const gs_probe *req,
              const int32_t *blocks_per_sm, int32_t final_cursor, int64_t plan_version);
/* reserve_memory (:169-174): GS_OK or GS_INFEASIBLE (False). */
int gs_reserve_memory(gs_device *dev, int64_t nbytes);
/* assign_memory (:176-178) and add_warps (:180-183). */
int gs_assign_memory(gs_device *dev, int32_t handle, int64_t nbytes);
int gs_add_warps(gs_device *dev, int32_t handle, int64_t warps);
/* allocate_raw (:185-190): GS_OK or GS_INFEASIBLE. */
int gs_allocate_raw(gs_device *dev, int32_t handle, int64_t nbytes);
/* release_task (:192-209): GS_OK + freed bytes, GS_ERR_CONTRACT if unknown. */
int gs_release(gs_device *dev, int32_t handle, int64_t *freed_bytes);
/* check_conservation (:220-245): GS_OK, or GS_ERR_CONTRACT with the first
 * violation's kind (GS_CHECK_*), SM index and the held sums. */
int gs_check_conservation(gs_device *dev, int32_t *kind, int32_t *sm,
                          int64_t *held_mem, int64_t *held_warps);
/* Read one residency row (+ blocks_per_sm when non-NULL). */
int gs_residency_read(gs_device *dev, int32_t handle, gs_residency *row,
                      int32_t *blocks_per_sm);

/* ---- scheduler: Scheduler (schedulers.py:71-218) ---------------------- */
int gs_sched_create(gs_engine *eng, gs_device *const *devices, int32_t n_devices,
                    int32_t policy, int32_t cg_ratio, int32_t skip_ahead,
                    gs_sched **out);
void gs_sched_destroy(gs_sched *s);
/* submit (schedulers.py:89-95): decide one request; DEFER queues it. */
int gs_submit(gs_sched *s, const gs_probe *req, gs_decision *out);
/* Decide n requests in order, each exactly as gs_submit would. */
int gs_submit_batch(gs_sched *s, const gs_probe *reqs, int32_t n, gs_decision *out);
/* on_release (schedulers.py:97-113): re-drive the FIFO.  Writes one
 * decision per tried entry in FIFO order (out may be NULL); *n_tried and
 * *n_admitted are set.  Admitted entries leave the device-side queue. */
int gs_on_release(gs_sched *s, gs_decision *out, int32_t out_cap,
                  int32_t *n_tried, int32_t *n_admitted);
/* A task's completion in one decision launch: DeviceState.release_task
 * (device_model.py:192-209) on the scheduler's device `dev_index`, then
 * on_release (schedulers.py:97-113) — the pair SimEngine runs at every
 * task end (sim_engine.py:541-547).  Outputs as gs_release + gs_on_release;
 * the re-drive runs even when the release names an unknown task (then
 * GS_ERR_CONTRACT is returned after it). */
int gs_release_redrive(gs_sched *s, int32_t dev_index, int32_t handle, int64_t *freed,
                       gs_decision *out, int32_t out_cap, int32_t *n_tried, int32_t *n_admitted);
/* job_ended (schedulers.py:115-123). */
int gs_job_ended(gs_sched *s, int32_t job);
int32_t gs_pending_count(gs_sched *s);
/* Job-granular state mirrors: sa_owner[d] (job handle or -1), cg_counts[d]. */
int gs_sched_job_state(gs_sched *s, int32_t *sa_owner, int32_t *cg_counts,
                       int32_t *cg_cursor);

/* ---- persistent decision kernel over a pinned host-mapped command ring --
 * The paper's probe channel (probes and scheduler talk
 * over shared memory) on B200: one resident decision warp polls the ring;
 * submit / on_release / job_ended of this scheduler and the ledger ops of
 * its devices become ring commands (no launch, no wait for a free SM).
 * Capacities (pending queue, task handles, job handles) are fixed at start;
 * the host must not write the ledgers while the ring runs.  An idle
 * watchdog retires the kernel after 200 ms idle; the next call relaunches it. */
int gs_sched_ring_start(gs_sched *s, int32_t max_pending, int32_t max_handles, int32_t max_jobs);
int gs_sched_ring_stop(gs_sched *s);
/* Decisions served so far (kernel-launched commands + ring commands). */
int64_t gs_engine_decisions(gs_engine *eng);

/* ---- placement sweep (BASELINE cfg 4) -------------------------------- */
/* Runs the whole synthetic stream on the GPU in one launch: for each probe
 * i: submit(i); then, if more than `max_resident` tasks are resident or the
 * queue is non-empty, release the oldest resident task and on_release().
 * Probe i uses handle i (the table is grown to n).  Writes the compact
 * event log: for every ASSIGN/DEFER/REJECT of a submit and every admit of a
 * drain, (kind, handle, device) with kind 0 submit-assign, 1 submit-defer,
 * 2 submit-reject, 3 drain-admit.  Returns the number of log entries in
 * *n_events and the kernel-only time in *kernel_ms.  The tasks still
 * resident at the end keep their ledger reservations, so a sweep consumes
 * the scheduler: later gs_submit / gs_submit_batch / gs_sweep calls on it
 * return GS_ERR_CONTRACT. */
int gs_sweep(gs_sched *s, const gs_probe *probes, int32_t n, int32_t max_resident,
             int32_t *events, int64_t events_cap, int64_t *n_events, float *kernel_ms);

#ifdef __cplusplus
}
#endif
#endif /* GS_H */
