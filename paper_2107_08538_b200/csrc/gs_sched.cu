// gs_sched.cu — B200-native ledger + placement engine (libgs).
//
// Replaces the reference's Python hot path:
//   DeviceState ledgers / try_place_blocks / commit   device_model.py:80-245
//   Scheduler.submit / on_release / job_ended         schedulers.py:89-123
//   _try_mgb_sm (Alg. 2) / _try_mgb_warps (Alg. 3)    schedulers.py:137-171
//   _try_sa / _try_cg / _impossible_everywhere        schedulers.py:173-199
//
// Design: one CTA of 256 threads is the single decision
// authority.  It stages every device ledger (free HBM, in-use warps, per-SM
// warps/TBs/regs/smem; 2.4 KB per 148-SM device) from pinned host-mapped
// memory into shared memory, interprets a command stream in arrival order
// (linearizable), and writes the dirty ledgers back.
//   * mgb-warps: lane d scores device d; ballot(free_mem >= mem) +
//     warp argmin over (in_use_warps, d).
//   * mgb-sm: warp w scores device w in parallel (per-SM residual capacity
//     over 148 SMs, 64-bit warp reductions); the first feasible device in
//     index order commits using the closed-form round-robin water-fill of
//     SURVEY.md App. A (binary search on full rounds + ballot prefix ranks
//     in cursor order) instead of the reference's one-block-per-visit loop.
//   * on_release: a parallel prefilter marks pending probes that cannot fit
//     the pass-start ledgers (exact: resources only shrink inside a pass),
//     then survivors are decided serially in FIFO order.
// Residency rows (_Residency, device_model.py:69-77) live in HBM, indexed
// by the interned task handle.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <stdio.h>
#include <stdlib.h>
#include <limits.h>
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>

#include "../../include/gs.h"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowHdrWords = sizeof(gs_residency) / 4;  // 12

enum Op : int32_t {
  OP_SUBMIT = 1,
  OP_ON_RELEASE = 2,
  OP_JOB_ENDED = 3,
  OP_RELEASE = 10,
  OP_ALLOC_RAW = 11,
  OP_RESERVE = 12,
  OP_ASSIGN = 13,
  OP_ADD_WARPS = 14,
  OP_TRY_PLACE = 15,
  OP_COMMIT = 16,
  OP_CHECK = 17,
};

struct Cmd {
  int32_t op, dev, handle, job;
  int64_t a, b;
  gs_probe probe;
};
static_assert(sizeof(gs_probe) == 64, "probe record must be 64 B");

struct SchedState {  // pinned host-mapped
  int32_t sa_owner[GS_MAX_DEVICES];
  int32_t cg_counts[GS_MAX_DEVICES];
  int32_t cg_cursor;
  int32_t pend_count;
  int32_t fifo_head, fifo_tail;
  int32_t n_tried, n_admitted;
  int32_t pad0, pad1;
  int64_t n_events;
};

struct KDev {
  gs_ledger *led;   // device pointer of the mapped ledger
  int32_t *res;     // residency rows in HBM
  int32_t stride;   // words per residency row
  int32_t n_sm;
  int32_t arr_pad;  // padded array length (ledger + smem)
  int32_t smem_off; // int offset of this device's arrays in dynamic smem
  gs_spec spec;
};

struct KParams {
  int32_t n_dev, policy, cg_ratio, skip_ahead;
  int32_t n_cmds, max_sm_pad, max_resident, sweep;
  KDev dev[GS_MAX_DEVICES];
  SchedState *st;
  const Cmd *cmds;
  gs_decision *results;
  gs_decision *drain_out;
  int32_t drain_cap;
  int32_t pend_cap;
  gs_probe *pend;
  int32_t *pend_flag;
  int32_t *claims;
  int32_t job_cap;
  int32_t fifo_cap;
  int32_t *fifo;
  int32_t *plan_io;
  int32_t *events;
  int64_t events_cap;
  const gs_probe *sweep_probes;
};

struct SLed {
  long long free_mem, in_use_warps, version, held_mem, held_warps;
  int rr_cursor, dirty;
};

struct Shape {
  long long mem, T, wpb, rpb, spb, tw;
};

__device__ __forceinline__ Shape shape_of(const gs_probe &p) {
  Shape s;
  s.mem = p.mem_bytes;
  s.T = p.thread_blocks;
  s.wpb = p.warps_per_block;
  s.rpb = (long long)p.regs_per_thread * (long long)p.threads_per_block;
  s.spb = p.smem_per_block;
  s.tw = p.total_warps;
  return s;
}

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_min64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, (long long)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_max32(int v) { return __reduce_max_sync(0xffffffffu, v); }

// Kernel-wide shared state (static part).
struct SmemStatic {
  SLed led[GS_MAX_DEVICES];
  SchedState st;
  Cmd cmd;
  int feas[GS_MAX_DEVICES];
  int chosen;
  int outcome;
  int cursor_out;
  int chk;
  long long scratch64;
};

__device__ __forceinline__ int *arr_warps(int *dyn, const KDev &D) { return dyn + D.smem_off; }
__device__ __forceinline__ int *arr_tbs(int *dyn, const KDev &D) { return dyn + D.smem_off + D.arr_pad; }
__device__ __forceinline__ int *arr_regs(int *dyn, const KDev &D) { return dyn + D.smem_off + 2 * D.arr_pad; }
__device__ __forceinline__ int *arr_smem(int *dyn, const KDev &D) { return dyn + D.smem_off + 3 * D.arr_pad; }

// Per-SM residual capacity for one more block of this shape, clamped to T.
// Mirrors _sm_admits (device_model.py:105-118) in closed form.
__device__ __forceinline__ int sm_cap(const KDev &D, int *dyn, int s, const Shape &sh) {
  const int *w = arr_warps(dyn, D), *t = arr_tbs(dyn, D), *r = arr_regs(dyn, D), *m = arr_smem(dyn, D);
  long long c = D.spec.max_tbs_per_sm - (long long)t[s];
  if (sh.wpb > 0) {
    long long num = D.spec.max_warps_per_sm - (long long)w[s];
    c = min(c, num < 0 ? -1LL : num / sh.wpb);
  } else if ((long long)w[s] > D.spec.max_warps_per_sm) {
    c = 0;
  }
  if (sh.rpb != 0) {
    long long num = D.spec.regs_per_sm - (long long)r[s];
    c = min(c, num < 0 ? -1LL : (sh.rpb > 0 ? num / sh.rpb : c));
  }
  if (sh.spb != 0) {
    long long num = D.spec.smem_per_sm_bytes - (long long)m[s];
    c = min(c, num < 0 ? -1LL : (sh.spb > 0 ? num / sh.spb : c));
  }
  if (c < 0) c = 0;
  if (c > sh.T) c = sh.T;
  return (int)c;
}

// Σ cap over the device's SMs (one warp).
__device__ __forceinline__ long long warp_total_cap(const KDev &D, int *dyn, const Shape &sh, int lane) {
  long long tot = 0;
  for (int s = lane; s < D.n_sm; s += 32) tot += sm_cap(D, dyn, s, sh);
  return warp_sum64(tot);
}

// occupancy_limit_per_sm (device_model.py:48-58) × sm_count.
__device__ __forceinline__ long long empty_capacity_blocks(const gs_spec &S, const Shape &sh) {
  long long lim = S.max_tbs_per_sm;
  if (sh.wpb > 0) lim = min(lim, S.max_warps_per_sm / sh.wpb);
  if (sh.rpb > 0) lim = min(lim, S.regs_per_sm / sh.rpb);
  if (sh.spb > 0) lim = min(lim, S.smem_per_sm_bytes / sh.spb);
  if (lim < 0) lim = 0;
  return lim * S.sm_count;
}

__device__ __forceinline__ int32_t *res_row(const KDev &D, int h) { return D.res + (size_t)h * D.stride; }

// _entry (device_model.py:211-216): create an empty residency row on demand.
__device__ __forceinline__ gs_residency *entry(const KDev &D, int h) {
  gs_residency *row = reinterpret_cast<gs_residency *>(res_row(D, h));
  if (!row->present) {
    row->mem_bytes = 0;
    row->warps = 0;
    row->regs_per_block = 0;
    row->smem_per_block = 0;
    row->has_blocks = 0;
    row->warps_per_block = 0;
    row->present = 1;
  }
  return row;
}

// Closed-form round-robin placement for one device, computed by one warp.
// Writes blocks into P[0..n) and returns the final cursor (all lanes), or -1
// when the blocks cannot fit (the reference's n-consecutive-misses None).
// Equivalent to try_place_blocks (device_model.py:120-139); SURVEY.md App. A.
__device__ int warp_plan(const KDev &D, int *dyn, const SLed &L, const Shape &sh, int *cap, int *P,
                         int lane) {
  const int n = D.n_sm;
  long long tot = 0;
  int mx = 0;
  for (int s = lane; s < n; s += 32) {
    int c = sm_cap(D, dyn, s, sh);
    cap[s] = c;
    tot += c;
    mx = max(mx, c);
  }
  tot = warp_sum64(tot);
  mx = warp_max32(mx);
  __syncwarp();
  if (tot < sh.T) return -1;
  int c0 = L.rr_cursor % n;
  if (c0 < 0) c0 += n;
  if (sh.T <= 0) {
    for (int s = lane; s < n; s += 32) P[s] = 0;
    __syncwarp();
    return c0;
  }
  // largest k in [0, mx] with S(k) = Σ min(cap, k) <= T  (full rounds)
  int lo = 0, hi = mx;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    long long sk = 0;
    for (int s = lane; s < n; s += 32) sk += min(cap[s], mid);
    sk = warp_sum64(sk);
    if (sk <= sh.T) lo = mid; else hi = mid - 1;
  }
  const int k = lo;
  long long sk = 0;
  for (int s = lane; s < n; s += 32) {
    int v = min(cap[s], k);
    P[s] = v;
    sk += v;
  }
  sk = warp_sum64(sk);
  __syncwarp();
  const long long rem = sh.T - sk;
  // walk the SMs in visit order from the cursor, 32 at a time
  int last = -1;
  long long run = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int base = 0; base < n; base += 32) {
    int p = base + lane;
    int s = p < n ? (c0 + p) % n : 0;
    bool q = false;
    if (p < n) q = rem > 0 ? (cap[s] > k) : (cap[s] >= k);
    unsigned b = __ballot_sync(0xffffffffu, q);
    if (rem > 0) {
      long long rank = run + __popc(b & lt);
      if (q && rank < rem) {
        P[s] = k + 1;
        if (rank == rem - 1) last = s;
      }
      run += __popc(b);
    } else if (b) {
      int lp = base + 31 - __clz(b);
      last = (c0 + lp) % n;
    }
  }
  last = __reduce_max_sync(0xffffffffu, last);
  __syncwarp();
  return (last + 1) % n;
}

// commit_placement (device_model.py:141-161), one warp.
__device__ void warp_commit(const KDev &D, int *dyn, SLed &L, int h, const Shape &sh, const int *P,
                            int cursor, int lane) {
  gs_residency *row = reinterpret_cast<gs_residency *>(res_row(D, h));
  if (lane == 0) entry(D, h);
  __syncwarp();
  int32_t *blocks = res_row(D, h) + kRowHdrWords;
  int *w = arr_warps(dyn, D), *t = arr_tbs(dyn, D), *r = arr_regs(dyn, D), *m = arr_smem(dyn, D);
  for (int s = lane; s < D.n_sm; s += 32) {
    int c = P[s];
    blocks[s] = c;
    if (c) {
      t[s] += c;
      w[s] += (int)(c * sh.wpb);
      r[s] += (int)(c * sh.rpb);
      m[s] += (int)(c * sh.spb);
    }
  }
  if (lane == 0) {
    L.rr_cursor = cursor;
    row->has_blocks = 1;
    row->regs_per_block = sh.rpb;
    row->smem_per_block = sh.spb;
    row->warps_per_block = (int32_t)sh.wpb;
    L.version += 1;
    L.dirty = 1;
  }
  __syncwarp();
}

// reserve + assign + add_warps for an admitted task (single thread).
__device__ void admit_accounting(const KDev &D, SLed &L, int h, const Shape &sh) {
  L.free_mem -= sh.mem;  // reserve_memory
  L.version += 1;
  gs_residency *row = entry(D, h);  // assign_memory
  row->mem_bytes += sh.mem;
  L.held_mem += sh.mem;
  L.version += 1;
  row->warps += sh.tw;  // add_warps
  L.in_use_warps += sh.tw;
  L.held_warps += sh.tw;
  L.version += 1;
  L.dirty = 1;
}

__device__ __forceinline__ void fifo_push(const KParams &p, SchedState &st, int d, int h) {
  if (!p.sweep) return;
  int pos = st.fifo_tail % p.fifo_cap;
  p.fifo[2 * pos] = d;
  p.fifo[2 * pos + 1] = h;
  st.fifo_tail++;
}

__device__ __forceinline__ void log_event(const KParams &p, SchedState &st, int kind, int h, int d) {
  if (!p.events) return;
  long long i = st.n_events++;
  if (i < p.events_cap) {
    p.events[3 * i] = kind;
    p.events[3 * i + 1] = h;
    p.events[3 * i + 2] = d;
  }
}

// One admission attempt (Scheduler._try, schedulers.py:127-135).  Called by
// all threads; returns outcome / device in S.outcome / S.chosen.
__device__ void decide(const KParams &p, SmemStatic &S, int *dyn, int *scratch, const gs_probe &pr,
                       int h, int job) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_dev = p.n_dev;
  if (p.policy == GS_POLICY_MGB_WARPS) {
    // _try_mgb_warps (schedulers.py:155-171)
    if (warp == 0) {
      const Shape sh = shape_of(pr);
      bool ok = lane < n_dev && S.led[lane].free_mem >= sh.mem;
      unsigned b = __ballot_sync(0xffffffffu, ok);
      if (b == 0) {
        // _impossible_everywhere(check_compute=False) (schedulers.py:191-199)
        bool possible = lane < n_dev && !(sh.mem > p.dev[lane].spec.mem_bytes);
        unsigned pb = __ballot_sync(0xffffffffu, possible);
        if (lane == 0) {
          S.outcome = pb ? GS_DEFER : GS_REJECTED;
          S.chosen = -1;
        }
      } else {
        long long key = ok ? S.led[lane].in_use_warps : LLONG_MAX;
        long long m = warp_min64(key);
        unsigned cand = __ballot_sync(0xffffffffu, ok && key == m);
        int d = __ffs(cand) - 1;
        if (lane == 0) {
          admit_accounting(p.dev[d], S.led[d], h, sh);
          S.outcome = GS_ASSIGN;
          S.chosen = d;
        }
      }
    }
    __syncthreads();
    return;
  }
  if (p.policy == GS_POLICY_MGB_SM) {
    // _try_mgb_sm (schedulers.py:137-153): devices in index order; score
    // all devices in parallel (one warp each), commit on the first feasible.
    const Shape sh = shape_of(pr);
    for (int d = warp; d < n_dev; d += kWarps) {
      int f = 0;
      if (S.led[d].free_mem >= sh.mem) {
        long long tot = warp_total_cap(p.dev[d], dyn, sh, lane);
        f = tot >= sh.T;
      }
      if (lane == 0) S.feas[d] = f;
    }
    __syncthreads();
    if (warp == 0) {
      bool f = lane < n_dev && S.feas[lane];
      unsigned b = __ballot_sync(0xffffffffu, f);
      if (b) {
        int d = __ffs(b) - 1;
        const KDev &D = p.dev[d];
        int *cap = scratch;
        int *P = scratch + p.max_sm_pad;
        int cur = warp_plan(D, dyn, S.led[d], sh, cap, P, lane);
        warp_commit(D, dyn, S.led[d], h, sh, P, cur, lane);
        if (lane == 0) {
          admit_accounting(D, S.led[d], h, sh);
          S.outcome = GS_ASSIGN;
          S.chosen = d;
        }
      } else {
        // _impossible_everywhere(check_compute=True)
        bool possible = false;
        if (lane < n_dev) {
          const gs_spec &sp = p.dev[lane].spec;
          possible = !(sh.mem > sp.mem_bytes) && !(empty_capacity_blocks(sp, sh) < sh.T);
        }
        unsigned pb = __ballot_sync(0xffffffffu, possible);
        if (lane == 0) {
          S.outcome = pb ? GS_DEFER : GS_REJECTED;
          S.chosen = -1;
        }
      }
    }
    __syncthreads();
    return;
  }
  if (tid == 0) {
    if (p.policy == GS_POLICY_SA) {
      // _try_sa (schedulers.py:173-178)
      S.outcome = GS_DEFER;
      S.chosen = -1;
      for (int d = 0; d < n_dev; ++d) {
        if (S.st.sa_owner[d] < 0) {
          S.st.sa_owner[d] = job;
          S.outcome = GS_ASSIGN;
          S.chosen = d;
          break;
        }
      }
    } else {
      // _try_cg (schedulers.py:180-189)
      S.outcome = GS_DEFER;
      S.chosen = -1;
      for (int step = 0; step < n_dev; ++step) {
        int d = (S.st.cg_cursor + step) % n_dev;
        if (S.st.cg_counts[d] < p.cg_ratio) {
          S.st.cg_counts[d] += 1;
          if (job >= 0 && job < p.job_cap) p.claims[job] = d;
          S.st.cg_cursor = (d + 1) % n_dev;
          S.outcome = GS_ASSIGN;
          S.chosen = d;
          break;
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void fill_decision(gs_decision &o, const SmemStatic &S, int outcome, int d,
                                              int pidx, int h) {
  o.outcome = outcome;
  o.device = d;
  o.free_mem_after = d >= 0 ? S.led[d].free_mem : 0;
  o.in_use_warps_after = d >= 0 ? S.led[d].in_use_warps : 0;
  o.pending_index = pidx;
  o.handle = h;
}

// Parallel feasibility prefilter for one pass (exact: see header).
__device__ void drain_prefilter(const KParams &p, SmemStatic &S, int *dyn, int P) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (p.policy == GS_POLICY_MGB_WARPS) {
    if (warp == 0) {
      long long f = lane < p.n_dev ? S.led[lane].free_mem : LLONG_MIN;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) f = max(f, (long long)__shfl_xor_sync(0xffffffffu, f, o));
      if (lane == 0) S.scratch64 = f;
    }
    __syncthreads();
    const long long maxfree = S.scratch64;
    for (int i = tid; i < P; i += kThreads) p.pend_flag[i] = p.pend[i].mem_bytes <= maxfree;
  } else if (p.policy == GS_POLICY_MGB_SM) {
    for (int i = warp; i < P; i += kWarps) {
      const Shape sh = shape_of(p.pend[i]);
      int ok = 0;
      for (int d = 0; d < p.n_dev && !ok; ++d) {
        if (S.led[d].free_mem < sh.mem) continue;
        if (warp_total_cap(p.dev[d], dyn, sh, lane) >= sh.T) ok = 1;
      }
      if (lane == 0) p.pend_flag[i] = ok;
    }
  } else {
    for (int i = tid; i < P; i += kThreads) p.pend_flag[i] = 1;
  }
  __syncthreads();
}

// Scheduler.on_release (schedulers.py:97-113).
__device__ void on_release(const KParams &p, SmemStatic &S, int *dyn, int *scratch, bool write_out) {
  const int tid = threadIdx.x;
  const int P = S.st.pend_count;
  drain_prefilter(p, S, dyn, P);
  int tried = 0, admitted = 0;
  for (int i = 0; i < P; ++i) {
    tried = i + 1;
    int outcome, d;
    const int h = p.pend[i].handle;
    if (!p.pend_flag[i]) {
      outcome = GS_DEFER;
      d = -1;
    } else {
      decide(p, S, dyn, scratch, p.pend[i], h, p.pend[i].job);
      outcome = S.outcome;
      d = S.chosen;
    }
    if (tid == 0) {
      if (write_out && i < p.drain_cap) fill_decision(p.drain_out[i], S, outcome, d, i, h);
      if (outcome == GS_ASSIGN) {
        fifo_push(p, S.st, d, h);
        log_event(p, S.st, 3, h, d);
      }
    }
    // pend_flag doubles as the "admitted" mark for compaction (2 = gone)
    if (outcome == GS_ASSIGN) {
      if (tid == 0) p.pend_flag[i] = 2;
      admitted++;
    } else if (!p.skip_ahead) {
      break;
    }
    __syncthreads();
  }
  __syncthreads();
  // stable in-place compaction of the survivors
  __shared__ int wsum[kWarps];
  __shared__ int base_out;
  if (tid == 0) base_out = 0;
  __syncthreads();
  for (int base = 0; base < P; base += kThreads) {
    int i = base + tid;
    gs_probe mine;
    bool keep = false;
    if (i < P) {
      keep = !(i < tried && p.pend_flag[i] == 2);
      if (keep) mine = p.pend[i];
    }
    unsigned b = __ballot_sync(0xffffffffu, keep);
    int lane = tid & 31, warp = tid >> 5;
    if (lane == 0) wsum[warp] = __popc(b);
    __syncthreads();
    int off = base_out;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    off += __popc(b & ((1u << lane) - 1u));
    __syncthreads();
    if (keep) p.pend[off] = mine;
    if (tid == kThreads - 1) {
      int tot = 0;
      for (int w = 0; w < kWarps; ++w) tot += wsum[w];
      base_out += tot;
    }
    __syncthreads();
  }
  if (tid == 0) {
    S.st.pend_count = base_out;
    S.st.n_tried = tried;
    S.st.n_admitted = admitted;
  }
  __syncthreads();
}

__device__ void submit(const KParams &p, SmemStatic &S, int *dyn, int *scratch, const gs_probe &pr,
                       gs_decision *out) {
  const int h = pr.handle;
  decide(p, S, dyn, scratch, pr, h, pr.job);
  if (threadIdx.x == 0) {
    const int oc = S.outcome, d = S.chosen;
    if (oc == GS_DEFER) {
      int pc = S.st.pend_count;
      if (pc < p.pend_cap) p.pend[pc] = pr;
      S.st.pend_count = pc + 1;
    }
    if (oc == GS_ASSIGN) fifo_push(p, S.st, d, h);
    log_event(p, S.st, oc == GS_ASSIGN ? 0 : (oc == GS_DEFER ? 1 : 2), h, d);
    if (out) fill_decision(*out, S, oc, d, -1, h);
  }
  __syncthreads();
}

// release_task (device_model.py:192-209), one warp.
__device__ int warp_release(const KDev &D, int *dyn, SLed &L, int h, long long *freed, int lane) {
  gs_residency *row = reinterpret_cast<gs_residency *>(res_row(D, h));
  int present = row->present;
  if (!present) return GS_ERR_CONTRACT;
  if (row->has_blocks) {
    const int32_t *blocks = res_row(D, h) + kRowHdrWords;
    int *w = arr_warps(dyn, D), *t = arr_tbs(dyn, D), *r = arr_regs(dyn, D), *m = arr_smem(dyn, D);
    for (int s = lane; s < D.n_sm; s += 32) {
      int c = blocks[s];
      if (c) {
        t[s] -= c;
        w[s] -= (int)(c * (long long)row->warps_per_block);
        r[s] -= (int)(c * row->regs_per_block);
        m[s] -= (int)(c * row->smem_per_block);
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    L.free_mem += row->mem_bytes;
    L.in_use_warps -= row->warps;
    L.held_mem -= row->mem_bytes;
    L.held_warps -= row->warps;
    L.version += 1;
    L.dirty = 1;
    *freed = row->mem_bytes;
    row->present = 0;
  }
  __syncwarp();
  return GS_OK;
}

__global__ void __launch_bounds__(kThreads, 1) gs_interp_kernel(KParams p) {
  extern __shared__ int dyn[];
  __shared__ SmemStatic S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int *scratch = dyn;  // per-warp scratch lives after the device arrays
  {
    int tot = 0;
    for (int d = 0; d < p.n_dev; ++d) tot = max(tot, p.dev[d].smem_off + 4 * p.dev[d].arr_pad);
    scratch = dyn + tot + warp * 2 * p.max_sm_pad;
  }
  // ---- stage ledgers + scheduler state into shared memory ----
  for (int d = 0; d < p.n_dev; ++d) {
    const KDev &D = p.dev[d];
    const int32_t *src = reinterpret_cast<const int32_t *>(D.led + 1);
    int *dst = dyn + D.smem_off;
    for (int i = tid; i < 4 * D.arr_pad; i += kThreads) dst[i] = src[i];
  }
  if (tid < p.n_dev) {
    const gs_ledger *g = p.dev[tid].led;
    SLed &L = S.led[tid];
    L.free_mem = g->free_mem;
    L.in_use_warps = g->in_use_warps;
    L.version = g->version;
    L.held_mem = g->held_mem;
    L.held_warps = g->held_warps;
    L.rr_cursor = g->rr_cursor;
    L.dirty = 0;
  }
  if (tid == 0) S.st = *p.st;
  __syncthreads();

  for (int ci = 0; ci < p.n_cmds; ++ci) {
    if (p.sweep) {
      // placement sweep (BASELINE cfg 4): submit probe ci, then maybe
      // release the oldest resident task and re-drive the FIFO.
      const gs_probe pr = p.sweep_probes[ci];
      submit(p, S, dyn, scratch, pr, nullptr);
      const int resident = S.st.fifo_tail - S.st.fifo_head;
      if (resident > p.max_resident || S.st.pend_count > 0) {
        if (resident > 0) {
          const int pos = S.st.fifo_head % p.fifo_cap;
          const int d = p.fifo[2 * pos], h = p.fifo[2 * pos + 1];
          if (warp == 0) {
            long long freed;
            warp_release(p.dev[d], dyn, S.led[d], h, &freed, lane);
          }
          __syncthreads();
          if (tid == 0) S.st.fifo_head++;
          __syncthreads();
        }
        on_release(p, S, dyn, scratch, false);
      }
      continue;
    }
    // copy the command into shared memory (one PCIe/L2 read per word)
    if (tid < (int)(sizeof(Cmd) / 4))
      reinterpret_cast<int32_t *>(&S.cmd)[tid] = reinterpret_cast<const int32_t *>(p.cmds + ci)[tid];
    __syncthreads();
    const Cmd &c = S.cmd;
    gs_decision *out = p.results + ci;
    switch (c.op) {
      case OP_SUBMIT:
        submit(p, S, dyn, scratch, c.probe, out);
        break;
      case OP_ON_RELEASE:
        on_release(p, S, dyn, scratch, true);
        if (tid == 0) {
          out->outcome = GS_OK;
          out->free_mem_after = S.st.n_tried;
          out->in_use_warps_after = S.st.n_admitted;
        }
        break;
      case OP_JOB_ENDED:
        // job_ended (schedulers.py:115-123)
        if (tid == 0) {
          for (int d = 0; d < p.n_dev; ++d)
            if (S.st.sa_owner[d] == c.job) S.st.sa_owner[d] = -1;
          if (p.policy == GS_POLICY_CG && c.job >= 0 && c.job < p.job_cap) {
            int d = p.claims[c.job];
            if (d >= 0) {
              S.st.cg_counts[d] -= 1;
              p.claims[c.job] = -1;
            }
          }
          out->outcome = GS_OK;
        }
        break;
      case OP_RELEASE:
        if (warp == 0) {
          long long freed = 0;
          int rc = warp_release(p.dev[c.dev], dyn, S.led[c.dev], c.handle, &freed, lane);
          if (lane == 0) {
            out->outcome = rc;
            out->free_mem_after = freed;
          }
        }
        break;
      case OP_RESERVE:
      case OP_ALLOC_RAW:
        if (tid == 0) {
          SLed &L = S.led[c.dev];
          if (c.a > L.free_mem) {
            out->outcome = GS_INFEASIBLE;
          } else {
            L.free_mem -= c.a;
            L.version += 1;
            L.dirty = 1;
            if (c.op == OP_ALLOC_RAW) {
              gs_residency *row = entry(p.dev[c.dev], c.handle);
              row->mem_bytes += c.a;
              L.held_mem += c.a;
              L.version += 1;
            }
            out->outcome = GS_OK;
          }
        }
        break;
      case OP_ASSIGN:
        if (tid == 0) {
          SLed &L = S.led[c.dev];
          gs_residency *row = entry(p.dev[c.dev], c.handle);
          row->mem_bytes += c.a;
          L.held_mem += c.a;
          L.version += 1;
          L.dirty = 1;
          out->outcome = GS_OK;
        }
        break;
      case OP_ADD_WARPS:
        if (tid == 0) {
          SLed &L = S.led[c.dev];
          gs_residency *row = entry(p.dev[c.dev], c.handle);
          row->warps += c.a;
          L.in_use_warps += c.a;
          L.held_warps += c.a;
          L.version += 1;
          L.dirty = 1;
          out->outcome = GS_OK;
        }
        break;
      case OP_TRY_PLACE:
        if (warp == 0) {
          const Shape sh = shape_of(c.probe);
          int *cap = scratch, *P = scratch + p.max_sm_pad;
          int cur = warp_plan(p.dev[c.dev], dyn, S.led[c.dev], sh, cap, P, lane);
          for (int s = lane; s < p.dev[c.dev].n_sm; s += 32) p.plan_io[s] = cur >= 0 ? P[s] : 0;
          if (lane == 0) {
            out->outcome = cur >= 0 ? GS_OK : GS_INFEASIBLE;
            out->device = cur;
            out->free_mem_after = S.led[c.dev].version;
          }
        }
        break;
      case OP_COMMIT:
        if (warp == 0) {
          SLed &L = S.led[c.dev];
          if (c.b != L.version) {
            if (lane == 0) {
              out->outcome = GS_ERR_CONTRACT;
              out->free_mem_after = L.version;
            }
          } else {
            const Shape sh = shape_of(c.probe);
            warp_commit(p.dev[c.dev], dyn, L, c.handle, sh, p.plan_io, (int)c.a, lane);
            if (lane == 0) out->outcome = GS_OK;
          }
        }
        break;
      case OP_CHECK: {
        // check_conservation (device_model.py:220-245)
        const KDev &D = p.dev[c.dev];
        const SLed &L = S.led[c.dev];
        if (tid == 0) {
          int k = GS_CHECK_OK;
          if (L.free_mem < 0 || L.free_mem + L.held_mem != D.spec.mem_bytes) k = GS_CHECK_MEM;
          else if (L.held_warps != L.in_use_warps) k = GS_CHECK_WARPS;
          S.chk = k ? -k : INT_MAX;
        }
        __syncthreads();
        if (S.chk == INT_MAX) {
          int *w = arr_warps(dyn, D), *t = arr_tbs(dyn, D), *r = arr_regs(dyn, D), *m = arr_smem(dyn, D);
          for (int s = tid; s < D.n_sm; s += kThreads) {
            int k = 0;
            if (!(t[s] >= 0 && t[s] <= D.spec.max_tbs_per_sm)) k = GS_CHECK_SM_TBS;
            else if (!(w[s] >= 0 && w[s] <= D.spec.max_warps_per_sm)) k = GS_CHECK_SM_WARPS;
            else if (!(r[s] >= 0 && r[s] <= D.spec.regs_per_sm)) k = GS_CHECK_SM_REGS;
            else if (!(m[s] >= 0 && m[s] <= D.spec.smem_per_sm_bytes)) k = GS_CHECK_SM_SMEM;
            if (k) atomicMin(&S.chk, s * 8 + k);
          }
        }
        __syncthreads();
        if (tid == 0) {
          int v = S.chk;
          if (v == INT_MAX) {
            out->outcome = GS_OK;
            out->device = 0;
            out->pending_index = -1;
          } else if (v < 0) {
            out->outcome = GS_ERR_CONTRACT;
            out->device = -v;
            out->pending_index = -1;
          } else {
            out->outcome = GS_ERR_CONTRACT;
            out->device = v & 7;
            out->pending_index = v >> 3;
          }
          out->free_mem_after = L.held_mem;
          out->in_use_warps_after = L.held_warps;
        }
        break;
      }
      default:
        if (tid == 0) out->outcome = GS_ERR_CONFIG;
        break;
    }
    __syncthreads();
  }

  // ---- write back dirty ledgers + scheduler state ----
  for (int d = 0; d < p.n_dev; ++d) {
    if (!S.led[d].dirty) continue;
    const KDev &D = p.dev[d];
    int32_t *dst = reinterpret_cast<int32_t *>(D.led + 1);
    const int *src = dyn + D.smem_off;
    for (int i = tid; i < 4 * D.arr_pad; i += kThreads) dst[i] = src[i];
    if (tid == 0) {
      gs_ledger *g = D.led;
      const SLed &L = S.led[d];
      g->free_mem = L.free_mem;
      g->in_use_warps = L.in_use_warps;
      g->version = L.version;
      g->held_mem = L.held_mem;
      g->held_warps = L.held_warps;
      g->rr_cursor = L.rr_cursor;
    }
  }
  if (tid == 0) *p.st = S.st;
  __threadfence_system();
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

thread_local std::string g_err;

int set_err(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return set_err(GS_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
struct Mapped {
  T *h = nullptr;
  T *d = nullptr;
  size_t n = 0;
  int alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    CU(cudaHostAlloc((void **)&h, count * sizeof(T), cudaHostAllocMapped | cudaHostAllocPortable));
    memset(h, 0, count * sizeof(T));
    CU(cudaHostGetDevicePointer((void **)&d, h, 0));
    n = count;
    return GS_OK;
  }
  void release() {
    if (h) cudaFreeHost(h);
    h = d = nullptr;
    n = 0;
  }
};

template <class T>
struct DevBuf {
  T *d = nullptr;
  size_t n = 0;
  int ensure(size_t count, cudaStream_t st, bool keep) {
    if (count <= n) return GS_OK;
    size_t nn = std::max(count, n * 2);
    T *nd = nullptr;
    CU(cudaMalloc((void **)&nd, nn * sizeof(T)));
    CU(cudaMemsetAsync(nd, 0, nn * sizeof(T), st));
    if (keep && d && n) CU(cudaMemcpyAsync(nd, d, n * sizeof(T), cudaMemcpyDeviceToDevice, st));
    CU(cudaStreamSynchronize(st));
    if (d) cudaFree(d);
    d = nd;
    n = nn;
    return GS_OK;
  }
  void release() {
    if (d) cudaFree(d);
    d = nullptr;
    n = 0;
  }
};

}  // namespace

struct gs_engine {
  int cuda_dev = 0;
  cudaStream_t stream = nullptr;
  std::recursive_mutex mu;
  int32_t res_cap = 0;
  std::vector<gs_device *> devices;
  Mapped<Cmd> cmds;
  Mapped<gs_decision> results;
  Mapped<int32_t> plan_io;
  Mapped<SchedState> dummy_state;
  DevBuf<Cmd> dcmds;
  int64_t launches = 0;
  int max_smem = 0;
};

struct gs_device {
  gs_engine *eng = nullptr;
  gs_spec spec{};
  int32_t index = 0;
  int32_t arr_pad = 0;
  int32_t stride = 0;
  Mapped<char> ledger;  // header + 4 arrays
  DevBuf<int32_t> res;
};

struct gs_sched {
  gs_engine *eng = nullptr;
  std::vector<gs_device *> devs;
  int32_t policy = 0, cg_ratio = 6, skip_ahead = 1;
  Mapped<SchedState> st;
  DevBuf<gs_probe> pend;
  DevBuf<int32_t> pend_flag;
  DevBuf<int32_t> claims;
  DevBuf<int32_t> fifo;
  DevBuf<int32_t> events;
  Mapped<gs_decision> drain;
};

namespace {

int pad4(int64_t n) { return (int)((n + 3) / 4 * 4); }

int grow_device_res(gs_device *dv, int32_t cap) {
  return dv->res.ensure((size_t)cap * dv->stride, dv->eng->stream, true);
}

struct Launch {
  KParams p{};
  size_t smem = 0;
};

int build_params(gs_engine *eng, gs_device *const *devs, int n, Launch &L) {
  if (n < 1 || n > GS_MAX_DEVICES) return set_err(GS_ERR_CONFIG, "fleet size must be 1..32");
  KParams &p = L.p;
  memset(&p, 0, sizeof(p));
  p.n_dev = n;
  int off = 0, max_pad = 0;
  for (int d = 0; d < n; ++d) {
    gs_device *dv = devs[d];
    KDev &k = p.dev[d];
    k.led = reinterpret_cast<gs_ledger *>(dv->ledger.d);
    k.res = dv->res.d;
    k.stride = dv->stride;
    k.n_sm = (int32_t)dv->spec.sm_count;
    k.arr_pad = dv->arr_pad;
    k.smem_off = off;
    k.spec = dv->spec;
    off += 4 * dv->arr_pad;
    max_pad = std::max(max_pad, dv->arr_pad);
  }
  p.max_sm_pad = max_pad;
  L.smem = (size_t)(off + kWarps * 2 * max_pad) * sizeof(int);
  if ((int)L.smem > eng->max_smem)
    return set_err(GS_ERR_CONFIG, "fleet ledgers exceed shared memory");
  p.st = eng->dummy_state.d;
  p.results = eng->results.d;
  p.plan_io = eng->plan_io.d;
  p.claims = nullptr;
  p.job_cap = 0;
  p.fifo_cap = 1;
  return GS_OK;
}

int launch(gs_engine *eng, Launch &L) {
  gs_interp_kernel<<<1, kThreads, L.smem, eng->stream>>>(L.p);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(eng->stream));
  eng->launches++;
  return GS_OK;
}

int ensure_cmds(gs_engine *eng, int n) {
  if ((size_t)n > eng->cmds.n) {
    int rc = eng->cmds.alloc(std::max<size_t>(n, eng->cmds.n * 2));
    if (rc) return rc;
  }
  if ((size_t)n > eng->results.n) {
    int rc = eng->results.alloc(std::max<size_t>(n, eng->results.n * 2));
    if (rc) return rc;
  }
  return GS_OK;
}

// Run `n` single-device commands on a one-device fleet.
int run_device_cmd(gs_device *dv, const Cmd &c, gs_decision *out) {
  gs_engine *eng = dv->eng;
  std::lock_guard<std::recursive_mutex> g(eng->mu);
  Launch L;
  gs_device *arr[1] = {dv};
  int rc = build_params(eng, arr, 1, L);
  if (rc) return rc;
  rc = ensure_cmds(eng, 1);
  if (rc) return rc;
  L.p.results = eng->results.d;
  eng->cmds.h[0] = c;
  eng->cmds.h[0].dev = 0;
  L.p.cmds = eng->cmds.d;
  L.p.n_cmds = 1;
  memset(eng->results.h, 0, sizeof(gs_decision));
  rc = launch(eng, L);
  if (rc) return rc;
  *out = eng->results.h[0];
  return GS_OK;
}

int sched_params(gs_sched *s, Launch &L) {
  int rc = build_params(s->eng, s->devs.data(), (int)s->devs.size(), L);
  if (rc) return rc;
  KParams &p = L.p;
  p.policy = s->policy;
  p.cg_ratio = s->cg_ratio;
  p.skip_ahead = s->skip_ahead;
  p.st = s->st.d;
  p.pend = s->pend.d;
  p.pend_cap = (int32_t)s->pend.n;
  p.pend_flag = s->pend_flag.d;
  p.claims = s->claims.d;
  p.job_cap = (int32_t)s->claims.n;
  p.drain_out = s->drain.d;
  p.drain_cap = (int32_t)s->drain.n;
  p.fifo = s->fifo.d;
  p.fifo_cap = std::max<int32_t>(1, (int32_t)(s->fifo.n / 2));
  return GS_OK;
}

int ensure_pending(gs_sched *s, int extra) {
  const size_t need = (size_t)s->st.h->pend_count + extra + 1;
  int rc = s->pend.ensure(need, s->eng->stream, true);
  if (rc) return rc;
  rc = s->pend_flag.ensure(need, s->eng->stream, false);
  if (rc) return rc;
  if (need > s->drain.n) {
    rc = s->drain.alloc(std::max(need, s->drain.n * 2));
    if (rc) return rc;
  }
  return GS_OK;
}

int ensure_jobs(gs_sched *s, int32_t job) {
  if (job < 0) return GS_OK;
  size_t old = s->claims.n;
  if ((size_t)job < old) return GS_OK;
  size_t nn = std::max<size_t>((size_t)job + 1, old * 2);
  int32_t *nd = nullptr;
  CU(cudaMalloc((void **)&nd, nn * sizeof(int32_t)));
  CU(cudaMemsetAsync(nd, 0xff, nn * sizeof(int32_t), s->eng->stream));  // -1
  if (old) CU(cudaMemcpyAsync(nd, s->claims.d, old * sizeof(int32_t), cudaMemcpyDeviceToDevice, s->eng->stream));
  CU(cudaStreamSynchronize(s->eng->stream));
  if (s->claims.d) cudaFree(s->claims.d);
  s->claims.d = nd;
  s->claims.n = nn;
  return GS_OK;
}

int check_handle(gs_engine *eng, int32_t h) {
  if (h < 0 || h >= eng->res_cap) return set_err(GS_ERR_CONFIG, "task handle out of range; reserve handles first");
  return GS_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

int gs_abi_version(void) { return GS_ABI_VERSION; }
const char *gs_last_error(void) { return g_err.c_str(); }

int gs_engine_open(int cuda_device, gs_engine **out) {
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return set_err(GS_ERR_CUDA, "no CUDA device visible: libgs has no CPU fallback");
  if (cuda_device < 0 || cuda_device >= count) return set_err(GS_ERR_CONFIG, "bad CUDA device index");
  CU(cudaSetDevice(cuda_device));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, cuda_device));
  if (prop.major < 10) return set_err(GS_ERR_CUDA, "libgs is built for sm_100a (B200)");
  auto *eng = new gs_engine();
  eng->cuda_dev = cuda_device;
  eng->max_smem = (int)prop.sharedMemPerBlockOptin - (int)sizeof(SmemStatic) - 2048;
  CU(cudaFuncSetAttribute(gs_interp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, eng->max_smem));
  CU(cudaStreamCreateWithFlags(&eng->stream, cudaStreamNonBlocking));
  int rc = eng->cmds.alloc(64);
  if (!rc) rc = eng->results.alloc(64);
  if (!rc) rc = eng->plan_io.alloc(4096);
  if (!rc) rc = eng->dummy_state.alloc(1);
  if (rc) {
    delete eng;
    return rc;
  }
  for (int d = 0; d < GS_MAX_DEVICES; ++d) eng->dummy_state.h->sa_owner[d] = -1;
  eng->res_cap = 0;
  *out = eng;
  return gs_engine_reserve_handles(eng, 256);
}

void gs_engine_close(gs_engine *eng) {
  if (!eng) return;
  cudaStreamSynchronize(eng->stream);
  eng->cmds.release();
  eng->results.release();
  eng->plan_io.release();
  eng->dummy_state.release();
  eng->dcmds.release();
  cudaStreamDestroy(eng->stream);
  delete eng;
}

int gs_engine_reserve_handles(gs_engine *eng, int32_t capacity) {
  std::lock_guard<std::recursive_mutex> g(eng->mu);
  if (capacity <= eng->res_cap) return GS_OK;
  int32_t cap = std::max(capacity, eng->res_cap * 2);
  for (gs_device *dv : eng->devices) {
    int rc = grow_device_res(dv, cap);
    if (rc) return rc;
  }
  eng->res_cap = cap;
  return GS_OK;
}

int32_t gs_engine_handle_capacity(gs_engine *eng) { return eng->res_cap; }
int64_t gs_engine_launches(gs_engine *eng) { return eng->launches; }

int gs_device_create(gs_engine *eng, const gs_spec *spec, int32_t index, gs_device **out) {
  std::lock_guard<std::recursive_mutex> g(eng->mu);
  *out = nullptr;
  if (spec->sm_count < 1 || spec->sm_count > 4096) return set_err(GS_ERR_CONFIG, "sm_count must be 1..4096");
  auto *dv = new gs_device();
  dv->eng = eng;
  dv->spec = *spec;
  dv->index = index;
  dv->arr_pad = pad4(spec->sm_count);
  dv->stride = pad4(kRowHdrWords + spec->sm_count);
  int rc = dv->ledger.alloc(sizeof(gs_ledger) + 4 * (size_t)dv->arr_pad * sizeof(int32_t));
  if (rc) {
    delete dv;
    return rc;
  }
  gs_ledger *L = reinterpret_cast<gs_ledger *>(dv->ledger.h);
  L->free_mem = spec->mem_bytes;
  L->sm_count = (int32_t)spec->sm_count;
  rc = grow_device_res(dv, eng->res_cap);
  if (rc) {
    dv->ledger.release();
    delete dv;
    return rc;
  }
  eng->devices.push_back(dv);
  *out = dv;
  return GS_OK;
}

void gs_device_destroy(gs_device *dv) {
  if (!dv) return;
  gs_engine *eng = dv->eng;
  std::lock_guard<std::recursive_mutex> g(eng->mu);
  eng->devices.erase(std::remove(eng->devices.begin(), eng->devices.end(), dv), eng->devices.end());
  dv->ledger.release();
  dv->res.release();
  delete dv;
}

gs_ledger *gs_device_ledger(gs_device *dv) { return reinterpret_cast<gs_ledger *>(dv->ledger.h); }

int32_t *gs_device_sm_array(gs_device *dv, int32_t which) {
  if (which < 0 || which > 3) return nullptr;
  int32_t *base = reinterpret_cast<int32_t *>(dv->ledger.h + sizeof(gs_ledger));
  return base + (size_t)which * dv->arr_pad;
}

int gs_try_place(gs_device *dv, const gs_probe *req, int32_t *blocks, int32_t *cursor, int64_t *version) {
  std::lock_guard<std::recursive_mutex> g(dv->eng->mu);
  if (dv->spec.sm_count > (int64_t)dv->eng->plan_io.n) return set_err(GS_ERR_CONFIG, "too many SMs");
  Cmd c{};
  c.op = OP_TRY_PLACE;
  c.probe = *req;
  gs_decision o{};
  int rc = run_device_cmd(dv, c, &o);
  if (rc) return rc;
  if (o.outcome != GS_OK) return GS_INFEASIBLE;
  if (blocks) memcpy(blocks, dv->eng->plan_io.h, sizeof(int32_t) * dv->spec.sm_count);
  if (cursor) *cursor = o.device;
  if (version) *version = o.free_mem_after;
  return GS_OK;
}

int gs_commit(gs_device *dv, int32_t handle, const gs_probe *req, const int32_t *blocks, int32_t cursor,
              int64_t plan_version) {
  std::lock_guard<std::recursive_mutex> g(dv->eng->mu);
  int rc = check_handle(dv->eng, handle);
  if (rc) return rc;
  memcpy(dv->eng->plan_io.h, blocks, sizeof(int32_t) * dv->spec.sm_count);
  Cmd c{};
  c.op = OP_COMMIT;
  c.handle = handle;
  c.a = cursor;
  c.b = plan_version;
  c.probe = *req;
  gs_decision o{};
  rc = run_device_cmd(dv, c, &o);
  if (rc) return rc;
  if (o.outcome == GS_ERR_CONTRACT) {
    char buf[160];
    snprintf(buf, sizeof buf, "placement plan is stale (device %d version %lld, plan version %lld)", dv->index,
             (long long)o.free_mem_after, (long long)plan_version);
    return set_err(GS_ERR_CONTRACT, buf);
  }
  return o.outcome;
}

static int simple_dev_op(gs_device *dv, int op, int32_t handle, int64_t a, gs_decision *o) {
  std::lock_guard<std::recursive_mutex> g(dv->eng->mu);
  if (op != OP_RESERVE && op != OP_CHECK) {
    int rc = check_handle(dv->eng, handle);
    if (rc) return rc;
  }
  Cmd c{};
  c.op = op;
  c.handle = handle;
  c.a = a;
  return run_device_cmd(dv, c, o);
}

int gs_reserve_memory(gs_device *dv, int64_t nbytes) {
  gs_decision o{};
  int rc = simple_dev_op(dv, OP_RESERVE, 0, nbytes, &o);
  return rc ? rc : o.outcome;
}
int gs_assign_memory(gs_device *dv, int32_t handle, int64_t nbytes) {
  gs_decision o{};
  int rc = simple_dev_op(dv, OP_ASSIGN, handle, nbytes, &o);
  return rc ? rc : o.outcome;
}
int gs_add_warps(gs_device *dv, int32_t handle, int64_t warps) {
  gs_decision o{};
  int rc = simple_dev_op(dv, OP_ADD_WARPS, handle, warps, &o);
  return rc ? rc : o.outcome;
}
int gs_allocate_raw(gs_device *dv, int32_t handle, int64_t nbytes) {
  gs_decision o{};
  int rc = simple_dev_op(dv, OP_ALLOC_RAW, handle, nbytes, &o);
  return rc ? rc : o.outcome;
}
int gs_release(gs_device *dv, int32_t handle, int64_t *freed) {
  gs_decision o{};
  int rc = simple_dev_op(dv, OP_RELEASE, handle, 0, &o);
  if (rc) return rc;
  if (o.outcome == GS_ERR_CONTRACT) return set_err(GS_ERR_CONTRACT, "release of unknown task");
  if (freed) *freed = o.free_mem_after;
  return GS_OK;
}
int gs_check_conservation(gs_device *dv, int32_t *kind, int32_t *sm, int64_t *held_mem, int64_t *held_warps) {
  gs_decision o{};
  int rc = simple_dev_op(dv, OP_CHECK, 0, 0, &o);
  if (rc) return rc;
  if (kind) *kind = o.outcome == GS_OK ? GS_CHECK_OK : o.device;
  if (sm) *sm = o.pending_index;
  if (held_mem) *held_mem = o.free_mem_after;
  if (held_warps) *held_warps = o.in_use_warps_after;
  return o.outcome == GS_OK ? GS_OK : set_err(GS_ERR_CONTRACT, "ledger conservation violated");
}

int gs_residency_read(gs_device *dv, int32_t handle, gs_residency *row, int32_t *blocks) {
  std::lock_guard<std::recursive_mutex> g(dv->eng->mu);
  int rc = check_handle(dv->eng, handle);
  if (rc) return rc;
  const int32_t *src = dv->res.d + (size_t)handle * dv->stride;
  CU(cudaMemcpyAsync(row, src, sizeof(gs_residency), cudaMemcpyDeviceToHost, dv->eng->stream));
  if (blocks)
    CU(cudaMemcpyAsync(blocks, src + kRowHdrWords, sizeof(int32_t) * dv->spec.sm_count, cudaMemcpyDeviceToHost,
                       dv->eng->stream));
  CU(cudaStreamSynchronize(dv->eng->stream));
  return GS_OK;
}

int gs_sched_create(gs_engine *eng, gs_device *const *devices, int32_t n, int32_t policy, int32_t cg_ratio,
                    int32_t skip_ahead, gs_sched **out) {
  std::lock_guard<std::recursive_mutex> g(eng->mu);
  *out = nullptr;
  if (n < 1 || n > GS_MAX_DEVICES) return set_err(GS_ERR_CONFIG, "fleet size must be 1..32");
  if (policy < GS_POLICY_SA || policy > GS_POLICY_MGB_WARPS) return set_err(GS_ERR_CONFIG, "unknown policy");
  if (policy == GS_POLICY_CG && cg_ratio < 1) return set_err(GS_ERR_CONFIG, "cg ratio must be >= 1");
  auto *s = new gs_sched();
  s->eng = eng;
  s->devs.assign(devices, devices + n);
  s->policy = policy;
  s->cg_ratio = cg_ratio;
  s->skip_ahead = skip_ahead;
  int rc = s->st.alloc(1);
  if (!rc) rc = s->drain.alloc(64);
  if (!rc) rc = s->pend.ensure(64, eng->stream, false);
  if (!rc) rc = s->pend_flag.ensure(64, eng->stream, false);
  if (!rc) rc = s->fifo.ensure(2, eng->stream, false);
  if (!rc) rc = ensure_jobs(s, 63);
  if (rc) {
    delete s;
    return rc;
  }
  for (int d = 0; d < GS_MAX_DEVICES; ++d) s->st.h->sa_owner[d] = -1;
  *out = s;
  return GS_OK;
}

void gs_sched_destroy(gs_sched *s) {
  if (!s) return;
  std::lock_guard<std::recursive_mutex> g(s->eng->mu);
  s->st.release();
  s->drain.release();
  s->pend.release();
  s->pend_flag.release();
  s->claims.release();
  s->fifo.release();
  s->events.release();
  delete s;
}

int gs_submit_batch(gs_sched *s, const gs_probe *reqs, int32_t n, gs_decision *out) {
  gs_engine *eng = s->eng;
  std::lock_guard<std::recursive_mutex> g(eng->mu);
  if (n <= 0) return GS_OK;
  int32_t maxh = -1, maxj = -1;
  for (int i = 0; i < n; ++i) {
    maxh = std::max(maxh, reqs[i].handle);
    maxj = std::max(maxj, reqs[i].job);
    if (reqs[i].handle < 0) return set_err(GS_ERR_CONFIG, "negative task handle");
  }
  int rc = gs_engine_reserve_handles(eng, maxh + 1);
  if (!rc) rc = ensure_jobs(s, maxj);
  if (!rc) rc = ensure_pending(s, n);
  if (!rc) rc = ensure_cmds(eng, n);
  if (rc) return rc;
  Launch L;
  rc = sched_params(s, L);
  if (rc) return rc;
  for (int i = 0; i < n; ++i) {
    Cmd &c = eng->cmds.h[i];
    memset(&c, 0, sizeof c);
    c.op = OP_SUBMIT;
    c.handle = reqs[i].handle;
    c.job = reqs[i].job;
    c.probe = reqs[i];
  }
  if (n > 32) {
    rc = eng->dcmds.ensure(n, eng->stream, false);
    if (rc) return rc;
    CU(cudaMemcpyAsync(eng->dcmds.d, eng->cmds.h, sizeof(Cmd) * n, cudaMemcpyHostToDevice, eng->stream));
    L.p.cmds = eng->dcmds.d;
  } else {
    L.p.cmds = eng->cmds.d;
  }
  L.p.n_cmds = n;
  L.p.results = eng->results.d;
  rc = launch(eng, L);
  if (rc) return rc;
  if (out) memcpy(out, eng->results.h, sizeof(gs_decision) * n);
  return GS_OK;
}

int gs_submit(gs_sched *s, const gs_probe *req, gs_decision *out) { return gs_submit_batch(s, req, 1, out); }

int gs_on_release(gs_sched *s, gs_decision *out, int32_t out_cap, int32_t *n_tried, int32_t *n_admitted) {
  gs_engine *eng = s->eng;
  std::lock_guard<std::recursive_mutex> g(eng->mu);
  int rc = ensure_pending(s, 0);
  if (!rc) rc = ensure_cmds(eng, 1);
  if (rc) return rc;
  Launch L;
  rc = sched_params(s, L);
  if (rc) return rc;
  Cmd &c = eng->cmds.h[0];
  memset(&c, 0, sizeof c);
  c.op = OP_ON_RELEASE;
  L.p.cmds = eng->cmds.d;
  L.p.n_cmds = 1;
  rc = launch(eng, L);
  if (rc) return rc;
  const int tried = s->st.h->n_tried, adm = s->st.h->n_admitted;
  if (n_tried) *n_tried = tried;
  if (n_admitted) *n_admitted = adm;
  if (out) memcpy(out, s->drain.h, sizeof(gs_decision) * std::min(tried, out_cap));
  return GS_OK;
}

int gs_job_ended(gs_sched *s, int32_t job) {
  gs_engine *eng = s->eng;
  std::lock_guard<std::recursive_mutex> g(eng->mu);
  int rc = ensure_jobs(s, job);
  if (!rc) rc = ensure_cmds(eng, 1);
  if (rc) return rc;
  Launch L;
  rc = sched_params(s, L);
  if (rc) return rc;
  Cmd &c = eng->cmds.h[0];
  memset(&c, 0, sizeof c);
  c.op = OP_JOB_ENDED;
  c.job = job;
  L.p.cmds = eng->cmds.d;
  L.p.n_cmds = 1;
  return launch(eng, L);
}

int32_t gs_pending_count(gs_sched *s) { return s->st.h->pend_count; }

int gs_sched_job_state(gs_sched *s, int32_t *sa_owner, int32_t *cg_counts, int32_t *cg_cursor) {
  const int n = (int)s->devs.size();
  for (int d = 0; d < n; ++d) {
    if (sa_owner) sa_owner[d] = s->st.h->sa_owner[d];
    if (cg_counts) cg_counts[d] = s->st.h->cg_counts[d];
  }
  if (cg_cursor) *cg_cursor = s->st.h->cg_cursor;
  return GS_OK;
}

int gs_sweep(gs_sched *s, const gs_probe *probes, int32_t n, int32_t max_resident, int32_t *events,
             int64_t events_cap, int64_t *n_events, float *kernel_ms) {
  gs_engine *eng = s->eng;
  std::lock_guard<std::recursive_mutex> g(eng->mu);
  if (n <= 0) return GS_OK;
  if (s->st.h->pend_count != 0 || s->st.h->fifo_tail != s->st.h->fifo_head)
    return set_err(GS_ERR_CONTRACT, "sweep needs a fresh scheduler");
  int rc = gs_engine_reserve_handles(eng, n);
  if (!rc) rc = ensure_pending(s, n);
  if (!rc) rc = s->fifo.ensure(2 * (size_t)n + 2, eng->stream, false);
  if (!rc) rc = s->events.ensure(3 * (size_t)std::max<int64_t>(events_cap, 1), eng->stream, false);
  if (rc) return rc;
  gs_probe *dprobes = nullptr;
  CU(cudaMalloc((void **)&dprobes, sizeof(gs_probe) * n));
  CU(cudaMemcpyAsync(dprobes, probes, sizeof(gs_probe) * n, cudaMemcpyHostToDevice, eng->stream));
  Launch L;
  rc = sched_params(s, L);
  if (rc) {
    cudaFree(dprobes);
    return rc;
  }
  L.p.sweep = 1;
  L.p.sweep_probes = dprobes;
  L.p.n_cmds = n;
  L.p.max_resident = max_resident;
  L.p.events = s->events.d;
  L.p.events_cap = events_cap;
  s->st.h->n_events = 0;
  s->st.h->fifo_head = s->st.h->fifo_tail = 0;
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  CU(cudaEventRecord(e0, eng->stream));
  gs_interp_kernel<<<1, kThreads, L.smem, eng->stream>>>(L.p);
  CU(cudaGetLastError());
  CU(cudaEventRecord(e1, eng->stream));
  CU(cudaStreamSynchronize(eng->stream));
  eng->launches++;
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (kernel_ms) *kernel_ms = ms;
  const int64_t ne = s->st.h->n_events;
  if (n_events) *n_events = ne;
  if (events)
    CU(cudaMemcpy(events, s->events.d, sizeof(int32_t) * 3 * std::min(ne, events_cap), cudaMemcpyDeviceToHost));
  cudaFree(dprobes);
  // the sweep's residents are bookkeeping of this run only
  s->st.h->fifo_head = s->st.h->fifo_tail = 0;
  return GS_OK;
}

}  // extern "C"
