// gs_sched.cu — B200-native ledger + placement engine (libgs).
//
// Replaces the reference's Python hot path:
//   DeviceState ledgers / try_place_blocks / commit   device_model.py:80-245
//   Scheduler.submit / on_release / job_ended         schedulers.py:89-123
//   _try_mgb_sm (Alg. 2) / _try_mgb_warps (Alg. 3)    schedulers.py:137-171
//   _try_sa / _try_cg / _impossible_everywhere        schedulers.py:173-199
//
// Design.  Decisions are a serial dependency chain (each
// ASSIGN mutates the ledgers the next decision reads), so the
// decision authority is ONE warp: no block barriers on the chain, all
// reductions are shuffles/ballots.  The warp stages every device ledger
// (free HBM, in-use warps, per-SM warps/TBs/regs/smem; 2.4 KB per 148-SM
// device, 19 KB for 8 x B200) into shared memory with 16-byte loads, runs a
// command stream in arrival order, and writes dirty ledgers back.
//   * mgb-warps: lane d scores device d: ballot(free_mem >= mem), then a
//     64-bit warp argmin over (in_use_warps, d).
//   * mgb-sm: devices in index order; per device the lanes compute per-SM
//     residual capacity over all SMs (warp-reduced); the first feasible
//     device commits through the closed-form round-robin water-fill of
//     SURVEY.md App. A (binary search on full rounds, ballot prefix ranks in
//     cursor order) instead of the reference's one-block-per-visit loop.
//   * on_release: only devices whose resources GREW since the scheduler's
//     last full pass can admit anything (pending requests were infeasible
//     everywhere at their last try, and resources otherwise only shrink), so
//     each pass scores pending probes against those devices only, first
//     with an O(1) aggregate-capacity bound (lane-parallel, 32 probes at a
//     time), then exactly, in FIFO order; admitted entries are compacted out
//     in place chunk by chunk.
// Residency rows (_Residency, device_model.py:69-77) live in HBM, indexed
// by the interned task handle; the rows a decision may touch are prefetched
// while the devices are being scored.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <stdio.h>
#include <stdlib.h>
#include <limits.h>
#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "gs_cache.h"
#include <algorithm>

#include "../../include/gs.h"

namespace {

constexpr int kThreads = 32;  // the decision chain runs on one warp
constexpr unsigned kFull = 0xffffffffu;
constexpr int kRowHdrWords = sizeof(gs_residency) / 4;  // 12
constexpr int kLedHdrWords = sizeof(gs_ledger) / 4;     // 16
static_assert(sizeof(gs_ledger) == 64, "ledger header must be 64 B");
static_assert(sizeof(gs_probe) == 64, "probe record must be 64 B");

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
  OP_STOP = 99,
};

struct Cmd {
  int32_t op, dev, handle, job;
  int64_t a, b;
  gs_probe probe;
};
static_assert(sizeof(Cmd) == 96, "command record is 96 B");

// Pinned host-mapped command ring of the persistent decision kernel
// (single producer: the host, under the engine mutex; single consumer: the
// decision warp).  tail / done are monotone command counters.
constexpr int kRingSlots = 64;
struct Ring {
  long long tail;
  long long pad0[7];
  long long done;
  long long pad1[7];
  int32_t alive;
  int32_t pad2[15];
  // globaltimer stamps of the last command (diagnostics, GS_RING_STAMPS):
  // [0] tail seen, [1] command read, [2] executed, [3] written back, [4] done published
  unsigned long long stamp[8];
  Cmd cmds[kRingSlots];
  gs_decision results[kRingSlots];
};

struct SchedState {  // pinned host-mapped
  int32_t sa_owner[GS_MAX_DEVICES];
  int32_t cg_counts[GS_MAX_DEVICES];
  int64_t seen_epoch[GS_MAX_DEVICES];
  int32_t cg_cursor;
  int32_t pend_count;
  int32_t fifo_head, fifo_tail;
  int32_t n_tried, n_admitted;
  int32_t error, pad;
  int64_t n_events;
};

struct KDev {
  gs_ledger *led;    // device pointer of the mapped ledger
  int32_t *res;      // residency rows in HBM
  int32_t stride;    // words per residency row
  int32_t n_sm;
  int32_t arr_pad;   // padded per-SM array length
  int32_t smem_off;  // int offset of this device's staged block in dyn smem
  int32_t fast;      // all spec per-SM limits < 2^22 (32-bit cap arithmetic)
  int32_t t_small;   // INT_MAX / n_sm: shapes with T <= this sum per-SM counts in 32 bits
  gs_spec spec;
};

struct KParams {
  int32_t n_dev, policy, cg_ratio, skip_ahead;
  int32_t n_cmds, max_sm_pad, max_resident, sweep;
  int32_t stage_q;   // int4 count of all staged ledger blocks
  int32_t scratch_off;
  int32_t fifo_off, fifo_cap, fifo_stride, sweep_fast;
  KDev dev[GS_MAX_DEVICES];
  SchedState *st;
  const Cmd *cmds;
  gs_decision *results;
  gs_decision *drain_out;
  int32_t drain_cap;
  int32_t pend_cap;
  gs_probe *pend;
  int32_t *claims;
  int32_t job_cap;
  int32_t pad;
  int32_t *plan_io;
  int32_t *events;
  int64_t events_cap;
  const gs_probe *sweep_probes;
  Ring *ring;
  long long ring_idle_ns;
  int ring_sleep_ns;  // poll interval of the idle decision warp
  int wb_mode;        // diagnostics (GS_RING_WB): 2 = system fence inside the per-command write-back
};

struct SLed {
  long long free_mem, in_use_warps, version, held_mem, held_warps, grow_epoch;
  int rr_cursor, dirty;  // dirty: bit 0 header changed, bit 1 per-SM arrays changed
};

struct Smem {
  SLed led[GS_MAX_DEVICES];
  // Σ over SMs of the positive residual (tbs, warps, regs, smem) per device:
  // an O(1) upper bound on the blocks a shape can still place there.
  // Maintained exactly while every SM's usage is within its limits
  // (agg_ok); recomputed at every launch.
  long long agg[GS_MAX_DEVICES][4];
  int agg_ok[GS_MAX_DEVICES];
  gs_probe cbuf[32];
  gs_probe cur;
  SchedState st;
  Cmd cmd;
};

struct Shape {
  long long mem, T, wpb, rpb, spb, tw;
  float iw, ir, is;  // reciprocals for the exact 32-bit division fast path
  bool fast;         // per-block amounts in [0, 2^22)
};

struct Dec {
  int outcome, dev;
};

constexpr long long kFastLim = 1LL << 22;

__device__ __forceinline__ Shape shape_of(const gs_probe &p) {
  Shape s;
  s.mem = p.mem_bytes;
  s.T = p.thread_blocks;
  s.wpb = p.warps_per_block;
  s.rpb = (long long)p.regs_per_thread * (long long)p.threads_per_block;
  s.spb = p.smem_per_block;
  s.tw = p.total_warps;
  s.fast = s.wpb >= 0 && s.wpb < kFastLim && s.rpb >= 0 && s.rpb < kFastLim && s.spb >= 0 && s.spb < kFastLim;
  s.iw = s.wpb > 0 ? 1.0f / (float)s.wpb : 0.f;
  s.ir = s.rpb > 0 ? 1.0f / (float)s.rpb : 0.f;
  s.is = s.spb > 0 ? 1.0f / (float)s.spb : 0.f;
  return s;
}

// floor(n / d) for 0 <= n < 2^22, 1 <= d < 2^22: float estimate (error < 1)
// corrected by one integer step each way — exact, ~8 instructions instead of
// an emulated 64-bit division.
__device__ __forceinline__ int fdiv(int n, int d, float inv) {
  int q = __float2int_rz(__int2float_rn(n) * inv);
  if (q * d > n) --q;
  else if ((q + 1) * d <= n) ++q;
  return q;
}

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ long long warp_min64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, (long long)__shfl_xor_sync(kFull, v, o));
  return v;
}

__device__ __forceinline__ unsigned all_mask(int n) { return n >= 32 ? kFull : ((1u << n) - 1u); }

// staged per-SM arrays: 0 warps, 1 tbs, 2 regs, 3 smem (ledger order)
__device__ __forceinline__ int *arr(int *dyn, const KDev &D, int which) {
  return dyn + D.smem_off + kLedHdrWords + which * D.arr_pad;
}

__device__ __forceinline__ int32_t *res_row(const KDev &D, int h) { return D.res + (size_t)h * D.stride; }

// Per-SM residual capacity for more blocks of this shape, clamped to T.
// _sm_admits (device_model.py:105-118) in closed form.
__device__ __forceinline__ int sm_cap(const KDev &D, int *dyn, int s, const Shape &sh) {
  const int w = arr(dyn, D, 0)[s], t = arr(dyn, D, 1)[s], r = arr(dyn, D, 2)[s], m = arr(dyn, D, 3)[s];
  if (D.fast && sh.fast && (w | t | r | m) >= 0) {
    // all residuals are below 2^22 here (spec < 2^22, usage >= 0)
    int c = (int)D.spec.max_tbs_per_sm - t;
    if (sh.wpb > 0) {
      const int num = (int)D.spec.max_warps_per_sm - w;
      c = min(c, num < 0 ? -1 : fdiv(num, (int)sh.wpb, sh.iw));
    } else if (w > (int)D.spec.max_warps_per_sm) {
      c = 0;
    }
    if (sh.rpb > 0) {
      const int num = (int)D.spec.regs_per_sm - r;
      c = min(c, num < 0 ? -1 : fdiv(num, (int)sh.rpb, sh.ir));
    }
    if (sh.spb > 0) {
      const int num = (int)D.spec.smem_per_sm_bytes - m;
      c = min(c, num < 0 ? -1 : fdiv(num, (int)sh.spb, sh.is));
    }
    c = max(c, 0);
    return (long long)c > sh.T ? (int)sh.T : c;
  }
  long long c = D.spec.max_tbs_per_sm - (long long)t;
  if (sh.wpb > 0) {
    long long num = D.spec.max_warps_per_sm - (long long)w;
    c = min(c, num < 0 ? -1LL : num / sh.wpb);
  } else if ((long long)w > D.spec.max_warps_per_sm) {
    c = 0;
  }
  if (sh.rpb > 0) {
    long long num = D.spec.regs_per_sm - (long long)r;
    c = min(c, num < 0 ? -1LL : num / sh.rpb);
  }
  if (sh.spb > 0) {
    long long num = D.spec.smem_per_sm_bytes - (long long)m;
    c = min(c, num < 0 ? -1LL : num / sh.spb);
  }
  if (c < 0) c = 0;
  if (c > sh.T) c = sh.T;
  return (int)c;
}

// Warp sum of per-SM block counts, each clamped to T: one redux.sync when
// n_sm * T fits in 31 bits (every partial and total sum does), else 64-bit
// shuffles.
__device__ __forceinline__ long long warp_sum_blocks(long long v, bool small) {
  return small ? (long long)__reduce_add_sync(kFull, (unsigned)v) : warp_sum64(v);
}
__device__ __forceinline__ bool blocks_small(const KDev &D, const Shape &sh) {
  return sh.T >= 0 && sh.T <= D.t_small;  // (a per-device constant: no division per reduction)
}

// Σ sm_cap over the device's SMs; also leaves every SM's cap in cap[] and
// the warp max in *mx for the warp_plan that follows an admission.
__device__ __forceinline__ long long warp_total_cap(const KDev &D, int *dyn, const Shape &sh, int *cap, int *mx,
                                                    int lane) {
  long long tot = 0;
  int m = 0;
  for (int s = lane; s < D.n_sm; s += 32) {
    const int c = sm_cap(D, dyn, s, sh);
    cap[s] = c;
    tot += c;
    m = max(m, c);
  }
  *mx = __reduce_max_sync(kFull, m);
  return warp_sum_blocks(tot, blocks_small(D, sh));
}

// occupancy_limit_per_sm (device_model.py:48-58) x sm_count.
__device__ __forceinline__ long long empty_capacity_blocks(const gs_spec &S, const Shape &sh) {
  long long lim = S.max_tbs_per_sm;
  if (sh.wpb > 0) lim = min(lim, S.max_warps_per_sm / sh.wpb);
  if (sh.rpb > 0) lim = min(lim, S.regs_per_sm / sh.rpb);
  if (sh.spb > 0) lim = min(lim, S.smem_per_sm_bytes / sh.spb);
  if (lim < 0) lim = 0;
  return lim * S.sm_count;
}

// _entry (device_model.py:211-216), single thread.
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

// ---- ledger staging -----------------------------------------------------


// Copy every staged ledger block mapped->smem (in) or smem->mapped (out,
// dirty devices only) with 16-byte accesses, 8 in flight per lane.  The
// loop runs per device (warp-uniform base pointers: the device table is a
// kernel parameter, and indexing it per lane with divergent devices
// serialized the constant-cache reads — a dirty 64 B header cost 24 us of
// per-command write-back in ring mode, tools/ring_bench.cpp).
__device__ void stage(const KParams &p, int *dyn, const Smem &S, bool in, int lane) {
  int4 *sm4 = reinterpret_cast<int4 *>(dyn);
  for (int d = 0; d < p.n_dev; ++d) {
    const int q0 = p.dev[d].smem_off >> 2;
    const int nq = (kLedHdrWords + 4 * p.dev[d].arr_pad) >> 2;
    int4 *g = reinterpret_cast<int4 *>(p.dev[d].led);
    int cnt = nq;
    if (!in) {
      // write-back: the 64 B header when it changed, the per-SM arrays only
      // when they did (mgb-warps never touches them: a 2.4 KB write-back over
      // PCIe per command became 64 B)
      const int dirty = S.led[d].dirty;
      cnt = (dirty & 2) ? nq : ((dirty & 1) ? 4 : 0);
    }
    for (int base = 0; base < cnt; base += 32 * 8) {
      int4 r[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int q = base + k * 32 + lane;
        if (q < cnt) {
          if (in) r[k] = g[q];
          else g[q] = sm4[q0 + q];
        }
      }
      if (in) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int q = base + k * 32 + lane;
          if (q < cnt) sm4[q0 + q] = r[k];
        }
      }
    }
  }
}

__device__ void led_from_stage(const KParams &p, int *dyn, Smem &S, int lane) {
  if (lane < p.n_dev) {
    const gs_ledger *g = reinterpret_cast<const gs_ledger *>(dyn + p.dev[lane].smem_off);
    SLed &L = S.led[lane];
    L.free_mem = g->free_mem;
    L.in_use_warps = g->in_use_warps;
    L.version = g->version;
    L.held_mem = g->held_mem;
    L.held_warps = g->held_warps;
    L.grow_epoch = g->grow_epoch;
    L.rr_cursor = g->rr_cursor;
    L.dirty = 0;
  }
  __syncwarp();
}

__device__ void led_to_stage(const KParams &p, int *dyn, Smem &S, int lane) {
  if (lane < p.n_dev && S.led[lane].dirty) {
    gs_ledger *g = reinterpret_cast<gs_ledger *>(dyn + p.dev[lane].smem_off);
    const SLed &L = S.led[lane];
    g->free_mem = L.free_mem;
    g->in_use_warps = L.in_use_warps;
    g->version = L.version;
    g->held_mem = L.held_mem;
    g->held_warps = L.held_warps;
    g->grow_epoch = L.grow_epoch;
    g->rr_cursor = L.rr_cursor;
  }
  __syncwarp();
}

// ---- placement plan / commit / release (one warp) ------------------------

// Closed-form round-robin placement == try_place_blocks
// (device_model.py:120-139).  Writes P[0..n) and returns the final cursor,
// or -1 when the blocks cannot fit (the reference's None).
// With caps_mx >= 0 the caller already left this shape's caps in cap[]
// (warp_total_cap, tot >= T) and caps_mx is their maximum.
__device__ int warp_plan(const KDev &D, int *dyn, const SLed &L, const Shape &sh, int *cap, int *P, int lane,
                         int caps_mx = -1) {
  const int n = D.n_sm;
  const bool small = blocks_small(D, sh);
  long long tot = sh.T;
  int mx = caps_mx;
  if (caps_mx < 0) {
    tot = 0;
    mx = 0;
    for (int s = lane; s < n; s += 32) {
      int c = sm_cap(D, dyn, s, sh);
      cap[s] = c;
      tot += c;
      mx = max(mx, c);
    }
    tot = warp_sum_blocks(tot, small);
    mx = __reduce_max_sync(kFull, mx);
  }
  __syncwarp();
  if (tot < sh.T) return -1;
  int c0 = L.rr_cursor % n;
  if (c0 < 0) c0 += n;
  if (sh.T <= 0) {
    for (int s = lane; s < n; s += 32) P[s] = 0;
    __syncwarp();
    return c0;
  }
  // largest k in [0, mx] with S(k) = sum min(cap, k) <= T  (full rounds)
  int lo = 0, hi = mx;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    long long sk = 0;
    for (int s = lane; s < n; s += 32) sk += min(cap[s], mid);
    sk = warp_sum_blocks(sk, small);
    if (sk <= sh.T) lo = mid; else hi = mid - 1;
  }
  const int k = lo;
  long long sk = 0;
  for (int s = lane; s < n; s += 32) {
    const int v = min(cap[s], k);
    P[s] = v;
    sk += v;
  }
  sk = warp_sum_blocks(sk, small);
  __syncwarp();
  const long long rem = sh.T - sk;
  int last = -1;
  long long run = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int base = 0; base < n; base += 32) {
    const int pos = base + lane;
    int s = c0 + pos;  // c0, pos < n: one conditional subtraction, not a modulo
    s = pos < n ? (s >= n ? s - n : s) : 0;
    bool q = false;
    if (pos < n) q = rem > 0 ? (cap[s] > k) : (cap[s] >= k);
    const unsigned b = __ballot_sync(kFull, q);
    if (rem > 0) {
      const long long rank = run + __popc(b & lt);
      if (q && rank < rem) {
        P[s] = k + 1;
        if (rank == rem - 1) last = s;
      }
      run += __popc(b);
      if (run >= rem) break;
    } else if (b) {
      last = c0 + base + 31 - __clz(b);
      last = last >= n ? last - n : last;
    }
  }
  last = __reduce_max_sync(kFull, last);
  __syncwarp();
  return (last + 1) % n;
}

// commit_placement's SM-array and block-row part (device_model.py:141-161).
// Also records Σ blocks in the row (for O(1) aggregate maintenance).
__device__ void warp_commit_blocks(const KDev &D, int *dyn, SLed &L, int h, const Shape &sh, const int *P,
                                   int cursor, int lane) {
  int32_t *blocks = res_row(D, h) + kRowHdrWords;
  int *w = arr(dyn, D, 0), *t = arr(dyn, D, 1), *r = arr(dyn, D, 2), *m = arr(dyn, D, 3);
  bool neg = false;
  int tot = 0;
  for (int s = lane; s < D.n_sm; s += 32) {
    const int c = P[s];
    blocks[s] = c;
    tot += c;
    if (c) {
      neg |= c < 0;
      t[s] += c;
      w[s] += (int)(c * sh.wpb);
      r[s] += (int)(c * sh.rpb);
      m[s] += (int)(c * sh.spb);
    }
  }
  neg = __any_sync(kFull, neg);
  tot = __reduce_add_sync(kFull, tot);
  if (lane == 0) {
    L.rr_cursor = cursor;
    L.version += 1;
    L.dirty |= 3;
    if (neg) L.grow_epoch += 1;
    reinterpret_cast<gs_residency *>(res_row(D, h))->thread_blocks = tot;
  }
  __syncwarp();
}

// commit_placement through the test API: _entry + blocks + header fields.
__device__ void warp_commit(const KDev &D, int *dyn, SLed &L, int h, const Shape &sh, const int *P, int cursor,
                            int lane) {
  if (lane == 0) {
    gs_residency *row = entry(D, h);
    row->has_blocks = 1;
    row->regs_per_block = sh.rpb;
    row->smem_per_block = sh.spb;
    row->warps_per_block = (int32_t)sh.wpb;
  }
  __syncwarp();
  warp_commit_blocks(D, dyn, L, h, sh, P, cursor, lane);
}

// Residency data of a release, from HBM or from the sweep's smem cache.
struct RelRow {
  long long mem, warps, rpb, spb;
  int present, has_blocks, wpb, T;
};

// Ledger side of release_task (device_model.py:192-209); c[k] holds the
// blocks of SMs lane + 32k (k < 8), SMs >= 256 are re-read from `rowp`.
__device__ void apply_release(const KDev &D, int *dyn, Smem &S, int d, const RelRow &rr, const int *c,
                              const int32_t *rowp, int lane) {
  SLed &L = S.led[d];
  const int n = D.n_sm;
  if (rr.has_blocks) {
    int *w = arr(dyn, D, 0), *t = arr(dyn, D, 1), *r = arr(dyn, D, 2), *m = arr(dyn, D, 3);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int s = lane + 32 * k;
      if (s < n && c[k]) {
        t[s] -= c[k];
        w[s] -= (int)((long long)c[k] * rr.wpb);
        r[s] -= (int)(c[k] * rr.rpb);
        m[s] -= (int)(c[k] * rr.spb);
      }
    }
    for (int s = lane + 256; s < n; s += 32) {  // devices with > 256 SMs
      const int cc = rowp[kRowHdrWords + s];
      if (cc) {
        t[s] -= cc;
        w[s] -= (int)((long long)cc * rr.wpb);
        r[s] -= (int)(cc * rr.rpb);
        m[s] -= (int)(cc * rr.spb);
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    L.free_mem += rr.mem;
    L.in_use_warps -= rr.warps;
    L.held_mem -= rr.mem;
    L.held_warps -= rr.warps;
    L.version += 1;
    L.grow_epoch += 1;
    L.dirty |= rr.has_blocks ? 3 : 1;
    if (rr.has_blocks && S.agg_ok[d]) {
      if (rr.wpb >= 0 && rr.rpb >= 0 && rr.spb >= 0) {
        S.agg[d][0] += rr.T;
        S.agg[d][1] += (long long)rr.T * rr.wpb;
        S.agg[d][2] += (long long)rr.T * rr.rpb;
        S.agg[d][3] += (long long)rr.T * rr.spb;
      } else {
        S.agg_ok[d] = 0;
      }
    }
    reinterpret_cast<gs_residency *>(const_cast<int32_t *>(rowp))->present = 0;
  }
  __syncwarp();
}

// release_task (device_model.py:192-209), one warp, one load round trip.
__device__ int warp_release(const KDev &D, int *dyn, Smem &S, int d, int h, long long *freed, int lane) {
  const int32_t *rowp = res_row(D, h);
  const int hw = lane < kRowHdrWords ? rowp[lane] : 0;
  int c[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int s = lane + 32 * k;
    c[k] = s < D.n_sm ? rowp[kRowHdrWords + s] : 0;
  }
  auto word = [&](int i) { return __shfl_sync(kFull, hw, i); };
  auto dword = [&](int i) {
    return (long long)(((unsigned long long)(unsigned)word(i + 1) << 32) | (unsigned)word(i));
  };
  RelRow rr;
  rr.present = word(8);
  rr.mem = dword(0);
  rr.warps = dword(2);
  rr.rpb = dword(4);
  rr.spb = dword(6);
  rr.has_blocks = word(9);
  rr.wpb = word(10);
  rr.T = word(11);
  if (!rr.present) return GS_ERR_CONTRACT;
  apply_release(D, dyn, S, d, rr, c, rowp, lane);
  *freed = rr.mem;
  return GS_OK;
}

// Σ positive residual per dimension for device d (kernel start).
__device__ void compute_agg(const KParams &p, int *dyn, Smem &S, int d, int lane) {
  const KDev &D = p.dev[d];
  long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  bool bad = false;
  for (int s = lane; s < D.n_sm; s += 32) {
    const long long w = arr(dyn, D, 0)[s], t = arr(dyn, D, 1)[s], r = arr(dyn, D, 2)[s], m = arr(dyn, D, 3)[s];
    bad |= t > D.spec.max_tbs_per_sm || w > D.spec.max_warps_per_sm || r > D.spec.regs_per_sm ||
           m > D.spec.smem_per_sm_bytes;
    a0 += max(0LL, D.spec.max_tbs_per_sm - t);
    a1 += max(0LL, D.spec.max_warps_per_sm - w);
    a2 += max(0LL, D.spec.regs_per_sm - r);
    a3 += max(0LL, D.spec.smem_per_sm_bytes - m);
  }
  a0 = warp_sum64(a0);
  a1 = warp_sum64(a1);
  a2 = warp_sum64(a2);
  a3 = warp_sum64(a3);
  bad = __any_sync(kFull, bad);
  if (lane == 0) {
    S.agg[d][0] = a0;
    S.agg[d][1] = a1;
    S.agg[d][2] = a2;
    S.agg[d][3] = a3;
    S.agg_ok[d] = !bad;
  }
  __syncwarp();
}

// O(1) necessary condition for T blocks of shape sh on device d:
// floor(A / x) >= T  <=>  A >= T * x  (no division).
__device__ __forceinline__ bool agg_admits(const Smem &S, int d, const Shape &sh) {
  if (!S.agg_ok[d] || sh.T <= 0) return true;
  if (S.agg[d][0] < sh.T) return false;
  if (sh.wpb > 0 && S.agg[d][1] < sh.T * sh.wpb) return false;
  if (sh.rpb > 0 && S.agg[d][2] < sh.T * sh.rpb) return false;
  if (sh.spb > 0 && S.agg[d][3] < sh.T * sh.spb) return false;
  return true;
}

// ---- decisions -------------------------------------------------------------

__device__ __forceinline__ void log_event(const KParams &p, Smem &S, int kind, int h, int d) {
  if (!p.events) return;
  const long long i = S.st.n_events++;
  if (i < p.events_cap) {
    p.events[3 * i] = kind;
    p.events[3 * i + 1] = h;
    p.events[3 * i + 2] = d;
  }
}

// Sweep mode: the resident FIFO lives in shared memory together with each
// resident task's residency data, so releasing the oldest task never waits
// on HBM.  Slot: [dev, handle, has_blocks, wpb, T, -, mem, warps, rpb, spb
// (int64 each)] + blocks[max_sm_pad].
constexpr int kSlotHdr = 14;

__device__ void fifo_push_slot(const KParams &p, Smem &S, int *dyn, int d, int h, const Shape &sh, long long mem,
                               long long warps, bool blocks, const int *P, int lane) {
  if (S.st.fifo_tail - S.st.fifo_head >= p.fifo_cap) {
    if (lane == 0) S.st.error = GS_ERR_NOMEM;
    __syncwarp();
    return;
  }
  int *slot = dyn + p.fifo_off + (S.st.fifo_tail % p.fifo_cap) * p.fifo_stride;
  if (blocks)
    for (int s = lane; s < p.dev[d].n_sm; s += 32) slot[kSlotHdr + s] = P[s];
  if (lane == 0) {
    slot[0] = d;
    slot[1] = h;
    slot[2] = blocks ? 1 : 0;
    slot[3] = (int)sh.wpb;
    slot[4] = (int)sh.T;
    long long *q = reinterpret_cast<long long *>(slot + 6);
    q[0] = mem;
    q[1] = warps;
    q[2] = blocks ? sh.rpb : 0;
    q[3] = blocks ? sh.spb : 0;
    S.st.fifo_tail++;
  }
  __syncwarp();
}

__device__ void fifo_pop_release(const KParams &p, Smem &S, int *dyn, int lane) {
  const int *slot = dyn + p.fifo_off + (S.st.fifo_head % p.fifo_cap) * p.fifo_stride;
  const int d = slot[0], h = slot[1];
  const KDev &D = p.dev[d];
  RelRow rr;
  rr.present = 1;
  rr.has_blocks = slot[2];
  rr.wpb = slot[3];
  rr.T = slot[4];
  const long long *q = reinterpret_cast<const long long *>(slot + 6);
  rr.mem = q[0];
  rr.warps = q[1];
  rr.rpb = q[2];
  rr.spb = q[3];
  int c[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int s = lane + 32 * k;
    c[k] = (rr.has_blocks && s < D.n_sm) ? slot[kSlotHdr + s] : 0;
  }
  apply_release(D, dyn, S, d, rr, c, res_row(D, h), lane);
  if (lane == 0) S.st.fifo_head++;
  __syncwarp();
}

// One admission attempt (Scheduler._try, schedulers.py:127-135) over the
// devices in `mask`.  Uniform result across the warp.
__device__ Dec decide(const KParams &p, Smem &S, int *dyn, const gs_probe &pr, unsigned mask, bool allow_reject,
                      int lane) {
  const int n_dev = p.n_dev;
  Dec out{GS_DEFER, -1};
  if (p.policy == GS_POLICY_MGB_WARPS || p.policy == GS_POLICY_MGB_SM) {
    const Shape sh = shape_of(pr);
    const int h = pr.handle;
    const bool fresh = (pr.level & GS_PROBE_FRESH) && (allow_reject || p.sweep);
    // prefetch the residency row this decision may accumulate into
    int r_present = 0;
    long long r_mem = 0, r_warps = 0;
    if (!fresh && lane < n_dev && ((mask >> lane) & 1)) {
      const gs_residency *row = reinterpret_cast<const gs_residency *>(res_row(p.dev[lane], h));
      r_present = row->present;
      r_mem = row->mem_bytes;
      r_warps = row->warps;
    }
    int chosen = -1, caps_mx = -1;
    if (p.policy == GS_POLICY_MGB_WARPS) {
      // _try_mgb_warps (schedulers.py:155-171): feasible = free_mem >= mem,
      // choose min((in_use_warps, idx))
      const bool ok = lane < n_dev && ((mask >> lane) & 1) && S.led[lane].free_mem >= sh.mem;
      if (__ballot_sync(kFull, ok)) {
        const long long key = ok ? S.led[lane].in_use_warps : LLONG_MAX;
        const long long m = warp_min64(key);
        chosen = __ffs(__ballot_sync(kFull, ok && key == m)) - 1;
      }
    } else {
      // _try_mgb_sm (schedulers.py:137-153): first device in index order
      // passing memory and per-SM placement.  Memory and the O(1)
      // aggregate bound are checked for all devices at once (lane d), the
      // exact per-SM count only for devices that pass both.
      const bool cand = lane < n_dev && ((mask >> lane) & 1) && S.led[lane].free_mem >= sh.mem &&
                        agg_admits(S, lane, sh);
      int *cap = dyn + p.scratch_off;
      for (unsigned m = __ballot_sync(kFull, cand); m; m &= m - 1) {
        const int d = __ffs(m) - 1;
        if (warp_total_cap(p.dev[d], dyn, sh, cap, &caps_mx, lane) >= sh.T) {
          chosen = d;
          break;
        }
      }
    }
    if (chosen < 0) {
      if (allow_reject) {
        // _impossible_everywhere (schedulers.py:191-199)
        bool possible = false;
        if (lane < n_dev) {
          const gs_spec &sp = p.dev[lane].spec;
          possible = !(sh.mem > sp.mem_bytes);
          if (p.policy == GS_POLICY_MGB_SM) possible = possible && !(empty_capacity_blocks(sp, sh) < sh.T);
        }
        if (!__ballot_sync(kFull, possible)) out.outcome = GS_REJECTED;
      }
      return out;
    }
    const int present = __shfl_sync(kFull, r_present, chosen);
    const long long pm = __shfl_sync(kFull, r_mem, chosen), pw = __shfl_sync(kFull, r_warps, chosen);
    const KDev &D = p.dev[chosen];
    SLed &L = S.led[chosen];
    gs_residency *row = reinterpret_cast<gs_residency *>(res_row(D, h));
    int *P = dyn + p.scratch_off + p.max_sm_pad;
    const bool sm_policy = p.policy == GS_POLICY_MGB_SM;
    if (sm_policy) {
      int *cap = dyn + p.scratch_off;
      const int cur = warp_plan(D, dyn, L, sh, cap, P, lane, caps_mx);
      warp_commit_blocks(D, dyn, L, h, sh, P, cur, lane);  // commit_placement
    }
    const long long new_mem = (present ? pm : 0) + sh.mem, new_warps = (present ? pw : 0) + sh.tw;
    if (lane == 0) {
      // commit header fields (mgb-sm), reserve_memory, assign_memory, add_warps
      row->mem_bytes = new_mem;
      row->warps = new_warps;
      if (sm_policy) {
        row->has_blocks = 1;
        row->regs_per_block = sh.rpb;
        row->smem_per_block = sh.spb;
        row->warps_per_block = (int32_t)sh.wpb;
        if (S.agg_ok[chosen]) {
          if (sh.wpb >= 0 && sh.rpb >= 0 && sh.spb >= 0) {
            S.agg[chosen][0] -= sh.T;
            S.agg[chosen][1] -= sh.T * sh.wpb;
            S.agg[chosen][2] -= sh.T * sh.rpb;
            S.agg[chosen][3] -= sh.T * sh.spb;
          } else {
            S.agg_ok[chosen] = 0;
          }
        }
      } else if (!present) {
        row->has_blocks = 0;
        row->regs_per_block = 0;
        row->smem_per_block = 0;
        row->warps_per_block = 0;
        row->thread_blocks = 0;
      }
      row->present = 1;
      L.free_mem -= sh.mem;
      L.held_mem += sh.mem;
      L.in_use_warps += sh.tw;
      L.held_warps += sh.tw;
      L.version += 3;
      L.dirty |= 1;
    }
    __syncwarp();
    if (p.sweep) fifo_push_slot(p, S, dyn, chosen, h, sh, new_mem, new_warps, sm_policy, P, lane);
    out.outcome = GS_ASSIGN;
    out.dev = chosen;
    return out;
  }
  int oc = GS_DEFER, dv = -1;
  if (lane == 0) {
    if (p.policy == GS_POLICY_SA) {
      // _try_sa (schedulers.py:173-178)
      for (int d = 0; d < n_dev; ++d) {
        if (S.st.sa_owner[d] < 0) {
          S.st.sa_owner[d] = pr.job;
          oc = GS_ASSIGN;
          dv = d;
          break;
        }
      }
    } else {
      // _try_cg (schedulers.py:180-189)
      for (int step = 0; step < n_dev; ++step) {
        const int d = (S.st.cg_cursor + step) % n_dev;
        if (S.st.cg_counts[d] < p.cg_ratio) {
          S.st.cg_counts[d] += 1;
          if (pr.job >= 0 && pr.job < p.job_cap) p.claims[pr.job] = d;
          S.st.cg_cursor = (d + 1) % n_dev;
          oc = GS_ASSIGN;
          dv = d;
          break;
        }
      }
    }
  }
  out.outcome = __shfl_sync(kFull, oc, 0);
  out.dev = __shfl_sync(kFull, dv, 0);
  __syncwarp();
  return out;
}

__device__ __forceinline__ void fill_decision(gs_decision &o, const Smem &S, int outcome, int d, int pidx,
                                              int h) {
  o.outcome = outcome;
  o.device = d;
  o.free_mem_after = d >= 0 ? S.led[d].free_mem : 0;
  o.in_use_warps_after = d >= 0 ? S.led[d].in_use_warps : 0;
  o.pending_index = pidx;
  o.handle = h;
}

// O(1) necessary condition for `pr` fitting one of the devices in `dirty`.
__device__ __forceinline__ bool bound_feasible(const KParams &p, const Smem &S, const gs_probe &pr, unsigned dirty) {
  const Shape sh = shape_of(pr);
  for (unsigned m = dirty; m; m &= m - 1) {
    const int d = __ffs(m) - 1;
    if (S.led[d].free_mem < sh.mem) continue;
    if (p.policy != GS_POLICY_MGB_SM || agg_admits(S, d, sh)) return true;
  }
  return false;
}

__device__ __forceinline__ void record_admit(const KParams &p, Smem &S, bool write_out, int i, const gs_probe &pr,
                                             Dec dc) {
  if (write_out && i < p.drain_cap) fill_decision(p.drain_out[i], S, dc.outcome, dc.dev, i, pr.handle);
  if (dc.outcome == GS_ASSIGN) log_event(p, S, 3, pr.handle, dc.dev);
}

// Scheduler.on_release (schedulers.py:97-113).
__device__ void on_release(const KParams &p, Smem &S, int *dyn, bool write_out, int lane) {
  const int P = S.st.pend_count;
  const bool mgb = p.policy == GS_POLICY_MGB_SM || p.policy == GS_POLICY_MGB_WARPS;
  const unsigned all = all_mask(p.n_dev);
  unsigned dirty = all;
  if (mgb) {
    const bool g = lane < p.n_dev && S.led[lane].grow_epoch != S.st.seen_epoch[lane];
    dirty = __ballot_sync(kFull, g);
  }
  const unsigned dmask = mgb ? dirty : all;
  if (mgb && !dirty && !write_out) {
    // no device's grow epoch moved since the last full pass: nothing pending
    // can fit (resources only shrank) — the pass below would try nothing
    // and keep the FIFO as is; skip reading it back from HBM
    if (lane == 0) {
      S.st.n_tried = P > 0 ? (p.skip_ahead ? P : 1) : 0;
      S.st.n_admitted = 0;
    }
    __syncwarp();
    return;
  }
  int w = 0, tried = 0, admitted = 0;
  bool stop = false;
  const unsigned lt = (1u << lane) - 1u;
  for (int base = 0; base < P; base += 32) {
    if (stop && w == base) {  // strict FIFO stopped and nothing moved: done
      w = P;
      break;
    }
    const int i = base + lane;
    const bool valid = i < P;
    const int cnt = min(32, P - base);
    gs_probe mine;
    if (valid) mine = p.pend[i];
    unsigned adm = 0;
    if (!stop) {
      const bool flag = valid && (!mgb || (dirty && bound_feasible(p, S, mine, dirty)));
      const unsigned fb = __ballot_sync(kFull, flag);
      if (valid) S.cbuf[lane] = mine;
      __syncwarp();
      if (p.skip_ahead) {
        if (write_out && valid && !flag && i < p.drain_cap)
          fill_decision(p.drain_out[i], S, GS_DEFER, -1, i, mine.handle);
        for (unsigned m = fb; m; m &= m - 1) {
          const int j = __ffs(m) - 1;
          const Dec dc = decide(p, S, dyn, S.cbuf[j], dmask, false, lane);
          if (lane == 0) record_admit(p, S, write_out, base + j, S.cbuf[j], dc);
          if (dc.outcome == GS_ASSIGN) adm |= 1u << j;
          __syncwarp();
        }
        tried = base + cnt;
      } else {
        for (int j = 0; j < cnt; ++j) {
          Dec dc{GS_DEFER, -1};
          if ((fb >> j) & 1) dc = decide(p, S, dyn, S.cbuf[j], dmask, false, lane);
          if (lane == 0) record_admit(p, S, write_out, base + j, S.cbuf[j], dc);
          __syncwarp();
          tried = base + j + 1;
          if (dc.outcome == GS_ASSIGN) {
            adm |= 1u << j;
          } else {
            stop = true;
            break;
          }
        }
      }
    }
    // in-place stable compaction of the survivors of this chunk
    const bool keep = valid && !((adm >> lane) & 1);
    const unsigned kb = __ballot_sync(kFull, keep);
    if ((w != base || adm) && keep) p.pend[w + __popc(kb & lt)] = mine;
    w += __popc(kb);
    admitted += __popc(adm);
    __syncwarp();
  }
  if (lane == 0) {
    S.st.pend_count = w;
    S.st.n_tried = tried;
    S.st.n_admitted = admitted;
  }
  if (mgb && !stop && lane < p.n_dev) S.st.seen_epoch[lane] = S.led[lane].grow_epoch;
  __syncwarp();
}

__device__ Dec submit(const KParams &p, Smem &S, int *dyn, const gs_probe &pr, gs_decision *out, int lane) {
  const Dec dc = decide(p, S, dyn, pr, all_mask(p.n_dev), true, lane);
  const int pc = S.st.pend_count;
  if (dc.outcome == GS_DEFER && pc < p.pend_cap && lane < 16)
    reinterpret_cast<int32_t *>(p.pend + pc)[lane] = reinterpret_cast<const int32_t *>(&pr)[lane];
  __syncwarp();
  if (lane == 0) {
    if (dc.outcome == GS_DEFER) S.st.pend_count = pc + 1;
    log_event(p, S, dc.outcome == GS_ASSIGN ? 0 : (dc.outcome == GS_DEFER ? 1 : 2), pr.handle, dc.dev);
    if (out) fill_decision(*out, S, dc.outcome, dc.dev, -1, pr.handle);
  }
  __syncwarp();
  return dc;
}

// One command of the interpreter (all lanes).
__device__ void exec_cmd(const KParams &p, Smem &S, int *dyn, const Cmd &c, gs_decision *out, int lane) {
  switch (c.op) {
    case OP_SUBMIT:
      submit(p, S, dyn, c.probe, out, lane);
      break;
    case OP_ON_RELEASE:
      on_release(p, S, dyn, true, lane);
      if (lane == 0) {
        out->outcome = GS_OK;
        out->free_mem_after = S.st.n_tried;
        out->in_use_warps_after = S.st.n_admitted;
      }
      break;
    case OP_JOB_ENDED:
      // job_ended (schedulers.py:115-123)
      if (lane == 0) {
        for (int d = 0; d < p.n_dev; ++d)
          if (S.st.sa_owner[d] == c.job) S.st.sa_owner[d] = -1;
        if (p.policy == GS_POLICY_CG && c.job >= 0 && c.job < p.job_cap) {
          const int d = p.claims[c.job];
          if (d >= 0) {
            S.st.cg_counts[d] -= 1;
            p.claims[c.job] = -1;
          }
        }
        out->outcome = GS_OK;
      }
      break;
    case OP_RELEASE: {
      long long freed = 0;
      const int rc = warp_release(p.dev[c.dev], dyn, S, c.dev, c.handle, &freed, lane);
      if (lane == 0) {
        out->outcome = rc;
        out->free_mem_after = freed;
      }
      break;
    }
    case OP_RESERVE:
    case OP_ALLOC_RAW:
      // reserve_memory (device_model.py:169-174) / allocate_raw (:185-190)
      if (lane == 0) {
        SLed &L = S.led[c.dev];
        if (c.a > L.free_mem) {
          out->outcome = GS_INFEASIBLE;
        } else {
          L.free_mem -= c.a;
          L.version += 1;
          L.dirty |= 1;
          if (c.a < 0) L.grow_epoch += 1;
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
      if (lane == 0) {
        SLed &L = S.led[c.dev];
        gs_residency *row = entry(p.dev[c.dev], c.handle);
        row->mem_bytes += c.a;
        L.held_mem += c.a;
        L.version += 1;
        L.dirty |= 1;
        out->outcome = GS_OK;
      }
      break;
    case OP_ADD_WARPS:
      if (lane == 0) {
        SLed &L = S.led[c.dev];
        gs_residency *row = entry(p.dev[c.dev], c.handle);
        row->warps += c.a;
        L.in_use_warps += c.a;
        L.held_warps += c.a;
        L.version += 1;
        L.dirty |= 1;
        out->outcome = GS_OK;
      }
      break;
    case OP_TRY_PLACE: {
      const Shape sh = shape_of(c.probe);
      int *cap = dyn + p.scratch_off, *P = cap + p.max_sm_pad;
      const int cur = warp_plan(p.dev[c.dev], dyn, S.led[c.dev], sh, cap, P, lane);
      for (int s = lane; s < p.dev[c.dev].n_sm; s += 32) p.plan_io[s] = cur >= 0 ? P[s] : 0;
      if (lane == 0) {
        out->outcome = cur >= 0 ? GS_OK : GS_INFEASIBLE;
        out->device = cur;
        out->free_mem_after = S.led[c.dev].version;
      }
      break;
    }
    case OP_COMMIT: {
      SLed &L = S.led[c.dev];
      if (c.b != L.version) {
        if (lane == 0) {
          out->outcome = GS_ERR_CONTRACT;
          out->free_mem_after = L.version;
        }
      } else {
        const Shape sh = shape_of(c.probe);
        warp_commit(p.dev[c.dev], dyn, L, c.handle, sh, p.plan_io, (int)c.a, lane);
        if (lane == 0) {
          out->outcome = GS_OK;
          S.agg_ok[c.dev] = 0;  // arbitrary plans: stop trusting the bound
        }
      }
      break;
    }
    case OP_CHECK: {
      // check_conservation (device_model.py:220-245), first violation
      const KDev &D = p.dev[c.dev];
      const SLed &L = S.led[c.dev];
      int k = GS_CHECK_OK, sm = -1;
      if (L.free_mem < 0 || L.free_mem + L.held_mem != D.spec.mem_bytes) k = GS_CHECK_MEM;
      else if (L.held_warps != L.in_use_warps) k = GS_CHECK_WARPS;
      if (k == GS_CHECK_OK) {
        int best = INT_MAX;
        const int *w = arr(dyn, D, 0), *t = arr(dyn, D, 1), *r = arr(dyn, D, 2), *m = arr(dyn, D, 3);
        for (int s = lane; s < D.n_sm && best == INT_MAX; s += 32) {
          int kk = 0;
          if (!(t[s] >= 0 && t[s] <= D.spec.max_tbs_per_sm)) kk = GS_CHECK_SM_TBS;
          else if (!(w[s] >= 0 && w[s] <= D.spec.max_warps_per_sm)) kk = GS_CHECK_SM_WARPS;
          else if (!(r[s] >= 0 && r[s] <= D.spec.regs_per_sm)) kk = GS_CHECK_SM_REGS;
          else if (!(m[s] >= 0 && m[s] <= D.spec.smem_per_sm_bytes)) kk = GS_CHECK_SM_SMEM;
          if (kk) best = s * 8 + kk;
        }
        best = __reduce_min_sync(kFull, best);
        if (best != INT_MAX) {
          k = best & 7;
          sm = best >> 3;
        }
      }
      if (lane == 0) {
        out->outcome = k == GS_CHECK_OK ? GS_OK : GS_ERR_CONTRACT;
        out->device = k;
        out->pending_index = sm;
        out->free_mem_after = L.held_mem;
        out->in_use_warps_after = L.held_warps;
      }
      break;
    }
    default:
      if (lane == 0) out->outcome = GS_ERR_CONFIG;
      break;
  }
  __syncwarp();
}

// Write dirty ledgers and the scheduler state back to mapped memory.
__device__ void writeback(const KParams &p, int *dyn, Smem &S, int lane, bool fence = true) {
  led_to_stage(p, dyn, S, lane);
  stage(p, dyn, S, false, lane);
  // every lane must have read the dirty flags (inside stage) before any lane
  // clears them — otherwise a fast lane 0 clears device d's flag while other
  // lanes still have d's chunks to write and they skip them
  __syncwarp();
  const int nw = sizeof(SchedState) / 4;
  for (int i = lane; i < nw; i += 32)
    reinterpret_cast<int32_t *>(p.st)[i] = reinterpret_cast<const int32_t *>(&S.st)[i];
  if (lane < p.n_dev) S.led[lane].dirty = 0;
  if (fence) __threadfence_system();
  __syncwarp();
}

__device__ __forceinline__ long long ld_acquire_sys(const long long *a) {
  long long v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(long long *a, long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Specialised mgb-warps sweep (BASELINE cfg 4).  The same decisions as
// submit / fifo_pop_release / on_release above, for the case the sweep
// stream is built of: fresh probes and an empty pending FIFO.  Lane d holds
// device d's ledger header in registers; _try_mgb_warps
// (schedulers.py:155-171: feasible = free_mem >= mem, choose
// min((in_use_warps, idx))) is one redux.sync min over the packed 32-bit
// key (in_use_warps << 5 | d), exact while every in_use_warps is in
// [0, 2^26); release_task (device_model.py:192-209) is a lane-local update.
// Only that chain is serial: the events and residency rows of a batch of 32
// probes are written afterwards, one lane per probe, while the next batch
// streams in from HBM.  The chain hands over to the general path, with
// identical state, at the first probe it does not cover (not fresh,
// deferred, a full resident FIFO, or a key out of range) and returns that
// probe's index.
constexpr long long kKeyLim = 1LL << 26;

__device__ int sweep_warps_fast(const KParams &p, Smem &S, int *dyn, int lane) {
  __shared__ long long q_mem[33], q_tw[33];
  __shared__ int q_h[33], q_lv[33];
  __shared__ int q_dev[32], q_rd[32], q_rh[32];  // decision, released (dev, handle)
  __shared__ int32_t *q_res[GS_MAX_DEVICES];
  __shared__ int q_stride[GS_MAX_DEVICES];
  const int n = p.n_cmds, nd = p.n_dev;
  const bool mine = lane < nd;
  if (mine) {
    q_res[lane] = p.dev[lane].res;
    q_stride[lane] = p.dev[lane].stride;
  }
  const long long cap = mine ? p.dev[lane].spec.mem_bytes : 0;
  long long fr = mine ? S.led[lane].free_mem : 0, iu = mine ? S.led[lane].in_use_warps : 0;
  const long long fr0 = fr, iu0 = iu;
  int nas = 0, nrel = 0;
  bool released = false;
  int head = S.st.fifo_head, tail = S.st.fifo_tail;
  int hs = head % p.fifo_cap, ts = tail % p.fifo_cap;
  long long ne = S.st.n_events;
  int stop_at = n;
  int *const fifo = dyn + p.fifo_off;
  const int fst = p.fifo_stride;
  const int32_t *src = reinterpret_cast<const int32_t *>(p.sweep_probes);
  // probe words: mem_bytes 0-1, total_warps 4-5, handle 13, level 15
  long long r_mem = 0, r_tw = 0;
  int r_h = 0, r_lv = 0;
  if (lane < n) {
    const int32_t *w = src + 16 * lane;
    r_mem = *reinterpret_cast<const long long *>(w);
    r_tw = *reinterpret_cast<const long long *>(w + 4);
    r_h = w[13];
    r_lv = w[15];
  }
  if (lane == 0) {  // sentinel after the last probe of a batch
    q_mem[32] = 0;
    q_tw[32] = 0;
    q_h[32] = 0;
    q_lv[32] = GS_PROBE_FRESH;
  }
  for (int base = 0; base < n && stop_at == n; base += 32) {
    __syncwarp();
    q_mem[lane] = r_mem;
    q_tw[lane] = r_tw;
    q_h[lane] = r_h;
    q_lv[lane] = r_lv;
    q_dev[lane] = -1;
    q_rd[lane] = -1;
    __syncwarp();
    const int nx = base + 32 + lane;  // next batch: loads in flight while this one is decided
    if (nx < n) {
      const int32_t *w = src + 16 * (size_t)nx;
      r_mem = *reinterpret_cast<const long long *>(w);
      r_tw = *reinterpret_cast<const long long *>(w + 4);
      r_h = w[13];
      r_lv = w[15];
    }
    // batch-level guards instead of per-probe ones: the chain covers the
    // probes before the first non-fresh one, and only while every key stays
    // packable — in_use_warps < 2^25 now and each total_warps < 2^20, so
    // 32 assignments keep it below 2^26 (releases only lower it)
    int cnt = min(32, n - base);
    {
      const unsigned nf = __ballot_sync(kFull, lane < cnt && (!(q_lv[lane] & GS_PROBE_FRESH) || q_tw[lane] < 0 ||
                                                              q_tw[lane] >= (1LL << 20)));
      if (nf) cnt = __ffs(nf) - 1;
      if (!__all_sync(kFull, !mine || (iu >= 0 && iu < (kKeyLim >> 1)))) cnt = 0;
    }
    const int full = min(32, n - base);
    int j = 0;
    long long mem = q_mem[0], tw = q_tw[0];
    int h = q_h[0];
    // the oldest resident's slot, read ahead of the push that may precede its pop
    int o_d = fifo[hs * fst], o_h = fifo[hs * fst + 1];
    long long o_m = *reinterpret_cast<const long long *>(fifo + hs * fst + 6);
    long long o_w = *reinterpret_cast<const long long *>(fifo + hs * fst + 8);
    for (; j < cnt; ++j) {
      const long long n_mem = q_mem[j + 1], n_tw = q_tw[j + 1];  // next probe, ahead of use
      const int n_h = q_h[j + 1];
      const bool ok = mine && fr >= mem;
      const unsigned m = __reduce_min_sync(kFull, ok ? ((unsigned)iu << 5) | (unsigned)lane : 0xffffffffu);
      if (m == 0xffffffffu) {
        if (__any_sync(kFull, mine && !(mem > cap))) break;  // deferred: the general path queues it
        // _impossible_everywhere: rejected (q_dev stays -1)
      } else {
        if (tail - head >= p.fifo_cap) break;  // the general path flags the overflow
        const int best = (int)(m & 31u);
        // assign (reserve_memory, assign_memory, add_warps)
        if (lane == best) {
          fr -= mem;
          iu += tw;
          ++nas;
        }
        if (lane == 0) {
          int *slot = fifo + ts * fst;
          slot[0] = best;
          slot[1] = h;
          slot[2] = 0;
          reinterpret_cast<long long *>(slot + 6)[0] = mem;
          reinterpret_cast<long long *>(slot + 6)[1] = tw;
          q_dev[j] = best;
        }
        if (ts == hs) {  // the FIFO was empty: the oldest resident is this task
          o_d = best;
          o_h = h;
          o_m = mem;
          o_w = tw;
        }
        ++tail;
        if (++ts == p.fifo_cap) ts = 0;
        if (tail - head > p.max_resident) {
          // release the oldest resident task, then on_release over an empty
          // pending FIFO (it only records the grow epochs)
          if (lane == o_d) {
            fr += o_m;
            iu -= o_w;
            ++nrel;
          }
          if (lane == 0) {
            q_rd[j] = o_d;
            q_rh[j] = o_h;
          }
          ++head;
          if (++hs == p.fifo_cap) hs = 0;
          released = true;
          __syncwarp();
          o_d = fifo[hs * fst];
          o_h = fifo[hs * fst + 1];
          o_m = *reinterpret_cast<const long long *>(fifo + hs * fst + 6);
          o_w = *reinterpret_cast<const long long *>(fifo + hs * fst + 8);
        }
      }
      mem = n_mem;
      tw = n_tw;
      h = n_h;
    }
    if (j < full) stop_at = base + j;
    __syncwarp();
    // this batch's outputs, one lane per probe: events, assigned rows, then
    // the released rows (ordered after the assignments by the warp barrier)
    if (lane < j) {
      const int d = q_dev[lane];
      const long long e = ne + lane;
      if (e < p.events_cap) {
        p.events[3 * e] = d >= 0 ? 0 : 2;
        p.events[3 * e + 1] = q_h[lane];
        p.events[3 * e + 2] = d;
      }
      if (d >= 0) {
        long long *row = reinterpret_cast<long long *>(q_res[d] + (size_t)q_h[lane] * q_stride[d]);
        row[0] = q_mem[lane];  // mem_bytes
        row[1] = q_tw[lane];   // warps
        row[2] = 0;            // regs_per_block
        row[3] = 0;            // smem_per_block
        row[4] = 1;            // present = 1, has_blocks = 0
        row[5] = 0;            // warps_per_block, thread_blocks
      }
    }
    __syncwarp();
    if (lane < j && q_rd[lane] >= 0) {
      const int d = q_rd[lane];
      reinterpret_cast<gs_residency *>(q_res[d] + (size_t)q_rh[lane] * q_stride[d])->present = 0;
    }
    ne += j;
  }
  __syncwarp();
  // hand the chain's state back to the shared ledgers
  if (mine) {
    SLed &L = S.led[lane];
    L.free_mem = fr;
    L.in_use_warps = iu;
    L.held_mem += fr0 - fr;
    L.held_warps += iu - iu0;
    L.version += 3LL * nas + nrel;
    L.grow_epoch += nrel;
    if (nas | nrel) L.dirty |= 1;
    if (released) S.st.seen_epoch[lane] = L.grow_epoch;
  }
  if (lane == 0) {
    if (released) {
      S.st.n_tried = 0;
      S.st.n_admitted = 0;
    }
    S.st.fifo_head = head;
    S.st.fifo_tail = tail;
    S.st.n_events = ne;
  }
  __syncwarp();
  return stop_at;
}

__global__ void __launch_bounds__(kThreads, 1) gs_interp_kernel(KParams p) {
  extern __shared__ __align__(16) int dyn[];
  __shared__ Smem S;
  const int lane = threadIdx.x;

  stage(p, dyn, S, true, lane);
  __syncwarp();
  led_from_stage(p, dyn, S, lane);
  {
    const int nw = sizeof(SchedState) / 4;
    for (int i = lane; i < nw; i += 32)
      reinterpret_cast<int32_t *>(&S.st)[i] = reinterpret_cast<const int32_t *>(p.st)[i];
  }
  __syncwarp();
  for (int d = 0; d < p.n_dev; ++d) compute_agg(p, dyn, S, d, lane);

  if (p.sweep) {
    // placement sweep (BASELINE cfg 4): submit probe i; then, if more than
    // max_resident tasks are resident or requests are queued, release the
    // oldest resident task and re-drive the FIFO.
    const int32_t *src = reinterpret_cast<const int32_t *>(p.sweep_probes);
    int ci0 = 0;
    if (p.sweep_fast && p.policy == GS_POLICY_MGB_WARPS) ci0 = sweep_warps_fast(p, S, dyn, lane);
    int nextw = (lane < 16 && ci0 < p.n_cmds) ? src[16 * ci0 + lane] : 0;
    for (int ci = ci0; ci < p.n_cmds; ++ci) {
      if (lane < 16) reinterpret_cast<int32_t *>(&S.cur)[lane] = nextw;
      __syncwarp();
      if (lane < 16 && ci + 1 < p.n_cmds) nextw = src[16 * (ci + 1) + lane];  // prefetch next probe
      submit(p, S, dyn, S.cur, nullptr, lane);
      const int resident = S.st.fifo_tail - S.st.fifo_head;
      if (resident > p.max_resident || S.st.pend_count > 0) {
        if (resident > 0) fifo_pop_release(p, S, dyn, lane);
        on_release(p, S, dyn, false, lane);
      }
      if (S.st.error) break;
    }
  } else if (p.ring) {
    // Persistent mode: poll the pinned host-mapped command ring; ledgers
    // stay in shared memory between commands, dirty ones are written back
    // after every command so host reads stay current.
    Ring *ring = p.ring;
    long long processed = ring->done;
    for (;;) {
      long long t = 0;
      if (lane == 0) {
        const unsigned long long t0 = globaltimer();
        // each poll is an acquire load of the tail: the command reads are
        // ordered after the poll that saw it (one PCIe round trip fewer than
        // relaxed polling + a separate acquire)
        while ((t = ld_acquire_sys(&ring->tail)) <= processed) {
          __nanosleep(p.ring_sleep_ns);
          if (globaltimer() - t0 > (unsigned long long)p.ring_idle_ns) {
            t = -1;
            break;
          }
        }
      }
      unsigned long long ts[5];
      ts[0] = globaltimer();
      t = __shfl_sync(kFull, t, 0);
      if (t < 0) break;  // idle watchdog: the host relaunches on demand
      const int slot = (int)(processed % kRingSlots);
      if (lane < (int)(sizeof(Cmd) / 4))
        reinterpret_cast<int32_t *>(&S.cmd)[lane] =
            reinterpret_cast<const volatile int32_t *>(ring->cmds + slot)[lane];
      __syncwarp();
      ts[1] = globaltimer();
      if (S.cmd.op == OP_STOP) {
        processed++;
        break;
      }
      exec_cmd(p, S, dyn, S.cmd, ring->results + slot, lane);
      ts[2] = globaltimer();
      // no system fence here: lane 0's st.release.sys of `done` below is
      // cumulative over the write-back the warp made before the __syncwarp
      // ending writeback(), so the host sees ledgers and results first
      // (GS_RING_WB=2 restores the fence, for measurement)
      writeback(p, dyn, S, lane, p.wb_mode == 2);
      ts[3] = globaltimer();
      processed++;
      if (lane == 0) st_release_sys(&ring->done, processed);
      ts[4] = globaltimer();
      if (lane == 0)  // lane 0's clock readings (the other lanes skip the poll loop)
        for (int k = 0; k < 5; ++k) ring->stamp[k] = ts[k];
      __syncwarp();
    }
    writeback(p, dyn, S, lane);
    if (lane == 0) {
      ring->alive = 0;
      st_release_sys(&ring->done, processed);
    }
    return;
  } else {
    for (int ci = 0; ci < p.n_cmds; ++ci) {
      if (lane < (int)(sizeof(Cmd) / 4))
        reinterpret_cast<int32_t *>(&S.cmd)[lane] = reinterpret_cast<const int32_t *>(p.cmds + ci)[lane];
      __syncwarp();
      exec_cmd(p, S, dyn, S.cmd, p.results + ci, lane);
    }
  }

  // ---- write back dirty ledgers + scheduler state ----
  writeback(p, dyn, S, lane);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

thread_local std::string g_err;

int set_err(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

}  // namespace

namespace gsw {
// shared by the job runners / executor (gs_work.cu, gs_exec.cu)
void set_last_error(const std::string &msg) { g_err = msg; }
}  // namespace gsw

namespace {

#define CU(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return set_err(GS_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

}  // namespace (reopened below)

namespace gscache {
namespace {
std::mutex g_mu;
std::multimap<std::pair<int, size_t>, void *> g_host, g_dev;
std::multimap<std::pair<int, int>, cudaStream_t> g_streams;
}  // namespace

cudaError_t host_alloc(void **p, size_t bytes) {
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_host.find({0, bytes});
    if (it != g_host.end()) {
      *p = it->second;
      g_host.erase(it);
      return cudaSuccess;
    }
  }
  return cudaHostAlloc(p, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
}
void host_free(void *p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> g(g_mu);
  g_host.insert({{0, bytes}, p});
}
static void (*g_oom_hook)(int) = nullptr;
void set_oom_hook(void (*hook)(int device)) { g_oom_hook = hook; }
cudaError_t dev_alloc(void **p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_dev.find({dev, bytes});
    if (it != g_dev.end()) {
      *p = it->second;
      g_dev.erase(it);
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation && g_oom_hook) {
    cudaGetLastError();
    g_oom_hook(dev);
    cudaSetDevice(dev);
    e = cudaMalloc(p, bytes);
  }
  return e;
}
void dev_free(void *p, size_t bytes, int device) {
  if (!p) return;
  std::lock_guard<std::mutex> g(g_mu);
  g_dev.insert({{device, bytes}, p});
}
cudaError_t stream_get(cudaStream_t *s, int prio) {
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_streams.find({dev, prio});
    if (it != g_streams.end()) {
      *s = it->second;
      g_streams.erase(it);
      return cudaSuccess;
    }
  }
  return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, prio);
}
void stream_put(cudaStream_t s, int device, int prio) {
  if (!s) return;
  std::lock_guard<std::mutex> g(g_mu);
  g_streams.insert({{device, prio}, s});
}
const cudaDeviceProp &device_props(int device) {
  static std::map<int, cudaDeviceProp> props;
  std::lock_guard<std::mutex> g(g_mu);
  auto it = props.find(device);
  if (it == props.end()) {
    cudaDeviceProp p;
    memset(&p, 0, sizeof p);
    cudaGetDeviceProperties(&p, device);
    it = props.emplace(device, p).first;
  }
  return it->second;
}
}  // namespace gscache

namespace {

template <class T>
struct Mapped {
  T *h = nullptr;
  T *d = nullptr;
  size_t n = 0;
  int alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    CU(gscache::host_alloc((void **)&h, count * sizeof(T)));
    memset(h, 0, count * sizeof(T));
    CU(cudaHostGetDevicePointer((void **)&d, h, 0));
    n = count;
    return GS_OK;
  }
  void release() {
    if (h) gscache::host_free(h, n * sizeof(T));
    h = d = nullptr;
    n = 0;
  }
};

template <class T>
struct DevBuf {
  T *d = nullptr;
  size_t n = 0;
  int dev = 0;
  int ensure(size_t count, cudaStream_t st, bool keep) {
    if (count <= n) return GS_OK;
    size_t nn = std::max(count, n * 2);
    T *nd = nullptr;
    int cur = 0;
    cudaGetDevice(&cur);
    CU(gscache::dev_alloc((void **)&nd, nn * sizeof(T)));
    CU(cudaMemsetAsync(nd, 0, nn * sizeof(T), st));
    if (keep && d && n) CU(cudaMemcpyAsync(nd, d, n * sizeof(T), cudaMemcpyDeviceToDevice, st));
    CU(cudaStreamSynchronize(st));
    release();
    d = nd;
    n = nn;
    dev = cur;
    return GS_OK;
  }
  void release() {
    if (d) gscache::dev_free(d, n * sizeof(T), dev);
    d = nullptr;
    n = 0;
  }
};

}  // namespace

struct gs_engine {
  int cuda_dev = 0;
  cudaStream_t stream = nullptr;
  int stream_prio = 0;
  std::recursive_mutex mu;
  int32_t res_cap = 0;
  std::vector<gs_device *> devices;
  Mapped<Cmd> cmds;
  Mapped<gs_decision> results;
  Mapped<int32_t> plan_io;
  Mapped<SchedState> dummy_state;
  DevBuf<Cmd> dcmds;
  int64_t launches = 0;
  int64_t decisions = 0;
  int rings_active = 0;
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
  gs_sched *ring_owner = nullptr;  // scheduler whose persistent kernel owns this ledger
  int32_t ring_index = -1;
};

struct gs_sched {
  gs_engine *eng = nullptr;
  std::vector<gs_device *> devs;
  int32_t policy = 0, cg_ratio = 6, skip_ahead = 1;
  Mapped<SchedState> st;
  DevBuf<gs_probe> pend;
  DevBuf<int32_t> claims;
  DevBuf<int32_t> events;
  Mapped<gs_decision> drain;
  // persistent decision kernel (command ring)
  Mapped<Ring> ring;
  bool ring_active = false;
  // a sweep leaves up to max_resident tasks holding ledger capacity that no
  // caller can release (their handles never left the kernel): the scheduler
  // and its ledgers are spent afterwards and every further decision call is
  // refused
  bool swept = false;
  cudaStream_t ring_stream = nullptr;
  size_t ring_smem = 0;
  KParams ring_params{};
};

namespace {

int pad4(int64_t n) { return (int)((n + 3) / 4 * 4); }

// Serializes engine calls (single decision authority) and makes the engine's
// device current for the duration of the call (worker threads of the
// executor keep their own device current between calls).
struct EngineLock {
  std::lock_guard<std::recursive_mutex> g;
  int prev = -1;
  explicit EngineLock(gs_engine *e) : g(e->mu) {
    cudaGetDevice(&prev);
    if (prev != e->cuda_dev) cudaSetDevice(e->cuda_dev);
  }
  ~EngineLock() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

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
    {
      const gs_spec &sp = dv->spec;
      const int64_t lim = 1LL << 22;
      k.t_small = (int32_t)(INT_MAX / std::max<int64_t>(dv->spec.sm_count, 1));
    k.fast = sp.max_tbs_per_sm >= 0 && sp.max_tbs_per_sm < lim && sp.max_warps_per_sm >= 0 &&
               sp.max_warps_per_sm < lim && sp.regs_per_sm >= 0 && sp.regs_per_sm < lim &&
               sp.smem_per_sm_bytes >= 0 && sp.smem_per_sm_bytes < lim;
    }
    off += kLedHdrWords + 4 * dv->arr_pad;
    max_pad = std::max(max_pad, dv->arr_pad);
  }
  p.max_sm_pad = max_pad;
  p.stage_q = off / 4;
  p.scratch_off = off;
  p.fifo_off = off + 2 * max_pad;
  p.fifo_cap = 0;
  L.smem = (size_t)(off + 2 * max_pad) * sizeof(int);
  if ((int)L.smem > eng->max_smem)
    return set_err(GS_ERR_CONFIG, "fleet ledgers exceed shared memory");
  p.st = eng->dummy_state.d;
  p.results = eng->results.d;
  p.plan_io = eng->plan_io.d;
  p.claims = nullptr;
  p.job_cap = 0;
  return GS_OK;
}

int launch(gs_engine *eng, Launch &L) {
  gs_interp_kernel<<<1, kThreads, L.smem, eng->stream>>>(L.p);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(eng->stream));
  eng->launches++;
  return GS_OK;
}

// ---- command ring (persistent decision kernel) ----------------------------

int ring_launch(gs_sched *s) {
  Ring *r = s->ring.h;
  r->alive = 1;
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
  KParams p = s->ring_params;
  p.ring = s->ring.d;
  gs_interp_kernel<<<1, kThreads, s->ring_smem, s->ring_stream>>>(p);
  CU(cudaGetLastError());
  s->eng->launches++;
  return GS_OK;
}

// Push n commands (in order) and wait for their results.  Caller holds the
// engine lock.
int ring_call(gs_sched *s, const Cmd *cmds, int n, gs_decision *results) {
  Ring *r = s->ring.h;
  for (int base = 0; base < n; base += kRingSlots) {
    const int m = std::min(n - base, kRingSlots);
    if (!__atomic_load_n(&r->alive, __ATOMIC_ACQUIRE)) {
      // the idle watchdog retired the kernel: ledgers were written back,
      // relaunch it (it restages from mapped memory)
      CU(cudaStreamSynchronize(s->ring_stream));
      int rc = ring_launch(s);
      if (rc) return rc;
    }
    long long t = __atomic_load_n(&r->tail, __ATOMIC_RELAXED);
    for (int k = 0; k < m; ++k) {
      Cmd &dst = r->cmds[(t + k) % kRingSlots];
      dst = cmds[base + k];
    }
    __atomic_store_n(&r->tail, t + m, __ATOMIC_RELEASE);
    const auto t0 = std::chrono::steady_clock::now();
    while (__atomic_load_n(&r->done, __ATOMIC_ACQUIRE) < t + m) {
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
      if (!__atomic_load_n(&r->alive, __ATOMIC_ACQUIRE) &&
          __atomic_load_n(&r->done, __ATOMIC_ACQUIRE) < t + m) {
        // retired between our check and the push: relaunch, it resumes at done
        CU(cudaStreamSynchronize(s->ring_stream));
        int rc = ring_launch(s);
        if (rc) return rc;
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
        return set_err(GS_ERR_CUDA, "decision ring did not answer within 30 s");
    }
    for (int k = 0; k < m; ++k) results[base + k] = r->results[(t + k) % kRingSlots];
    s->eng->decisions += m;
  }
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
  EngineLock g(eng);
  if (dv->ring_owner && dv->ring_owner->ring_active) {
    Cmd rc = c;
    rc.dev = dv->ring_index;
    return ring_call(dv->ring_owner, &rc, 1, out);
  }
  eng->decisions++;
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
  p.claims = s->claims.d;
  p.job_cap = (int32_t)s->claims.n;
  p.drain_out = s->drain.d;
  p.drain_cap = (int32_t)s->drain.n;
  return GS_OK;
}

int ensure_pending(gs_sched *s, int extra) {
  const size_t need = (size_t)s->st.h->pend_count + extra + 1;
  if (s->ring_active) {
    if (need > s->pend.n || need > s->drain.n)
      return set_err(GS_ERR_NOMEM, "pending queue capacity reserved at ring start exceeded");
    return GS_OK;
  }
  int rc = s->pend.ensure(need, s->eng->stream, true);
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
  if (s->ring_active) return set_err(GS_ERR_NOMEM, "job capacity reserved at ring start exceeded");
  size_t nn = std::max<size_t>((size_t)job + 1, old * 2);
  int32_t *nd = nullptr;
  int cur = 0;
  cudaGetDevice(&cur);
  CU(gscache::dev_alloc((void **)&nd, nn * sizeof(int32_t)));
  CU(cudaMemsetAsync(nd, 0xff, nn * sizeof(int32_t), s->eng->stream));  // -1
  if (old) CU(cudaMemcpyAsync(nd, s->claims.d, old * sizeof(int32_t), cudaMemcpyDeviceToDevice, s->eng->stream));
  CU(cudaStreamSynchronize(s->eng->stream));
  s->claims.release();
  s->claims.d = nd;
  s->claims.n = nn;
  s->claims.dev = cur;
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
  const cudaDeviceProp &prop = gscache::device_props(cuda_device);
  if (prop.major < 10) return set_err(GS_ERR_CUDA, "libgs is built for sm_100a (B200)");
  auto *eng = new gs_engine();
  eng->cuda_dev = cuda_device;
  {
    // dynamic shared memory left next to the kernel's static arrays
    cudaFuncAttributes fa;
    CU(cudaFuncGetAttributes(&fa, gs_interp_kernel));
    eng->max_smem = ((int)prop.sharedMemPerBlockOptin - (int)fa.sharedSizeBytes) & ~15;
  }
  CU(cudaFuncSetAttribute(gs_interp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, eng->max_smem));
  {
    // decisions preempt workload blocks at the block scheduler
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(gscache::stream_get(&eng->stream, hi));
    eng->stream_prio = hi;
  }
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
  gscache::stream_put(eng->stream, eng->cuda_dev, eng->stream_prio);
  delete eng;
}

int gs_engine_reserve_handles(gs_engine *eng, int32_t capacity) {
  EngineLock g(eng);
  if (capacity <= eng->res_cap) return GS_OK;
  if (eng->rings_active) return set_err(GS_ERR_NOMEM, "handle capacity reserved at ring start exceeded");
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
  EngineLock g(eng);
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
  EngineLock g(eng);
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
  EngineLock g(dv->eng);
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
  EngineLock g(dv->eng);
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
  EngineLock g(dv->eng);
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
  EngineLock g(dv->eng);
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
  EngineLock g(eng);
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
  gs_sched_ring_stop(s);
  EngineLock g(s->eng);
  s->st.release();
  s->drain.release();
  s->pend.release();
  s->claims.release();
  s->events.release();
  delete s;
}

int gs_submit_batch(gs_sched *s, const gs_probe *reqs, int32_t n, gs_decision *out) {
  gs_engine *eng = s->eng;
  EngineLock g(eng);
  if (n <= 0) return GS_OK;
  if (s->swept) return set_err(GS_ERR_CONTRACT, "scheduler already consumed by a sweep");
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
  eng->decisions += s->ring_active ? 0 : n;
  if (s->ring_active) {
    rc = ring_call(s, eng->cmds.h, n, eng->results.h);
    if (rc) return rc;
    if (out) memcpy(out, eng->results.h, sizeof(gs_decision) * n);
    return GS_OK;
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

// diagnostics (not in gs.h): globaltimer stamps of the ring's last command
int gs_ring_stamps(gs_sched *s, unsigned long long *out5) {
  if (!s || !s->ring_active) return set_err(GS_ERR_CONFIG, "ring not running");
  for (int i = 0; i < 5; ++i) out5[i] = s->ring.h->stamp[i];
  return GS_OK;
}

int gs_on_release(gs_sched *s, gs_decision *out, int32_t out_cap, int32_t *n_tried, int32_t *n_admitted) {
  gs_engine *eng = s->eng;
  EngineLock g(eng);
  int rc = ensure_pending(s, 0);
  if (!rc) rc = ensure_cmds(eng, 1);
  if (rc) return rc;
  Launch L;
  rc = sched_params(s, L);
  if (rc) return rc;
  Cmd &c = eng->cmds.h[0];
  memset(&c, 0, sizeof c);
  c.op = OP_ON_RELEASE;
  if (s->ring_active) {
    rc = ring_call(s, &c, 1, eng->results.h);
  } else {
    eng->decisions++;
    L.p.cmds = eng->cmds.d;
    L.p.n_cmds = 1;
    rc = launch(eng, L);
  }
  if (rc) return rc;
  const int tried = s->st.h->n_tried, adm = s->st.h->n_admitted;
  if (n_tried) *n_tried = tried;
  if (n_admitted) *n_admitted = adm;
  if (out) memcpy(out, s->drain.h, sizeof(gs_decision) * std::min(tried, out_cap));
  return GS_OK;
}

int gs_release_redrive(gs_sched *s, int32_t dev_index, int32_t handle, int64_t *freed, gs_decision *out,
                       int32_t out_cap, int32_t *n_tried, int32_t *n_admitted) {
  gs_engine *eng = s->eng;
  EngineLock g(eng);
  if (dev_index < 0 || dev_index >= (int32_t)s->devs.size()) return set_err(GS_ERR_CONFIG, "bad device index");
  int rc = check_handle(eng, handle);
  if (!rc) rc = ensure_pending(s, 0);
  if (!rc) rc = ensure_cmds(eng, 2);
  if (rc) return rc;
  Launch L;
  rc = sched_params(s, L);
  if (rc) return rc;
  Cmd *c = eng->cmds.h;
  memset(c, 0, 2 * sizeof(Cmd));
  c[0].op = OP_RELEASE;
  c[0].dev = dev_index;
  c[0].handle = handle;
  c[1].op = OP_ON_RELEASE;
  gs_decision res[2];
  if (s->ring_active) {
    rc = ring_call(s, c, 2, res);
  } else {
    eng->decisions++;
    L.p.cmds = eng->cmds.d;
    L.p.n_cmds = 2;
    L.p.results = eng->results.d;
    rc = launch(eng, L);
    if (!rc) memcpy(res, eng->results.h, sizeof res);
  }
  if (rc) return rc;
  const int tried = s->st.h->n_tried, adm = s->st.h->n_admitted;
  if (n_tried) *n_tried = tried;
  if (n_admitted) *n_admitted = adm;
  if (out) memcpy(out, s->drain.h, sizeof(gs_decision) * std::min(tried, out_cap));
  if (res[0].outcome == GS_ERR_CONTRACT) return set_err(GS_ERR_CONTRACT, "release of unknown task");
  if (freed) *freed = res[0].free_mem_after;
  return GS_OK;
}

int gs_job_ended(gs_sched *s, int32_t job) {
  gs_engine *eng = s->eng;
  EngineLock g(eng);
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
  if (s->ring_active) return ring_call(s, &c, 1, eng->results.h);
  eng->decisions++;
  L.p.cmds = eng->cmds.d;
  L.p.n_cmds = 1;
  return launch(eng, L);
}

int gs_sched_ring_start(gs_sched *s, int32_t max_pending, int32_t max_handles, int32_t max_jobs) {
  gs_engine *eng = s->eng;
  EngineLock g(eng);
  if (s->ring_active) return GS_OK;
  for (gs_device *dv : s->devs)
    if (dv->ring_owner) return set_err(GS_ERR_CONTRACT, "a device of this fleet is owned by another ring");
  int rc = gs_engine_reserve_handles(eng, std::max(max_handles, 1));
  if (!rc) rc = ensure_jobs(s, std::max(max_jobs, 1));
  if (!rc) rc = ensure_pending(s, std::max(max_pending, 1));
  if (!rc) rc = ensure_cmds(eng, kRingSlots);
  if (!rc && !s->ring.h) rc = s->ring.alloc(1);
  if (rc) return rc;
  Launch L;
  rc = sched_params(s, L);
  if (rc) return rc;
  s->ring_params = L.p;
  // idle watchdog: an idle ring retires after 200 ms (the next call relaunches
  // it in ~10 us), so a resident decision kernel never pins the device for long
  s->ring_params.ring_idle_ns = 200LL * 1000 * 1000;
  {
    const char *sl = getenv("GS_RING_SLEEP_NS");
    s->ring_params.ring_sleep_ns = sl ? atoi(sl) : 0;
    const char *wb = getenv("GS_RING_WB");
    s->ring_params.wb_mode = wb ? atoi(wb) : 0;
  }
  s->ring_smem = L.smem;
  if (!s->ring_stream) {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const char *pr = getenv("GS_RING_PRIO");  // experiment knob: 0 = default priority
    CU(cudaStreamCreateWithPriority(&s->ring_stream, cudaStreamNonBlocking, (pr && pr[0] == '0') ? lo : hi));
  }
  memset(s->ring.h, 0, sizeof(Ring));
  rc = ring_launch(s);
  if (rc) return rc;
  s->ring_active = true;
  eng->rings_active++;
  for (size_t d = 0; d < s->devs.size(); ++d) {
    s->devs[d]->ring_owner = s;
    s->devs[d]->ring_index = (int32_t)d;
  }
  return GS_OK;
}

int gs_sched_ring_stop(gs_sched *s) {
  gs_engine *eng = s->eng;
  EngineLock g(eng);
  if (!s->ring_active) return GS_OK;
  Ring *r = s->ring.h;
  int rc = GS_OK;
  if (__atomic_load_n(&r->alive, __ATOMIC_ACQUIRE)) {
    Cmd stop;
    memset(&stop, 0, sizeof stop);
    stop.op = OP_STOP;
    const long long t = __atomic_load_n(&r->tail, __ATOMIC_RELAXED);
    r->cmds[t % kRingSlots] = stop;
    __atomic_store_n(&r->tail, t + 1, __ATOMIC_RELEASE);
  }
  cudaError_t e = cudaStreamSynchronize(s->ring_stream);
  if (e != cudaSuccess) rc = set_err(GS_ERR_CUDA, cudaGetErrorString(e));
  s->ring_active = false;
  eng->rings_active--;
  for (gs_device *dv : s->devs) {
    dv->ring_owner = nullptr;
    dv->ring_index = -1;
  }
  return rc;
}

int64_t gs_engine_decisions(gs_engine *eng) { return eng->decisions; }

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
  EngineLock g(eng);
  if (n <= 0) return GS_OK;
  if (s->ring_active) return set_err(GS_ERR_CONTRACT, "stop the decision ring before a sweep");
  if (s->swept) return set_err(GS_ERR_CONTRACT, "scheduler already consumed by a sweep");
  if (s->st.h->pend_count != 0 || s->st.h->fifo_tail != s->st.h->fifo_head)
    return set_err(GS_ERR_CONTRACT, "sweep needs a fresh scheduler");
  int rc = gs_engine_reserve_handles(eng, n);
  if (!rc) rc = ensure_pending(s, n);
  if (!rc) rc = s->events.ensure(3 * (size_t)std::max<int64_t>(events_cap, 1), eng->stream, false);
  if (rc) return rc;
  // every return path below gives back the probe copy and the events
  gs_probe *dprobes = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  struct Guard {
    gs_probe *&p;
    cudaEvent_t &a, &b;
    ~Guard() {
      if (p) cudaFree(p);
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } guard{dprobes, e0, e1};
  CU(cudaMalloc((void **)&dprobes, sizeof(gs_probe) * n));
  CU(cudaMemcpyAsync(dprobes, probes, sizeof(gs_probe) * n, cudaMemcpyHostToDevice, eng->stream));
  Launch L;
  rc = sched_params(s, L);
  if (rc) return rc;
  L.p.sweep = 1;
  L.p.sweep_probes = dprobes;
  {
    // GS_SWEEP_GENERAL=1: every probe through the general interpreter path
    // (the specialised mgb-warps chain is checked against it in the tests)
    const char *g = getenv("GS_SWEEP_GENERAL");
    L.p.sweep_fast = !(g && g[0] == '1');
  }
  {
    // resident FIFO slots with cached residency data (kSlotHdr + blocks)
    int stride = kSlotHdr + (s->policy == GS_POLICY_MGB_SM ? L.p.max_sm_pad : 0);
    stride = (stride + 1) & ~1;
    L.p.fifo_stride = stride;
    const size_t room = (size_t)eng->max_smem > L.smem ? ((size_t)eng->max_smem - L.smem) / (stride * sizeof(int)) : 0;
    L.p.fifo_cap = (int32_t)std::min<size_t>((size_t)n + 1, room);
    if (L.p.fifo_cap < 64) return set_err(GS_ERR_NOMEM, "no shared memory left for the resident FIFO");
    L.smem += (size_t)L.p.fifo_cap * stride * sizeof(int);
  }
  L.p.n_cmds = n;
  L.p.max_resident = max_resident;
  L.p.events = s->events.d;
  L.p.events_cap = events_cap;
  s->st.h->n_events = 0;
  s->st.h->error = 0;
  s->st.h->fifo_head = s->st.h->fifo_tail = 0;
  // from the launch on, the ledgers carry the sweep's residents
  s->swept = true;
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
  if (kernel_ms) *kernel_ms = ms;
  const int64_t ne = s->st.h->n_events;
  if (n_events) *n_events = ne;
  if (events)
    CU(cudaMemcpy(events, s->events.d, sizeof(int32_t) * 3 * std::min(ne, events_cap), cudaMemcpyDeviceToHost));
  s->st.h->fifo_head = s->st.h->fifo_tail = 0;
  if (s->st.h->error) return set_err(s->st.h->error, "sweep overflowed the resident FIFO");
  return GS_OK;
}

}  // extern "C"
