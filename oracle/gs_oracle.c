/*
 * gs_oracle.c — CPU restatement of the reference placement path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker or the timed CPU baseline; the product path
 * (libgs, csrc/gs_sched.cu) never calls it.
 *
 * It restates, line for line in behaviour, /root/reference/pkg/src/gpushare:
 *   occupancy_limit_per_sm        device_model.py:48-58
 *   DeviceState._sm_admits        device_model.py:105-118
 *   DeviceState.try_place_blocks  device_model.py:120-139  (the reference's
 *                                 one-block-per-visit loop, NOT the GPU's
 *                                 closed form — that is what is checked)
 *   commit_placement              device_model.py:141-161
 *   reserve/assign/add_warps/allocate_raw/release_task  :169-209
 *   check_conservation            device_model.py:220-245
 *   Scheduler.submit/on_release/job_ended  schedulers.py:89-123
 *   _try_mgb_sm / _try_mgb_warps / _try_sa / _try_cg / _impossible_everywhere
 *                                 schedulers.py:137-199
 * Parity is pinned against golden event streams recorded from the
 * reference itself (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/gs.h"

typedef struct {
    int64_t mem, warps, rpb, spb;
    int32_t wpb, present, has_blocks;
    int32_t *blocks;
} ores;

typedef struct odev {
    gs_spec spec;
    int32_t index;
    int64_t free_mem, in_use_warps, version;
    int32_t rr_cursor;
    int32_t *sm_warps, *sm_tbs, *sm_regs, *sm_smem;
    ores *res;
    int32_t res_cap;
} odev;

typedef struct osched {
    odev **devs;
    int32_t n, policy, cg_ratio, skip_ahead;
    gs_probe *pend;
    int32_t pend_n, pend_cap;
    int32_t sa_owner[GS_MAX_DEVICES];
    int32_t cg_counts[GS_MAX_DEVICES];
    int32_t cg_cursor;
    int32_t *claims;
    int32_t claims_cap;
} osched;

/* ---- device ----------------------------------------------------------- */

odev *o_dev_new(const gs_spec *spec, int32_t index) {
    odev *d = (odev *)calloc(1, sizeof(odev));
    int64_t n = spec->sm_count;
    d->spec = *spec;
    d->index = index;
    d->free_mem = spec->mem_bytes;
    d->sm_warps = (int32_t *)calloc(n, 4);
    d->sm_tbs = (int32_t *)calloc(n, 4);
    d->sm_regs = (int32_t *)calloc(n, 4);
    d->sm_smem = (int32_t *)calloc(n, 4);
    return d;
}

void o_dev_free(odev *d) {
    for (int i = 0; i < d->res_cap; ++i) free(d->res[i].blocks);
    free(d->res);
    free(d->sm_warps);
    free(d->sm_tbs);
    free(d->sm_regs);
    free(d->sm_smem);
    free(d);
}

/* ledger snapshot: free_mem, in_use_warps, version, rr_cursor */
void o_ledger(const odev *d, int64_t *out) {
    out[0] = d->free_mem;
    out[1] = d->in_use_warps;
    out[2] = d->version;
    out[3] = d->rr_cursor;
}

void o_set_ledger(odev *d, const int64_t *in) {
    d->free_mem = in[0];
    d->in_use_warps = in[1];
    d->version = in[2];
    d->rr_cursor = (int32_t)in[3];
}

int32_t *o_sm_array(odev *d, int32_t which) {
    switch (which) {
        case 0: return d->sm_warps;
        case 1: return d->sm_tbs;
        case 2: return d->sm_regs;
        default: return d->sm_smem;
    }
}

/* _entry (device_model.py:211-216) */
static ores *entry(odev *d, int32_t h) {
    if (h >= d->res_cap) {
        int32_t nc = d->res_cap ? d->res_cap : 64;
        while (nc <= h) nc *= 2;
        d->res = (ores *)realloc(d->res, sizeof(ores) * nc);
        memset(d->res + d->res_cap, 0, sizeof(ores) * (nc - d->res_cap));
        d->res_cap = nc;
    }
    ores *e = &d->res[h];
    if (!e->present) {
        int32_t *keep = e->blocks;
        memset(e, 0, sizeof(*e));
        e->blocks = keep;
        e->present = 1;
    }
    return e;
}

int32_t o_is_resident(const odev *d, int32_t h) { return h < d->res_cap && d->res[h].present; }

/* Python floor division for the signed cases the ledgers can reach. */
static int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

int64_t o_occupancy_limit_per_sm(const gs_spec *s, const gs_probe *r) {
    int64_t lim = s->max_tbs_per_sm;
    if (r->warps_per_block > 0) {
        int64_t v = floordiv(s->max_warps_per_sm, r->warps_per_block);
        if (v < lim) lim = v;
    }
    int64_t rpb = (int64_t)r->regs_per_thread * r->threads_per_block;
    if (rpb > 0) {
        int64_t v = floordiv(s->regs_per_sm, rpb);
        if (v < lim) lim = v;
    }
    if (r->smem_per_block > 0) {
        int64_t v = floordiv(s->smem_per_sm_bytes, r->smem_per_block);
        if (v < lim) lim = v;
    }
    return lim < 0 ? 0 : lim;
}

/* _sm_admits (device_model.py:105-118) */
static int sm_admits(const odev *d, int sm, const gs_probe *r, const int64_t *extra) {
    const gs_spec *s = &d->spec;
    if (d->sm_tbs[sm] + extra[sm] + 1 > s->max_tbs_per_sm) return 0;
    int64_t wpb = r->warps_per_block;
    if (d->sm_warps[sm] + extra[sm] * wpb + wpb > s->max_warps_per_sm) return 0;
    int64_t rpb = (int64_t)r->regs_per_thread * r->threads_per_block;
    if (rpb && d->sm_regs[sm] + extra[sm] * rpb + rpb > s->regs_per_sm) return 0;
    int64_t spb = r->smem_per_block;
    if (spb && d->sm_smem[sm] + extra[sm] * spb + spb > s->smem_per_sm_bytes) return 0;
    return 1;
}

/* try_place_blocks (device_model.py:120-139): 0 = plan, 1 = None */
int32_t o_try_place(const odev *d, const gs_probe *r, int32_t *blocks, int32_t *cursor_out,
                    int64_t *version_out) {
    int64_t n = d->spec.sm_count;
    int64_t *placed = (int64_t *)calloc(n, sizeof(int64_t));
    int64_t remaining = r->thread_blocks;
    int64_t cursor = d->rr_cursor;
    int64_t misses = 0;
    while (remaining > 0) {
        int64_t sm = ((cursor % n) + n) % n;
        cursor += 1;
        if (sm_admits(d, (int)sm, r, placed)) {
            placed[sm] += 1;
            remaining -= 1;
            misses = 0;
        } else {
            misses += 1;
            if (misses >= n) {
                free(placed);
                return GS_INFEASIBLE;
            }
        }
    }
    for (int64_t i = 0; i < n; ++i) blocks[i] = (int32_t)placed[i];
    *cursor_out = (int32_t)(((cursor % n) + n) % n);
    *version_out = d->version;
    free(placed);
    return GS_OK;
}

/* commit_placement (device_model.py:141-161) */
int32_t o_commit(odev *d, int32_t h, const gs_probe *r, const int32_t *blocks, int32_t cursor,
                 int64_t plan_version) {
    if (plan_version != d->version) return GS_ERR_CONTRACT;
    int64_t rpb = (int64_t)r->regs_per_thread * r->threads_per_block;
    for (int64_t sm = 0; sm < d->spec.sm_count; ++sm) {
        int64_t c = blocks[sm];
        if (!c) continue;
        d->sm_tbs[sm] += (int32_t)c;
        d->sm_warps[sm] += (int32_t)(c * r->warps_per_block);
        d->sm_regs[sm] += (int32_t)(c * rpb);
        d->sm_smem[sm] += (int32_t)(c * r->smem_per_block);
    }
    d->rr_cursor = cursor;
    ores *e = entry(d, h);
    if (!e->blocks) e->blocks = (int32_t *)malloc(4 * d->spec.sm_count);
    memcpy(e->blocks, blocks, 4 * d->spec.sm_count);
    e->has_blocks = 1;
    e->rpb = rpb;
    e->spb = r->smem_per_block;
    e->wpb = r->warps_per_block;
    d->version += 1;
    return GS_OK;
}

int32_t o_reserve(odev *d, int64_t n) {
    if (n > d->free_mem) return GS_INFEASIBLE;
    d->free_mem -= n;
    d->version += 1;
    return GS_OK;
}

void o_assign(odev *d, int32_t h, int64_t n) {
    entry(d, h)->mem += n;
    d->version += 1;
}

void o_add_warps(odev *d, int32_t h, int64_t w) {
    entry(d, h)->warps += w;
    d->in_use_warps += w;
    d->version += 1;
}

int32_t o_alloc_raw(odev *d, int32_t h, int64_t n) {
    if (o_reserve(d, n) != GS_OK) return GS_INFEASIBLE;
    o_assign(d, h, n);
    return GS_OK;
}

int32_t o_release(odev *d, int32_t h, int64_t *freed) {
    if (!o_is_resident(d, h)) return GS_ERR_CONTRACT;
    ores *e = &d->res[h];
    d->free_mem += e->mem;
    d->in_use_warps -= e->warps;
    if (e->has_blocks) {
        for (int64_t sm = 0; sm < d->spec.sm_count; ++sm) {
            int64_t c = e->blocks[sm];
            if (!c) continue;
            d->sm_tbs[sm] -= (int32_t)c;
            d->sm_warps[sm] -= (int32_t)(c * e->wpb);
            d->sm_regs[sm] -= (int32_t)(c * e->rpb);
            d->sm_smem[sm] -= (int32_t)(c * e->spb);
        }
    }
    d->version += 1;
    if (freed) *freed = e->mem;
    e->present = 0;
    return GS_OK;
}

/* check_conservation (device_model.py:220-245): 0 ok, else kind (GS_CHECK_*) */
int32_t o_check(const odev *d, int32_t *sm_out, int64_t *held_out, int64_t *warps_out) {
    int64_t held = 0, warps = 0;
    for (int i = 0; i < d->res_cap; ++i)
        if (d->res[i].present) {
            held += d->res[i].mem;
            warps += d->res[i].warps;
        }
    *sm_out = -1;
    *held_out = held;
    *warps_out = warps;
    if (d->free_mem < 0 || d->free_mem + held != d->spec.mem_bytes) return GS_CHECK_MEM;
    if (warps != d->in_use_warps) return GS_CHECK_WARPS;
    const gs_spec *s = &d->spec;
    for (int64_t sm = 0; sm < s->sm_count; ++sm) {
        *sm_out = (int32_t)sm;
        if (!(0 <= d->sm_tbs[sm] && d->sm_tbs[sm] <= s->max_tbs_per_sm)) return GS_CHECK_SM_TBS;
        if (!(0 <= d->sm_warps[sm] && d->sm_warps[sm] <= s->max_warps_per_sm)) return GS_CHECK_SM_WARPS;
        if (!(0 <= d->sm_regs[sm] && d->sm_regs[sm] <= s->regs_per_sm)) return GS_CHECK_SM_REGS;
        if (!(0 <= d->sm_smem[sm] && d->sm_smem[sm] <= s->smem_per_sm_bytes)) return GS_CHECK_SM_SMEM;
    }
    *sm_out = -1;
    return GS_CHECK_OK;
}

/* ---- scheduler -------------------------------------------------------- */

osched *o_sched_new(odev **devs, int32_t n, int32_t policy, int32_t cg_ratio, int32_t skip_ahead) {
    osched *s = (osched *)calloc(1, sizeof(osched));
    s->devs = (odev **)malloc(sizeof(odev *) * n);
    memcpy(s->devs, devs, sizeof(odev *) * n);
    s->n = n;
    s->policy = policy;
    s->cg_ratio = cg_ratio;
    s->skip_ahead = skip_ahead;
    for (int i = 0; i < GS_MAX_DEVICES; ++i) s->sa_owner[i] = -1;
    return s;
}

void o_sched_free(osched *s) {
    free(s->devs);
    free(s->pend);
    free(s->claims);
    free(s);
}

int32_t o_pending_count(const osched *s) { return s->pend_n; }

static void set_claim(osched *s, int32_t job, int32_t dev) {
    if (job < 0) return;
    if (job >= s->claims_cap) {
        int32_t nc = s->claims_cap ? s->claims_cap : 64;
        while (nc <= job) nc *= 2;
        s->claims = (int32_t *)realloc(s->claims, 4 * nc);
        for (int i = s->claims_cap; i < nc; ++i) s->claims[i] = -1;
        s->claims_cap = nc;
    }
    s->claims[job] = dev;
}

/* _impossible_everywhere (schedulers.py:191-199) */
static int impossible_everywhere(const osched *s, const gs_probe *r, int check_compute) {
    for (int i = 0; i < s->n; ++i) {
        const odev *d = s->devs[i];
        if (r->mem_bytes > d->spec.mem_bytes) continue;
        if (check_compute && o_occupancy_limit_per_sm(&d->spec, r) * d->spec.sm_count < r->thread_blocks)
            continue;
        return 0;
    }
    return 1;
}

/* _try (schedulers.py:127-135) and the four policy cores */
static int32_t try_one(osched *s, const gs_probe *r, int32_t *dev_out) {
    *dev_out = -1;
    if (s->policy == GS_POLICY_MGB_SM) {
        int32_t *blocks = NULL;
        for (int i = 0; i < s->n; ++i) {
            odev *d = s->devs[i];
            if (d->free_mem < r->mem_bytes) continue;
            blocks = (int32_t *)realloc(blocks, 4 * d->spec.sm_count);
            int32_t cur;
            int64_t ver;
            if (o_try_place(d, r, blocks, &cur, &ver) != GS_OK) continue;
            o_commit(d, r->handle, r, blocks, cur, ver);
            o_reserve(d, r->mem_bytes);
            o_assign(d, r->handle, r->mem_bytes);
            o_add_warps(d, r->handle, r->total_warps);
            free(blocks);
            *dev_out = i;
            return GS_ASSIGN;
        }
        free(blocks);
        return impossible_everywhere(s, r, 1) ? GS_REJECTED : GS_DEFER;
    }
    if (s->policy == GS_POLICY_MGB_WARPS) {
        int best = -1;
        for (int i = 0; i < s->n; ++i) {
            odev *d = s->devs[i];
            if (d->free_mem < r->mem_bytes) continue;
            if (best < 0 || d->in_use_warps < s->devs[best]->in_use_warps) best = i;
        }
        if (best < 0) return impossible_everywhere(s, r, 0) ? GS_REJECTED : GS_DEFER;
        odev *d = s->devs[best];
        o_reserve(d, r->mem_bytes);
        o_assign(d, r->handle, r->mem_bytes);
        o_add_warps(d, r->handle, r->total_warps);
        *dev_out = best;
        return GS_ASSIGN;
    }
    if (s->policy == GS_POLICY_SA) {
        for (int i = 0; i < s->n; ++i)
            if (s->sa_owner[i] < 0) {
                s->sa_owner[i] = r->job;
                *dev_out = i;
                return GS_ASSIGN;
            }
        return GS_DEFER;
    }
    for (int step = 0; step < s->n; ++step) {
        int idx = (s->cg_cursor + step) % s->n;
        if (s->cg_counts[idx] < s->cg_ratio) {
            s->cg_counts[idx] += 1;
            set_claim(s, r->job, idx);
            s->cg_cursor = (idx + 1) % s->n;
            *dev_out = idx;
            return GS_ASSIGN;
        }
    }
    return GS_DEFER;
}

static void fill(gs_decision *o, const osched *s, int32_t outcome, int32_t dev, int32_t pidx, int32_t h) {
    o->outcome = outcome;
    o->device = dev;
    o->free_mem_after = dev >= 0 ? s->devs[dev]->free_mem : 0;
    o->in_use_warps_after = dev >= 0 ? s->devs[dev]->in_use_warps : 0;
    o->pending_index = pidx;
    o->handle = h;
}

/* submit (schedulers.py:89-95) */
int32_t o_submit(osched *s, const gs_probe *r, gs_decision *out) {
    int32_t dev;
    int32_t oc = try_one(s, r, &dev);
    if (oc == GS_DEFER) {
        if (s->pend_n == s->pend_cap) {
            s->pend_cap = s->pend_cap ? 2 * s->pend_cap : 64;
            s->pend = (gs_probe *)realloc(s->pend, sizeof(gs_probe) * s->pend_cap);
        }
        s->pend[s->pend_n++] = *r;
    }
    if (out) fill(out, s, oc, dev, -1, r->handle);
    return oc;
}

/* on_release (schedulers.py:97-113) */
int32_t o_on_release(osched *s, gs_decision *out, int32_t out_cap, int32_t *n_tried, int32_t *n_admitted) {
    int32_t n = s->pend_n, tried = 0, adm = 0, w = 0;
    char *gone = (char *)calloc(n ? n : 1, 1);
    for (int32_t i = 0; i < n; ++i) {
        int32_t dev;
        int32_t oc = try_one(s, &s->pend[i], &dev);
        tried = i + 1;
        if (out && i < out_cap) fill(&out[i], s, oc, dev, i, s->pend[i].handle);
        if (oc == GS_ASSIGN) {
            gone[i] = 1;
            adm++;
        } else if (!s->skip_ahead) {
            break;
        }
    }
    for (int32_t i = 0; i < n; ++i)
        if (!gone[i]) s->pend[w++] = s->pend[i];
    s->pend_n = w;
    free(gone);
    *n_tried = tried;
    *n_admitted = adm;
    return GS_OK;
}

/* job_ended (schedulers.py:115-123) */
void o_job_ended(osched *s, int32_t job) {
    for (int i = 0; i < s->n; ++i)
        if (s->sa_owner[i] == job) s->sa_owner[i] = -1;
    if (s->policy == GS_POLICY_CG && job >= 0 && job < s->claims_cap && s->claims[job] >= 0) {
        s->cg_counts[s->claims[job]] -= 1;
        s->claims[job] = -1;
    }
}

void o_job_state(const osched *s, int32_t *sa_owner, int32_t *cg_counts, int32_t *cg_cursor) {
    for (int i = 0; i < s->n; ++i) {
        sa_owner[i] = s->sa_owner[i];
        cg_counts[i] = s->cg_counts[i];
    }
    *cg_cursor = s->cg_cursor;
}

/* The placement sweep driver (BASELINE cfg 4; same stream as gs_sweep):
 * submit probe i (handle i); then if more than max_resident tasks are
 * resident or the queue is non-empty, release the oldest resident task and
 * re-drive the FIFO.  Event log entries: (kind, handle, device). */
int32_t o_sweep(osched *s, const gs_probe *probes, int32_t n, int32_t max_resident, int32_t *events,
                int64_t events_cap, int64_t *n_events) {
    int32_t *fifo = (int32_t *)malloc(sizeof(int32_t) * 2 * ((size_t)n + 1));
    int64_t head = 0, tail = 0, ne = 0;
    gs_decision *drain = NULL;
    int32_t drain_cap = 0;
#define EV(k, h, d)                                  \
    do {                                             \
        if (ne < events_cap) {                       \
            events[3 * ne] = (k);                    \
            events[3 * ne + 1] = (h);                \
            events[3 * ne + 2] = (d);                \
        }                                            \
        ne++;                                        \
    } while (0)
    for (int32_t i = 0; i < n; ++i) {
        gs_probe r = probes[i];
        r.handle = i;
        gs_decision o;
        int32_t oc = o_submit(s, &r, &o);
        if (oc == GS_ASSIGN) {
            fifo[2 * tail] = o.device;
            fifo[2 * tail + 1] = i;
            tail++;
        }
        EV(oc == GS_ASSIGN ? 0 : (oc == GS_DEFER ? 1 : 2), i, o.device);
        if (tail - head > max_resident || s->pend_n > 0) {
            if (tail > head) {
                o_release(s->devs[fifo[2 * head]], fifo[2 * head + 1], NULL);
                head++;
            }
            if (s->pend_n > drain_cap) {
                drain_cap = s->pend_n * 2;
                drain = (gs_decision *)realloc(drain, sizeof(gs_decision) * drain_cap);
            }
            int32_t tried, adm;
            o_on_release(s, drain, drain_cap, &tried, &adm);
            for (int32_t k = 0; k < tried; ++k)
                if (drain[k].outcome == GS_ASSIGN) {
                    fifo[2 * tail] = drain[k].device;
                    fifo[2 * tail + 1] = drain[k].handle;
                    tail++;
                    EV(3, drain[k].handle, drain[k].device);
                }
        }
    }
#undef EV
    free(fifo);
    free(drain);
    *n_events = ne;
    return GS_OK;
}
