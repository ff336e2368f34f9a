/*
 * kernels_cpu.c — CPU restatement of the co-scheduled workload kernels.
 *
 * TEST INFRASTRUCTURE ONLY (checker + timed CPU baseline; see gs_oracle.c).
 *
 * The reference ships no kernels ("parity unpinned"):
 * its jobs are catalog entries (gpushare/data/catalog.json) standing for
 * Rodinia v3.1 programs.  These restate the public
 * Rodinia algorithms — bfs, hotspot, srad (v2), kmeans, backprop, needle
 * (Needleman-Wunsch), lud — with the exact arithmetic order the GPU
 * kernels use (explicit fmaf, no contraction: build with
 * -ffp-contract=off), so integer outputs match bit for bit and float
 * outputs match to IEEE rounding (1e-5 relative is the stated bound).
 * Inputs come from the shared generator in include/gs_work.h.
 * OpenMP parallelises the data-parallel loops for the CPU baseline.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/gs_work.h"

static const int BLOSUM62[24][24] = GS_BLOSUM62_INIT;

/* ---- bfs: level-synchronous top-down (Rodinia bfs) --------------------- */
int32_t cpu_bfs(int64_t n, uint64_t seed, int32_t *level) {
    int32_t *q = (int32_t *)malloc(sizeof(int32_t) * n);
    int32_t *q2 = (int32_t *)malloc(sizeof(int32_t) * n);
    for (int64_t v = 0; v < n; ++v) level[v] = -1;
    level[0] = 0;
    q[0] = 0;
    int64_t qn = 1;
    int32_t depth = 0;
    while (qn > 0) {
        int64_t q2n = 0;
        for (int64_t k = 0; k < qn; ++k) {
            const int64_t v = q[k];
            for (int64_t e = v * GS_BFS_DEGREE; e < (v + 1) * GS_BFS_DEGREE; ++e) {
                const int32_t u = gs_bfs_col(seed, (uint64_t)e, n);
                if (level[u] < 0) {
                    level[u] = depth + 1;
                    q2[q2n++] = u;
                }
            }
        }
        int32_t *t = q;
        q = q2;
        q2 = t;
        qn = q2n;
        depth++;
    }
    free(q);
    free(q2);
    return depth;
}

/* ---- hotspot (Rodinia hotspot single_iteration) ------------------------- */
void cpu_hotspot(int64_t n, int32_t iters, uint64_t seed, float *out) {
    float cc, rx1, ry1, rz1;
    gs_hotspot_coeffs(&cc, &rx1, &ry1, &rz1);
    const int64_t nn = n * n;
    float *t = (float *)malloc(sizeof(float) * nn), *t2 = (float *)malloc(sizeof(float) * nn);
    float *p = (float *)malloc(sizeof(float) * nn);
#pragma omp parallel for
    for (int64_t i = 0; i < nn; ++i) {
        t[i] = gs_hotspot_temp0(seed, (uint64_t)i);
        p[i] = gs_hotspot_power(seed, (uint64_t)i);
    }
    for (int32_t it = 0; it < iters; ++it) {
#pragma omp parallel for
        for (int64_t r = 0; r < n; ++r) {
            const int64_t rn = r > 0 ? r - 1 : 0, rs = r < n - 1 ? r + 1 : n - 1;
            for (int64_t c = 0; c < n; ++c) {
                const int64_t cw = c > 0 ? c - 1 : 0, ce = c < n - 1 ? c + 1 : n - 1;
                const float tc = t[r * n + c];
                const float a = fmaf(-2.0f, tc, t[rs * n + c] + t[rn * n + c]);
                const float b = fmaf(-2.0f, tc, t[r * n + ce] + t[r * n + cw]);
                const float e = GS_HOTSPOT_AMB - tc;
                float d = fmaf(a, ry1, p[r * n + c]);
                d = fmaf(b, rx1, d);
                d = fmaf(e, rz1, d);
                t2[r * n + c] = fmaf(cc, d, tc);
            }
        }
        float *x = t;
        t = t2;
        t2 = x;
    }
    memcpy(out, t, sizeof(float) * nn);
    free(t);
    free(t2);
    free(p);
}

/* ---- srad v2 (Rodinia srad_v2: ROI statistics, diffusion coefficient,
 * update; ROI rows/cols 0..127) ------------------------------------------- */
void cpu_srad(int64_t n, int32_t iters, uint64_t seed, float *out) {
    const int64_t nn = n * n;
    float *J = (float *)malloc(sizeof(float) * nn), *J2 = (float *)malloc(sizeof(float) * nn);
    float *C = (float *)malloc(sizeof(float) * nn);
#pragma omp parallel for
    for (int64_t i = 0; i < nn; ++i) J[i] = gs_srad_j0(seed, (uint64_t)i);
    const int64_t roi = n < 128 ? n : 128;
    for (int32_t it = 0; it < iters; ++it) {
        double sum = 0.0, sum2 = 0.0;
        for (int64_t r = 0; r < roi; ++r)
            for (int64_t c = 0; c < roi; ++c) {
                const double v = J[r * n + c];
                sum += v;
                sum2 += v * v;
            }
        const double size = (double)(roi * roi);
        const double mean = sum / size;
        const double var = sum2 / size - mean * mean;
        const float q0sqr = (float)(var / (mean * mean));
#pragma omp parallel for
        for (int64_t r = 0; r < n; ++r) {
            const int64_t rn = r > 0 ? r - 1 : 0, rs = r < n - 1 ? r + 1 : n - 1;
            for (int64_t c = 0; c < n; ++c) {
                const int64_t cw = c > 0 ? c - 1 : 0, ce = c < n - 1 ? c + 1 : n - 1;
                const float jc = J[r * n + c];
                const float dN = J[rn * n + c] - jc, dS = J[rs * n + c] - jc;
                const float dW = J[r * n + cw] - jc, dE = J[r * n + ce] - jc;
                float g2 = dN * dN + dS * dS;
                g2 = g2 + dW * dW;
                g2 = g2 + dE * dE;
                g2 = g2 / (jc * jc);
                float l = dN + dS;
                l = l + dW;
                l = l + dE;
                l = l / jc;
                const float num = 0.5f * g2 - (1.0f / 16.0f) * (l * l);
                float den = 1.0f + 0.25f * l;
                const float qsqr = num / (den * den);
                den = (qsqr - q0sqr) / (q0sqr * (1.0f + q0sqr));
                float cv = 1.0f / (1.0f + den);
                cv = cv < 0.0f ? 0.0f : (cv > 1.0f ? 1.0f : cv);
                C[r * n + c] = cv;
            }
        }
#pragma omp parallel for
        for (int64_t r = 0; r < n; ++r) {
            const int64_t rn = r > 0 ? r - 1 : 0, rs = r < n - 1 ? r + 1 : n - 1;
            for (int64_t c = 0; c < n; ++c) {
                const int64_t cw = c > 0 ? c - 1 : 0, ce = c < n - 1 ? c + 1 : n - 1;
                const float jc = J[r * n + c];
                const float dN = J[rn * n + c] - jc, dS = J[rs * n + c] - jc;
                const float dW = J[r * n + cw] - jc, dE = J[r * n + ce] - jc;
                const float cN = C[r * n + c], cS = C[rs * n + c], cW = C[r * n + c], cE = C[r * n + ce];
                float d = cN * dN + cS * dS;
                d = d + cW * dW;
                d = d + cE * dE;
                J2[r * n + c] = jc + (0.25f * GS_SRAD_LAMBDA) * d;
            }
        }
        float *x = J;
        J = J2;
        J2 = x;
    }
    memcpy(out, J, sizeof(float) * nn);
    free(J);
    free(J2);
    free(C);
}

/* ---- kmeans (Rodinia kmeans: nearest-centroid assignment + recentering;
 * fixed-point exact centroid sums) ---------------------------------------- */
void cpu_kmeans(int64_t n, int32_t nf, int32_t iters, uint64_t seed, int32_t *membership, float *centroids) {
    const int K = GS_KMEANS_K;
    float *x = (float *)malloc(sizeof(float) * n * nf);
#pragma omp parallel for
    for (int64_t i = 0; i < n * nf; ++i) x[i] = gs_kmeans_feature(seed, (uint64_t)i);
    float *c = centroids;
    for (int k = 0; k < K; ++k)
        for (int f = 0; f < nf; ++f) c[k * nf + f] = x[(int64_t)f * n + k];
    int64_t *sumq = (int64_t *)malloc(sizeof(int64_t) * K * nf);
    int64_t cnt[GS_KMEANS_K];
    for (int32_t it = 0; it < iters; ++it) {
#pragma omp parallel for
        for (int64_t p = 0; p < n; ++p) {
            int best = 0;
            float bd = 0.0f;
            for (int k = 0; k < K; ++k) {
                float acc = 0.0f;
                for (int f = 0; f < nf; ++f) {
                    const float d = x[(int64_t)f * n + p] - c[k * nf + f];
                    acc = fmaf(d, d, acc);
                }
                if (k == 0 || acc < bd) {
                    bd = acc;
                    best = k;
                }
            }
            membership[p] = best;
        }
        memset(sumq, 0, sizeof(int64_t) * K * nf);
        memset(cnt, 0, sizeof(cnt));
        for (int64_t p = 0; p < n; ++p) cnt[membership[p]]++;
#pragma omp parallel for
        for (int f = 0; f < nf; ++f)
            for (int64_t p = 0; p < n; ++p)
                sumq[membership[p] * nf + f] += (int64_t)(x[(int64_t)f * n + p] * 16777216.0f);
        for (int k = 0; k < K; ++k)
            if (cnt[k] > 0)
                for (int f = 0; f < nf; ++f)
                    c[k * nf + f] = (float)((double)sumq[k * nf + f] / 16777216.0 / (double)cnt[k]);
    }
    free(x);
    free(sumq);
}

/* ---- backprop (Rodinia backprop: layerforward + adjust_weights; hidden
 * sums accumulated in double) --------------------------------------------- */
static float squash(float v) { return 1.0f / (1.0f + expf(-v)); }

void cpu_backprop(int64_t n_in, int32_t n_hid, int32_t iters, uint64_t seed, float *w1, float *w2, float *hidden,
                  float *output) {
    const int64_t ni = n_in + 1;
    float *x = (float *)malloc(sizeof(float) * ni);
    float *ow1 = (float *)calloc((size_t)n_hid * ni, sizeof(float));
    float ow2[64] = {0};
    float dh[64];
    for (int64_t i = 0; i < ni; ++i) x[i] = gs_bp_input(seed, (uint64_t)i);
    /* element-major [input][hidden] (Rodinia input_weights); value of (j, i) from index j * ni + i */
#pragma omp parallel for
    for (int64_t i = 0; i < ni; ++i)
        for (int j = 0; j < n_hid; ++j) w1[i * n_hid + j] = gs_bp_w1(seed, (uint64_t)(j * ni + i));
    for (int j = 0; j <= n_hid; ++j) w2[j] = gs_bp_w2(seed, (uint64_t)j);
    float o = 0.0f;
    for (int32_t it = 0; it < iters; ++it) {
        hidden[0] = 1.0f;
        /* double dot products, summed in fixed chunks of inputs (cache-friendly
         * over the element-major rows; deterministic chunk order) */
        {
            const int64_t chunk = 1 << 16;
            const int64_t nch = (ni + chunk - 1) / chunk;
            double *part = (double *)calloc((size_t)nch * n_hid, sizeof(double));
#pragma omp parallel for
            for (int64_t c = 0; c < nch; ++c) {
                double *pc = part + c * n_hid;
                const int64_t i1 = (c + 1) * chunk < ni ? (c + 1) * chunk : ni;
                for (int64_t i = c * chunk; i < i1; ++i)
                    for (int j = 0; j < n_hid; ++j) pc[j] += (double)w1[i * n_hid + j] * (double)x[i];
            }
            for (int j = 0; j < n_hid; ++j) {
                double s = 0.0;
                for (int64_t c = 0; c < nch; ++c) s += part[c * n_hid + j];
                hidden[j + 1] = squash((float)s);
            }
            free(part);
        }
        float so = 0.0f;
        for (int j = 0; j <= n_hid; ++j) so = fmaf(w2[j], hidden[j], so);
        o = squash(so);
        const float delta_o = o * (1.0f - o) * (GS_BP_TARGET - o);
        for (int j = 1; j <= n_hid; ++j) dh[j] = hidden[j] * (1.0f - hidden[j]) * (w2[j] * delta_o);
        for (int j = 0; j <= n_hid; ++j) {
            float t1 = GS_BP_ETA * delta_o;
            t1 = t1 * hidden[j];
            const float nd = t1 + GS_BP_MOMENTUM * ow2[j];
            w2[j] = w2[j] + nd;
            ow2[j] = nd;
        }
        float e[64];
        for (int j = 0; j < n_hid; ++j) e[j] = GS_BP_ETA * dh[j + 1];
#pragma omp parallel for
        for (int64_t i = 0; i < ni; ++i)
            for (int j = 0; j < n_hid; ++j) {
                const float t1 = e[j] * x[i];
                const float nd = t1 + GS_BP_MOMENTUM * ow1[i * n_hid + j];
                w1[i * n_hid + j] = w1[i * n_hid + j] + nd;
                ow1[i * n_hid + j] = nd;
            }
    }
    *output = o;
    free(x);
    free(ow1);
}

/* ---- needle (Rodinia nw: Needleman-Wunsch with BLOSUM62, penalty 10) ---- */
void cpu_needle(int64_t n, uint64_t seed, int32_t *score) {
    const int64_t w = n + 1;
    int32_t *s1 = (int32_t *)malloc(sizeof(int32_t) * w), *s2 = (int32_t *)malloc(sizeof(int32_t) * w);
    for (int64_t i = 1; i <= n; ++i) {
        s1[i] = gs_nw_seq(seed, (uint64_t)i);
        s2[i] = gs_nw_seq(seed + 1, (uint64_t)i);
    }
    for (int64_t j = 0; j < w; ++j) score[j] = (int32_t)(-j * GS_NW_PENALTY);
    for (int64_t i = 1; i < w; ++i) {
        score[i * w] = (int32_t)(-i * GS_NW_PENALTY);
        const int *brow = BLOSUM62[s1[i]];
        for (int64_t j = 1; j < w; ++j) {
            const int32_t a = score[(i - 1) * w + j - 1] + brow[s2[j]];
            const int32_t b = score[i * w + j - 1] - GS_NW_PENALTY;
            const int32_t c = score[(i - 1) * w + j] - GS_NW_PENALTY;
            int32_t m = a > b ? a : b;
            score[i * w + j] = m > c ? m : c;
        }
    }
    free(s1);
    free(s2);
}

/* ---- lud (Rodinia lud: blocked, no pivoting; diagonal / perimeter /
 * internal in the GPU's exact order) -------------------------------------- */
void cpu_lud(int64_t n, uint64_t seed, float *a) {
    const int64_t B = GS_LUD_BS;
#pragma omp parallel for
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) a[i * n + j] = gs_lud_a(seed, i, j, n);
    for (int64_t o = 0; o < n; o += B) {
        /* diagonal block: Doolittle row by row */
        for (int64_t i = 0; i < B; ++i) {
            for (int64_t j = i; j < B; ++j) {
                float acc = a[(o + i) * n + o + j];
                for (int64_t k = 0; k < i; ++k) acc = fmaf(-a[(o + i) * n + o + k], a[(o + k) * n + o + j], acc);
                a[(o + i) * n + o + j] = acc;
            }
            for (int64_t j = i + 1; j < B; ++j) {
                float acc = a[(o + j) * n + o + i];
                for (int64_t k = 0; k < i; ++k) acc = fmaf(-a[(o + j) * n + o + k], a[(o + k) * n + o + i], acc);
                a[(o + j) * n + o + i] = acc / a[(o + i) * n + o + i];
            }
        }
        if (o + B >= n) break;
        /* perimeter: U12 = L11^-1 A12 (columns), L21 = A21 U11^-1 (rows) */
#pragma omp parallel for
        for (int64_t j = o + B; j < n; ++j)
            for (int64_t i = 0; i < B; ++i) {
                float acc = a[(o + i) * n + j];
                for (int64_t k = 0; k < i; ++k) acc = fmaf(-a[(o + i) * n + o + k], a[(o + k) * n + j], acc);
                a[(o + i) * n + j] = acc;
            }
#pragma omp parallel for
        for (int64_t r = o + B; r < n; ++r)
            for (int64_t j = 0; j < B; ++j) {
                float acc = a[r * n + o + j];
                for (int64_t k = 0; k < j; ++k) acc = fmaf(-a[r * n + o + k], a[(o + k) * n + o + j], acc);
                a[r * n + o + j] = acc / a[(o + j) * n + o + j];
            }
        /* internal: A22 -= L21 U12 */
#pragma omp parallel for
        for (int64_t r = o + B; r < n; ++r)
            for (int64_t c = o + B; c < n; ++c) {
                float acc = 0.0f;
                for (int64_t k = 0; k < B; ++k) acc = fmaf(a[r * n + o + k], a[(o + k) * n + c], acc);
                a[r * n + c] = a[r * n + c] - acc;
            }
    }
}
