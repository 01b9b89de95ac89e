/*
 * vlc_oracle.c -- CPU oracle for the VL-Cache compress + decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2410_23317_b200/ links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and only as the checker.
 *
 * This is a plain-C restatement of the reference's compiled kernels
 * (reference: pkg/src/vlcache/_kernels/_core.pyx).  The arithmetic order is
 * reproduced on purpose so that, built with the same contraction behaviour
 * (-O3 -mfma, GNU default -ffp-contract=fast), it is bit-identical to the
 * reference extension; tests/test_oracle_golden.py pins that against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py) and
 * against oracle/_ref when it is present.
 *
 * Precision contract restated (reference attention.py:3-9, _core.pyx:1-12):
 *   logit   = (float)( fp64 dot(q, k) * (1/sqrt(d)) )          _core.pyx:144-145
 *   pass 1  : running f32 row max, f64 row sum with exp(double)  _core.pyx:147-155
 *             rescale, tile sums of (double)expf(l - max)
 *   pass 2  : e = expf(l - rowmax); col += (double)e * (1/rowsum) _core.pyx:199-205
 *             below += ((double)e < p); causal += 1
 *   decode  : f32 dots, expf, f64 denominator, w = (float)(e/s),  _core.pyx:245-278
 *             f32 accumulation in key order
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

/* fp64 dot with sixteen interleaved accumulators combined as a balanced tree
 * (reference _core.pyx:34-62).  Sixteen independent chains, lane t%16. */
static double dot16_f64(const double *restrict x, const double *restrict y, ptrdiff_t n)
{
    double acc[16] = {0};
    ptrdiff_t t = 0;
    for (; t + 16 <= n; t += 16)
        for (int c = 0; c < 16; ++c)
            acc[c] += x[t + c] * y[t + c];
    for (; t < n; ++t)
        acc[0] += x[t] * y[t];
    double lo = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    double hi = ((acc[8] + acc[9]) + (acc[10] + acc[11])) + ((acc[12] + acc[13]) + (acc[14] + acc[15]));
    return lo + hi;
}

/* Same shape in float32 (reference _core.pyx:64-92). */
static float dot16_f32(const float *restrict x, const float *restrict y, ptrdiff_t n)
{
    float acc[16] = {0};
    ptrdiff_t t = 0;
    for (; t + 16 <= n; t += 16)
        for (int c = 0; c < 16; ++c)
            acc[c] += x[t + c] * y[t + c];
    for (; t < n; ++t)
        acc[0] += x[t] * y[t];
    float lo = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    float hi = ((acc[8] + acc[9]) + (acc[10] + acc[11])) + ((acc[12] + acc[13]) + (acc[14] + acc[15]));
    return lo + hi;
}

static void widen(const float *src, double *dst, ptrdiff_t count)
{
    for (ptrdiff_t i = 0; i < count; ++i)
        dst[i] = (double)src[i];
}

static ptrdiff_t min_pd(ptrdiff_t a, ptrdiff_t b) { return a < b ? a : b; }

/*
 * Tiled two-pass attention statistics for one (layer, head) query window.
 * q [w, d], keys [n, d] (row-major float32); row r has absolute index q_base+r
 * and attends to keys j <= q_base + r.  Outputs are written (not accumulated):
 * row_max f32[w], row_sum f64[w], col_score f64[n], below i64[n], causal i64[n].
 * Returns 0, or -1 on allocation failure.
 */
int vlo_stats_tiled(const float *q, ptrdiff_t w, const float *keys, ptrdiff_t n, ptrdiff_t d,
                    ptrdiff_t q_base, double p, ptrdiff_t tile,
                    float *row_max, double *row_sum, double *col_score,
                    int64_t *below, int64_t *causal)
{
    const double inv = 1.0 / sqrt((double)d);
    float *lbuf = (float *)malloc((size_t)tile * sizeof(float));
    double *qbuf = (double *)malloc((size_t)(tile * d) * sizeof(double));
    double *kbuf = (double *)malloc((size_t)(tile * d) * sizeof(double));
    if (!lbuf || !qbuf || !kbuf) {
        free(lbuf); free(qbuf); free(kbuf);
        return -1;
    }
    for (ptrdiff_t r = 0; r < w; ++r) { row_max[r] = -INFINITY; row_sum[r] = 0.0; }
    memset(col_score, 0, (size_t)n * sizeof(double));
    memset(below, 0, (size_t)n * sizeof(int64_t));
    memset(causal, 0, (size_t)n * sizeof(int64_t));

    /* pass 1: query tiles outer, key tiles inner, online max / sum
     * (reference _core.pyx:110-157) */
    for (ptrdiff_t q0 = 0; q0 < w; q0 += tile) {
        ptrdiff_t q1 = min_pd(q0 + tile, w);
        widen(q + q0 * d, qbuf, (q1 - q0) * d);
        for (ptrdiff_t k0 = 0; k0 < n && k0 <= q_base + q1 - 1; k0 += tile) {
            ptrdiff_t k1 = min_pd(k0 + tile, n);
            widen(keys + k0 * d, kbuf, (k1 - k0) * d);
            for (ptrdiff_t r = q0; r < q1; ++r) {
                ptrdiff_t jend = min_pd(q_base + r + 1, k1);
                if (k0 >= jend)
                    continue;
                const double *qr = qbuf + (r - q0) * d;
                float tmax = -FLT_MAX;
                for (ptrdiff_t j = k0; j < jend; ++j) {
                    float l = (float)(dot16_f64(qr, kbuf + (j - k0) * d, d) * inv);
                    lbuf[j - k0] = l;
                    if (l > tmax) tmax = l;
                }
                if (tmax > row_max[r]) {
                    row_sum[r] *= exp((double)row_max[r] - (double)tmax);
                    row_max[r] = tmax;
                }
                double s = 0.0;
                for (ptrdiff_t j = k0; j < jend; ++j)
                    s += (double)expf(lbuf[j - k0] - row_max[r]);
                row_sum[r] += s;
            }
        }
    }

    /* pass 2: key tiles outer, query tiles inner, column statistics against
     * the stored row max / sum (reference _core.pyx:160-207) */
    for (ptrdiff_t k0 = 0; k0 < n; k0 += tile) {
        ptrdiff_t k1 = min_pd(k0 + tile, n);
        widen(keys + k0 * d, kbuf, (k1 - k0) * d);
        for (ptrdiff_t q0 = 0; q0 < w; q0 += tile) {
            ptrdiff_t q1 = min_pd(q0 + tile, w);
            if (k0 > q_base + q1 - 1)
                continue;
            widen(q + q0 * d, qbuf, (q1 - q0) * d);
            for (ptrdiff_t r = q0; r < q1; ++r) {
                ptrdiff_t jend = min_pd(q_base + r + 1, k1);
                const double *qr = qbuf + (r - q0) * d;
                for (ptrdiff_t j = k0; j < jend; ++j)
                    lbuf[j - k0] = (float)(dot16_f64(qr, kbuf + (j - k0) * d, d) * inv);
                float rmax = row_max[r];
                double inv_sum = 1.0 / row_sum[r];
                for (ptrdiff_t j = k0; j < jend; ++j) {
                    float e = expf(lbuf[j - k0] - rmax);
                    col_score[j] += (double)e * inv_sum;
                    below[j] += ((double)e < p);
                    causal[j] += 1;
                }
            }
        }
    }
    free(lbuf); free(qbuf); free(kbuf);
    return 0;
}

/*
 * One decode attention pass: q [g, d] against keys/values [n, d]; out [g, d]
 * (reference _core.pyx:245-278).  Returns 0, or -1 on allocation failure.
 */
int vlo_decode_step(const float *q, ptrdiff_t g, const float *keys, const float *values,
                    ptrdiff_t n, ptrdiff_t d, float *out)
{
    float *ebuf = (float *)malloc((size_t)(n > 0 ? n : 1) * sizeof(float));
    if (!ebuf)
        return -1;
    const float inv = (float)(1.0 / sqrt((double)d));
    memset(out, 0, (size_t)(g * d) * sizeof(float));
    for (ptrdiff_t h = 0; h < g; ++h) {
        float mx = -FLT_MAX;
        for (ptrdiff_t j = 0; j < n; ++j) {
            float l = dot16_f32(q + h * d, keys + j * d, d) * inv;
            ebuf[j] = l;
            if (l > mx) mx = l;
        }
        double s = 0.0;
        for (ptrdiff_t j = 0; j < n; ++j) {
            float e = expf(ebuf[j] - mx);
            ebuf[j] = e;
            s += (double)e;
        }
        float *o = out + h * d;
        for (ptrdiff_t j = 0; j < n; ++j) {
            float wj = (float)((double)ebuf[j] / s);
            const float *v = values + j * d;
            for (ptrdiff_t t = 0; t < d; ++t)
                o[t] += wj * v[t];
        }
    }
    free(ebuf);
    return 0;
}

/* Smallest float32 x with (double)expf(x) >= p, i.e. the threshold t* such
 * that "(double)expf(x) < p" <=> "x < t*" for the monotone libm expf
 * (the below-threshold test of reference _core.pyx:201-204). */
float vlo_threshold_logit(double p)
{
    float x = (float)log(p);
    /* walk down while still >= p, then up until >= p */
    while ((double)expf(x) >= p)
        x = nextafterf(x, -INFINITY);
    while ((double)expf(x) < p)
        x = nextafterf(x, INFINITY);
    return x;
}
