/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference lmKAN forward
 * path, used solely as the parity checker (see lmkan_oracle.h). Compile with
 * -O2 -ffp-contract=off and no -ffast-math so every fp64 operation rounds
 * exactly as the reference's Release build does (proj/CMakeLists.txt:6-8 sets
 * no -march, so GCC emits no FMA there either).
 */
#include "lmkan_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* grid.hpp:14-17: one exp(-|x|); x > 0 ? 1 - t/2 : t/2. NaN falls into the
 * else-branch and propagates. */
double lmko_sigma(double x) {
    const double t = exp(-fabs(x));
    return x > 0.0 ? 1.0 - 0.5 * t : 0.5 * t;
}

/* grid.hpp:44-68 */
int lmko_build_grid(int G, double* points, double* inv_areas) {
    if (G < 3) return -1; /* grid.hpp:45-46 throws std::invalid_argument */
    for (int k = 0; k <= G; ++k) points[k] = 0.0;
    for (int k = 1; 2 * k < G; ++k) { /* grid.hpp:50-54, mirrored halves */
        const double v = log(2.0 * k / G);
        points[k] = v;
        points[G - k] = -v;
    }
    if (G % 2 == 0) points[G / 2] = 0.0;            /* grid.hpp:55 */
    points[0] = 2.0 * points[1] - points[2];         /* grid.hpp:56, ghost */
    points[G] = 2.0 * points[G - 1] - points[G - 2]; /* grid.hpp:57, ghost */
    for (int i1 = 0; i1 < G; ++i1) {                 /* grid.hpp:59-66 */
        const double h1 = points[i1 + 1] - points[i1];
        for (int i2 = 0; i2 < G; ++i2) {
            const double h2 = points[i2 + 1] - points[i2];
            inv_areas[i1 * G + i2] = 1.0 / (h1 * h2);
        }
    }
    return 0;
}

/* grid.hpp:72-75. static_cast<int>(floor(NaN)) is x86 cvttsd2si's INT_MIN,
 * which the clamp maps to 0; restated explicitly here. */
int lmko_interval_index(int G, double x) {
    const double f = floor(lmko_sigma(x) * G);
    const int i = isnan(f) ? INT32_MIN : (int)f;
    return i < 0 ? 0 : (i >= G ? G - 1 : i);
}

/* grid.hpp:87-101 */
void lmko_preamble(int G, const double* points, const double* inv_areas, double x1, double x2,
                   int* i1, int* i2, double* w) {
    const int a1 = lmko_interval_index(G, x1);
    const int a2 = lmko_interval_index(G, x2);
    const double a = points[a1 + 1] - x1;
    const double b = x1 - points[a1];
    const double c = points[a2 + 1] - x2;
    const double d = x2 - points[a2];
    const double inv = inv_areas[a1 * G + a2];
    w[0] = a * c * inv; /* w00 */
    w[1] = b * c * inv; /* w10 */
    w[2] = a * d * inv; /* w01 */
    w[3] = b * d * inv; /* w11 */
    *i1 = a1;
    *i2 = a2;
}

/* layer.hpp:96-101 applied to every row */
void lmko_locate(int G, const double* points, const double* inv_areas, int n_in, const double* X,
                 int64_t rows, int32_t* i1, int32_t* i2, double* w) {
    const int pairs = n_in / 2;
    for (int64_t r = 0; r < rows; ++r)
        for (int p = 0; p < pairs; ++p) {
            const int64_t k = r * pairs + p;
            int a1, a2;
            lmko_preamble(G, points, inv_areas, X[r * n_in + 2 * p], X[r * n_in + 2 * p + 1], &a1,
                          &a2, w + 4 * k);
            i1[k] = a1;
            i2[k] = a2;
        }
}

typedef struct {
    int n_in, n_out, G;
    const double *points, *inv_areas, *P;
    double gamma;
    const double* X;
    double* Y;
    int64_t rb, re;
} fwd_job;

/* layer.hpp:116-133 for rows [rb, re) */
static void* fwd_rows(void* arg) {
    const fwd_job* j = (const fwd_job*)arg;
    const int pairs = j->n_in / 2, n_out = j->n_out, G1 = j->G + 1;
    const size_t per_node = (size_t)pairs * n_out; /* layer.hpp:34-37 */
    int* ci1 = (int*)malloc(sizeof(int) * pairs);
    int* ci2 = (int*)malloc(sizeof(int) * pairs);
    double* cw = (double*)malloc(sizeof(double) * 4 * pairs);
    for (int64_t r = j->rb; r < j->re; ++r) {
        const double* x = j->X + r * j->n_in;
        for (int p = 0; p < pairs; ++p) /* stage 1: row_preambles */
            lmko_preamble(j->G, j->points, j->inv_areas, x[2 * p], x[2 * p + 1], &ci1[p], &ci2[p],
                          cw + 4 * p);
        double* y = j->Y + r * n_out;
        for (int q = 0; q < n_out; ++q) y[q] = 0.0;
        for (int p = 0; p < pairs; ++p) { /* stage 2, layer.hpp:122-130 */
            const double w00 = cw[4 * p], w10 = cw[4 * p + 1], w01 = cw[4 * p + 2],
                         w11 = cw[4 * p + 3];
            const double* p00 = j->P + ((size_t)ci1[p] * G1 + ci2[p]) * per_node + (size_t)p * n_out;
            const double* p10 = p00 + (size_t)G1 * per_node;
            const double* p01 = p00 + per_node;
            const double* p11 = p10 + per_node;
            for (int q = 0; q < n_out; ++q)
                y[q] += w00 * p00[q] + w10 * p10[q] + w01 * p01[q] + w11 * p11[q];
        }
        for (int q = 0; q < n_out; ++q) y[q] *= j->gamma; /* layer.hpp:131 */
    }
    free(ci1);
    free(ci2);
    free(cw);
    return NULL;
}

void lmko_forward(int n_in, int n_out, int G, const double* points, const double* inv_areas,
                  const double* P, double gamma, const double* X, int64_t rows, double* Y,
                  int threads) {
    if (threads < 1) threads = 1;
    if (threads > rows) threads = rows > 0 ? (int)rows : 1;
    fwd_job* jobs = (fwd_job*)calloc((size_t)threads, sizeof(fwd_job));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    const int64_t chunk = (rows + threads - 1) / threads; /* threading.hpp:33-39 */
    for (int t = 0; t < threads; ++t) {
        fwd_job* j = &jobs[t];
        j->n_in = n_in; j->n_out = n_out; j->G = G;
        j->points = points; j->inv_areas = inv_areas; j->P = P;
        j->gamma = gamma; j->X = X; j->Y = Y;
        j->rb = t * chunk < rows ? t * chunk : rows;
        j->re = j->rb + chunk < rows ? j->rb + chunk : rows;
    }
    if (threads == 1) {
        fwd_rows(&jobs[0]);
    } else {
        for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, fwd_rows, &jobs[t]);
        for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    }
    free(jobs);
    free(tid);
}

/* layer.hpp:141-202, one worker (the row loop of worker 0 accumulates straight
 * into dP, layer.hpp:162-163; the per-q loop order and expression grouping of
 * layer.hpp:182-191 are kept, so with -ffp-contract=off this is bit-identical
 * to the reference at workers = 1). */
void lmko_backward(int n_in, int n_out, int G, const double* points, const double* inv_areas,
                   const double* P, double gamma, const double* X, const double* dY, int64_t rows,
                   double* dP, double* dX) {
    const int pairs = n_in / 2;
    const int G1 = G + 1;
    const size_t per_node = (size_t)pairs * n_out;
    for (int64_t r = 0; r < rows; ++r) {
        const double* x = X + r * n_in;
        const double* g = dY + r * n_out;
        for (int p = 0; p < pairs; ++p) {
            int i1, i2;
            double w[4];
            lmko_preamble(G, points, inv_areas, x[2 * p], x[2 * p + 1], &i1, &i2, w);
            const size_t base = ((size_t)i1 * G1 + i2) * per_node + (size_t)p * n_out;
            double* d00 = dP + base;
            double* d10 = dP + base + (size_t)G1 * per_node;
            double* d01 = dP + base + per_node;
            double* d11 = d10 + per_node;
            const double* p00 = P + base;
            const double* p10 = p00 + (size_t)G1 * per_node;
            const double* p01 = p00 + per_node;
            const double* p11 = p10 + per_node;
            const double inv = inv_areas[i1 * G + i2];
            const double r2 = points[i2 + 1] - x[2 * p + 1];
            const double l2 = x[2 * p + 1] - points[i2];
            const double r1 = points[i1 + 1] - x[2 * p];
            const double l1 = x[2 * p] - points[i1];
            double acc1 = 0.0, acc2 = 0.0;
            for (int q = 0; q < n_out; ++q) {
                const double gq = gamma * g[q];
                d00[q] += w[0] * gq;
                d10[q] += w[1] * gq;
                d01[q] += w[2] * gq;
                d11[q] += w[3] * gq;
                acc1 += gq * ((p10[q] - p00[q]) * r2 + (p11[q] - p01[q]) * l2);
                acc2 += gq * ((p01[q] - p00[q]) * r1 + (p11[q] - p10[q]) * l1);
            }
            if (dX) {
                dX[r * n_in + 2 * p] = acc1 * inv;
                dX[r * n_in + 2 * p + 1] = acc2 * inv;
            }
        }
    }
}

/* ---- threshold derivation (not in the reference; derived FROM it) ---- */

/* Monotone maps between finite floating values and unsigned keys. */
static uint64_t key64(double x) {
    uint64_t u;
    memcpy(&u, &x, 8);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
static double unkey64(uint64_t k) {
    const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double x;
    memcpy(&x, &u, 8);
    return x;
}
static uint32_t key32(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    return (u >> 31) ? ~u : (u | 0x80000000u);
}
static float unkey32(uint32_t k) {
    const uint32_t u = (k >> 31) ? (k & 0x7fffffffu) : ~k;
    float x;
    memcpy(&x, &u, 4);
    return x;
}

int lmko_thresholds_f64(int G, double* t) {
    if (G < 3) return -1;
    for (int k = 1; k <= G - 1; ++k) {
        uint64_t lo = key64(-INFINITY), hi = key64(INFINITY); /* idx(lo)=0<k, idx(hi)=G-1>=k */
        while (hi - lo > 1) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (lmko_interval_index(G, unkey64(mid)) >= k) hi = mid; else lo = mid;
        }
        t[k - 1] = unkey64(hi);
    }
    return 0;
}

int lmko_thresholds_f32(int G, float* t) {
    if (G < 3) return -1;
    for (int k = 1; k <= G - 1; ++k) {
        uint32_t lo = key32(-INFINITY), hi = key32(INFINITY);
        while (hi - lo > 1) {
            const uint32_t mid = lo + (hi - lo) / 2;
            if (lmko_interval_index(G, (double)unkey32(mid)) >= k) hi = mid; else lo = mid;
        }
        t[k - 1] = unkey32(hi);
    }
    return 0;
}

typedef struct {
    int G;
    const float* t;
    uint64_t lo, hi; /* inclusive bit-pattern range */
    int64_t bad;
} verify_job;

static void* verify_range(void* arg) {
    verify_job* j = (verify_job*)arg;
    int64_t bad = 0;
    for (uint64_t b = j->lo; b <= j->hi; ++b) {
        const uint32_t bits = (uint32_t)b;
        float x;
        memcpy(&x, &bits, 4);
        int cnt = 0;
        for (int k = 0; k < j->G - 1; ++k) cnt += x >= j->t[k];
        if (cnt != lmko_interval_index(j->G, (double)x)) ++bad;
    }
    j->bad = bad;
    return NULL;
}

int64_t lmko_verify_thresholds_f32(int G, const float* t, uint32_t lo, uint32_t hi, int threads) {
    if (threads < 1) threads = 1;
    const uint64_t n = (uint64_t)hi - lo + 1;
    if ((uint64_t)threads > n) threads = (int)n;
    verify_job* jobs = (verify_job*)calloc((size_t)threads, sizeof(verify_job));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    const uint64_t chunk = (n + threads - 1) / threads;
    for (int i = 0; i < threads; ++i) {
        jobs[i].G = G;
        jobs[i].t = t;
        jobs[i].lo = lo + i * chunk;
        jobs[i].hi = jobs[i].lo + chunk - 1 > hi ? hi : jobs[i].lo + chunk - 1;
        pthread_create(&tid[i], NULL, verify_range, &jobs[i]);
    }
    int64_t bad = 0;
    for (int i = 0; i < threads; ++i) {
        pthread_join(tid[i], NULL);
        bad += jobs[i].bad;
    }
    free(jobs);
    free(tid);
    return bad;
}
