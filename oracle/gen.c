/*
 * gen.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Input generators for the reference arm of bench.py and for the parity
 * tests, so that the CPU reference can be fed the bench workload without
 * loading anything from the B200 package.  They restate the contract of the
 * package's synthetic generators (as_gen_powerlaw / as_fill_uniform,
 * include/autosage_b200.h): every row draws from its own counter-based
 * splitmix64 stream, so the output is a pure function of the arguments and
 * independent of the thread count.  tests/test_oracle.py checks that both
 * produce the same bytes.
 *
 * The reference's own generators (proj/src/generate.cpp:41-132: ER, hub-skew,
 * fixed hubs) have no heavy-tailed degree model, which the BASELINE configs
 * need (Reddit / Products shapes, Zipf sweeps); their libstdc++ <random>
 * streams are reached through oracle/_ref (ref_gen) instead.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

/* a splitmix64 stream: state advances by the golden gamma, output = mix */
typedef struct {
    uint64_t s;
} stream_t;

static uint64_t st_next(stream_t* r) {
    const uint64_t z = mix64(r->s);
    r->s += 0x9E3779B97F4A7C15ULL;
    return z;
}
static double st_unit(stream_t* r) { return (double)(st_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static float st_unitf(stream_t* r) { return (float)(st_next(r) >> 40) * (1.0f / 16777216.0f); }
static uint64_t st_below(stream_t* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)st_next(r) * n) >> 64);
}

/* ---- a tiny row-range thread pool ------------------------------------- */
typedef void (*range_fn)(void* ctx, uint64_t r0, uint64_t r1);
typedef struct {
    range_fn fn;
    void* ctx;
    uint64_t r0, r1;
} range_job;

static void* range_tramp(void* p) {
    range_job* j = (range_job*)p;
    j->fn(j->ctx, j->r0, j->r1);
    return NULL;
}

static void for_ranges(uint64_t n, range_fn fn, void* ctx) {
    long nt = sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if (nt > 64) nt = 64;
    if (n < 4096 || nt == 1) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t th[64];
    range_job jobs[64];
    const uint64_t chunk = (n + (uint64_t)nt - 1) / (uint64_t)nt;
    int started = 0;
    for (long t = 0; t < nt; ++t) {
        const uint64_t a = (uint64_t)t * chunk, b = a + chunk < n ? a + chunk : n;
        if (a >= b) break;
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].r0 = a;
        jobs[t].r1 = b;
        pthread_create(&th[t], NULL, range_tramp, &jobs[t]);
        ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

/* d distinct column ids of [0, m), ascending.  Dense requests (2d > m) pick
 * the m-d ids to leave out by rejection; sparse ones draw the deficit,
 * sort and de-duplicate until d distinct ids remain (so the result is the
 * sorted set of every id drawn). */
static void pick_columns(uint64_t d, uint64_t m, stream_t* r, uint32_t* out, uint32_t** buf,
                         uint64_t* cap) {
    if (d == 0) return;
    if (d >= m) {
        for (uint64_t i = 0; i < m; ++i) out[i] = (uint32_t)i;
        return;
    }
    if (2 * d > m) {
        unsigned char* skip = (unsigned char*)calloc(m, 1);
        for (uint64_t left = m - d; left;) {
            const uint64_t t = st_below(r, m);
            if (!skip[t]) {
                skip[t] = 1;
                --left;
            }
        }
        uint64_t o = 0;
        for (uint64_t i = 0; i < m; ++i)
            if (!skip[i]) out[o++] = (uint32_t)i;
        free(skip);
        return;
    }
    if (*cap < d) {
        free(*buf);
        *buf = (uint32_t*)malloc(d * sizeof(uint32_t));
        *cap = d;
    }
    uint32_t* s = *buf;
    uint64_t have = 0;
    while (have < d) {
        const uint64_t need = d - have;
        for (uint64_t i = 0; i < need; ++i) s[have + i] = (uint32_t)st_below(r, m);
        have += need;
        qsort(s, have, sizeof(uint32_t), cmp_u32);
        uint64_t u = 0;
        for (uint64_t i = 0; i < have; ++i)
            if (u == 0 || s[i] != s[u - 1]) s[u++] = s[i];
        have = u;
    }
    memcpy(out, s, d * sizeof(uint32_t));
}

typedef struct {
    uint64_t seed, d_min, cap;
    double expo;
    uint64_t* deg;
} deg_ctx;

static void deg_range(void* p, uint64_t r0, uint64_t r1) {
    deg_ctx* c = (deg_ctx*)p;
    for (uint64_t i = r0; i < r1; ++i) {
        stream_t r = {mix64(c->seed * 0x632BE59BD9B4E019ULL + i)};
        double u = st_unit(&r);
        if (u < 1e-300) u = 1e-300;
        double d = floor((double)c->d_min * pow(u, c->expo));
        if (!(d < (double)c->cap)) d = (double)c->cap;
        c->deg[i] = (uint64_t)d;
    }
}

typedef struct {
    uint64_t seed, n_cols;
    const uint64_t* rowptr;
    uint32_t* colind;
    float* val;
} col_ctx;

static void col_range(void* p, uint64_t r0, uint64_t r1) {
    col_ctx* c = (col_ctx*)p;
    uint32_t* buf = NULL;
    uint64_t cap = 0;
    for (uint64_t i = r0; i < r1; ++i) {
        stream_t r = {mix64(c->seed * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL * (i + 1))};
        const uint64_t e0 = c->rowptr[i], e1 = c->rowptr[i + 1];
        pick_columns(e1 - e0, c->n_cols, &r, c->colind + e0, &buf, &cap);
        if (c->val)
            for (uint64_t e = e0; e < e1; ++e) c->val[e] = st_unitf(&r);
    }
    free(buf);
}

int orc_gen_powerlaw_degrees(uint64_t n_rows, uint64_t n_cols, uint64_t nnz_target, double alpha,
                             uint64_t d_min, uint64_t d_max, uint64_t seed, uint64_t* rowptr) {
    if (!(alpha > 1.0)) return -1;
    if (n_cols == 0 && n_rows > 0 && nnz_target > 0) return -1;
    const uint64_t cap = d_max < n_cols ? d_max : n_cols;
    if (nnz_target > 0 && nnz_target > cap * n_rows) return -1;
    uint64_t* deg = (uint64_t*)malloc((n_rows ? n_rows : 1) * sizeof(uint64_t));
    deg_ctx dc = {seed, d_min, cap, -1.0 / (alpha - 1.0), deg};
    for_ranges(n_rows, deg_range, &dc);
    if (nnz_target > 0) {
        uint64_t total = 0;
        for (uint64_t i = 0; i < n_rows; ++i) total += deg[i];
        if (total > 0) {
            const double s = (double)nnz_target / (double)total;
            total = 0;
            for (uint64_t i = 0; i < n_rows; ++i) {
                const uint64_t d = (uint64_t)floor((double)deg[i] * s);
                deg[i] = d < cap ? d : cap;
                total += deg[i];
            }
        }
        /* settle the remainder one entry per row, cycling */
        uint64_t i = 0;
        while (total < nnz_target) {
            if (deg[i] < cap) ++deg[i], ++total;
            i = (i + 1) % n_rows;
        }
        while (total > nnz_target) {
            if (deg[i] > 0) --deg[i], --total;
            i = (i + 1) % n_rows;
        }
    }
    rowptr[0] = 0;
    for (uint64_t i = 0; i < n_rows; ++i) rowptr[i + 1] = rowptr[i] + deg[i];
    free(deg);
    return 0;
}

void orc_gen_powerlaw_columns(uint64_t n_rows, uint64_t n_cols, uint64_t seed, const uint64_t* rowptr,
                              uint32_t* colind, float* val) {
    col_ctx cc = {seed, n_cols, rowptr, colind, val};
    for_ranges(n_rows, col_range, &cc);
}

typedef struct {
    uint64_t seed;
    float* out;
} fill_ctx;

static void fill_range(void* p, uint64_t i0, uint64_t i1) {
    fill_ctx* c = (fill_ctx*)p;
    for (uint64_t i = i0; i < i1; ++i) {
        const uint64_t h = mix64(c->seed * 0xA0761D6478BD642FULL + i);
        c->out[i] = (float)(h >> 40) * (2.0f / 16777216.0f) - 1.0f;
    }
}

void orc_fill_uniform(float* out, uint64_t n, uint64_t seed) {
    fill_ctx fc = {seed, out};
    for_ranges(n, fill_range, &fc);
}
