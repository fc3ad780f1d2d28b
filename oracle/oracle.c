/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain-C restatement of the AutoSAGE reference CPU algorithm.  Written for
 * clarity and exactness, not speed: single-threaded, the same arithmetic in
 * the same order as the reference (no FMA contraction: build with
 * -ffp-contract=off, as the reference's x86-64 build emits mulsd/addsd).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- SpMM -- */

/* src/kernels.cpp:210-228 */
void orc_spmm_baseline(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                       uint64_t n_rows, const float* b, uint64_t f, float* c) {
    double* acc = (double*)calloc(f ? f : 1, sizeof(double));
    for (uint64_t i = 0; i < n_rows; ++i) {
        for (uint64_t t = 0; t < f; ++t) acc[t] = 0.0;
        for (uint64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            const float* brow = b + (uint64_t)colind[e] * f;
            const double v = val ? (double)val[e] : 1.0;
            for (uint64_t t = 0; t < f; ++t) acc[t] += v * (double)brow[t];
        }
        for (uint64_t t = 0; t < f; ++t) c[i * f + t] = (float)acc[t];
    }
    free(acc);
}

/* src/kernels.cpp:260-334 (pieces: :129-142, reduce: :310-332) */
void orc_spmm_hubsplit(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                       uint64_t n_rows, const float* b, uint64_t f, uint64_t hub_t, float* c) {
    double* acc = (double*)calloc(f ? f : 1, sizeof(double));
    double* part = (double*)calloc(f ? f : 1, sizeof(double));
    for (uint64_t i = 0; i < n_rows; ++i) {
        const uint64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        if (e1 - e0 < hub_t) {
            for (uint64_t t = 0; t < f; ++t) acc[t] = 0.0;
            for (uint64_t e = e0; e < e1; ++e) {
                const float* brow = b + (uint64_t)colind[e] * f;
                const double v = val ? (double)val[e] : 1.0;
                for (uint64_t t = 0; t < f; ++t) acc[t] += v * (double)brow[t];
            }
            for (uint64_t t = 0; t < f; ++t) c[i * f + t] = (float)acc[t];
            continue;
        }
        /* heavy row: s starts at 0.0 and adds each piece partial in order */
        for (uint64_t t = 0; t < f; ++t) acc[t] = 0.0; /* acc = running s */
        for (uint64_t p0 = e0; p0 < e1; p0 += ORC_HUB_NNZ_CHUNK) {
            const uint64_t p1 = (p0 + ORC_HUB_NNZ_CHUNK < e1) ? p0 + ORC_HUB_NNZ_CHUNK : e1;
            for (uint64_t t = 0; t < f; ++t) part[t] = 0.0;
            for (uint64_t e = p0; e < p1; ++e) {
                const float* brow = b + (uint64_t)colind[e] * f;
                const double v = val ? (double)val[e] : 1.0;
                for (uint64_t t = 0; t < f; ++t) part[t] += v * (double)brow[t];
            }
            for (uint64_t t = 0; t < f; ++t) acc[t] += part[t];
        }
        for (uint64_t t = 0; t < f; ++t) c[i * f + t] = (float)acc[t];
    }
    free(acc);
    free(part);
}

/* --------------------------------------------------------------- SDDMM -- */

/* src/kernels.cpp:45-47 */
static uint64_t effective_tile(uint64_t f_tile, uint64_t f) {
    uint64_t fm = f > 1 ? f : 1;
    uint64_t t = f_tile < fm ? f_tile : fm;
    return t > 1 ? t : 1;
}

/* src/kernels.cpp:103-127 */
static double sddmm_dot(const float* xr, const float* yr, uint64_t f, uint64_t ft, int vec) {
    double acc = 0.0;
    for (uint64_t b0 = 0; b0 < f; b0 += ft) {
        const uint64_t fw = (ft < f - b0) ? ft : f - b0;
        if (vec) {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            const uint64_t fw4 = fw & ~(uint64_t)3;
            uint64_t t = 0;
            for (; t < fw4; t += 4) {
                a0 += (double)xr[b0 + t + 0] * (double)yr[b0 + t + 0];
                a1 += (double)xr[b0 + t + 1] * (double)yr[b0 + t + 1];
                a2 += (double)xr[b0 + t + 2] * (double)yr[b0 + t + 2];
                a3 += (double)xr[b0 + t + 3] * (double)yr[b0 + t + 3];
            }
            double tail = 0.0;
            for (; t < fw; ++t) tail += (double)xr[b0 + t] * (double)yr[b0 + t];
            acc += ((a0 + a1) + (a2 + a3)) + tail;
        } else {
            for (uint64_t t = 0; t < fw; ++t) acc += (double)xr[b0 + t] * (double)yr[b0 + t];
        }
    }
    return acc;
}

/* src/kernels.cpp:336-355 (vec=0) and :357-429 (tiling/vec per sddmm_dot).
 * HubSplit only redistributes work for SDDMM (pieces write disjoint
 * outputs, :414-427), so it needs no separate restatement. */
void orc_sddmm(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
               const float* x, const float* y, uint64_t f, uint64_t f_tile, int vec,
               float* out) {
    const uint64_t ft = effective_tile(f_tile, f);
    for (uint64_t i = 0; i < n_rows; ++i) {
        const float* xr = x + i * f;
        for (uint64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            const float* yr = y + (uint64_t)colind[e] * f;
            out[e] = (float)sddmm_dot(xr, yr, f, ft, vec);
        }
    }
}

/* ------------------------------------------------------------- softmax -- */

/* src/kernels.cpp:431-461; std::max(a,b) is (a < b) ? b : a. */
void orc_row_softmax(const uint64_t* rowptr, uint64_t n_rows, const float* vals_in,
                     float* vals_out) {
    for (uint64_t i = 0; i < n_rows; ++i) {
        const uint64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        if (e0 == e1) continue;
        float mx = vals_in[e0];
        for (uint64_t e = e0 + 1; e < e1; ++e) mx = (mx < vals_in[e]) ? vals_in[e] : mx;
        double sum = 0.0;
        for (uint64_t e = e0; e < e1; ++e) {
            const float ex = (float)exp((double)vals_in[e] - (double)mx);
            vals_out[e] = ex;
            sum += (double)ex;
        }
        for (uint64_t e = e0; e < e1; ++e) vals_out[e] = (float)((double)vals_out[e] / sum);
    }
}

/* ----------------------------------------------------------- attention -- */

/* src/attention.cpp:9-40: scores = sddmm(pattern, q, k) -> row_softmax ->
 * spmm(p, v).  Pattern values are ignored; empty rows give zero rows. */
void orc_attention(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
                   const float* q, const float* k, uint64_t f, const float* v, uint64_t fv,
                   uint64_t sddmm_ft, int sddmm_vec, uint64_t spmm_hub_t, float* out) {
    const uint64_t nnz = rowptr[n_rows];
    float* scores = (float*)malloc((nnz ? nnz : 1) * sizeof(float));
    float* p = (float*)malloc((nnz ? nnz : 1) * sizeof(float));
    orc_sddmm(rowptr, colind, n_rows, q, k, f, sddmm_ft, sddmm_vec, scores);
    orc_row_softmax(rowptr, n_rows, scores, p);
    if (spmm_hub_t == 0)
        orc_spmm_baseline(rowptr, colind, p, n_rows, v, fv, out);
    else
        orc_spmm_hubsplit(rowptr, colind, p, n_rows, v, fv, spmm_hub_t, out);
    free(scores);
    free(p);
}

/* ----------------------------------------------------------- graph_sig -- */

/* src/cache.cpp:18-29 */
static uint64_t fnv_bytes(uint64_t h, const void* data, uint64_t n) {
    const unsigned char* p = (const unsigned char*)data;
    for (uint64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    return h;
}

/* src/cache.cpp:66-74 */
uint64_t orc_graph_sig(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
                       uint64_t n_cols, uint64_t nnz) {
    uint64_t h = 14695981039346656037ULL;
    h = fnv_bytes(h, &n_rows, 8);
    h = fnv_bytes(h, &n_cols, 8);
    h = fnv_bytes(h, &nnz, 8);
    h = fnv_bytes(h, rowptr, (n_rows + 1) * 8);
    h = fnv_bytes(h, colind, nnz * 4);
    return h;
}

/* ------------------------------------------------------------ features -- */

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return (x > y) - (x < y);
}

/* src/csr.cpp:98-104: rank = ceil(q*n), clamped to [1, n] */
static uint64_t nearest_rank(const uint64_t* sorted, uint64_t n, double q) {
    if (n == 0) return 0;
    uint64_t rank = (uint64_t)ceil(q * (double)n);
    if (rank == 0) rank = 1;
    if (rank > n) rank = n;
    return sorted[rank - 1];
}

/* src/csr.cpp:108-135 */
void orc_extract_features(const uint64_t* rowptr, uint64_t n_rows, uint64_t n_cols,
                          uint64_t hub_t, orc_features* gf) {
    memset(gf, 0, sizeof *gf);
    gf->n_rows = n_rows;
    gf->n_cols = n_cols;
    gf->nnz = rowptr[n_rows];
    gf->hub_threshold = hub_t;
    if (n_rows == 0) return;
    uint64_t* deg = (uint64_t*)malloc(n_rows * sizeof(uint64_t));
    uint64_t heavy = 0, empty = 0;
    for (uint64_t i = 0; i < n_rows; ++i) {
        deg[i] = rowptr[i + 1] - rowptr[i];
        if (deg[i] >= hub_t) ++heavy;
        if (deg[i] == 0) ++empty;
    }
    qsort(deg, n_rows, sizeof(uint64_t), cmp_u64);
    gf->deg_p25 = nearest_rank(deg, n_rows, 0.25);
    gf->deg_p50 = nearest_rank(deg, n_rows, 0.50);
    gf->deg_p75 = nearest_rank(deg, n_rows, 0.75);
    gf->deg_p90 = nearest_rank(deg, n_rows, 0.90);
    gf->deg_p99 = nearest_rank(deg, n_rows, 0.99);
    gf->deg_max = deg[n_rows - 1];
    gf->mean_degree = (double)gf->nnz / (double)n_rows;
    gf->heavy_row_fraction = (double)heavy / (double)n_rows;
    gf->empty_row_fraction = (double)empty / (double)n_rows;
    free(deg);
}

/* ------------------------------------------------------------ sampling -- */

/* src/generate.cpp:134-153.  std::stable_sort by degree descending equals a
 * stable counting sort on (max_degree - degree). */
uint64_t orc_sample_row_indices(const uint64_t* rowptr, uint64_t n_rows, double frac,
                                uint64_t min_rows, uint64_t* rows_out) {
    if (frac <= 0.0 || frac > 1.0) return UINT64_MAX;
    if (n_rows == 0) return 0;
    uint64_t s = (uint64_t)ceil(frac * (double)n_rows);
    if (s < min_rows) s = min_rows;
    if (s > n_rows) s = n_rows;

    /* stable sort by degree descending: merge sort on indices */
    uint64_t* order = (uint64_t*)malloc(n_rows * sizeof(uint64_t));
    uint64_t* tmp = (uint64_t*)malloc(n_rows * sizeof(uint64_t));
    for (uint64_t i = 0; i < n_rows; ++i) order[i] = i;
    for (uint64_t width = 1; width < n_rows; width *= 2) {
        for (uint64_t lo = 0; lo < n_rows; lo += 2 * width) {
            uint64_t mid = lo + width < n_rows ? lo + width : n_rows;
            uint64_t hi = lo + 2 * width < n_rows ? lo + 2 * width : n_rows;
            uint64_t a = lo, b = mid, o = lo;
            while (a < mid && b < hi) {
                uint64_t da = rowptr[order[a] + 1] - rowptr[order[a]];
                uint64_t db = rowptr[order[b] + 1] - rowptr[order[b]];
                /* take b first only when strictly greater degree (stability) */
                if (db > da) tmp[o++] = order[b++];
                else tmp[o++] = order[a++];
            }
            while (a < mid) tmp[o++] = order[a++];
            while (b < hi) tmp[o++] = order[b++];
        }
        uint64_t* sw = order;
        order = tmp;
        tmp = sw;
    }
    uint64_t stride = n_rows / s;
    if (stride < 1) stride = 1;
    for (uint64_t r = 0; r < s; ++r) rows_out[r] = order[r * stride];
    free(order);
    free(tmp);
    return s;
}

/* src/generate.cpp:155-176 */
uint64_t orc_slice_rows(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                        const uint64_t* rows, uint64_t n_sel, uint64_t* rowptr_out,
                        uint32_t* colind_out, float* val_out) {
    uint64_t nnz = 0;
    rowptr_out[0] = 0;
    for (uint64_t r = 0; r < n_sel; ++r) {
        const uint64_t i = rows[r];
        const uint64_t d = rowptr[i + 1] - rowptr[i];
        if (colind_out) memcpy(colind_out + nnz, colind + rowptr[i], d * sizeof(uint32_t));
        if (val && val_out) memcpy(val_out + nnz, val + rowptr[i], d * sizeof(float));
        nnz += d;
        rowptr_out[r + 1] = nnz;
    }
    return nnz;
}

/* ---------------------------------------------------------------- cost -- */

/* src/cost.cpp:9-43 */
double orc_estimate_cost(const orc_variant* v, const orc_features* gf, uint64_t f,
                         double bw_eff, double flops_eff, uint64_t cores) {
    if (bw_eff <= 0.0 || flops_eff <= 0.0) return -1.0; /* reference throws */
    if (gf->nnz == 0) return 0.0;
    const double nnz = (double)gf->nnz;
    const double n = (double)gf->n_rows;
    const double fd = (double)f;
    double bytes;
    if (v->op == 0)
        bytes = 8.0 * nnz + 4.0 * nnz * fd + 4.0 * n * fd + 8.0 * (n + 1.0);
    else
        bytes = 8.0 * nnz + 4.0 * nnz * fd * 2.0 + 4.0 * nnz;
    const double flops = 2.0 * nnz * fd;
    const double tb = bytes / bw_eff, tf = flops / flops_eff;
    const double seconds = tb > tf ? tb : tf;
    double penalty = 1.0;
    if (v->mapping != 2) {
        const double mean = gf->mean_degree;
        double imbalance = 0.0;
        if (mean > 0.0)
            imbalance = ((double)gf->deg_max / mean - 1.0) / (double)(cores > 1 ? cores : 1);
        if (imbalance < 0.0) imbalance = 0.0;
        if (imbalance > 4.0) imbalance = 4.0;
        penalty = 1.0 + imbalance;
    }
    return seconds * 1e3 * penalty;
}

typedef struct {
    double cost;
    orc_variant v;
} ranked;

/* rank tuple (cost, mapping==rowparallel?0:1, f_tile, vec?0:1, rpc); src/cost.cpp:69-73 */
static int rank_less(const ranked* a, const ranked* b) {
    if (a->cost != b->cost) return a->cost < b->cost;
    int ma = a->v.mapping == 1 ? 0 : 1, mb = b->v.mapping == 1 ? 0 : 1;
    if (ma != mb) return ma < mb;
    if (a->v.f_tile != b->v.f_tile) return a->v.f_tile < b->v.f_tile;
    int va = a->v.vectorized ? 0 : 1, vb = b->v.vectorized ? 0 : 1;
    if (va != vb) return va < vb;
    return a->v.rows_per_chunk < b->v.rows_per_chunk;
}

/* src/cost.cpp:45-79: grid order mapping x tile x rpc x (vec first), then a
 * stable sort (insertion sort is stable). */
int orc_shortlist(const orc_features* gf, uint64_t f, int op, double bw_eff,
                  double flops_eff, uint64_t cores, orc_variant* out) {
    static const uint64_t tiles[3] = {32, 64, 128};
    static const uint64_t rpcs[3] = {1, 4, 16};
    const int vec_eligible = f > 0 && f % 4 == 0;
    ranked grid[36];
    int n = 0;
    for (int m = 1; m <= 2; ++m)
        for (int ti = 0; ti < 3; ++ti)
            for (int ri = 0; ri < 3; ++ri)
                for (int vec = vec_eligible ? 1 : 0; vec >= 0; --vec) {
                    orc_variant v = {op, m, tiles[ti], rpcs[ri], vec, 256};
                    grid[n].v = v;
                    grid[n].cost = orc_estimate_cost(&v, gf, f, bw_eff, flops_eff, cores);
                    ++n;
                }
    for (int i = 1; i < n; ++i) {
        ranked key = grid[i];
        int j = i - 1;
        while (j >= 0 && rank_less(&key, &grid[j])) {
            grid[j + 1] = grid[j];
            --j;
        }
        grid[j + 1] = key;
    }
    for (int i = 0; i < n; ++i) out[i] = grid[i].v;
    return n;
}

/* -------------------------------------------------------------- timing -- */

/* src/timing.cpp:22-61 (warm-up counted in launches and max_run_ms) */
int orc_time_kernel_policy(const double* script, int script_len, int iters, double cap_ms,
                           double warmup_ms, orc_timed_stats* st) {
    if (iters < 1) return -1;
    memset(st, 0, sizeof *st);
    st->max_run_ms = warmup_ms;
    st->launches = 1;
    double* times = (double*)malloc((size_t)iters * sizeof(double));
    double total = 0.0;
    int n = 0;
    for (int k = 0; k < iters; ++k) {
        if (n >= script_len) {
            free(times);
            return -2; /* FakeTimer: script exhausted */
        }
        const double t = script[n];
        ++st->launches;
        times[n++] = t;
        total += t;
        if (t > st->max_run_ms) st->max_run_ms = t;
        if (total > cap_ms && k + 1 < iters) {
            st->capped = 1;
            break;
        }
    }
    st->completed = n;
    for (int i = 1; i < n; ++i) { /* sort ascending */
        double key = times[i];
        int j = i - 1;
        while (j >= 0 && times[j] > key) {
            times[j + 1] = times[j];
            --j;
        }
        times[j + 1] = key;
    }
    st->median_ms = times[(n - 1) / 2];
    free(times);
    return 0;
}

/* ----------------------------------------------------------- partition -- */

void orc_partition_rows(const uint64_t* rowptr, uint64_t n_rows, uint32_t g, uint64_t* cuts) {
    const uint64_t nnz = rowptr[n_rows];
    cuts[0] = 0;
    for (uint32_t k = 1; k < g; ++k) {
        const uint64_t target = (uint64_t)(((unsigned __int128)k * nnz) / g);
        uint64_t lo = 0, hi = n_rows; /* first i with rowptr[i] >= target */
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (rowptr[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        cuts[k] = lo < cuts[k - 1] ? cuts[k - 1] : lo;
    }
    cuts[g] = n_rows;
}

/* ------------------------------------------------ backward (new; N4) -- */
/* The reference has no backward pass (PAPER.md:334 lists it
 * as an extension).  These restate the gradients of the forward operators
 * above with the same accumulation rules, so the device backward can be
 * held to the same bar: structure bit-exact, SpMM/SDDMM gradients bit-exact
 * (they ARE SpMM/SDDMM calls), softmax backward bit-exact (f64 sum in entry
 * order). */

/* Transpose of a canonical CSR (csr.hpp:24-45 invariants): counting sort by
 * column, entries of a column kept in row order (so the result is canonical
 * too).  perm[k] = source entry of transposed entry k. */
void orc_transpose(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
                   uint64_t n_cols, uint64_t* rowptr_t, uint32_t* colind_t, uint32_t* perm) {
    const uint64_t nnz = rowptr[n_rows];
    for (uint64_t j = 0; j <= n_cols; ++j) rowptr_t[j] = 0;
    for (uint64_t e = 0; e < nnz; ++e) rowptr_t[colind[e] + 1]++;
    for (uint64_t j = 0; j < n_cols; ++j) rowptr_t[j + 1] += rowptr_t[j];
    uint64_t* next = (uint64_t*)malloc((n_cols ? n_cols : 1) * sizeof(uint64_t));
    for (uint64_t j = 0; j < n_cols; ++j) next[j] = rowptr_t[j];
    for (uint64_t i = 0; i < n_rows; ++i)
        for (uint64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            const uint64_t k = next[colind[e]]++;
            colind_t[k] = (uint32_t)i;
            perm[k] = (uint32_t)e;
        }
    free(next);
}

/* Gradient of row_softmax (src/kernels.cpp:431-461): with p = softmax(s) and
 * upstream g, ds[e] = p[e] * (g[e] - sum_row p*g).  The products f64(p)*f64(g)
 * are exact; they are summed in a fixed order chosen for the GPU (the
 * reference defines none): 256 strided partials (partial l takes the row's
 * entries l, l+256, l+512, ... in order), folded pairwise part[l] += part[l+o]
 * for o = 128, 64, ..., 1.  ds = f32(f64(p) * (f64(g) - dot)).  Empty rows
 * untouched. */
void orc_row_softmax_backward(const uint64_t* rowptr, uint64_t n_rows, const float* p,
                              const float* g, float* ds) {
    for (uint64_t i = 0; i < n_rows; ++i) {
        const uint64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        double part[256];
        for (int l = 0; l < 256; ++l) part[l] = 0.0;
        for (uint64_t e = e0; e < e1; ++e) part[(e - e0) & 255] += (double)p[e] * (double)g[e];
        for (int o = 128; o > 0; o >>= 1)
            for (int l = 0; l < o; ++l) part[l] += part[l + o];
        const double dot = part[0];
        for (uint64_t e = e0; e < e1; ++e) ds[e] = (float)((double)p[e] * ((double)g[e] - dot));
    }
}

/* Column-blocked SpMM (the B200 library's as_spmm_blocked_*): each segment
 * -- a row, or under HubSplit (hub_t > 0) a 2048-nnz piece of a row with
 * degree >= hub_t (src/kernels.cpp:129-142) -- keeps one f64 accumulator per
 * feature across the column blocks [cuts[b], cuts[b+1]), visited in ascending
 * order; C[i] = f32(0.0 + s_0 + s_1 + ...) over the row's segments
 * (src/kernels.cpp:320-331).  Equal to orc_spmm_baseline / orc_spmm_hubsplit
 * bit for bit for every cut vector (columns are sorted within a row). */
void orc_spmm_blocked(const uint64_t* rowptr, const uint32_t* colind, const float* val, uint64_t n_rows,
                      const float* b, uint64_t f, uint64_t hub_t, const uint64_t* cuts, uint32_t n_blocks,
                      float* c) {
    double* acc = (double*)calloc(f ? f : 1, sizeof(double));
    double* sum = (double*)calloc(f ? f : 1, sizeof(double));
    for (uint64_t i = 0; i < n_rows; ++i) {
        const uint64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        const uint64_t step = (hub_t && e1 - e0 >= hub_t) ? ORC_HUB_NNZ_CHUNK : (e1 > e0 ? e1 - e0 : 1);
        for (uint64_t t = 0; t < f; ++t) sum[t] = 0.0;
        for (uint64_t s0 = e0; s0 < e1; s0 += step) {
            const uint64_t s1 = s0 + step < e1 ? s0 + step : e1;
            for (uint64_t t = 0; t < f; ++t) acc[t] = 0.0;
            uint64_t e = s0;
            for (uint32_t blk = 0; blk < n_blocks; ++blk) {
                /* this block's run of the segment: columns below cuts[blk + 1] */
                for (; e < s1 && colind[e] < cuts[blk + 1]; ++e) {
                    const float* brow = b + (uint64_t)colind[e] * f;
                    const double v = val ? (double)val[e] : 1.0;
                    for (uint64_t t = 0; t < f; ++t) acc[t] += v * (double)brow[t];
                }
            }
            for (uint64_t t = 0; t < f; ++t) sum[t] += acc[t];
        }
        for (uint64_t t = 0; t < f; ++t) c[i * f + t] = (float)sum[t];
    }
    free(acc);
    free(sum);
}
