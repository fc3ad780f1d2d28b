/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the AutoSAGE reference algorithm for the CSR
 * SpMM / SDDMM / row-softmax / attention hot path and the host-side policy
 * helpers the scheduler depends on.  It is the *checker* for the B200
 * library: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.  The product path (paper_2511_17594_b200) never links or
 * calls anything in this directory.
 *
 * Parity pinning: every function here is checked in tests/test_oracle.py
 * against (a) the known-answer vectors of the reference's own doctest suite
 * and (b) the reference library itself, compiled from /root/reference by
 * oracle/Makefile into oracle/_ref/libautosage_ref.so, plus committed golden
 * fixtures under tests/golden/ produced by tests/golden/make_golden.py.
 *
 * Citations are /root/reference/proj/<path>:<line>.
 */
#ifndef AUTOSAGE_ORACLE_H
#define AUTOSAGE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* src/kernels.cpp:21 -- nnz per heavy-row piece in HubSplit. */
#define ORC_HUB_NNZ_CHUNK 2048u

/* SpMM, src/kernels.cpp:210-228: C[i,:] = sum_e val[e]*B[col[e],:] with a
 * double accumulator per feature, entries in CSR order, rounded to f32.
 * val == NULL means implicit 1.0 (pattern-only CSR). */
void orc_spmm_baseline(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                       uint64_t n_rows, const float* b, uint64_t f, float* c);

/* SpMM HubSplit, src/kernels.cpp:260-334: rows with degree >= hub_t are cut
 * into 2048-nnz pieces with double partials, reduced in piece order from
 * 0.0; light rows as the baseline (every RowParallel tiling is bitwise equal
 * to it, src/kernels.cpp:55-94). */
void orc_spmm_hubsplit(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                       uint64_t n_rows, const float* b, uint64_t f, uint64_t hub_t, float* c);

/* SDDMM, src/kernels.cpp:336-355 (vec=0: sequential double dot, tiling is a
 * no-op) and src/kernels.cpp:103-127 (vec=1: per f_tile block, four strided
 * partial sums combined as ((a0+a1)+(a2+a3))+tail).  f_tile is clamped as
 * effective_tile (src/kernels.cpp:45-47). */
void orc_sddmm(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
               const float* x, const float* y, uint64_t f, uint64_t f_tile, int vec,
               float* out);

/* Row softmax, src/kernels.cpp:431-461: f32 max, f32(exp(f64 v - f64 mx)),
 * f64 sum in entry order, f32(f64 ex / sum).  Empty rows untouched. */
void orc_row_softmax(const uint64_t* rowptr, uint64_t n_rows, const float* vals_in,
                     float* vals_out);

/* CSR attention, src/attention.cpp:9-40 with an SDDMM variant (ft, vec) and
 * an SpMM variant (hub_t == 0: row-parallel/baseline order, else hubsplit). */
void orc_attention(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
                   const float* q, const float* k, uint64_t f, const float* v, uint64_t fv,
                   uint64_t sddmm_ft, int sddmm_vec, uint64_t spmm_hub_t, float* out);

/* graph_sig, src/cache.cpp:18-29,66-74: FNV-1a 64 over u64 n_rows, n_cols,
 * nnz, rowptr bytes, colind bytes (little endian). */
uint64_t orc_graph_sig(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
                       uint64_t n_cols, uint64_t nnz);

/* GraphFeatures, include/autosage/csr.hpp:93-107; src/csr.cpp:97-135. */
typedef struct {
    uint64_t n_rows, n_cols, nnz;
    uint64_t deg_p25, deg_p50, deg_p75, deg_p90, deg_p99, deg_max;
    double mean_degree, heavy_row_fraction, empty_row_fraction;
    uint64_t hub_threshold;
} orc_features;
void orc_extract_features(const uint64_t* rowptr, uint64_t n_rows, uint64_t n_cols,
                          uint64_t hub_t, orc_features* out);

/* sample_row_indices, src/generate.cpp:134-153.  Writes min(n, max(min_rows,
 * ceil(frac*n))) row ids to rows_out (capacity n_rows) and returns the count;
 * returns UINT64_MAX when frac is outside (0,1]. */
uint64_t orc_sample_row_indices(const uint64_t* rowptr, uint64_t n_rows, double frac,
                                uint64_t min_rows, uint64_t* rows_out);

/* slice_rows, src/generate.cpp:155-176.  rowptr_out has n_sel+1 entries;
 * colind_out/val_out must hold the sliced nnz (returned). val may be NULL. */
uint64_t orc_slice_rows(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                        const uint64_t* rows, uint64_t n_sel, uint64_t* rowptr_out,
                        uint32_t* colind_out, float* val_out);

/* estimate_cost / shortlist, src/cost.cpp:9-79.  op: 0 spmm, 1 sddmm;
 * mapping: 0 baseline, 1 rowparallel, 2 hubsplit. */
typedef struct {
    int op, mapping;
    uint64_t f_tile, rows_per_chunk;
    int vectorized;
    uint64_t hub_threshold;
} orc_variant;
double orc_estimate_cost(const orc_variant* v, const orc_features* gf, uint64_t f,
                         double bw_eff, double flops_eff, uint64_t cores);
/* Fills up to 36 variants in rank order, returns the count (36 or 18). */
int orc_shortlist(const orc_features* gf, uint64_t f, int op, double bw_eff,
                  double flops_eff, uint64_t cores, orc_variant* out);

/* time_kernel policy, src/timing.cpp:22-61, on a scripted list of timed run
 * durations (the warm-up is not part of the script, as with FakeTimer). */
typedef struct {
    double median_ms;
    int completed, capped, launches;
    double max_run_ms;
} orc_timed_stats;
int orc_time_kernel_policy(const double* script, int script_len, int iters, double cap_ms,
                           double warmup_ms, orc_timed_stats* out);

/* nnz-balanced row partition (new for multi-GPU; no reference counterpart):
 * cut_k = lower_bound(rowptr, floor(k*nnz/g)), k = 1..g-1; cuts[0]=0,
 * cuts[g]=n_rows. */
void orc_partition_rows(const uint64_t* rowptr, uint64_t n_rows, uint32_t g, uint64_t* cuts);


/* ---- backward (new; SURVEY 8(f) N4 -- the reference has none) ---- */
/* CSR transpose by stable counting sort on the column (csr.hpp:24-45
 * invariants preserved); perm[k] = source entry of transposed entry k. */
void orc_transpose(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
                   uint64_t n_cols, uint64_t* rowptr_t, uint32_t* colind_t, uint32_t* perm);
/* d row_softmax (src/kernels.cpp:431-461): ds = f32(p * (g - dot)), dot =
 * 256 strided f64 partials of f64(p)*f64(g) folded in a fixed pairwise tree. */
void orc_row_softmax_backward(const uint64_t* rowptr, uint64_t n_rows, const float* p,
                              const float* g, float* ds);

/* Column-blocked SpMM restated (see oracle.c): segment accumulators carried
 * across ascending column blocks [cuts[b], cuts[b+1]); hub_t == 0 for row
 * chains (baseline / RowParallel), else HubSplit pieces. */
void orc_spmm_blocked(const uint64_t* rowptr, const uint32_t* colind, const float* val, uint64_t n_rows,
                      const float* b, uint64_t f, uint64_t hub_t, const uint64_t* cuts, uint32_t n_blocks,
                      float* c);

/* ---- input generators (gen.c; no reference counterpart -- see gen.c) ---- */
/* Heavy-tailed degrees: deg_i = min(cap, floor(d_min * u^(-1/(alpha-1)))),
 * u from row i's own stream, rescaled to nnz_target (0 = keep) and settled
 * one entry per row; writes rowptr[n_rows+1].  Returns -1 on bad args. */
int orc_gen_powerlaw_degrees(uint64_t n_rows, uint64_t n_cols, uint64_t nnz_target, double alpha,
                             uint64_t d_min, uint64_t d_max, uint64_t seed, uint64_t* rowptr);
/* Distinct ascending columns per row (and U[0,1) values when val != NULL). */
void orc_gen_powerlaw_columns(uint64_t n_rows, uint64_t n_cols, uint64_t seed, const uint64_t* rowptr,
                              uint32_t* colind, float* val);
/* out[i] = U[-1, 1) from splitmix64(seed * 0xA0761D6478BD642F + i). */
void orc_fill_uniform(float* out, uint64_t n, uint64_t seed);

#ifdef __cplusplus
}
#endif

#endif
