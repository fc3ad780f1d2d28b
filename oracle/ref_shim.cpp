// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" face of the *reference library itself*, compiled from the
// untouched sources under /root/reference/proj/src with
// -Dautosage=autosage_ref (oracle/Makefile).  Python tests load
// oracle/_ref/libautosage_ref.so through ctypes to (a) pin the C
// restatement in oracle/oracle.c and (b) time the reference CPU path as the
// bench's `cpu_baseline` / `--impl reference` arm.  Nothing in the product
// links this file.

#include "autosage/attention.hpp"
#include "autosage/cache.hpp"
#include "autosage/cost.hpp"
#include "autosage/csr.hpp"
#include "autosage/device.hpp"
#include "autosage/generate.hpp"
#include "autosage/kernels.hpp"
#include "autosage/parallel.hpp"
#include "autosage/scheduler.hpp"

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

namespace R = autosage_ref;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown";
        return 1;
    }
}

R::CsrMatrix make_csr(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                      uint64_t n_rows, uint64_t n_cols, uint64_t nnz) {
    R::CsrMatrix m;
    m.n_rows = n_rows;
    m.n_cols = n_cols;
    m.rowptr.assign(rowptr, rowptr + n_rows + 1);
    m.colind.assign(colind, colind + nnz);
    if (val) m.val.assign(val, val + nnz);
    return m;
}

R::DenseMatrix make_dense(const float* d, uint64_t rows, uint64_t cols) {
    R::DenseMatrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data(), d, rows * cols * sizeof(float));
    return m;
}

void copy_out(const R::DenseMatrix& m, float* out) {
    if (m.size()) std::memcpy(out, m.data(), m.size() * sizeof(float));
}

struct Graph {
    R::CsrMatrix m;
};
struct Dense {
    R::DenseMatrix m;
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- persistent operands (so timed loops do not re-copy) -----------------
void* ref_graph_new(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                    uint64_t n_rows, uint64_t n_cols, uint64_t nnz) {
    return new Graph{make_csr(rowptr, colind, val, n_rows, n_cols, nnz)};
}
void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }
void* ref_dense_new(const float* d, uint64_t rows, uint64_t cols) {
    return new Dense{make_dense(d, rows, cols)};
}
void ref_dense_free(void* d) { delete static_cast<Dense*>(d); }

// ---- kernels (src/kernels.cpp) ------------------------------------------
int ref_spmm_baseline(void* g, void* b, float* out) {
    return guard([&] {
        copy_out(R::spmm_baseline(static_cast<Graph*>(g)->m, static_cast<Dense*>(b)->m), out);
    });
}

// dispatch(variant, a, b, workers) -- src/kernels.cpp:485-510
int ref_spmm_dispatch(const char* variant, void* g, void* b, uint64_t workers, float* out,
                      int* vectorized_path) {
    return guard([&] {
        auto r = R::dispatch(R::variant_from_string(variant), static_cast<Graph*>(g)->m,
                             static_cast<Dense*>(b)->m, workers);
        if (out) copy_out(r.output, out);
        if (vectorized_path) *vectorized_path = r.vectorized_path ? 1 : 0;
    });
}

int ref_sddmm_baseline(void* g, void* x, void* y, float* out) {
    return guard([&] {
        auto v = R::sddmm_baseline(static_cast<Graph*>(g)->m, static_cast<Dense*>(x)->m,
                                   static_cast<Dense*>(y)->m);
        if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(float));
    });
}

int ref_sddmm_dispatch(const char* variant, void* g, void* x, void* y, uint64_t workers,
                       float* out) {
    return guard([&] {
        auto r = R::dispatch(R::variant_from_string(variant), static_cast<Graph*>(g)->m,
                             static_cast<Dense*>(x)->m, static_cast<Dense*>(y)->m, workers);
        if (out && !r.values.empty())
            std::memcpy(out, r.values.data(), r.values.size() * sizeof(float));
    });
}

// row_softmax over the graph's values -- src/kernels.cpp:431-461
int ref_row_softmax(void* g, uint64_t workers, float* out) {
    return guard([&] {
        auto r = R::row_softmax(static_cast<Graph*>(g)->m, workers);
        if (!r.val.empty()) std::memcpy(out, r.val.data(), r.val.size() * sizeof(float));
    });
}

// ---- policy helpers ------------------------------------------------------
int ref_graph_sig(void* g, uint64_t* out) {
    return guard([&] { *out = R::graph_sig(static_cast<Graph*>(g)->m); });
}

// writes 14 fields: n_rows n_cols nnz p25 p50 p75 p90 p99 max (u64 as double)
// mean heavy empty hub_t
int ref_extract_features(void* g, uint64_t hub_t, double* out14) {
    return guard([&] {
        auto f = R::extract_features(static_cast<Graph*>(g)->m, hub_t);
        double v[14] = {double(f.n_rows),  double(f.n_cols),  double(f.nnz),
                        double(f.deg_p25), double(f.deg_p50), double(f.deg_p75),
                        double(f.deg_p90), double(f.deg_p99), double(f.deg_max),
                        f.mean_degree,     f.heavy_row_fraction, f.empty_row_fraction,
                        double(f.hub_threshold), 0.0};
        std::memcpy(out14, v, sizeof v);
    });
}

int ref_sample_row_indices(void* g, double frac, uint64_t min_rows, uint64_t* rows_out,
                           uint64_t* count) {
    return guard([&] {
        auto rows = R::sample_row_indices(static_cast<Graph*>(g)->m, frac, min_rows);
        for (size_t i = 0; i < rows.size(); ++i) rows_out[i] = rows[i];
        *count = rows.size();
    });
}

// shortlist as newline-separated variant strings -- src/cost.cpp:45-79
int ref_shortlist(void* g, uint64_t f, int op, double bw, double flops, uint64_t cores,
                  char* buf, uint64_t cap) {
    return guard([&] {
        auto gf = R::extract_features(static_cast<Graph*>(g)->m);
        auto dp = R::DeviceProfile::fixed(bw, flops, cores, "test");
        auto list = R::shortlist(gf, f, op == 0 ? R::Op::SpMM : R::Op::SDDMM, dp);
        std::string s;
        for (auto& v : list) s += R::variant_to_string(v) + "\n";
        std::snprintf(buf, cap, "%s", s.c_str());
    });
}

int ref_estimate_cost(void* g, const char* variant, uint64_t f, double bw, double flops,
                      uint64_t cores, double* out) {
    return guard([&] {
        auto gf = R::extract_features(static_cast<Graph*>(g)->m);
        auto dp = R::DeviceProfile::fixed(bw, flops, cores, "test");
        *out = R::estimate_cost(R::variant_from_string(variant), gf, f, dp);
    });
}

int ref_record_line(const char* dev, uint64_t sig, uint64_t f, int op, const char* choice,
                    double t_b, double t_star, double alpha, uint64_t ts, const char* tool,
                    char* buf, uint64_t cap) {
    return guard([&] {
        R::CacheRecord rec;
        rec.key = {dev, sig, f, op == 0 ? R::Op::SpMM : R::Op::SDDMM};
        rec.choice = choice;
        rec.t_b = t_b;
        rec.t_star = t_star;
        rec.alpha = alpha;
        rec.timestamp = ts;
        rec.toolchain = tool;
        std::snprintf(buf, cap, "%s", R::record_to_line(rec).c_str());
    });
}

// ---- generators (src/generate.cpp) used to build the reference's own ------
// ---- test fixtures; arrays are malloc'ed and freed with ref_free ----------
static void export_csr(const R::CsrMatrix& m, uint64_t** rowptr, uint32_t** colind,
                       float** val, uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz) {
    *n_rows = m.n_rows;
    *n_cols = m.n_cols;
    *nnz = m.nnz();
    *rowptr = static_cast<uint64_t*>(std::malloc((m.n_rows + 1) * 8));
    std::memcpy(*rowptr, m.rowptr.data(), (m.n_rows + 1) * 8);
    *colind = static_cast<uint32_t*>(std::malloc(m.nnz() * 4 + 4));
    if (m.nnz()) std::memcpy(*colind, m.colind.data(), m.nnz() * 4);
    *val = nullptr;
    if (m.has_values()) {
        *val = static_cast<float*>(std::malloc(m.nnz() * 4 + 4));
        std::memcpy(*val, m.val.data(), m.nnz() * 4);
    }
}

int ref_gen(int kind, uint64_t n, double p, uint64_t k, uint64_t hubs, uint64_t hub_deg,
            uint64_t other_deg, uint64_t seed, uint64_t** rowptr, uint32_t** colind,
            float** val, uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz) {
    return guard([&] {
        R::CsrMatrix m;
        if (kind == 0) m = R::gen_er(n, p, seed);
        else if (kind == 1) m = R::gen_hubskew(n, k, p, seed, hubs ? hubs : 64);
        else m = R::gen_hub_fixed(n, hubs, hub_deg, other_deg, seed);
        export_csr(m, rowptr, colind, val, n_rows, n_cols, nnz);
    });
}
void ref_free(void* p) { std::free(p); }

// ---- the reference's input-aware path, as its bench runs it ---------------
// decide once (host profile, probes) -> variant string; src/scheduler.cpp:195-239
int ref_decide(void* g, void* x, void* y, int op, char* choice, uint64_t cap,
               double* probe_ms) {
    return guard([&] {
        R::ProbeConfig cfg;
        R::ScheduleContext ctx;
        R::ScheduleDecision d =
            op == 0 ? R::decide_spmm(static_cast<Graph*>(g)->m, static_cast<Dense*>(y)->m, cfg,
                                     ctx)
                    : R::decide_sddmm(static_cast<Graph*>(g)->m, static_cast<Dense*>(x)->m,
                                      static_cast<Dense*>(y)->m, cfg, ctx);
        std::snprintf(choice, cap, "%s", d.choice_string().c_str());
        if (probe_ms) *probe_ms = d.report.probe_wall_ms;
    });
}

uint64_t ref_default_workers() { return R::default_workers(); }

// csr_attention_forward with default probing and a private cache
int ref_attention(void* g, void* q, void* k, void* v, float* out) {
    return guard([&] {
        R::ProbeConfig cfg;
        R::ScheduleCache cache;
        R::ScheduleContext ctx;
        ctx.cache = &cache;
        auto o = R::csr_attention_forward(static_cast<Graph*>(g)->m, static_cast<Dense*>(q)->m,
                                          static_cast<Dense*>(k)->m, static_cast<Dense*>(v)->m,
                                          cfg, ctx);
        copy_out(o, out);
    });
}

} // extern "C"
