// capi.cpp -- the extern "C" boundary (include/autosage_b200.h).
// Exceptions never cross it: each entry point maps them to as_status and a
// thread-local message (the reference's exception texts where it throws).
#include "autosage_b200.h"

#include "cache.hpp"
#include "engine.hpp"
#include "ops.hpp"
#include "policy.hpp"

#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <new>

namespace asb {
struct BlockedPlan;
BlockedPlan* blocked_plan_create(Graph& g, const as_variant* v, const std::uint64_t* cuts,
                                 std::uint32_t n_blocks);
void blocked_plan_run(BlockedPlan& p, std::uint32_t block, const float* vals, const float* b, std::uint64_t b_rows,
                      std::uint64_t f, float* c, cudaStream_t s);
void blocked_plan_destroy(BlockedPlan* p);
Graph& blocked_plan_graph(BlockedPlan& p);
void gen_powerlaw(std::uint64_t, std::uint64_t, std::uint64_t, double, std::uint64_t,
                  std::uint64_t, std::uint64_t, bool, std::vector<std::uint64_t>&,
                  std::vector<std::uint32_t>&, std::vector<float>&);
void fill_uniform(float*, std::uint64_t, std::uint64_t);
void save_csr(const std::string&, const std::uint64_t*, const std::uint32_t*, const float*,
              std::uint64_t, std::uint64_t, std::uint64_t);
void load_csr(const std::string&, std::vector<std::uint64_t>&, std::vector<std::uint32_t>&,
              std::vector<float>&, std::uint64_t&, std::uint64_t&);
} // namespace asb

using namespace asb;

namespace {

thread_local std::string t_err;

template <class F>
as_status guard(F&& f) {
    try {
        f();
        return AS_OK;
    } catch (const InvalidArgument& e) {
        t_err = e.what();
        return AS_INVALID_ARGUMENT;
    } catch (const CacheError& e) {
        t_err = e.what();
        return AS_CACHE_ERROR;
    } catch (const IoError& e) {
        t_err = e.what();
        return AS_IO_ERROR;
    } catch (const ReplayMissError& e) {
        t_err = e.what();
        return AS_REPLAY_MISS;
    } catch (const OutOfMemory& e) {
        t_err = e.what();
        return AS_OUT_OF_MEMORY;
    } catch (const CudaError& e) {
        t_err = e.what();
        return AS_CUDA_ERROR;
    } catch (const LogicError& e) {
        t_err = e.what();
        return AS_LOGIC_ERROR;
    } catch (const std::invalid_argument& e) {
        t_err = e.what();
        return AS_INVALID_ARGUMENT;
    } catch (const std::bad_alloc&) {
        t_err = "host allocation failed";
        return AS_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        t_err = e.what();
        return AS_INTERNAL;
    } catch (...) {
        t_err = "unknown error";
        return AS_INTERNAL;
    }
}

Graph& G(as_graph g) {
    if (!g) throw InvalidArgument("null graph handle");
    return *reinterpret_cast<Graph*>(g);
}

ScheduleCache* C(as_cache c) { return reinterpret_cast<ScheduleCache*>(c); }

TimeOnce wrap_timer(as_time_once_fn fn, void* user) {
    if (!fn) return {};
    return [fn, user](const std::string& label, const std::function<void()>& run) {
        struct Tramp {
            const std::function<void()>* run;
            std::exception_ptr err;
        } t{&run, nullptr};
        auto tramp = [](void* arg) {
            auto* tp = static_cast<Tramp*>(arg);
            try {
                (*tp->run)();
            } catch (...) {
                tp->err = std::current_exception();
            }
        };
        const double ms = fn(user, label.c_str(), tramp, &t);
        if (t.err) std::rethrow_exception(t.err);
        if (ms < 0.0) throw LogicError("timer: script exhausted");
        return ms;
    };
}

Context make_ctx(const as_context* c) {
    Context ctx;
    if (!c) return ctx;
    ctx.device = c->device;
    ctx.cache = C(c->cache);
    ctx.timer = wrap_timer(c->timer, c->timer_user);
    ctx.replay = c->replay;
    ctx.stream = static_cast<cudaStream_t>(c->stream);
    return ctx;
}

as_probe_config cfg_or_default(const as_probe_config* cfg) {
    return cfg ? *cfg : probe_config_default();
}

void fill_result(as_kernel_result* res, const KernelResult& r) {
    if (!res) return;
    res->variant = r.variant;
    res->vectorized_path = r.vectorized_path ? 1 : 0;
    res->elapsed_ms = r.elapsed_ms;
}

template <class T>
T* malloc_copy(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(std::max<std::size_t>(v.size(), 1) * sizeof(T)));
    if (!p) throw std::bad_alloc();
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}

} // namespace

extern "C" {

const char* as_last_error(void) { return t_err.c_str(); }
int as_abi_version(void) { return AS_ABI_VERSION; }
const char* as_artifact_version(void) { return kArtifactVersion; }
uint64_t as_kernel_launch_count(void) { return g_kernel_launches.load(); }

// ---- variants -------------------------------------------------------------------
void as_variant_default(as_variant* v) {
    if (v) *v = default_variant();
}

as_status as_variant_to_string(const as_variant* v, char* buf, size_t cap) {
    return guard([&] {
        if (!v || !buf) throw InvalidArgument("null argument");
        std::snprintf(buf, cap, "%s", variant_to_string(*v).c_str());
    });
}

as_status as_variant_from_string(const char* s, as_variant* out) {
    return guard([&] {
        if (!s || !out) throw InvalidArgument("null argument");
        *out = variant_from_string(s);
    });
}

int as_vec4_eligible(uint64_t f, const void* const* bases, int n_bases) {
    return vec4_eligible(f, bases, n_bases) ? 1 : 0;
}

// ---- graphs ------------------------------------------------------------------------
as_status as_graph_create(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                          uint64_t n_rows, uint64_t n_cols, uint64_t nnz, int device,
                          as_graph* out) {
    return guard([&] {
        if (!out) throw InvalidArgument("null output");
        *out = reinterpret_cast<as_graph>(
            graph_create_host(rowptr, colind, val, n_rows, n_cols, nnz, device, true).release());
    });
}

as_status as_graph_create_device(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                                 uint64_t n_rows, uint64_t n_cols, uint64_t nnz, int device, void* stream,
                                 as_graph* out) {
    return guard([&] {
        if (!out) throw InvalidArgument("null output");
        *out = reinterpret_cast<as_graph>(graph_create_device(rowptr, colind, val, n_rows, n_cols, nnz, device,
                                                              static_cast<cudaStream_t>(stream))
                                              .release());
    });
}

as_status as_graph_destroy(as_graph g) {
    return guard([&] { delete reinterpret_cast<Graph*>(g); });
}

as_status as_graph_shape(as_graph g, uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz,
                         int* has_values) {
    return guard([&] {
        Graph& gr = G(g);
        if (n_rows) *n_rows = gr.n_rows;
        if (n_cols) *n_cols = gr.n_cols;
        if (nnz) *nnz = gr.nnz;
        if (has_values) *has_values = gr.has_val ? 1 : 0;
    });
}

as_status as_graph_device_arrays(as_graph g, const uint64_t** rowptr, const uint32_t** colind,
                                 const float** val) {
    return guard([&] {
        Graph& gr = G(g);
        if (rowptr) *rowptr = gr.rowptr.get();
        if (colind) *colind = gr.colind.get();
        if (val) *val = gr.has_val ? gr.val.get() : nullptr;
    });
}

as_status as_graph_set_values(as_graph g, const float* vals, int vals_on_device) {
    return guard([&] {
        Graph& gr = G(g);
        DeviceGuard dg(gr.device);
        if (!vals || gr.nnz == 0) {
            gr.val.release();
            gr.has_val = false;
            return;
        }
        gr.val.ensure(gr.nnz);
        ASB_CUDA(cudaMemcpyAsync(gr.val.get(), vals, gr.nnz * 4,
                                 vals_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 gr.stream));
        ASB_CUDA(cudaStreamSynchronize(gr.stream));
        gr.has_val = true;
    });
}

as_status as_validate(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                      uint64_t rowptr_len, uint64_t n_rows, uint64_t n_cols, uint64_t nnz,
                      uint64_t val_len, int* violated, char* buf, size_t cap, uint64_t* index) {
    (void)val;
    return guard([&] {
        auto v = validate_csr(rowptr, rowptr_len, colind, nnz, val_len, n_rows, n_cols);
        if (violated) *violated = v ? 1 : 0;
        if (v) {
            if (buf) std::snprintf(buf, cap, "%s", v->invariant.c_str());
            if (index) *index = v->index;
        }
    });
}

as_status as_graph_sig(as_graph g, uint64_t* out) {
    return guard([&] { *out = graph_sig(G(g)); });
}

uint64_t as_graph_sig_host(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
                           uint64_t n_cols, uint64_t nnz) {
    return graph_sig_host(rowptr, colind, n_rows, n_cols, nnz);
}

as_status as_graph_features(as_graph g, uint64_t hub_threshold, as_features* out) {
    return guard([&] { *out = graph_features(G(g), hub_threshold); });
}

as_status as_sample_row_indices(as_graph g, double frac, uint64_t min_rows, uint64_t* rows_out,
                                uint64_t* count) {
    return guard([&] {
        const auto rows = sample_row_indices(G(g), frac, min_rows);
        if (rows_out && !rows.empty()) std::memcpy(rows_out, rows.data(), rows.size() * 8);
        if (count) *count = rows.size();
    });
}

as_status as_slice_rows(as_graph g, const uint64_t* rows_host, uint64_t n_sel, as_graph* out) {
    return guard([&] {
        Graph& gr = G(g);
        std::vector<std::uint64_t> rows(rows_host, rows_host + n_sel);
        *out = reinterpret_cast<as_graph>(slice_rows(gr, rows, graph_values(gr, nullptr)).release());
    });
}

as_status as_graph_download(as_graph g, uint64_t* rowptr, uint32_t* colind, float* val) {
    return guard([&] {
        Graph& gr = G(g);
        DeviceGuard dg(gr.device);
        if (rowptr) std::memcpy(rowptr, gr.h_rowptr.data(), (gr.n_rows + 1) * 8);
        if (colind && gr.nnz)
            ASB_CUDA(cudaMemcpyAsync(colind, gr.colind.get(), gr.nnz * 4, cudaMemcpyDeviceToHost,
                                     gr.stream));
        if (val && gr.has_val && gr.nnz)
            ASB_CUDA(cudaMemcpyAsync(val, gr.val.get(), gr.nnz * 4, cudaMemcpyDeviceToHost, gr.stream));
        ASB_CUDA(cudaStreamSynchronize(gr.stream));
    });
}

// ---- operators -------------------------------------------------------------------
static as_status spmm_entry(const as_variant* v, as_graph a, const float* vals_dev, const float* b_dev,
                            uint64_t b_rows, uint64_t f, float* c_dev, void* stream, as_kernel_result* res) {
    return guard([&] {
        Graph& g = G(a);
        cudaStream_t s = resolve_stream(g, stream);
        GraphUse use(g, s);
        if (!v) {
            KernelResult r;
            r.variant = default_variant();
            r.variant.mapping = AS_MAP_BASELINE;
            if (g.n_cols != b_rows) throw InvalidArgument("spmm: a.n_cols != b.n_rows");
            DeviceGuard dg(g.device);
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (res) {
                ASB_CUDA(cudaEventCreate(&e0));
                ASB_CUDA(cudaEventCreate(&e1));
                ASB_CUDA(cudaEventRecord(e0, s));
            }
            spmm_baseline(g, graph_values(g, vals_dev), b_dev, b_rows, f, c_dev, s);
            if (res) {
                ASB_CUDA(cudaEventRecord(e1, s));
                ASB_CUDA(cudaEventSynchronize(e1));
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                r.elapsed_ms = ms;
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
            }
            fill_result(res, r);
            return;
        }
        const KernelResult r = dispatch_spmm(*v, g, vals_dev, b_dev, b_rows, f, c_dev, s, res != nullptr);
        fill_result(res, r);
    });
}

as_status as_spmm(const as_variant* v, as_graph a, const float* b_dev, uint64_t b_rows, uint64_t f,
                  float* c_dev, void* stream, as_kernel_result* res) {
    return spmm_entry(v, a, nullptr, b_dev, b_rows, f, c_dev, stream, res);
}

as_status as_spmm_values(const as_variant* v, as_graph a, const float* vals_dev, const float* b_dev,
                         uint64_t b_rows, uint64_t f, float* c_dev, void* stream, as_kernel_result* res) {
    if (!vals_dev && a && G(a).nnz) {
        t_err = "spmm_values: values required";
        return AS_INVALID_ARGUMENT;
    }
    return spmm_entry(v, a, vals_dev, b_dev, b_rows, f, c_dev, stream, res);
}

as_status as_spmm_rowparallel(const as_variant* v, as_graph a, const float* b_dev, uint64_t b_rows,
                              uint64_t f, float* c_dev, void* stream) {
    return guard([&] {
        if (!v) throw InvalidArgument("null variant");
        Graph& g = G(a);
        GraphUse use(g, resolve_stream(g, stream));
        spmm_mapped(*v, AS_MAP_ROWPARALLEL, g, graph_values(g, nullptr), b_dev, b_rows, f, c_dev,
                    resolve_stream(g, stream));
    });
}

as_status as_spmm_hubsplit(const as_variant* v, as_graph a, const float* b_dev, uint64_t b_rows,
                           uint64_t f, float* c_dev, void* stream) {
    return guard([&] {
        if (!v) throw InvalidArgument("null variant");
        Graph& g = G(a);
        GraphUse use(g, resolve_stream(g, stream));
        spmm_mapped(*v, AS_MAP_HUBSPLIT, g, graph_values(g, nullptr), b_dev, b_rows, f, c_dev,
                    resolve_stream(g, stream));
    });
}

as_status as_sddmm(const as_variant* v, as_graph pattern, const float* x_dev, uint64_t x_rows,
                   const float* y_dev, uint64_t y_rows, uint64_t f, float* out_dev, void* stream,
                   as_kernel_result* res) {
    return guard([&] {
        Graph& g = G(pattern);
        cudaStream_t s = resolve_stream(g, stream);
        GraphUse use(g, s);
        if (!v) {
            KernelResult r;
            r.variant = default_variant();
            r.variant.op = AS_OP_SDDMM;
            r.variant.mapping = AS_MAP_BASELINE;
            DeviceGuard dg(g.device);
            ensure_chunk_rows(g);
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (res) {
                ASB_CUDA(cudaEventCreate(&e0));
                ASB_CUDA(cudaEventCreate(&e1));
                ASB_CUDA(cudaEventRecord(e0, s));
            }
            sddmm_baseline(g, x_dev, x_rows, y_dev, y_rows, f, out_dev, s);
            if (res) {
                ASB_CUDA(cudaEventRecord(e1, s));
                ASB_CUDA(cudaEventSynchronize(e1));
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                r.elapsed_ms = ms;
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
            }
            fill_result(res, r);
            return;
        }
        fill_result(res, dispatch_sddmm(*v, g, x_dev, x_rows, y_dev, y_rows, f, out_dev, s,
                                        res != nullptr));
    });
}

as_status as_sddmm_rowparallel(const as_variant* v, as_graph pattern, const float* x_dev,
                               uint64_t x_rows, const float* y_dev, uint64_t y_rows, uint64_t f,
                               float* out_dev, void* stream) {
    return guard([&] {
        if (!v) throw InvalidArgument("null variant");
        Graph& g = G(pattern);
        GraphUse use(g, resolve_stream(g, stream));
        sddmm_mapped(*v, g, x_dev, x_rows, y_dev, y_rows, f, out_dev, resolve_stream(g, stream));
    });
}

as_status as_row_softmax(as_graph m, const float* vals_dev, float* out_dev, void* stream) {
    return guard([&] {
        Graph& g = G(m);
        GraphUse use(g, resolve_stream(g, stream));
        row_softmax(g, graph_values(g, vals_dev), out_dev, resolve_stream(g, stream));
    });
}

// Host-buffer forms (engine.cpp host pipeline): H2D on the graph's copy-in
// stream, kernels on its stream, D2H on its copy-out stream; the SDDMM
// values come back in slices that overlap the remaining kernels.
as_status as_spmm_host(const as_variant* v, as_graph a, const float* b_host, uint64_t b_rows,
                       uint64_t f, float* c_host, as_kernel_result* res) {
    return guard([&] {
        GraphUse use(G(a), G(a).stream);
        fill_result(res, spmm_host(v, G(a), b_host, b_rows, f, c_host, true));
    });
}

as_status as_sddmm_host(const as_variant* v, as_graph pattern, const float* x_host, uint64_t x_rows,
                        const float* y_host, uint64_t y_rows, uint64_t f, float* out_host,
                        as_kernel_result* res) {
    return guard([&] {
        GraphUse use(G(pattern), G(pattern).stream);
        fill_result(res, sddmm_host(v, G(pattern), x_host, x_rows, y_host, y_rows, f, out_host, true));
    });
}

as_status as_spmm_host_async(const as_variant* v, as_graph a, const float* b_host, uint64_t b_rows,
                             uint64_t f, float* c_host, as_kernel_result* res) {
    return guard([&] {
        GraphUse use(G(a), G(a).stream);
        fill_result(res, spmm_host(v, G(a), b_host, b_rows, f, c_host, false));
    });
}

as_status as_sddmm_host_async(const as_variant* v, as_graph pattern, const float* x_host,
                              uint64_t x_rows, const float* y_host, uint64_t y_rows, uint64_t f,
                              float* out_host, as_kernel_result* res) {
    return guard([&] {
        GraphUse use(G(pattern), G(pattern).stream);
        fill_result(res, sddmm_host(v, G(pattern), x_host, x_rows, y_host, y_rows, f, out_host, false));
    });
}

as_status as_graph_synchronize(as_graph g) {
    return guard([&] { host_synchronize(G(g)); });
}

as_status as_row_softmax_host(as_graph m, const float* vals_host, float* out_host) {
    return guard([&] {
        Graph& g = G(m);
        DeviceGuard dg(g.device);
        GraphUse use(g, g.stream);
        const float* vin = nullptr;
        if (vals_host) {
            g.stage_in.ensure(std::max<std::uint64_t>(g.nnz, 1));
            if (g.nnz)
                ASB_CUDA(cudaMemcpyAsync(g.stage_in.get(), vals_host, g.nnz * 4, cudaMemcpyHostToDevice,
                                         g.stream));
            vin = g.stage_in.get();
        } else {
            vin = graph_values(g, nullptr);
        }
        g.stage_out.ensure(std::max<std::uint64_t>(g.nnz, 1));
        row_softmax(g, vin, g.stage_out.get(), g.stream);
        if (g.nnz)
            ASB_CUDA(cudaMemcpyAsync(out_host, g.stage_out.get(), g.nnz * 4, cudaMemcpyDeviceToHost,
                                     g.stream));
        ASB_CUDA(cudaStreamSynchronize(g.stream));
    });
}

// ---- device profile / cost -------------------------------------------------------
as_status as_device_profile_gpu(int device, as_device_profile* out) {
    return guard([&] {
        if (device < 0) ASB_CUDA(cudaGetDevice(&device));
        *out = gpu_profile(device);
    });
}

void as_device_profile_fixed(double bw_eff, double flops_eff, uint64_t cores, const char* sig_tag,
                             as_device_profile* out) {
    // DeviceProfile::fixed, src/device.cpp:103-111
    as_device_profile dp{};
    std::snprintf(dp.device_sig, sizeof dp.device_sig, "%s|cores=%llu|%s",
                  sig_tag ? sig_tag : "fixed", (unsigned long long)cores, kArtifactVersion);
    dp.bw_eff = bw_eff;
    dp.flops_eff = flops_eff;
    dp.cores = cores;
    *out = dp;
}

as_status as_estimate_cost(const as_variant* v, const as_features* gf, uint64_t f,
                           const as_device_profile* dp, double* out_ms) {
    return guard([&] { *out_ms = estimate_cost(*v, *gf, f, *dp); });
}

as_status as_shortlist(const as_features* gf, uint64_t f, int op, const as_device_profile* dp,
                       as_variant* out, int* count) {
    return guard([&] {
        const auto list = shortlist(*gf, f, op, *dp);
        for (std::size_t i = 0; i < list.size() && i < AS_MAX_CANDIDATES; ++i) out[i] = list[i];
        *count = int(list.size());
    });
}

// ---- timing -------------------------------------------------------------------------
as_status as_time_kernel(const char* label, void (*run)(void*), void* run_arg, int iters,
                         double cap_ms, as_time_once_fn timer, void* timer_user,
                         as_timed_stats* out) {
    return guard([&] {
        std::function<void()> fn = [run, run_arg] {
            if (run) run(run_arg);
        };
        TimeOnce t = wrap_timer(timer, timer_user);
        if (!t) {
            cudaStream_t s = nullptr;  // legacy default stream
            t = [s](const std::string&, const std::function<void()>& r) {
                cudaEvent_t e0, e1;
                ASB_CUDA(cudaEventCreate(&e0));
                ASB_CUDA(cudaEventCreate(&e1));
                ASB_CUDA(cudaEventRecord(e0, s));
                r();
                ASB_CUDA(cudaEventRecord(e1, s));
                ASB_CUDA(cudaEventSynchronize(e1));
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
                return double(ms);
            };
        }
        *out = time_kernel(label ? label : "", fn, iters, cap_ms, t);
    });
}

// ---- cache --------------------------------------------------------------------------
as_status as_cache_create(as_cache* out) {
    return guard([&] { *out = reinterpret_cast<as_cache>(new ScheduleCache()); });
}
as_status as_cache_destroy(as_cache c) {
    return guard([&] { delete C(c); });
}
as_status as_cache_get(as_cache c, const as_key* key, as_record* out, int* found) {
    return guard([&] {
        auto r = C(c)->get(key_from_c(*key));
        *found = r ? 1 : 0;
        if (r && out) *out = record_to_c(*r);
    });
}
as_status as_cache_put(as_cache c, const as_record* rec) {
    return guard([&] { C(c)->put(record_from_c(*rec)); });
}
as_status as_cache_size(as_cache c, uint64_t* n) {
    return guard([&] { *n = C(c)->size(); });
}
as_status as_cache_snapshot(as_cache c, as_record* out, uint64_t cap, uint64_t* n) {
    return guard([&] {
        const auto snap = C(c)->snapshot();
        if (n) *n = snap.size();
        if (out)
            for (std::size_t i = 0; i < snap.size() && i < cap; ++i) out[i] = record_to_c(snap[i]);
    });
}
as_status as_cache_clear(as_cache c) {
    return guard([&] { C(c)->clear(); });
}
as_status as_cache_load(as_cache c, const char* path) {
    return guard([&] { C(c)->load(path); });
}
as_status as_cache_store(as_cache c, const char* path) {
    return guard([&] { C(c)->store(path); });
}
as_status as_record_to_line(const as_record* rec, char* buf, size_t cap) {
    return guard([&] { std::snprintf(buf, cap, "%s", record_to_line(record_from_c(*rec)).c_str()); });
}
as_status as_record_from_line(const char* line, as_record* out) {
    return guard([&] { *out = record_to_c(record_from_line(line)); });
}
as_status as_key_to_string(const as_key* key, char* buf, size_t cap) {
    return guard([&] { std::snprintf(buf, cap, "%s", key_from_c(*key).to_string().c_str()); });
}
const char* as_toolchain_tag(void) {
    static const std::string tag = toolchain_tag();
    return tag.c_str();
}

// ---- scheduler -------------------------------------------------------------------------
void as_probe_config_default(as_probe_config* out) { *out = probe_config_default(); }
void as_probe_config_from_env(as_probe_config* out) { *out = probe_config_from_env(); }
void as_replay_policy_from_env(as_replay_policy* out) { *out = replay_policy_from_env(); }

as_status as_decide_spmm(const as_context* ctx, const as_probe_config* cfg, as_graph a,
                         const float* b_dev, uint64_t b_rows, uint64_t f, as_decision* out) {
    return guard([&] {
        const Context c = make_ctx(ctx);
        GraphUse use(G(a), c.stream ? c.stream : G(a).stream);
        *out = decide_spmm(c, cfg_or_default(cfg), G(a), nullptr, b_dev, b_rows, f);
    });
}

as_status as_decide_sddmm(const as_context* ctx, const as_probe_config* cfg, as_graph pattern,
                          const float* x_dev, uint64_t x_rows, const float* y_dev, uint64_t y_rows,
                          uint64_t f, as_decision* out) {
    return guard([&] {
        const Context c = make_ctx(ctx);
        GraphUse use(G(pattern), c.stream ? c.stream : G(pattern).stream);
        *out = decide_sddmm(c, cfg_or_default(cfg), G(pattern), x_dev, x_rows, y_dev, y_rows, f);
    });
}

as_status as_spmm_auto(const as_context* ctx, const as_probe_config* cfg, as_graph a,
                       const float* b_dev, uint64_t b_rows, uint64_t f, float* c_dev,
                       as_decision* decision) {
    return guard([&] {
        const Context c = make_ctx(ctx);
        GraphUse use(G(a), c.stream ? c.stream : G(a).stream);
        spmm_auto(c, cfg_or_default(cfg), G(a), nullptr, b_dev, b_rows, f, c_dev, decision);
    });
}

as_status as_spmm_auto_values(const as_context* ctx, const as_probe_config* cfg, as_graph a,
                              const float* vals_dev, const float* b_dev, uint64_t b_rows, uint64_t f,
                              float* c_dev, as_decision* decision) {
    return guard([&] {
        Graph& g = G(a);
        if (!vals_dev && g.nnz) throw InvalidArgument("spmm_auto_values: values required");
        const Context c = make_ctx(ctx);
        GraphUse use(g, c.stream ? c.stream : g.stream);
        spmm_auto(c, cfg_or_default(cfg), g, vals_dev, b_dev, b_rows, f, c_dev, decision);
    });
}

as_status as_sddmm_auto(const as_context* ctx, const as_probe_config* cfg, as_graph pattern,
                        const float* x_dev, uint64_t x_rows, const float* y_dev, uint64_t y_rows,
                        uint64_t f, float* out_dev, as_decision* decision) {
    return guard([&] {
        const Context c = make_ctx(ctx);
        GraphUse use(G(pattern), c.stream ? c.stream : G(pattern).stream);
        sddmm_auto(c, cfg_or_default(cfg), G(pattern), x_dev, x_rows, y_dev, y_rows, f, out_dev, decision);
    });
}

uint64_t as_probe_launch_count(void) { return probe_launch_count(); }
void as_reset_probe_launch_count(void) { reset_probe_launch_count(); }

as_status as_decide_host(const as_context* ctx, const as_probe_config* cfg, uint64_t graph_sig,
                         const as_features* gf, uint64_t f, int op, uint64_t sample_rows,
                         as_decision* out) {
    return guard([&] {
        *out = decide_host(make_ctx(ctx), cfg_or_default(cfg), graph_sig, *gf, f, op, sample_rows);
    });
}

as_status as_csr_attention_forward(const as_context* ctx, const as_probe_config* cfg,
                                   as_graph pattern, const float* q_dev, uint64_t q_rows,
                                   const float* k_dev, uint64_t k_rows, const float* v_dev,
                                   uint64_t v_rows, uint64_t f, uint64_t fv, float* out_dev,
                                   int fused, as_decision* sd, as_decision* pd) {
    return guard([&] {
        const Context c = make_ctx(ctx);
        GraphUse use(G(pattern), c.stream ? c.stream : G(pattern).stream);
        attention_forward(c, cfg_or_default(cfg), G(pattern), q_dev, q_rows, k_dev, k_rows, v_dev, v_rows, f,
                          fv, out_dev, fused != 0, sd, pd);
    });
}

as_status as_csr_attention_forward_heads(const as_context* ctx, const as_probe_config* cfg, as_graph pattern,
                                         uint32_t n_heads, const float* const* q_devs, uint64_t q_rows,
                                         const float* const* k_devs, uint64_t k_rows, const float* const* v_devs,
                                         uint64_t v_rows, uint64_t f, uint64_t fv, float* const* out_devs, int fused,
                                         as_decision* sd, as_decision* pd) {
    return guard([&] {
        if (n_heads && (!q_devs || !k_devs || !v_devs || !out_devs))
            throw InvalidArgument("attention_heads: null head array");
        Context c = make_ctx(ctx);
        ScheduleCache local;  // heads 2..n replay head 1's decisions
        if (!c.cache) c.cache = &local;
        Graph& g = G(pattern);
        GraphUse use(g, c.stream ? c.stream : g.stream);
        const as_probe_config pc = cfg_or_default(cfg);
        for (std::uint32_t h = 0; h < n_heads; ++h)
            attention_forward(c, pc, g, q_devs[h], q_rows, k_devs[h], k_rows, v_devs[h], v_rows, f, fv,
                              out_devs[h], fused != 0, sd, pd);
    });
}

as_status as_csr_attention_forward_p(const as_context* ctx, const as_probe_config* cfg, as_graph pattern,
                                     const float* q_dev, uint64_t q_rows, const float* k_dev, uint64_t k_rows,
                                     const float* v_dev, uint64_t v_rows, uint64_t f, uint64_t fv, float* out_dev,
                                     float* p_dev, as_decision* sd, as_decision* pd) {
    return guard([&] {
        Graph& g = G(pattern);
        if (g.nnz && !p_dev) throw InvalidArgument("attention: p output required");
        const Context c = make_ctx(ctx);
        GraphUse use(g, c.stream ? c.stream : g.stream);
        attention_forward(c, cfg_or_default(cfg), g, q_dev, q_rows, k_dev, k_rows, v_dev, v_rows, f,
                          fv, out_dev, false, sd, pd, p_dev);
    });
}

// ---- multi-GPU partition ------------------------------------------------------------
as_status as_partition_rows(const uint64_t* rowptr_host, uint64_t n_rows, uint32_t g,
                            uint64_t* cuts) {
    return guard([&] { partition_rows(rowptr_host, n_rows, g, cuts); });
}

as_status as_graph_row_range(as_graph g, uint64_t r0, uint64_t r1, as_graph* out) {
    return guard([&] { *out = reinterpret_cast<as_graph>(row_range(G(g), r0, r1).release()); });
}

as_status as_spmm_blocked_create(as_graph a, const as_variant* v, const uint64_t* col_cuts, uint32_t n_blocks,
                                 as_blocked* out) {
    return guard([&] {
        if (!out || !col_cuts) throw InvalidArgument("spmm_blocked: null argument");
        *out = reinterpret_cast<as_blocked>(blocked_plan_create(G(a), v, col_cuts, n_blocks));
    });
}

as_status as_spmm_blocked_run(as_blocked p, uint32_t block, const float* vals_dev, const float* b_dev,
                              uint64_t b_rows, uint64_t f, float* c_dev, void* stream) {
    return guard([&] {
        if (!p) throw InvalidArgument("spmm_blocked: null plan");
        auto& plan = *reinterpret_cast<BlockedPlan*>(p);
        Graph& g = blocked_plan_graph(plan);
        const cudaStream_t s = resolve_stream(g, stream);
        GraphUse use(g, s);
        blocked_plan_run(plan, block, graph_values(g, vals_dev), b_dev, b_rows, f, c_dev, s);
    });
}

as_status as_spmm_blocked_destroy(as_blocked p) {
    return guard([&] { blocked_plan_destroy(reinterpret_cast<BlockedPlan*>(p)); });
}

// ---- backward (backward.cu) -----------------------------------------------------------
as_status as_graph_transpose(as_graph g, as_graph* out) {
    return guard([&] {
        if (!out) throw InvalidArgument("transpose: null output");
        *out = reinterpret_cast<as_graph>(transpose_graph(G(g)).release());
    });
}

as_status as_graph_transpose_perm(as_graph gt, const uint32_t** perm) {
    return guard([&] {
        Graph& g = G(gt);
        if (!g.is_transpose) throw InvalidArgument("transpose_perm: graph is not a transpose");
        *perm = g.src_perm.get();
    });
}

// ValPermScope: the graph reads its values through its transpose
// permutation for one call, set and cleared while the caller holds the
// graph (GraphUse), so no other operator sees it
struct ValPermScope {
    Graph& g;
    explicit ValPermScope(Graph& gr) : g(gr) { g.val_perm = g.src_perm.get(); }
    ~ValPermScope() { g.val_perm = nullptr; }
};

as_status as_spmm_transpose_values(const as_variant* v, as_graph gt, const float* vals_src_dev,
                                   const float* b_dev, uint64_t b_rows, uint64_t f, float* c_dev, void* stream,
                                   as_kernel_result* res) {
    Graph* gp = nullptr;
    const as_status st = guard([&] {
        Graph& g = G(gt);
        if (!g.is_transpose) throw InvalidArgument("spmm_transpose_values: graph is not a transpose");
        if (g.nnz && !vals_src_dev) throw InvalidArgument("spmm_transpose_values: values required");
        gp = &g;
    });
    if (st != AS_OK) return st;
    std::unique_ptr<GraphUse> use;
    const as_status st2 = guard([&] { use = std::make_unique<GraphUse>(*gp, resolve_stream(*gp, stream)); });
    if (st2 != AS_OK) return st2;
    ValPermScope scope(*gp);
    return spmm_entry(v, gt, vals_src_dev, b_dev, b_rows, f, c_dev, stream, res);
}

as_status as_permute_values(as_graph gt, const float* src_dev, float* dst_dev, void* stream) {
    return guard([&] {
        Graph& g = G(gt);
        if (!g.is_transpose) throw InvalidArgument("permute_values: graph is not a transpose");
        if (g.nnz && (!src_dev || !dst_dev)) throw InvalidArgument("permute_values: null array");
        DeviceGuard dg(g.device);
        GraphUse use(g, resolve_stream(g, stream));
        launch_permute(src_dev, g.src_perm.get(), g.nnz, dst_dev, resolve_stream(g, stream));
    });
}

static as_status spmm_half_entry(const as_variant* v, as_graph a, const float* vals_dev, const uint16_t* b_dev,
                                 uint64_t b_rows, uint64_t f, float* c_dev, void* stream, as_kernel_result* res,
                                 int wt, const char* name) {
    return guard([&] {
        Graph& g = G(a);
        // B is read only through entries: a graph without entries may pass
        // an empty (null) B, as the f32 entry points allow
        if ((g.n_rows && f && !c_dev) || (g.nnz && f && !b_dev))
            throw InvalidArgument(std::string(name) + ": null operand");
        GraphUse use(g, resolve_stream(g, stream));
        const KernelResult r = dispatch_spmm_half(v, g, vals_dev, b_dev, b_rows, f, c_dev,
                                                  resolve_stream(g, stream), res != nullptr, wt);
        fill_result(res, r);
    });
}

as_status as_spmm_bf16(const as_variant* v, as_graph a, const float* vals_dev, const uint16_t* b_dev,
                       uint64_t b_rows, uint64_t f, float* c_dev, void* stream, as_kernel_result* res) {
    return spmm_half_entry(v, a, vals_dev, b_dev, b_rows, f, c_dev, stream, res, 1, "spmm_bf16");
}

as_status as_spmm_f16(const as_variant* v, as_graph a, const float* vals_dev, const uint16_t* b_dev,
                      uint64_t b_rows, uint64_t f, float* c_dev, void* stream, as_kernel_result* res) {
    return spmm_half_entry(v, a, vals_dev, b_dev, b_rows, f, c_dev, stream, res, 2, "spmm_f16");
}

static as_status sddmm_half_entry(const as_variant* v, as_graph pattern, const uint16_t* x_dev, uint64_t x_rows,
                                  const uint16_t* y_dev, uint64_t y_rows, uint64_t f, float* out_dev, void* stream,
                                  as_kernel_result* res, int wt, const char* name) {
    return guard([&] {
        Graph& g = G(pattern);
        if (g.nnz && f && (!x_dev || !y_dev || !out_dev)) throw InvalidArgument(std::string(name) + ": null operand");
        GraphUse use(g, resolve_stream(g, stream));
        const KernelResult r = dispatch_sddmm_half(v, g, x_dev, x_rows, y_dev, y_rows, f, out_dev,
                                                   resolve_stream(g, stream), res != nullptr, wt);
        fill_result(res, r);
    });
}

as_status as_sddmm_bf16(const as_variant* v, as_graph pattern, const uint16_t* x_dev, uint64_t x_rows,
                        const uint16_t* y_dev, uint64_t y_rows, uint64_t f, float* out_dev, void* stream,
                        as_kernel_result* res) {
    return sddmm_half_entry(v, pattern, x_dev, x_rows, y_dev, y_rows, f, out_dev, stream, res, 1, "sddmm_bf16");
}

as_status as_sddmm_f16(const as_variant* v, as_graph pattern, const uint16_t* x_dev, uint64_t x_rows,
                       const uint16_t* y_dev, uint64_t y_rows, uint64_t f, float* out_dev, void* stream,
                       as_kernel_result* res) {
    return sddmm_half_entry(v, pattern, x_dev, x_rows, y_dev, y_rows, f, out_dev, stream, res, 2, "sddmm_f16");
}

as_status as_csr_attention_half(as_graph pattern, const as_variant* sddmm_v, const as_variant* spmm_v,
                                const uint16_t* q_dev, uint64_t q_rows, const uint16_t* k_dev, uint64_t k_rows,
                                const uint16_t* v_dev, uint64_t v_rows, uint64_t f, uint64_t fv, float* out_dev,
                                float* p_dev, int wt, int fused, void* stream) {
    return guard([&] {
        Graph& g = G(pattern);
        if (wt != 1 && wt != 2) throw InvalidArgument("attention_half: wt must be 1 (bf16) or 2 (f16)");
        if (g.n_rows && fv && !out_dev) throw InvalidArgument("attention_half: null output");
        if (g.nnz && f && (!q_dev || !k_dev)) throw InvalidArgument("attention_half: null operand");
        if (g.nnz && fv && !v_dev) throw InvalidArgument("attention_half: null operand");
        const cudaStream_t s = resolve_stream(g, stream);
        GraphUse use(g, s);
        attention_half(g, sddmm_v, spmm_v, q_dev, q_rows, k_dev, k_rows, v_dev, v_rows, f, fv, out_dev, p_dev,
                       fused != 0, wt, s);
    });
}

as_status as_row_softmax_backward(as_graph m, const float* p_dev, const float* grad_dev, float* ds_dev,
                                  void* stream) {
    return guard([&] {
        Graph& g = G(m);
        if (g.nnz && (!p_dev || !grad_dev || !ds_dev))
            throw InvalidArgument("row_softmax_backward: null array");
        DeviceGuard dg(g.device);
        GraphUse use(g, resolve_stream(g, stream));
        launch_row_softmax_backward(g, p_dev, grad_dev, ds_dev, resolve_stream(g, stream));
    });
}

// ---- synthetic inputs / io ------------------------------------------------------------
as_status as_gen_powerlaw(uint64_t n_rows, uint64_t n_cols, uint64_t nnz_target, double alpha,
                          uint64_t d_min, uint64_t d_max, uint64_t seed, int with_values,
                          uint64_t** rowptr, uint32_t** colind, float** val, uint64_t* nnz) {
    return guard([&] {
        std::vector<std::uint64_t> rp;
        std::vector<std::uint32_t> ci;
        std::vector<float> vv;
        gen_powerlaw(n_rows, n_cols, nnz_target, alpha, d_min, d_max, seed, with_values != 0, rp, ci, vv);
        *rowptr = malloc_copy(rp);
        *colind = malloc_copy(ci);
        *val = with_values ? malloc_copy(vv) : nullptr;
        *nnz = ci.size();
    });
}

as_status as_fill_uniform(float* host, uint64_t n, uint64_t seed) {
    return guard([&] { fill_uniform(host, n, seed); });
}

void as_free(void* p) { std::free(p); }

as_status as_save_csr(const char* path, const uint64_t* rowptr, const uint32_t* colind,
                      const float* val, uint64_t n_rows, uint64_t n_cols, uint64_t nnz) {
    return guard([&] { save_csr(path, rowptr, colind, val, n_rows, n_cols, nnz); });
}

as_status as_load_csr(const char* path, uint64_t** rowptr, uint32_t** colind, float** val,
                      uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz) {
    return guard([&] {
        std::vector<std::uint64_t> rp;
        std::vector<std::uint32_t> ci;
        std::vector<float> vv;
        load_csr(path, rp, ci, vv, *n_rows, *n_cols);
        *rowptr = malloc_copy(rp);
        *colind = malloc_copy(ci);
        *val = vv.empty() ? nullptr : malloc_copy(vv);
        *nnz = ci.size();
    });
}

as_status as_host_alloc(void** p, uint64_t bytes) {
    return guard([&] { ASB_CUDA(cudaMallocHost(p, std::max<std::uint64_t>(bytes, 1))); });
}

as_status as_host_free(void* p) {
    return guard([&] { ASB_CUDA(cudaFreeHost(p)); });
}

} // extern "C"
