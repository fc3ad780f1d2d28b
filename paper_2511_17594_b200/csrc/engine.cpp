// engine.cpp -- operator dispatch (src/kernels.cpp:465-531), the
// input-aware scheduler (src/scheduler.cpp:18-247) and the CSR attention
// pipeline (src/attention.cpp:9-46) over device graphs.
//
// Decision procedure (decide_common, src/scheduler.cpp:86-167), unchanged:
//   key = (device_sig, graph_sig, F, op) -> forced env knobs -> cache hit
//   (cached / replayed) -> replay-only miss (warn + baseline, or ReplayMiss)
//   -> features -> roofline shortlist[:top_k] -> probe lock -> time the
//   baseline kernel, then each candidate (strict < keeps the first of equal
//   medians) -> accept iff best >= 0 and t* <= alpha * t_b -> cache put.
// B200 changes: the probe sample (a degree-stratified induced row slice)
// is built on device and only when a probe actually runs -- the reference
// builds it before the cache lookup (src/scheduler.cpp:198-199); graph_sig
// is memoized per graph handle; probes are timed with CUDA events on the
// probe stream.
#include "engine.hpp"
#include "ops.hpp"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>

namespace asb {

namespace {

std::atomic<std::uint64_t> g_probe_launches{0};
std::mutex g_probe_mutex;  // one probe in flight per process (src/scheduler.cpp:20-22)

std::optional<as_variant> forced_env_variant(int op) {  // src/scheduler.cpp:46-59
    auto ft = env::get_int("AUTOSAGE_FTILE");
    auto wpb = env::get_int("AUTOSAGE_WPB");
    auto hub = env::get_int("AUTOSAGE_HUB_T");
    if (!ft && !wpb && !hub) return std::nullopt;
    as_variant v = default_variant();
    v.op = op;
    v.mapping = hub ? AS_MAP_HUBSPLIT : AS_MAP_ROWPARALLEL;
    if (ft && *ft > 0) v.f_tile = std::uint64_t(*ft);
    if (wpb && *wpb > 0) v.rows_per_chunk = std::uint64_t(*wpb);
    if (hub && *hub > 0) v.hub_threshold = std::uint64_t(*hub);
    v.vectorized = 0;
    return v;
}

void set_key(as_decision& d, const as_device_profile& dp, std::uint64_t sig, std::uint64_t f,
             int op) {
    std::snprintf(d.key.device_sig, sizeof d.key.device_sig, "%s", dp.device_sig);
    d.key.graph_sig = sig;
    d.key.f = f;
    d.key.op = op;
}

std::string choice_string(const as_decision& d) {
    return d.has_choice ? variant_to_string(d.choice) : std::string("baseline");
}

void from_record(const Record& rec, int source, as_decision& d) {  // src/scheduler.cpp:61-70
    d.key = key_to_c(rec.key);
    d.alpha = rec.alpha;
    d.source = source;
    d.has_choice = rec.choice != "baseline";
    if (d.has_choice) d.choice = variant_from_string(rec.choice);
    d.baseline_ms = rec.t_b;
    d.t_star = rec.t_star;
}

Record to_record(const as_decision& d) {  // src/scheduler.cpp:72-82
    Record rec;
    rec.key = key_from_c(d.key);
    rec.choice = choice_string(d);
    rec.t_b = d.baseline_ms;
    rec.t_star = d.t_star;
    rec.alpha = d.alpha;
    rec.timestamp = unix_now();
    rec.toolchain = toolchain_tag();
    return rec;
}

// AUTOSAGE_PROBE_FLUSH_L2=<MiB> (default: twice the device's L2, 0 = off):
// before each timed probe run, overwrite that many bytes on the probe
// stream, outside the timed events, so candidates are timed from a cold L2
// -- the condition of a step whose operands were evicted since the last op
// (bench.py flushes between steps).  A warm-L2 probe on the small sample
// ranks mappings whose cold costs differ: c1 (1.6M nnz, F=64) picked
// rowparallel (0.143-0.147 ms on a cold step) in 3 of 3 runs, the cold probe
// hub-split (0.105 ms) in 3 of 3; Reddit-shape picks are unchanged.  The
// buffer lives for one decide call (allocated only when the CUDA-event timer
// runs) and is freed with it.
std::size_t probe_flush_bytes() {
    const auto knob = env::get_int("AUTOSAGE_PROBE_FLUSH_L2");
    if (knob) return *knob > 0 ? std::size_t(*knob) << 20 : 0;
    int dev = 0, l2 = 0;
    ASB_CUDA(cudaGetDevice(&dev));
    ASB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    return std::size_t(std::max(l2, 1 << 20)) * 2;
}

TimeOnce event_timer(cudaStream_t s, std::shared_ptr<DevBuf<char>> flush) {
    return [s, flush](const std::string&, const std::function<void()>& run) {
        cudaEvent_t e0, e1;
        ASB_CUDA(cudaEventCreate(&e0));
        ASB_CUDA(cudaEventCreate(&e1));
        if (flush && flush->size())
            ASB_CUDA(cudaMemsetAsync(flush->get(), 0x5a, flush->size(), s));
        ASB_CUDA(cudaEventRecord(e0, s));
        run();
        ASB_CUDA(cudaEventRecord(e1, s));
        ASB_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        ASB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return double(ms);
    };
}

struct ProbeHooks {
    std::function<as_features()> features;                 // full-graph features
    std::function<std::uint64_t()> prepare;                // build the sample, return its rows
    std::function<void()> run_baseline;
    std::function<void(const as_variant&)> run_candidate;
    cudaStream_t stream = nullptr;
};

as_decision decide_common(const Context& ctx, const as_probe_config& cfg,
                          const as_device_profile& dp, const std::function<std::uint64_t()>& sig,
                          std::uint64_t f, int op, ProbeHooks& hooks) {
    check_probe_config(cfg);
    using clk = std::chrono::steady_clock;
    auto ms_since = [](clk::time_point t) {
        return std::chrono::duration<double, std::milli>(clk::now() - t).count();
    };
    const auto call0 = clk::now();
    as_decision d{};
    d.best_index = -1;
    set_key(d, dp, sig(), f, op);
    d.sig_ms = ms_since(call0);
    d.alpha = cfg.alpha;
    struct WallOnExit {
        as_decision& d;
        clk::time_point t0;
        ~WallOnExit() { d.decide_wall_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count(); }
    } wall_on_exit{d, call0};

    if (auto forced = forced_env_variant(op)) {
        d.has_choice = 1;
        d.choice = *forced;
        d.source = AS_SRC_FORCED_ENV;
        return d;
    }
    if (ctx.cache) {
        if (auto rec = ctx.cache->get(key_from_c(d.key))) {
            from_record(*rec, ctx.replay.replay_only ? AS_SRC_REPLAYED : AS_SRC_CACHED, d);
            return d;
        }
    }
    if (ctx.replay.replay_only) {
        const std::string k = key_from_c(d.key).to_string();
        if (ctx.replay.strict) throw ReplayMissError("replay miss for key " + k);
        std::fprintf(stderr, "autosage: warning: replay miss for %s, using baseline\n", k.c_str());
        d.source = AS_SRC_REPLAYED;
        d.has_choice = 0;
        return d;
    }

    auto t_phase = clk::now();
    const as_features gf = hooks.features();
    d.features_ms = ms_since(t_phase);
    auto candidates = shortlist(gf, f, op, dp);
    if (dp.model == AS_MODEL_B200) {
        l2_tile_rule(candidates, f, gf.n_cols);
        candidates = distinct_gpu_configs(candidates, f);
    }
    if (candidates.size() > std::size_t(cfg.top_k)) candidates.resize(std::size_t(cfg.top_k));
    t_phase = clk::now();
    const std::uint64_t sample_rows = hooks.prepare ? hooks.prepare() : 0;
    d.sample_ms = ms_since(t_phase);

    std::shared_ptr<DevBuf<char>> flush;
    if (!ctx.timer) {
        flush = std::make_shared<DevBuf<char>>();
        if (const std::size_t fb = probe_flush_bytes()) flush->alloc(fb);
    }
    TimeOnce timer = ctx.timer ? ctx.timer : event_timer(hooks.stream, flush);
    std::lock_guard<std::mutex> probe_lock(g_probe_mutex);
    cudaStream_t ps = hooks.stream;
    set_warmup_sync(ps ? std::function<void()>([ps] { cudaStreamSynchronize(ps); })
                       : std::function<void()>());
    const auto wall0 = std::chrono::steady_clock::now();

    d.sample_rows = sample_rows;
    auto tb = time_kernel("baseline", hooks.run_baseline, cfg.iters, cfg.cap_ms, timer);
    g_probe_launches += std::uint64_t(tb.launches);
    d.baseline_ms = tb.median_ms;
    d.baseline_completed = tb.completed;
    d.baseline_capped = tb.capped;
    d.max_single_run_ms = tb.max_run_ms;

    double t_star = std::numeric_limits<double>::infinity();
    int best = -1;
    for (std::size_t c = 0; c < candidates.size(); ++c) {
        const as_variant cand = candidates[c];
        auto st = time_kernel(variant_to_string(cand), [&] { hooks.run_candidate(cand); },
                              cfg.iters, cfg.cap_ms, timer);
        g_probe_launches += std::uint64_t(st.launches);
        if (d.n_candidates < AS_MAX_CANDIDATES) {
            as_candidate_timing& ct = d.candidates[d.n_candidates++];
            ct.variant = cand;
            ct.median_ms = st.median_ms;
            ct.completed = st.completed;
            ct.capped = st.capped;
        }
        d.max_single_run_ms = std::max(d.max_single_run_ms, st.max_run_ms);
        if (st.median_ms < t_star) {
            t_star = st.median_ms;
            best = int(c);
        }
    }
    set_warmup_sync({});
    d.t_star = t_star;
    d.best_index = best;
    d.probe_wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
    if (best >= 0 && t_star <= cfg.alpha * d.baseline_ms) {
        d.has_choice = 1;
        d.choice = candidates[std::size_t(best)];
    } else {
        d.has_choice = 0;
    }
    d.source = AS_SRC_PROBED;
    if (ctx.cache) ctx.cache->put(to_record(d));
    return d;
}

const as_device_profile& profile_for(const Context& ctx, int device) {
    return ctx.device ? *ctx.device : gpu_profile(device);
}

struct TimedRegion {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaStream_t s;
    bool on;
    TimedRegion(cudaStream_t st, bool enable) : s(st), on(enable) {
        if (!on) return;
        ASB_CUDA(cudaEventCreate(&e0));
        ASB_CUDA(cudaEventCreate(&e1));
        ASB_CUDA(cudaEventRecord(e0, s));
    }
    double stop() {
        if (!on) return 0.0;
        ASB_CUDA(cudaEventRecord(e1, s));
        ASB_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        ASB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        return double(ms);
    }
    ~TimedRegion() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

void check_spmm_dims(const Graph& a, std::uint64_t b_rows) {  // src/kernels.cpp:33-37
    if (a.n_cols != b_rows) throw InvalidArgument("spmm: a.n_cols != b.n_rows");
}

void check_sddmm_dims(const Graph& p, std::uint64_t x_rows, std::uint64_t y_rows) {
    if (x_rows != p.n_rows) throw InvalidArgument("sddmm: x.n_rows != pattern.n_rows");
    if (y_rows != p.n_cols) throw InvalidArgument("sddmm: y.n_rows != pattern.n_cols");
}

// Device flag enabling the ALU re-bias half of the f32 -> f64 widening
// (widen.cuh), or nullptr for the all-F2F path.  The scan costs a full read
// of the dense operand; it pays only when the gathers are L2-resident and the
// XU pipe is a limiter.  A gathered operand larger than ~3/4 of L2 streams from
// DRAM, where the widening is not on the critical path (Products-shape B,
// 980 MB: the scan alone was 0.15 ms per call).
// A probe sample scans its operand once (decide_*'s prepare hook) and
// freezes the flag, so candidate timings do not include a scan the
// baseline's do not.
// Finite scan of the dense operand (gates the ALU re-bias widening).
// Operands above the cap skip it and widen every component on the XU pipe.
// SpMM: 128 MiB -- Reddit F=128 (B 119 MB) 4.16 -> 4.04 ms with it, but
// further past the L2 the gathers bound the kernel and the scan is pure
// cost (Reddit F=256 8.38 -> 8.72 ms, Products F=100 8.98 -> 9.54 ms).  SDDMM: no cap -- its dot is XU-bound at any size (F=128 5.77 ->
// 5.25 ms, F=256 11.72 -> 10.58 ms, Products 11.98 -> 11.85 ms with it,
// scan included; profiles/r02o_mix_scan.md).  AUTOSAGE_DEV_MIX_SCAN_MB
// (MiB) overrides both caps (A/B knob).
// Small products skip it too: the scan is a separate ~10 us launch in front
// of a latency-bound op whose XU is not the limit -- c1 (1.6M nnz x 64)
// SpMM 0.080 -> 0.066 ms, SDDMM 0.105 -> 0.095 ms without it
// (profiles/r02aj_small_scan.md).  Rule: scan only when the op multiplies at
// least 2^28 entry-features (nnz x F); AUTOSAGE_DEV_MIX_MIN_WORK overrides.
const unsigned* mix_flag(Graph& g, const float* p, std::uint64_t n, cudaStream_t s, bool sddmm = false) {
    const auto knob = env::get_int("AUTOSAGE_DEV_MIX_SCAN_MB");
    const std::uint64_t dflt = sddmm ? ~0ull : std::uint64_t(128) << 20;
    const std::uint64_t max_bytes = knob && *knob >= 0 ? std::uint64_t(*knob) << 20 : dflt;
    if (n * 4 > max_bytes) return nullptr;
    {
        const auto w = env::get_int("AUTOSAGE_DEV_MIX_MIN_WORK");
        const std::uint64_t min_work = w && *w >= 0 ? std::uint64_t(*w) : (std::uint64_t(1) << 28);
        const std::uint64_t nnz = g.plan_nnz ? g.plan_nnz : g.nnz;
        const std::uint64_t f = n / std::max<std::uint64_t>(g.n_cols, 1);
        if (nnz * f < min_work) return nullptr;
    }
    if (g.flag_frozen) return g.flag.get();
    return finite_flag(g, p, n, s);
}

void freeze_mix_flag(Graph& g, const float* p, std::uint64_t n, cudaStream_t s, bool sddmm = false) {
    g.flag_frozen = false;
    mix_flag(g, p, n, s, sddmm);
    g.flag_frozen = true;
}

// rmax/rsum (softmax mode, fused attention): vals are the stats pass's ex and
// the kernels turn them into probabilities on the fly (ops.hpp)
void run_spmm_variant(const as_variant& v, Graph& a, const float* vals, const float* b,
                      std::uint64_t f, float* c, cudaStream_t s, bool vec,
                      const float* rmax = nullptr, const double* rsum = nullptr) {
    switch (v.mapping) {
        case AS_MAP_BASELINE:
            launch_spmm_baseline(a, vals, b, std::uint32_t(f), c, s);
            break;
        case AS_MAP_ROWPARALLEL: {
            ensure_order(a);
            const unsigned* fin = mix_flag(a, b, a.n_cols * f, s);
            launch_spmm_rows(a, vals, 0, a.n_rows, b, std::uint32_t(f), c, v.f_tile, vec,
                             std::uint32_t(std::min<std::uint64_t>(v.rows_per_chunk, 16)), s, fin, rmax,
                             rsum);
            break;
        }
        case AS_MAP_HUBSPLIT: {
            const unsigned* fin = mix_flag(a, b, a.n_cols * f, s);
            launch_spmm_hubsplit(a, vals, b, std::uint32_t(f), c, v.f_tile, vec,
                                 std::uint32_t(std::min<std::uint64_t>(v.rows_per_chunk, 16)),
                                 v.hub_threshold, s, fin, rmax, rsum);
            break;
        }
    }
}

} // namespace

// ---- operators --------------------------------------------------------------

void spmm_baseline(Graph& a, const float* vals, const float* b, std::uint64_t b_rows,
                   std::uint64_t f, float* c, cudaStream_t s) {
    check_spmm_dims(a, b_rows);
    DeviceGuard dg(a.device);
    launch_spmm_baseline(a, vals, b, std::uint32_t(f), c, s);
}

void spmm_mapped(const as_variant& v, int expect_mapping, Graph& a, const float* vals,
                 const float* b, std::uint64_t b_rows, std::uint64_t f, float* c, cudaStream_t s) {
    check_spmm_dims(a, b_rows);
    check_variant(v);
    if (v.mapping != expect_mapping)
        throw InvalidArgument(expect_mapping == AS_MAP_ROWPARALLEL
                                  ? "spmm_rowparallel: variant mapping mismatch"
                                  : "spmm_hubsplit: variant mapping mismatch");
    DeviceGuard dg(a.device);
    const void* bases[1] = {b};
    // SpMM numerics do not depend on the vec flag (per-feature CSR order,
    // src/kernels.cpp:63-80), so the kernels load float4 whenever the gate
    // passes; `vectorized` only selects what the reference reports.
    run_spmm_variant(v, a, graph_values(a, vals), b, f, c, s, vec4_eligible(f, bases, 1));
}

KernelResult dispatch_spmm(const as_variant& v, Graph& a, const float* vals, const float* b,
                           std::uint64_t b_rows, std::uint64_t f, float* c, cudaStream_t s,
                           bool timed) {
    if (v.op != AS_OP_SPMM)
        throw InvalidArgument("dispatch: spmm operands given to a non-spmm variant");
    check_spmm_dims(a, b_rows);
    KernelResult r;
    r.variant = apply_env_overrides(v);
    check_variant(r.variant);
    const void* bases[1] = {b};
    const bool vec = r.variant.vectorized && vec4_eligible(f, bases, 1);
    DeviceGuard dg(a.device);
    if (r.variant.mapping == AS_MAP_ROWPARALLEL) ensure_order(a);
    if (r.variant.mapping == AS_MAP_HUBSPLIT) ensure_hub_plan(a, r.variant.hub_threshold);
    TimedRegion tr(s, timed);
    run_spmm_variant(r.variant, a, graph_values(a, vals), b, f, c, s, vec4_eligible(f, bases, 1));
    r.elapsed_ms = tr.stop();
    r.vectorized_path = vec && r.variant.mapping != AS_MAP_BASELINE;
    return r;
}

// SpMM with a 16-bit B (bf16 or f16 words, wt):
// the same kernels reading half the gather bytes.  Either -> f32 is exact, so
// the result equals the f32
// SpMM on float(B) bit for bit.  v == nullptr: baseline.  The 4-wide path
// (8-byte loads) needs f % 4 == 0 and an 8-byte aligned base; the ring
// kernel and the softmax mode stay f32-only.
KernelResult dispatch_spmm_half(const as_variant* v, Graph& a, const float* vals, const std::uint16_t* b,
                                std::uint64_t b_rows, std::uint64_t f, float* c, cudaStream_t s, bool timed,
                                int wt) {
    check_spmm_dims(a, b_rows);
    KernelResult r;
    if (v) {
        if (v->op != AS_OP_SPMM) throw InvalidArgument("dispatch: spmm operands given to a non-spmm variant");
        r.variant = apply_env_overrides(*v);
        check_variant(r.variant);
    } else {
        r.variant = default_variant();
        r.variant.mapping = AS_MAP_BASELINE;
    }
    const bool vec_ok = f > 0 && f % 4 == 0 && (reinterpret_cast<std::uintptr_t>(b) & 7) == 0;
    DeviceGuard dg(a.device);
    const float* va = graph_values(a, vals);
    const std::uint32_t wpb = std::uint32_t(std::min<std::uint64_t>(r.variant.rows_per_chunk, 16));
    const unsigned* fin = nullptr;
    if (r.variant.mapping != AS_MAP_BASELINE) {
        if (r.variant.mapping == AS_MAP_ROWPARALLEL) ensure_order(a);
        else ensure_hub_plan(a, r.variant.hub_threshold);
        if (a.n_cols * f * 2 <= (std::uint64_t(96) << 20)) fin = finite_flag_half(a, b, a.n_cols * f, s, wt);
    }
    TimedRegion tr(s, timed);
    switch (r.variant.mapping) {
        case AS_MAP_BASELINE:
            launch_spmm_baseline(a, va, b, std::uint32_t(f), c, s, wt);
            break;
        case AS_MAP_ROWPARALLEL:
            launch_spmm_rows(a, va, 0, a.n_rows, b, std::uint32_t(f), c, r.variant.f_tile, vec_ok, wpb, s, fin,
                             nullptr, nullptr, wt);
            break;
        case AS_MAP_HUBSPLIT:
            launch_spmm_hubsplit(a, va, b, std::uint32_t(f), c, r.variant.f_tile, vec_ok, wpb,
                                 r.variant.hub_threshold, s, fin, nullptr, nullptr, wt);
            break;
    }
    r.elapsed_ms = tr.stop();
    r.vectorized_path = r.variant.vectorized && vec_ok && r.variant.mapping != AS_MAP_BASELINE;
    return r;
}

// SDDMM on bf16 X and Y (raw words).  The vec flag selects the reference's
// four-way block order (src/kernels.cpp:103-127) whenever f % 4 == 0 -- the
// gate the f32 copies of X and Y would pass -- so the result is as_sddmm on
// float(X), float(Y) with the same variant, bit for bit.
KernelResult dispatch_sddmm_half(const as_variant* v, Graph& p, const std::uint16_t* x, std::uint64_t x_rows,
                                 const std::uint16_t* y, std::uint64_t y_rows, std::uint64_t f, float* out,
                                 cudaStream_t s, bool timed, int wt) {
    check_sddmm_dims(p, x_rows, y_rows);
    KernelResult r;
    if (v) {
        if (v->op != AS_OP_SDDMM) throw InvalidArgument("dispatch: sddmm operands given to a non-sddmm variant");
        r.variant = apply_env_overrides(*v);
        check_variant(r.variant);
    } else {
        r.variant = default_variant();
        r.variant.op = AS_OP_SDDMM;
        r.variant.mapping = AS_MAP_BASELINE;
    }
    const bool baseline = r.variant.mapping == AS_MAP_BASELINE;
    const int ord = !baseline && r.variant.vectorized && f > 0 && f % 4 == 0 ? 1 : 0;
    const std::uint32_t ft = std::uint32_t(baseline ? std::max<std::uint64_t>(f, 1) : effective_tile(r.variant.f_tile, f));
    DeviceGuard dg(p.device);
    TimedRegion tr(s, timed);
    launch_sddmm_half(p, x, y, std::uint32_t(f), out, ft, ord, baseline, s, wt);
    r.elapsed_ms = tr.stop();
    r.vectorized_path = ord == 1;
    return r;
}

void sddmm_baseline(Graph& p, const float* x, std::uint64_t x_rows, const float* y,
                    std::uint64_t y_rows, std::uint64_t f, float* out, cudaStream_t s) {
    check_sddmm_dims(p, x_rows, y_rows);
    DeviceGuard dg(p.device);
    launch_sddmm_baseline(p, x, y, std::uint32_t(f), out, s);
}

void sddmm_mapped(const as_variant& v, Graph& p, const float* x, std::uint64_t x_rows,
                  const float* y, std::uint64_t y_rows, std::uint64_t f, float* out,
                  cudaStream_t s) {
    check_sddmm_dims(p, x_rows, y_rows);
    check_variant(v);
    if (v.mapping == AS_MAP_BASELINE)
        throw InvalidArgument("sddmm_rowparallel: variant mapping mismatch");
    const void* bases[2] = {x, y};
    const bool vec = v.vectorized && vec4_eligible(f, bases, 2);
    DeviceGuard dg(p.device);
    const unsigned* fin = mix_flag(p, y, y_rows * f, s, true);
    launch_sddmm_chunks(p, x, y, std::uint32_t(f), out, v.f_tile, vec,
                        std::uint32_t(std::min<std::uint64_t>(v.rows_per_chunk, 16)), s, fin);
}

KernelResult dispatch_sddmm(const as_variant& v, Graph& p, const float* x, std::uint64_t x_rows,
                            const float* y, std::uint64_t y_rows, std::uint64_t f, float* out,
                            cudaStream_t s, bool timed) {
    if (v.op != AS_OP_SDDMM)
        throw InvalidArgument("dispatch: sddmm operands given to a non-sddmm variant");
    check_sddmm_dims(p, x_rows, y_rows);
    KernelResult r;
    r.variant = apply_env_overrides(v);
    check_variant(r.variant);
    const void* bases[2] = {x, y};
    const bool vec = r.variant.vectorized && vec4_eligible(f, bases, 2);
    DeviceGuard dg(p.device);
    ensure_chunk_rows(p);
    TimedRegion tr(s, timed);
    if (r.variant.mapping == AS_MAP_BASELINE) {
        launch_sddmm_baseline(p, x, y, std::uint32_t(f), out, s);
    } else {
        const unsigned* fin = mix_flag(p, y, y_rows * f, s, true);
        launch_sddmm_chunks(p, x, y, std::uint32_t(f), out, r.variant.f_tile, vec,
                            std::uint32_t(std::min<std::uint64_t>(r.variant.rows_per_chunk, 16)), s,
                            fin);
    }
    r.elapsed_ms = tr.stop();
    r.vectorized_path = vec && r.variant.mapping != AS_MAP_BASELINE;
    return r;
}

// ---- host-buffer pipeline ------------------------------------------------------------
namespace {

void ensure_pipe(Graph& g) {
    auto& P = g.pipe;
    if (P.h2d) return;
    ASB_CUDA(cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking));
    ASB_CUDA(cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&P.spmm_in, &P.spmm_done, &P.spmm_out, &P.sddmm_in, &P.sddmm_done,
                           &P.sddmm_out})
        ASB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

void ensure_slices(Graph& g, std::size_t k) {
    for (auto* v : {&g.pipe.slice, &g.pipe.slice_x})
        while (v->size() < k) {
            cudaEvent_t e;
            ASB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            v->push_back(e);
        }
}

// row holding entry e (host rowptr mirror)
std::uint64_t host_row_of(const Graph& g, std::uint64_t e) {
    const auto it = std::upper_bound(g.h_rowptr.begin(), g.h_rowptr.end(), e);
    return std::uint64_t(it - g.h_rowptr.begin()) - 1;
}

std::uint64_t host_slices() {
    const auto k = env::get_int("AUTOSAGE_HOST_SLICES");
    return k && *k > 0 ? std::uint64_t(*k) : 16;
}

// first host slice = 1/head of an even slice (AUTOSAGE_HOST_HEAD; 1 = even)
std::uint64_t host_head() {
    const auto h = env::get_int("AUTOSAGE_HOST_HEAD");
    return h && *h > 0 ? std::uint64_t(*h) : 8;
}

}  // namespace

KernelResult spmm_host(const as_variant* v, Graph& g, const float* b_host, std::uint64_t b_rows,
                       std::uint64_t f, float* c_host, bool sync) {
    check_spmm_dims(g, b_rows);
    DeviceGuard dg(g.device);
    ensure_pipe(g);
    auto& P = g.pipe;
    P.b.ensure(std::max<std::uint64_t>(b_rows * f, 1));
    P.c.ensure(std::max<std::uint64_t>(g.n_rows * f, 1));
    // the previous SpMM's kernel must have finished reading the staging B
    ASB_CUDA(cudaStreamWaitEvent(P.h2d, P.spmm_done, 0));
    if (b_rows && f)
        ASB_CUDA(cudaMemcpyAsync(P.b.get(), b_host, b_rows * f * 4, cudaMemcpyHostToDevice, P.h2d));
    ASB_CUDA(cudaEventRecord(P.spmm_in, P.h2d));
    ASB_CUDA(cudaStreamWaitEvent(g.stream, P.spmm_in, 0));
    ASB_CUDA(cudaStreamWaitEvent(g.stream, P.spmm_out, 0));  // staging C free again
    KernelResult r;
    if (v) {
        r = dispatch_spmm(*v, g, nullptr, P.b.get(), b_rows, f, P.c.get(), g.stream, false);
    } else {
        r.variant = default_variant();
        r.variant.mapping = AS_MAP_BASELINE;
        launch_spmm_baseline(g, graph_values(g, nullptr), P.b.get(), std::uint32_t(f), P.c.get(), g.stream);
    }
    ASB_CUDA(cudaEventRecord(P.spmm_done, g.stream));
    ASB_CUDA(cudaStreamWaitEvent(P.d2h, P.spmm_done, 0));
    if (g.n_rows && f)
        ASB_CUDA(cudaMemcpyAsync(c_host, P.c.get(), g.n_rows * f * 4, cudaMemcpyDeviceToHost, P.d2h));
    ASB_CUDA(cudaEventRecord(P.spmm_out, P.d2h));
    if (sync) ASB_CUDA(cudaEventSynchronize(P.spmm_out));
    return r;
}

KernelResult sddmm_host(const as_variant* v, Graph& g, const float* x_host, std::uint64_t x_rows,
                        const float* y_host, std::uint64_t y_rows, std::uint64_t f, float* out_host,
                        bool sync) {
    check_sddmm_dims(g, x_rows, y_rows);
    DeviceGuard dg(g.device);
    ensure_pipe(g);
    ensure_chunk_rows(g);
    auto& P = g.pipe;
    KernelResult r;
    if (v) {
        if (v->op != AS_OP_SDDMM)
            throw InvalidArgument("dispatch: sddmm operands given to a non-sddmm variant");
        r.variant = apply_env_overrides(*v);
        check_variant(r.variant);
    } else {
        r.variant = default_variant();
        r.variant.op = AS_OP_SDDMM;
        r.variant.mapping = AS_MAP_BASELINE;
    }
    P.x.ensure(std::max<std::uint64_t>(x_rows * f, 1));
    P.y.ensure(std::max<std::uint64_t>(y_rows * f, 1));
    P.v.ensure(std::max<std::uint64_t>(g.nnz, 1));
    ASB_CUDA(cudaStreamWaitEvent(P.h2d, P.sddmm_done, 0));
    // Y first (every slice gathers from all of it); X follows slice by slice
    if (y_rows && f)
        ASB_CUDA(cudaMemcpyAsync(P.y.get(), y_host, y_rows * f * 4, cudaMemcpyHostToDevice, P.h2d));
    ASB_CUDA(cudaEventRecord(P.sddmm_in, P.h2d));
    ASB_CUDA(cudaStreamWaitEvent(g.stream, P.sddmm_in, 0));
    ASB_CUDA(cudaStreamWaitEvent(g.stream, P.sddmm_out, 0));

    const float *x = P.x.get(), *y = P.y.get();
    float* out = P.v.get();
    const void* bases[2] = {x, y};
    const bool vec = r.variant.vectorized && vec4_eligible(f, bases, 2);
    r.vectorized_path = vec && r.variant.mapping != AS_MAP_BASELINE;
    const std::uint64_t n_chunks = (g.nnz + 31) / 32;
    const std::uint64_t k = std::max<std::uint64_t>(1, std::min(host_slices(), n_chunks));
    const std::uint64_t per = (n_chunks + k - 1) / std::max<std::uint64_t>(k, 1);
    // the first slice is cut short (1/head of the others) so the D2H link,
    // the step's bottleneck, starts as soon as Y has landed; the rest stay even
    const std::uint64_t head = std::max<std::uint64_t>(1, per / host_head());
    const std::uint64_t rest = k > 1 ? (n_chunks - std::min(n_chunks, head) + k - 2) / (k - 1) : per;
    auto slice_begin = [&](std::uint64_t i) {
        if (k == 1 || i == 0) return i == 0 ? std::uint64_t(0) : n_chunks;
        return std::min(n_chunks, head + (i - 1) * rest);
    };
    ensure_slices(g, std::size_t(k));
    const unsigned* fin = nullptr;
    const std::uint32_t wpb = std::uint32_t(std::min<std::uint64_t>(r.variant.rows_per_chunk, 16));
    if (r.variant.mapping != AS_MAP_BASELINE) fin = mix_flag(g, y, y_rows * f, g.stream, true);
    std::uint64_t x_done = 0;  // X rows [0, x_done) queued
    for (std::uint64_t i = 0; i < k && n_chunks; ++i) {
        const std::uint64_t c0 = slice_begin(i), c1 = i + 1 == k ? n_chunks : slice_begin(i + 1);
        if (c0 >= c1) break;
        // X rows of this slice's entries
        const std::uint64_t ra = host_row_of(g, c0 * 32);
        const std::uint64_t rb = host_row_of(g, std::min(c1 * 32, g.nnz) - 1) + 1;
        if (rb > x_done && f) {
            const std::uint64_t from = std::max(ra, x_done);
            ASB_CUDA(cudaMemcpyAsync(P.x.get() + from * f, x_host + from * f, (rb - from) * f * 4,
                                     cudaMemcpyHostToDevice, P.h2d));
            x_done = rb;
        }
        ASB_CUDA(cudaEventRecord(P.slice_x[i], P.h2d));
        ASB_CUDA(cudaStreamWaitEvent(g.stream, P.slice_x[i], 0));
        if (r.variant.mapping != AS_MAP_BASELINE)
            sddmm_chunks_prepare(g, x, y, std::uint32_t(f), r.variant.f_tile, vec, g.stream, fin, ra, rb);
        if (r.variant.mapping == AS_MAP_BASELINE)
            launch_sddmm_baseline(g, x, y, std::uint32_t(f), out, g.stream, c0, c1);
        else
            launch_sddmm_chunks(g, x, y, std::uint32_t(f), out, r.variant.f_tile, vec, wpb, g.stream, fin, c0,
                                c1, false);
        ASB_CUDA(cudaEventRecord(P.slice[i], g.stream));
        ASB_CUDA(cudaStreamWaitEvent(P.d2h, P.slice[i], 0));
        const std::uint64_t e0 = c0 * 32, e1 = std::min(c1 * 32, g.nnz);
        ASB_CUDA(cudaMemcpyAsync(out_host + e0, out + e0, (e1 - e0) * 4, cudaMemcpyDeviceToHost, P.d2h));
    }
    if (x_done < x_rows && f)  // rows after the last entry (empty rows): keep P.x complete
        ASB_CUDA(cudaMemcpyAsync(P.x.get() + x_done * f, x_host + x_done * f, (x_rows - x_done) * f * 4,
                                 cudaMemcpyHostToDevice, P.h2d));
    ASB_CUDA(cudaEventRecord(P.sddmm_done, g.stream));
    ASB_CUDA(cudaStreamWaitEvent(P.d2h, P.sddmm_done, 0));
    ASB_CUDA(cudaEventRecord(P.sddmm_out, P.d2h));
    if (sync) ASB_CUDA(cudaEventSynchronize(P.sddmm_out));
    return r;
}

void host_synchronize(Graph& g) {
    DeviceGuard dg(g.device);
    if (g.pipe.d2h) ASB_CUDA(cudaStreamSynchronize(g.pipe.d2h));
    if (g.pipe.h2d) ASB_CUDA(cudaStreamSynchronize(g.pipe.h2d));
    ASB_CUDA(cudaStreamSynchronize(g.stream));
}

void row_softmax(Graph& m, const float* vin, float* vout, cudaStream_t s) {
    if (m.nnz > 0 && vin == nullptr) throw InvalidArgument("row_softmax: values required");
    DeviceGuard dg(m.device);
    launch_row_softmax(m, vin, vout, s);
}

// ---- scheduler ---------------------------------------------------------------

// Probe sample rows.  The reference takes max(min_rows, ceil(frac*N))
// (src/generate.cpp:134-181).  A 2% sample of a mid-size graph is a few
// microseconds of GPU work -- launch latency, not the kernels -- so under the
// B200 model the sample is raised until it holds about
// AUTOSAGE_GPU_PROBE_NNZ (default 4M) entries at the graph's mean degree;
// the row selection itself is unchanged.
std::uint64_t probe_min_rows(const Graph& g, const as_probe_config& cfg, const as_device_profile& dp) {
    std::uint64_t rows = cfg.min_rows;
    if (dp.model != AS_MODEL_B200 || g.n_rows == 0 || g.nnz == 0) return rows;
    const auto knob = env::get_int("AUTOSAGE_GPU_PROBE_NNZ");
    const double want = knob && *knob > 0 ? double(*knob) : 4.0e6;
    const double mean = double(g.nnz) / double(g.n_rows);
    const auto need = std::uint64_t(std::ceil(want / std::max(mean, 1.0)));
    return std::min<std::uint64_t>(g.n_rows, std::max(rows, need));
}

as_decision decide_spmm(const Context& ctx, const as_probe_config& cfg, Graph& a,
                        const float* vals, const float* b, std::uint64_t b_rows, std::uint64_t f) {
    if (a.n_cols != b_rows) throw InvalidArgument("decide_spmm: dimension mismatch");
    DeviceGuard dg(a.device);
    cudaStream_t s = ctx.stream ? ctx.stream : a.stream;
    std::unique_ptr<Graph> sample;
    DevBuf<float> cbuf;
    ProbeHooks h;
    h.stream = s;
    h.features = [&] { return graph_features(a, kDefaultHubThreshold); };
    const as_device_profile& dp = profile_for(ctx, a.device);
    h.prepare = [&]() -> std::uint64_t {
        const auto rows = sample_row_indices(a, cfg.frac, probe_min_rows(a, cfg, dp));
        sample = slice_rows(a, rows, graph_values(a, vals));
        ensure_order(*sample);
        freeze_mix_flag(*sample, b, a.n_cols * f, s);
        cbuf.alloc(std::max<std::uint64_t>(rows.size() * f, 1));
        return rows.size();
    };
    h.run_baseline = [&] {
        launch_spmm_baseline(*sample, graph_values(*sample, nullptr), b, std::uint32_t(f), cbuf.get(), s);
    };
    h.run_candidate = [&](const as_variant& v) {
        dispatch_spmm(v, *sample, nullptr, b, b_rows, f, cbuf.get(), s, false);
    };
    return decide_common(ctx, cfg, dp, [&] { return graph_sig(a); }, f, AS_OP_SPMM, h);
}

as_decision decide_sddmm(const Context& ctx, const as_probe_config& cfg, Graph& p,
                         const float* x, std::uint64_t x_rows, const float* y,
                         std::uint64_t y_rows, std::uint64_t f) {
    if (x_rows != p.n_rows || y_rows != p.n_cols)
        throw InvalidArgument("decide_sddmm: dimension mismatch");
    DeviceGuard dg(p.device);
    cudaStream_t s = ctx.stream ? ctx.stream : p.stream;
    std::unique_ptr<Graph> sample;
    DevBuf<float> xs, obuf;
    std::uint64_t ns = 0;
    ProbeHooks h;
    h.stream = s;
    h.features = [&] { return graph_features(p, kDefaultHubThreshold); };
    const as_device_profile& dp = profile_for(ctx, p.device);
    h.prepare = [&]() -> std::uint64_t {
        const auto rows = sample_row_indices(p, cfg.frac, probe_min_rows(p, cfg, dp));
        sample = slice_rows(p, rows, nullptr);  // SDDMM ignores pattern values
        ensure_chunk_rows(*sample);
        // the slice renumbers rows: gather the matching x rows (src/scheduler.cpp:214-220)
        ns = rows.size();
        xs.alloc(std::max<std::uint64_t>(ns * f, 1));
        gather_dense_rows(x, f, rows, xs.get(), s);
        obuf.alloc(std::max<std::uint64_t>(sample->nnz, 1));
        freeze_mix_flag(*sample, y, y_rows * f, s, true);
        return ns;
    };
    h.run_baseline = [&] { launch_sddmm_baseline(*sample, xs.get(), y, std::uint32_t(f), obuf.get(), s); };
    h.run_candidate = [&](const as_variant& v) {
        dispatch_sddmm(v, *sample, xs.get(), ns, y, y_rows, f, obuf.get(), s, false);
    };
    return decide_common(ctx, cfg, dp, [&] { return graph_sig(p); }, f, AS_OP_SDDMM, h);
}

as_decision decide_host(const Context& ctx, const as_probe_config& cfg, std::uint64_t sig,
                        const as_features& gf, std::uint64_t f, int op, std::uint64_t sample_rows) {
    if (!ctx.device) throw InvalidArgument("decide_host: a device profile is required");
    if (!ctx.timer) throw InvalidArgument("decide_host: a timer is required");
    ProbeHooks h;
    h.features = [&] { return gf; };
    h.prepare = [&] { return sample_rows; };
    h.run_baseline = [] {};
    h.run_candidate = [](const as_variant&) {};
    return decide_common(ctx, cfg, *ctx.device, [&] { return sig; }, f, op, h);
}

void spmm_auto(const Context& ctx, const as_probe_config& cfg, Graph& a, const float* vals,
               const float* b, std::uint64_t b_rows, std::uint64_t f, float* c, as_decision* out) {
    const as_decision d = decide_spmm(ctx, cfg, a, vals, b, b_rows, f);
    cudaStream_t s = ctx.stream ? ctx.stream : a.stream;
    if (d.has_choice) dispatch_spmm(d.choice, a, vals, b, b_rows, f, c, s, false);
    else spmm_baseline(a, graph_values(a, vals), b, b_rows, f, c, s);
    if (out) *out = d;
}

void sddmm_auto(const Context& ctx, const as_probe_config& cfg, Graph& p, const float* x,
                std::uint64_t x_rows, const float* y, std::uint64_t y_rows, std::uint64_t f,
                float* out, as_decision* dout) {
    const as_decision d = decide_sddmm(ctx, cfg, p, x, x_rows, y, y_rows, f);
    cudaStream_t s = ctx.stream ? ctx.stream : p.stream;
    if (d.has_choice) dispatch_sddmm(d.choice, p, x, x_rows, y, y_rows, f, out, s, false);
    else sddmm_baseline(p, x, x_rows, y, y_rows, f, out, s);
    if (dout) *dout = d;
}

std::uint64_t probe_launch_count() { return g_probe_launches.load(); }
void reset_probe_launch_count() { g_probe_launches.store(0); }

// ---- attention (src/attention.cpp:9-46) --------------------------------------

void attention_forward(const Context& ctx, const as_probe_config& cfg, Graph& pattern,
                       const float* q, std::uint64_t q_rows, const float* k, std::uint64_t k_rows,
                       const float* v, std::uint64_t v_rows, std::uint64_t f, std::uint64_t fv,
                       float* out, bool fused, as_decision* sd_out, as_decision* pd_out, float* p_out) {
    if (q_rows != pattern.n_rows || k_rows != pattern.n_cols || v_rows != pattern.n_cols)
        throw InvalidArgument("attention: operand row counts incompatible with pattern");
    DeviceGuard dg(pattern.device);
    cudaStream_t s = ctx.stream ? ctx.stream : pattern.stream;

    const as_decision sd = decide_sddmm(ctx, cfg, pattern, q, q_rows, k, k_rows, f);
    pattern.att_buf.ensure(std::max<std::uint64_t>(2 * pattern.nnz, 2));
    float* scores = pattern.att_buf.get();
    float* p = p_out ? p_out : scores + pattern.nnz;
    bool p_ready = false;
    auto make_p = [&] {
        if (p_ready) return;
        if (sd.has_choice) dispatch_sddmm(sd.choice, pattern, q, q_rows, k, k_rows, f, scores, s, false);
        else sddmm_baseline(pattern, q, q_rows, k, k_rows, f, scores, s);
        row_softmax(pattern, scores, p, s);
        p_ready = true;
    };
    if (!fused || p_out) make_p();

    // decide_spmm on p = softmax(scores): same structure (same graph_sig), the
    // probe sample slices p's values -- materialized only if a probe runs
    as_decision pd;
    {
        if (pattern.n_cols != v_rows) throw InvalidArgument("decide_spmm: dimension mismatch");
        std::unique_ptr<Graph> sample;
        DevBuf<float> cbuf;
        ProbeHooks h;
        h.stream = s;
        h.features = [&] { return graph_features(pattern, kDefaultHubThreshold); };
        h.prepare = [&]() -> std::uint64_t {
            make_p();
            const auto rows = sample_row_indices(pattern, cfg.frac,
                                                 probe_min_rows(pattern, cfg, profile_for(ctx, pattern.device)));
            sample = slice_rows(pattern, rows, p);
            ensure_order(*sample);
            cbuf.alloc(std::max<std::uint64_t>(rows.size() * fv, 1));
            return rows.size();
        };
        h.run_baseline = [&] {
            launch_spmm_baseline(*sample, graph_values(*sample, nullptr), v, std::uint32_t(fv),
                                 cbuf.get(), s);
        };
        h.run_candidate = [&](const as_variant& var) {
            dispatch_spmm(var, *sample, nullptr, v, v_rows, fv, cbuf.get(), s, false);
        };
        pd = decide_common(ctx, cfg, profile_for(ctx, pattern.device),
                           [&] { return graph_sig(pattern); }, fv, AS_OP_SPMM, h);
    }

    bool done = false;
    if (fused && !p_ready && pd.has_choice) {
        // SDDMM -> per-row (max, sum) and per-entry ex -> SpMM that turns each
        // ex into its probability as it loads it: p never touches memory, and
        // the bits are those of the staged pipeline (same softmax.cuh arithmetic)
        const as_variant pv = apply_env_overrides(pd.choice);
        check_variant(pv);
        const void* vv[1] = {v};
        if (pv.mapping != AS_MAP_BASELINE && fv % 4 == 0 && vec4_eligible(fv, vv, 1)) {
            if (sd.has_choice) dispatch_sddmm(sd.choice, pattern, q, q_rows, k, k_rows, f, scores, s, false);
            else sddmm_baseline(pattern, q, q_rows, k, k_rows, f, scores, s);
            pattern.att_max.ensure(std::max<std::uint64_t>(pattern.n_rows, 1));
            pattern.att_sum.ensure(std::max<std::uint64_t>(pattern.n_rows, 1));
            float* ex = scores + pattern.nnz;  // p's slot, unused on this path
            launch_row_softmax_stats(pattern, scores, ex, pattern.att_max.get(), pattern.att_sum.get(), s);
            run_spmm_variant(pv, pattern, ex, v, fv, out, s, true, pattern.att_max.get(), pattern.att_sum.get());
            done = true;
        }
    }
    if (!done) {
        make_p();
        if (pd.has_choice) dispatch_spmm(pd.choice, pattern, p, v, v_rows, fv, out, s, false);
        else spmm_baseline(pattern, p, v, v_rows, fv, out, s);
    }
    if (sd_out) *sd_out = sd;
    if (pd_out) *pd_out = pd;
}

// CSR attention on 16-bit q, k, v words (wt: 1 bf16, 2 f16)
// with given variants (the torch training path fixes them): scores =
// SDDMM(q, k) -> row softmax -> SpMM over v.  fused: SDDMM -> per-row (max,
// sum) -> the SpMM turning each score into its probability as it loads it
// (softmax.cuh, as the f32 fused path); p_out, when given, receives p (the
// staged form).  Either way the bits are those of the f32 staged pipeline on
// float(q), float(k), float(v) with the same variants.
void attention_half(Graph& pattern, const as_variant* sv, const as_variant* pv, const std::uint16_t* q,
                    std::uint64_t q_rows, const std::uint16_t* k, std::uint64_t k_rows, const std::uint16_t* v,
                    std::uint64_t v_rows, std::uint64_t f, std::uint64_t fv, float* out, float* p_out, bool fused,
                    int wt, cudaStream_t s) {
    if (q_rows != pattern.n_rows || k_rows != pattern.n_cols || v_rows != pattern.n_cols)
        throw InvalidArgument("attention: operand row counts incompatible with pattern");
    if (sv && sv->op != AS_OP_SDDMM) throw InvalidArgument("attention: sddmm variant expected");
    if (pv && pv->op != AS_OP_SPMM) throw InvalidArgument("attention: spmm variant expected");
    DeviceGuard dg(pattern.device);
    pattern.att_buf.ensure(std::max<std::uint64_t>(2 * pattern.nnz, 2));
    float* scores = pattern.att_buf.get();
    dispatch_sddmm_half(sv, pattern, q, q_rows, k, k_rows, f, scores, s, false, wt);
    as_variant pvar = pv ? apply_env_overrides(*pv) : default_variant();
    if (!pv) pvar.mapping = AS_MAP_BASELINE;
    check_variant(pvar);
    const bool vec_ok = fv % 4 == 0 && (reinterpret_cast<std::uintptr_t>(v) & 7) == 0;
    if (fused && !p_out && pvar.mapping != AS_MAP_BASELINE && vec_ok && pattern.nnz) {
        pattern.att_max.ensure(std::max<std::uint64_t>(pattern.n_rows, 1));
        pattern.att_sum.ensure(std::max<std::uint64_t>(pattern.n_rows, 1));
        float* ex = scores + pattern.nnz;  // p's slot, unused on this path
        launch_row_softmax_stats(pattern, scores, ex, pattern.att_max.get(), pattern.att_sum.get(), s);
        const std::uint32_t wpb = std::uint32_t(std::min<std::uint64_t>(pvar.rows_per_chunk, 16));
        if (pvar.mapping == AS_MAP_ROWPARALLEL) {
            ensure_order(pattern);
            launch_spmm_rows(pattern, ex, 0, pattern.n_rows, v, std::uint32_t(fv), out, pvar.f_tile, true, wpb, s,
                             nullptr, pattern.att_max.get(), pattern.att_sum.get(), wt);
        } else {
            launch_spmm_hubsplit(pattern, ex, v, std::uint32_t(fv), out, pvar.f_tile, true, wpb,
                                 pvar.hub_threshold, s, nullptr, pattern.att_max.get(), pattern.att_sum.get(), wt);
        }
        return;
    }
    float* p = p_out ? p_out : scores + pattern.nnz;
    if (pattern.nnz) row_softmax(pattern, scores, p, s);
    dispatch_spmm_half(pv, pattern, p, v, v_rows, fv, out, s, false, wt);
}

} // namespace asb
