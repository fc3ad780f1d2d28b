// policy.cpp -- host-side policy of the B200 AutoSAGE library: env parsing,
// variant strings, the vec4 gate, CSR validation, the roofline cost model
// and shortlist, the time_kernel probe policy.  Behaviour follows the
// reference contracts cited per function (paths under /root/reference/proj).
#include "internal.hpp"
#include "policy.hpp"

#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <tuple>
#include <vector>

namespace asb {

std::atomic<std::uint64_t> g_kernel_launches{0};
const char* const kArtifactVersion = "autosage-b200-0.1.0";

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    if (e == cudaErrorMemoryAllocation) throw OutOfMemory(buf);
    throw CudaError(buf);
}

void check_launch(const char* name) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw_cuda(e, name, __FILE__, __LINE__);
    count_launch();
}

// ---- env: include/autosage/env.hpp:9-40 -----------------------------------
namespace env {
std::optional<std::string> get_string(const char* name) {
    const char* v = std::getenv(name);
    if (v == nullptr || *v == '\0') return std::nullopt;
    return std::string(v);
}
std::optional<long long> get_int(const char* name) {
    auto s = get_string(name);
    if (!s) return std::nullopt;
    char* end = nullptr;
    long long v = std::strtoll(s->c_str(), &end, 10);
    if (end == s->c_str() || *end != '\0') return std::nullopt;
    return v;
}
std::optional<double> get_double(const char* name) {
    auto s = get_string(name);
    if (!s) return std::nullopt;
    char* end = nullptr;
    double v = std::strtod(s->c_str(), &end);
    if (end == s->c_str() || *end != '\0') return std::nullopt;
    return v;
}
bool get_flag(const char* name, bool fallback) {
    auto s = get_string(name);
    if (!s) return fallback;
    std::string v = *s;
    for (auto& c : v) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return !(v == "0" || v == "false" || v == "off");
}
} // namespace env

// ---- variants: src/kernels.cpp:146-208 -----------------------------------
as_variant default_variant() {
    as_variant v{};
    v.op = AS_OP_SPMM;
    v.mapping = AS_MAP_ROWPARALLEL;
    v.f_tile = 64;
    v.rows_per_chunk = 4;
    v.vectorized = 0;
    v.hub_threshold = kDefaultHubThreshold;
    return v;
}

const char* op_name(int op) { return op == AS_OP_SPMM ? "spmm" : "sddmm"; }

const char* mapping_name(int m) {
    switch (m) {
        case AS_MAP_BASELINE: return "baseline";
        case AS_MAP_ROWPARALLEL: return "rowparallel";
        case AS_MAP_HUBSPLIT: return "hubsplit";
    }
    return "?";
}

std::string variant_to_string(const as_variant& v) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "%s:%s:ft=%llu:rpc=%llu:vec=%d:hubt=%llu", op_name(v.op),
                  mapping_name(v.mapping), (unsigned long long)v.f_tile,
                  (unsigned long long)v.rows_per_chunk, v.vectorized ? 1 : 0,
                  (unsigned long long)v.hub_threshold);
    return buf;
}

namespace {
std::uint64_t parse_field(const std::string& p, const char* prefix) {
    const std::size_t n = std::strlen(prefix);
    if (p.compare(0, n, prefix) != 0)
        throw InvalidArgument("variant_from_string: expected " + std::string(prefix));
    const std::string digits = p.substr(n);
    // std::stoull semantics: leading whitespace/sign accepted, junk after the
    // number ignored, no digits -> invalid_argument
    try {
        return static_cast<std::uint64_t>(std::stoull(digits));
    } catch (const std::invalid_argument&) {
        throw InvalidArgument("stoull");
    } catch (const std::out_of_range&) {
        throw InvalidArgument("stoull");
    }
}
} // namespace

as_variant variant_from_string(const std::string& s) {
    std::vector<std::string> parts;
    std::size_t start = 0;
    while (true) {
        auto pos = s.find(':', start);
        parts.push_back(s.substr(start, pos - start));
        if (pos == std::string::npos) break;
        start = pos + 1;
    }
    if (parts.size() != 6) throw InvalidArgument("variant_from_string: bad format: " + s);
    as_variant v = default_variant();
    if (parts[0] == "spmm") v.op = AS_OP_SPMM;
    else if (parts[0] == "sddmm") v.op = AS_OP_SDDMM;
    else throw InvalidArgument("variant_from_string: bad op: " + parts[0]);
    if (parts[1] == "baseline") v.mapping = AS_MAP_BASELINE;
    else if (parts[1] == "rowparallel") v.mapping = AS_MAP_ROWPARALLEL;
    else if (parts[1] == "hubsplit") v.mapping = AS_MAP_HUBSPLIT;
    else throw InvalidArgument("variant_from_string: bad mapping: " + parts[1]);
    v.f_tile = parse_field(parts[2], "ft=");
    v.rows_per_chunk = parse_field(parts[3], "rpc=");
    v.vectorized = parse_field(parts[4], "vec=") != 0;
    v.hub_threshold = parse_field(parts[5], "hubt=");
    return v;
}

bool variant_equal(const as_variant& a, const as_variant& b) {
    return a.op == b.op && a.mapping == b.mapping && a.f_tile == b.f_tile &&
           a.rows_per_chunk == b.rows_per_chunk && (a.vectorized != 0) == (b.vectorized != 0) &&
           a.hub_threshold == b.hub_threshold;
}

void check_variant(const as_variant& v) {
    if (v.f_tile == 0) throw InvalidArgument("variant: f_tile must be > 0");
    if (v.rows_per_chunk == 0) throw InvalidArgument("variant: rows_per_chunk must be > 0");
    if (v.mapping == AS_MAP_HUBSPLIT && v.hub_threshold == 0)
        throw InvalidArgument("variant: hub_threshold must be > 0 for hubsplit");
    if (v.mapping < AS_MAP_BASELINE || v.mapping > AS_MAP_HUBSPLIT)
        throw InvalidArgument("variant: bad mapping");
    if (v.op != AS_OP_SPMM && v.op != AS_OP_SDDMM) throw InvalidArgument("variant: bad op");
}

as_variant apply_env_overrides(as_variant v) {
    if (auto ft = env::get_int("AUTOSAGE_FTILE"); ft && *ft > 0) v.f_tile = std::uint64_t(*ft);
    if (auto w = env::get_int("AUTOSAGE_WPB"); w && *w > 0) v.rows_per_chunk = std::uint64_t(*w);
    if (auto h = env::get_int("AUTOSAGE_HUB_T"); h && *h > 0) v.hub_threshold = std::uint64_t(*h);
    return v;
}

std::uint64_t effective_tile(std::uint64_t ft, std::uint64_t f) {
    return std::max<std::uint64_t>(1, std::min(ft, std::max<std::uint64_t>(f, 1)));
}

bool vec4_eligible(std::uint64_t f, const void* const* bases, int n) {
    if (f == 0 || f % 4 != 0) return false;
    for (int i = 0; i < n; ++i) {
        if (reinterpret_cast<std::uintptr_t>(bases[i]) % 16 != 0) return false;
    }
    return true;
}

// ---- FNV-1a, src/cache.cpp:18-29 ------------------------------------------
std::uint64_t fnv1a(std::uint64_t h, const void* data, std::size_t n) {
    const auto* p = static_cast<const unsigned char*>(data);
    // 8-way manual unroll; the recurrence is inherently serial
    std::size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        h = (h ^ p[i + 0]) * 1099511628211ULL;
        h = (h ^ p[i + 1]) * 1099511628211ULL;
        h = (h ^ p[i + 2]) * 1099511628211ULL;
        h = (h ^ p[i + 3]) * 1099511628211ULL;
        h = (h ^ p[i + 4]) * 1099511628211ULL;
        h = (h ^ p[i + 5]) * 1099511628211ULL;
        h = (h ^ p[i + 6]) * 1099511628211ULL;
        h = (h ^ p[i + 7]) * 1099511628211ULL;
    }
    for (; i < n; ++i) h = (h ^ p[i]) * 1099511628211ULL;
    return h;
}

std::uint64_t graph_sig_host(const std::uint64_t* rowptr, const std::uint32_t* colind,
                             std::uint64_t n_rows, std::uint64_t n_cols, std::uint64_t nnz) {
    std::uint64_t h = kFnvOffset;
    h = fnv1a(h, &n_rows, 8);
    h = fnv1a(h, &n_cols, 8);
    h = fnv1a(h, &nnz, 8);
    h = fnv1a(h, rowptr, (n_rows + 1) * 8);
    h = fnv1a(h, colind, nnz * 4);
    return h;
}

std::string toolchain_tag() {
    char buf[64];
#if defined(__clang__)
    std::snprintf(buf, sizeof buf, "clang-%d.%d.%d", __clang_major__, __clang_minor__,
                  __clang_patchlevel__);
#elif defined(__GNUC__)
    std::snprintf(buf, sizeof buf, "gcc-%d.%d.%d", __GNUC__, __GNUC_MINOR__, __GNUC_PATCHLEVEL__);
#else
    std::snprintf(buf, sizeof buf, "unknown");
#endif
    return buf;
}

std::uint64_t unix_now() {
    return static_cast<std::uint64_t>(std::chrono::duration_cast<std::chrono::seconds>(
                                          std::chrono::system_clock::now().time_since_epoch())
                                          .count());
}

// ---- validate, src/csr.cpp:62-93 ------------------------------------------
std::optional<Violation> validate_csr(const std::uint64_t* rowptr, std::uint64_t rowptr_len,
                                      const std::uint32_t* colind, std::uint64_t nnz,
                                      std::uint64_t val_len, std::uint64_t n_rows,
                                      std::uint64_t n_cols) {
    if (rowptr_len != n_rows + 1) return Violation{"rowptr length", rowptr_len};
    if (rowptr[0] != 0) return Violation{"rowptr[0] nonzero", 0};
    for (std::uint64_t i = 1; i <= n_rows; ++i)
        if (rowptr[i] < rowptr[i - 1]) return Violation{"rowptr non-decreasing", i};
    if (rowptr[n_rows] != nnz) return Violation{"rowptr/nnz mismatch", n_rows};
    for (std::uint64_t e = 0; e < nnz; ++e)
        if (colind[e] >= n_cols) return Violation{"colind out of range", e};
    for (std::uint64_t i = 0; i < n_rows; ++i)
        for (std::uint64_t e = rowptr[i] + 1; e < rowptr[i + 1]; ++e)
            if (colind[e] <= colind[e - 1]) return Violation{"colind not strictly increasing", e};
    if (val_len != 0 && val_len != nnz) return Violation{"val length mismatch", val_len};
    return std::nullopt;
}

// ---- cost model, src/cost.cpp:9-79 ----------------------------------------
double estimate_cost(const as_variant& v, const as_features& gf, std::uint64_t f,
                     const as_device_profile& dp) {
    if (dp.bw_eff <= 0.0 || dp.flops_eff <= 0.0)
        throw InvalidArgument("estimate_cost: device profile not calibrated");
    if (gf.nnz == 0) return 0.0;
    const double nnz = double(gf.nnz), n = double(gf.n_rows), fd = double(f);
    double bytes;
    if (v.op == AS_OP_SPMM)
        bytes = 8.0 * nnz + 4.0 * nnz * fd + 4.0 * n * fd + 8.0 * (n + 1.0);
    else
        bytes = 8.0 * nnz + 4.0 * nnz * fd * 2.0 + 4.0 * nnz;
    const double flops = 2.0 * nnz * fd;
    if (dp.model == AS_MODEL_B200) {
        // B200 refinement (not in the reference): the sm_100a kernels re-read
        // colind/val once per f_tile pass of SpMM; SDDMM runs the same
        // balanced nnz-chunk kernel for both mappings (no imbalance term).
        if (v.op == AS_OP_SPMM) {
            const double ft = double(effective_tile(v.f_tile, f));
            const double passes = std::ceil(fd / std::max(ft, 1.0));
            bytes += 8.0 * nnz * (passes - 1.0);
        } else {
            return std::max(bytes / dp.bw_eff, flops / dp.flops_eff) * 1e3;
        }
    }
    const double seconds = std::max(bytes / dp.bw_eff, flops / dp.flops_eff);
    double penalty = 1.0;
    if (v.mapping != AS_MAP_HUBSPLIT) {
        const double mean = gf.mean_degree;
        double imbalance = 0.0;
        if (mean > 0.0)
            imbalance = (double(gf.deg_max) / mean - 1.0) /
                        double(std::max<std::uint64_t>(dp.cores, 1));
        imbalance = std::clamp(imbalance, 0.0, 4.0);
        penalty = 1.0 + imbalance;
    }
    return seconds * 1e3 * penalty;
}

std::vector<as_variant> shortlist(const as_features& gf, std::uint64_t f, int op,
                                  const as_device_profile& dp) {
    static constexpr std::uint64_t kTiles[] = {32, 64, 128};
    static constexpr std::uint64_t kRpc[] = {1, 4, 16};
    const bool vec_ok = f > 0 && f % 4 == 0;
    std::vector<as_variant> grid;
    for (int mapping : {AS_MAP_ROWPARALLEL, AS_MAP_HUBSPLIT})
        for (auto ft : kTiles)
            for (auto rpc : kRpc)
                for (int vec = vec_ok ? 1 : 0; vec >= 0; --vec) {
                    as_variant v = default_variant();
                    v.op = op;
                    v.mapping = mapping;
                    v.f_tile = ft;
                    v.rows_per_chunk = rpc;
                    v.vectorized = vec;
                    v.hub_threshold = kDefaultHubThreshold;
                    grid.push_back(v);
                }
    auto rank = [&](const as_variant& v) {
        return std::make_tuple(estimate_cost(v, gf, f, dp), v.mapping == AS_MAP_ROWPARALLEL ? 0 : 1,
                               v.f_tile, v.vectorized ? 0 : 1, v.rows_per_chunk);
    };
    std::stable_sort(grid.begin(), grid.end(),
                     [&](const as_variant& a, const as_variant& b) { return rank(a) < rank(b); });
    return grid;
}

// B200: several reference variants compile to the same sm_100a launch (SpMM:
// vec only selects the reported path and rows_per_chunk no longer sizes
// anything; SDDMM: both mappings run the nnz-chunk kernel, and f_tile only
// matters to the vec order).  Keep the first of each class in rank order so
// the top_k probes compare distinct kernels.
std::vector<as_variant> distinct_gpu_configs(const std::vector<as_variant>& ranked, std::uint64_t f) {
    std::vector<as_variant> out;
    std::vector<std::tuple<int, int, std::uint64_t, int, std::uint64_t>> seen;
    for (const auto& v : ranked) {
        const std::uint64_t ft = effective_tile(v.f_tile, f);
        std::tuple<int, int, std::uint64_t, int, std::uint64_t> key;
        if (v.op == AS_OP_SPMM)
            key = {v.op, v.mapping, ft, 0, v.mapping == AS_MAP_HUBSPLIT ? v.hub_threshold : 0};
        else
            key = {v.op, 0, v.vectorized ? ft : 0, v.vectorized, 0};
        if (std::find(seen.begin(), seen.end(), key) != seen.end()) continue;
        seen.push_back(key);
        out.push_back(v);
    }
    return out;
}

// B200, SpMM at F > 64: the lane-group kernels walk feature tiles
// tile-major, so with 64-wide tiles only a 64-column slice of B is live at a
// time and it stays in the L2 where the whole B does not.  A probe sample
// never fills the L2, so it cannot see this and ranks wider tiles first (one
// colind pass fewer).  Where B is over the L2 budget and a 64-column slice is
// within it, every SpMM candidate therefore takes f_tile 64 (all f_tiles give
// the same bits).  Reddit-shape: F=128 3.49 ms at ft 64 vs 3.93 at ft 128,
// F=192 6.44 vs 8.21, F=256 8.60 vs 8.65 (profiles/r02at_ftile.md).
void l2_tile_rule(std::vector<as_variant>& cands, std::uint64_t f, std::uint64_t n_cols) {
    constexpr std::uint64_t kL2Budget = std::uint64_t(96) << 20;  // l2hint.cuh kKeepMaxBytes
    if (f <= 64 || n_cols * f * 4 <= kL2Budget || n_cols * 64 * 4 > kL2Budget) return;
    for (auto& v : cands)
        if (v.op == AS_OP_SPMM && v.mapping != AS_MAP_BASELINE) v.f_tile = 64;
}

// ---- time_kernel, src/timing.cpp:22-61 -----------------------------------
namespace {
thread_local std::function<void()> t_warmup_sync;
}
void set_warmup_sync(std::function<void()> sync) { t_warmup_sync = std::move(sync); }
void sync_current_stream_for_timing() {
    if (t_warmup_sync) t_warmup_sync();
}

as_timed_stats time_kernel(const std::string& label, const std::function<void()>& run, int iters,
                           double cap_ms, const TimeOnce& time_once) {
    if (iters < 1) throw InvalidArgument("time_kernel: iters must be >= 1");
    as_timed_stats st{};
    const auto wall0 = std::chrono::steady_clock::now();
    {
        // untimed warm-up; its wall time still counts toward max_run_ms
        const auto w0 = std::chrono::steady_clock::now();
        run();
        sync_current_stream_for_timing();
        st.max_run_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
        st.launches = 1;
    }
    std::vector<double> times;
    times.reserve(std::size_t(iters));
    double total = 0.0;
    for (int k = 0; k < iters; ++k) {
        const double t = time_once(label, run);
        ++st.launches;
        times.push_back(t);
        total += t;
        st.max_run_ms = std::max(st.max_run_ms, t);
        if (total > cap_ms && k + 1 < iters) {
            st.capped = 1;
            break;
        }
    }
    st.completed = int(times.size());
    std::sort(times.begin(), times.end());
    st.median_ms = times[(times.size() - 1) / 2];
    st.wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
    return st;
}

// ---- probe config / replay policy -----------------------------------------
as_probe_config probe_config_default() {
    as_probe_config c{};
    c.frac = 0.02;
    c.min_rows = 512;
    c.iters = 5;
    c.cap_ms = 1.0;
    c.top_k = 3;
    c.alpha = 0.95;
    return c;
}

as_probe_config probe_config_from_env() {  // src/scheduler.cpp:171-179
    as_probe_config c = probe_config_default();
    if (auto v = env::get_double("AUTOSAGE_PROBE_FRAC")) c.frac = *v;
    if (auto v = env::get_int("AUTOSAGE_PROBE_ITERS")) c.iters = int(*v);
    if (auto v = env::get_double("AUTOSAGE_PROBE_CAP_MS")) c.cap_ms = *v;
    if (auto v = env::get_int("AUTOSAGE_PROBE_TOPK")) c.top_k = int(*v);
    if (auto v = env::get_double("AUTOSAGE_GUARDRAIL")) c.alpha = *v;
    return c;
}

as_replay_policy replay_policy_from_env() {  // src/cache.cpp:223-228
    as_replay_policy p{};
    p.replay_only = env::get_flag("AUTOSAGE_REPLAY_ONLY");
    p.strict = env::get_flag("AUTOSAGE_REPLAY_STRICT");
    return p;
}

void check_probe_config(const as_probe_config& cfg) {  // src/scheduler.cpp:24-33
    if (!(cfg.frac > 0.0 && cfg.frac <= 1.0))
        throw InvalidArgument("probe config: frac must be in (0,1]");
    if (cfg.iters < 1) throw InvalidArgument("probe config: iters must be >= 1");
    if (!(cfg.alpha > 0.0 && cfg.alpha <= 1.0))
        throw InvalidArgument("probe config: alpha must be in (0,1]");
    if (cfg.top_k < 1) throw InvalidArgument("probe config: top_k must be >= 1");
}

// ---- partition (new) ----------------------------------------
void partition_rows(const std::uint64_t* rowptr, std::uint64_t n_rows, std::uint32_t g,
                    std::uint64_t* cuts) {
    if (g == 0) throw InvalidArgument("partition_rows: g must be >= 1");
    const std::uint64_t nnz = rowptr[n_rows];
    cuts[0] = 0;
    for (std::uint32_t k = 1; k < g; ++k) {
        const std::uint64_t target =
            static_cast<std::uint64_t>((static_cast<unsigned __int128>(k) * nnz) / g);
        const std::uint64_t lo =
            std::uint64_t(std::lower_bound(rowptr, rowptr + n_rows, target) - rowptr);
        cuts[k] = std::max(lo, cuts[k - 1]);
    }
    cuts[g] = n_rows;
}

} // namespace asb
