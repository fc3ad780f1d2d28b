// policy.hpp -- host policy declarations (see policy.cpp).
#pragma once

#include "internal.hpp"

#include <functional>
#include <string>
#include <vector>

namespace asb {

struct Violation {
    std::string invariant;
    std::uint64_t index = 0;
};

std::optional<Violation> validate_csr(const std::uint64_t* rowptr, std::uint64_t rowptr_len,
                                      const std::uint32_t* colind, std::uint64_t nnz,
                                      std::uint64_t val_len, std::uint64_t n_rows,
                                      std::uint64_t n_cols);

std::uint64_t graph_sig_host(const std::uint64_t* rowptr, const std::uint32_t* colind,
                             std::uint64_t n_rows, std::uint64_t n_cols, std::uint64_t nnz);

double estimate_cost(const as_variant& v, const as_features& gf, std::uint64_t f,
                     const as_device_profile& dp);
std::vector<as_variant> shortlist(const as_features& gf, std::uint64_t f, int op,
                                  const as_device_profile& dp);
// B200 model: drop variants that launch the same kernel as a better-ranked one.
std::vector<as_variant> distinct_gpu_configs(const std::vector<as_variant>& ranked, std::uint64_t f);
// SpMM candidates take f_tile 64 where B overflows the L2 but a 64-column
// slice fits (tile-major walk; policy.cpp)
void l2_tile_rule(std::vector<as_variant>& cands, std::uint64_t f, std::uint64_t n_cols);

// ProbeTimer::time_once_ms (include/autosage/timing.hpp:10-15)
using TimeOnce = std::function<double(const std::string&, const std::function<void()>&)>;
// Completes outstanding device work of `run` (used after the untimed
// warm-up so its wall time covers the launch); empty for host-only use.
void set_warmup_sync(std::function<void()> sync);
void sync_current_stream_for_timing();

as_timed_stats time_kernel(const std::string& label, const std::function<void()>& run, int iters,
                           double cap_ms, const TimeOnce& time_once);

as_probe_config probe_config_default();
as_probe_config probe_config_from_env();
as_replay_policy replay_policy_from_env();
void check_probe_config(const as_probe_config& cfg);

void partition_rows(const std::uint64_t* rowptr, std::uint64_t n_rows, std::uint32_t g,
                    std::uint64_t* cuts);

} // namespace asb
