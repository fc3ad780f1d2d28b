// internal.hpp -- shared internals of libautosage_b200 (host C++ + CUDA).
//
// Error model: internal code throws typed exceptions; the C-ABI layer
// (capi.cpp) maps them onto as_status codes and the thread-local message.
#pragma once

#include "autosage_b200.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <optional>
#include <stdexcept>
#include <string>

namespace asb {

// Mirrors of the reference's exception types (by role, not by name).
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct CacheError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ReplayMissError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct OutOfMemory : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct LogicError : std::logic_error {
    using std::logic_error::logic_error;
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define ASB_CUDA(call)                                                      \
    do {                                                                    \
        cudaError_t asb_e_ = (call);                                        \
        if (asb_e_ != cudaSuccess) ::asb::throw_cuda(asb_e_, #call, __FILE__, __LINE__); \
    } while (0)

// Kernel launch bookkeeping: every launch of one of our kernels bumps this.
extern std::atomic<std::uint64_t> g_kernel_launches;
inline void count_launch(std::uint64_t n = 1) { g_kernel_launches += n; }
void check_launch(const char* name);

// ---- env (include/autosage/env.hpp:9-40 semantics) ----------------------
namespace env {
std::optional<std::string> get_string(const char* name);
std::optional<long long> get_int(const char* name);
std::optional<double> get_double(const char* name);
bool get_flag(const char* name, bool fallback = false);
} // namespace env

// ---- variants ------------------------------------------------------------
constexpr std::uint64_t kDefaultHubThreshold = 256;  // include/autosage/csr.hpp:18
constexpr std::uint64_t kHubNnzChunk = 2048;         // src/kernels.cpp:21
extern const char* const kArtifactVersion;           // include/autosage/version.hpp:6

as_variant default_variant();
std::string variant_to_string(const as_variant& v);
as_variant variant_from_string(const std::string& s);
bool variant_equal(const as_variant& a, const as_variant& b);
void check_variant(const as_variant& v);                 // src/kernels.cpp:25-31
as_variant apply_env_overrides(as_variant v);            // src/kernels.cpp:465-476
std::uint64_t effective_tile(std::uint64_t ft, std::uint64_t f);  // src/kernels.cpp:45-47
bool vec4_eligible(std::uint64_t f, const void* const* bases, int n);
const char* op_name(int op);
const char* mapping_name(int m);

// ---- misc host helpers -----------------------------------------------------
std::uint64_t fnv1a(std::uint64_t h, const void* data, std::size_t n);
constexpr std::uint64_t kFnvOffset = 14695981039346656037ULL;
std::string toolchain_tag();
std::uint64_t unix_now();

} // namespace asb
