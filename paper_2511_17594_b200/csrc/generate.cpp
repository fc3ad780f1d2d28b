// generate.cpp -- synthetic inputs and ASCR I/O.
//
// The reference's generators (src/generate.cpp:41-132) cover Erdos-Renyi
// and fixed hub shapes; the B200 configs need heavy-tailed (power-law /
// Zipf) degree graphs at Reddit/Products scale, so this is a new,
// multi-threaded generator.  Every row draws from its own counter-based
// stream (splitmix64 of seed and row), so the output is a pure function of
// the arguments and independent of the thread count.
//
// ASCR v1 container (src/io.cpp:48-93): "ASCR", u32 version=1, u64 n_rows,
// u64 n_cols, u64 nnz, u8 has_values, rowptr u64[n+1], colind u32[nnz],
// val f32[nnz] if has_values; load validates (src/csr.cpp:62-93).
#include "internal.hpp"
#include "policy.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <thread>
#include <vector>

namespace asb {

namespace {

inline std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

struct Rng {
    std::uint64_t s;
    explicit Rng(std::uint64_t seed) : s(seed) {}
    std::uint64_t next() {
        s += 0x9E3779B97F4A7C15ULL;
        std::uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double uniform01() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }  // [0,1)
    float uniformf() { return float(next() >> 40) * (1.0f / 16777216.0f); }          // [0,1)
    std::uint64_t below(std::uint64_t n) {  // unbiased enough for n << 2^64
        return std::uint64_t((static_cast<unsigned __int128>(next()) * n) >> 64);
    }
};

unsigned n_threads() {
    unsigned t = std::thread::hardware_concurrency();
    return std::max(1u, std::min(t, 64u));
}

template <class F>
void parallel_rows(std::uint64_t n, F&& fn) {
    const unsigned nt = n_threads();
    if (n < 4096 || nt == 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> th;
    const std::uint64_t chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const std::uint64_t r0 = t * chunk, r1 = std::min(n, r0 + chunk);
        if (r0 >= r1) break;
        th.emplace_back([&, r0, r1] { fn(r0, r1); });
    }
    for (auto& x : th) x.join();
}

// d distinct sorted values in [0, m) from rng
void distinct_sorted(std::uint64_t d, std::uint64_t m, Rng& rng, std::uint32_t* out,
                     std::vector<std::uint32_t>& scratch) {
    if (d == 0) return;
    if (d >= m) {
        for (std::uint64_t i = 0; i < m; ++i) out[i] = std::uint32_t(i);
        return;
    }
    if (d * 2 > m) {
        // complement: choose m-d values to drop
        std::vector<char> drop(m, 0);
        std::uint64_t k = m - d;
        while (k) {
            const std::uint64_t t = rng.below(m);
            if (!drop[t]) {
                drop[t] = 1;
                --k;
            }
        }
        std::uint64_t o = 0;
        for (std::uint64_t i = 0; i < m; ++i)
            if (!drop[i]) out[o++] = std::uint32_t(i);
        return;
    }
    scratch.clear();
    // draw exactly the deficit each round; duplicates shrink it geometrically
    while (scratch.size() < d) {
        const std::uint64_t need = d - scratch.size();
        for (std::uint64_t i = 0; i < need; ++i) scratch.push_back(std::uint32_t(rng.below(m)));
        std::sort(scratch.begin(), scratch.end());
        scratch.erase(std::unique(scratch.begin(), scratch.end()), scratch.end());
    }
    std::copy(scratch.begin(), scratch.end(), out);
}

} // namespace

void gen_powerlaw(std::uint64_t n_rows, std::uint64_t n_cols, std::uint64_t nnz_target, double alpha,
                  std::uint64_t d_min, std::uint64_t d_max, std::uint64_t seed, bool with_values,
                  std::vector<std::uint64_t>& rowptr, std::vector<std::uint32_t>& colind,
                  std::vector<float>& val) {
    if (alpha <= 1.0) throw InvalidArgument("gen_powerlaw: alpha must be > 1");
    if (n_cols == 0 && n_rows > 0 && nnz_target > 0)
        throw InvalidArgument("gen_powerlaw: n_cols must be > 0");
    const std::uint64_t cap = std::min(d_max, n_cols);
    std::vector<std::uint64_t> deg(n_rows);
    const double expo = -1.0 / (alpha - 1.0);
    parallel_rows(n_rows, [&](std::uint64_t r0, std::uint64_t r1) {
        for (std::uint64_t i = r0; i < r1; ++i) {
            Rng rng(splitmix64(seed * 0x632BE59BD9B4E019ULL + i));
            double u = rng.uniform01();
            if (u < 1e-300) u = 1e-300;
            double d = std::floor(double(d_min) * std::pow(u, expo));
            if (!(d < double(cap))) d = double(cap);
            deg[i] = std::uint64_t(d);
        }
    });
    if (nnz_target > 0) {
        std::uint64_t total = 0;
        for (auto d : deg) total += d;
        if (nnz_target > cap * n_rows) throw InvalidArgument("gen_powerlaw: nnz_target unreachable");
        if (total > 0) {
            const double s = double(nnz_target) / double(total);
            total = 0;
            for (auto& d : deg) {
                d = std::min<std::uint64_t>(cap, std::uint64_t(std::floor(double(d) * s)));
                total += d;
            }
        }
        // settle the remainder one entry at a time, cycling over rows
        std::uint64_t i = 0;
        while (total < nnz_target) {
            if (deg[i] < cap) {
                ++deg[i];
                ++total;
            }
            i = (i + 1) % n_rows;
        }
        while (total > nnz_target) {
            if (deg[i] > 0) {
                --deg[i];
                --total;
            }
            i = (i + 1) % n_rows;
        }
    }
    rowptr.assign(n_rows + 1, 0);
    for (std::uint64_t i = 0; i < n_rows; ++i) rowptr[i + 1] = rowptr[i] + deg[i];
    const std::uint64_t nnz = rowptr[n_rows];
    colind.resize(nnz);
    val.clear();
    if (with_values) val.resize(nnz);
    parallel_rows(n_rows, [&](std::uint64_t r0, std::uint64_t r1) {
        std::vector<std::uint32_t> scratch;
        for (std::uint64_t i = r0; i < r1; ++i) {
            Rng rng(splitmix64(seed * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL * (i + 1)));
            distinct_sorted(deg[i], n_cols, rng, colind.data() + rowptr[i], scratch);
            if (with_values)
                for (std::uint64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) val[e] = rng.uniformf();
        }
    });
}

void fill_uniform(float* out, std::uint64_t n, std::uint64_t seed) {
    parallel_rows(n, [&](std::uint64_t i0, std::uint64_t i1) {
        for (std::uint64_t i = i0; i < i1; ++i) {
            const std::uint64_t h = splitmix64(seed * 0xA0761D6478BD642FULL + i);
            out[i] = float(h >> 40) * (2.0f / 16777216.0f) - 1.0f;  // U[-1, 1)
        }
    });
}

// ---- ASCR v1 ------------------------------------------------------------------
void save_csr(const std::string& path, const std::uint64_t* rowptr, const std::uint32_t* colind,
              const float* val, std::uint64_t n_rows, std::uint64_t n_cols, std::uint64_t nnz) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw IoError("save_csr: cannot open " + path);
    const std::uint32_t version = 1;
    const std::uint8_t hv = val ? 1 : 0;
    f.write("ASCR", 4);
    f.write(reinterpret_cast<const char*>(&version), 4);
    f.write(reinterpret_cast<const char*>(&n_rows), 8);
    f.write(reinterpret_cast<const char*>(&n_cols), 8);
    f.write(reinterpret_cast<const char*>(&nnz), 8);
    f.write(reinterpret_cast<const char*>(&hv), 1);
    f.write(reinterpret_cast<const char*>(rowptr), std::streamsize((n_rows + 1) * 8));
    f.write(reinterpret_cast<const char*>(colind), std::streamsize(nnz * 4));
    if (val) f.write(reinterpret_cast<const char*>(val), std::streamsize(nnz * 4));
    if (!f) throw IoError("save_csr: write failed for " + path);
}

void load_csr(const std::string& path, std::vector<std::uint64_t>& rowptr,
              std::vector<std::uint32_t>& colind, std::vector<float>& val, std::uint64_t& n_rows,
              std::uint64_t& n_cols) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("load_csr: cannot open " + path);
    char magic[4];
    f.read(magic, 4);
    if (!f || std::memcmp(magic, "ASCR", 4) != 0) throw IoError("load_csr: bad magic in " + path);
    auto rd = [&](void* p, std::size_t n, const char* field) {
        f.read(static_cast<char*>(p), std::streamsize(n));
        if (!f) throw IoError(std::string("load_csr: truncated ") + field);
    };
    std::uint32_t version = 0;
    rd(&version, 4, "version");
    if (version != 1) throw IoError("load_csr: unsupported version " + std::to_string(version));
    std::uint64_t nnz = 0;
    std::uint8_t hv = 0;
    rd(&n_rows, 8, "n_rows");
    rd(&n_cols, 8, "n_cols");
    rd(&nnz, 8, "nnz");
    rd(&hv, 1, "has_values");
    if (hv > 1) throw IoError("load_csr: bad has_values flag");
    rowptr.resize(n_rows + 1);
    rd(rowptr.data(), (n_rows + 1) * 8, "rowptr");
    colind.resize(nnz);
    rd(colind.data(), nnz * 4, "colind");
    val.clear();
    if (hv) {
        val.resize(nnz);
        rd(val.data(), nnz * 4, "val");
    }
    if (auto v = validate_csr(rowptr.data(), rowptr.size(), colind.data(), nnz, val.size(), n_rows,
                              n_cols))
        throw IoError("load_csr: " + v->invariant + " at index " + std::to_string(v->index));
}

} // namespace asb
