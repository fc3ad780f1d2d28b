// cache.hpp -- persistent (device_sig, graph_sig, F, op) decision cache.
// Contract: include/autosage/cache.hpp:23-91 and src/cache.cpp:76-218.
#pragma once

#include "internal.hpp"

#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

namespace asb {

struct Key {
    std::string device_sig;
    std::uint64_t graph_sig = 0;
    std::uint64_t f = 0;
    int op = AS_OP_SPMM;
    bool operator<(const Key& o) const {
        return std::tie(device_sig, graph_sig, f, op) <
               std::tie(o.device_sig, o.graph_sig, o.f, o.op);
    }
    bool operator==(const Key& o) const {
        return device_sig == o.device_sig && graph_sig == o.graph_sig && f == o.f && op == o.op;
    }
    std::string to_string() const;  // src/cache.cpp:76-81
};

struct Record {
    Key key;
    std::string choice;  // "baseline" or a variant string
    double t_b = 0.0, t_star = 0.0, alpha = 0.0;
    std::uint64_t timestamp = 0;
    std::uint32_t schema_version = 1;
    std::string toolchain;
};

std::string record_to_line(const Record& rec);
Record record_from_line(const std::string& line);

class ScheduleCache {
public:
    std::optional<Record> get(const Key& key) const;
    void put(const Record& rec);
    std::size_t size() const;
    std::vector<Record> snapshot() const;
    void clear();
    void load(const std::string& path);
    void store(const std::string& path) const;

private:
    mutable std::mutex mu_;
    std::map<Key, Record> records_;
};

Key key_from_c(const as_key& k);
as_key key_to_c(const Key& k);
Record record_from_c(const as_record& r);
as_record record_to_c(const Record& r);

} // namespace asb
