// config.hpp -- host-side ngram_config restatement used by the C-ABI (shape algebra,
// validation and JSON of config.hpp:25-77 / config.cpp:23-183).  Host logic only.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ngram_b200.h"

namespace ngh {

// Error carrying the C-ABI status it maps to (the reference exception type).
struct Error : std::runtime_error {
    int status;
    Error(int st, const std::string& msg) : std::runtime_error(msg), status(st) {}
};

struct Config {
    int max_order = 4;        // N
    int sub_tables = 2;       // K
    uint32_t base_vocab = 0;  // V0
    int dim = 0;              // D
    int variant = 1;          // 0 averaged_v1, 1 subtable_v2
    int amp = 0;              // 0 none, 1 scale_sqrt_d, 2 layer_norm
    std::vector<uint64_t> sub_vocab;  // V_{n,k} in branch order b = (n-2)K + (k-1)

    int branch_count() const { return max_order < 2 ? 0 : (max_order - 1) * sub_tables; }  // config.hpp:35-37
    int branch_dim() const {                                                                // config.hpp:40-45
        return (variant == 0 || branch_count() == 0) ? dim : dim / branch_count();
    }
    int branch_index(int n, int k) const { return (n - 2) * sub_tables + (k - 1); }  // config.hpp:48-50
    int merge_denominator() const { return variant == 0 ? max_order : branch_count() + 1; }  // config.hpp:53-56
};

// ngram_config_from_json + validate (config.cpp:124-139, 32-77).  Throws Error.
Config parse_config(const std::string& json_text);
void validate(const Config& c);
std::string to_json(const Config& c);                                                 // config.cpp:109-122
Config default_config(uint32_t base_vocab, int dim, int max_order, int sub_tables);  // config.cpp:163-183

}  // namespace ngh
