// config.cpp -- see config.hpp.  Validation messages and order follow config.cpp:32-77.
#include "config.hpp"

#include <map>
#include <utility>

#include <json.hpp>

namespace ngh {

namespace {

uint64_t half_multiple_size(uint64_t v0, uint64_t multiple) { return ((2 * multiple + 1) * v0 + 1) / 2; }

[[noreturn]] void invalid(const std::string& m) { throw Error(NGRAM_EINVAL, "ngram_config: " + m); }

}  // namespace

void validate(const Config& c) {
    if (c.max_order < 1) invalid("max_order must be >= 1");
    if (c.sub_tables < 1) invalid("sub_tables must be >= 1");
    if (c.base_vocab < 2) invalid("base_vocab must be >= 2");
    if (c.dim < 1) invalid("dim must be >= 1");
    if (c.variant == 0 && c.sub_tables != 1)
        invalid("the averaged variant has a single full-width table per order (sub_tables must be 1)");
    if (c.max_order == 1) {
        if (!c.sub_vocab.empty()) invalid("base-only config must have no sub-table vocabularies");
        return;
    }
    if (c.variant == 1 && c.dim % c.branch_count() != 0)
        invalid("dim " + std::to_string(c.dim) + " not divisible by (max_order-1)*sub_tables = " +
                std::to_string(c.branch_count()));
    if (c.sub_vocab.size() != size_t(c.branch_count()))
        invalid("expected " + std::to_string(c.branch_count()) + " sub-table vocabulary sizes, got " +
                std::to_string(c.sub_vocab.size()));
    for (uint64_t v : c.sub_vocab)
        if (v < 1) invalid("every V_{n,k} must be >= 1");
}

Config parse_config(const std::string& json_text) {
    Config c;
    std::map<std::pair<int, int>, uint64_t> sv;
    try {
        const auto j = nlohmann::json::parse(json_text);
        c.max_order = j.at("max_order").get<int>();
        c.sub_tables = j.at("sub_tables").get<int>();
        c.base_vocab = j.at("base_vocab").get<uint32_t>();
        c.dim = j.at("dim").get<int>();
        const std::string var = j.at("variant").get<std::string>();
        if (var == "averaged_v1") c.variant = 0;
        else if (var == "subtable_v2") c.variant = 1;
        else invalid("unknown variant '" + var + "'");
        const std::string amp = j.at("amplification").get<std::string>();
        if (amp == "none") c.amp = 0;
        else if (amp == "scale_sqrt_d") c.amp = 1;
        else if (amp == "layer_norm") c.amp = 2;
        else invalid("unknown amplification '" + amp + "'");
        for (const auto& e : j.at("sub_vocab"))
            sv[{e.at("n").get<int>(), e.at("k").get<int>()}] = e.at("vocab").get<uint64_t>();
    } catch (const nlohmann::json::exception& e) {
        throw Error(NGRAM_EPARSE, std::string("bad config JSON: ") + e.what());
    }
    // The reference keeps a (n,k) map; validate() checks its size, then looks every branch
    // up (config.cpp:56-76, vocab_of :23-30).  Same order here, on the map.
    Config probe = c;
    probe.sub_vocab.assign(sv.size(), 1);  // size-only stand-in for the checks before the lookups
    validate(probe);
    if (c.max_order >= 2) {
        for (int n = 2; n <= c.max_order; ++n)
            for (int k = 1; k <= c.sub_tables; ++k) {
                auto it = sv.find({n, k});
                if (it == sv.end())
                    invalid("missing vocabulary size for (n=" + std::to_string(n) + ", k=" + std::to_string(k) + ")");
                c.sub_vocab.push_back(it->second);
            }
    }
    validate(c);
    return c;
}

std::string to_json(const Config& c) {
    nlohmann::json j;
    j["max_order"] = c.max_order;
    j["sub_tables"] = c.sub_tables;
    j["base_vocab"] = c.base_vocab;
    j["dim"] = c.dim;
    j["variant"] = c.variant == 0 ? "averaged_v1" : "subtable_v2";
    j["amplification"] = c.amp == 0 ? "none" : (c.amp == 1 ? "scale_sqrt_d" : "layer_norm");
    auto& sv = j["sub_vocab"] = nlohmann::json::array();
    for (int n = 2; n <= c.max_order; ++n)
        for (int k = 1; k <= c.sub_tables; ++k)
            sv.push_back({{"n", n}, {"k", k}, {"vocab", c.sub_vocab[size_t(c.branch_index(n, k))]}});
    return j.dump(2);
}

Config default_config(uint32_t base_vocab, int dim, int max_order, int sub_tables) {
    Config c;
    c.max_order = max_order;
    c.sub_tables = sub_tables;
    c.base_vocab = base_vocab;
    c.dim = dim;
    c.variant = 1;
    c.amp = 1;
    for (int n = 2; n <= max_order; ++n)
        for (int k = 1; k <= sub_tables; ++k) {
            const uint64_t multiple = 8ULL * uint64_t(n - 1) + 4ULL * uint64_t(k - 1);
            c.sub_vocab.push_back(half_multiple_size(base_vocab, multiple));
        }
    validate(c);
    return c;
}

}  // namespace ngh
