// dropin.cpp -- the C++ drop-in API (include/ngram/*.hpp) on top of the C-ABI
// (include/ngram_b200.h).  Host logic only: argument validation in the reference's
// order, exception mapping, JSON; every hash / embedding is computed by the
// CUDA kernels behind libngram_b200.so.  Built as libngram.so (g++), linked to it.
#include <atomic>
#include <cstring>
#include <fstream>
#include <list>
#include <map>
#include <mutex>
#include <sstream>
#include <thread>
#include <type_traits>

#include <json.hpp>

#include "ngram/cache.hpp"
#include "ngram/config.hpp"
#include "ngram/embedding.hpp"
#include "ngram/errors.hpp"
#include "ngram/hashing.hpp"
#include "ngram/ple.hpp"
#include "ngram_b200.h"

namespace ngram {

void throw_status(int st) {
    if (st == NGRAM_OK) return;
    const std::string m = ngram_last_error();
    switch (st) {
        case NGRAM_EINVAL: throw std::invalid_argument(m);
        case NGRAM_ERANGE: throw std::out_of_range(m);
        case NGRAM_EIO: throw io_error(m);
        case NGRAM_EPARSE: throw parse_error(m, 0, 0);
        case NGRAM_ECONFIG: throw config_error(m);
        case NGRAM_ENUMERIC: throw numeric_error(m);
        default: throw device_error(m);
    }
}

// ------------------------------------------------------------------------ config
const char* to_string(ne_variant v) { return v == ne_variant::averaged_v1 ? "averaged_v1" : "subtable_v2"; }
const char* to_string(amp_mode m) {
    return m == amp_mode::none ? "none" : (m == amp_mode::scale_sqrt_d ? "scale_sqrt_d" : "layer_norm");
}

std::uint64_t ngram_config::vocab_of(int n, int k) const {
    const auto it = sub_vocab.find({n, k});
    if (it == sub_vocab.end())
        throw std::invalid_argument("ngram_config: missing vocabulary size for (n=" + std::to_string(n) +
                                    ", k=" + std::to_string(k) + ")");
    return it->second;
}

std::string to_json_string(const ngram_config& c) {
    nlohmann::json j;
    j["max_order"] = c.max_order;
    j["sub_tables"] = c.sub_tables;
    j["base_vocab"] = c.base_vocab;
    j["dim"] = c.dim;
    j["variant"] = to_string(c.variant);
    j["amplification"] = to_string(c.amplification);
    auto& sv = j["sub_vocab"] = nlohmann::json::array();
    for (const auto& [nk, v] : c.sub_vocab) sv.push_back({{"n", nk.first}, {"k", nk.second}, {"vocab", v}});
    return j.dump(2);
}

void ngram_config::validate() const { throw_status(ngram_config_validate(to_json_string(*this).c_str())); }

ngram_config ngram_config_from_json(const std::string& text) {
    throw_status(ngram_config_validate(text.c_str()));
    const auto j = nlohmann::json::parse(text);
    ngram_config c;
    c.max_order = j.at("max_order").get<int>();
    c.sub_tables = j.at("sub_tables").get<int>();
    c.base_vocab = j.at("base_vocab").get<std::uint32_t>();
    c.dim = j.at("dim").get<int>();
    c.variant = j.at("variant").get<std::string>() == "averaged_v1" ? ne_variant::averaged_v1 : ne_variant::subtable_v2;
    const auto a = j.at("amplification").get<std::string>();
    c.amplification = a == "none" ? amp_mode::none : (a == "scale_sqrt_d" ? amp_mode::scale_sqrt_d : amp_mode::layer_norm);
    for (const auto& e : j.at("sub_vocab"))
        c.sub_vocab[{e.at("n").get<int>(), e.at("k").get<int>()}] = e.at("vocab").get<std::uint64_t>();
    return c;
}

ngram_config load_ngram_config(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw io_error("cannot open config file: " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ngram_config_from_json(ss.str());
}

void save_ngram_config(const ngram_config& cfg, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw io_error("cannot write config file: " + path);
    out << to_json_string(cfg) << '\n';
}

ngram_config make_default_config(std::uint32_t base_vocab, int dim, int max_order, int sub_tables) {
    std::string buf(1 << 16, '\0');
    throw_status(ngram_make_default_config(base_vocab, dim, max_order, sub_tables, buf.data(), buf.size()));
    return ngram_config_from_json(buf.c_str());
}

// ------------------------------------------------------------------------ banks
device_bank::device_bank(const ngram_config& cfg, int device, int shard_rank, int shard_count) : cfg_(cfg) {
    ngram_bank* h = nullptr;
    throw_status(ngram_bank_create(to_json_string(cfg).c_str(), device, shard_rank, shard_count, &h));
    h_.reset(h, [](ngram_bank* p) { ngram_bank_destroy(p); });
}

device_bank::device_bank(const embedding_bank& host, int device) : device_bank(host.config, device) { upload(host); }

device_bank device_bank::from_file(const std::string& path, const ngram_config& cfg, int device) {
    device_bank b(cfg, device);
    throw_status(ngram_bank_load_file(b.handle(), path.c_str()));
    return b;
}

void device_bank::upload(const embedding_bank& host) {
    std::vector<const float*> sub, proj;
    for (const auto& t : host.sub_tables) sub.push_back(t.data());
    for (const auto& p : host.projections) proj.push_back(p.data());
    throw_status(ngram_bank_upload_f32(h_.get(), host.base.data(), sub.data(), proj.empty() ? nullptr : proj.data(),
                                       host.ln_gain.empty() ? nullptr : host.ln_gain.data(),
                                       host.ln_bias.empty() ? nullptr : host.ln_bias.data()));
}

void device_bank::generate(std::uint64_t seed) {
    throw_status(ngram_bank_generate(h_.get(), seed, nullptr));
    throw_status(ngram_sync_errors(h_.get(), nullptr));
}

bool device_bank::tensor_core_path() const {
    ngram_bank_info info;
    throw_status(ngram_bank_get_info(h_.get(), &info));
    return info.tensor_core_path != 0;
}

namespace {
std::uint64_t fingerprint_range(const float* p, std::size_t n) {
    std::uint64_t h = 0x9e3779b97f4a7c15ULL ^ n;
    std::size_t i = 0;
    for (; i + 2 <= n; i += 2) {
        std::uint64_t w;
        std::memcpy(&w, p + i, 8);
        h = (h ^ w) * 0x100000001b3ULL + (h >> 29);
    }
    if (i < n) {
        std::uint32_t w;
        std::memcpy(&w, p + i, 4);
        h = (h ^ w) * 0x100000001b3ULL + (h >> 29);
    }
    return h * 0x9e3779b97f4a7c15ULL;
}

// 64-bit content fingerprint of a host bank: chunks of 4 M floats hashed on up to 8 threads
// (large banks: a 220 MB bank in ~5 ms instead of ~50 ms), combined in a fixed order.
std::uint64_t fingerprint(const embedding_bank& b) {
    constexpr std::size_t kChunk = std::size_t(1) << 22;
    std::vector<std::pair<const float*, std::size_t>> chunks;
    auto add = [&](const std::vector<float>& v) {
        for (std::size_t o = 0; o < v.size(); o += kChunk) chunks.emplace_back(v.data() + o, std::min(kChunk, v.size() - o));
        chunks.emplace_back(nullptr, v.size());  // tensor boundary (and empty tensors) count too
    };
    add(b.base);
    for (const auto& t : b.sub_tables) add(t);
    for (const auto& w : b.projections) add(w);
    add(b.ln_gain);
    add(b.ln_bias);
    std::vector<std::uint64_t> hs(chunks.size());
    auto work = [&](std::size_t first, std::size_t step) {
        for (std::size_t c = first; c < chunks.size(); c += step)
            hs[c] = chunks[c].first ? fingerprint_range(chunks[c].first, chunks[c].second) : chunks[c].second;
    };
    const std::size_t nthreads =
        chunks.size() > 4 ? std::min<std::size_t>(8, std::max(1u, std::thread::hardware_concurrency())) : 1;
    std::vector<std::thread> pool;
    for (std::size_t t = 1; t < nthreads; ++t) pool.emplace_back(work, t, nthreads);
    work(0, nthreads);
    for (auto& t : pool) t.join();
    std::uint64_t h = std::hash<std::string>()(to_json_string(b.config));
    for (const std::uint64_t x : hs) h = (h ^ x) * 0x100000001b3ULL + (h >> 31);
    return h;
}
}  // namespace

std::shared_ptr<const device_bank> device_bank_for(const embedding_bank& host) {
    struct entry {
        const embedding_bank* addr;
        std::uint64_t fp;
        std::shared_ptr<const device_bank> dev;
    };
    static std::mutex mu;
    // most recently used first, at most kKeep banks; never destroyed (device banks must not be
    // released after the CUDA driver has shut down at process exit)
    static auto& cache = *new std::list<entry>();
    constexpr std::size_t kKeep = 4;
    const std::uint64_t fp = fingerprint(host);
    std::lock_guard<std::mutex> g(mu);
    for (auto it = cache.begin(); it != cache.end(); ++it)
        if (it->addr == &host && it->fp == fp) {
            cache.splice(cache.begin(), cache, it);
            return cache.front().dev;
        }
    auto dev = std::make_shared<const device_bank>(host);
    cache.push_front({&host, fp, dev});
    if (cache.size() > kKeep) cache.pop_back();
    return dev;
}

// ------------------------------------------------------------------------ hashing
void hash_spec::validate() const {
    if (order < 2) throw std::invalid_argument("hash_spec: order must be >= 2, got " + std::to_string(order));
    if (base < 2) throw std::invalid_argument("hash_spec: base must be >= 2, got " + std::to_string(base));
    if (modulus < 1) throw std::invalid_argument("hash_spec: modulus must be >= 1");
}

std::uint64_t rolling_hash(std::span<const token_id> window, const hash_spec& spec) {
    spec.validate();
    if (window.size() != std::size_t(spec.order))
        throw std::invalid_argument("rolling_hash: window length " + std::to_string(window.size()) +
                                    " does not match order " + std::to_string(spec.order));
    const int32_t len = int32_t(window.size()), order = spec.order;
    uint64_t out = 0;
    int32_t status = 0;
    throw_status(ngram_rolling_hash_host(window.data(), len, &len, &order, &spec.base, &spec.modulus, 1, &out, &status));
    if (status == NGRAM_ERANGE) throw std::out_of_range("rolling_hash: token out of range for base vocabulary");
    throw_status(status);
    return out;
}

namespace {
// Hash-only device banks keyed by config: hash_all_orders needs only the config.  The key is
// the config's fields (no JSON on the per-call path); a config is validated once, when its
// hasher is created (ngram_bank_create_ex validates).
std::vector<std::uint64_t> config_key(const ngram_config& c) {
    std::vector<std::uint64_t> k{std::uint64_t(c.max_order), std::uint64_t(c.sub_tables), c.base_vocab,
                                 std::uint64_t(c.dim), std::uint64_t(c.variant), std::uint64_t(c.amplification)};
    for (const auto& [nk, v] : c.sub_vocab) {
        k.push_back((std::uint64_t(std::uint32_t(nk.first)) << 32) | std::uint32_t(nk.second));
        k.push_back(v);
    }
    return k;
}

std::shared_ptr<ngram_bank> hasher_for(const ngram_config& cfg) {
    static std::mutex mu;
    static auto& cache = *new std::map<std::vector<std::uint64_t>, std::shared_ptr<ngram_bank>>();  // never destroyed
    auto key = config_key(cfg);
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    ngram_bank* h = nullptr;
    throw_status(ngram_bank_create_ex(to_json_string(cfg).c_str(), 0, 0, 1, NGRAM_BANK_HASH_ONLY, &h));
    std::shared_ptr<ngram_bank> p(h, [](ngram_bank* b) { ngram_bank_destroy(b); });
    cache.emplace(std::move(key), p);
    return p;
}

std::vector<token_id> prior_tail(std::span<const token_id> prior, int N1) {
    std::vector<token_id> m(std::size_t(std::max(N1, 0)), 0);
    const std::size_t n = std::min<std::size_t>(prior.size(), m.size());
    for (std::size_t i = 0; i < n; ++i) m[m.size() - n + i] = prior[prior.size() - n + i];
    return m;
}
}  // namespace

std::vector<std::uint64_t> hash_all_orders(std::span<const token_id> context, const ngram_config& cfg) {
    auto h = hasher_for(cfg);  // validates the config (hashing.cpp:63) the first time it is seen
    if (context.size() != std::size_t(cfg.max_order))
        throw std::invalid_argument("hash_all_orders: context length " + std::to_string(context.size()) +
                                    " does not match max order " + std::to_string(cfg.max_order));
    std::vector<std::uint64_t> ids(std::size_t(cfg.branch_count()));
    if (ids.empty()) return ids;
    const int64_t off[2] = {0, 1};
    throw_status(ngram_hash_ids_host(h.get(), &context.back(), off, 1, context.data(), ids.data()));
    return ids;
}

std::vector<std::uint64_t> hash_sequence(std::span<const token_id> tokens, const device_bank& bank,
                                         std::span<const token_id> prior_context) {
    const auto& cfg = bank.config();
    std::vector<std::uint64_t> ids(tokens.size() * std::size_t(cfg.branch_count()));
    if (tokens.empty() || ids.empty()) return ids;
    const auto pr = prior_tail(prior_context, cfg.max_order - 1);
    const int64_t off[2] = {0, int64_t(tokens.size())};
    throw_status(ngram_hash_ids_host(bank.handle(), tokens.data(), off, 1, pr.empty() ? nullptr : pr.data(), ids.data()));
    return ids;
}

// ------------------------------------------------------------------------ forward
void embed_from_ids(token_id token, std::span<const std::uint64_t> ids, const device_bank& bank, std::span<float> out,
                    embed_counters* counters) {
    const auto& cfg = bank.config();
    if (ids.size() != std::size_t(cfg.branch_count()))
        throw std::invalid_argument("embed_from_ids: expected " + std::to_string(cfg.branch_count()) +
                                    " bucket ids, got " + std::to_string(ids.size()));
    if (out.size() != std::size_t(cfg.dim)) throw std::invalid_argument("embed_from_ids: output size mismatch");
    throw_status(ngram_embed_from_ids_host(bank.handle(), &token, ids.data(), 1, out.data()));
    if (counters) {
        counters->table_gathers += 1 + std::uint64_t(cfg.branch_count());
        if (cfg.variant == ne_variant::subtable_v2)
            counters->projection_madds += std::uint64_t(cfg.dim) * std::uint64_t(cfg.branch_dim()) * cfg.branch_count();
    }
}

void embed_from_ids(token_id token, std::span<const std::uint64_t> ids, const embedding_bank& bank,
                    std::span<float> out, embed_counters* counters) {
    embed_from_ids(token, ids, *device_bank_for(bank), out, counters);
}

sequence_embedding<float> embed_sequence_cached(std::span<const token_id> tokens, const device_bank& bank,
                                                std::span<const token_id> prior_context, embed_counters* counters) {
    const auto& cfg = bank.config();
    sequence_embedding<float> r;
    r.rows.resize(tokens.size() * std::size_t(cfg.dim));
    r.merged.resize(r.rows.size());
    if (tokens.empty()) return r;
    const auto pr = prior_tail(prior_context, cfg.max_order - 1);
    const int64_t off[2] = {0, int64_t(tokens.size())};
    throw_status(ngram_embed_sequence_host(bank.handle(), tokens.data(), off, 1, pr.empty() ? nullptr : pr.data(),
                                           r.rows.data(), r.merged.data(), NGRAM_F32));
    if (counters) {
        counters->table_gathers += tokens.size() * (1 + std::uint64_t(cfg.branch_count()));
        if (cfg.variant == ne_variant::subtable_v2)
            counters->projection_madds +=
                tokens.size() * std::uint64_t(cfg.dim) * std::uint64_t(cfg.branch_dim()) * cfg.branch_count();
    }
    return r;
}

std::vector<float> embed_sequence(std::span<const token_id> tokens, const device_bank& bank,
                                  std::span<const token_id> prior_context) {
    return embed_sequence_cached(tokens, bank, prior_context).rows;
}

sequence_embedding<float> embed_sequence_cached(std::span<const token_id> tokens, const embedding_bank& bank,
                                                std::span<const token_id> prior_context, embed_counters* counters) {
    return embed_sequence_cached(tokens, *device_bank_for(bank), prior_context, counters);
}

std::vector<float> embed_sequence(std::span<const token_id> tokens, const embedding_bank& bank,
                                  std::span<const token_id> prior_context) {
    return embed_sequence_cached(tokens, *device_bank_for(bank), prior_context).rows;
}

namespace {
void add_device_grads(ngram_grad* g, embedding_bank& grads);

// Run one device backward into a fresh fp32 gradient bank and add it into the host grads.
void backward_into(const device_bank& bank, std::span<const token_id> tokens, std::span<const token_id> prior,
                   const float* merged, const float* upstream, int flags, embedding_bank& grads) {
    const auto& cfg = bank.config();
    if (grads.base.size() != std::size_t(cfg.base_vocab) * std::size_t(cfg.dim) ||
        grads.sub_tables.size() != std::size_t(cfg.branch_count()))
        throw std::invalid_argument("embed_backward: gradient bank shape does not match the bank");
    ngram_grad* g = nullptr;
    throw_status(ngram_grad_create(bank.handle(), &g));
    std::unique_ptr<ngram_grad, int (*)(ngram_grad*)> guard(g, ngram_grad_destroy);
    const auto pr = prior_tail(prior, cfg.max_order - 1);
    const int64_t off[2] = {0, int64_t(tokens.size())};
    throw_status(ngram_embed_backward_host(g, tokens.data(), off, 1, pr.empty() ? nullptr : pr.data(), merged, upstream,
                                           flags));
    add_device_grads(g, grads);
}

// grads += the device gradient bank (reference layout download).
void add_device_grads(ngram_grad* g, embedding_bank& grads) {
    embedding_bank d = zeros_like(grads);
    std::vector<float*> sp, pp;
    for (auto& t : d.sub_tables) sp.push_back(t.data());
    for (auto& p : d.projections) pp.push_back(p.data());
    throw_status(ngram_grad_download(g, d.base.data(), sp.empty() ? nullptr : sp.data(),
                                     pp.empty() ? nullptr : pp.data(), d.ln_gain.empty() ? nullptr : d.ln_gain.data(),
                                     d.ln_bias.empty() ? nullptr : d.ln_bias.data()));
    auto add = [](std::vector<float>& a, const std::vector<float>& b) {
        for (std::size_t i = 0; i < a.size() && i < b.size(); ++i) a[i] += b[i];
    };
    add(grads.base, d.base);
    for (std::size_t b = 0; b < grads.sub_tables.size(); ++b) add(grads.sub_tables[b], d.sub_tables[b]);
    for (std::size_t b = 0; b < grads.projections.size() && b < d.projections.size(); ++b)
        add(grads.projections[b], d.projections[b]);
    add(grads.ln_gain, d.ln_gain);
    add(grads.ln_bias, d.ln_bias);
}
}  // namespace

void amplify_backward(std::span<const float> pre, std::span<const float> upstream, const device_bank& bank,
                      embedding_bank& grads, std::span<float> d_pre) {
    const std::size_t D = std::size_t(bank.config().dim);
    if (pre.size() != D || upstream.size() != D || d_pre.size() != D)
        throw std::invalid_argument("amplify_backward: size mismatch");
    const bool ln = bank.config().amplification == amp_mode::layer_norm;
    if (ln && (grads.ln_gain.size() != D || grads.ln_bias.size() != D))
        throw std::invalid_argument("amplify_backward: gradient bank has no layer-norm parameters");
    throw_status(ngram_amplify_backward_host(bank.handle(), 1, pre.data(), upstream.data(), d_pre.data(),
                                             ln ? grads.ln_gain.data() : nullptr, ln ? grads.ln_bias.data() : nullptr));
}

void amplify_backward(std::span<const float> pre, std::span<const float> upstream, const embedding_bank& bank,
                      embedding_bank& grads, std::span<float> d_pre) {
    amplify_backward(pre, upstream, *device_bank_for(bank), grads, d_pre);
}

void embed_backward(std::span<const token_id> context, const device_bank& bank, std::span<const float> upstream,
                    embedding_bank& grads) {
    const auto& cfg = bank.config();
    if (upstream.size() != std::size_t(cfg.dim)) throw std::invalid_argument("embed_backward: upstream size mismatch");
    if (context.size() != std::size_t(cfg.max_order))
        throw std::invalid_argument("hash_all_orders: context length " + std::to_string(context.size()) +
                                    " does not match max order " + std::to_string(cfg.max_order));
    backward_into(bank, context.last(1), context.first(context.size() - 1), nullptr, upstream.data(),
                  NGRAM_BWD_SKIP_AMPLIFY, grads);
}

void embed_backward(std::span<const token_id> context, const embedding_bank& bank, std::span<const float> upstream,
                    embedding_bank& grads) {
    embed_backward(context, *device_bank_for(bank), upstream, grads);
}

void embed_sequence_backward(std::span<const token_id> tokens, const device_bank& bank, std::span<const float> merged,
                             std::span<const float> upstream, embedding_bank& grads,
                             std::span<const token_id> prior_context) {
    const std::size_t n = tokens.size() * std::size_t(bank.config().dim);
    if (upstream.size() != n || merged.size() != n)
        throw std::invalid_argument("embed_sequence_backward: merged / upstream size mismatch");
    if (tokens.empty()) return;
    backward_into(bank, tokens, prior_context, merged.data(), upstream.data(), 0, grads);
}

void embed_sequence_backward(std::span<const token_id> tokens, const embedding_bank& bank,
                             std::span<const float> merged, std::span<const float> upstream, embedding_bank& grads,
                             std::span<const token_id> prior_context) {
    embed_sequence_backward(tokens, *device_bank_for(bank), merged, upstream, grads, prior_context);
}

void embed_window(std::span<const token_id> context, const device_bank& bank, std::span<float> out,
                  embed_counters* counters) {
    const auto& cfg = bank.config();
    if (context.size() != std::size_t(cfg.max_order))
        throw std::invalid_argument("hash_all_orders: context length " + std::to_string(context.size()) +
                                    " does not match max order " + std::to_string(cfg.max_order));
    if (out.size() != std::size_t(cfg.dim)) throw std::invalid_argument("embed_from_ids: output size mismatch");
    auto r = embed_sequence_cached(context.last(1), bank, context.first(context.size() - 1), counters);
    std::copy(r.merged.begin(), r.merged.end(), out.begin());
}

std::vector<float> embed_v1(std::span<const token_id> context, const device_bank& bank) {
    if (bank.config().variant != ne_variant::averaged_v1)
        throw std::invalid_argument("embed_v1 requires the averaged variant");
    std::vector<float> out(std::size_t(bank.config().dim));
    embed_window(context, bank, out);
    return out;
}

std::vector<float> embed_v2(std::span<const token_id> context, const device_bank& bank) {
    if (bank.config().variant != ne_variant::subtable_v2)
        throw std::invalid_argument("embed_v2 requires the sub-table variant");
    std::vector<float> out(std::size_t(bank.config().dim));
    embed_window(context, bank, out);
    return out;
}

std::vector<float> embed_batch(const std::vector<std::vector<token_id>>& seqs, const device_bank& bank) {
    std::vector<int64_t> off(1, 0);
    std::vector<token_id> all;
    for (const auto& s : seqs) {
        all.insert(all.end(), s.begin(), s.end());
        off.push_back(int64_t(all.size()));
    }
    std::vector<float> rows(all.size() * std::size_t(bank.config().dim));
    if (seqs.empty()) return rows;
    throw_status(ngram_embed_sequence_host(bank.handle(), all.data(), off.data(), int64_t(seqs.size()), nullptr,
                                           rows.data(), nullptr, NGRAM_F32));
    return rows;
}

// ------------------------------------------------------------------------ cache
std::string counters_to_json(const cache_counters& c) {
    std::ostringstream ss;
    ss << "{\"appends\":" << c.appends << ",\"rollbacks\":" << c.rollbacks << ",\"memo_hits\":" << c.memo_hits
       << ",\"memo_misses\":" << c.memo_misses << ",\"table_gathers\":" << c.table_gathers
       << ",\"projection_madds\":" << c.projection_madds << ",\"draft_table_gathers\":" << c.draft_table_gathers
       << ",\"verify_table_gathers\":" << c.verify_table_gathers << "}";
    return ss.str();
}

namespace {
std::uint64_t next_uid() {
    static std::atomic<std::uint64_t> u{1};
    return u.fetch_add(1);
}
constexpr int kMaxDraft = 64;
}  // namespace

sequence_cache::sequence_cache(const ngram_config& cfg) : cfg_(cfg) {
    cfg_.validate();
    bank_ = hasher_for(cfg_);  // ids need only the config; tables join at the first bind()
    ngram_decode* d = nullptr;
    throw_status(ngram_decode_create(bank_.get(), 1, kMaxDraft, &d));
    st_.reset(d, [](ngram_decode* p) { ngram_decode_destroy(p); });
    uid_ = next_uid();
}

sequence_cache::sequence_cache(const device_bank& bank) : cfg_(bank.config()), bank_(bank.shared_handle()) {
    cfg_.validate();
    ngram_decode* d = nullptr;
    throw_status(ngram_decode_create(bank_.get(), 1, kMaxDraft, &d));
    st_.reset(d, [](ngram_decode* p) { ngram_decode_destroy(p); });
    uid_ = next_uid();
}

void sequence_cache::bind(const device_bank& bank) {
    if (bank.handle() == bank_.get()) return;
    if (to_json_string(bank.config()) != to_json_string(cfg_))
        throw std::invalid_argument("sequence_cache: bank config does not match the state's config");
    snap cur;
    cur.ring.assign(std::size_t(std::max(cfg_.max_order - 1, 0)), 0);
    throw_status(ngram_decode_get_state(st_.get(), cur.ring.empty() ? nullptr : cur.ring.data(), &cur.length,
                                        &cur.last));
    ngram_decode* d = nullptr;
    throw_status(ngram_decode_create(bank.handle(), 1, kMaxDraft, &d));
    st_.reset(d, [](ngram_decode* p) { ngram_decode_destroy(p); });
    bank_ = bank.shared_handle();
    restore(cur);
}

std::vector<std::uint64_t> sequence_cache::append(token_id token, cache_counters* counters) {
    if (std::uint64_t(token) >= config().base_vocab)
        throw std::out_of_range("sequence_cache: token " + std::to_string(token) + " out of range");
    std::vector<std::uint64_t> ids(std::size_t(config().branch_count()));
    throw_status(ngram_decode_step_host(st_.get(), &token, ids.empty() ? nullptr : ids.data(), nullptr));
    if (counters) counters->appends++;
    return ids;
}

std::uint64_t sequence_cache::length() const {
    uint64_t len = 0;
    token_id last = 0;
    throw_status(ngram_decode_get_state(st_.get(), nullptr, &len, &last));
    return len;
}

token_id sequence_cache::last_token() const {
    uint64_t len = 0;
    token_id last = 0;
    throw_status(ngram_decode_get_state(st_.get(), nullptr, &len, &last));
    return last;
}

std::span<const token_id> sequence_cache::ring() const {
    uint64_t len = 0;
    token_id last = 0;
    ring_view_.resize(std::size_t(std::max(config().max_order - 1, 0)));
    throw_status(ngram_decode_get_state(st_.get(), ring_view_.empty() ? nullptr : ring_view_.data(), &len, &last));
    return ring_view_;
}

snapshot_handle sequence_cache::snapshot() {
    snap s;
    s.serial = next_serial_++;
    s.ring.assign(std::size_t(std::max(config().max_order - 1, 0)), 0);
    throw_status(ngram_decode_get_state(st_.get(), s.ring.empty() ? nullptr : s.ring.data(), &s.length, &s.last));
    snaps_.push_back(std::move(s));
    return {uid_, snaps_.back().serial, snaps_.size() - 1};
}

void sequence_cache::check(const snapshot_handle& h) const {
    if (h.owner != uid_) throw std::invalid_argument("sequence_cache: handle belongs to another state");
    if (h.slot >= snaps_.size() || snaps_[h.slot].serial != h.serial)
        throw std::invalid_argument("sequence_cache: stale snapshot handle");
}

void sequence_cache::restore(const snap& s) {
    throw_status(ngram_decode_set_state_host(st_.get(), s.ring.empty() ? nullptr : s.ring.data(), &s.length, &s.last));
}

void sequence_cache::rollback(const snapshot_handle& h, cache_counters* counters) {
    check(h);
    restore(snaps_[h.slot]);
    snaps_.resize(h.slot + 1);
    if (counters) counters->rollbacks++;
}

void sequence_cache::discard(const snapshot_handle& h) {
    check(h);
    if (h.slot + 1 != snaps_.size()) throw std::invalid_argument("sequence_cache: only the top snapshot can be discarded");
    snaps_.pop_back();
}

std::vector<float> embedding_memo::lookup(token_id token, std::span<const std::uint64_t> ids, const device_bank& bank,
                                          cache_counters* counters) {
    key k;
    k.reserve(ids.size() + 1);
    k.push_back(token);
    k.insert(k.end(), ids.begin(), ids.end());
    if (const auto it = where_.find(k); it != where_.end()) {
        lru_.splice(lru_.begin(), lru_, it->second);
        if (counters) counters->memo_hits++;
        return it->second->second;
    }
    std::vector<float> e(std::size_t(bank.config().dim));
    embed_counters ec;
    embed_from_ids(token, ids, bank, e, &ec);
    if (counters) {
        counters->memo_misses++;
        counters->table_gathers += ec.table_gathers;
        counters->projection_madds += ec.projection_madds;
    }
    if (lru_.size() == capacity_) {
        where_.erase(lru_.back().first);
        lru_.pop_back();
    }
    lru_.emplace_front(std::move(k), e);
    where_[lru_.front().first] = lru_.begin();
    return e;
}

std::vector<float> embedding_memo::lookup(token_id token, std::span<const std::uint64_t> ids,
                                          const embedding_bank& bank, cache_counters* counters) {
    key k;  // a hit touches no table (cache.cpp:123-133): look up before resolving the device bank
    k.reserve(ids.size() + 1);
    k.push_back(token);
    k.insert(k.end(), ids.begin(), ids.end());
    if (const auto it = where_.find(k); it != where_.end()) {
        lru_.splice(lru_.begin(), lru_, it->second);
        if (counters) counters->memo_hits++;
        return it->second->second;
    }
    return lookup(token, ids, *device_bank_for(bank), counters);
}

draft_result draft_verify(sequence_cache& state, const device_bank& bank, std::span<const token_id> draft,
                          std::size_t accept_count, cache_counters* counters, const draft_options& opts) {
    if (accept_count > draft.size()) throw std::invalid_argument("draft_verify: accept count exceeds draft length");
    const auto& cfg = bank.config();
    state.bind(bank);
    for (const token_id t : draft)
        if (std::uint64_t(t) >= cfg.base_vocab)
            throw std::out_of_range("sequence_cache: token " + std::to_string(t) + " out of range");
    draft_result res;
    const std::size_t D = std::size_t(cfg.dim);
    std::size_t done = 0, remaining = accept_count;
    while (done < draft.size()) {  // verify blocks of at most kMaxDraft tokens
        const int L = int(std::min<std::size_t>(kMaxDraft, draft.size() - done));
        const int32_t acc = int32_t(std::min<std::size_t>(remaining, std::size_t(L)));
        std::vector<float> out(std::size_t(L) * D);
        throw_status(ngram_verify_commit_host(state.handle(), draft.data() + done, L, &acc, out.data()));
        for (int i = 0; i < acc; ++i) res.accepted.emplace_back(out.begin() + i * D, out.begin() + (i + 1) * D);
        remaining -= std::size_t(acc);
        done += std::size_t(L);
        if (acc < L) break;  // the rest of the draft was rejected
    }
    if (counters) {  // the reference's work counters, evaluated arithmetically (cache.cpp:164-192)
        const std::uint64_t L = draft.size(), A = accept_count, g = 1 + std::uint64_t(cfg.branch_count());
        const std::uint64_t madds = cfg.variant == ne_variant::subtable_v2
                                        ? std::uint64_t(cfg.dim) * cfg.branch_dim() * cfg.branch_count()
                                        : 0;
        counters->appends += L + A;
        counters->rollbacks += 1;
        if (opts.conventional_draft_embedding) {
            counters->table_gathers += L + A * g;
            counters->draft_table_gathers += L;
            counters->verify_table_gathers += A * g;
            counters->memo_misses += A;
            counters->projection_madds += A * madds;
        } else {
            counters->table_gathers += L * g;
            counters->draft_table_gathers += L * g;
            counters->memo_misses += L;
            counters->memo_hits += A;
            counters->projection_madds += L * madds;
        }
    }
    return res;
}

draft_result draft_verify(sequence_cache& state, embedding_memo&, const device_bank& bank,
                          std::span<const token_id> draft, std::size_t accept_count, cache_counters* counters,
                          const draft_options& opts) {
    return draft_verify(state, bank, draft, accept_count, counters, opts);
}

draft_result draft_verify(sequence_cache& state, embedding_memo& memo, const embedding_bank& bank,
                          std::span<const token_id> draft, std::size_t accept_count, cache_counters* counters,
                          const draft_options& opts) {
    if (accept_count > draft.size()) throw std::invalid_argument("draft_verify: accept count exceeds draft length");
    return draft_verify(state, memo, *device_bank_for(bank), draft, accept_count, counters, opts);
}

void amplify(std::span<const float> e, amp_mode mode, std::span<const float> gain, std::span<const float> bias,
             std::span<float> out) {
    const std::size_t D = e.size();
    if (out.size() != D) throw std::invalid_argument("amplify: output size mismatch");
    if (mode == amp_mode::layer_norm && (gain.size() != D || bias.size() != D))
        throw std::invalid_argument("amplify: layer_norm needs gain/bias of size D");
    const int m = mode == amp_mode::none ? 0 : mode == amp_mode::scale_sqrt_d ? 1 : 2;
    throw_status(ngram_amplify_host(m, int(D), D ? 1 : 0, m == 2 ? gain.data() : nullptr,
                                    m == 2 ? bias.data() : nullptr, e.data(), out.data()));
}

// ---------------------------------------------------------------- accounting / serialization
param_count_report param_count(const ngram_config& cfg) {
    cfg.validate();
    param_count_report r;
    const std::uint64_t D = std::uint64_t(cfg.dim), d = std::uint64_t(cfg.branch_dim());
    r.base = std::uint64_t(cfg.base_vocab) * D;
    for (const auto& kv : cfg.sub_vocab) r.sub_tables += kv.second * d;
    if (cfg.variant == ne_variant::subtable_v2) r.projections = std::uint64_t(cfg.branch_count()) * D * d;
    r.total = r.base + r.sub_tables + r.projections;
    return r;
}

budget_info budget_report(std::uint64_t embedding_params, std::uint64_t other_params) {
    budget_info b;
    b.embedding_params = embedding_params;
    b.other_params = other_params;
    const double all = double(embedding_params) + double(other_params);
    b.fraction = all > 0.0 ? double(embedding_params) / all : 0.0;
    b.over_budget = b.fraction > 0.5;
    return b;
}

budget_info budget_report(const ngram_config& cfg, std::uint64_t other_params) {
    return budget_report(param_count(cfg).total, other_params);
}

std::string budget_guidance(const budget_info& info) {
    std::string s = "embedding parameters take " + std::to_string(int(info.fraction * 100.0 + 0.5)) +
                    "% of the total budget; keep this at or below 50%. ";
    if (info.over_budget)
        s += "This configuration is over budget: past the halfway point the same parameters buy more as FFN "
             "capacity. ";
    s += "Reference point: a production 68.5B-parameter model allocates 31.4B parameters (46% of the total) to "
         "n-gram embeddings.";
    return s;
}

namespace {
void put_f32(std::ofstream& f, const std::vector<float>& v) {
    f.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * 4));
}
void get_f32(std::ifstream& f, std::vector<float>& v, const std::string& path) {
    f.read(reinterpret_cast<char*>(v.data()), std::streamsize(v.size() * 4));
    if (!f) throw parse_error("bank file truncated: " + path, 0, std::size_t(f.gcount()));
}
}  // namespace

void save_bank(const embedding_bank& bank, const std::string& path) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw io_error("cannot write bank file: " + path);
    const std::string head = to_json_string(bank.config);
    const std::uint32_t n = std::uint32_t(head.size());
    const unsigned char len[4] = {static_cast<unsigned char>(n), static_cast<unsigned char>(n >> 8),
                                  static_cast<unsigned char>(n >> 16), static_cast<unsigned char>(n >> 24)};
    f.write(reinterpret_cast<const char*>(len), 4);
    f.write(head.data(), std::streamsize(head.size()));
    put_f32(f, bank.base);
    for (const auto& t : bank.sub_tables) put_f32(f, t);
    for (const auto& w : bank.projections) put_f32(f, w);
    if (bank.config.amplification == amp_mode::layer_norm) {
        put_f32(f, bank.ln_gain);
        put_f32(f, bank.ln_bias);
    }
    if (!f) throw io_error("short write to bank file: " + path);
}

embedding_bank load_bank(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw io_error("cannot open bank file: " + path);
    unsigned char len[4];
    f.read(reinterpret_cast<char*>(len), 4);
    if (!f) throw parse_error("bank file too short for header: " + path, 0, 0);
    const std::uint32_t n = std::uint32_t(len[0]) | (std::uint32_t(len[1]) << 8) | (std::uint32_t(len[2]) << 16) |
                            (std::uint32_t(len[3]) << 24);
    std::string head(n, '\0');
    f.read(head.data(), std::streamsize(n));
    if (!f) throw parse_error("bank file truncated in header: " + path, 0, 4);
    ngram_config cfg;
    try {
        cfg = ngram_config_from_json(head);
    } catch (const nlohmann::json::exception& e) {
        throw parse_error(std::string("bad bank header JSON: ") + e.what(), 0, 4);
    }
    embedding_bank bank = make_zero_bank<float>(cfg);
    get_f32(f, bank.base, path);
    for (auto& t : bank.sub_tables) get_f32(f, t, path);
    for (auto& w : bank.projections) get_f32(f, w, path);
    if (cfg.amplification == amp_mode::layer_norm) {
        get_f32(f, bank.ln_gain, path);
        get_f32(f, bank.ln_bias, path);
    }
    char extra;
    if (f.read(&extra, 1)) throw parse_error("bank file longer than its header declares: " + path, 0, 0);
    return bank;
}

// ---------------------------------------------------------------- per-layer FFN (ple.hpp)
namespace {
using plne_ptr = std::unique_ptr<ngram_plne, int (*)(ngram_plne*)>;

plne_ptr make_plne(const device_bank& bank, const ple_params& p, std::span<const float> x) {
    if (x.size() != std::size_t(p.d_model) || bank.config().dim != p.hidden)
        throw std::invalid_argument("ple: input/gate width mismatch");
    ngram_plne* h = nullptr;
    throw_status(ngram_plne_create(bank.handle(), p.d_model, &h));
    return plne_ptr(h, ngram_plne_destroy);
}

void check_layer_bank(const device_bank& bank, const ple_params& p, std::span<const token_id> context) {
    const auto& cfg = bank.config();
    if (cfg.dim != p.hidden) throw std::invalid_argument("ffn_plne: layer bank width must equal gate width");
    if (cfg.amplification != amp_mode::none) throw std::invalid_argument("ffn_plne: layer banks use no amplification");
    if (context.size() != std::size_t(cfg.max_order))
        throw std::invalid_argument("hash_all_orders: context length " + std::to_string(context.size()) +
                                    " does not match max order " + std::to_string(cfg.max_order));
}

// ffn_ple's table as a base-only layer bank (max_order 1, merge scale 1, E0 = table)
device_bank table_bank(const ple_params& p) {
    ngram_config cfg;
    cfg.max_order = 1;
    cfg.sub_tables = 1;
    cfg.base_vocab = p.base_vocab;
    cfg.dim = p.hidden;
    cfg.variant = ne_variant::subtable_v2;
    cfg.amplification = amp_mode::none;
    embedding_bank host;
    host.config = cfg;
    host.base = p.table;
    return device_bank(host);
}
}  // namespace

std::vector<float> ffn_plne(std::span<const float> x, std::span<const token_id> context, const device_bank& layer_bank,
                            const ple_params& p) {
    check_layer_bank(layer_bank, p, context);
    auto h = make_plne(layer_bank, p, x);
    const auto pr = prior_tail(context.first(context.size() - 1), layer_bank.config().max_order - 1);
    const int64_t off[2] = {0, 1};
    std::vector<float> y(std::size_t(p.d_model));
    throw_status(ngram_plne_forward_host(h.get(), p.gate.data(), p.down.data(), x.data(), context.data() + context.size() - 1,
                                         off, 1, pr.empty() ? nullptr : pr.data(), y.data()));
    return y;
}

std::vector<float> ffn_plne(std::span<const float> x, std::span<const token_id> context,
                            const embedding_bank& layer_bank, const ple_params& p) {
    return ffn_plne(x, context, *device_bank_for(layer_bank), p);
}

void ffn_plne_backward(std::span<const float> x, std::span<const token_id> context, const device_bank& layer_bank,
                       const ple_params& p, std::span<const float> upstream, ple_params& grads,
                       embedding_bank& bank_grads, std::span<float> dx) {
    check_layer_bank(layer_bank, p, context);
    if (upstream.size() != std::size_t(p.d_model) || dx.size() != std::size_t(p.d_model))
        throw std::invalid_argument("ple: input/gate width mismatch");
    auto h = make_plne(layer_bank, p, x);
    ngram_grad* g = nullptr;
    throw_status(ngram_grad_create(layer_bank.handle(), &g));
    std::unique_ptr<ngram_grad, int (*)(ngram_grad*)> guard(g, ngram_grad_destroy);
    const auto pr = prior_tail(context.first(context.size() - 1), layer_bank.config().max_order - 1);
    const int64_t off[2] = {0, 1};
    throw_status(ngram_plne_backward_host(h.get(), g, p.gate.data(), p.down.data(), x.data(),
                                          context.data() + context.size() - 1, off, 1, pr.empty() ? nullptr : pr.data(),
                                          upstream.data(), grads.gate.data(), grads.down.data(), dx.data()));
    add_device_grads(g, bank_grads);
}

void ffn_plne_backward(std::span<const float> x, std::span<const token_id> context, const embedding_bank& layer_bank,
                       const ple_params& p, std::span<const float> upstream, ple_params& grads,
                       embedding_bank& bank_grads, std::span<float> dx) {
    ffn_plne_backward(x, context, *device_bank_for(layer_bank), p, upstream, grads, bank_grads, dx);
}

std::vector<float> ffn_ple(std::span<const float> x, token_id token, const ple_params& p) {
    if (std::uint64_t(token) >= p.base_vocab) throw std::out_of_range("ffn_ple: token out of range");
    const token_id ctx[1] = {token};
    return ffn_plne(x, ctx, table_bank(p), p);
}

void ffn_ple_backward(std::span<const float> x, token_id token, const ple_params& p, std::span<const float> upstream,
                      ple_params& grads, std::span<float> dx) {
    if (std::uint64_t(token) >= p.base_vocab) throw std::out_of_range("ffn_ple: token out of range");
    const device_bank bank = table_bank(p);
    embedding_bank bg;  // the base-only bank's gradient: its E0 rows are the table's
    bg.config = bank.config();
    bg.base.assign(grads.table.size(), 0.0f);
    const token_id ctx[1] = {token};
    ffn_plne_backward(x, ctx, bank, p, upstream, grads, bg, dx);
    for (std::size_t i = 0; i < grads.table.size(); ++i) grads.table[i] += bg.base[i];
}

// ============================================================== the reference's templates
// (embedding.hpp:205-459, ple.hpp:148-198) over host banks: float -> the device float path,
// double -> the device fp64 instantiation (include/ngram_b200.h, ngram_f64_*).
namespace {
struct F64View {  // C-ABI view of a host embedding_bank_t<double>
    std::string cfg;
    std::vector<const double*> sub, proj;
    explicit F64View(const embedding_bank_t<double>& b) : cfg(to_json_string(b.config)) {
        for (const auto& t : b.sub_tables) sub.push_back(t.data());
        for (const auto& w : b.projections) proj.push_back(w.data());
    }
};

void check_window(std::span<const token_id> context, const ngram_config& cfg) {
    if (context.size() != std::size_t(cfg.max_order))
        throw std::invalid_argument("hash_all_orders: context length " + std::to_string(context.size()) +
                                    " does not match max order " + std::to_string(cfg.max_order));
}

// merged (and amplified) rows of one sequence in fp64 on the device
void f64_sequence(std::span<const token_id> tokens, const embedding_bank_t<double>& bank,
                  std::span<const token_id> prior, double* merged, double* rows) {
    if (tokens.empty()) return;
    const F64View v(bank);
    throw_status(ngram_f64_forward(v.cfg.c_str(), bank.base.data(), v.sub.data(), v.proj.empty() ? nullptr : v.proj.data(),
                                   bank.ln_gain.empty() ? nullptr : bank.ln_gain.data(),
                                   bank.ln_bias.empty() ? nullptr : bank.ln_bias.data(), tokens.data(),
                                   int64_t(tokens.size()), prior.empty() ? nullptr : prior.data(), int64_t(prior.size()),
                                   merged, rows));
}

void f64_backward(std::span<const token_id> tokens, const embedding_bank_t<double>& bank,
                  std::span<const token_id> prior, const double* merged, const double* upstream,
                  embedding_bank_t<double>& grads) {
    if (tokens.empty()) return;
    const auto& cfg = bank.config;
    if (grads.base.size() != bank.base.size() || grads.sub_tables.size() != bank.sub_tables.size())
        throw std::invalid_argument("embed_backward: gradient bank shape does not match the bank");
    const F64View v(bank);
    std::vector<double*> gs, gp;
    for (auto& t : grads.sub_tables) gs.push_back(t.data());
    for (auto& w : grads.projections) gp.push_back(w.data());
    const bool ln = cfg.amplification == amp_mode::layer_norm && merged;
    throw_status(ngram_f64_backward(v.cfg.c_str(), bank.base.data(), v.sub.data(),
                                    v.proj.empty() ? nullptr : v.proj.data(),
                                    bank.ln_gain.empty() ? nullptr : bank.ln_gain.data(),
                                    bank.ln_bias.empty() ? nullptr : bank.ln_bias.data(), tokens.data(),
                                    int64_t(tokens.size()), prior.empty() ? nullptr : prior.data(),
                                    int64_t(prior.size()), merged, upstream, grads.base.data(), gs.data(),
                                    gp.empty() ? nullptr : gp.data(), ln ? grads.ln_gain.data() : nullptr,
                                    ln ? grads.ln_bias.data() : nullptr));
}

int amp_code(amp_mode m) { return m == amp_mode::none ? 0 : m == amp_mode::scale_sqrt_d ? 1 : 2; }
}  // namespace

template <typename T>
void embed_window(std::span<const token_id> context, const embedding_bank_t<T>& bank, std::span<T> out,
                  embed_counters* counters) {
    if constexpr (std::is_same_v<T, float>) {
        embed_window(context, *device_bank_for(bank), out, counters);
    } else {
        const auto& cfg = bank.config;
        check_window(context, cfg);
        if (out.size() != std::size_t(cfg.dim)) throw std::invalid_argument("embed_from_ids: output size mismatch");
        f64_sequence(context.last(1), bank, context.first(context.size() - 1), out.data(), nullptr);
        if (counters) {
            counters->table_gathers += 1 + std::uint64_t(cfg.branch_count());
            if (cfg.variant == ne_variant::subtable_v2)
                counters->projection_madds += std::uint64_t(cfg.dim) * std::uint64_t(cfg.branch_dim()) * cfg.branch_count();
        }
    }
}

template <typename T>
std::vector<T> embed_v1(std::span<const token_id> context, const embedding_bank_t<T>& bank) {
    if (bank.config.variant != ne_variant::averaged_v1) throw std::invalid_argument("embed_v1 requires the averaged variant");
    std::vector<T> out(std::size_t(bank.config.dim));
    embed_window<T>(context, bank, std::span<T>(out));
    return out;
}

template <typename T>
std::vector<T> embed_v2(std::span<const token_id> context, const embedding_bank_t<T>& bank) {
    if (bank.config.variant != ne_variant::subtable_v2) throw std::invalid_argument("embed_v2 requires the sub-table variant");
    std::vector<T> out(std::size_t(bank.config.dim));
    embed_window<T>(context, bank, std::span<T>(out));
    return out;
}

template <typename T>
sequence_embedding<T> embed_sequence_cached(std::span<const token_id> tokens, const embedding_bank_t<T>& bank,
                                            std::span<const token_id> prior_context, embed_counters* counters) {
    if constexpr (std::is_same_v<T, float>) {
        return embed_sequence_cached(tokens, *device_bank_for(bank), prior_context, counters);
    } else {
        const auto& cfg = bank.config;
        sequence_embedding<double> r;
        r.rows.resize(tokens.size() * std::size_t(cfg.dim));
        r.merged.resize(r.rows.size());
        f64_sequence(tokens, bank, prior_context, r.merged.data(), r.rows.data());
        if (counters) {
            counters->table_gathers += tokens.size() * (1 + std::uint64_t(cfg.branch_count()));
            if (cfg.variant == ne_variant::subtable_v2)
                counters->projection_madds +=
                    tokens.size() * std::uint64_t(cfg.dim) * std::uint64_t(cfg.branch_dim()) * cfg.branch_count();
        }
        return r;
    }
}

template <typename T>
std::vector<T> embed_sequence(std::span<const token_id> tokens, const embedding_bank_t<T>& bank,
                              std::span<const token_id> prior_context) {
    return embed_sequence_cached<T>(tokens, bank, prior_context).rows;
}

template <typename T>
void amplify(std::span<const T> e, amp_mode mode, std::span<const T> gain, std::span<const T> bias, std::span<T> out) {
    if constexpr (std::is_same_v<T, float>) {
        amplify(e, mode, gain, bias, out);  // the non-template float entry
    } else {
        const std::size_t D = e.size();
        if (out.size() != D) throw std::invalid_argument("amplify: output size mismatch");
        if (mode == amp_mode::layer_norm && (gain.size() != D || bias.size() != D))
            throw std::invalid_argument("amplify: layer_norm needs gain/bias of size D");
        const bool ln = mode == amp_mode::layer_norm;
        throw_status(ngram_f64_amplify(amp_code(mode), int64_t(D), ln ? gain.data() : nullptr,
                                       ln ? bias.data() : nullptr, e.data(), out.data()));
    }
}

template <typename T>
void amplify_backward(std::span<const T> pre, std::span<const T> upstream, const embedding_bank_t<T>& bank,
                      embedding_bank_t<T>& grads, std::span<T> d_pre) {
    if constexpr (std::is_same_v<T, float>) {
        amplify_backward(pre, upstream, *device_bank_for(bank), grads, d_pre);
    } else {
        const std::size_t D = std::size_t(bank.config.dim);
        if (pre.size() != D || upstream.size() != D || d_pre.size() != D)
            throw std::invalid_argument("amplify_backward: size mismatch");
        const bool ln = bank.config.amplification == amp_mode::layer_norm;
        if (ln && (grads.ln_gain.size() != D || grads.ln_bias.size() != D))
            throw std::invalid_argument("amplify_backward: gradient bank has no layer-norm parameters");
        throw_status(ngram_f64_amplify_backward(amp_code(bank.config.amplification), int64_t(D), pre.data(),
                                                upstream.data(), ln ? bank.ln_gain.data() : nullptr, d_pre.data(),
                                                ln ? grads.ln_gain.data() : nullptr, ln ? grads.ln_bias.data() : nullptr));
    }
}

template <typename T>
void embed_backward(std::span<const token_id> context, const embedding_bank_t<T>& bank, std::span<const T> upstream,
                    embedding_bank_t<T>& grads) {
    if constexpr (std::is_same_v<T, float>) {
        embed_backward(context, *device_bank_for(bank), upstream, grads);
    } else {
        if (upstream.size() != std::size_t(bank.config.dim))
            throw std::invalid_argument("embed_backward: upstream size mismatch");
        check_window(context, bank.config);
        f64_backward(context.last(1), bank, context.first(context.size() - 1), nullptr, upstream.data(), grads);
    }
}

template <typename T>
void embed_sequence_backward(std::span<const token_id> tokens, const embedding_bank_t<T>& bank,
                             std::span<const T> merged, std::span<const T> upstream, embedding_bank_t<T>& grads,
                             std::span<const token_id> prior_context) {
    if constexpr (std::is_same_v<T, float>) {
        embed_sequence_backward(tokens, *device_bank_for(bank), merged, upstream, grads, prior_context);
    } else {
        const std::size_t n = tokens.size() * std::size_t(bank.config.dim);
        if (upstream.size() != n || merged.size() != n)
            throw std::invalid_argument("embed_sequence_backward: merged / upstream size mismatch");
        f64_backward(tokens, bank, prior_context, merged.data(), upstream.data(), grads);
    }
}

template <typename T>
std::vector<T> ffn_ple(std::span<const T> x, token_id token, const ple_params_t<T>& p) {
    if constexpr (std::is_same_v<T, float>) {
        return ffn_ple(x, token, static_cast<const ple_params&>(p));
    } else {
        if (std::uint64_t(token) >= p.base_vocab) throw std::out_of_range("ffn_ple: token out of range");
        if (x.size() != std::size_t(p.d_model)) throw std::invalid_argument("ple: input/gate width mismatch");
        std::vector<double> y(std::size_t(p.d_model));
        throw_status(ngram_f64_gated_ffn(p.d_model, p.hidden, p.gate.data(), p.down.data(), x.data(),
                                         p.table.data() + std::size_t(token) * std::size_t(p.hidden), y.data()));
        return y;
    }
}

template <typename T>
void ffn_ple_backward(std::span<const T> x, token_id token, const ple_params_t<T>& p, std::span<const T> upstream,
                      ple_params_t<T>& grads, std::span<T> dx) {
    if constexpr (std::is_same_v<T, float>) {
        ffn_ple_backward(x, token, static_cast<const ple_params&>(p), upstream, static_cast<ple_params&>(grads), dx);
    } else {
        if (std::uint64_t(token) >= p.base_vocab) throw std::out_of_range("ffn_ple: token out of range");
        const std::size_t row = std::size_t(token) * std::size_t(p.hidden);
        // dL/dg accumulates straight into the table row's gradient (ple.hpp:163-165)
        throw_status(ngram_f64_gated_ffn_backward(p.d_model, p.hidden, p.gate.data(), p.down.data(), x.data(),
                                                  p.table.data() + row, upstream.data(), grads.gate.data(),
                                                  grads.down.data(), dx.data(), grads.table.data() + row));
    }
}

template <typename T>
std::vector<T> ffn_plne(std::span<const T> x, std::span<const token_id> context, const embedding_bank_t<T>& layer_bank,
                        const ple_params_t<T>& p) {
    if constexpr (std::is_same_v<T, float>) {
        return ffn_plne(x, context, static_cast<const embedding_bank&>(layer_bank), static_cast<const ple_params&>(p));
    } else {
        if (layer_bank.config.dim != p.hidden)
            throw std::invalid_argument("ffn_plne: layer bank width must equal gate width");
        if (layer_bank.config.amplification != amp_mode::none)
            throw std::invalid_argument("ffn_plne: layer banks use no amplification");
        std::vector<double> g(std::size_t(p.hidden)), y(std::size_t(p.d_model));
        embed_window<double>(context, layer_bank, std::span<double>(g));
        if (x.size() != std::size_t(p.d_model)) throw std::invalid_argument("ple: input/gate width mismatch");
        throw_status(ngram_f64_gated_ffn(p.d_model, p.hidden, p.gate.data(), p.down.data(), x.data(), g.data(),
                                         y.data()));
        return y;
    }
}

template <typename T>
void ffn_plne_backward(std::span<const T> x, std::span<const token_id> context, const embedding_bank_t<T>& layer_bank,
                       const ple_params_t<T>& p, std::span<const T> upstream, ple_params_t<T>& grads,
                       embedding_bank_t<T>& bank_grads, std::span<T> dx) {
    if constexpr (std::is_same_v<T, float>) {
        ffn_plne_backward(x, context, static_cast<const embedding_bank&>(layer_bank), static_cast<const ple_params&>(p),
                          upstream, static_cast<ple_params&>(grads), static_cast<embedding_bank&>(bank_grads), dx);
    } else {
        std::vector<double> g(std::size_t(p.hidden)), dg(std::size_t(p.hidden), 0.0);
        embed_window<double>(context, layer_bank, std::span<double>(g));
        throw_status(ngram_f64_gated_ffn_backward(p.d_model, p.hidden, p.gate.data(), p.down.data(), x.data(), g.data(),
                                                  upstream.data(), grads.gate.data(), grads.down.data(), dx.data(),
                                                  dg.data()));
        embed_backward<double>(context, layer_bank, dg, bank_grads);  // ple.hpp:196-197
    }
}

#define NGRAM_INSTANTIATE(T)                                                                                        \
    template void embed_window<T>(std::span<const token_id>, const embedding_bank_t<T>&, std::span<T>,              \
                                  embed_counters*);                                                                 \
    template std::vector<T> embed_v1<T>(std::span<const token_id>, const embedding_bank_t<T>&);                    \
    template std::vector<T> embed_v2<T>(std::span<const token_id>, const embedding_bank_t<T>&);                    \
    template sequence_embedding<T> embed_sequence_cached<T>(std::span<const token_id>, const embedding_bank_t<T>&, \
                                                            std::span<const token_id>, embed_counters*);           \
    template std::vector<T> embed_sequence<T>(std::span<const token_id>, const embedding_bank_t<T>&,               \
                                              std::span<const token_id>);                                          \
    template void amplify<T>(std::span<const T>, amp_mode, std::span<const T>, std::span<const T>, std::span<T>);   \
    template void amplify_backward<T>(std::span<const T>, std::span<const T>, const embedding_bank_t<T>&,         \
                                      embedding_bank_t<T>&, std::span<T>);                                          \
    template void embed_backward<T>(std::span<const token_id>, const embedding_bank_t<T>&, std::span<const T>,     \
                                    embedding_bank_t<T>&);                                                          \
    template void embed_sequence_backward<T>(std::span<const token_id>, const embedding_bank_t<T>&,                \
                                             std::span<const T>, std::span<const T>, embedding_bank_t<T>&,          \
                                             std::span<const token_id>);                                            \
    template std::vector<T> ffn_ple<T>(std::span<const T>, token_id, const ple_params_t<T>&);                      \
    template void ffn_ple_backward<T>(std::span<const T>, token_id, const ple_params_t<T>&, std::span<const T>,   \
                                      ple_params_t<T>&, std::span<T>);                                              \
    template std::vector<T> ffn_plne<T>(std::span<const T>, std::span<const token_id>, const embedding_bank_t<T>&, \
                                        const ple_params_t<T>&);                                                    \
    template void ffn_plne_backward<T>(std::span<const T>, std::span<const token_id>, const embedding_bank_t<T>&, \
                                       const ple_params_t<T>&, std::span<const T>, ple_params_t<T>&,               \
                                       embedding_bank_t<T>&, std::span<T>);
NGRAM_INSTANTIATE(float)
NGRAM_INSTANTIATE(double)
#undef NGRAM_INSTANTIATE

}  // namespace ngram
