// embedding.hpp -- drop-in for proj/include/ngram/embedding.hpp (hot-path parts).
//
// embedding_bank_t<T> stays the reference's host-side parameter store (same layout,
// same make_bank RNG order -> bit-identical banks).  The forward runs on the GPU:
// a device_bank holds the B200 layout (bf16 tables, W_cat, E0) and every embed_* call
// goes through the C-ABI (no CPU fallback).  The overloads taking a host
// embedding_bank_t<float> keep reference call sites compiling: they upload to a
// transient device_bank per call (convenience for small banks); production code keeps
// a device_bank.
#pragma once
#include <cmath>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "ngram/config.hpp"
#include "ngram/errors.hpp"
#include "ngram/hashing.hpp"
#include "ngram/rng.hpp"

struct ngram_bank;

namespace ngram {

struct embed_counters {
    std::uint64_t table_gathers = 0;
    std::uint64_t projection_madds = 0;
};

template <typename T>
struct embedding_bank_t {
    ngram_config config;
    std::vector<T> base;
    std::vector<std::vector<T>> sub_tables;
    std::vector<std::vector<T>> projections;
    std::vector<T> ln_gain;
    std::vector<T> ln_bias;

    std::span<const T> base_row(token_id t) const {
        if (std::uint64_t(t) >= config.base_vocab)
            throw std::out_of_range("embedding: token " + std::to_string(t) + " out of range for base vocabulary " +
                                    std::to_string(config.base_vocab));
        return std::span<const T>(base).subspan(std::size_t(t) * std::size_t(config.dim), std::size_t(config.dim));
    }
    std::span<T> base_row(token_id t) {
        auto r = static_cast<const embedding_bank_t&>(*this).base_row(t);
        return {const_cast<T*>(r.data()), r.size()};
    }
    std::span<const T> sub_row(int branch, std::uint64_t bucket) const {
        const auto& table = sub_tables.at(std::size_t(branch));
        const std::size_t w = std::size_t(config.branch_dim());
        if ((bucket + 1) * w > table.size())
            throw std::out_of_range("embedding: bucket " + std::to_string(bucket) + " out of range for sub-table " +
                                    std::to_string(branch));
        return std::span<const T>(table).subspan(std::size_t(bucket) * w, w);
    }
    std::span<T> sub_row(int branch, std::uint64_t bucket) {
        auto r = static_cast<const embedding_bank_t&>(*this).sub_row(branch, bucket);
        return {const_cast<T*>(r.data()), r.size()};
    }
};

using embedding_bank = embedding_bank_t<float>;

// make_bank (embedding.hpp:76-110): identical RNG consumption order.
template <typename T>
embedding_bank_t<T> make_bank(const ngram_config& cfg, std::uint64_t seed) {
    cfg.validate();
    embedding_bank_t<T> bank;
    bank.config = cfg;
    rng64 g(seed);
    const std::size_t D = std::size_t(cfg.dim), d = std::size_t(cfg.branch_dim());
    bank.base.resize(std::size_t(cfg.base_vocab) * D);
    for (auto& x : bank.base) x = T(0.02 * gaussian(g));
    const int B = cfg.branch_count();
    bank.sub_tables.resize(std::size_t(B));
    bank.projections.resize(cfg.variant == ne_variant::subtable_v2 ? std::size_t(B) : 0);
    for (int n = 2; n <= cfg.max_order; ++n)
        for (int k = 1; k <= cfg.sub_tables; ++k) {
            const int b = cfg.branch_index(n, k);
            auto& tab = bank.sub_tables[std::size_t(b)];
            tab.resize(std::size_t(cfg.vocab_of(n, k)) * d);
            for (auto& x : tab) x = T(0.02 * gaussian(g));
            if (cfg.variant == ne_variant::subtable_v2) {
                auto& p = bank.projections[std::size_t(b)];
                p.resize(D * d);
                const double sigma = 0.02 / std::sqrt(double(d));
                for (auto& x : p) x = T(sigma * gaussian(g));
            }
        }
    if (cfg.amplification == amp_mode::layer_norm) {
        bank.ln_gain.assign(D, T(1));
        bank.ln_bias.assign(D, T(0));
    }
    return bank;
}

template <typename T>
embedding_bank_t<T> make_zero_bank(const ngram_config& cfg) {
    auto bank = make_bank<T>(cfg, 0);
    for (auto* v : {&bank.base}) std::fill(v->begin(), v->end(), T(0));
    for (auto& t : bank.sub_tables) std::fill(t.begin(), t.end(), T(0));
    for (auto& p : bank.projections) std::fill(p.begin(), p.end(), T(0));
    return bank;
}

// The B200-resident bank (include/ngram_b200.h, ngram_bank).
class device_bank {
  public:
    explicit device_bank(const ngram_config& cfg, int device = 0, int shard_rank = 0, int shard_count = 1);
    explicit device_bank(const embedding_bank& host, int device = 0);  // upload (f32 -> bf16)
    static device_bank from_file(const std::string& path, const ngram_config& cfg, int device = 0);  // save_bank format
    void upload(const embedding_bank& host);
    void generate(std::uint64_t seed);  // synthetic LongCat-scale tables, on device
    const ngram_config& config() const { return cfg_; }
    ngram_bank* handle() const { return h_.get(); }
    bool tensor_core_path() const;

    const std::shared_ptr<ngram_bank>& shared_handle() const { return h_; }

  private:
    ngram_config cfg_;
    std::shared_ptr<ngram_bank> h_;
};

// The device copy of a host bank, cached across calls: keyed by the bank's address and a
// 64-bit fingerprint of its contents, so a bank edited in place between calls is re-uploaded
// and an unchanged one is not.  Every embedding_bank overload below goes through it.
std::shared_ptr<const device_bank> device_bank_for(const embedding_bank& host);

// embed_from_ids (embedding.hpp:163-201): merged, pre-amplification.
void embed_from_ids(token_id token, std::span<const std::uint64_t> ids, const device_bank& bank, std::span<float> out,
                    embed_counters* counters = nullptr);
void embed_from_ids(token_id token, std::span<const std::uint64_t> ids, const embedding_bank& bank,
                    std::span<float> out, embed_counters* counters = nullptr);
// The reference's template form (embed_from_ids<float>(...), embedding.hpp:163): float banks
// run on the device; the double instantiation of the reference is a CPU gradient-check tool
// and has no device path here.
template <typename T>
void embed_from_ids(token_id token, std::span<const std::uint64_t> ids, const embedding_bank_t<T>& bank,
                    std::span<T> out, embed_counters* counters = nullptr) {
    static_assert(std::is_same_v<T, float>, "device embeddings are computed from float banks");
    embed_from_ids(token, ids, static_cast<const embedding_bank&>(bank), out, counters);
}

// embed_window / embed_v1 / embed_v2 (embedding.hpp:205-237): merged embedding of one window.
void embed_window(std::span<const token_id> context, const device_bank& bank, std::span<float> out,
                  embed_counters* counters = nullptr);
std::vector<float> embed_v1(std::span<const token_id> context, const device_bank& bank);
std::vector<float> embed_v2(std::span<const token_id> context, const device_bank& bank);

template <typename T>
struct sequence_embedding {
    std::vector<T> rows;    // len x D, amplified
    std::vector<T> merged;  // len x D, before amplification
};

// embed_sequence(_cached) (embedding.hpp:409-436).
sequence_embedding<float> embed_sequence_cached(std::span<const token_id> tokens, const device_bank& bank,
                                                std::span<const token_id> prior_context = {},
                                                embed_counters* counters = nullptr);
std::vector<float> embed_sequence(std::span<const token_id> tokens, const device_bank& bank,
                                  std::span<const token_id> prior_context = {});
sequence_embedding<float> embed_sequence_cached(std::span<const token_id> tokens, const embedding_bank& bank,
                                                std::span<const token_id> prior_context = {},
                                                embed_counters* counters = nullptr);
std::vector<float> embed_sequence(std::span<const token_id> tokens, const embedding_bank& bank,
                                  std::span<const token_id> prior_context = {});

// Batched extension: many sequences in one launch (rows concatenated, len_total x D).
std::vector<float> embed_batch(const std::vector<std::vector<token_id>>& sequences, const device_bank& bank);

// ---- the reference's template entry points over host banks (embedding.hpp:205-459) ----------
// T = float runs the device float path on the bank's cached device copy (device_bank_for);
// T = double runs the device fp64 instantiation (ngram_f64_*, include/ngram_b200.h) -- the
// precision the reference's own gradient checks use.  Explicitly instantiated for float and
// double in libngram.so.
template <typename T>
std::vector<T> embed_v1(std::span<const token_id> context, const embedding_bank_t<T>& bank);
template <typename T>
std::vector<T> embed_v2(std::span<const token_id> context, const embedding_bank_t<T>& bank);
template <typename T>
void embed_window(std::span<const token_id> context, const embedding_bank_t<T>& bank, std::span<T> out,
                  embed_counters* counters = nullptr);
template <typename T>
sequence_embedding<T> embed_sequence_cached(std::span<const token_id> tokens, const embedding_bank_t<T>& bank,
                                            std::span<const token_id> prior_context = {},
                                            embed_counters* counters = nullptr);
template <typename T>
std::vector<T> embed_sequence(std::span<const token_id> tokens, const embedding_bank_t<T>& bank,
                              std::span<const token_id> prior_context = {});
template <typename T>
void amplify(std::span<const T> e, amp_mode mode, std::span<const T> gain, std::span<const T> bias, std::span<T> out);
template <typename T>
std::vector<T> amplify(std::span<const T> e, const embedding_bank_t<T>& bank) {
    std::vector<T> out(e.size());
    amplify<T>(e, bank.config.amplification, bank.ln_gain, bank.ln_bias, std::span<T>(out));
    return out;
}
template <typename T>
void amplify_backward(std::span<const T> pre, std::span<const T> upstream, const embedding_bank_t<T>& bank,
                      embedding_bank_t<T>& grads, std::span<T> d_pre);
template <typename T>
void embed_backward(std::span<const token_id> context, const embedding_bank_t<T>& bank,
                    std::span<const T> upstream, embedding_bank_t<T>& grads);
template <typename T>
void embed_sequence_backward(std::span<const token_id> tokens, const embedding_bank_t<T>& bank,
                             std::span<const T> merged, std::span<const T> upstream, embedding_bank_t<T>& grads,
                             std::span<const token_id> prior_context = {});

// ---- parameter accounting (embedding.hpp:461-484, embedding.cpp:13-56): host arithmetic
struct param_count_report {
    std::uint64_t base = 0;
    std::uint64_t sub_tables = 0;
    std::uint64_t projections = 0;
    std::uint64_t total = 0;
};
param_count_report param_count(const ngram_config& cfg);

struct budget_info {
    std::uint64_t embedding_params = 0;
    std::uint64_t other_params = 0;
    double fraction = 0.0;     // embedding / (embedding + other)
    bool over_budget = false;  // fraction strictly above 1/2
};
budget_info budget_report(std::uint64_t embedding_params, std::uint64_t other_params);
budget_info budget_report(const ngram_config& cfg, std::uint64_t other_params);
std::string budget_guidance(const budget_info& info);

// ---- serialization (embedding.hpp:486-493): the reference's single-file format (u32 LE
// header length, JSON config, raw LE f32 tensors).  A device_bank reads the same file with
// device_bank::from_file (streamed f32 -> bf16 on the GPU).
void save_bank(const embedding_bank& bank, const std::string& path);
embedding_bank load_bank(const std::string& path);

// bank_cast (embedding.hpp:140-156): element-wise conversion of a host bank.
template <typename From, typename To>
embedding_bank_t<To> bank_cast(const embedding_bank_t<From>& bank) {
    auto conv = [](const std::vector<From>& v) { return std::vector<To>(v.begin(), v.end()); };
    embedding_bank_t<To> out;
    out.config = bank.config;
    out.base = conv(bank.base);
    for (const auto& t : bank.sub_tables) out.sub_tables.push_back(conv(t));
    for (const auto& p : bank.projections) out.projections.push_back(conv(p));
    out.ln_gain = conv(bank.ln_gain);
    out.ln_bias = conv(bank.ln_bias);
    return out;
}

// amplify (embedding.hpp:239-287) of one merged row, on the device (float).
void amplify(std::span<const float> e, amp_mode mode, std::span<const float> gain, std::span<const float> bias,
             std::span<float> out);

// zeros_like (embedding.hpp:123-134): a zero bank of the same shape (the gradient store).
template <typename T>
embedding_bank_t<T> zeros_like(const embedding_bank_t<T>& bank) {
    embedding_bank_t<T> z;
    z.config = bank.config;
    z.base.assign(bank.base.size(), T(0));
    for (const auto& t : bank.sub_tables) z.sub_tables.emplace_back(t.size(), T(0));
    for (const auto& p : bank.projections) z.projections.emplace_back(p.size(), T(0));
    z.ln_gain.assign(bank.ln_gain.size(), T(0));
    z.ln_bias.assign(bank.ln_bias.size(), T(0));
    return z;
}

// amplify_backward (embedding.hpp:291-336) of one row, on the device: d_pre from the
// amplification input `pre` and `upstream`; layer_norm accumulates grads.ln_gain / ln_bias.
void amplify_backward(std::span<const float> pre, std::span<const float> upstream, const device_bank& bank,
                      embedding_bank& grads, std::span<float> d_pre);
void amplify_backward(std::span<const float> pre, std::span<const float> upstream, const embedding_bank& bank,
                      embedding_bank& grads, std::span<float> d_pre);

// Backward (embedding.hpp:338-459), computed on the device (ngram_embed_backward_host:
// fp32 atomics + fp32 GEMMs) and ACCUMULATED into the host gradient bank `grads`.
// embed_backward: `upstream` is d(merged) of one window (no amplification step).
void embed_backward(std::span<const token_id> context, const device_bank& bank, std::span<const float> upstream,
                    embedding_bank& grads);
void embed_backward(std::span<const token_id> context, const embedding_bank& bank, std::span<const float> upstream,
                    embedding_bank& grads);
// embed_sequence_backward: `merged` = embed_sequence_cached(...).merged, `upstream` = dL/d(rows).
void embed_sequence_backward(std::span<const token_id> tokens, const device_bank& bank, std::span<const float> merged,
                             std::span<const float> upstream, embedding_bank& grads,
                             std::span<const token_id> prior_context = {});
void embed_sequence_backward(std::span<const token_id> tokens, const embedding_bank& bank,
                             std::span<const float> merged, std::span<const float> upstream, embedding_bank& grads,
                             std::span<const token_id> prior_context = {});

}  // namespace ngram
