// ref_shim.cpp -- extern "C" handle onto the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with the
// reference's own sources, where they lie under /root/reference/proj/src, into
// oracle/_ref/libngram_ref.so.  Nothing here re-implements reference arithmetic: every
// entry point calls the reference function named in its comment.  Used to
//   * generate tests/golden/ (tests/golden/make_golden.py),
//   * pin oracle/ngram_oracle.c against the reference (tests/test_oracle_golden.py),
//   * time the reference CPU path for bench.py --impl reference / cpu_baseline.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <functional>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ngram/analysis.hpp"
#include "ngram/cache.hpp"
#include "ngram/config.hpp"
#include "ngram/corpus.hpp"
#include "ngram/embedding.hpp"
#include "ngram/errors.hpp"
#include "ngram/hashing.hpp"
#include "ngram/ple.hpp"

using namespace ngram;

namespace {

thread_local std::string g_err;

int map_exc() {
    try {
        throw;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return -2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const parse_error& e) {
        g_err = e.what();
        return -4;
    } catch (const io_error& e) {
        g_err = e.what();
        return -3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -9;
    }
}

struct ref_bank {
    embedding_bank bank;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// config.cpp:163-183 make_default_config -> JSON (config.cpp:109-122)
int ref_make_default_config_json(uint32_t v0, int dim, int max_order, int sub_tables, char* buf, int64_t cap) {
    try {
        const auto s = to_json_string(make_default_config(v0, dim, max_order, sub_tables));
        if ((int64_t)s.size() + 1 > cap) return -1;
        std::memcpy(buf, s.c_str(), s.size() + 1);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// config.cpp:124-139 ngram_config_from_json (validates)
int ref_config_validate_json(const char* json) {
    try {
        ngram_config_from_json(json);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// hashing.cpp:33-59
int ref_rolling_hash(const uint32_t* window, int64_t len, int order, uint64_t base, uint64_t modulus, uint64_t* out) {
    try {
        *out = rolling_hash(std::span<const token_id>(window, std::size_t(len)), hash_spec{order, base, modulus});
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// Reproduces tests/test_hashing.cpp:40-57's sample stream (rng64(seed), n in 2..8,
// base < 2^17, log-uniform modulus < 2^48) and evaluates reference rolling_hash on it.
// windows: count x 8 (unused tail zero).
int ref_rolling_hash_cases(uint64_t seed, int count, int32_t* n_out, uint64_t* base_out, uint64_t* mod_out,
                           uint32_t* windows, uint64_t* hash_out) {
    try {
        rng64 rng(seed);
        for (int trial = 0; trial < count; ++trial) {
            const int n = 2 + int(uniform_below(rng, 7));
            const std::uint64_t base = 2 + uniform_below(rng, (1u << 17) - 1);
            const int bits = 1 + int(uniform_below(rng, 48));
            const std::uint64_t modulus = 1 + uniform_below(rng, (std::uint64_t(1) << bits));
            std::vector<token_id> w(static_cast<std::size_t>(n));
            for (auto& t : w) t = token_id(uniform_below(rng, base));
            n_out[trial] = n;
            base_out[trial] = base;
            mod_out[trial] = modulus;
            for (int j = 0; j < 8; ++j) windows[trial * 8 + j] = j < n ? w[std::size_t(j)] : 0u;
            hash_out[trial] = rolling_hash(w, hash_spec{n, base, modulus});
        }
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// hashing.cpp:61-81 over every position of a sequence; windows built by the
// reference's own detail::fill_context (embedding.hpp:391-405). ids: len x B.
int ref_hash_sequence(const char* cfg_json, const uint32_t* tokens, int64_t len, const uint32_t* prior,
                      int64_t prior_len, uint64_t* ids) {
    try {
        const auto cfg = ngram_config_from_json(cfg_json);
        const std::size_t B = std::size_t(cfg.branch_count());
        std::vector<token_id> ctx;
        std::span<const token_id> toks(tokens, std::size_t(len));
        std::span<const token_id> pr(prior, std::size_t(prior_len));
        for (int64_t pos = 0; pos < len; ++pos) {
            detail::fill_context(toks, std::size_t(pos), cfg.max_order, pr, ctx);
            const auto v = hash_all_orders(ctx, cfg);
            std::memcpy(ids + pos * int64_t(B), v.data(), B * sizeof(uint64_t));
        }
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// embedding.hpp:76-110 make_bank<float>; optionally bf16-round every value (RNE)
// so the bf16 device bank and this float bank hold identical numbers.
void* ref_bank_create(const char* cfg_json, uint64_t seed, int round_bf16) {
    try {
        auto cfg = ngram_config_from_json(cfg_json);
        auto rb = std::make_unique<ref_bank>();
        rb->bank = make_bank<float>(cfg, seed);
        if (round_bf16) {
            auto rnd = [](std::vector<float>& v) {
                for (auto& x : v) {
                    uint32_t u;
                    std::memcpy(&u, &x, 4);
                    u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
                    std::memcpy(&x, &u, 4);
                }
            };
            rnd(rb->bank.base);
            for (auto& t : rb->bank.sub_tables) rnd(t);
            for (auto& p : rb->bank.projections) rnd(p);
            rnd(rb->bank.ln_gain);
            rnd(rb->bank.ln_bias);
        }
        return rb.release();
    } catch (...) {
        map_exc();
        return nullptr;
    }
}

// embedding.cpp:100-140 load_bank
void* ref_bank_load(const char* path) {
    try {
        auto rb = std::make_unique<ref_bank>();
        rb->bank = load_bank(path);
        return rb.release();
    } catch (...) {
        map_exc();
        return nullptr;
    }
}

// embedding.cpp:77-98 save_bank
int ref_bank_save(void* h, const char* path) {
    try {
        save_bank(static_cast<ref_bank*>(h)->bank, path);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

void ref_bank_destroy(void* h) { delete static_cast<ref_bank*>(h); }

// Raw tensor views (row-major, embedding.hpp:31-38). which: 0 base, 1 sub[b], 2 proj[b], 3 gain, 4 bias.
const float* ref_bank_tensor(void* h, int which, int b, int64_t* numel) {
    auto& bk = static_cast<ref_bank*>(h)->bank;
    const std::vector<float>* v = nullptr;
    switch (which) {
        case 0: v = &bk.base; break;
        case 1: v = &bk.sub_tables.at(std::size_t(b)); break;
        case 2: v = &bk.projections.at(std::size_t(b)); break;
        case 3: v = &bk.ln_gain; break;
        case 4: v = &bk.ln_bias; break;
        default: return nullptr;
    }
    *numel = int64_t(v->size());
    return v->data();
}

// Overwrite the LN gain/bias (the reference tests draw them non-trivially, test_embedding.cpp:211-214).
int ref_bank_set_ln(void* h, const float* gain, const float* bias) {
    auto& bk = static_cast<ref_bank*>(h)->bank;
    if (bk.ln_gain.empty()) return -1;
    std::memcpy(bk.ln_gain.data(), gain, bk.ln_gain.size() * 4);
    std::memcpy(bk.ln_bias.data(), bias, bk.ln_bias.size() * 4);
    return 0;
}

// embedding.hpp:438-459 embed_sequence_backward<double> on bank_cast<float,double>, grads
// accumulated from zeros_like (the reference's gradient-check setup, gradcases.hpp:35-36).
// Outputs in the reference layout: base V0 x D, sub[b] V_b x d, proj[b] D x d, gain, bias.
int ref_embed_sequence_backward_f64(void* h, const uint32_t* tokens, int64_t len, const uint32_t* prior,
                                    int64_t prior_len, const double* merged, const double* upstream, double* g_base,
                                    double* const* g_sub, double* const* g_proj, double* g_gain, double* g_bias) {
    try {
        auto& bk = static_cast<ref_bank*>(h)->bank;
        const auto bd = bank_cast<float, double>(bk);
        auto g = zeros_like(bd);
        const std::size_t D = std::size_t(bk.config.dim);
        embed_sequence_backward<double>(std::span<const token_id>(tokens, std::size_t(len)), bd,
                                        std::span<const double>(merged, std::size_t(len) * D),
                                        std::span<const double>(upstream, std::size_t(len) * D), g,
                                        std::span<const token_id>(prior, std::size_t(prior_len)));
        std::memcpy(g_base, g.base.data(), g.base.size() * 8);
        for (std::size_t b = 0; b < g.sub_tables.size(); ++b)
            std::memcpy(g_sub[b], g.sub_tables[b].data(), g.sub_tables[b].size() * 8);
        for (std::size_t b = 0; b < g.projections.size(); ++b)
            std::memcpy(g_proj[b], g.projections[b].data(), g.projections[b].size() * 8);
        if (g_gain && !g.ln_gain.empty()) std::memcpy(g_gain, g.ln_gain.data(), g.ln_gain.size() * 8);
        if (g_bias && !g.ln_bias.empty()) std::memcpy(g_bias, g.ln_bias.data(), g.ln_bias.size() * 8);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// ple.hpp:168-181 ffn_plne<double> on bank_cast<float,double> (n-gram form: empty table).
static ple_params_t<double> plne_params(const double* gate, const double* down, int d_model, int hidden,
                                        std::uint32_t v0) {
    ple_params_t<double> p;
    p.d_model = d_model;
    p.hidden = hidden;
    p.base_vocab = v0;
    p.gate.assign(gate, gate + std::size_t(hidden) * std::size_t(d_model));
    p.down.assign(down, down + std::size_t(d_model) * std::size_t(hidden));
    return p;
}

int ref_ffn_plne_f64(void* h, const double* gate, const double* down, int d_model, const double* x,
                     const uint32_t* ctx, double* y) {
    try {
        auto& bk = static_cast<ref_bank*>(h)->bank;
        const auto bd = bank_cast<float, double>(bk);
        const auto p = plne_params(gate, down, d_model, bk.config.dim, bk.config.base_vocab);
        const auto r = ffn_plne<double>(std::span<const double>(x, std::size_t(d_model)),
                                        std::span<const token_id>(ctx, std::size_t(bk.config.max_order)), bd, p);
        std::memcpy(y, r.data(), r.size() * 8);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// ple.hpp:183-196 ffn_plne_backward<double>: fresh zero grads per call (ple_zeros_like,
// zeros_like), copied out in the reference layouts; dx starts at zero.
int ref_ffn_plne_backward_f64(void* h, const double* gate, const double* down, int d_model, const double* x,
                              const uint32_t* ctx, const double* up, double* g_gate, double* g_down, double* g_base,
                              double* const* g_sub, double* const* g_proj, double* dx) {
    try {
        auto& bk = static_cast<ref_bank*>(h)->bank;
        const auto bd = bank_cast<float, double>(bk);
        const auto p = plne_params(gate, down, d_model, bk.config.dim, bk.config.base_vocab);
        auto gp = ple_zeros_like(p);
        auto gb = zeros_like(bd);
        std::vector<double> d(std::size_t(d_model), 0.0);
        ffn_plne_backward<double>(std::span<const double>(x, std::size_t(d_model)),
                                  std::span<const token_id>(ctx, std::size_t(bk.config.max_order)), bd, p,
                                  std::span<const double>(up, std::size_t(d_model)), gp, gb, std::span<double>(d));
        std::memcpy(g_gate, gp.gate.data(), gp.gate.size() * 8);
        std::memcpy(g_down, gp.down.data(), gp.down.size() * 8);
        std::memcpy(g_base, gb.base.data(), gb.base.size() * 8);
        for (std::size_t b = 0; b < gb.sub_tables.size(); ++b)
            std::memcpy(g_sub[b], gb.sub_tables[b].data(), gb.sub_tables[b].size() * 8);
        for (std::size_t b = 0; b < gb.projections.size(); ++b)
            std::memcpy(g_proj[b], gb.projections[b].data(), gb.projections[b].size() * 8);
        std::memcpy(dx, d.data(), d.size() * 8);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// analysis.cpp:44-176: corpus_analyzer over the batch (add_sequence per sequence, the error of
// a bad token caught), then stats().  meta: [sequences, tokens]; seen / distinct [n_orders];
// buckets [n_orders][n_moduli].  Returns the add's status (-2 = out_of_range) after filling
// the stats, or the constructor's error.
int ref_corpus_analyze(uint64_t v0, const int* orders, int n_orders, const uint64_t* moduli, int n_moduli,
                       const uint32_t* tokens, const int64_t* off, int64_t nseq, uint64_t* meta, uint64_t* seen,
                       uint64_t* distinct, uint64_t* buckets) {
    try {
        corpus_analyzer an(v0, std::vector<int>(orders, orders + n_orders),
                           std::vector<std::uint64_t>(moduli, moduli + n_moduli));
        int rc = 0;
        try {
            for (int64_t s = 0; s < nseq; ++s)
                an.add_sequence(std::span<const token_id>(tokens + off[s], std::size_t(off[s + 1] - off[s])));
        } catch (...) {
            rc = map_exc();
        }
        const auto st = an.stats();
        meta[0] = st.sequences_seen;
        meta[1] = st.tokens_seen;
        for (int i = 0; i < n_orders; ++i) {
            seen[i] = st.ngrams_seen.at(orders[i]);
            distinct[i] = st.distinct_ngrams.at(orders[i]);
            for (int j = 0; j < n_moduli; ++j)
                buckets[i * n_moduli + j] = st.distinct_buckets.at({orders[i], moduli[j]});
        }
        return rc;
    } catch (...) {
        return map_exc();
    }
}

// corpus.cpp:211-271 generate_zipf_markov: sequences x seq_len tokens, row-major.
int ref_generate_zipf_markov(uint32_t vocab, int64_t sequences, int64_t seq_len, uint64_t seed, double exponent,
                             double markov_prob, uint32_t* out) {
    try {
        const auto c = generate_zipf_markov(vocab, std::size_t(sequences), std::size_t(seq_len), seed, exponent,
                                            markov_prob);
        for (std::size_t s = 0; s < c.size(); ++s)
            std::memcpy(out + s * std::size_t(seq_len), c[s].data(), c[s].size() * 4);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// embedding.hpp:409-429 embed_sequence_cached<float>: rows (amplified) and merged.
int ref_embed_sequence_f32(void* h, const uint32_t* tokens, int64_t len, const uint32_t* prior, int64_t prior_len,
                           float* rows, float* merged) {
    try {
        auto& bk = static_cast<ref_bank*>(h)->bank;
        auto r = embed_sequence_cached<float>(std::span<const token_id>(tokens, std::size_t(len)), bk,
                                              std::span<const token_id>(prior, std::size_t(prior_len)));
        if (rows) std::memcpy(rows, r.rows.data(), r.rows.size() * 4);
        if (merged) std::memcpy(merged, r.merged.data(), r.merged.size() * 4);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// Same in double on bank_cast<float,double> (embedding.hpp:140-156): the tolerance reference.
int ref_embed_sequence_f64(void* h, const uint32_t* tokens, int64_t len, const uint32_t* prior, int64_t prior_len,
                           double* rows, double* merged) {
    try {
        auto& bk = static_cast<ref_bank*>(h)->bank;
        const auto bd = bank_cast<float, double>(bk);
        auto r = embed_sequence_cached<double>(std::span<const token_id>(tokens, std::size_t(len)), bd,
                                               std::span<const token_id>(prior, std::size_t(prior_len)));
        if (rows) std::memcpy(rows, r.rows.data(), r.rows.size() * 8);
        if (merged) std::memcpy(merged, r.merged.data(), r.merged.size() * 8);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// embed_sequence_cached<double> (embedding.hpp:409-429) evaluated at selected positions of a
// batch, the bank cast to double ONCE (a LongCat/config-B-size bank is ~9 GB in float): position
// p of sequence s is the single-token call on tokens[p] with prior_context = the (up to) N-1
// tokens of s before p -- the same window fill_context builds for p in the whole-sequence call
// (embedding.hpp:391-405).  positions: global indices into tokens; rows / merged: npos x D.
int ref_embed_positions_f64(void* h, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                            const int64_t* positions, int64_t npos, double* rows, double* merged) {
    try {
        auto& bk = static_cast<ref_bank*>(h)->bank;
        const auto bd = bank_cast<float, double>(bk);
        const int64_t D = bk.config.dim, ctx = bk.config.max_order - 1;
        for (int64_t i = 0; i < npos; ++i) {
            const int64_t p = positions[i];
            int64_t s = 0;
            while (s + 1 < nseq && seq_offsets[s + 1] <= p) ++s;
            const int64_t a = std::max(seq_offsets[s], p - ctx);
            auto r = embed_sequence_cached<double>(std::span<const token_id>(tokens + p, 1), bd,
                                                   std::span<const token_id>(tokens + a, std::size_t(p - a)));
            if (rows) std::memcpy(rows + i * D, r.rows.data(), std::size_t(D) * 8);
            if (merged) std::memcpy(merged + i * D, r.merged.data(), std::size_t(D) * 8);
        }
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// The reference CPU path run over a batch of sequences, one sequence per std::thread
// (embed_sequence is pure and the bank read-only). Used as the
// timed CPU baseline. seq_offsets: nseq+1 prefix offsets into tokens; rows: total x D.
int ref_embed_batch_mt(void* h, const uint32_t* tokens, const int64_t* seq_offsets, int nseq, int nthreads,
                       float* rows) {
    auto& bk = static_cast<ref_bank*>(h)->bank;
    const int64_t D = bk.config.dim;
    std::vector<std::thread> pool;
    std::vector<int> rc(std::size_t(nseq), 0);
    std::atomic<int> next{0};
    if (nthreads < 1) nthreads = 1;
    for (int w = 0; w < nthreads; ++w) {
        pool.emplace_back([&]() {
            for (;;) {
                const int s = next.fetch_add(1);
                if (s >= nseq) return;
                try {
                    const int64_t a = seq_offsets[s], b = seq_offsets[s + 1];
                    const auto r = embed_sequence<float>(std::span<const token_id>(tokens + a, std::size_t(b - a)), bk);
                    std::memcpy(rows + a * D, r.data(), r.size() * 4);
                } catch (...) {
                    rc[std::size_t(s)] = -1;
                }
            }
        });
    }
    for (auto& t : pool) t.join();
    for (int x : rc)
        if (x) return x;
    return 0;
}

// --- cache.cpp ---------------------------------------------------------------
void* ref_cache_create(const char* cfg_json) {
    try {
        return new sequence_cache(ngram_config_from_json(cfg_json));
    } catch (...) {
        map_exc();
        return nullptr;
    }
}
void ref_cache_destroy(void* h) { delete static_cast<sequence_cache*>(h); }

// cache.cpp:37-57
int ref_cache_append(void* h, uint32_t token, uint64_t* ids) {
    try {
        const auto v = static_cast<sequence_cache*>(h)->append(token);
        std::memcpy(ids, v.data(), v.size() * 8);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_cache_ring(void* h, uint32_t* ring, uint64_t* length, uint32_t* last) {
    auto* c = static_cast<sequence_cache*>(h);
    const auto r = c->ring();
    std::memcpy(ring, r.data(), r.size() * 4);
    *length = c->length();
    *last = c->last_token();
    return int(r.size());
}

// cache.cpp:152-195 draft_verify with a fresh memo of `memo_capacity`: accepted merged
// vectors (accept x D) and counters (8 x u64, cache.hpp:17-26 order).
int ref_draft_verify(void* cache, void* bank, const uint32_t* draft, int64_t len, int64_t accept, int64_t memo_capacity,
                     int conventional, float* accepted, uint64_t* counters) {
    try {
        auto& bk = static_cast<ref_bank*>(bank)->bank;
        embedding_memo memo{static_cast<std::size_t>(memo_capacity)};
        cache_counters c;
        draft_options opts;
        opts.conventional_draft_embedding = conventional != 0;
        const auto r = draft_verify(*static_cast<sequence_cache*>(cache), memo, bk,
                                    std::span<const token_id>(draft, std::size_t(len)), std::size_t(accept), &c, opts);
        const std::size_t D = std::size_t(bk.config.dim);
        for (std::size_t i = 0; i < r.accepted.size(); ++i) std::memcpy(accepted + i * D, r.accepted[i].data(), D * 4);
        const uint64_t cv[8] = {c.appends,          c.rollbacks,        c.memo_hits,           c.memo_misses,
                                c.table_gathers,    c.projection_madds, c.draft_table_gathers, c.verify_table_gathers};
        std::memcpy(counters, cv, sizeof(cv));
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// --- CPU baselines for the decode / verify workloads and the index stage -------------
// (bench.py cpu_baseline of configs D / E and of hash_all_orders alone; BASELINE.md "CPU
// baseline plan").  Every stream owns a sequence_cache and an embedding_memo; streams are
// independent, so they are spread over `nthreads` std::threads.  The reference calls are
// the stock ones:
//   mode 0 (decode step, config D):  ids = sequence_cache::append(t) (cache.cpp:37-57),
//                                    e = embedding_memo::lookup(t, ids, bank) (cache.cpp:123-150)
//   mode 1 (verify block, config E): draft_verify(state, memo, bank, draft[L], accept)
//                                    (cache.cpp:152-195)
// prior: [nstreams][prior_len] tokens appended first (the prefill hand-off); tokens:
// [nstreams][steps * L]; accept: [nstreams][steps] (mode 1).  last_out: [nstreams][D], the
// last merged vector each stream produced (so the work cannot be optimised away).
int ref_decode_mt(void* bank, int mode, int nstreams, int nthreads, const uint32_t* prior, int prior_len,
                  const uint32_t* tokens, int steps, int L, const int32_t* accept, int64_t memo_capacity,
                  float* last_out) {
    auto& bk = static_cast<ref_bank*>(bank)->bank;
    const std::size_t D = std::size_t(bk.config.dim);
    std::vector<int> rc(std::size_t(nstreams), 0);
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    if (nthreads < 1) nthreads = 1;
    const int per = mode == 0 ? steps : steps * L;
    for (int w = 0; w < nthreads; ++w) {
        pool.emplace_back([&]() {
            for (;;) {
                const int s = next.fetch_add(1);
                if (s >= nstreams) return;
                try {
                    sequence_cache state(bk.config);
                    embedding_memo memo{std::size_t(memo_capacity)};
                    for (int i = 0; i < prior_len; ++i) state.append(prior[std::size_t(s) * prior_len + i]);
                    const uint32_t* tk = tokens + std::size_t(s) * std::size_t(per);
                    std::vector<float> last(D, 0.0f);
                    if (mode == 0) {
                        for (int i = 0; i < steps; ++i) {
                            const auto ids = state.append(tk[i]);
                            last = memo.lookup(tk[i], ids, bk);
                        }
                    } else {
                        for (int r = 0; r < steps; ++r) {
                            const auto res = draft_verify(state, memo, bk,
                                                          std::span<const token_id>(tk + std::size_t(r) * L, std::size_t(L)),
                                                          std::size_t(accept[std::size_t(s) * steps + r]));
                            if (!res.accepted.empty()) last = res.accepted.back();
                        }
                    }
                    std::memcpy(last_out + std::size_t(s) * D, last.data(), D * 4);
                } catch (...) {
                    rc[std::size_t(s)] = map_exc();
                }
            }
        });
    }
    for (auto& t : pool) t.join();
    for (int x : rc)
        if (x) return x;
    return 0;
}

// hashing.cpp:61-81 hash_all_orders over every position of `len` tokens (one zero-padded
// sequence; windows via corpus.cpp:273-280 window_at), positions split over nthreads.
// ids: len x branch_count.
int ref_hash_all_orders_mt(const char* cfg_json, const uint32_t* tokens, int64_t len, int nthreads, uint64_t* ids) {
    try {
        const auto cfg = ngram_config_from_json(cfg_json);
        const std::vector<token_id> seq(tokens, tokens + len);
        const std::size_t nb = std::size_t(cfg.branch_count());
        std::vector<std::thread> pool;
        std::vector<int> rc(std::size_t(std::max(nthreads, 1)), 0);
        if (nthreads < 1) nthreads = 1;
        for (int w = 0; w < nthreads; ++w) {
            pool.emplace_back([&, w]() {
                try {
                    std::vector<token_id> window;
                    const int64_t a = len * w / nthreads, b = len * (w + 1) / nthreads;
                    for (int64_t p = a; p < b; ++p) {
                        window_at(seq, std::size_t(p), cfg.max_order, window);
                        const auto v = hash_all_orders(window, cfg);
                        std::memcpy(ids + std::size_t(p) * nb, v.data(), nb * 8);
                    }
                } catch (...) {
                    rc[std::size_t(w)] = map_exc();
                }
            });
        }
        for (auto& t : pool) t.join();
        for (int x : rc)
            if (x) return x;
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// Per-call latency of the reference's one-token entries on one host thread (ns per call, median
// of `reps` timed batches of 16 calls): rolling_hash (order 3), hash_all_orders,
// sequence_cache::append, embedding_memo::lookup (a miss: embed_from_ids), draft_verify (4 drafts,
// accept 2).  out: 5 doubles.  bench.py --workload dropin (the drop-in's per-call latency beside it).
int ref_time_calls(void* bank, int reps, double* out) {
    try {
        auto& bk = static_cast<ref_bank*>(bank)->bank;
        const auto& cfg = bk.config;
        auto med = [&](const std::function<void()>& f) {
            for (int i = 0; i < 3; ++i) f();
            std::vector<double> t;
            for (int r = 0; r < reps; ++r) {
                const auto a = std::chrono::steady_clock::now();
                for (int i = 0; i < 16; ++i) f();
                t.push_back(std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - a).count() / 16);
            }
            std::sort(t.begin(), t.end());
            return t[t.size() / 2];
        };
        std::vector<token_id> ctx{5, 6, 7, 8};
        ctx.resize(std::size_t(cfg.max_order), 1);
        volatile uint64_t sink = 0;
        sequence_cache st(cfg);
        embedding_memo memo(1);  // capacity 1: every lookup of a new key is a miss (embed_from_ids)
        token_id tk = 1;
        out[0] = med([&] { sink = sink + rolling_hash(std::span<const token_id>(ctx).last(2), {2, cfg.base_vocab, 997}); });
        out[1] = med([&] { sink = sink + hash_all_orders(ctx, cfg)[0]; });
        out[2] = med([&] { sink = sink + st.append(tk = (tk * 7 + 3) % cfg.base_vocab)[0]; });
        out[3] = med([&] {
            tk = (tk * 7 + 3) % cfg.base_vocab;
            const auto ids = st.append(tk);
            sink = sink + uint64_t(memo.lookup(tk, ids, bk)[0] != 0.0f);
        });
        std::vector<token_id> draft{3, 1, 4, 1};
        out[4] = med([&] { sink = sink + draft_verify(st, memo, bk, draft, 2).accepted.size(); });
        return 0;
    } catch (...) {
        return map_exc();
    }
}

}  // extern "C"
