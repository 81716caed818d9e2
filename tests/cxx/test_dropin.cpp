// test_dropin.cpp -- the reference's own test cases (proj/tests/test_hashing.cpp,
// test_embedding.cpp, test_cache.cpp), rewritten against the DROP-IN headers
// include/ngram/*.hpp: same calls, same expected values / exceptions, executed on the
// GPU through libngram.so -> libngram_b200.so.  Built by paper_2601_21204_b200/build.py,
// run by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "ngram/analysis.hpp"
#include "ngram/cache.hpp"
#include "ngram/config.hpp"
#include "ngram/embedding.hpp"
#include "ngram/ple.hpp"
#include "ngram/hashing.hpp"

using namespace ngram;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                  \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(c)) {                                                               \
            ++g_fail;                                                             \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);              \
        }                                                                         \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                  \
    do {                                                                          \
        ++g_checks;                                                               \
        bool ok = false;                                                          \
        try {                                                                     \
            (void)(expr);                                                         \
        } catch (const T&) {                                                      \
            ok = true;                                                            \
        } catch (...) {                                                           \
        }                                                                         \
        if (!ok) {                                                                \
            ++g_fail;                                                             \
            std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
        }                                                                         \
    } while (0)

static void test_case(const char* name, const std::function<void()>& f) {
    const int before = g_fail;
    try {
        f();
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("FAIL %s: unexpected exception %s\n", name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name);
}

static ngram_config v2_config(std::uint32_t v0, int dim, int order, int k, amp_mode amp = amp_mode::none) {
    ngram_config cfg;
    cfg.max_order = order;
    cfg.sub_tables = k;
    cfg.base_vocab = v0;
    cfg.dim = dim;
    cfg.variant = ne_variant::subtable_v2;
    cfg.amplification = amp;
    for (int n = 2; n <= order; ++n)
        for (int kk = 1; kk <= k; ++kk) cfg.sub_vocab[{n, kk}] = 13 + 8 * std::uint64_t(n) + 3 * std::uint64_t(kk);
    cfg.validate();
    return cfg;
}

static bool close_rows(const std::vector<float>& a, const std::vector<float>& b, double tol = 1e-5) {
    if (a.size() != b.size()) return false;
    double mx = 0, err = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        mx = std::max(mx, std::fabs(double(b[i])));
        err = std::max(err, std::fabs(double(a[i]) - double(b[i])));
    }
    return err <= tol * (mx + 1e-30);
}

// test_analysis.cpp:18-48: two-pass set oracle and random corpora (the reference's bigint
// polynomial hash is exact here in 128 bits: V0 < 2^8, order <= 4).
struct two_pass_counts {
    std::uint64_t ngrams = 0, buckets = 0;
};

static two_pass_counts two_pass(const std::vector<token_sequence>& corpus, std::uint64_t v0, int order,
                                std::uint64_t m) {
    std::set<std::vector<token_id>> ng;
    std::set<std::uint64_t> bk;
    std::vector<token_id> w;
    for (const auto& seq : corpus)
        for (std::size_t pos = 0; pos < seq.size(); ++pos) {
            window_at(seq, pos, order, w);
            ng.insert(w);
            unsigned __int128 h = 0;
            for (const token_id t : w) h = h * v0 + t;
            bk.insert(std::uint64_t(h % m));
        }
    return {ng.size(), bk.size()};
}

static std::vector<token_sequence> random_corpus(rng64& rng, std::uint32_t v0, std::size_t seqs, std::size_t max_len) {
    std::vector<token_sequence> c(seqs);
    for (auto& q : c) {
        q.resize(1 + uniform_below(rng, max_len));
        for (auto& t : q) t = token_id(uniform_below(rng, v0));
    }
    return c;
}

int main() {
    test_case("rolling_hash worked examples", [] {  // test_hashing.cpp:12-26
        std::vector<token_id> w{3, 5};
        CHECK(rolling_hash(w, {2, 10, 7}) == 0);
        std::vector<token_id> zeros(5, 0);
        CHECK(rolling_hash(zeros, {5, 1000, 12345}) == 0);
        CHECK(rolling_hash(std::span(zeros).first(2), {2, 7, 3}) == 0);
        std::vector<token_id> padded{0, 0, 7};
        CHECK(rolling_hash(padded, {3, 128000, 13}) == 7);
    });
    test_case("rolling_hash input validation", [] {  // test_hashing.cpp:28-38
        std::vector<token_id> w{1, 2, 3};
        CHECK_THROWS_AS(rolling_hash(w, {2, 10, 7}), std::invalid_argument);
        CHECK_THROWS_AS(rolling_hash(w, {4, 10, 7}), std::invalid_argument);
        std::vector<token_id> oob{1, 12};
        CHECK_THROWS_AS(rolling_hash(oob, {2, 10, 7}), std::out_of_range);
        CHECK_THROWS_AS(rolling_hash(w, {3, 1, 7}), std::invalid_argument);
        CHECK_THROWS_AS(rolling_hash(w, {3, 10, 0}), std::invalid_argument);
        std::vector<token_id> one{5};
        CHECK_THROWS_AS(rolling_hash(one, {1, 10, 7}), std::invalid_argument);
    });
    test_case("hash_all_orders worked example", [] {  // test_hashing.cpp:83-101
        ngram_config cfg;
        cfg.max_order = 3;
        cfg.sub_tables = 1;
        cfg.base_vocab = 16;
        cfg.dim = 4;
        cfg.variant = ne_variant::averaged_v1;
        cfg.sub_vocab[{2, 1}] = 101;
        cfg.sub_vocab[{3, 1}] = 103;
        std::vector<token_id> ctx{0, 4, 9};
        const auto ids = hash_all_orders(ctx, cfg);
        CHECK(ids.size() == 2);
        CHECK(ids[std::size_t(cfg.branch_index(2, 1))] == 73);
        CHECK(ids[std::size_t(cfg.branch_index(3, 1))] == 73);
        std::vector<token_id> zeros{0, 0, 0};
        for (auto id : hash_all_orders(zeros, cfg)) CHECK(id == 0);
    });
    test_case("hash_all_orders matches per-window rolling_hash", [] {  // test_hashing.cpp:122-138
        ngram_config cfg = make_default_config(50, 24, 4, 2);
        rng64 rng(99);
        for (int trial = 0; trial < 50; ++trial) {
            std::vector<token_id> ctx(4);
            for (auto& t : ctx) t = token_id(uniform_below(rng, 50));
            const auto ids = hash_all_orders(ctx, cfg);
            for (int n = 2; n <= 4; ++n)
                for (int k = 1; k <= 2; ++k)
                    CHECK(ids[std::size_t(cfg.branch_index(n, k))] ==
                          rolling_hash(std::span<const token_id>(ctx).last(std::size_t(n)),
                                       {n, 50, cfg.vocab_of(n, k)}));
        }
        std::vector<token_id> bad{0, 3, 10};
        CHECK_THROWS_AS(hash_all_orders(bad, make_default_config(10, 12, 3, 2)), std::out_of_range);
        std::vector<token_id> shortc{3, 4};
        CHECK_THROWS_AS(hash_all_orders(shortc, make_default_config(10, 12, 3, 2)), std::invalid_argument);
    });
    test_case("embed_sequence: first row uses the zero-padded window", [] {  // test_embedding.cpp:143-153
        const auto cfg = v2_config(16, 12, 4, 2);
        const auto host = make_bank<float>(cfg, 7);
        const device_bank bank(host);
        std::vector<token_id> seq{9};
        const auto rows = embed_sequence(seq, bank);
        std::vector<token_id> padded{0, 0, 0, 9};
        const auto want = embed_v2(padded, bank);
        CHECK(rows.size() == 12);
        for (std::size_t i = 0; i < 12; ++i) CHECK(rows[i] == want[i]);  // amp none: rows == merged
    });
    test_case("embed_sequence: split with carried context equals whole-sequence run", [] {  // :155-174
        const auto cfg = v2_config(32, 12, 3, 2, amp_mode::scale_sqrt_d);
        const device_bank bank(make_bank<float>(cfg, 11));
        rng64 rng(13);
        std::vector<token_id> seq(20);
        for (auto& t : seq) t = token_id(uniform_below(rng, 32));
        const auto whole = embed_sequence(seq, bank);
        const std::size_t cut = 7;
        const auto head = std::span<const token_id>(seq).first(cut);
        const auto tail = std::span<const token_id>(seq).subspan(cut);
        const auto p1 = embed_sequence(head, bank);
        const auto p2 = embed_sequence(tail, bank, head);
        for (std::size_t i = 0; i < cut * 12; ++i) CHECK(whole[i] == p1[i]);
        for (std::size_t i = 0; i < (seq.size() - cut) * 12; ++i) CHECK(whole[cut * 12 + i] == p2[i]);
    });
    test_case("embed_sequence: zero bank is the zero matrix", [] {  // :176-181
        const auto cfg = v2_config(8, 6, 3, 1);
        const device_bank bank(make_zero_bank<float>(cfg));
        std::vector<token_id> seq{1, 2, 3, 4};
        for (const float x : embed_sequence(seq, bank)) CHECK(x == 0.0f);
    });
    test_case("tensor-core shape: device == host-bank overload == embed_from_ids", [] {
        auto cfg = make_default_config(500, 256, 3, 2);
        const auto host = make_bank<float>(cfg, 5);
        const device_bank bank(host);
        CHECK(bank.tensor_core_path());
        rng64 rng(3);
        std::vector<token_id> seq(300);
        for (auto& t : seq) t = token_id(uniform_below(rng, 500));
        const auto a = embed_sequence_cached(seq, bank);
        const auto b = embed_sequence_cached(seq, host);
        CHECK(a.rows == b.rows && a.merged == b.merged);
        const auto ids = hash_sequence(seq, bank);
        std::vector<float> one(256);
        embed_from_ids(seq[100], std::span<const std::uint64_t>(ids).subspan(100 * 4, 4), bank, one);
        CHECK(close_rows(one, std::vector<float>(a.merged.begin() + 100 * 256, a.merged.begin() + 101 * 256)));
        CHECK_THROWS_AS(embed_from_ids(seq[0], std::span<const std::uint64_t>(ids).first(3), bank, one),
                        std::invalid_argument);
    });
    test_case("append stream equals from-scratch batch", [] {  // test_cache.cpp:54-65
        const auto cfg = v2_config(32, 384, 4, 2);
        const device_bank bank(make_bank<float>(cfg, 5));
        sequence_cache state(bank);
        rng64 rng(1);
        std::vector<token_id> confirmed;
        for (int i = 0; i < 40; ++i) {
            const token_id t = token_id(uniform_below(rng, 32));
            const auto ids = state.append(t);
            confirmed.push_back(t);
            const auto all = hash_sequence(confirmed, bank);
            CHECK(std::equal(ids.begin(), ids.end(), all.end() - long(ids.size())));
        }
        CHECK(state.length() == 40);
        CHECK_THROWS_AS(state.append(32), std::out_of_range);
    });
    test_case("snapshot / rollback / stale handles", [] {  // test_cache.cpp:81-126
        const auto cfg = v2_config(32, 384, 4, 2);
        const device_bank bank(make_bank<float>(cfg, 5));
        sequence_cache a(bank), b(bank);
        const auto ha = a.snapshot();
        CHECK_THROWS_AS(b.rollback(ha), std::invalid_argument);
        const auto h1 = a.snapshot();
        a.append(1);
        const auto h2 = a.snapshot();
        a.append(2);
        a.rollback(h1);
        CHECK_THROWS_AS(a.rollback(h2), std::invalid_argument);
        a.rollback(ha);
        CHECK(a.length() == 0);
    });
    test_case("draft_verify: accept all / none / too many", [] {  // test_cache.cpp:221-262
        const auto cfg = v2_config(32, 384, 4, 2);
        const device_bank bank(make_bank<float>(cfg, 9));
        embedding_memo memo(256);
        sequence_cache state(bank);
        state.append(11);
        std::vector<token_id> draft{3, 1, 4, 1, 5};
        cache_counters c;
        const auto result = draft_verify(state, memo, bank, draft, draft.size(), &c);
        CHECK(result.accepted.size() == 5);
        std::vector<token_id> seq{11, 3, 1, 4, 1, 5};
        const auto want = embed_sequence_cached(seq, bank).merged;
        for (std::size_t i = 0; i < 5; ++i)
            CHECK(close_rows(result.accepted[i], std::vector<float>(want.begin() + long((i + 1) * 384),
                                                                    want.begin() + long((i + 2) * 384))));
        CHECK(state.length() == 6 && state.last_token() == 5 && state.snapshot_depth() == 0);
        CHECK(c.verify_table_gathers == 0 && c.rollbacks == 1);
        sequence_cache s2(bank);
        s2.append(2);
        s2.append(8);
        std::vector<token_id> d2{9, 9, 9};
        CHECK(draft_verify(s2, memo, bank, d2, 0).accepted.empty());
        CHECK(s2.length() == 2 && s2.last_token() == 8);
        CHECK_THROWS_AS(draft_verify(s2, memo, bank, d2, 4), std::invalid_argument);
        CHECK(counters_to_json(c).find("\"rollbacks\":1") != std::string::npos);
    });
    test_case("config validation and JSON round-trip", [] {  // test_embedding.cpp:424-444
        ngram_config cfg = v2_config(16, 8, 3, 2);
        cfg.dim = 9;
        CHECK_THROWS_AS(cfg.validate(), std::invalid_argument);
        ngram_config missing = v2_config(16, 8, 3, 2);
        missing.sub_vocab.erase({3, 2});
        CHECK_THROWS_AS(missing.validate(), std::invalid_argument);
        CHECK_THROWS_AS(v2_config(1, 8, 3, 2), std::invalid_argument);
        const auto c2 = v2_config(128, 24, 4, 2, amp_mode::layer_norm);
        CHECK(ngram_config_from_json(to_json_string(c2)) == c2);
    });
    test_case("backward: sequence backward == sum of per-window embed_backward, accumulates", [] {
        auto cfg = make_default_config(500, 256, 3, 2);
        cfg.amplification = amp_mode::none;  // embed_backward takes d(merged) directly
        const auto host = make_bank<float>(cfg, 11);
        const device_bank bank(host);
        rng64 rng(21);
        std::vector<token_id> seq(40);
        for (auto& t : seq) t = token_id(uniform_below(rng, 500));
        std::vector<float> up(seq.size() * 256);
        for (auto& u : up) u = float(gaussian(rng));
        const auto fwd = embed_sequence_cached(seq, bank);
        auto a = zeros_like(host);
        embed_sequence_backward(seq, bank, fwd.merged, up, a);
        auto b = zeros_like(host);
        for (std::size_t pos = 0; pos < seq.size(); ++pos) {
            std::vector<token_id> ctx(3, 0);
            for (int j = 0; j < 3; ++j)
                if (long(pos) - 2 + j >= 0) ctx[std::size_t(j)] = seq[pos - 2 + std::size_t(j)];
            embed_backward(ctx, bank, std::span<const float>(up).subspan(pos * 256, 256), b);
        }
        CHECK(close_rows(a.base, b.base));
        for (std::size_t i = 0; i < a.sub_tables.size(); ++i) CHECK(close_rows(a.sub_tables[i], b.sub_tables[i]));
        for (std::size_t i = 0; i < a.projections.size(); ++i) CHECK(close_rows(a.projections[i], b.projections[i]));
        auto twice = a;
        embed_sequence_backward(seq, bank, fwd.merged, up, twice);
        std::vector<float> dbl(a.base.size());
        for (std::size_t i = 0; i < dbl.size(); ++i) dbl[i] = 2.0f * a.base[i];
        CHECK(close_rows(twice.base, dbl));
        CHECK_THROWS_AS(embed_backward(std::span<const token_id>(seq).first(3), bank,
                                       std::span<const float>(up).first(255), b),
                        std::invalid_argument);
        auto bad = seq;
        bad[7] = 500;
        const auto before = a.base;
        CHECK_THROWS_AS(embed_sequence_backward(bad, bank, fwd.merged, up, a), std::out_of_range);
        CHECK(a.base == before);
    });
    // ---- per-layer FFN (test_ple.cpp:60-200, float + bf16-representable tables)
    auto bf16 = [](std::vector<float>& v) {
        for (auto& x : v) {
            std::uint32_t u;
            std::memcpy(&u, &x, 4);
            u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
            std::memcpy(&x, &u, 4);
        }
    };
    auto layer_config = [](std::uint32_t v0, int width, int order, int k) {  // test_ple.cpp:43-57
        ngram_config cfg;
        cfg.max_order = order;
        cfg.sub_tables = k;
        cfg.base_vocab = v0;
        cfg.dim = width;
        cfg.variant = ne_variant::subtable_v2;
        cfg.amplification = amp_mode::none;
        for (int n = 2; n <= order; ++n)
            for (int kk = 1; kk <= k; ++kk) cfg.sub_vocab[{n, kk}] = 19 + 6 * std::uint64_t(n) + std::uint64_t(kk);
        cfg.validate();
        return cfg;
    };
    test_case("ffn_ple: zero input / zero table row give zero output", [&] {
        auto p = make_ple_params<float>(4, 6, 10, 1);
        bf16(p.table);
        std::vector<float> x(4, 0.0f);
        for (const float y : ffn_ple(x, 3, p)) CHECK(y == 0.0f);
        std::fill(p.table.begin() + 3 * 6, p.table.begin() + 4 * 6, 0.0f);
        rng64 rng(4);
        for (auto& v : x) v = float(gaussian(rng));
        for (const float y : ffn_ple(x, 3, p)) CHECK(y == 0.0f);
    });
    test_case("ffn_ple matches the straight-line oracle; rejects bad tokens / shapes", [&] {
        auto p = make_ple_params<float>(4, 6, 10, 7);
        bf16(p.table);
        rng64 rng(8);
        for (int trial = 0; trial < 20; ++trial) {
            std::vector<float> x(4);
            for (auto& v : x) v = float(gaussian(rng));
            const token_id t = token_id(uniform_below(rng, 10));
            const auto got = ffn_ple(x, t, p);
            std::vector<float> want(4);
            std::vector<double> h(6);
            for (int r = 0; r < 6; ++r) {
                double u = 0;
                for (int c = 0; c < 4; ++c) u += double(p.gate[r * 4 + c]) * x[c];
                h[r] = u / (1.0 + std::exp(-u)) * p.table[t * 6 + r];
            }
            for (int r = 0; r < 4; ++r) {
                double acc = 0;
                for (int c = 0; c < 6; ++c) acc += double(p.down[r * 6 + c]) * h[c];
                want[r] = float(acc);
            }
            CHECK(close_rows(got, want, 1e-5));
        }
        std::vector<float> x(4, 0.1f), short_x(3, 0.1f);
        CHECK_THROWS_AS(ffn_ple(x, 10, p), std::out_of_range);
        CHECK_THROWS_AS(ffn_ple(short_x, 2, p), std::invalid_argument);
    });
    test_case("ffn_plne: zero bank, all-pad context = ffn_ple / denom, base-only bank = ffn_ple", [&] {
        const auto cfg = layer_config(10, 6, 3, 3);
        auto p = make_ple_params<float>(4, 6, 10, 5);
        bf16(p.table);
        rng64 rng(9);
        std::vector<float> x(4);
        for (auto& v : x) v = float(gaussian(rng));
        std::vector<token_id> ctx{1, 2, 3}, pads{0, 0, 0};
        for (const float y : ffn_plne(x, ctx, make_zero_bank<float>(cfg), p)) CHECK(y == 0.0f);
        auto bank = make_zero_bank<float>(cfg);
        bank.base = p.table;
        const auto plne = ffn_plne(x, pads, bank, p);
        auto ple = ffn_ple(x, 0, p);
        for (auto& v : ple) v /= float(cfg.merge_denominator());
        CHECK(close_rows(plne, ple, 1e-5));
        ngram_config c1;
        c1.max_order = 1;
        c1.sub_tables = 1;
        c1.base_vocab = 10;
        c1.dim = 6;
        c1.variant = ne_variant::subtable_v2;
        c1.validate();
        auto b1 = make_zero_bank<float>(c1);
        b1.base = p.table;
        const device_bank d1(b1);
        for (token_id t = 0; t < 10; ++t) {
            const token_id one[1] = {t};
            CHECK(ffn_plne(x, one, d1, p) == ffn_ple(x, t, p));
        }
        CHECK_THROWS_AS(ffn_plne(x, ctx, make_bank<float>(layer_config(10, 8, 3, 2), 2), p), std::invalid_argument);
    });
    test_case("ffn_plne_backward: dx matches finite differences; ffn_ple_backward == base-only plne", [&] {
        const auto cfg = layer_config(10, 8, 3, 2);
        auto host = make_bank<float>(cfg, 3);
        for (auto* v : {&host.base}) bf16(*v);
        for (auto& t : host.sub_tables) bf16(t);
        for (auto& w : host.projections) bf16(w);
        const device_bank bank(host);
        auto p = make_ple_params<float>(5, 8, 10, 6);
        rng64 rng(12);
        std::vector<float> x(5), u(5);
        for (auto& v : x) v = float(gaussian(rng));
        for (auto& v : u) v = float(gaussian(rng));
        std::vector<token_id> ctx{4, 7, 1};
        auto grads = ple_zeros_like(p);
        auto bg = zeros_like(host);
        std::vector<float> dx(5, 0.0f);
        ffn_plne_backward(x, ctx, bank, p, u, grads, bg, dx);
        for (int c = 0; c < 5; ++c) {
            auto xp = x, xm = x;
            xp[c] += 1e-2f;
            xm[c] -= 1e-2f;
            const auto yp = ffn_plne(xp, ctx, bank, p), ym = ffn_plne(xm, ctx, bank, p);
            double fd = 0;
            for (int r = 0; r < 5; ++r) fd += double(u[r]) * (double(yp[r]) - double(ym[r])) / 2e-2;
            CHECK(std::fabs(fd - dx[c]) <= 1e-3 * std::max(1.0, std::fabs(fd)) + 1e-6);
        }
        bool any = false;
        for (const float v : bg.base) any = any || v != 0.0f;
        CHECK(any);
        auto p2 = make_ple_params<float>(4, 6, 10, 7);
        bf16(p2.table);
        auto g1 = ple_zeros_like(p2);
        std::vector<float> x2(4, 0.3f), u2(4, 1.0f), d1(4, 0.0f);
        ffn_ple_backward(x2, 2, p2, u2, g1, d1);
        bool row = false;
        for (int i = 0; i < 6; ++i) row = row || g1.table[2 * 6 + i] != 0.0f;
        CHECK(row);
        CHECK(g1.table[3 * 6] == 0.0f);
    });
    test_case("param_count / budget_report / save_bank round trip", [] {  // test_embedding.cpp accounting
        const auto cfg = make_default_config(1000, 256, 3, 2);
        const auto pc = param_count(cfg);
        CHECK(pc.base == 1000ull * 256);
        CHECK(pc.projections == 4ull * 256 * 64);
        CHECK(pc.total == pc.base + pc.sub_tables + pc.projections);
        const auto b = budget_report(cfg, pc.total);
        CHECK(b.fraction == 0.5 && !b.over_budget);
        CHECK(budget_report(3, 1).over_budget);
        CHECK(budget_guidance(budget_report(3, 1)).find("over budget") != std::string::npos);
        auto host = make_bank<float>(make_default_config(50, 128, 3, 1), 4);
        const std::string path = "/tmp/ngram_dropin_bank.bin";
        save_bank(host, path);
        const auto back = load_bank(path);
        CHECK(back.base == host.base && back.sub_tables == host.sub_tables && back.projections == host.projections);
        CHECK(back.config == host.config);
        CHECK_THROWS_AS(load_bank("/nonexistent/dir/bank.bin"), io_error);
        const device_bank a(host), c = device_bank::from_file(path, host.config);
        std::vector<token_id> seq{1, 2, 3, 4, 5};
        CHECK(embed_sequence(seq, a) == embed_sequence(seq, c));
    });
    test_case("amplify (device) matches the reference formulas; bank_cast round trip", [] {
        rng64 rng(17);
        std::vector<float> e(300), gain(300), bias(300), out(300);
        for (auto& v : e) v = float(gaussian(rng));
        for (auto& v : gain) v = 1.0f + 0.1f * float(gaussian(rng));
        for (auto& v : bias) v = 0.05f * float(gaussian(rng));
        amplify(e, amp_mode::none, {}, {}, out);
        CHECK(out == e);
        amplify(e, amp_mode::scale_sqrt_d, {}, {}, out);
        const float s = float(std::sqrt(300.0));
        for (int i = 0; i < 300; ++i) CHECK(out[i] == e[i] * s);
        amplify(e, amp_mode::layer_norm, gain, bias, out);
        double mean = 0, var = 0;
        for (float v : e) mean += v;
        mean /= 300;
        for (float v : e) var += (v - mean) * (v - mean);
        var /= 300;
        std::vector<float> want(300);
        for (int i = 0; i < 300; ++i) want[i] = float(gain[i] * (e[i] - mean) / std::sqrt(var + 1e-5) + bias[i]);
        CHECK(close_rows(out, want, 1e-5));
        CHECK_THROWS_AS(amplify(e, amp_mode::layer_norm, std::span<const float>(gain).first(3), bias, out),
                        std::invalid_argument);
        const auto host = make_bank<float>(make_default_config(40, 64, 3, 1), 2);
        const auto back = bank_cast<double, float>(bank_cast<float, double>(host));
        CHECK(back.base == host.base && back.sub_tables == host.sub_tables);
    });
    test_case("one device_bank shared by host threads (bank read-only across threads, SPEC.md:283)", [] {
        const auto host = make_bank<float>(make_default_config(500, 256, 3, 2), 8);
        const device_bank bank(host);
        std::vector<std::vector<token_id>> seqs(4);
        rng64 rng(5);
        for (auto& q : seqs) {
            q.resize(100 + 37 * (&q - seqs.data()));
            for (auto& t : q) t = token_id(uniform_below(rng, 500));
        }
        std::vector<std::vector<float>> want;
        for (const auto& q : seqs) want.push_back(embed_sequence(q, bank));
        std::vector<int> ok(seqs.size(), 1);
        std::vector<std::thread> th;
        for (std::size_t i = 0; i < seqs.size(); ++i)
            th.emplace_back([&, i] {
                sequence_cache cache(bank);
                for (int rep = 0; rep < 10; ++rep) {
                    if (embed_sequence(seqs[i], bank) != want[i]) ok[i] = 0;
                    cache.append(seqs[i][std::size_t(rep)]);
                }
            });
        for (auto& t : th) t.join();
        for (const int v : ok) CHECK(v == 1);
    });
    test_case("embedding_memo: hits are bit-identical, LRU eviction, counters (test_cache.cpp:264-314)", [] {
        const auto cfg = make_default_config(300, 256, 3, 2);
        const device_bank bank(make_bank<float>(cfg, 13));
        embedding_memo memo(2);
        cache_counters c;
        const std::vector<token_id> a{1, 2, 3}, b{4, 5, 6}, d{7, 8, 9};
        const auto ia = hash_all_orders(a, cfg), ib = hash_all_orders(b, cfg), id = hash_all_orders(d, cfg);
        const auto x1 = memo.lookup(3, ia, bank, &c);
        const auto x2 = memo.lookup(3, ia, bank, &c);
        CHECK(x1 == x2 && c.memo_hits == 1 && c.memo_misses == 1);
        std::vector<float> direct(256);
        embed_from_ids(3, ia, bank, direct);
        CHECK(x1 == direct);
        memo.lookup(6, ib, bank, &c);
        memo.lookup(9, id, bank, &c);  // evicts the least recently used (token 3)
        CHECK(memo.size() == 2 && c.memo_misses == 3);
        memo.lookup(3, ia, bank, &c);
        CHECK(c.memo_misses == 4 && c.table_gathers == 4 * 5);
        CHECK_THROWS_AS(embedding_memo(0), std::invalid_argument);
    });
    test_case("amplify_backward + embed_backward == embed_sequence_backward for one window (layer_norm)", [] {
        auto cfg = make_default_config(300, 256, 3, 2);
        cfg.amplification = amp_mode::layer_norm;
        auto host = make_bank<float>(cfg, 23);
        rng64 rng(3);
        for (auto& g : host.ln_gain) g = 1.0f + 0.1f * float(gaussian(rng));
        const device_bank bank(host);
        const std::vector<token_id> ctx{5, 9, 11};
        std::vector<float> up(256);
        for (auto& u : up) u = float(gaussian(rng));
        std::vector<float> merged(256);
        embed_window(ctx, bank, merged);
        auto a = zeros_like(host);
        std::vector<float> d_pre(256);
        amplify_backward(merged, up, bank, a, d_pre);
        embed_backward(ctx, bank, d_pre, a);
        auto b = zeros_like(host);
        embed_sequence_backward(std::span<const token_id>(ctx).last(1), bank, merged, up, b,
                                std::span<const token_id>(ctx).first(2));
        CHECK(close_rows(a.base, b.base, 1e-5) && close_rows(a.ln_gain, b.ln_gain, 1e-5) &&
              close_rows(a.ln_bias, b.ln_bias, 1e-5));
        for (std::size_t i = 0; i < a.projections.size(); ++i) CHECK(close_rows(a.projections[i], b.projections[i], 1e-5));
    });
    test_case("generate_zipf_markov reproduces the reference stream", [] {  // corpus.cpp:211-271
        // values printed by the reference (oracle/_ref) for vocab 1000, 2 x 64, seed 99
        const auto z = generate_zipf_markov(1000, 2, 64, 99, 1.1, 0.85);
        const std::vector<token_id> head{7, 4, 0, 7, 4, 9, 1, 43, 0, 7, 4, 9}, tail{296, 11, 14, 0, 7, 4};
        CHECK(z.size() == 2 && z[0].size() == 64);
        CHECK(std::equal(head.begin(), head.end(), z[0].begin()));
        CHECK(std::equal(tail.begin(), tail.end(), z[1].end() - 6));
        std::uint64_t sum = 0;
        for (const auto& q : z)
            for (auto t : q) sum += t;
        CHECK(sum == 1946);
    });
    test_case("analysis: hit rates and worked collision examples", [] {  // test_analysis.cpp:50-113
        std::vector<token_sequence> one{{5}};
        CHECK(std::fabs(compute_hit_rate(one, {2, 10, 100}) - 0.01) < 1e-12);
        std::vector<token_sequence> pairs;
        for (std::uint32_t a = 0; a < 7; ++a)
            for (std::uint32_t b = 0; b < 7; ++b) pairs.push_back({a, b});
        CHECK(compute_hit_rate(pairs, {2, 7, 49}) == 1.0);
        CHECK(compute_hit_rate(pairs, {2, 7, 30}) == 1.0);
        const auto z = generate_zipf_markov(1000, 16, 4096, 99, 1.1, 0.85);
        CHECK(compute_hit_rate(z, {4, 1000, 4999}) > compute_hit_rate(z, {2, 1000, 4999}));
        std::vector<token_sequence> ex{{1, 5}, {3, 5}, {5, 5}};
        CHECK(count_collisions(ex, {2, 10, 20}) == 2);
        CHECK(count_collisions(ex, {2, 10, 23}) == 0);
        std::vector<token_sequence> inj{{1, 2, 3, 4, 5, 6, 7, 8, 9}};
        CHECK(count_collisions(inj, {2, 10, 1000000}) == 0);
        rng64 rng(42);
        for (int trial = 0; trial < 20; ++trial) {
            const auto c = random_corpus(rng, 6, 4, 50);
            CHECK(count_collisions(c, {2, 6, 36}) == 0);
            CHECK(count_collisions(c, {3, 6, 216}) == 0);
        }
    });
    test_case("analysis: streaming equals the two-pass oracle", [] {  // test_analysis.cpp:115-129
        rng64 rng(0xabc);
        for (int trial = 0; trial < 25; ++trial) {
            const std::uint32_t v0 = 3 + std::uint32_t(uniform_below(rng, 200));
            const auto c = random_corpus(rng, v0, 1 + uniform_below(rng, 6), 80);
            const int order = 2 + int(uniform_below(rng, 3));
            const std::uint64_t m = 1 + uniform_below(rng, 3000);
            const auto want = two_pass(c, v0, order, m);
            const hash_spec spec{order, v0, m};
            CHECK(compute_hit_rate(c, spec) == double(want.buckets) / double(m));
            CHECK(count_collisions(c, spec) == want.ngrams - want.buckets);
        }
    });
    test_case("analysis: sweeps, advised sizes, monotonicity", [] {  // test_analysis.cpp:131-195
        const auto corpus = generate_zipf_markov(100, 8, 512, 7, 1.1, 0.85);
        const std::vector<std::uint64_t> moduli{101, 250, 999};
        const auto r = sweep_vocab_sizes(corpus, 2, 100, moduli, "c");
        CHECK(r.size() == 3);
        for (std::size_t i = 0; i < r.size(); ++i) {
            CHECK(r[i].modulus == moduli[i] && r[i].order == 2 && r[i].corpus_id == "c");
            CHECK(r[i].hit_rate == compute_hit_rate(corpus, {2, 100, moduli[i]}));
            CHECK(r[i].collision_count == count_collisions(corpus, {2, 100, moduli[i]}));
            CHECK(r[i].tokens_processed == total_tokens(corpus));
        }
        CHECK(sweep_vocab_sizes(corpus, 2, 100, {}).empty());
        CHECK_THROWS_AS(sweep_vocab_sizes(corpus, 2, 100, {250, 101}), std::invalid_argument);
        const auto big = generate_zipf_markov(1000, 24, 4096, 20260809, 1.1, 0.85);
        const auto rr = sweep_vocab_sizes(big, 2, 1000, {2000, 2500});
        CHECK(rr.size() == 2 && rr[0].collision_count > rr[1].collision_count);
        const auto o1 = two_pass(big, 1000, 2, 2000), o2 = two_pass(big, 1000, 2, 2500);
        CHECK(rr[0].collision_count == o1.ngrams - o1.buckets && rr[1].collision_count == o2.ngrams - o2.buckets);
        CHECK(advise_vocab_size(128000, 30) == 3904000 && advise_vocab_size(10, 2) == 25 && advise_vocab_size(2, 1) == 3);
        CHECK_THROWS_AS(advise_vocab_size(1, 3), std::invalid_argument);
        CHECK_THROWS_AS(advise_vocab_size(10, 0), std::invalid_argument);
        CHECK(advise_vocab_size(1000, 30) == 30500);
        CHECK(count_collisions(big, {2, 1000, 30500}) <= count_collisions(big, {2, 1000, 30000}));
        rng64 rng(0xfeed);
        for (int trial = 0; trial < 10; ++trial) {
            auto c = random_corpus(rng, 50, 6, 60);
            std::vector<token_sequence> prefix(c.begin(), c.begin() + 3);
            CHECK(compute_hit_rate(c, {2, 50, 40}) >= compute_hit_rate(prefix, {2, 50, 40}));
            CHECK(count_collisions(c, {2, 50, 40}) >= count_collisions(prefix, {2, 50, 40}));
        }
    });
    test_case("analysis: sharded analyzers merge to the single pass", [] {  // test_analysis.cpp:197-240
        rng64 rng(0x5eed);
        const auto corpus = random_corpus(rng, 120, 9, 100);
        const std::vector<int> orders{2, 3};
        const std::vector<std::uint64_t> moduli{37, 240, 4000};
        corpus_analyzer whole(120, orders, moduli);
        whole.add_corpus(corpus);
        corpus_analyzer a(120, orders, moduli), b(120, orders, moduli), c(120, orders, moduli);
        for (std::size_t i = 0; i < corpus.size(); ++i) (i % 3 == 0 ? a : i % 3 == 1 ? b : c).add_sequence(corpus[i]);
        c.merge(a);
        c.merge(b);
        const auto sw = whole.stats(), sc = c.stats();
        CHECK(sw.sequences_seen == sc.sequences_seen && sw.ngrams_seen == sc.ngrams_seen);
        CHECK(sw.distinct_ngrams == sc.distinct_ngrams && sw.distinct_buckets == sc.distinct_buckets);
        rng64 r2(31337);
        const auto c2 = random_corpus(r2, 40, 8, 120);
        corpus_analyzer an(40, {2, 3, 4}, {17, 1000, 70000});
        an.add_corpus(c2);
        const auto s = an.stats();
        for (const auto& [order, distinct] : s.distinct_ngrams) {
            CHECK(distinct <= s.ngrams_seen.at(order));
            for (const auto& [key, nb] : s.distinct_buckets)
                if (key.first == order) CHECK(nb <= distinct && nb <= key.second);
        }
    });
    test_case("analysis: error paths and CSV", [] {  // test_analysis.cpp:241-262
        std::vector<token_sequence> empty;
        CHECK_THROWS_AS(compute_hit_rate(empty, {2, 10, 5}), std::invalid_argument);
        std::vector<token_sequence> empty_seqs{{}, {}};
        CHECK_THROWS_AS(compute_hit_rate(empty_seqs, {2, 10, 5}), std::invalid_argument);
        std::vector<token_sequence> oob{{3, 11}};
        CHECK_THROWS_AS(count_collisions(oob, {2, 10, 5}), std::out_of_range);
        CHECK_THROWS_AS(corpus_analyzer(1 << 17, {8}, {100}), std::invalid_argument);
        std::vector<collision_report> reports(2);
        reports[0] = {2, 2000, 0.5, 123, "c", 4096};
        reports[1] = {3, 2500, 0.125, 0, "c", 4096};
        std::ostringstream ss;
        write_reports_csv(ss, reports);
        CHECK(ss.str() == "order,modulus,hit_rate,collision_count,tokens_processed\n2,2000,0.5,123,4096\n"
                          "3,2500,0.125,0,4096\n");
    });
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
