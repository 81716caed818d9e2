// bench_dropin.cpp -- per-call latency of the C++ drop-in (include/ngram/*.hpp) entries a
// reference call site uses one token at a time: rolling_hash, hash_all_orders,
// sequence_cache::append (+ embedding_memo::lookup), embed_from_ids and draft_verify.  Each
// such call is a synchronous host -> device -> host round trip through the C-ABI; this
// prints one JSON line with the median microseconds per call (after warm-up), so a
// reference loop's cost through the drop-in can be compared with the reference's CPU numbers
// (append 948 ns/token at N=4, K=4).  Built by paper_2601_21204_b200/build.py,
// run by bench.py --workload dropin.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "ngram/cache.hpp"
#include "ngram/config.hpp"
#include "ngram/embedding.hpp"
#include "ngram/hashing.hpp"

using namespace ngram;

static double median_us(int reps, const std::function<void()>& f) {
    for (int i = 0; i < 5; ++i) f();
    std::vector<double> t;
    t.reserve(std::size_t(reps));
    for (int i = 0; i < reps; ++i) {
        const auto a = std::chrono::steady_clock::now();
        f();
        t.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count());
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main(int argc, char** argv) {
    const int D = argc > 1 ? std::stoi(argv[1]) : 3072;
    const int reps = argc > 2 ? std::stoi(argv[2]) : 200;
    // LongCat-shaped config (N = 4, K = 4, D), reduced vocabulary so the host bank is small
    const auto cfg = make_default_config(1000, D, 4, 4);
    const auto host = make_bank<float>(cfg, 3);
    device_bank bank(host);
    std::vector<token_id> ctx{5, 6, 7, 8};
    const auto ids = hash_all_orders(ctx, cfg);
    std::vector<float> out(static_cast<std::size_t>(D));
    sequence_cache st(bank);
    token_id t = 1;
    embedding_memo memo(1);  // capacity 1: lookups of new keys miss (embed_from_ids on the GPU)
    const double us_rolling = median_us(reps, [&] { (void)rolling_hash(std::span(ctx).last(3), {3, 1000, 997}); });
    const double us_hash = median_us(reps, [&] { (void)hash_all_orders(ctx, cfg); });
    const double us_append = median_us(reps, [&] { (void)st.append(t = (t * 7 + 3) % 1000); });
    const double us_embed = median_us(reps, [&] { embed_from_ids(ctx.back(), ids, bank, out); });
    const double us_embed_host = median_us(reps, [&] { embed_from_ids(ctx.back(), ids, host, out); });
    const double us_append_memo = median_us(reps, [&] {
        t = (t * 7 + 3) % 1000;
        const auto i2 = st.append(t);
        (void)memo.lookup(t, i2, bank);
    });
    std::vector<token_id> draft{3, 1, 4, 1};
    const double us_verify = median_us(reps, [&] { (void)draft_verify(st, memo, bank, draft, 2); });
    std::printf(
        "{\"D\": %d, \"reps\": %d, \"us_per_call\": {\"rolling_hash\": %.2f, \"hash_all_orders\": %.2f, "
        "\"sequence_cache_append\": %.2f, \"embed_from_ids_device_bank\": %.2f, \"embed_from_ids_host_bank\": %.2f, "
        "\"append_plus_memo_lookup_miss\": %.2f, \"draft_verify_4_accept_2\": %.2f}}\n",
        D, reps, us_rolling, us_hash, us_append, us_embed, us_embed_host, us_append_memo, us_verify);
    return 0;
}
