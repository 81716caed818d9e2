// analysis_dropin.cpp -- include/ngram/analysis.hpp + corpus.hpp on top of the C-ABI.  Host
// logic only (argument checks in the reference's order, report arithmetic, CSV); the counting
// runs in the analysis kernels behind ngram_analyzer_*.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <ostream>
#include <stdexcept>

#include "ngram/analysis.hpp"
#include "ngram/errors.hpp"
#include "ngram/rng.hpp"
#include "ngram_b200.h"

namespace ngram {

// ------------------------------------------------------------------------ corpus.hpp
std::size_t total_tokens(const std::vector<token_sequence>& corpus) {
    std::size_t n = 0;
    for (const auto& q : corpus) n += q.size();
    return n;
}

void window_at(const token_sequence& seq, std::size_t pos, int order, std::vector<token_id>& out) {
    out.assign(std::size_t(order), 0);
    for (int j = 0; j < order; ++j) {  // out[order-1] is the token at pos
        const std::ptrdiff_t src = std::ptrdiff_t(pos) - j;
        if (src >= 0) out[std::size_t(order - 1 - j)] = seq[std::size_t(src)];
    }
}

namespace {

// P(i) ~ 1/(i+1)^s over [0, vocab), sampled by inverting the running-sum CDF.
class zipf_table {
  public:
    zipf_table(std::uint32_t vocab, double s) : cdf_(vocab) {
        double acc = 0.0;
        for (std::uint32_t i = 0; i < vocab; ++i) cdf_[i] = acc += 1.0 / std::pow(double(i) + 1.0, s);
        for (double& c : cdf_) c /= acc;
    }
    token_id sample(rng64& g) const {
        const auto it = std::upper_bound(cdf_.begin(), cdf_.end(), uniform01(g));
        return token_id(std::min<std::size_t>(std::size_t(it - cdf_.begin()), cdf_.size() - 1));
    }

  private:
    std::vector<double> cdf_;
};

}  // namespace

// corpus.cpp:211-271: function-token pool with Zipf successors, content tokens mapped back to
// the pool by id block, fresh Zipf draws over the active half (never two in a row), 0.1 %
// uniform noise.  The draw order is the reference's, so a seed gives the same corpus.
std::vector<token_sequence> generate_zipf_markov(std::uint32_t vocab, std::size_t sequences, std::size_t seq_len,
                                                 std::uint64_t seed, double exponent, double markov_prob) {
    rng64 g(seed);
    const zipf_table zipf(vocab, exponent);
    const std::uint32_t pool = std::min<std::uint32_t>(vocab, std::max<std::uint32_t>(2, vocab * 3 / 50));
    const std::uint32_t block = std::max<std::uint32_t>(1, vocab / 20);
    const std::uint32_t active = std::max<std::uint32_t>(pool, vocab / 2);
    std::vector<token_id> next_of(vocab);
    for (std::uint32_t v = 0; v < vocab; ++v) {
        if (v >= pool) {
            next_of[v] = token_id((2 * (v / block) + 1) % pool);
            continue;
        }
        token_id s = zipf.sample(g);
        while (s >= pool) s = zipf.sample(g);
        next_of[v] = s;
    }
    std::vector<token_sequence> out(sequences, token_sequence(seq_len));
    for (auto& seq : out) {
        token_id prev = 0;
        bool fresh = true;
        for (auto& t : seq) {
            if (!fresh && uniform01(g) >= markov_prob) {
                if (uniform01(g) < 0.001) {
                    t = token_id(uniform_below(g, vocab));
                } else {
                    t = zipf.sample(g);
                    while (t >= active) t = zipf.sample(g);
                }
                fresh = true;
            } else {
                t = next_of[prev];
                fresh = false;
            }
            prev = t;
        }
    }
    return out;
}

// ------------------------------------------------------------------------ analysis.hpp
corpus_analyzer::corpus_analyzer(std::uint64_t base_vocab, std::vector<int> orders, std::vector<std::uint64_t> moduli)
    : base_vocab_(base_vocab), orders_(std::move(orders)), moduli_(std::move(moduli)) {
    throw_status(ngram_analyzer_create(0, base_vocab_, orders_.data(), int(orders_.size()), moduli_.data(),
                                       int(moduli_.size()), &h_));
}

corpus_analyzer::~corpus_analyzer() { ngram_analyzer_destroy(h_); }

corpus_analyzer::corpus_analyzer(corpus_analyzer&& o) noexcept
    : base_vocab_(o.base_vocab_), orders_(std::move(o.orders_)), moduli_(std::move(o.moduli_)), h_(o.h_) {
    o.h_ = nullptr;
}

corpus_analyzer& corpus_analyzer::operator=(corpus_analyzer&& o) noexcept {
    if (this != &o) {
        ngram_analyzer_destroy(h_);
        base_vocab_ = o.base_vocab_;
        orders_ = std::move(o.orders_);
        moduli_ = std::move(o.moduli_);
        h_ = o.h_;
        o.h_ = nullptr;
    }
    return *this;
}

void corpus_analyzer::add_sequence(std::span<const token_id> seq) {
    const int64_t off[2] = {0, int64_t(seq.size())};
    throw_status(ngram_analyzer_add_host(h_, seq.data(), off, 1));
}

void corpus_analyzer::add_corpus(const std::vector<token_sequence>& corpus) {
    std::vector<int64_t> off(corpus.size() + 1, 0);
    std::vector<token_id> flat;
    flat.reserve(total_tokens(corpus));
    for (std::size_t i = 0; i < corpus.size(); ++i) {
        flat.insert(flat.end(), corpus[i].begin(), corpus[i].end());
        off[i + 1] = int64_t(flat.size());
    }
    throw_status(ngram_analyzer_add_host(h_, flat.data(), off.data(), int64_t(corpus.size())));
}

void corpus_analyzer::merge(const corpus_analyzer& other) {
    if (other.base_vocab_ != base_vocab_ || other.orders_ != orders_ || other.moduli_ != moduli_)
        throw std::invalid_argument("corpus_analyzer: merge of mismatched analyzers");
    throw_status(ngram_analyzer_merge(h_, other.h_, nullptr));
}

corpus_stats corpus_analyzer::stats() const {
    const std::size_t no = orders_.size(), nm = moduli_.size();
    std::vector<std::uint64_t> seen(no), dist(no), bk(no * nm);
    corpus_stats s;
    std::uint64_t sq = 0, tk = 0;
    throw_status(ngram_analyzer_stats(h_, &sq, &tk, seen.data(), dist.data(), bk.data()));
    s.sequences_seen = sq;
    s.tokens_seen = tk;
    for (std::size_t i = 0; i < no; ++i) {
        s.ngrams_seen[orders_[i]] = seen[i];
        s.distinct_ngrams[orders_[i]] = dist[i];
        for (std::size_t j = 0; j < nm; ++j) s.distinct_buckets[{orders_[i], moduli_[j]}] = bk[i * nm + j];
    }
    return s;
}

std::vector<collision_report> corpus_analyzer::reports(const std::string& corpus_id) const {
    const corpus_stats s = stats();
    if (s.tokens_seen == 0) throw std::invalid_argument("corpus_analyzer: empty corpus");
    std::vector<collision_report> out;
    for (const int n : orders_)
        for (const std::uint64_t m : moduli_) {
            const std::uint64_t b = s.distinct_buckets.at({n, m});
            out.push_back({n, m, double(b) / double(m), s.distinct_ngrams.at(n) - b, corpus_id, s.tokens_seen});
        }
    return out;
}

namespace {

corpus_analyzer analyze_single(const std::vector<token_sequence>& corpus, const hash_spec& spec) {
    spec.validate();
    if (total_tokens(corpus) == 0) throw std::invalid_argument("analysis: empty corpus");
    corpus_analyzer an(spec.base, {spec.order}, {spec.modulus});
    an.add_corpus(corpus);
    return an;
}

}  // namespace

double compute_hit_rate(const std::vector<token_sequence>& corpus, const hash_spec& spec) {
    return analyze_single(corpus, spec).reports("").front().hit_rate;
}

std::uint64_t count_collisions(const std::vector<token_sequence>& corpus, const hash_spec& spec) {
    return analyze_single(corpus, spec).reports("").front().collision_count;
}

std::vector<collision_report> sweep_vocab_sizes(const std::vector<token_sequence>& corpus, int order,
                                                std::uint64_t base_vocab, const std::vector<std::uint64_t>& moduli,
                                                const std::string& corpus_id) {
    if (moduli.empty()) return {};
    if (!std::is_sorted(moduli.begin(), moduli.end()))
        throw std::invalid_argument("sweep_vocab_sizes: moduli must be sorted ascending");
    if (total_tokens(corpus) == 0) throw std::invalid_argument("analysis: empty corpus");
    corpus_analyzer an(base_vocab, {order}, moduli);
    an.add_corpus(corpus);
    return an.reports(corpus_id);
}

std::uint64_t advise_vocab_size(std::uint64_t base_vocab, std::uint64_t target_multiple) {
    if (base_vocab < 2) throw std::invalid_argument("advise_vocab_size: base vocabulary must be >= 2");
    if (target_multiple < 1) throw std::invalid_argument("advise_vocab_size: target multiple must be >= 1");
    return ((2 * target_multiple + 1) * base_vocab + 1) / 2;  // round((m + 1/2) V0)
}

void write_reports_csv(std::ostream& out, std::span<const collision_report> reports) {
    out << "order,modulus,hit_rate,collision_count,tokens_processed\n";
    for (const auto& r : reports) {
        char rate[64];
        std::snprintf(rate, sizeof(rate), "%.9g", r.hit_rate);
        out << r.order << ',' << r.modulus << ',' << rate << ',' << r.collision_count << ',' << r.tokens_processed
            << '\n';
    }
}

}  // namespace ngram
