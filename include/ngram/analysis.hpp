// analysis.hpp -- drop-in for proj/include/ngram/analysis.hpp (analysis.hpp:19-124): corpus
// collision analysis computed on the GPU (ngram_analyzer_* in ngram_b200.h, kernels in
// analysis.cu).  Same types, same numbers, same exceptions.  corpus_analyzer owns a device
// analyzer on CUDA device 0: movable, not copyable.
#pragma once
#include <cstdint>
#include <iosfwd>
#include <map>
#include <span>
#include <string>
#include <vector>

#include "ngram/corpus.hpp"
#include "ngram/hashing.hpp"

struct ngram_analyzer;

namespace ngram {

struct corpus_stats {
    std::uint64_t sequences_seen = 0;
    std::uint64_t tokens_seen = 0;
    std::map<int, std::uint64_t> ngrams_seen;      // per order
    std::map<int, std::uint64_t> distinct_ngrams;  // per order
    std::map<std::pair<int, std::uint64_t>, std::uint64_t> distinct_buckets;  // per (order, modulus)
};

// hit_rate = distinct buckets / modulus; collision_count = distinct n-grams - distinct buckets
struct collision_report {
    int order = 0;
    std::uint64_t modulus = 0;
    double hit_rate = 0.0;
    std::uint64_t collision_count = 0;
    std::string corpus_id;
    std::uint64_t tokens_processed = 0;
};

class corpus_analyzer {
  public:
    corpus_analyzer(std::uint64_t base_vocab, std::vector<int> orders, std::vector<std::uint64_t> moduli);
    ~corpus_analyzer();
    corpus_analyzer(corpus_analyzer&& o) noexcept;
    corpus_analyzer& operator=(corpus_analyzer&& o) noexcept;
    corpus_analyzer(const corpus_analyzer&) = delete;
    corpus_analyzer& operator=(const corpus_analyzer&) = delete;

    void add_sequence(std::span<const token_id> seq);
    void add_corpus(const std::vector<token_sequence>& corpus);  // one device pass
    void merge(const corpus_analyzer& other);

    corpus_stats stats() const;
    std::vector<collision_report> reports(const std::string& corpus_id) const;

    const std::vector<int>& orders() const { return orders_; }
    const std::vector<std::uint64_t>& moduli() const { return moduli_; }

  private:
    std::uint64_t base_vocab_;
    std::vector<int> orders_;
    std::vector<std::uint64_t> moduli_;
    ::ngram_analyzer* h_ = nullptr;
};

double compute_hit_rate(const std::vector<token_sequence>& corpus, const hash_spec& spec);
std::uint64_t count_collisions(const std::vector<token_sequence>& corpus, const hash_spec& spec);
std::vector<collision_report> sweep_vocab_sizes(const std::vector<token_sequence>& corpus, int order,
                                                std::uint64_t base_vocab, const std::vector<std::uint64_t>& moduli,
                                                const std::string& corpus_id = "");
std::uint64_t advise_vocab_size(std::uint64_t base_vocab, std::uint64_t target_multiple);
void write_reports_csv(std::ostream& out, std::span<const collision_report> reports);

}  // namespace ngram
