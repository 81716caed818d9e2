// corpus.hpp -- drop-in for the parts of proj/include/ngram/corpus.hpp the analysis API and its
// tests use: the sequence type, total_tokens, window_at (corpus.cpp:273-280) and the
// synthetic Zipf-Markov generator (corpus.cpp:186-271, same rng stream => same tokens).
// Corpus file I/O is outside this library's scope.
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

#include "ngram/config.hpp"

namespace ngram {

using token_sequence = std::vector<token_id>;

std::size_t total_tokens(const std::vector<token_sequence>& corpus);

std::vector<token_sequence> generate_zipf_markov(std::uint32_t vocab, std::size_t sequences, std::size_t seq_len,
                                                 std::uint64_t seed, double exponent = 1.1,
                                                 double markov_prob = 0.35);

// The trailing window ending at `pos`, zero-padded before the sequence start.
void window_at(const token_sequence& seq, std::size_t pos, int order, std::vector<token_id>& out);

}  // namespace ngram
