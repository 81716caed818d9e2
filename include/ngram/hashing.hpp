// hashing.hpp -- drop-in for proj/include/ngram/hashing.hpp (hashing.hpp:13-38), computed
// by the K1 hash-index kernel (bit-exact) behind the C-ABI.
#pragma once
#include <cstdint>
#include <span>
#include <vector>

#include "ngram/config.hpp"

namespace ngram {

class device_bank;

struct hash_spec {
    int order = 2;
    std::uint64_t base = 2;
    std::uint64_t modulus = 1;
    void validate() const;
};

// rolling_hash (hashing.cpp:33-59): one window, oldest first.
std::uint64_t rolling_hash(std::span<const token_id> window, const hash_spec& spec);
// hash_all_orders (hashing.cpp:61-81): ids of every (n,k) branch over the N-token context.
std::vector<std::uint64_t> hash_all_orders(std::span<const token_id> context, const ngram_config& cfg);

// Batched extension: ids [len][branch_count] of every position of one sequence (the
// windows of embed_sequence, embedding.hpp:391-405), prior_context as in embed_sequence.
std::vector<std::uint64_t> hash_sequence(std::span<const token_id> tokens, const device_bank& bank,
                                         std::span<const token_id> prior_context = {});

}  // namespace ngram
