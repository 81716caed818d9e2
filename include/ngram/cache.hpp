// cache.hpp -- drop-in for proj/include/ngram/cache.hpp (cache.hpp:14-136).  The decode
// state (ring of N-1 tokens, length, last) lives on the device (ngram_decode); appends,
// verification and the accepted-prefix commit run as kernels.
#pragma once
#include <cstdint>
#include <list>
#include <map>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "ngram/embedding.hpp"

struct ngram_decode;

namespace ngram {

struct cache_counters {
    std::uint64_t appends = 0;
    std::uint64_t rollbacks = 0;
    std::uint64_t memo_hits = 0;
    std::uint64_t memo_misses = 0;
    std::uint64_t table_gathers = 0;
    std::uint64_t projection_madds = 0;
    std::uint64_t draft_table_gathers = 0;
    std::uint64_t verify_table_gathers = 0;
};

std::string counters_to_json(const cache_counters& c);

struct snapshot_handle {
    std::uint64_t owner = 0;
    std::uint64_t serial = 0;
    std::size_t slot = 0;
};

// Single-owner decode stream.  Constructed from a config (the reference's form,
// cache.hpp:45) the state hashes on a shared hash-only device bank; the first draft_verify /
// memo lookup against a bank with tables moves the state onto that bank's device copy.
class sequence_cache {
  public:
    explicit sequence_cache(const ngram_config& cfg);
    explicit sequence_cache(const device_bank& bank);
    std::vector<std::uint64_t> append(token_id token, cache_counters* counters = nullptr);
    snapshot_handle snapshot();
    void rollback(const snapshot_handle& h, cache_counters* counters = nullptr);
    void discard(const snapshot_handle& h);
    std::uint64_t length() const;
    std::size_t snapshot_depth() const { return snaps_.size(); }
    token_id last_token() const;
    const ngram_config& config() const { return cfg_; }
    // The trailing N-1 confirmed tokens, oldest first (a view valid until the next call on
    // this state, as the reference's span into its ring).
    std::span<const token_id> ring() const;
    ngram_decode* handle() const { return st_.get(); }
    // Move the state (ring, length, last) onto `bank`'s device copy if it lives elsewhere, so
    // verify blocks gather from that bank's tables.
    void bind(const device_bank& bank);

  private:
    struct snap {
        std::uint64_t serial, length;
        token_id last;
        std::vector<token_id> ring;
    };
    void check(const snapshot_handle& h) const;
    void restore(const snap& s);
    ngram_config cfg_;
    std::shared_ptr<ngram_bank> bank_;  // the device bank the decode state runs on
    std::shared_ptr<ngram_decode> st_;
    mutable std::vector<token_id> ring_view_;
    std::uint64_t uid_ = 0, next_serial_ = 1;
    std::vector<snap> snaps_;
};

// embedding_memo (cache.hpp:82-113, cache.cpp:98-150): an LRU of merged (pre-amplification)
// vectors keyed by the exact (token, bucket ids); a miss runs embed_from_ids on the GPU and
// inserts, a hit returns the stored vector (bit-identical to recomputing).  draft_verify does
// not need it on the GPU -- a verify block computes every draft position in one launch and
// the accepted prefix is read from it -- but direct lookups behave as the reference's.
// Externally synchronised when shared, as the reference's.
class embedding_memo {
  public:
    explicit embedding_memo(std::size_t capacity) : capacity_(capacity) {
        if (capacity_ < 1) throw std::invalid_argument("embedding_memo: capacity must be >= 1");
    }
    std::vector<float> lookup(token_id token, std::span<const std::uint64_t> ids, const device_bank& bank,
                              cache_counters* counters = nullptr);
    std::vector<float> lookup(token_id token, std::span<const std::uint64_t> ids, const embedding_bank& bank,
                              cache_counters* counters = nullptr);
    std::size_t capacity() const { return capacity_; }
    std::size_t size() const { return lru_.size(); }

  private:
    using key = std::vector<std::uint64_t>;  // token, then the ids
    std::size_t capacity_;
    std::list<std::pair<key, std::vector<float>>> lru_;  // front = most recently used
    std::map<key, decltype(lru_)::iterator> where_;
};

struct draft_options {
    bool conventional_draft_embedding = false;
};

struct draft_result {
    std::vector<std::vector<float>> accepted;  // merged (pre-amplification) embeddings
};

// draft_verify (cache.cpp:152-195): verify block + commit of the accepted prefix.
draft_result draft_verify(sequence_cache& state, const device_bank& bank, std::span<const token_id> draft,
                          std::size_t accept_count, cache_counters* counters = nullptr, const draft_options& opts = {});
draft_result draft_verify(sequence_cache& state, embedding_memo& memo, const device_bank& bank,
                          std::span<const token_id> draft, std::size_t accept_count, cache_counters* counters = nullptr,
                          const draft_options& opts = {});
// The reference's signature (cache.hpp:131-136): the host bank's device copy is cached
// (see device_bank_for), so repeated rounds against one bank upload it once.
draft_result draft_verify(sequence_cache& state, embedding_memo& memo, const embedding_bank& bank,
                          std::span<const token_id> draft, std::size_t accept_count, cache_counters* counters = nullptr,
                          const draft_options& opts = {});

}  // namespace ngram
