// shard.cpp -- placeholder, replaced by the row-sharded exchange.
#include "api_util.hpp"
#include "bank.hpp"
using namespace ngh;
extern "C" {
int ngram_shard_group_create(ngram_bank*, int64_t, ngram_shard_group**) { return set_error(NGRAM_EINVAL, "not built"); }
int ngram_shard_group_destroy(ngram_shard_group*) { return NGRAM_OK; }
int ngram_shard_export(ngram_shard_group*, void*) { return set_error(NGRAM_EINVAL, "not built"); }
int ngram_shard_open(ngram_shard_group*, int, const void*) { return set_error(NGRAM_EINVAL, "not built"); }
int ngram_shard_scatter_rows(ngram_shard_group*, const uint32_t*, const int64_t*, int64_t, int64_t, const int64_t*,
                             const uint32_t*, void*) { return set_error(NGRAM_EINVAL, "not built"); }
int ngram_shard_project(ngram_shard_group*, const uint32_t*, int64_t, void*, void*, int, void*) {
    return set_error(NGRAM_EINVAL, "not built");
}
}
