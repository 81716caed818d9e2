// analysis.cpp -- C-ABI of the device corpus analyzer (corpus_analyzer, analysis.hpp:45-93,
// analysis.cpp:44-176).  Kernels in kernels/analysis.cu.
//
// State on the device: per order an open-addressing set of the exact 128-bit window values,
// per (order, modulus) a bitmap of m bits (m <= 2^32) or a set of buckets, the distinct
// counters, and [sequences, tokens, ngrams_seen per order].  The host keeps an upper bound on
// every set's occupancy (last synchronised count + positions submitted since) and grows a set
// (rehash into twice the slots) before an add could push it past load 1/2, synchronising only
// when the bound says it might.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "api_util.hpp"
#include "bank.hpp"

using namespace ngh;

namespace {

constexpr uint64_t kBitmapMax = uint64_t(1) << 32;  // moduli up to 2^32 use a bitmap (512 MiB)
constexpr uint64_t kMinSlots = uint64_t(1) << 12;
constexpr int kMaxOrders = 62;                       // meta = 2 + n_orders words, one merge block

struct DevSet {
    DevBuf<ulonglong2> slots;
    uint64_t n = 0;      // slots (power of two)
    uint64_t bound = 0;  // upper bound on occupied slots
    uint64_t limit = ~uint64_t(0);  // keys can never exceed this (buckets of a modulus)
};

uint64_t pow2_at_least(uint64_t x) {
    uint64_t p = kMinSlots;
    while (p < x) p <<= 1;
    return p;
}

}  // namespace

struct ngram_analyzer {
    int device = 0;
    int num_sms = 148;
    uint64_t V0 = 0;
    std::vector<int> orders;
    std::vector<uint64_t> moduli;
    int max_order = 0;

    DevBuf<int> d_orders;
    DevBuf<ulonglong2> d_vpow;
    DevBuf<uint64_t> d_moduli, d_barrett, d_c64;
    std::vector<DevSet> sets;                   // [n_orders]
    std::vector<DevSet> bsets;                  // [n_orders * n_moduli] (large moduli only)
    std::vector<DevBuf<unsigned long long>> bits;  // [n_orders * n_moduli] (bitmap moduli)
    std::vector<uint64_t> nwords;               // bitmap words per modulus (0: set)
    DevBuf<ngk::AnSet> d_sets;
    DevBuf<ngk::AnBucket> d_buckets;
    DevBuf<unsigned long long> counts;  // [n_orders + n_orders * n_moduli]
    DevBuf<unsigned long long> meta;    // [2 + n_orders]
    DevBuf<unsigned long long> scratch; // [0] first bad / insert limit, [1] overflow flag, [2..3] first error
    DevBuf<uint32_t> h_tok;
    DevBuf<int64_t> h_off;
    std::mutex mu;

    size_t n_pairs() const { return orders.size() * moduli.size(); }

    ngk::AnDev dev() {
        ngk::AnDev a{};
        a.V0 = V0;
        a.n_orders = int(orders.size());
        a.n_moduli = int(moduli.size());
        a.orders = d_orders.p;
        a.vpow = d_vpow.p;
        a.moduli = d_moduli.p;
        a.barrett = d_barrett.p;
        a.c64 = d_c64.p;
        a.ngram_sets = d_sets.p;
        a.buckets = d_buckets.p;
        a.counts = counts.p;
        a.err = scratch.p + 1;
        return a;
    }

    // Upload the set / bitmap descriptors (after creation or a grow; the stream is idle).
    void upload_descriptors() {
        std::vector<ngk::AnSet> hs(orders.size());
        for (size_t i = 0; i < orders.size(); ++i) hs[i] = {sets[i].slots.p, sets[i].n - 1};
        std::vector<ngk::AnBucket> hb(n_pairs());
        for (size_t k = 0; k < n_pairs(); ++k) {
            hb[k].bits = bits[k].p;
            hb[k].set = {bsets[k].slots.p, bsets[k].n ? bsets[k].n - 1 : 0};
        }
        NGH_CUDA(cudaMemcpy(d_sets.p, hs.data(), hs.size() * sizeof(ngk::AnSet), cudaMemcpyHostToDevice));
        NGH_CUDA(cudaMemcpy(d_buckets.p, hb.data(), hb.size() * sizeof(ngk::AnBucket), cudaMemcpyHostToDevice));
    }

    void alloc_set(DevSet& s, uint64_t n) {
        s.slots.alloc(size_t(n));
        NGH_CUDA(cudaMemset(s.slots.p, 0xff, size_t(n) * sizeof(ulonglong2)));
        s.n = n;
    }

    // Make every set able to take `extra` more keys at load <= 1/2.  Synchronises only when
    // an upper bound says a set might overflow.
    void reserve(uint64_t extra, cudaStream_t st) {
        auto need = [&](const DevSet& s) {
            return s.n && std::min(s.bound + extra, s.limit) > s.n / 2;
        };
        bool any = false;
        for (auto& s : sets) any |= need(s);
        for (auto& s : bsets) any |= need(s);
        if (!any) return;
        NGH_CUDA(cudaStreamSynchronize(st));
        std::vector<unsigned long long> c(counts.n);
        NGH_CUDA(cudaMemcpy(c.data(), counts.p, counts.n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        const size_t no = orders.size();
        bool grown = false;
        auto grow = [&](DevSet& s, uint64_t count) {
            s.bound = count;
            const uint64_t want = std::min(count + extra, s.limit);
            if (want <= s.n / 2) return;
            DevSet ns;
            alloc_set(ns, pow2_at_least(2 * want));
            ns.bound = count;
            ns.limit = s.limit;
            ngk::launch_an_rehash(s.slots.p, s.n, ngk::AnSet{ns.slots.p, ns.n - 1}, scratch.p + 1, num_sms, st);
            NGH_CUDA(cudaStreamSynchronize(st));
            std::swap(s.slots.p, ns.slots.p);
            std::swap(s.slots.n, ns.slots.n);
            s.n = ns.n;
            grown = true;
        };
        for (size_t i = 0; i < no; ++i) grow(sets[i], c[i]);
        for (size_t k = 0; k < n_pairs(); ++k)
            if (bsets[k].n) grow(bsets[k], c[no + k]);
        if (grown) upload_descriptors();
    }

    void account(uint64_t positions) {
        for (auto& s : sets) s.bound += positions;
        for (auto& s : bsets)
            if (s.n) s.bound = std::min(s.bound + positions, s.limit);
    }

    // Overflow of a device set (internal invariant) always; the first out-of-range token of
    // the adds since the last check when `range` (then cleared).
    void check_errors(cudaStream_t st, bool range) {
        unsigned long long e[3];
        NGH_CUDA(cudaMemcpyAsync(e, scratch.p + 1, sizeof(e), cudaMemcpyDeviceToHost, st));
        NGH_CUDA(cudaStreamSynchronize(st));
        if (e[0]) throw Error(NGRAM_ECUDA, "corpus analyzer: a device set overflowed (internal load bound violated)");
        if (range && e[1] != ~0ull) {
            const unsigned long long clear[2] = {~0ull, ~0ull};
            NGH_CUDA(cudaMemcpy(scratch.p + 2, clear, sizeof(clear), cudaMemcpyHostToDevice));
            throw Error(NGRAM_ERANGE, "corpus_analyzer: token " + std::to_string(e[2]) +
                                          " out of range for base vocabulary " + std::to_string(V0));
        }
    }

    void add(const uint32_t* tokens, const int64_t* off, int64_t nseq, int64_t T, cudaStream_t st) {
        reserve(uint64_t(T), st);
        NGH_CUDA(cudaMemsetAsync(scratch.p, 0xff, sizeof(unsigned long long), st));
        ngk::launch_an_add(dev(), tokens, off, nseq, T, scratch.p, meta.p, scratch.p + 2, num_sms, st);
        NGH_CUDA(cudaGetLastError());
        account(uint64_t(T));
    }
};

namespace {

void check_same(const ngram_analyzer* a, const ngram_analyzer* b) {
    if (a->V0 != b->V0 || a->orders != b->orders || a->moduli != b->moduli)
        throw Error(NGRAM_EINVAL, "corpus_analyzer: merge of mismatched analyzers");
    if (a->device != b->device) throw Error(NGRAM_EINVAL, "corpus_analyzer: merge across devices is not supported");
}

}  // namespace

extern "C" {

int ngram_analyzer_create(int device, uint64_t base_vocab, const int* orders, int n_orders, const uint64_t* moduli,
                          int n_moduli, ngram_analyzer** out) {
    NGRAM_API_BEGIN
    if (!out) throw Error(NGRAM_EINVAL, "ngram_analyzer_create: null out");
    *out = nullptr;
    // analysis.cpp:44-77: the reference's checks and messages, in its order
    if (base_vocab < 2) throw Error(NGRAM_EINVAL, "corpus_analyzer: base vocabulary must be >= 2");
    if (n_orders < 1 || n_moduli < 1 || !orders || !moduli)
        throw Error(NGRAM_EINVAL, "corpus_analyzer: need at least one order and one modulus");
    if (n_orders > kMaxOrders) throw Error(NGRAM_EINVAL, "corpus_analyzer: at most 62 orders per analyzer");
    int max_order = 0;
    for (int i = 0; i < n_orders; ++i) {
        if (orders[i] < 2) throw Error(NGRAM_EINVAL, "corpus_analyzer: orders must be >= 2");
        max_order = std::max(max_order, orders[i]);
    }
    for (int i = 0; i < n_moduli; ++i)
        if (moduli[i] < 1) throw Error(NGRAM_EINVAL, "corpus_analyzer: moduli must be >= 1");
    std::vector<ulonglong2> vpow(size_t(max_order) + 1);
    unsigned __int128 pw = 1;
    vpow[0] = {1ull, 0ull};
    for (int j = 1; j <= max_order; ++j) {
        if (pw > (~(unsigned __int128)0) / base_vocab)
            throw Error(NGRAM_EINVAL,
                        "corpus_analyzer: V0^order exceeds 128 bits; exact distinct n-gram counting is limited to "
                        "order*log2(V0) < 128");
        pw *= base_vocab;
        vpow[size_t(j)] = {(unsigned long long)pw, (unsigned long long)(pw >> 64)};
    }
    DeviceGuard g(device);
    auto a = std::make_unique<ngram_analyzer>();
    a->device = device;
    NGH_CUDA(cudaDeviceGetAttribute(&a->num_sms, cudaDevAttrMultiProcessorCount, device));
    a->V0 = base_vocab;
    a->orders.assign(orders, orders + n_orders);
    a->moduli.assign(moduli, moduli + n_moduli);
    a->max_order = max_order;
    std::vector<uint64_t> mu(static_cast<size_t>(n_moduli)), c64(static_cast<size_t>(n_moduli));
    for (int i = 0; i < n_moduli; ++i) {
        const uint64_t m = moduli[i];
        const bool fast = m >= 2 && m <= kBitmapMax;
        mu[size_t(i)] = fast ? uint64_t(((unsigned __int128)1 << 64) / m) : 0;
        c64[size_t(i)] = m >= 2 ? uint64_t(((unsigned __int128)1 << 64) % m) : 0;
    }
    a->d_orders.alloc(size_t(n_orders));
    a->d_vpow.alloc(vpow.size());
    a->d_moduli.alloc(size_t(n_moduli));
    a->d_barrett.alloc(size_t(n_moduli));
    a->d_c64.alloc(size_t(n_moduli));
    NGH_CUDA(cudaMemcpy(a->d_orders.p, orders, size_t(n_orders) * sizeof(int), cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(a->d_vpow.p, vpow.data(), vpow.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(a->d_moduli.p, moduli, size_t(n_moduli) * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(a->d_barrett.p, mu.data(), size_t(n_moduli) * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(a->d_c64.p, c64.data(), size_t(n_moduli) * 8, cudaMemcpyHostToDevice));

    a->sets.resize(size_t(n_orders));
    for (auto& s : a->sets) a->alloc_set(s, kMinSlots);
    const size_t np = a->n_pairs();
    a->bsets.resize(np);
    a->bits.resize(np);
    a->nwords.assign(size_t(n_moduli), 0);
    for (int mi = 0; mi < n_moduli; ++mi)
        if (moduli[mi] <= kBitmapMax) a->nwords[size_t(mi)] = (moduli[mi] + 63) / 64;
    for (int oi = 0; oi < n_orders; ++oi)
        for (int mi = 0; mi < n_moduli; ++mi) {
            const size_t k = size_t(oi) * size_t(n_moduli) + size_t(mi);
            if (a->nwords[size_t(mi)]) {
                a->bits[k].alloc(size_t(a->nwords[size_t(mi)]));
                NGH_CUDA(cudaMemset(a->bits[k].p, 0, size_t(a->nwords[size_t(mi)]) * 8));
            } else {
                a->bsets[k].limit = moduli[mi];
                a->alloc_set(a->bsets[k], kMinSlots);
            }
        }
    a->d_sets.alloc(size_t(n_orders));
    a->d_buckets.alloc(np);
    a->upload_descriptors();
    a->counts.alloc(size_t(n_orders) + np);
    NGH_CUDA(cudaMemset(a->counts.p, 0, a->counts.n * 8));
    a->meta.alloc(size_t(2 + n_orders));
    NGH_CUDA(cudaMemset(a->meta.p, 0, a->meta.n * 8));
    a->scratch.alloc(4);
    const unsigned long long init[4] = {~0ull, 0ull, ~0ull, ~0ull};
    NGH_CUDA(cudaMemcpy(a->scratch.p, init, sizeof(init), cudaMemcpyHostToDevice));
    *out = a.release();
    NGRAM_API_END
}

void ngram_analyzer_destroy(ngram_analyzer* a) {
    if (!a) return;
    DeviceGuard g(a->device);
    cudaDeviceSynchronize();
    delete a;
}

int ngram_analyzer_add(ngram_analyzer* a, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq, int64_t T,
                       void* stream) {
    NGRAM_API_BEGIN
    if (!a || !seq_offsets || nseq < 0 || T < 0 || (T > 0 && !tokens))
        throw Error(NGRAM_EINVAL, "ngram_analyzer_add: bad argument");
    if (nseq == 0) return NGRAM_OK;
    std::lock_guard<std::mutex> lk(a->mu);
    DeviceGuard g(a->device);
    a->add(tokens, seq_offsets, nseq, T, static_cast<cudaStream_t>(stream));
    NGRAM_API_END
}

int ngram_analyzer_add_host(ngram_analyzer* a, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq) {
    NGRAM_API_BEGIN
    if (!a || !seq_offsets || nseq < 0) throw Error(NGRAM_EINVAL, "ngram_analyzer_add_host: bad argument");
    if (nseq == 0) return NGRAM_OK;
    if (seq_offsets[0] != 0) throw Error(NGRAM_EINVAL, "seq_offsets must start at 0");
    for (int64_t i = 0; i < nseq; ++i)
        if (seq_offsets[i + 1] < seq_offsets[i]) throw Error(NGRAM_EINVAL, "seq_offsets must be non-decreasing");
    const int64_t T = seq_offsets[nseq];
    if (T > 0 && !tokens) throw Error(NGRAM_EINVAL, "ngram_analyzer_add_host: null tokens");
    std::lock_guard<std::mutex> lk(a->mu);
    DeviceGuard g(a->device);
    a->h_tok.ensure(size_t(std::max<int64_t>(T, 1)));
    a->h_off.ensure(size_t(nseq + 1));
    if (T > 0) NGH_CUDA(cudaMemcpy(a->h_tok.p, tokens, size_t(T) * 4, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(a->h_off.p, seq_offsets, size_t(nseq + 1) * 8, cudaMemcpyHostToDevice));
    a->add(a->h_tok.p, a->h_off.p, nseq, T, nullptr);
    a->check_errors(nullptr, true);  // the reference throws out_of_range from add_sequence itself
    NGRAM_API_END
}

int ngram_analyzer_merge(ngram_analyzer* dst, ngram_analyzer* src, void* stream) {
    NGRAM_API_BEGIN
    if (!dst || !src) throw Error(NGRAM_EINVAL, "ngram_analyzer_merge: null analyzer");
    if (dst == src) throw Error(NGRAM_EINVAL, "ngram_analyzer_merge: an analyzer cannot merge itself");
    check_same(dst, src);
    std::scoped_lock lk(dst->mu, src->mu);
    DeviceGuard g(dst->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the union can add at most the source's distinct counts to each set
    NGH_CUDA(cudaStreamSynchronize(st));
    NGH_CUDA(cudaDeviceSynchronize());  // src may have work on another stream
    std::vector<unsigned long long> c(src->counts.n);
    NGH_CUDA(cudaMemcpy(c.data(), src->counts.p, c.size() * 8, cudaMemcpyDeviceToHost));
    uint64_t most = 0;
    for (auto v : c) most = std::max<uint64_t>(most, v);
    dst->reserve(most, st);
    const size_t no = dst->orders.size(), nm = dst->moduli.size();
    for (size_t i = 0; i < no; ++i)
        ngk::launch_an_merge_set(src->sets[i].slots.p, src->sets[i].n,
                                 ngk::AnSet{dst->sets[i].slots.p, dst->sets[i].n - 1}, dst->counts.p + i,
                                 dst->scratch.p + 1, dst->num_sms, st);
    for (size_t oi = 0; oi < no; ++oi)
        for (size_t mi = 0; mi < nm; ++mi) {
            const size_t k = oi * nm + mi;
            if (dst->nwords[mi])
                ngk::launch_an_merge_bits(src->bits[k].p, dst->nwords[mi], dst->bits[k].p, dst->counts.p + no + k,
                                          dst->num_sms, st);
            else
                ngk::launch_an_merge_set(src->bsets[k].slots.p, src->bsets[k].n,
                                         ngk::AnSet{dst->bsets[k].slots.p, dst->bsets[k].n - 1},
                                         dst->counts.p + no + k, dst->scratch.p + 1, dst->num_sms, st);
        }
    ngk::launch_an_merge_meta(src->meta.p, dst->meta.p, int(dst->meta.n), st);
    NGH_CUDA(cudaGetLastError());
    for (size_t i = 0; i < no; ++i) dst->sets[i].bound += c[i];
    for (size_t k = 0; k < dst->n_pairs(); ++k)
        if (dst->bsets[k].n) dst->bsets[k].bound = std::min<uint64_t>(dst->bsets[k].bound + c[no + k], dst->bsets[k].limit);
    NGRAM_API_END
}

int ngram_analyzer_reserve(ngram_analyzer* a, uint64_t windows) {
    NGRAM_API_BEGIN
    if (!a) throw Error(NGRAM_EINVAL, "ngram_analyzer_reserve: null analyzer");
    std::lock_guard<std::mutex> lk(a->mu);
    DeviceGuard g(a->device);
    // like unordered_set::reserve: grow now so the next `windows` positions add no rehash
    a->reserve(windows, nullptr);
    NGRAM_API_END
}

int ngram_analyzer_sync_errors(ngram_analyzer* a) {
    NGRAM_API_BEGIN
    if (!a) throw Error(NGRAM_EINVAL, "ngram_analyzer_sync_errors: null analyzer");
    std::lock_guard<std::mutex> lk(a->mu);
    DeviceGuard g(a->device);
    NGH_CUDA(cudaDeviceSynchronize());
    a->check_errors(nullptr, true);
    NGRAM_API_END
}

int ngram_analyzer_stats(ngram_analyzer* a, uint64_t* sequences, uint64_t* tokens, uint64_t* ngrams_seen,
                         uint64_t* distinct_ngrams, uint64_t* distinct_buckets) {
    NGRAM_API_BEGIN
    if (!a) throw Error(NGRAM_EINVAL, "ngram_analyzer_stats: null analyzer");
    std::lock_guard<std::mutex> lk(a->mu);
    DeviceGuard g(a->device);
    NGH_CUDA(cudaDeviceSynchronize());
    a->check_errors(nullptr, false);
    const size_t no = a->orders.size();
    std::vector<unsigned long long> m(a->meta.n), c(a->counts.n);
    NGH_CUDA(cudaMemcpy(m.data(), a->meta.p, m.size() * 8, cudaMemcpyDeviceToHost));
    NGH_CUDA(cudaMemcpy(c.data(), a->counts.p, c.size() * 8, cudaMemcpyDeviceToHost));
    if (sequences) *sequences = m[0];
    if (tokens) *tokens = m[1];
    for (size_t i = 0; i < no; ++i) {
        if (ngrams_seen) ngrams_seen[i] = m[2 + i];
        if (distinct_ngrams) distinct_ngrams[i] = c[i];
    }
    if (distinct_buckets)
        for (size_t k = 0; k < a->n_pairs(); ++k) distinct_buckets[k] = c[no + k];
    // the bounds can tighten to the exact counts now
    for (size_t i = 0; i < no; ++i) a->sets[i].bound = c[i];
    for (size_t k = 0; k < a->n_pairs(); ++k)
        if (a->bsets[k].n) a->bsets[k].bound = c[no + k];
    NGRAM_API_END
}

}  // extern "C"
