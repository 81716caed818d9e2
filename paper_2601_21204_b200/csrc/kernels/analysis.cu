// analysis.cu -- corpus collision analysis on the device (corpus_analyzer, analysis.cpp:93-121;
// SURVEY.md 8(f) row 4).  Every position of every sequence contributes one zero-padded window
// per order (no carry across sequences, analysis.cpp:104-112).  The window's exact identity is
// its polynomial value poly = sum_j V0^j * tok[pos-j] (newest token weight V0^0, < 2^128 by the
// constructor's check), its bucket under modulus m is poly mod m -- congruent to the rolling
// hash of hashing.cpp:33-59, computed here directly from the 128-bit value:
//   m <= 2^32: poly mod m = ((hi mod m) * (2^64 mod m) + lo mod m) mod m, four Barrett steps;
//   m >  2^32: the 128-bit remainder.
// Distinct windows per order live in an open-addressing set of 128-bit keys (linear probing,
// inserted with atom.global.cas.b128; the all-ones key is never a valid window because
// V0^order <= 2^128 - 1).  Distinct buckets per (order, modulus) live in a bitmap of m bits
// (m <= 2^32) or in the same kind of set.  New-entry counts are aggregated per warp before one
// atomicAdd.  The host (csrc/host/analysis.cpp) keeps every set at load <= 1/2.
//
// HBM / L2 bound integer work: per position n_orders * (n token loads, cached) plus one
// 16-byte CAS per order and one 8-byte atomicOr (or CAS) per (order, modulus).
#include <algorithm>

#include "hashdev.cuh"
#include "kernels.h"

namespace ngk {
namespace {

constexpr unsigned long long kEmpty = ~0ull;

__device__ __forceinline__ ulonglong2 cas128(ulonglong2* p, unsigned long long clo, unsigned long long chi,
                                             unsigned long long vlo, unsigned long long vhi) {
    ulonglong2 old;
    asm volatile(
        "{\n\t.reg .b128 c, v, d;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 v, {%4, %5};\n\t"
        "atom.global.cas.b128 d, [%6], c, v;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(old.x), "=l"(old.y)
        : "l"(clo), "l"(chi), "l"(vlo), "l"(vhi), "l"(p)
        : "memory");
    return old;
}

__device__ __forceinline__ ulonglong2 ld_cg128(const ulonglong2* p) {
    ulonglong2 v;
    asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
    return v;
}

__device__ __forceinline__ uint64_t mix128(uint64_t lo, uint64_t hi) {
    uint64_t x = lo ^ (hi * 0x9e3779b97f4a7c15ull);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

// true when (lo, hi) was not yet in the set.  Every slot goes EMPTY -> key exactly once, so a
// plain read that already shows the key proves a duplicate -- except a torn read (one half
// EMPTY) could fake a key with an all-ones half, so those keys always take the CAS.
__device__ bool set_insert(const AnSet& s, uint64_t lo, uint64_t hi, unsigned long long* err) {
    uint64_t slot = mix128(lo, hi) & s.mask;
    const bool fast = lo != kEmpty && hi != kEmpty;
    for (uint64_t probe = 0; probe <= s.mask; ++probe) {
        ulonglong2* p = s.slots + slot;
        if (fast) {
            const ulonglong2 cur = ld_cg128(p);
            if (cur.x == lo && cur.y == hi) return false;
        }
        const ulonglong2 old = cas128(p, kEmpty, kEmpty, lo, hi);
        if (old.x == kEmpty && old.y == kEmpty) return true;
        if (old.x == lo && old.y == hi) return false;
        slot = (slot + 1) & s.mask;
    }
    atomicExch(err, 1ull);  // full table: the host's load bound was violated
    return false;
}

__device__ __forceinline__ void warp_count(bool is_new, unsigned long long* counter) {
    const unsigned m = __ballot_sync(0xffffffffu, is_new);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(counter, (unsigned long long)__popc(m));
}

__device__ __forceinline__ uint64_t poly_mod(unsigned __int128 poly, uint64_t m, uint64_t mu, uint64_t c64) {
    if (m <= 1) return 0;
    if (mu) {  // m <= 2^32
        const uint64_t lo = barrett_mod((uint64_t)poly, m, mu);
        const uint64_t hi = barrett_mod((uint64_t)(poly >> 64), m, mu);
        uint64_t r = barrett_mod(hi * c64, m, mu) + lo;  // < 2m
        return r >= m ? r - m : r;
    }
    return (uint64_t)(poly % m);
}

// Thread per position t < limit (positions >= limit belong to or follow the first sequence
// holding a bad token, analysis.cpp:101-106).  The loop bound is warp-uniform so the
// per-warp ballots see every lane.
// New-entry counters: per block in shared memory (one global atomicAdd per counter per block
// at the end) when they fit, else straight to global.  All counters of an analyzer share a
// few L2 lines, so per-warp global atomics would serialise on one L2 slice.
__global__ void __launch_bounds__(256) an_insert_kernel(AnDev a, const uint32_t* __restrict__ tokens,
                                                        const int64_t* __restrict__ off, int64_t nseq,
                                                        const unsigned long long* __restrict__ limit_p,
                                                        int smem_counts) {
    extern __shared__ unsigned long long s_cnt[];
    const int ncnt = a.n_orders * (1 + a.n_moduli);
    if (smem_counts) {
        for (int i = threadIdx.x; i < ncnt; i += blockDim.x) s_cnt[i] = 0;
        __syncthreads();
    }
    unsigned long long* cnt = smem_counts ? s_cnt : a.counts;
    const int64_t limit = (int64_t)*limit_p;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < limit; base += stride) {
        const int64_t t = base + threadIdx.x;
        const bool live = t < limit;
        int64_t p = 0;
        if (live) p = t - __ldg(off + find_seq(off, nseq, t));
        for (int oi = 0; oi < a.n_orders; ++oi) {
            const int n = a.orders[oi];
            unsigned __int128 poly = 0;
            if (live) {
                const int jn = p + 1 < (int64_t)n ? (int)(p + 1) : n;
                for (int j = 0; j < jn; ++j) {
                    const ulonglong2 vp = a.vpow[j];
                    const unsigned __int128 w = ((unsigned __int128)vp.y << 64) | vp.x;
                    poly += w * __ldg(tokens + t - j);
                }
            }
            const uint64_t plo = (uint64_t)poly, phi = (uint64_t)(poly >> 64);
            const bool nw = live && set_insert(a.ngram_sets[oi], plo, phi, a.err);
            warp_count(nw, cnt + oi);
            for (int mi = 0; mi < a.n_moduli; ++mi) {
                const int k = oi * a.n_moduli + mi;
                bool bn = false;
                if (live) {
                    const uint64_t bucket = poly_mod(poly, a.moduli[mi], a.barrett[mi], a.c64[mi]);
                    const AnBucket& bk = a.buckets[k];
                    if (bk.bits) {  // a plain read first: most bits are set after warm-up
                        unsigned long long* w = bk.bits + (bucket >> 6);
                        const unsigned long long bit = 1ull << (bucket & 63);
                        if (!(*reinterpret_cast<volatile unsigned long long*>(w) & bit))
                            bn = !(atomicOr(w, bit) & bit);
                    } else {
                        bn = set_insert(bk.set, bucket, 0, a.err);
                    }
                }
                warp_count(bn, cnt + a.n_orders + k);
            }
        }
    }
    if (smem_counts) {
        __syncthreads();
        for (int i = threadIdx.x; i < ncnt; i += blockDim.x)
            if (s_cnt[i]) atomicAdd(a.counts + i, s_cnt[i]);
    }
}

__global__ void an_validate_kernel(const uint32_t* __restrict__ tokens, int64_t T, uint64_t V0,
                                   unsigned long long* first_bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += stride)
        if (__ldg(tokens + t) >= V0) atomicMin(first_bad, (unsigned long long)t);
}

// One thread: the counters of this call (analysis.cpp:98-100: a sequence counts, with its full
// length, as soon as it is started; positions before the first bad token are inserted) and the
// insert limit; records the first error of the analyzer (position, token) for the host.
__global__ void an_account_kernel(const uint32_t* __restrict__ tokens, const int64_t* __restrict__ off,
                                  int64_t nseq, unsigned long long* first_bad, unsigned long long* meta,
                                  int n_orders, unsigned long long* err_pos) {
    const int64_t T = off[nseq];
    const unsigned long long g = *first_bad;
    int64_t limit = T, seqs = nseq, toks = T;
    if (g != kEmpty) {
        int64_t lo = 0, hi = nseq - 1;  // sequence holding position g: largest s with off[s] <= g
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (off[mid] <= (int64_t)g) lo = mid;
            else hi = mid - 1;
        }
        limit = (int64_t)g;
        seqs = lo + 1;
        toks = off[lo + 1];
        if (err_pos[0] == kEmpty) {
            err_pos[0] = g;
            err_pos[1] = tokens[g];
        }
    }
    meta[0] += (unsigned long long)seqs;
    meta[1] += (unsigned long long)toks;
    for (int oi = 0; oi < n_orders; ++oi) meta[2 + oi] += (unsigned long long)limit;
    *first_bad = (unsigned long long)limit;  // reused as the insert limit
}

__global__ void an_rehash_kernel(const ulonglong2* __restrict__ old_slots, uint64_t old_n, AnSet dst,
                                 unsigned long long* err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)old_n; i += stride) {
        const ulonglong2 k = old_slots[i];
        if (!(k.x == kEmpty && k.y == kEmpty)) set_insert(dst, k.x, k.y, err);
    }
}

__global__ void __launch_bounds__(256) an_merge_set_kernel(const ulonglong2* __restrict__ src, uint64_t n, AnSet dst,
                                                           unsigned long long* counter, unsigned long long* err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < (int64_t)n; base += stride) {
        const int64_t i = base + threadIdx.x;
        bool nw = false;
        if (i < (int64_t)n) {
            const ulonglong2 k = src[i];
            if (!(k.x == kEmpty && k.y == kEmpty)) nw = set_insert(dst, k.x, k.y, err);
        }
        warp_count(nw, counter);
    }
}

__global__ void __launch_bounds__(256) an_merge_bits_kernel(const unsigned long long* __restrict__ src, uint64_t nw,
                                                            unsigned long long* dst, unsigned long long* counter) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < (int64_t)nw; base += stride) {
        const int64_t i = base + threadIdx.x;
        int add = 0;
        if (i < (int64_t)nw) {
            const unsigned long long s = src[i];
            if (s) add = __popcll(s & ~atomicOr(dst + i, s));
        }
        for (int o = 16; o; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
        if ((threadIdx.x & 31) == 0 && add) atomicAdd(counter, (unsigned long long)add);
    }
}

__global__ void an_merge_meta_kernel(const unsigned long long* __restrict__ src, unsigned long long* dst, int n) {
    if (threadIdx.x < n) dst[threadIdx.x] += src[threadIdx.x];
}

int grid_for(int64_t n, int num_sms) {
    const int64_t b = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms * 8));
}

}  // namespace

void launch_an_add(const AnDev& a, const uint32_t* tokens, const int64_t* off, int64_t nseq, int64_t T,
                   unsigned long long* first_bad, unsigned long long* meta, unsigned long long* err_pos,
                   int num_sms, cudaStream_t st) {
    if (T > 0) {
        an_validate_kernel<<<grid_for(T, num_sms), 256, 0, st>>>(tokens, T, a.V0, first_bad);
        count_launch();
    }
    an_account_kernel<<<1, 1, 0, st>>>(tokens, off, nseq, first_bad, meta, a.n_orders, err_pos);
    count_launch();
    if (T > 0) {
        const int ncnt = a.n_orders * (1 + a.n_moduli);
        const int smem = ncnt <= 6144 ? ncnt * 8 : 0;
        an_insert_kernel<<<grid_for(T, num_sms), 256, smem, st>>>(a, tokens, off, nseq, first_bad, smem != 0);
        count_launch();
    }
}

void launch_an_rehash(const ulonglong2* old_slots, uint64_t old_n, const AnSet& dst, unsigned long long* err,
                      int num_sms, cudaStream_t st) {
    an_rehash_kernel<<<grid_for((int64_t)old_n, num_sms), 256, 0, st>>>(old_slots, old_n, dst, err);
    count_launch();
}

void launch_an_merge_set(const ulonglong2* src, uint64_t n, const AnSet& dst, unsigned long long* counter,
                         unsigned long long* err, int num_sms, cudaStream_t st) {
    an_merge_set_kernel<<<grid_for((int64_t)n, num_sms), 256, 0, st>>>(src, n, dst, counter, err);
    count_launch();
}

void launch_an_merge_bits(const unsigned long long* src, uint64_t nwords, unsigned long long* dst,
                          unsigned long long* counter, int num_sms, cudaStream_t st) {
    an_merge_bits_kernel<<<grid_for((int64_t)nwords, num_sms), 256, 0, st>>>(src, nwords, dst, counter);
    count_launch();
}

void launch_an_merge_meta(const unsigned long long* src, unsigned long long* dst, int n, cudaStream_t st) {
    an_merge_meta_kernel<<<1, 64, 0, st>>>(src, dst, n);
    count_launch();
}

}  // namespace ngk
