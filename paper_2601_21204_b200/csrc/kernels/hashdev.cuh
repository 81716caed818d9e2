// hashdev.cuh -- device helpers of K1 shared by the hash kernels and the gather warps of
// the fused K1+K2+K3 kernel: Barrett / 128-bit modular products, the sequence lookup,
// and the warp-per-position hash + row gather (restating hashing.cpp:33-81 over the
// windows of embedding.hpp:391-405; see hash.cu for the exactness argument).
#pragma once
#include <cstdint>

#include "kernels.h"

namespace ngk {

__device__ __forceinline__ uint64_t barrett_mod(uint64_t x, uint64_t m, uint64_t mu) {
    const uint64_t q = __umul64hi(x, mu);
    uint64_t r = x - q * m;
    if (r >= m) r -= m;
    if (r >= m) r -= m;
    return r;
}

__device__ __forceinline__ uint64_t mulmod128(uint64_t a, uint64_t b, uint64_t m) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) % m);
}

// Position t of the concatenated batch -> sequence index (largest s with off[s] <= t).
__device__ __forceinline__ int64_t find_seq(const int64_t* __restrict__ off, int64_t nseq, int64_t t) {
    // equal-length batches (decode steps, verify blocks, uniform prefill): two dependent
    // loads instead of log2(nseq); the check keeps the result identical to the search below
    const int64_t total = __ldg(off + nseq);
    if (nseq > 1 && total > 0 && total % nseq == 0) {
        const int64_t sq = t / (total / nseq);
        if (sq < nseq && __ldg(off + sq) <= t && __ldg(off + sq + 1) > t) return sq;
    }
    int64_t lo = 0, hi = nseq - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Bucket of branch b for the window w (oldest first, N tokens):
//   h = sum_{j < n} (w[N-1-j] mod V_b) * (V0^j mod V_b)  mod V_b        (hashing.cpp:33-59)
// The loop runs over the window slot k = N-1-j (a compile-time register index; indexing w by
// the runtime N-1-j would put the window in local memory).  The terms are summed in another
// order than the reference's, which leaves the residue unchanged.  Common case (every token
// < V0 <= V_b <= 2^30): w mod V_b = w and each term < V_b^2 <= 2^60, so n <= 16 terms sum
// below 2^64 and ONE Barrett reduction of the plain sum gives the same residue.
template <int MAXN>
__device__ __forceinline__ uint64_t branch_hash(const Shape& s, const HashTables* __restrict__ ht,
                                                const uint32_t (&w)[MAXN], int b) {
    const int N = s.N;
    const int n = 2 + b / s.K;
    const uint64_t m = __ldg(&ht->modulus[b]);
    if (m <= 1) return 0;
    uint64_t acc = 0;
    if (s.fast_hash) {
        const uint64_t mu = __ldg(&ht->barrett[b]);
        if (m <= (1ull << 30) && (uint64_t)s.V0 <= m) {
#pragma unroll
            for (int k = 0; k < MAXN; ++k)
                if (k < N && k >= N - n) acc += (uint64_t)w[k] * (uint32_t)__ldg(&ht->pow[b][N - 1 - k]);
            return barrett_mod(acc, m, mu);
        }
#pragma unroll
        for (int k = 0; k < MAXN; ++k)
            if (k < N && k >= N - n) {
                const uint64_t tm = barrett_mod((uint64_t)w[k], m, mu);
                acc += barrett_mod(tm * __ldg(&ht->pow[b][N - 1 - k]), m, mu);
            }
        return barrett_mod(acc, m, mu);  // acc < n * 2^32
    }
#pragma unroll
    for (int k = 0; k < MAXN; ++k)
        if (k < N && k >= N - n) acc = (acc + mulmod128((uint64_t)w[k] % m, __ldg(&ht->pow[b][N - 1 - k]), m)) % m;
    return acc;
}

// A block's shared-memory copy of the hash constants of its B branches (moduli, Barrett
// factors, V0^j mod V_b, shard row ranges): one cooperative load, then every hash of the block
// reads shared memory instead of running a global-latency chain (hash_all_orders alone:
// 22.9 -> 14.3 us at config C).  load() must be reached by every thread of the block.
template <int MAXN>
struct HashSmem {
    uint64_t m[kMaxBranches], mu[kMaxBranches], pw[kMaxBranches][MAXN];
    int64_t lo[kMaxBranches], hi[kMaxBranches], base[kMaxBranches];

    __device__ __forceinline__ void load(const HashTables* __restrict__ ht, int B) {
        for (int i = threadIdx.x; i < B * MAXN; i += blockDim.x) {
            const int b = i / MAXN, j = i % MAXN;
            pw[b][j] = j < kMaxOrder ? __ldg(&ht->pow[b][j]) : 0ull;
            if (j == 0) {
                m[b] = __ldg(&ht->modulus[b]);
                mu[b] = __ldg(&ht->barrett[b]);
                lo[b] = __ldg(&ht->row_lo[b]);
                hi[b] = __ldg(&ht->row_hi[b]);
                base[b] = __ldg(&ht->row_base[b]);
            }
        }
        __syncthreads();
    }
    // branch_hash (above) from the shared copy: the same residue
    __device__ __forceinline__ uint64_t hash(const Shape& s, const uint32_t (&w)[MAXN], int b) const {
        const int N = s.N, n = 2 + b / s.K;
        const uint64_t mb = m[b];
        if (mb <= 1) return 0;
        uint64_t acc = 0;
        if (s.fast_hash) {
            const uint64_t mub = mu[b];
            if (mb <= (1ull << 30) && (uint64_t)s.V0 <= mb) {
#pragma unroll
                for (int k = 0; k < MAXN; ++k)
                    if (k < N && k >= N - n) acc += (uint64_t)w[k] * (uint32_t)pw[b][N - 1 - k];
            } else {
#pragma unroll
                for (int k = 0; k < MAXN; ++k)
                    if (k < N && k >= N - n)
                        acc += barrett_mod(barrett_mod((uint64_t)w[k], mb, mub) * pw[b][N - 1 - k], mb, mub);
            }
            return barrett_mod(acc, mb, mub);
        }
#pragma unroll
        for (int k = 0; k < MAXN; ++k)
            if (k < N && k >= N - n) acc = (acc + mulmod128((uint64_t)w[k] % mb, pw[b][N - 1 - k], mb)) % mb;
        return acc;
    }
    // storage_row (below) from the shared copy; -1 when the bucket is not on this shard
    __device__ __forceinline__ int32_t row(int b, uint64_t h) const {
        const int64_t hh = (int64_t)h;
        return (hh >= lo[b] && hh < hi[b]) ? (int32_t)(base[b] + (hh - lo[b])) : -1;
    }
};

// Storage row of bucket h of branch b on this shard (fallback row 0 when not local).
__device__ __forceinline__ int32_t storage_row(const HashTables* __restrict__ ht, int b, uint64_t h, bool* local) {
    const int64_t lo = __ldg(&ht->row_lo[b]), hi = __ldg(&ht->row_hi[b]);
    const bool in = (int64_t)h >= lo && (int64_t)h < hi;
    if (local) *local = in;
    return in ? (int32_t)(__ldg(&ht->row_base[b]) + ((int64_t)h - lo)) : 0;
}

// One warp: window of position t; returns false (warp-uniform) when it holds a token >= V0.
// uniform_len > 0: every sequence has that length (decode steps / verify blocks; the host
// knows it), so the sequence of t needs no offset loads at all.
template <int MAXN>
__device__ __forceinline__ bool load_window(const Shape& s, const uint32_t* __restrict__ tokens,
                                            const int64_t* __restrict__ seq_off, int64_t nseq,
                                            const uint32_t* __restrict__ prior, int64_t t, uint32_t (&w)[MAXN],
                                            int64_t uniform_len = 0) {
    const int N = s.N;
    const int64_t sq = uniform_len > 0 ? t / uniform_len : find_seq(seq_off, nseq, t);
    const int64_t base = uniform_len > 0 ? sq * uniform_len : __ldg(seq_off + sq);
    const int64_t p = t - base;
    if (p < 0) return false;  // malformed device offsets (off[0] > t): never read out of bounds
    bool bad = false;
#pragma unroll
    for (int j = 0; j < MAXN; ++j) {
        if (j < N) {
            const int64_t idx = p - (N - 1) + j;
            const uint32_t v = idx >= 0 ? __ldg(tokens + base + idx)
                                        : (prior ? __ldg(prior + sq * (N - 1) + (N - 1) + idx) : 0u);
            w[j] = v;
            bad |= (v >= s.V0);
        }
    }
    return !bad;
}

// One warp: hash the B branches of position t (lane = branch) and copy the B d-wide rows
// into xrow = X + t*D with 16-byte vectors, U independent loads in flight per lane.
template <int MAXN, int U>
__device__ __forceinline__ void gather_position(const Shape& s, const HashTables* __restrict__ ht,
                                                const uint32_t (&w)[MAXN], const __nv_bfloat16* __restrict__ sub,
                                                __nv_bfloat16* __restrict__ xrow_base, int32_t* grow, int64_t Tpad,
                                                int64_t t, int lane) {
    const int B = s.B, d = s.d;
    for (int b0 = 0; b0 < B; b0 += 32) {
        const int b = b0 + lane;
        int32_t row = 0;
        if (b < B) {
            row = storage_row(ht, b, branch_hash<MAXN>(s, ht, w, b), nullptr);
            if (grow) grow[(int64_t)b * Tpad + t] = row;
        }
        const int vpr = d / 8;
        const int nv = min(32, B - b0) * vpr;
        uint4* xrow = reinterpret_cast<uint4*>(xrow_base + (int64_t)b0 * d);
        for (int v0 = lane; v0 - lane < nv; v0 += 32 * U) {  // warp-uniform trip count (shfl inside)
            uint4 val[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + u * 32;
                const int bb = v / vpr;
                const int32_t r = __shfl_sync(0xffffffffu, row, bb & 31);
                if (v < nv) val[u] = __ldg(reinterpret_cast<const uint4*>(sub + (int64_t)r * d) + (v - bb * vpr));
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (v0 + u * 32 < nv) xrow[v0 + u * 32] = val[u];
        }
    }
}

}  // namespace ngk
