// hash.cu -- K1, the n-gram hash-index kernel (bit-exact restatement of the reference's
// polynomial rolling hash, hashing.cpp:33-81, over the windows of embed_sequence,
// embedding.hpp:391-405).
//
// One thread per position.  For branch b=(n-2)K+(k-1) the bucket is
//     h_b = ( sum_{j<n} (w[N-1-j] mod V_b) * (V0^j mod V_b) ) mod V_b
// -- the same residue the reference accumulates step by step (exact integer arithmetic,
// so the result is identical).  Fast path (every V_b <= 2^32): all products fit in
// 64 bits and every reduction is a Barrett step with mu = floor(2^64 / V_b) (quotient
// estimate low by at most 2, so two conditional subtractions are exact).  General path
// (any V_b < 2^64): 128-bit products, as the reference's mulmod (hashing.cpp:11-15).
//
// HBM: reads N tokens (L1/L2 hits, 4 B/token from DRAM), writes B ids (u32) and B
// storage rows (i32): 4 + 8B bytes/token -- purely bandwidth/latency bound.
//
// Kernels: hash_ids_kernel (K1 alone: ids / storage rows), rolling_hash_kernel (the
// reference's single-window API), hash_gather_block_kernel (K1+K2 fused, the prefill
// default: 16 positions per block hashed in parallel, then their X rows streamed as one
// flat array), hash_gather_kernel (warp-per-position fallback), hash_gather_rows_kernel
// (warp per (position, branch): small T), validate_tokens_kernel.
#include <cstdint>
#include <cstdlib>

#include "hashdev.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace ngk {

namespace {

template <int MAXN>
__global__ void __launch_bounds__(256) hash_ids_kernel(Shape s, const HashTables* __restrict__ ht,
                                                        const uint32_t* __restrict__ tokens,
                                                        const int64_t* __restrict__ seq_off, int64_t nseq, int64_t T,
                                                        const uint32_t* __restrict__ prior, void* __restrict__ ids_tok,
                                                        int ids_u64, int32_t* __restrict__ grow, int64_t Tpad,
                                                        unsigned long long* err) {
    const int N = s.N, K = s.K, B = s.B;
    __shared__ HashSmem<MAXN> hs;  // the block's hash constants (hashdev.cuh)
    hs.load(ht, B);
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= Tpad) return;
    if (t >= T) {  // padding rows of the GEMM's last m-tile: a valid (row 0) address, never stored
        if (grow)
            for (int b = 0; b < B; ++b) grow[(int64_t)b * Tpad + t] = 0;
        return;
    }
    const int64_t sq = find_seq(seq_off, nseq, t);
    const int64_t p = t - __ldg(seq_off + sq);
    const int64_t base = __ldg(seq_off + sq);

    uint32_t w[MAXN];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < MAXN; ++j) {
        if (j < N) {
            const int64_t idx = p - (N - 1) + j;
            uint32_t v;
            if (idx >= 0) v = __ldg(tokens + base + idx);
            else v = prior ? __ldg(prior + sq * (N - 1) + (N - 1) + idx) : 0u;
            w[j] = v;
            bad |= (v >= s.V0);
        }
    }
    if (bad) {  // the reference throws out_of_range at the first window holding the token
        atomicMin(err, (unsigned long long)t);
        return;
    }
    for (int b = 0; b < B; ++b) {
        const uint64_t h = hs.hash(s, w, b);  // hashing.cpp:33-59 (branch_hash, hashdev.cuh)
        if (ids_tok) {
            if (ids_u64) static_cast<uint64_t*>(ids_tok)[t * B + b] = h;
            else static_cast<uint32_t*>(ids_tok)[t * B + b] = (uint32_t)h;
        }
        if (grow) grow[(int64_t)b * Tpad + t] = hs.row(b, h);
    }
}

// Reference rolling_hash, one window per thread, with its validation order
// (hash_spec::validate, then length check, then per-token range check while hashing).
__global__ void rolling_hash_kernel(const uint32_t* __restrict__ windows, int64_t stride,
                                    const int32_t* __restrict__ lengths, const int32_t* __restrict__ orders,
                                    const uint64_t* __restrict__ bases, const uint64_t* __restrict__ moduli,
                                    int64_t count, uint64_t* __restrict__ out, int32_t* __restrict__ status) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int order = orders[i];
    const uint64_t base = bases[i], m = moduli[i];
    const int len = lengths ? lengths[i] : order;
    if (order < 2 || base < 2 || m < 1 || len != order) {
        status[i] = 1;  // NGRAM_EINVAL
        out[i] = 0;
        return;
    }
    const uint32_t* w = windows + i * stride;
    const uint64_t base_mod = base % m;
    uint64_t acc = 0, power = 1 % m;
    for (int j = 0; j < order; ++j) {
        const uint32_t t = w[len - 1 - j];
        if ((uint64_t)t >= base) {
            status[i] = 2;  // NGRAM_ERANGE
            out[i] = 0;
            return;
        }
        acc = (acc + mulmod128((uint64_t)t % m, power, m)) % m;
        power = mulmod128(power, base_mod, m);
    }
    out[i] = acc;
    status[i] = 0;
}

// User-supplied global bucket ids -> storage rows, with embedding_bank_t::sub_row /
// base_row range checks (embedding.hpp:41-44, 58-62).
__global__ void ids_to_rows_kernel(Shape s, const HashTables* __restrict__ ht, const uint64_t* __restrict__ ids,
                                   const uint32_t* __restrict__ tokens, int64_t T, int32_t* __restrict__ grow,
                                   int64_t Tpad, unsigned long long* err) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= Tpad) return;
    const int B = s.B;
    if (t >= T) {
        for (int b = 0; b < B; ++b) grow[(int64_t)b * Tpad + t] = 0;
        return;
    }
    bool bad = tokens[t] >= s.V0;
    for (int b = 0; b < B; ++b) {
        const uint64_t h = ids[t * B + b];
        bad |= h >= __ldg(&ht->modulus[b]);
        const int64_t lo = __ldg(&ht->row_lo[b]), hi = __ldg(&ht->row_hi[b]);
        const int64_t hh = (int64_t)h;
        grow[(int64_t)b * Tpad + t] = (hh >= lo && hh < hi) ? (int32_t)(__ldg(&ht->row_base[b]) + (hh - lo)) : -1;
    }
    if (bad) atomicMin(err, (unsigned long long)t);
}

// K1+K2 fused (X path): one warp per position (hashdev.cuh gather_position).  Lane b < B hashes branch b (the B
// hashes of a position run in parallel instead of serially), then the warp copies the
// position's B sub-table rows into X[t, b*d:(b+1)*d] with 16-byte vectors, several
// independent loads in flight per lane.  Also writes the storage rows (for callers that
// need them) when grow != null.
template <int MAXN>
__global__ void __launch_bounds__(256) hash_gather_kernel(Shape s, const HashTables* __restrict__ ht,
                                                          const uint32_t* __restrict__ tokens,
                                                          const int64_t* __restrict__ seq_off, int64_t nseq,
                                                          int64_t T, const uint32_t* __restrict__ prior,
                                                          const __nv_bfloat16* __restrict__ sub,
                                                          __nv_bfloat16* __restrict__ X, int32_t* __restrict__ grow,
                                                          int64_t Tpad, unsigned long long* err, int64_t t_begin,
                                                          int64_t t_end, int64_t x_row0) {
    const int lane = threadIdx.x & 31;
    const int64_t t = t_begin + (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (t >= t_end) return;
    uint32_t w[MAXN];
    if (!load_window<MAXN>(s, tokens, seq_off, nseq, prior, t, w)) {
        if (lane == 0) atomicMin(err, (unsigned long long)t);
        return;
    }
    gather_position<MAXN, 4>(s, ht, w, sub, X + (t - x_row0) * (int64_t)s.D, grow, Tpad, t, lane);
}

// K1+K2, block-decoupled form (default when D == B*d, B <= 32 and d/8 is a power of two):
// a block takes P positions at a time; phase A hashes all P*B (position, branch) pairs in
// parallel, one thread each, into shared memory; phase B streams the P*D*2 bytes of X as
// one flat array of 16-byte vectors (X rows of consecutive positions are contiguous), U
// independent loads in flight per thread -- the access pattern of a plain row gather.
template <int MAXN, int LOG_VPR, int U, int kGatherP>
__global__ void __launch_bounds__(256) hash_gather_block_kernel(Shape s, const HashTables* __restrict__ ht,
                                                                const uint32_t* __restrict__ tokens,
                                                                const int64_t* __restrict__ seq_off, int64_t nseq,
                                                                int64_t T, const uint32_t* __restrict__ prior,
                                                                const __nv_bfloat16* __restrict__ sub,
                                                                __nv_bfloat16* __restrict__ X,
                                                                int32_t* __restrict__ grow, int64_t Tpad,
                                                                unsigned long long* err, int64_t t_begin,
                                                                int64_t t_end, int64_t x_row0) {
    __shared__ int32_t srow[kGatherP * 32];
    __shared__ HashSmem<MAXN> hs;  // the block's hash constants (hashdev.cuh)
    const int B = s.B;
    hs.load(ht, B);
    constexpr int VPR = 1 << LOG_VPR;  // 16-byte vectors per sub-table row
    const uint4* sub4 = reinterpret_cast<const uint4*>(sub);
    uint4* X4 = reinterpret_cast<uint4*>(X);
    const int64_t vpos = (int64_t)B * VPR;  // vectors per X row
    for (int64_t t0 = t_begin + (int64_t)blockIdx.x * kGatherP; t0 < t_end; t0 += (int64_t)gridDim.x * kGatherP) {
        const int np = (int)(t_end - t0 < kGatherP ? t_end - t0 : kGatherP);
        for (int i = threadIdx.x; i < np * B; i += blockDim.x) {
            const int p = i / B, b = i - p * B;
            const int64_t t = t0 + p;
            uint32_t w[MAXN];
            int32_t row = -1;
            if (load_window<MAXN>(s, tokens, seq_off, nseq, prior, t, w)) {
                row = hs.row(b, hs.hash(s, w, b));
                if (row < 0) row = 0;  // not on this shard: storage_row's fallback row
                if (grow) grow[(int64_t)b * Tpad + t] = row;
            } else if (b == 0) {
                atomicMin(err, (unsigned long long)t);
            }
            srow[i] = row;
        }
        __syncthreads();
        const int n = np * B * VPR;
        uint4* dst = X4 + (t0 - x_row0) * vpos;  // X row 0 holds position x_row0
        for (int v0 = threadIdx.x; v0 < n; v0 += blockDim.x * U) {
            uint4 val[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + u * (int)blockDim.x;
                if (v < n) {
                    const int32_t row = srow[v >> LOG_VPR];
                    if (row >= 0) val[u] = __ldg(sub4 + (int64_t)row * VPR + (v & (VPR - 1)));
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + u * (int)blockDim.x;
                if (v < n && srow[v >> LOG_VPR] >= 0) dst[v] = val[u];
            }
        }
        __syncthreads();
    }
}

// Small-T variant (decode / verify): one warp per (position, branch), so a position's B
// rows are fetched by B warps in a single round of loads instead of serially by one warp.
template <int MAXN>
__global__ void __launch_bounds__(256) hash_gather_rows_kernel(Shape s, const HashTables* __restrict__ ht,
                                                               const uint32_t* __restrict__ tokens,
                                                               const int64_t* __restrict__ seq_off, int64_t nseq,
                                                               int64_t T, const uint32_t* __restrict__ prior,
                                                               const __nv_bfloat16* __restrict__ sub,
                                                               __nv_bfloat16* __restrict__ X,
                                                               unsigned long long* err, int64_t uniform_len) {
    griddep_launch_dependents();  // the decode GEMM may start its set-up (it waits for us)
    __shared__ HashSmem<MAXN> hs;  // the block's hash constants (hashdev.cuh)
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const bool active = w < T * s.B;
    const int64_t t = active ? w / s.B : 0;
    const int b = active ? (int)(w - t * s.B) : 0;
    uint32_t win[MAXN];
    // the window loads are issued before the constants' cooperative load, so the two global
    // round trips overlap instead of running back to back
    const bool ok = active && load_window<MAXN>(s, tokens, seq_off, nseq, prior, t, win, uniform_len);
    hs.load(ht, s.B);
    if (!active) return;
    if (!ok) {
        if (lane == 0 && b == 0) atomicMin(err, (unsigned long long)t);
        return;
    }
    int32_t row = hs.row(b, hs.hash(s, win, b));
    if (row < 0) row = 0;  // not on this shard: storage_row's fallback row
    const uint4* src = reinterpret_cast<const uint4*>(sub + (int64_t)row * s.d);
    uint4* dst = reinterpret_cast<uint4*>(X + t * (int64_t)s.D + (int64_t)b * s.d);
    for (int c = lane; c < s.d / 8; c += 32) dst[c] = __ldg(src + c);
}

__global__ void validate_tokens_kernel(uint32_t V0, const uint32_t* __restrict__ tokens, int64_t T,
                                       const int64_t* __restrict__ seq_off, int64_t nseq, const uint32_t* prior,
                                       int R, unsigned long long* err) {
    griddep_launch_dependents();  // the fused prefill kernel may start (it waits before any output)
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < T) {
        if (__ldg(tokens + i) >= V0) atomicMin(err, (unsigned long long)i);
    } else if (prior && i < T + nseq * R) {  // prior tokens are in the window of the sequence's position 0
        const int64_t k = i - T, sq = k / R;
        const int64_t a = __ldg(seq_off + sq), b = __ldg(seq_off + sq + 1);
        if (b > a && __ldg(prior + k) >= V0) atomicMin(err, (unsigned long long)a);
    }
}

}  // namespace

void launch_validate_tokens(const Shape& s, const uint32_t* tokens, int64_t T, const int64_t* seq_off, int64_t nseq,
                            const uint32_t* prior, unsigned long long* err, cudaStream_t st) {
    const int R = s.N > 1 ? s.N - 1 : 0;
    const int64_t n = T + (prior ? nseq * R : 0);
    if (n <= 0) return;
    validate_tokens_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s.V0, tokens, T, seq_off, nseq, prior, R, err);
    count_launch();
}

void launch_hash_gather(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* seq_off,
                        int64_t nseq, int64_t T, const uint32_t* prior, const __nv_bfloat16* sub, __nv_bfloat16* X,
                        int32_t* grow, int64_t Tpad, unsigned long long* err, cudaStream_t st, int64_t t_begin,
                        int64_t t_end, int64_t x_row0) {
    if (t_end < 0) t_end = T;
    if (t_end <= t_begin) return;
    static const bool warp_form = getenv("NGRAM_GATHER_WARP") != nullptr;  // A/B switch
    const int vpr = s.d / 8;
    const bool block_form = !warp_form && s.variant == 1 && s.B >= 1 && s.B <= 32 && s.d % 8 == 0 &&
                            (vpr & (vpr - 1)) == 0 && vpr <= 64 && s.N <= 8 && (int64_t)s.B * s.d == s.D;
    if (block_form) {
        // one P-position tile per block, not persistent: block turnover overlaps one block's
        // hashing phase with its neighbours' copy phases (measured: 0.145 vs 0.153 ms persistent)
        constexpr int P = 16;
        const int64_t blocks = (t_end - t_begin + P - 1) / P;
        auto go = [&](auto kern) {
            kern<<<(unsigned)blocks, 256, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, sub, X, grow, Tpad, err,
                                                    t_begin, t_end, x_row0);
        };
        const int lv = __builtin_ctz((unsigned)vpr);
        if (s.N <= 4) {
            switch (lv) {
                case 0: go(hash_gather_block_kernel<4, 0, 8, P>); break;
                case 1: go(hash_gather_block_kernel<4, 1, 8, P>); break;
                case 2: go(hash_gather_block_kernel<4, 2, 8, P>); break;
                case 3: go(hash_gather_block_kernel<4, 3, 8, P>); break;
                case 4: go(hash_gather_block_kernel<4, 4, 8, P>); break;
                case 5: go(hash_gather_block_kernel<4, 5, 8, P>); break;
                default: go(hash_gather_block_kernel<4, 6, 8, P>); break;
            }
        } else {
            switch (lv) {
                case 0: go(hash_gather_block_kernel<8, 0, 8, P>); break;
                case 1: go(hash_gather_block_kernel<8, 1, 8, P>); break;
                case 2: go(hash_gather_block_kernel<8, 2, 8, P>); break;
                case 3: go(hash_gather_block_kernel<8, 3, 8, P>); break;
                case 4: go(hash_gather_block_kernel<8, 4, 8, P>); break;
                case 5: go(hash_gather_block_kernel<8, 5, 8, P>); break;
                default: go(hash_gather_block_kernel<8, 6, 8, P>); break;
            }
        }
        count_launch();
        return;
    }
    const unsigned blocks = (unsigned)((t_end - t_begin + 7) / 8);  // 8 warps (positions) per block
    if (s.N <= 4)
        hash_gather_kernel<4><<<blocks, 256, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, sub, X, grow, Tpad, err,
                                                      t_begin, t_end, x_row0);
    else if (s.N <= 8)
        hash_gather_kernel<8><<<blocks, 256, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, sub, X, grow, Tpad, err,
                                                      t_begin, t_end, x_row0);
    else
        hash_gather_kernel<16><<<blocks, 256, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, sub, X, grow, Tpad,
                                                       err, t_begin, t_end, x_row0);
    count_launch();
}

void launch_hash_gather_rows(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* seq_off,
                             int64_t nseq, int64_t T, const uint32_t* prior, const __nv_bfloat16* sub,
                             __nv_bfloat16* X, unsigned long long* err, cudaStream_t st, int64_t uniform_len) {
    const int64_t warps = T * s.B;
    if (warps <= 0) return;
    const unsigned blocks = (unsigned)((warps + 7) / 8);
    if (s.N <= 4)
        hash_gather_rows_kernel<4><<<blocks, 256, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, sub, X, err, uniform_len);
    else if (s.N <= 8)
        hash_gather_rows_kernel<8><<<blocks, 256, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, sub, X, err, uniform_len);
    else
        hash_gather_rows_kernel<16><<<blocks, 256, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, sub, X, err, uniform_len);
    count_launch();
}

void launch_hash_ids(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* seq_off,
                     int64_t nseq, int64_t T, const uint32_t* prior, void* ids_tok, int ids_u64, int32_t* grow,
                     int64_t Tpad, unsigned long long* err, cudaStream_t st) {
    const int64_t n = grow ? Tpad : T;
    if (n <= 0) return;
    const int threads = 256;
    const unsigned blocks = (unsigned)((n + threads - 1) / threads);
    if (s.N <= 4)
        hash_ids_kernel<4><<<blocks, threads, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, ids_tok, ids_u64, grow,
                                                       grow ? Tpad : T, err);
    else if (s.N <= 8)
        hash_ids_kernel<8><<<blocks, threads, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, ids_tok, ids_u64, grow,
                                                       grow ? Tpad : T, err);
    else
        hash_ids_kernel<16><<<blocks, threads, 0, st>>>(s, ht, tokens, seq_off, nseq, T, prior, ids_tok, ids_u64,
                                                        grow, grow ? Tpad : T, err);
    count_launch();
}

void launch_rolling_hash_batch(const uint32_t* windows, int64_t stride, const int32_t* lengths, const int32_t* orders,
                               const uint64_t* bases, const uint64_t* moduli, int64_t count, uint64_t* out,
                               int32_t* status, cudaStream_t st) {
    if (count <= 0) return;
    const int threads = 256;
    rolling_hash_kernel<<<(unsigned)((count + threads - 1) / threads), threads, 0, st>>>(
        windows, stride, lengths, orders, bases, moduli, count, out, status);
    count_launch();
}

void launch_ids_to_rows(const Shape& s, const HashTables* ht, const uint64_t* ids, const uint32_t* tokens, int64_t T,
                        int32_t* grow, int64_t Tpad, unsigned long long* err, cudaStream_t st) {
    if (Tpad <= 0) return;
    const int threads = 256;
    ids_to_rows_kernel<<<(unsigned)((Tpad + threads - 1) / threads), threads, 0, st>>>(s, ht, ids, tokens, T, grow,
                                                                                        Tpad, err);
    count_launch();
}

}  // namespace ngk
