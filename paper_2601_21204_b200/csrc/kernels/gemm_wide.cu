// gemm_wide.cu -- fused prefill for narrow models (D <= 768): K1 (hash) + K2 (row gather) +
// K3 (projection + base add + scale + amplify) in ONE persistent tcgen05 kernel, no X.
//
//   Y[t, :] = amplify( (E0[tok_t, :] + X[t, :] . W_cat^T) * fp32(1/denom) ),
//   X[t, b*d:(b+1)*d] = E_b[id_b(t)]            (embedding.hpp:163-201, 239-287)
//
// Why a separate kernel: at D = 768 (SURVEY config B) the layer is HBM-bound (403 MB of
// algorithmic bytes vs 47 us of tensor work), and the X path moves 605 MB (X written by
// K1+K2 and read back by K3).  The pair kernel with gathering producers re-gathers an
// m-block's rows once per 256-column N-tile (3x at D = 768) as 128-byte requests.  Here a CTA
// pair owns a whole 256-row m-block: its producers hash the rows' windows and tile::gather4
// the D/64 K-blocks of A ONCE into shared memory, where they stay resident while the MMA warp
// sweeps all D/256 N-tiles over them (the W_cat tiles stream from L2 through a small ring).
// The accumulators (2 x 256 TMEM columns) alternate between N-tiles so the epilogue of one
// overlaps the MMAs of the next; each A slot is refilled for the next m-block as soon as the
// last N-tile's MMA of that K-block has retired (its commit frees the slot).
//
// Shared memory per CTA: A = D/64 slots x 16 KB (128 rows x 64 bf16, SWIZZLE_128B K-major),
// B ring = 16 KB stages (this CTA's 128 W_cat rows x 64): D = 768 -> 192 + 2 x 16 KB.
// The epilogue has no staging buffer left, so it goes straight from registers: TMEM is read
// with tcgen05.ld.16x256b (4 lanes share a row, 8-byte column pairs), which makes every fp32
// output store a full 32-byte sector per row; E0 pairs are read the same way (L2-prefetched
// a tile ahead).  Warp roles: 0-3 A producers (thread = tile row), 4 W producer, 5-12
// epilogue (two per TMEM lane quadrant, one column half each), 13 MMA issuer (highest id:
// the warp arbiter serves it first).
//
// Arithmetic is identical to the X path (same A rows, same MMA shape and K order, same
// epilogue roundings), so outputs are bit-identical to it (tested).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "hashdev.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace ngk {

namespace {

constexpr int kWSlot = 128 * 64 * 2;  // one A K-block slot of this CTA: 128 rows x 64 bf16 = 16 KB
constexpr int kWBN = 256;             // N-tile width (pair MMA 256 x 256; 256 x 128 measured 1.8x slower)
// W stage depth: 64 (128 rows x 64 bf16, SWIZZLE_128B, 16 KB: two stages at D = 768) or 32
// (SWIZZLE_64B, 8 KB: four stages).  Measured at config B: 64 -> 141 us, 32 -> 146 us (the
// extra commit + barrier round per K-block costs more than the finer ring gains).
constexpr int kWBK = 64;
constexpr int kWStage = (kWBN / 2) * kWBK * 2;
constexpr int kWAcc = 512 / kWBN;     // TMEM accumulators (512 columns)
constexpr int kWSteps = kWBN / 32;    // epilogue steps per tile and warp (2 row halves x 32-column chunks)
constexpr int kWMaxB = 12;            // branches (N-1)K: B * d = D <= 768 with d >= 64
constexpr int kWMaxN = 8;             // max order (window length)
constexpr int kWProd = 4;             // A producer warps
constexpr int kWWWarp = 4;            // W producer warp
constexpr int kWEpi0 = 5;             // epilogue warps 5..12
constexpr int kWEpiWarps = 8;
constexpr int kWMmaWarp = 13;
constexpr int kWThreads = 14 * 32;
constexpr int kWSmemMax = 232448;     // sm_100 dynamic shared memory per block
// the kernel's hash constants (B <= 12 branches, windows <= 8): moduli, Barrett factors, V0^j,
// shard row ranges, copied to shared memory once (the K1 kernels gained 10-40 % from it)
struct WideHash {
    uint64_t m[kWMaxB], mu[kWMaxB], pw[kWMaxB][kWMaxN];
    int64_t lo[kWMaxB], hi[kWMaxB], base[kWMaxB];
};
constexpr int kWSmemExtra = 1024 /*align*/ + 512 /*barriers*/ + (int)sizeof(WideHash);

__host__ __device__ constexpr int wide_stages(int KB) {
    return (kWSmemMax - kWSmemExtra - KB * kWSlot) / kWStage > 8 ? 8
                                                                : (kWSmemMax - kWSmemExtra - KB * kWSlot) / kWStage;
}
__host__ __device__ constexpr int wide_smem(int KB) { return kWSmemExtra + KB * kWSlot + wide_stages(KB) * kWStage; }

struct WideParams {
    Shape s;
    const HashTables* ht;
    const uint32_t* tokens;
    const int64_t* seq_off;
    int64_t nseq;
    const uint32_t* prior;
    const __nv_bfloat16* sub;
    const __nv_bfloat16* e0;
    void* rows_out;
    void* merged_out;
    int out_bf16;
    int write_rows;
    int64_t T;
    float scale, amp;
    const unsigned long long* err;
    int dbg;    // diagnostics only (NGRAM_DEBUG_WIDE bits): 1 no hashing (synthetic rows), 2 no epilogue memory
                // traffic, 4 no A copies (cp.async mode), 8 no W loads
    int a_tma;  // A producer: 0 = cp.async (default), 1 = TMA tile::gather4 (NGRAM_WIDE_GATHER4=1)
    int pdl;    // launched as a programmatic dependent of the token check: only the epilogue waits
};

// 16 TMEM lanes x 32 columns: thread i gets lane (base + i/4) in r[4j], r[4j+1] and lane
// (base + 8 + i/4) in r[4j+2], r[4j+3], columns 8j + 2(i%4) + {0, 1}, j = 0..3 (layout
// measured on the B200: scratch probe recorded in profiles/README.md).
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}

// fp32 output pairs: no L1 allocation (measured at config B: 123.7-123.9 us vs 124.6-125.0 with
// the streaming .cs operator, 125.8-127.1 with the default write-back; profiles/README.md)
__device__ __forceinline__ void st_na_f2(float* p, float a, float b) {
    asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void st_cs_u32(void* p, uint32_t v) {
    asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Window of position t NEWEST first (wr[j] = token at t - j; the sequence's prior context,
// then zeros, before its start -- embedding.hpp:391-405): load_window's w[N-1-j] with static
// register indices (load_window + branch_hash index w by the runtime N, which puts the window
// in local memory).
__device__ __forceinline__ bool window_rev(const Shape& s, const uint32_t* __restrict__ tokens,
                                           const int64_t* __restrict__ seq_off, int64_t nseq,
                                           const uint32_t* __restrict__ prior, int64_t t, uint32_t (&wr)[kWMaxN]) {
    const int N = s.N;
    const int64_t sq = find_seq(seq_off, nseq, t);
    const int64_t base = __ldg(seq_off + sq);
    const int64_t pos = t - base;
    if (pos < 0) return false;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < kWMaxN; ++j) {
        uint32_t v = 0;
        if (j < N) {
            const int64_t idx = pos - j;
            v = idx >= 0 ? __ldg(tokens + base + idx) : (prior ? __ldg(prior + sq * (N - 1) + (N - 1) + idx) : 0u);
            bad |= v >= s.V0;
        }
        wr[j] = v;
    }
    return !bad;
}

// The general forms, out of line (rare: a token may exceed the modulus, or the modulus is
// above 2^30; the unrolled __int128 / double-Barrett code would bloat the producer loop):
// hashdev.cuh branch_hash term for term.
struct Win8 {
    uint32_t v[kWMaxN];
};
__device__ __noinline__ uint64_t hash_rev_general(const Shape s, const HashTables* __restrict__ ht, Win8 wr, int n,
                                                  int b, uint64_t m) {
    uint64_t acc = 0;
    if (s.fast_hash) {
        const uint64_t mu = __ldg(&ht->barrett[b]);
#pragma unroll
        for (int j = 0; j < kWMaxN; ++j)
            if (j < n) acc += barrett_mod(barrett_mod((uint64_t)wr.v[j], m, mu) * __ldg(&ht->pow[b][j]), m, mu);
        return barrett_mod(acc, m, mu);  // acc < n * 2^32
    }
#pragma unroll
    for (int j = 0; j < kWMaxN; ++j)
        if (j < n) acc = (acc + mulmod128((uint64_t)wr.v[j] % m, __ldg(&ht->pow[b][j]), m)) % m;
    return acc;
}

// branch_hash (hashdev.cuh; hashing.cpp:33-81) over a newest-first window: the same residue
// sum_j (w_{t-j} mod V_b) * (V0^j mod V_b) mod V_b.  Common case inline: every token < V0 <=
// V_b <= 2^30, so w mod V_b = w, each term < 2^62 / 8 and the n <= 8 terms sum below 2^64:
// ONE Barrett reduction of the plain sum (the same residue as reducing every term).
__device__ __forceinline__ uint64_t hash_rev(const Shape& s, const HashTables* __restrict__ ht,
                                             const uint32_t (&wr)[kWMaxN], int b) {
    const int n = 2 + b / s.K;
    const uint64_t m = __ldg(&ht->modulus[b]);
    if (m <= 1) return 0;
    if (s.fast_hash && m <= (1ull << 30) && (uint64_t)s.V0 <= m) {
        uint64_t acc = 0;
#pragma unroll
        for (int j = 0; j < kWMaxN; ++j)
            if (j < n) acc += (uint64_t)wr[j] * (uint32_t)__ldg(&ht->pow[b][j]);
        return barrett_mod(acc, m, __ldg(&ht->barrett[b]));
    }
    Win8 w8;
#pragma unroll
    for (int j = 0; j < kWMaxN; ++j) w8.v[j] = wr[j];
    return hash_rev_general(s, ht, w8, n, b, m);
}

// OUT: 1 = amplified rows in fp32 only (the prefill call), 0 = any combination (runtime)
// hash_rev from the shared constants (the general forms fall back to the global tables)
__device__ __forceinline__ uint64_t hash_rev_s(const Shape& s, const HashTables* __restrict__ ht, const WideHash& h,
                                               const uint32_t (&wr)[kWMaxN], int b) {
    const int n = 2 + b / s.K;
    const uint64_t m = h.m[b];
    if (m <= 1) return 0;
    if (s.fast_hash && m <= (1ull << 30) && (uint64_t)s.V0 <= m) {
        uint64_t acc = 0;
#pragma unroll
        for (int j = 0; j < kWMaxN; ++j)
            if (j < n) acc += (uint64_t)wr[j] * (uint32_t)h.pw[b][j];
        return barrett_mod(acc, m, h.mu[b]);
    }
    return hash_rev(s, ht, wr, b);
}
__device__ __forceinline__ int32_t wide_row(const WideHash& h, int b, uint64_t v) {
    const int64_t hh = (int64_t)v;
    return (hh >= h.lo[b] && hh < h.hi[b]) ? (int32_t)(h.base[b] + (hh - h.lo[b])) : 0;
}

template <int KB, int OUT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kWThreads, 1)
    forward_wide_kernel(const __grid_constant__ CUtensorMap tmap_sub, const __grid_constant__ CUtensorMap tmap_w,
                        WideParams p) {
    constexpr int SB = wide_stages(KB);
    constexpr int nN = KB * 64 / kWBN;  // N-tiles
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* aslot = smem;
    uint8_t* bstage = smem + KB * kWSlot;
    uint64_t* afull = reinterpret_cast<uint64_t*>(bstage + SB * kWStage);
    uint64_t* aempty = afull + KB;
    uint64_t* bfull = aempty + KB;
    uint64_t* bempty = bfull + SB;
    uint64_t* tfull = bempty + SB;
    uint64_t* tempty = tfull + kWAcc;
    uint64_t* lfull = tempty + kWAcc;  // cp.async producers of the peer CTA: its own slot arrivals (relayed)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lfull + KB);
    WideHash* wh = reinterpret_cast<WideHash*>(smem + KB * kWSlot + SB * kWStage + 512);

    // a token was out of range (the validation kernel before this one): no output.  Launched as
    // its programmatic dependent, the kernel starts while the check still runs -- hashing,
    // gathers and MMAs only read -- and the epilogue waits for the verdict before any store.
    if (!p.pdl && *p.err != ~0ull) return;

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int64_t pair = cluster_id_x();
    const int64_t npairs = nclusters_x();
    const int64_t nM = (p.T + 255) / 256;
    const int KPB = p.s.d / 64;  // K-blocks per branch

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < KB; ++i) {
            // gather4: the leader's producer warps (each expects both CTAs' rows); cp.async: every
            // leader producer thread's copy-completion arrive + the peer's relay
            mbar_init(&afull[i], p.a_tma ? kWProd : kWProd * 32 + 1);
            mbar_init(&lfull[i], kWProd * 32);
            mbar_init(&aempty[i], 1);  // the leader's multicast commit after the last N-tile
        }
        for (int i = 0; i < SB; ++i) {
            mbar_init(&bfull[i], 1);
            mbar_init(&bempty[i], 1);
        }
        for (int i = 0; i < kWAcc; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 2 * kWEpiWarps);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmap_sub);
        tma_prefetch_desc(&tmap_w);
    }
    if (warp < kWProd)  // the producers' hash constants (read only by this CTA's producer warps)
        for (int i = threadIdx.x; i < p.s.B * kWMaxN; i += kWProd * 32) {
            const int b = i / kWMaxN, j = i % kWMaxN;
            wh->pw[b][j] = __ldg(&p.ht->pow[b][j]);
            if (j == 0) {
                wh->m[b] = __ldg(&p.ht->modulus[b]);
                wh->mu[b] = __ldg(&p.ht->barrett[b]);
                wh->lo[b] = __ldg(&p.ht->row_lo[b]);
                wh->hi[b] = __ldg(&p.ht->row_hi[b]);
                wh->base[b] = __ldg(&p.ht->row_base[b]);
            }
        }
    if (warp == kWMmaWarp) tmem_alloc_2cta<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < kWProd) {
        // ------------------------------------------------ A producers: hash + gather4 (both CTAs)
        const int r = warp * 32 + lane;  // this thread's tile row
        // storage rows of the thread's row for every branch of m-block m, computed one m-block
        // ahead: the hashing runs while the MMA sweeps the current block, so each slot is
        // refilled the moment its last N-tile's MMA frees it (rows past T / bad windows: any
        // valid row, never stored)
        int32_t rr[kWMaxB];
        // rr[b] with a runtime b, kept in registers: a select chain (a runtime loop over the
        // branches keeps the producer's code small -- unrolled per-branch code overflowed the
        // instruction cache, measured)
        auto row_of = [&](int b) {
            int32_t v = rr[0];
#pragma unroll
            for (int k = 1; k < kWMaxB; ++k) v = b == k ? rr[k] : v;
            return v;
        };
        auto rows_for = [&](int64_t m) {
            const int64_t t = m * 256 + (int64_t)rank * 128 + r;
            uint32_t w[kWMaxN];
            const bool ok = !(p.dbg & 1) && t < p.T && window_rev(p.s, p.tokens, p.seq_off, p.nseq, p.prior, t, w);
#pragma unroll 1
            for (int b = 0; b < p.s.B; ++b) {  // (four chains per trip measured no faster)
                const int32_t v = ok ? wide_row(*wh, b, hash_rev_s(p.s, p.ht, *wh, w, b))
                                     : (p.dbg & 1) ? (int32_t)((t * 7919 + b * 104729) % 1000000) : 0;
#pragma unroll
                for (int k = 0; k < kWMaxB; ++k) rr[k] = b == k ? v : rr[k];
            }
        };
        // one call site each (code size): hash block mh, then issue it on the next trip while
        // hashing the block after
        const int q8 = lane & 7;
        const int l4 = 4 * q8;
        uint64_t* arrive_bar = leader ? afull : lfull;
        int64_t mh = pair;
        int it = -1;
        while (true) {
            if (it >= 0) {
                const uint32_t par = (uint32_t)(it & 1) ^ 1u;
                int kb = 0;
#pragma unroll 1
                for (int b = 0; b < p.s.B; ++b) {
                    const int32_t rb = row_of(b);
                    if (p.a_tma) {
                        const int32_t r0 = __shfl_sync(0xffffffffu, rb, l4), r1 = __shfl_sync(0xffffffffu, rb, l4 + 1);
                        const int32_t r2 = __shfl_sync(0xffffffffu, rb, l4 + 2), r3 = __shfl_sync(0xffffffffu, rb, l4 + 3);
                        for (int c = 0; c < KPB; ++c, ++kb) {
                            mbar_wait(&aempty[kb], par);
                            if (leader && lane == 0) mbar_arrive_expect_tx(&afull[kb], 2 * 32 * 128);
                            __syncwarp();
                            if (lane < 8)
                                tma_gather4_2cta(aslot + kb * kWSlot + (warp * 32 + l4) * 128, &tmap_sub,
                                                 leader_bar(&afull[kb]), c * 64, r0, r1, r2, r3);
                        }
                    } else {
                        // cp.async: 8 lanes per 128-byte row segment (coalesced), 4 rows per
                        // instruction, written in the SWIZZLE_128B K-major layout.  Completion is
                        // signalled by the copies themselves (arrive.noinc): the leader's threads
                        // on afull, the peer's on lfull, which its idle MMA warp relays to the leader.
                        int32_t src[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) src[j] = __shfl_sync(0xffffffffu, rb, 4 * j + (lane >> 3));
                        for (int c = 0; c < KPB; ++c, ++kb) {
                            mbar_wait(&aempty[kb], par);
                            const uint32_t a_base = smem_u32(aslot + kb * kWSlot);
                            const __nv_bfloat16* col = p.sub + c * 64 + q8 * 8;
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const int rs = warp * 32 + 4 * j + (lane >> 3);
                                if (!(p.dbg & 4))
                                    cp_async_16(a_base + rs * 128 + ((q8 ^ (rs & 7)) << 4), col + (int64_t)src[j] * p.s.d);
                            }
                            cp_async_mbar_arrive_noinc(&arrive_bar[kb]);
                        }
                    }
                }
            }
            if (mh >= nM) break;
            rows_for(mh);
            mh += npairs;
            ++it;
        }
        if (!p.a_tma) cp_async_wait<0>();
    } else if (warp == kWWWarp) {
        // ------------------------------------------------ W_cat producer (both CTAs)
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();  // W_cat stays L2-resident
            int s = 0;
            uint32_t ph = 0;
            for (int64_t m = pair; m < nM; m += npairs)
                for (int n = 0; n < nN; ++n)
                    for (int kh = 0; kh < KB * (64 / kWBK); ++kh) {  // W stages of kWBK columns
                        mbar_wait(&bempty[s], ph ^ 1);
                        if (p.dbg & 8) {  // diagnostics: no W loads
                            if (leader) mbar_arrive(&bfull[s]);
                            if (++s == SB) {
                                s = 0;
                                ph ^= 1;
                            }
                            continue;
                        }
                        if (leader) mbar_arrive_expect_tx(&bfull[s], 2 * kWStage);
                        tma_load_2d_2cta(bstage + s * kWStage, &tmap_w, leader_bar(&bfull[s]), kh * kWBK,
                                         n * kWBN + (int)rank * (kWBN / 2), pol);
                        if (++s == SB) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
        }
        __syncwarp();
    } else if (warp == kWMmaWarp) {
        // ------------------------------------------------ MMA issuer (leader only)
        if (!leader && !p.a_tma) {
            // relay: this CTA's rows of slot kb landed (its producers' cp.async arrivals) ->
            // ordered for the async proxy -> one relaxed arrive on the leader's afull
            if (lane == 0) {
                int it = 0;
                for (int64_t m = pair; m < nM; m += npairs, ++it)
                    for (int kb = 0; kb < KB; ++kb) {
                        mbar_wait(&lfull[kb], (uint32_t)(it & 1));
                        fence_proxy_async_smem();
                        mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&afull[kb]), 0));
                    }
            }
            __syncwarp();
        }
        if (leader) {
            constexpr uint32_t idesc = idesc_bf16_f32(256, kWBN);
            int s = 0, acc = 0, it = 0;
            uint32_t ph = 0, acc_ph = 0;
            for (int64_t m = pair; m < nM; m += npairs, ++it) {
                const uint32_t par = (uint32_t)(it & 1);
                for (int n = 0; n < nN; ++n) {
                    mbar_wait(&tempty[acc], acc_ph ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + (uint32_t)(acc * kWBN);
#pragma unroll 1
                    for (int kb = 0; kb < KB; ++kb) {
                        mbar_wait(&afull[kb], par);  // completes once per m-block; later N-tiles pass through
                        if (!p.a_tma && n == 0) fence_proxy_async_smem();  // the producers' cp.async rows
                        const uint64_t adesc = smem_desc_sw128(smem_u32(aslot + kb * kWSlot));
#pragma unroll
                        for (int hf = 0; hf < 64 / kWBK; ++hf) {  // the K-block's W stages
                            mbar_wait(&bfull[s], ph);
                            tc_fence_after();
                            if (lane == 0) {
                                const uint32_t baddr = smem_u32(bstage + s * kWStage);
                                const uint64_t bdesc = kWBK == 64 ? smem_desc_sw128(baddr) : smem_desc_sw64(baddr);
#pragma unroll
                                for (int k = 0; k < kWBK / 16; ++k)
                                    tc_mma_bf16_2cta(d_tmem, adesc + (uint64_t)(hf * (kWBK / 8) + k * 2),
                                                     bdesc + (uint64_t)(k * 2), idesc, (kb | hf | k) != 0);
                                tc_commit_2cta_mc(&bempty[s], 0x3);
                                if (hf == 64 / kWBK - 1 && n == nN - 1)
                                    tc_commit_2cta_mc(&aempty[kb], 0x3);  // slot free for the next m-block
                            }
                            __syncwarp();
                            if (++s == SB) {
                                s = 0;
                                ph ^= 1;
                            }
                        }
                    }
                    if (lane == 0) tc_commit_2cta_mc(&tfull[acc], 0x3);
                    __syncwarp();
                    if (++acc == kWAcc) {
                        acc = 0;
                        acc_ph ^= 1;
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (both CTAs)
        bool no_out = false;
        if (p.pdl) {
            griddep_wait();  // the token check has completed
            no_out = *p.err != ~0ull;
        }
        // Warp (quadrant q, half h) drains rows 32 q .. 32 q + 31 x columns h kWBN/2 .. + kWBN/2
        // of each tile in kWSteps steps: row half hh (16 TMEM lanes) x 32-column chunk ch.  E0
        // words come through a 4-slot register ring loaded 4 steps ahead (across tiles); the
        // next tile's E0 segments are L2-prefetched a tile ahead of that.
        const int ew = warp - kWEpi0;  // 0..7
        const int q = warp & 3;        // TMEM lane quadrant this warp may access
        const int h = ew >> 2;         // column half of the tile
        const int g = lane >> 2, c2 = 2 * (lane & 3);
        const int D = p.s.D;
        const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
        int acc = 0;
        uint32_t acc_ph = 0;
        // the thread's four rows of an m-block: g, g + 8, g + 16, g + 24 of its quadrant
        auto row0_of = [&](int64_t m) { return m * 256 + (int64_t)rank * 128 + q * 32 + g; };
        auto toks_of = [&](int64_t r0, uint32_t (&tok)[4]) {
#pragma unroll
            for (int i = 0; i < 4; ++i)  // rows past T: row 0 (never stored)
                tok[i] = r0 + 8 * i < p.T ? __ldg(p.tokens + r0 + 8 * i) : 0u;
        };
        auto prefetch_e0 = [&](const uint32_t (&tok)[4], int col0) {  // kWBN/2 bf16 per row (128-byte lines)
            if ((lane & 3) == 0) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int c = 0; c < kWBN / 2; c += 64) prefetch_l2(p.e0 + (int64_t)tok[i] * D + col0 + c);
            }
        };
        // E0 words of step s of a tile whose warp columns start at col0: rows g + 16 hh + 8 i2
        auto load_step = [&](const uint32_t (&tk)[4], int col0, int s, uint32_t (&e)[8]) {
            if (p.dbg & 2) return;
            const int hh = s / (kWSteps / 2), ch = s % (kWSteps / 2);
#pragma unroll
            for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    e[4 * i2 + j] = __ldg(reinterpret_cast<const uint32_t*>(p.e0 + (int64_t)tk[2 * hh + i2] * D + col0 +
                                                                            ch * 32 + 8 * j + c2));
        };
        int64_t r0 = row0_of(pair);
        uint32_t tok[4], ntok[4];
        uint32_t E[4][8];  // E0 ring: step s's words in slot s
        const int hcol = h * (kWBN / 2);
        if (pair < nM) {
            toks_of(r0, tok);
            prefetch_e0(tok, hcol);
#pragma unroll
            for (int s = 0; s < 4; ++s) load_step(tok, hcol, s, E[s]);
        }
        int64_t m = pair;
        int n = 0;
        while (m < nM) {
            const int col0 = n * kWBN + hcol;
            int64_t m2 = m;
            int n2 = n + 1;
            if (n2 == nN) {
                n2 = 0;
                m2 += npairs;
            }
            const bool has_next = m2 < nM, same_m = m2 == m;
            // tokens of the next m-block; L2 prefetch of the next tile's E0 segments
            if (has_next && !same_m) toks_of(row0_of(m2), ntok);
            if (has_next) {
                if (same_m) prefetch_e0(tok, n2 * kWBN + hcol);
                else prefetch_e0(ntok, hcol);
            }
            mbar_wait(&tfull[acc], acc_ph);
            tc_fence_after();
#pragma unroll
            for (int s = 0; s < kWSteps; ++s) {
                const int hh = s / (kWSteps / 2), ch = s % (kWSteps / 2);
                uint32_t v[16];
                tmem_ld_16x256b_x4(tmem_base + ((uint32_t)(q * 32 + 16 * hh) << 16) +
                                       (uint32_t)(acc * kWBN + hcol + ch * 32), v);
                tmem_ld_wait();
                if (s == kWSteps - 1) {  // accumulator fully read (the loads have completed): release it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader + 8u * (uint32_t)acc);
                }
#pragma unroll
                for (int i2 = 0; i2 < 2; ++i2) {
                    const int64_t tr = r0 + 16 * hh + 8 * i2;
                    if (tr >= p.T || no_out || (p.dbg & 2)) continue;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t ew2 = E[s & 3][4 * i2 + j];
                        const float m0 = __fmul_rn(__fadd_rn(bf16_bits_to_f32(ew2 & 0xffffu),
                                                             __uint_as_float(v[4 * j + 2 * i2])), p.scale);
                        const float m1 = __fmul_rn(__fadd_rn(bf16_bits_to_f32(ew2 >> 16),
                                                             __uint_as_float(v[4 * j + 2 * i2 + 1])), p.scale);
                        const int64_t o = tr * D + col0 + ch * 32 + 8 * j + c2;
                        if (OUT == 1) {
                            st_na_f2(static_cast<float*>(p.rows_out) + o, __fmul_rn(m0, p.amp), __fmul_rn(m1, p.amp));
                            continue;
                        }
                        if (p.merged_out) {
                            if (p.out_bf16) st_cs_u32(static_cast<__nv_bfloat16*>(p.merged_out) + o, pack_bf16x2(m0, m1));
                            else st_na_f2(static_cast<float*>(p.merged_out) + o, m0, m1);
                        }
                        if (p.write_rows) {
                            const float a0 = __fmul_rn(m0, p.amp), a1 = __fmul_rn(m1, p.amp);
                            if (p.out_bf16) st_cs_u32(static_cast<__nv_bfloat16*>(p.rows_out) + o, pack_bf16x2(a0, a1));
                            else st_na_f2(static_cast<float*>(p.rows_out) + o, a0, a1);
                        }
                    }
                }
                // refill the slot with the step four ahead (this tile's, or the next tile's first)
                if (s + 4 < kWSteps) {
                    load_step(tok, col0, s + 4, E[s & 3]);
                } else if (has_next) {
                    if (same_m) load_step(tok, n2 * kWBN + hcol, s + 4 - kWSteps, E[s & 3]);
                    else load_step(ntok, hcol, s + 4 - kWSteps, E[s & 3]);
                }
            }
            if (++acc == kWAcc) {
                acc = 0;
                acc_ph ^= 1;
            }
            if (has_next && !same_m) {
                r0 = row0_of(m2);
#pragma unroll
                for (int i = 0; i < 4; ++i) tok[i] = ntok[i];
            }
            m = m2;
            n = n2;
        }
    }

    tc_fence_before();
    cluster_sync();  // every MMA retired and every remote arrive delivered before TMEM is freed
    if (warp == kWMmaWarp) {
        tc_fence_after();
        tmem_dealloc_2cta<512>(tmem_base);
    }
}

template <int KB, int OUT>
void launch_wide_out(const FwdArgs& a, const WideParams& p, int num_sms, cudaStream_t st) {
    const int64_t nM = (a.T + 255) / 256;
    int64_t pairs = std::min<int64_t>(num_sms / 2, nM);
    if (pairs < 1) pairs = 1;
    cudaFuncSetAttribute(forward_wide_kernel<KB, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, wide_smem(KB));
    const CUtensorMap& mw = kWBK == 64 ? *a.tmap_w2 : *a.tmap_w32;
    if (!p.pdl) {
        forward_wide_kernel<KB, OUT><<<(unsigned)(2 * pairs), kWThreads, wide_smem(KB), st>>>(*a.tmap_sub, mw, p);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * pairs));
    cfg.blockDim = dim3(kWThreads);
    cfg.dynamicSmemBytes = wide_smem(KB);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, forward_wide_kernel<KB, OUT>, *a.tmap_sub, mw, p);
}
template <int KB>
void launch_wide(const FwdArgs& a, const WideParams& p, int num_sms, cudaStream_t st) {
    if (p.write_rows && !p.merged_out && !p.out_bf16) launch_wide_out<KB, 1>(a, p, num_sms, st);
    else launch_wide_out<KB, 0>(a, p, num_sms, st);
}

}  // namespace

static_assert(wide_smem(12) <= kWSmemMax && wide_stages(12) >= 2, "D = 768 needs two W stages");

bool wide_prefill_shape(const Shape& s) {
    return s.variant == 1 && s.D % 256 == 0 && s.D <= 768 && s.d % 64 == 0 && s.B >= 1 && s.B <= kWMaxB &&
           s.N >= 2 && s.N <= kWMaxN && (int64_t)s.B * s.d == s.D;
}

void launch_forward_wide(const FwdArgs& a, int num_sms, cudaStream_t st) {
    if (a.T <= 0) return;
    WideParams p{};
    p.s = a.s;
    p.ht = a.ht;
    p.tokens = a.tokens;
    p.seq_off = a.seq_off;
    p.nseq = a.nseq;
    p.prior = a.prior;
    p.sub = a.sub;
    p.e0 = a.e0;
    p.rows_out = a.rows_out;
    p.merged_out = a.merged_out;
    p.out_bf16 = a.out_bf16;
    p.write_rows = (a.rows_out != nullptr && a.s.amp != kAmpLN) ? 1 : 0;
    p.T = a.T;
    p.scale = 1.0f / (float)a.s.denom;
    p.amp = a.s.amp == kAmpSqrt ? (float)__builtin_sqrt((double)a.s.D) : 1.0f;
    p.err = a.err;
    static const int a_tma = getenv("NGRAM_WIDE_GATHER4") ? atoi(getenv("NGRAM_WIDE_GATHER4")) : 0;
    p.a_tma = a_tma;
    static const int dbg = getenv("NGRAM_DEBUG_WIDE") ? atoi(getenv("NGRAM_DEBUG_WIDE")) : 0;
    p.dbg = dbg;
    static const bool pdl = !(getenv("NGRAM_PDL") && atoi(getenv("NGRAM_PDL")) == 0);
    p.pdl = pdl ? 1 : 0;  // the caller launched the token check right before (forward.cpp)
    switch (a.s.D / 64) {
        case 4: launch_wide<4>(a, p, num_sms, st); break;
        case 8: launch_wide<8>(a, p, num_sms, st); break;
        default: launch_wide<12>(a, p, num_sms, st); break;
    }
    count_launch();
}

}  // namespace ngk
