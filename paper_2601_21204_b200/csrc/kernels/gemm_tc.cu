// gemm_tc.cu -- K3: the projection GEMM on the 5th-gen tensor cores, with the base-row
// add, 1/denom scale and amplification in the epilogue.
//
//   Y[t, :] = amplify( (E0[tok_t, :] + X[t, :] . W_cat^T) * fp32(1/denom) )
//   X[t, b*d:(b+1)*d] = E_b[id_b(t)]
//
// This is embed_from_ids (embedding.hpp:163-201) + amplify (:239-287): the reference's
// per-token D x d matvec per branch (its >99% hot loop, embedding.hpp:189-195) becomes ONE
// bf16 GEMM with K = (N-1)K*d = D (branch-concatenated), fp32 accumulation in TMEM.  The A
// operand is either X materialised by the fused K1+K2 kernel (hash.cu; TMA 2D tiles) or the
// sub-table rows gathered straight into shared memory (tile::gather4 / cp.async).
//
// Kernels (persistent, warp-specialised; the MMA issuer is always the highest warp id
// because the warp arbiter serves the highest eligible id first):
//   forward_tc2_kernel   2-CTA pairs (cta_group::2), 256 x 256 tiles, 8 epilogue warps,
//                        TMEM double-buffered; the production path for D % 256 == 0 and
//                        T > 256.  EPI 4 (default) / 1: all epilogue traffic by TMA (E0
//                        rows gathered 64 / 32 columns at a time into a smem ring, outputs
//                        staged and bulk-stored); EPI 0: direct.
//   forward_tc_kernel    1 CTA, 128 x BN tiles: shapes the pair kernel does not take, and
//                        the small-T split-K GEMM (raw fp32 partials, BN = 128; MODE 2
//                        hashes in its producers, opt-in).
//   splitk_reduce_kernel S partials + E0 + scales (+ the decode-state commit), PDL-launched.
// Tiles are ordered n-fastest so the CTAs running concurrently share an m-block's A rows
// through L2; W_cat (2*D^2 bytes) stays L2-resident (evict_last).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "decodedev.cuh"
#include "hashdev.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace ngk {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one SWIZZLE_128B atom of bf16
constexpr int kStages = 4;
constexpr int kLag = 2;  // cp.async mode: K-blocks in flight per producer warp before retiring
constexpr int kMaxDecodeN = 8;  // MODE 2 (hash in the producer): max_order <= 8

template <int BN, int NP>
struct Cfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int kEpiWarp0 = NP;     // epilogue warps NP..NP+3
    static constexpr int kMmaWarp = NP + 4;  // MMA issuer last: highest arbiter priority
    static constexpr int kThreads = (NP + 5) * 32;
    static constexpr int kRowsPerWarp = BM / NP;
};

struct TcParams {
    Shape s;
    const uint32_t* tokens;
    const int32_t* grow;
    const __nv_bfloat16* sub;
    const __nv_bfloat16* e0;
    void* rows_out;
    void* merged_out;
    int out_bf16;
    int write_rows;  // amp != LN
    int64_t T, Tpad;  // rows of this call, grow row stride
    float scale, amp;
    const unsigned long long* err;
    int use_x;  // A operand from materialised X (tmap_a is X) instead of gathered sub-table rows
    int hash_lsu;  // pair kernel: producers hash the windows and cp.async the rows (K1+K2+K3 in one)
    int epi_skip;  // diagnostics only (NGRAM_DEBUG_EPI_SKIP): 1 drain TMEM without loads/stores,
                   // 2 (pair kernel) skip the E0 loads, 3 (pair kernel) skip the output stores
    int diag_skip_a;  // diagnostics only (NGRAM_DEBUG_SKIP_A): X-path pair kernel loads W tiles only
    int pdl;          // launched with programmatic stream serialization (decode chain)
    int tempty_relaxed;  // pair kernel TMA epilogue: relaxed accumulator release (NGRAM_TEMPTY_RELAXED, default 1)
    int ksplit;      // split-K factor (small-T path); >1 => raw fp32 partials to `partial`
    float* partial;  // [ksplit][T][D] fp32
    // MODE 2 (small-T GEMM hashing in its producers): the windows of `tokens`
    const HashTables* ht;
    const int64_t* seq_off;
    int64_t nseq;
    const uint32_t* prior;
};

__device__ __forceinline__ void store_chunk(void* out, int out_bf16, int64_t o, const float (&mv)[32]) {
    if (out_bf16) {
        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + o);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16x2(mv[8 * i], mv[8 * i + 1]), pack_bf16x2(mv[8 * i + 2], mv[8 * i + 3]),
                                pack_bf16x2(mv[8 * i + 4], mv[8 * i + 5]), pack_bf16x2(mv[8 * i + 6], mv[8 * i + 7]));
    } else {
        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(out) + o);
#pragma unroll
        for (int i = 0; i < 8; ++i) dst[i] = make_float4(mv[4 * i], mv[4 * i + 1], mv[4 * i + 2], mv[4 * i + 3]);
    }
}

template <int BN, int NP, int MODE>
__global__ void __launch_bounds__(Cfg<BN, NP>::kThreads, 1)
    forward_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_w,
                      TcParams p) {
    using C = Cfg<BN, NP>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    // PDL launch (decode chain): the set-up below overlaps the previous kernel's tail; the
    // error word and X are read only after griddep_wait.
    if (!p.pdl && *p.err != ~0ull) return;  // a token was out of range: produce no output (uniform)

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int D = p.s.D;
    const int nN = D / BN;
    const int64_t nM = (p.T + BM - 1) / BM;
    const int S = p.ksplit;
    const int64_t tiles = nM * nN * S;  // split-K: tile = (s * nM + m) * nN + n
    const int KB = D / BK / S;   // K-blocks per tile
    const int KPB = p.s.d / BK;  // K-blocks per branch (gather mode)

    if (warp == 0 && lane == 0) {
        // full: one arrive per producer warp (+1 for the W TMA in cp.async mode), or one in X mode
        const uint32_t full_count = p.use_x ? 1u : (MODE != 1 ? (uint32_t)NP : (uint32_t)NP + 1);
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], full_count);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_w);
    }
    if (warp == C::kMmaWarp) tmem_alloc<C::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (p.pdl) {
        griddep_launch_dependents();  // the reduce kernel may launch and park in its own wait
        griddep_wait();               // gather kernel done: X and the error word are final
        if (*p.err != ~0ull) {        // uniform: release TMEM, produce nothing
            if (warp == C::kMmaWarp) tmem_dealloc<C::kTmemCols>(tmem_base);
            return;
        }
    }

    if (warp < NP) {
        // ------------------------------------------------------------ producers
        int stage = 0;
        uint32_t phase = 0;
        const uint64_t pol_w = policy_evict_last();
        if (p.use_x) {
            for (int64_t tile = blockIdx.x; warp == 0 && tile < tiles; tile += gridDim.x) {
                const int64_t mn = tile % (nM * nN);
                const int ks = (int)(tile / (nM * nN));
                const int64_t m = mn / nN;
                const int n = (int)(mn - m * nN);
                for (int kb = ks * KB; kb < (ks + 1) * KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (lane == 0) {
                        uint8_t* a_dst = smem + stage * C::kStageBytes;
                        mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                        tma_load_2d(a_dst, &tmap_a, &full[stage], kb * BK, (int32_t)(m * BM));
                        tma_load_2d_hint(a_dst + C::kABytes, &tmap_w, &full[stage], kb * BK, n * BN, pol_w);
                    }
                    __syncwarp();
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        } else if (MODE == 2) {
            // Small-T split-K with K1 fused into the producer: each lane of a producer warp
            // hashes 4 of the warp's 32 tile rows for the branch its K-blocks belong to and
            // gathers them with tile::gather4 straight from the sub-tables (no X round trip,
            // no separate gather launch).  Rows past T gather row 0 (never stored); a bad
            // window sets the error word, which the reduce kernel checks before any output.
            const int r0 = warp * C::kRowsPerWarp;
            for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
                const int64_t mn = tile % (nM * nN);
                const int ks = (int)(tile / (nM * nN));
                const int64_t m = mn / nN;
                const int n = (int)(mn - m * nN);
                uint32_t win[4][kMaxDecodeN];
                bool ok[4];
                if (lane < C::kRowsPerWarp / 4) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int64_t t = m * BM + r0 + 4 * lane + i;
                        ok[i] = t < p.T && load_window<kMaxDecodeN>(p.s, p.tokens, p.seq_off, p.nseq, p.prior, t,
                                                                     win[i]);
                        if (t < p.T && !ok[i]) atomicMin(const_cast<unsigned long long*>(p.err),
                                                         (unsigned long long)t);
                    }
                }
                int cur_b = -1;
                int4 rows4 = make_int4(0, 0, 0, 0);
                for (int kb = ks * KB; kb < (ks + 1) * KB; ++kb) {
                    const int b = kb / KPB, c = kb - b * KPB;
                    if (b != cur_b && lane < C::kRowsPerWarp / 4) {
                        int r[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            r[i] = ok[i] ? storage_row(p.ht, b, branch_hash<kMaxDecodeN>(p.s, p.ht, win[i], b), nullptr)
                                         : 0;
                        rows4 = make_int4(r[0], r[1], r[2], r[3]);
                    }
                    cur_b = b;
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a_dst = smem + stage * C::kStageBytes;
                    if (lane == 0)
                        mbar_arrive_expect_tx(&full[stage], (warp == 0 ? C::kBBytes : 0) + C::kRowsPerWarp * BK * 2);
                    __syncwarp();
                    if (lane < C::kRowsPerWarp / 4)
                        tma_gather4(a_dst + (r0 + 4 * lane) * (BK * 2), &tmap_a, &full[stage], c * BK, rows4.x,
                                    rows4.y, rows4.z, rows4.w);
                    if (warp == 0 && lane == 0)
                        tma_load_2d_hint(a_dst + C::kABytes, &tmap_w, &full[stage], kb * BK, n * BN, pol_w);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        } else {
        const int r0 = warp * C::kRowsPerWarp;  // first tile row of this warp
        int retired_stage = 0, pending = 0;     // cp.async mode bookkeeping
        for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const int64_t m = tile / nN;
            const int n = (int)(tile - m * nN);
            const int64_t t0 = m * BM;
            for (int b = 0; b < p.s.B; ++b) {
                const int32_t* gb = p.grow + (int64_t)b * p.Tpad + t0 + r0;
                int4 rows4 = make_int4(0, 0, 0, 0);
                int32_t row1 = 0;
                if (MODE == 0) {
                    if (lane < C::kRowsPerWarp / 4) rows4 = *reinterpret_cast<const int4*>(gb + 4 * lane);
                } else {
                    row1 = gb[lane];  // lane l holds the storage row of tile row r0 + l
                }
                for (int c = 0; c < KPB; ++c) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a_dst = smem + stage * C::kStageBytes;
                    const int kcol = c * BK;
                    if (MODE == 0) {
                        if (lane == 0)
                            mbar_arrive_expect_tx(&full[stage],
                                                  (warp == 0 ? C::kBBytes : 0) + C::kRowsPerWarp * BK * 2);
                        __syncwarp();
                        if (lane < C::kRowsPerWarp / 4)
                            tma_gather4(a_dst + (r0 + 4 * lane) * (BK * 2), &tmap_a, &full[stage], kcol, rows4.x,
                                        rows4.y, rows4.z, rows4.w);
                        if (warp == 0 && lane == 0)
                            tma_load_2d_hint(a_dst + C::kABytes, &tmap_w, &full[stage], (b * KPB + c) * BK, n * BN,
                                             pol_w);
                    } else {
                        if (warp == 0 && lane == 0) {
                            mbar_arrive_expect_tx(&full[stage], C::kBBytes);
                            tma_load_2d_hint(a_dst + C::kABytes, &tmap_w, &full[stage], (b * KPB + c) * BK, n * BN,
                                             pol_w);
                        }
                        const uint32_t a_base = smem_u32(a_dst);
                        const int q = lane & 7;  // 16-B chunk of the 128-B row segment
#pragma unroll
                        for (int j = 0; j < C::kRowsPerWarp / 4; ++j) {
                            const int rl = 4 * j + (lane >> 3);  // row within this warp's slab
                            const int r = r0 + rl;               // row within the tile
                            const int32_t src_row = __shfl_sync(0xffffffffu, row1, rl);
                            const __nv_bfloat16* src = p.sub + (int64_t)src_row * p.s.d + kcol + q * 8;
                            cp_async_16(a_base + r * 128 + ((q ^ (r & 7)) << 4), src);
                        }
                        cp_async_commit();
                        if (++pending > kLag) {  // retire the K-block issued kLag steps ago
                            cp_async_wait<kLag>();
                            fence_proxy_async_smem();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&full[retired_stage]);
                            if (++retired_stage == kStages) retired_stage = 0;
                            --pending;
                        }
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        if (MODE == 1) {
            cp_async_wait<0>();
            fence_proxy_async_smem();
            __syncwarp();
            for (; pending > 0; --pending) {
                if (lane == 0) mbar_arrive(&full[retired_stage]);
                if (++retired_stage == kStages) retired_stage = 0;
            }
        }
        }  // gather mode
    } else if (warp == C::kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
            for (int kb = 0; kb < KB; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a_addr = smem_u32(smem + stage * C::kStageBytes);
                    const uint64_t adesc = smem_desc_sw128(a_addr);
                    const uint64_t bdesc = smem_desc_sw128(a_addr + C::kABytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        // advance the start address by k * 16 bf16 = 32 B inside the swizzle atom
                        tc_mma_bf16(d_tmem, adesc + (uint64_t)(k * 2), bdesc + (uint64_t)(k * 2), idesc,
                                    (kb | k) != 0);
                    }
                    tc_commit(&empty[stage]);  // smem slot free once these MMAs retire
                }
                __syncwarp();
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (lane == 0) tc_commit(&tfull[acc]);  // accumulator ready for the epilogue
            __syncwarp();
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        const int r = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const int64_t mn = tile % (nM * nN);
            const int ks = (int)(tile / (nM * nN));
            const int64_t m = mn / nN;
            const int n = (int)(mn - m * nN);
            const int64_t t = m * BM + r;
            const bool valid = t < p.T && !p.epi_skip;
            const uint32_t tok = valid ? __ldg(p.tokens + t) : 0u;
            const __nv_bfloat16* e0row = p.e0 + (int64_t)tok * D + n * BN;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
                if (S > 1) {  // split-K: raw fp32 partial sums, reduced + epilogued by splitk_reduce_kernel
                    tmem_ld_wait();
                    if (valid) {
                        float4* dst = reinterpret_cast<float4*>(p.partial + ((int64_t)ks * p.T + t) * D +
                                                                (int64_t)n * BN + c * 32);
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                                 __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                    }
                    continue;
                }
                uint4 e[4];
                if (valid) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) e[i] = __ldg(reinterpret_cast<const uint4*>(e0row + c * 32) + i);
                }
                tmem_ld_wait();
                if (valid) {
                    float mv[32];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t w[4] = {e[i].x, e[i].y, e[i].z, e[i].w};
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const int j = i * 8 + h * 2;
                            mv[j] = __fmul_rn(__fadd_rn(bf16_bits_to_f32(w[h] & 0xffffu), __uint_as_float(v[j])),
                                              p.scale);
                            mv[j + 1] = __fmul_rn(
                                __fadd_rn(bf16_bits_to_f32(w[h] >> 16), __uint_as_float(v[j + 1])), p.scale);
                        }
                    }
                    const int64_t o = t * D + (int64_t)n * BN + c * 32;
                    if (p.merged_out) store_chunk(p.merged_out, p.out_bf16, o, mv);
                    if (p.write_rows) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) mv[j] = __fmul_rn(mv[j], p.amp);
                        store_chunk(p.rows_out, p.out_bf16, o, mv);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == C::kMmaWarp) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}


// ============================================================================ 2-CTA variant
// cta_group::2: a CTA pair computes a 256 x 256 tile (M = 256 tokens, 128 per CTA; the
// W tile is split, 128 rows per CTA), so each SM streams 16 KB of W per K-block instead
// of 32 KB -- shared-memory traffic per SM drops from 96 KB to 64 KB per K-block, under
// the ~128 B/clk smem port.  The leader CTA (rank 0) owns the full barriers and the
// accumulator-empty barrier and issues every tcgen05.mma.cta_group::2; the peer's TMA
// loads (.cta_group::2) complete on the leader's barriers, the leader's commits arrive on
// both CTAs' empty / accumulator-full barriers (multicast).
constexpr int BM2 = 256;   // tokens per pair tile
constexpr int BN2 = 256;   // output columns per pair tile
constexpr int kStages2 = 6;
constexpr int NP2 = 4;     // producer warps per CTA

constexpr int kEpiWarps2 = 8;  // two per TMEM lane quadrant, each owning half the columns

// Epilogue modes.  0: E0 loaded and outputs stored by every thread straight from
// registers (one token row per lane: 32 rows per warp instruction).  1: all epilogue
// memory traffic by TMA -- each warp gathers its 32 rows x 32 columns of E0 per chunk with
// tile::gather4 into a 2-slot SWIZZLE_64B ring (issued two chunks ahead, across tile
// boundaries) and stages every output box in SWIZZLE_128B (fp32) / SWIZZLE_64B (bf16) smem
// for a bulk tensor store.  Mode 1 costs one pipeline stage of smem.
// Mode 1 = 5 stages, 2 E0 slots, 1 output buffer per warp.  Measured equal within noise and
// removed (profiles/README.md): 4 stages with 2 output buffers, or with 4 E0 slots.
// Mode 4 (production): as mode 1 with E0 gathered 64 columns (128-byte rows, SWIZZLE_128B)
// per gather4 -- half the TMA gather operations; each ring slot serves two chunks; 4 stages
// (the wider slots take the fifth stage's smem).  K3 0.853 vs 0.859 ms at config C.
constexpr int stages2(int epi) { return epi == 0 ? kStages2 : epi == 1 ? kStages2 - 1 : kStages2 - 2; }
constexpr int epi_ring(int) { return 2; }
constexpr int epi_obufs(int) { return 1; }
constexpr int kE0Box = 32 * 32 * 2;   // one E0 chunk: 32 rows x 32 bf16 columns
constexpr int e0box(int epi) { return epi == 4 ? 2 * kE0Box : kE0Box; }
constexpr int kOutBox = 32 * 32 * 4;  // one staged output box (fp32 worst case)
constexpr int epi_smem(int epi) {
    return epi ? kEpiWarps2 * (epi_ring(epi) * e0box(epi) + epi_obufs(epi) * kOutBox) : 0;
}

struct Cfg2 {
    static constexpr int kABytes = 128 * BK * 2;           // this CTA's 128 token rows
    static constexpr int kBBytes = (BN2 / 2) * BK * 2;     // this CTA's half of the W tile
    static constexpr int kStageBytes = kABytes + kBBytes;  // 32 KB
    static constexpr int kTmemCols = 2 * BN2;              // double-buffered 128 x 256 fp32
    static constexpr int smem_bytes(int epi) {
        return stages2(epi) * kStageBytes + epi_smem(epi) + 1024 + 512;
    }
    // Warp roles: producers [0, NP2), epilogue [NP2, NP2+8), and the single MMA-issuing warp
    // LAST: the warp arbiter picks the highest eligible warp id first, so the tensor-core
    // issue is never starved.
    static constexpr int kEpiWarp0 = NP2;
    static constexpr int kMmaWarp = NP2 + kEpiWarps2;
    static constexpr int kThreads = (NP2 + kEpiWarps2 + 1) * 32;
    static constexpr int kRowsPerWarp = 128 / NP2;
};

// SWIZZLE_64B / SWIZZLE_128B smem address of 16-byte chunk j of row r of a box whose rows
// are 64 / 128 bytes (buffers 512 / 1024-byte aligned): the TMA unit applies the same XOR
// of address bits [4, 6) / [4, 7) with bits [7, 9) / [7, 10), and one row per lane makes
// every warp-wide v4 access bank-conflict free.
__device__ __forceinline__ uint32_t sw64(uint32_t base, int r, int j) {
    return base + (uint32_t)r * 64u + (uint32_t)((j ^ ((r >> 1) & 3)) << 4);
}
__device__ __forceinline__ uint32_t sw128(uint32_t base, int r, int j) {
    return base + (uint32_t)r * 128u + (uint32_t)((j ^ (r & 7)) << 4);
}

// Stage one 32 x 32 output box (lane = row) and hand it to TMA.  The staging buffer is
// rewritten only after the bulk group that last read it has finished reading smem.
template <int NBUF>
__device__ __forceinline__ void epi_store_box(uint8_t* obuf, int lane, const float (&mv)[32], float mul, bool scaled,
                                              int out_bf16, const CUtensorMap* map, int32_t col, int32_t row,
                                              uint64_t pol) {
    if (lane == 0) bulk_wait_group_read<NBUF - 1>();
    __syncwarp();
    const uint32_t base = smem_u32(obuf);
    float f[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] = scaled ? __fmul_rn(mv[j], mul) : mv[j];
    if (out_bf16) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            st_shared_v4u(sw64(base, lane, j),
                          make_uint4(pack_bf16x2(f[8 * j], f[8 * j + 1]), pack_bf16x2(f[8 * j + 2], f[8 * j + 3]),
                                     pack_bf16x2(f[8 * j + 4], f[8 * j + 5]), pack_bf16x2(f[8 * j + 6], f[8 * j + 7])));
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            st_shared_v4(sw128(base, lane, j), make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]));
    }
    fence_proxy_async_smem();  // generic-proxy smem writes -> async-proxy (TMA) reads
    __syncwarp();
    if (lane == 0) {
        tma_store_2d(map, obuf, col, row, pol);
        bulk_commit_group();
    }
}

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg2::kThreads, 1)
    forward_tc2_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_w,
                       const __grid_constant__ CUtensorMap tmap_rows, const __grid_constant__ CUtensorMap tmap_merged,
                       const __grid_constant__ CUtensorMap tmap_e0, TcParams p) {
    using C = Cfg2;
    constexpr int kStages2 = stages2(EPI);  // shadows the namespace constant
    constexpr int kMmaWarp = C::kMmaWarp;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* staging = smem + kStages2 * C::kStageBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(staging + epi_smem(EPI));
    uint64_t* empty = full + kStages2;
    uint64_t* tfull = empty + kStages2;
    uint64_t* tempty = tfull + 2;
    uint64_t* e0bar = tempty + 2;  // [kEpiWarps2][ring] E0 ring slots (mode 1)
    uint64_t* lfull = e0bar + epi_ring(EPI) * kEpiWarps2;  // hash_lsu: the peer's own stage barriers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lfull + kStages2);

    if (*p.err != ~0ull) return;  // uniform across the grid

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int64_t pair = cluster_id_x();
    const int64_t npairs = nclusters_x();
    const int D = p.s.D;
    const int nN = D / BN2;
    const int64_t nM = (p.T + BM2 - 1) / BM2;
    const int64_t tiles = nM * nN;
    const int KB = D / BK;
    const int KPB = p.s.d / BK;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kStages2; ++i) {
            // leader's: X path one (expect_tx); gather4 path one per leader producer warp; hash_lsu
            // one cp.async arrival per leader producer thread + the peer's relay + the W expect_tx
            mbar_init(&full[i], p.use_x ? 1 : p.hash_lsu ? NP2 * 32 + 2 : NP2);
            mbar_init(&lfull[i], NP2 * 32);  // hash_lsu, peer CTA: its producer threads' cp.async
            mbar_init(&empty[i], 1);                 // leader's multicast commit
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 2 * kEpiWarps2);  // epilogue warps of both CTAs (leader's copy)
        }
        if (EPI)
            for (int i = 0; i < epi_ring(EPI) * kEpiWarps2; ++i) mbar_init(&e0bar[i], 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_w);
    }
    if (warp == kMmaWarp) tmem_alloc_2cta<C::kTmemCols>(tmem_slot);
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised, TMEM allocated, before any remote signal
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < NP2) {
        // ------------------------------------------------------------ producers (both CTAs)
        int stage = 0;
        uint32_t phase = 0;
        const uint64_t pol_w = policy_evict_last();
        const int r0 = warp * C::kRowsPerWarp;
        // X path: one thread issues both TMA loads per stage; producer warps 1..3 (needed by the
        // gathering modes) leave at once instead of spinning on the same barriers
        for (int64_t tile = pair; p.use_x && warp == 0 && lane == 0 && tile < tiles; tile += npairs) {
            const int64_t m = tile / nN;
            const int n = (int)(tile - m * nN);
            const int64_t t0 = m * BM2 + (int64_t)rank * 128;  // this CTA's first token row
            const int wrow = n * BN2 + (int)rank * (BN2 / 2);  // this CTA's first W row
            for (int kb = 0; kb < KB; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* a_dst = smem + stage * C::kStageBytes;
                if (leader) mbar_arrive_expect_tx(&full[stage], p.diag_skip_a ? 2 * C::kBBytes : 2 * C::kStageBytes);
                if (!p.diag_skip_a)
                    tma_load_2d_2cta(a_dst, &tmap_a, leader_bar(&full[stage]), kb * BK, (int32_t)t0, 0);
                tma_load_2d_2cta(a_dst + C::kABytes, &tmap_w, leader_bar(&full[stage]), kb * BK, wrow, pol_w);
                if (++stage == kStages2) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        if (p.hash_lsu) {
            // K1 + K2 in the producers (no X, no grow): lane l of producer warp w owns tile row
            // r = 32 w + l -- it loads its window once per tile, hashes one branch per d-wide
            // slab, and the warp copies its 32 rows of each 64-column K-block with cp.async
            // (4 rows x 8 16-byte chunks per instruction: every 128-byte row segment is one
            // coalesced request) into the SWIZZLE_128B A slab.  Completion is signalled by the
            // copies themselves (cp.async.mbarrier.arrive.noinc): the producer never waits on its
            // own loads, so as many K-blocks are in flight as there are free stages.  The leader's
            // threads arrive on its full barrier directly; the peer's arrive on a local barrier
            // that the peer's (otherwise idle) MMA warp relays to the leader -- a remote arrive
            // from a thread with cp.async in flight would fence on all of them (measured: the
            // release-cluster arrive serialised every stage).  Tokens were range-checked by the
            // validation kernel before this launch (a bad call produces no output).
            const int rw = warp * 32;
            const int q = lane & 7;
            uint64_t* arrive_bar = leader ? full : lfull;  // the peer's rows are relayed (MMA warp)
            // L2 prefetch of the rows PB branches ahead (crossing into the next tile): the
            // random-row DRAM latency is paid by the prefetch, the cp.async of a stage hits L2 --
            // four smem stages alone cover ~1 us of load latency, the random rows take longer
            const int PB = (4 + KPB - 1) / KPB;
            const int rowbytes = p.s.d * 2;
            auto window_of = [&](int64_t tile, uint32_t (&w)[kMaxDecodeN]) {
                if (tile >= tiles) return false;
                const int64_t t = (tile / nN) * BM2 + (int64_t)rank * 128 + rw + lane;
                return t < p.T && load_window<kMaxDecodeN>(p.s, p.tokens, p.seq_off, p.nseq, p.prior, t, w);
            };
            auto prefetch_row = [&](bool okw, const uint32_t (&w)[kMaxDecodeN], int b) {
                if (!okw) return;
                const int32_t r = storage_row(p.ht, b, branch_hash<kMaxDecodeN>(p.s, p.ht, w, b), nullptr);
                const char* base = reinterpret_cast<const char*>(p.sub + (int64_t)r * p.s.d);
                for (int o = 0; o < rowbytes; o += 128) prefetch_l2(base + o);
            };
            uint32_t win[kMaxDecodeN], nwin[kMaxDecodeN];
            bool ok = window_of(pair, win);
            constexpr bool kPrefetchL2 = false;  // measured slower (B 205 -> 339 us, C 1.95 -> 2.38 ms)
            for (int b = 0; kPrefetchL2 && b < PB && b < p.s.B; ++b) prefetch_row(ok, win, b);
            for (int64_t tile = pair; tile < tiles; tile += npairs) {
                const int64_t m = tile / nN;
                const int n = (int)(tile - m * nN);
                const int wrow = n * BN2 + (int)rank * (BN2 / 2);
                const bool nok = window_of(tile + npairs, nwin);
                for (int b = 0; b < p.s.B; ++b) {
                    const int32_t row1 = ok ? storage_row(p.ht, b, branch_hash<kMaxDecodeN>(p.s, p.ht, win, b), nullptr)
                                            : 0;  // rows past T: any valid row (never stored)
                    if (kPrefetchL2) {
                        if (b + PB < p.s.B) prefetch_row(ok, win, b + PB);
                        else prefetch_row(nok, nwin, b + PB - p.s.B);
                    }
                    for (int c = 0; c < KPB; ++c) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* a_dst = smem + stage * C::kStageBytes;
                        if (warp == 0 && lane == 0) {
                            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::kBBytes);
                            tma_load_2d_2cta(a_dst + C::kABytes, &tmap_w, leader_bar(&full[stage]),
                                             (b * KPB + c) * BK, wrow, pol_w);
                        }
                        const uint32_t a_base = smem_u32(a_dst);
                        const __nv_bfloat16* col = p.sub + c * BK + q * 8;
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int rl = 4 * j + (lane >> 3);
                            const int r = rw + rl;
                            const int32_t src = __shfl_sync(0xffffffffu, row1, rl);
                            cp_async_16(a_base + r * 128 + ((q ^ (r & 7)) << 4), col + (int64_t)src * p.s.d);
                        }
                        cp_async_mbar_arrive_noinc(&arrive_bar[stage]);
                        if (++stage == kStages2) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
                ok = nok;
#pragma unroll
                for (int j = 0; j < kMaxDecodeN; ++j) win[j] = nwin[j];
            }
            cp_async_wait<0>();
        } else if (!p.use_x) {
            // Gather producers: the storage rows of (tile, branch) unit u are loaded kAhead units
            // ahead (across tile boundaries), so a stage only issues gathers -- a row-index load
            // per stage put a global-memory latency (~0.7 us) on every K-block, against 0.26 us
            // of MMA per stage at D = 768 (the fused path ran at 43 % of the X path's speed).
            constexpr int kAhead = 4;
            const int B = p.s.B;
            const int64_t my_tiles = pair < tiles ? (tiles - pair + npairs - 1) / npairs : 0;
            const int64_t units = my_tiles * B;
            auto load_unit = [&](int64_t u) {
                int4 r = make_int4(0, 0, 0, 0);
                if (u < units && lane < C::kRowsPerWarp / 4) {
                    const int64_t tile = pair + (u / B) * npairs;
                    const int64_t t0 = (tile / nN) * BM2 + (int64_t)rank * 128;
                    r = *reinterpret_cast<const int4*>(p.grow + (int64_t)(u % B) * p.Tpad + t0 + r0 + 4 * lane);
                }
                return r;
            };
            int4 rq[kAhead];
#pragma unroll
            for (int j = 0; j < kAhead; ++j) rq[j] = load_unit(j);
            for (int64_t u0 = 0; u0 < units; u0 += kAhead) {
#pragma unroll
                for (int j = 0; j < kAhead; ++j) {
                    const int64_t u = u0 + j;
                    if (u >= units) break;
                    const int4 rows4 = rq[j];
                    rq[j] = load_unit(u + kAhead);
                    const int64_t tile = pair + (u / B) * npairs;
                    const int b = (int)(u % B);
                    const int n = (int)(tile % nN);
                    const int wrow = n * BN2 + (int)rank * (BN2 / 2);
                    for (int c = 0; c < KPB; ++c) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* a_dst = smem + stage * C::kStageBytes;
                        if (leader && lane == 0)  // expect this warp's rows of BOTH CTAs (+ both W halves)
                            mbar_arrive_expect_tx(&full[stage], 2 * (C::kRowsPerWarp * BK * 2) +
                                                                    (warp == 0 ? 2 * C::kBBytes : 0));
                        __syncwarp();
                        if (lane < C::kRowsPerWarp / 4)
                            tma_gather4_2cta(a_dst + (r0 + 4 * lane) * (BK * 2), &tmap_a, leader_bar(&full[stage]),
                                             c * BK, rows4.x, rows4.y, rows4.z, rows4.w);
                        if (warp == 0 && lane == 0)
                            tma_load_2d_2cta(a_dst + C::kABytes, &tmap_w, leader_bar(&full[stage]),
                                             (b * KPB + c) * BK, wrow, pol_w);
                        if (++stage == kStages2) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer (leader only)
        if (!leader && p.hash_lsu) {
            // relay: each stage's rows of this CTA landed (its producers' cp.async arrivals) ->
            // ordered for the async proxy -> one arrive on the leader's full barrier
            if (lane == 0) {
                int stage = 0;
                uint32_t phase = 0;
                const int64_t steps = (pair < tiles ? (tiles - pair + npairs - 1) / npairs : 0) * KB;
                for (int64_t i = 0; i < steps; ++i) {
                    mbar_wait(&lfull[stage], phase);
                    fence_proxy_async_smem();
                    // the rows are complete and fenced for this SM's tensor core (which reads them
                    // for the pair MMA): a relaxed arrive suffices and avoids a GPU-scope MEMBAR
                    // per stage (measured: the release arrive serialised the peer's stages)
                    mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&full[stage]), 0));
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            __syncwarp();
        }
        if (leader) {
            constexpr uint32_t idesc = idesc_bf16_f32(BM2, BN2);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t tile = pair; tile < tiles; tile += npairs) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN2);
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (p.hash_lsu) fence_proxy_async_smem();  // the producers' cp.async rows -> async proxy
                    if (lane == 0) {
                        const uint32_t a_addr = smem_u32(smem + stage * C::kStageBytes);
                        const uint64_t adesc = smem_desc_sw128(a_addr);
                        const uint64_t bdesc = smem_desc_sw128(a_addr + C::kABytes);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            tc_mma_bf16_2cta(d_tmem, adesc + (uint64_t)(k * 2), bdesc + (uint64_t)(k * 2), idesc,
                                             (kb | k) != 0);
                        tc_commit_2cta_mc(&empty[stage], 0x3);
                    }
                    __syncwarp();
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (lane == 0) tc_commit_2cta_mc(&tfull[acc], 0x3);
                __syncwarp();
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (EPI) {
        // ------------------------------------------------------------ TMA epilogue (both CTAs)
        // Chunk g of this warp = columns [col0 + 32 (g % 4), +32) of tile pair + (g / 4) npairs.
        const int ew = warp - C::kEpiWarp0;  // 0..7
        const int q = warp & 3;              // TMEM lane quadrant this warp may access
        const int half = ew >> 2;            // column half of the tile this warp owns
        const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
        const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty[1]), 0);
        constexpr int kChunks = BN2 / 2 / 32;
        constexpr int R = epi_ring(EPI);
        constexpr int OB = epi_obufs(EPI);
        constexpr bool kWide = EPI == 4;        // one E0 slot = two chunks (64 columns)
        constexpr int EB = e0box(EPI);
        constexpr int kPer = kWide ? 2 : 1;     // chunks per E0 slot
        uint8_t* e0ring = staging + ew * (R * EB);
        uint8_t* obuf0 = staging + kEpiWarps2 * R * EB + ew * OB * kOutBox;
        int ob = 0;
        uint64_t* ebar = e0bar + R * ew;
        const uint64_t pol_out = policy_evict_first();
        const int64_t nchunks = ((tiles - pair + npairs - 1) / npairs) * kChunks;
        const int64_t nslots = nchunks / kPer;
        // gather the E0 rows of slot-load g (kPer chunks) into ring slot g % R (4 rows per
        // gather4, lanes 0..7)
        auto issue_e0 = [&](int64_t g) {
            const int64_t tile = pair + (g / (kChunks / kPer)) * npairs;
            const int c = (int)(g % (kChunks / kPer));
            const int64_t m = tile / nN;
            const int n = (int)(tile - m * nN);
            const int64_t t = m * BM2 + (int64_t)rank * 128 + q * 32 + lane;
            const int tok = t < p.T ? (int)__ldg(p.tokens + t) : 0;  // rows past T: any valid row
            const int l4 = 4 * (lane & 7);
            const int r0 = __shfl_sync(0xffffffffu, tok, l4), r1 = __shfl_sync(0xffffffffu, tok, l4 + 1);
            const int r2 = __shfl_sync(0xffffffffu, tok, l4 + 2), r3 = __shfl_sync(0xffffffffu, tok, l4 + 3);
            uint64_t* bar = &ebar[g % R];
            if (lane == 0) mbar_arrive_expect_tx(bar, EB);
            __syncwarp();
            if (lane < 8)
                tma_gather4(e0ring + (g % R) * EB + lane * 4 * (64 * kPer), &tmap_e0, bar,
                            n * BN2 + half * (BN2 / 2) + c * 32 * kPer, r0, r1, r2, r3);
        };
        for (int64_t g0 = 0; g0 < R && g0 < nslots; ++g0) issue_e0(g0);
        int acc = 0;
        uint32_t acc_phase = 0;
        int64_t g = 0;
        for (int64_t tile = pair; tile < tiles; tile += npairs) {
            const int64_t m = tile / nN;
            const int n = (int)(tile - m * nN);
            const int32_t orow = (int32_t)(m * BM2 + (int64_t)rank * 128 + q * 32);
            const int col0 = n * BN2 + half * (BN2 / 2);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < kChunks; ++c, ++g) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) +
                                       (uint32_t)(acc * BN2 + half * (BN2 / 2) + c * 32),
                                   v);
                const int64_t gs = g / kPer;  // E0 slot-load holding this chunk
                mbar_wait(&ebar[gs % R], (uint32_t)((gs / R) & 1));
                const uint32_t eb = smem_u32(e0ring + (gs % R) * EB);
                uint4 e[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    e[i] = ld_shared_v4u(kWide ? sw128(eb, lane, (int)(g & 1) * 4 + i) : sw64(eb, lane, i));
                if (!kWide || (g & 1)) {
                    fence_proxy_async_smem();  // generic reads of the slot before TMA refills it
                    __syncwarp();
                    if (gs + R < nslots) issue_e0(gs + R);
                }
                tmem_ld_wait();
                float mv[32];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t w[4] = {e[i].x, e[i].y, e[i].z, e[i].w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const int j = i * 8 + h * 2;
                        mv[j] = __fmul_rn(__fadd_rn(bf16_bits_to_f32(w[h] & 0xffffu), __uint_as_float(v[j])),
                                          p.scale);
                        mv[j + 1] =
                            __fmul_rn(__fadd_rn(bf16_bits_to_f32(w[h] >> 16), __uint_as_float(v[j + 1])), p.scale);
                    }
                }
                if (c + 1 == kChunks) {  // accumulator fully read: release it to the MMA warp
                    tc_fence_before();
                    __syncwarp();
                    // relaxed: the TMEM loads have completed (tcgen05.wait::ld above) and nothing
                    // else is published -- a release arrive cost a GPU-scope MEMBAR behind the
                    // warp's outstanding stores on every tile (ncu: 11 % of the samples at config B)
                    if (lane == 0) {
                        const uint32_t bar = acc == 0 ? tempty_leader0 : tempty_leader1;
                        if (p.tempty_relaxed) mbar_arrive_cluster_relaxed(bar);
                        else mbar_arrive_cluster(bar);
                    }
                }
                // rows past T are clipped by the output tensor maps
                if (p.merged_out) {
                    epi_store_box<OB>(obuf0 + ob * kOutBox, lane, mv, 1.0f, false, p.out_bf16, &tmap_merged,
                                      col0 + c * 32, orow, pol_out);
                    ob = (ob + 1) % OB;
                }
                if (p.write_rows) {
                    epi_store_box<OB>(obuf0 + ob * kOutBox, lane, mv, p.amp, true, p.out_bf16, &tmap_rows,
                                      col0 + c * 32, orow, pol_out);
                    ob = (ob + 1) % OB;
                }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) bulk_wait_group<0>();  // output stores complete before exit
    } else {
        // ------------------------------------------------------------ epilogue (both CTAs)
        const int ew = warp - C::kEpiWarp0;  // 0..7
        const int q = warp & 3;                   // TMEM lane quadrant this warp may access
        const int half = ew >> 2;                 // column half of the tile this warp owns
        const int r = q * 32 + lane;
        const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
        const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty[1]), 0);
        constexpr int kChunks = BN2 / 2 / 32;     // 32-column chunks per warp
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t tile = pair; tile < tiles; tile += npairs) {
            const int64_t m = tile / nN;
            const int n = (int)(tile - m * nN);
            const int64_t t = m * BM2 + (int64_t)rank * 128 + r;
            const bool valid = t < p.T && p.epi_skip != 1;
            const bool load_e0 = valid && p.epi_skip != 2;
            const uint32_t tok = valid ? __ldg(p.tokens + t) : 0u;
            const int col0 = n * BN2 + half * (BN2 / 2);
            const __nv_bfloat16* e0row = p.e0 + (int64_t)tok * D + col0;
            uint4 e[4], en[4];
            if (!load_e0) {
#pragma unroll
                for (int i = 0; i < 4; ++i) e[i] = en[i] = make_uint4(0, 0, 0, 0);
            }
            if (load_e0) {  // E0 chunk 0, loaded before the accumulator is ready
#pragma unroll
                for (int i = 0; i < 4; ++i) e[i] = __ldg(reinterpret_cast<const uint4*>(e0row) + i);
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < kChunks; ++c) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) +
                                       (uint32_t)(acc * BN2 + half * (BN2 / 2) + c * 32),
                                   v);
                if (load_e0 && c + 1 < kChunks) {  // prefetch the next E0 chunk
#pragma unroll
                    for (int i = 0; i < 4; ++i) en[i] = __ldg(reinterpret_cast<const uint4*>(e0row + (c + 1) * 32) + i);
                }
                tmem_ld_wait();
                if (valid) {
                    float mv[32];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t w[4] = {e[i].x, e[i].y, e[i].z, e[i].w};
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const int j = i * 8 + h * 2;
                            mv[j] = __fmul_rn(__fadd_rn(bf16_bits_to_f32(w[h] & 0xffffu), __uint_as_float(v[j])),
                                              p.scale);
                            mv[j + 1] = __fmul_rn(
                                __fadd_rn(bf16_bits_to_f32(w[h] >> 16), __uint_as_float(v[j + 1])), p.scale);
                        }
                    }
                    const int64_t o = t * D + col0 + c * 32;
                    if (p.epi_skip == 3 && mv[0] != 1.2345e-30f) continue;  // diagnostics: no stores
                    if (p.merged_out) store_chunk(p.merged_out, p.out_bf16, o, mv);
                    if (p.write_rows) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) mv[j] = __fmul_rn(mv[j], p.amp);
                        store_chunk(p.rows_out, p.out_bf16, o, mv);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) e[i] = en[i];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc == 0 ? tempty_leader0 : tempty_leader1);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }

    tc_fence_before();
    cluster_sync();  // every MMA retired and every remote arrive delivered before TMEM is freed
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc_2cta<C::kTmemCols>(tmem_base);
    }
}

// Diagnostics switches (read once): NGRAM_DEBUG_EPI_SKIP=1/2/3, NGRAM_DEBUG_SKIP_A.
static int debug_epi_skip() {
    static const int v = getenv("NGRAM_DEBUG_EPI_SKIP") ? atoi(getenv("NGRAM_DEBUG_EPI_SKIP")) : 0;
    return v;
}
static int debug_skip_a() {
    static const int v = getenv("NGRAM_DEBUG_SKIP_A") ? 1 : 0;
    return v;
}

template <int BN, int NP, int MODE>
void launch_cfg(const FwdArgs& a, int num_sms, cudaStream_t st, int ksplit = 1, float* partial = nullptr,
                bool pdl = false) {
    using C = Cfg<BN, NP>;
    TcParams p{};
    p.ksplit = ksplit;
    p.partial = partial;
    p.s = a.s;
    p.tokens = a.tokens;
    p.grow = a.grow;
    p.sub = a.sub;
    p.e0 = a.e0;
    p.rows_out = a.rows_out;
    p.merged_out = a.merged_out;
    p.out_bf16 = a.out_bf16;
    p.write_rows = (a.rows_out != nullptr && a.s.amp != kAmpLN) ? 1 : 0;
    p.T = a.T;
    p.Tpad = a.Tpad;
    p.scale = 1.0f / (float)a.s.denom;
    p.amp = a.s.amp == kAmpSqrt ? (float)__builtin_sqrt((double)a.s.D) : 1.0f;
    p.err = a.err;
    p.use_x = a.tmap_x != nullptr;
    p.epi_skip = debug_epi_skip();
    p.diag_skip_a = debug_skip_a();
    p.ht = a.ht;
    p.seq_off = a.seq_off;
    p.nseq = a.nseq;
    p.prior = a.prior;
    const int64_t tiles = ((a.T + BM - 1) / BM) * (a.s.D / BN) * ksplit;
    int grid = (int)(tiles < num_sms ? tiles : num_sms);
    if (grid < 1) grid = 1;
    // the W box must match BN rows: tmap_w2 always has a 128-row box, tmap_w has BN(D) rows
    const CUtensorMap* wmap = (BN == 128) ? a.tmap_w2 : a.tmap_w;
    cudaFuncSetAttribute(forward_tc_kernel<BN, NP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    p.pdl = pdl ? 1 : 0;
    if (pdl) {  // programmatic stream serialization: set-up overlaps the gather kernel's tail
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(C::kThreads);
        cfg.dynamicSmemBytes = C::kSmemBytes;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, forward_tc_kernel<BN, NP, MODE>, a.tmap_x ? *a.tmap_x : *a.tmap_sub, *wmap, p);
    } else {
        forward_tc_kernel<BN, NP, MODE><<<grid, C::kThreads, C::kSmemBytes, st>>>(
            a.tmap_x ? *a.tmap_x : *a.tmap_sub, *wmap, p);
    }
    count_launch();
}

int tma_epi_mode() {
    static const int v = [] {
        const char* e = getenv("NGRAM_TMA_EPI");
        const int m = e ? atoi(e) : 4;
        return m == 4 ? 4 : std::min(1, std::max(0, m));
    }();
    return v;
}

void launch_tc2(const FwdArgs& a, int num_sms, cudaStream_t st) {
    TcParams p{};
    p.ksplit = 1;
    p.partial = nullptr;
    p.s = a.s;
    p.tokens = a.tokens;
    p.grow = a.grow;
    p.sub = a.sub;
    p.e0 = a.e0;
    p.rows_out = a.rows_out;
    p.merged_out = a.merged_out;
    p.out_bf16 = a.out_bf16;
    p.write_rows = (a.rows_out != nullptr && a.s.amp != kAmpLN) ? 1 : 0;
    p.T = a.T;
    p.Tpad = a.Tpad;
    p.scale = 1.0f / (float)a.s.denom;
    p.amp = a.s.amp == kAmpSqrt ? (float)__builtin_sqrt((double)a.s.D) : 1.0f;
    p.err = a.err;
    p.use_x = a.tmap_x != nullptr;
    p.hash_lsu = !p.use_x && a.seq_off != nullptr;
    p.ht = a.ht;
    p.seq_off = a.seq_off;
    p.nseq = a.nseq;
    p.prior = a.prior;
    p.epi_skip = debug_epi_skip();
    p.diag_skip_a = debug_skip_a();
    static const int trel = getenv("NGRAM_TEMPTY_RELAXED") ? atoi(getenv("NGRAM_TEMPTY_RELAXED")) : 1;
    p.tempty_relaxed = trel;
    const int64_t tiles = ((a.T + BM2 - 1) / BM2) * (a.s.D / BN2);
    int64_t pairs = num_sms / 2;
    if (tiles < pairs) pairs = tiles;
    if (pairs < 1) pairs = 1;
    // TMA epilogue when every written output has a map (NGRAM_TMA_EPI=0 selects mode 0)
    const bool maps_ok = a.tmap_e0 && (!p.merged_out || a.tmap_merged_out) && (!p.write_rows || a.tmap_rows_out);
    const int epi = maps_ok && !p.epi_skip ? tma_epi_mode() : 0;
    const CUtensorMap& ma = a.tmap_x ? *a.tmap_x : *a.tmap_sub;
    const CUtensorMap& mr = a.tmap_rows_out ? *a.tmap_rows_out : *a.tmap_w2;
    const CUtensorMap& mm = a.tmap_merged_out ? *a.tmap_merged_out : *a.tmap_w2;
    const unsigned grid = (unsigned)(2 * pairs);
    const CUtensorMap& me = a.tmap_e0 ? *a.tmap_e0 : *a.tmap_w2;
    if (epi == 4 && a.tmap_e0w) {
        cudaFuncSetAttribute(forward_tc2_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg2::smem_bytes(4));
        forward_tc2_kernel<4><<<grid, Cfg2::kThreads, Cfg2::smem_bytes(4), st>>>(ma, *a.tmap_w2, mr, mm, *a.tmap_e0w,
                                                                                   p);
    } else if (epi >= 1) {
        cudaFuncSetAttribute(forward_tc2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg2::smem_bytes(1));
        forward_tc2_kernel<1><<<grid, Cfg2::kThreads, Cfg2::smem_bytes(1), st>>>(ma, *a.tmap_w2, mr, mm, me, p);
    } else {
        cudaFuncSetAttribute(forward_tc2_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg2::smem_bytes(0));
        forward_tc2_kernel<0><<<grid, Cfg2::kThreads, Cfg2::smem_bytes(0), st>>>(ma, *a.tmap_w2, mr, mm, me, p);
    }
    count_launch();
}

TcParams tc2_params(const FwdArgs& a) {
    TcParams p{};
    p.ksplit = 1;
    p.s = a.s;
    p.tokens = a.tokens;
    p.grow = a.grow;
    p.sub = a.sub;
    p.e0 = a.e0;
    p.rows_out = a.rows_out;
    p.merged_out = a.merged_out;
    p.out_bf16 = a.out_bf16;
    p.write_rows = (a.rows_out != nullptr && a.s.amp != kAmpLN) ? 1 : 0;
    p.T = a.T;
    p.Tpad = a.Tpad;
    p.scale = 1.0f / (float)a.s.denom;
    p.amp = a.s.amp == kAmpSqrt ? (float)__builtin_sqrt((double)a.s.D) : 1.0f;
    p.err = a.err;
    p.use_x = 1;
    p.epi_skip = debug_epi_skip();
    p.diag_skip_a = debug_skip_a();
    return p;
}

// A-producer: 0 = TMA tile::gather4, 1 = cp.async (default).  NGRAM_PRODUCER overrides
// (kept for the A/B measurement recorded in DESIGN.md / profiles/).
int producer_mode() {
    static int mode = [] {
        const char* e = getenv("NGRAM_PRODUCER");
        return e ? atoi(e) : 1;
    }();
    return mode;
}

}  // namespace

// Split-K reduction + epilogue: out = amp((E0[tok] + sum_s partial[s]) * 1/denom); the
// partials are summed in split order (deterministic).  Latency shape (decode / verify): the
// E0 row is gathered BEFORE the programmatic-launch wait (tokens and E0 do not depend on the
// GEMM; a token >= V0 reads row 0, its output is never written), and the S partial loads are
// issued back to back (independent, one L2 round trip instead of S); 128-thread blocks spread
// a small batch over more SMs.
constexpr int kReduceThreads = 128;
constexpr int kReduceMaxS = 8;
__global__ void __launch_bounds__(kReduceThreads) splitk_reduce_kernel(const float* __restrict__ partial, int S,
                                                                       int64_t T, int D,
                                                            const uint32_t* __restrict__ tokens,
                                                            const __nv_bfloat16* __restrict__ e0, uint32_t V0,
                                                            float scale, float amp, int write_rows, void* rows,
                                                            void* merged, int out_bf16,
                                                            const unsigned long long* err, DecodeCommit commit,
                                                            int commit_sep) {
    const int64_t n4 = T * D / 4;
    // commit_sep: the decode-state commit runs in a block of its own (block 0, dispatched
    // first), beside the reduction blocks instead of ahead of block 0's share of the reduction
    const bool commit_here = commit.ring && blockIdx.x == 0;
    const unsigned sep = commit.ring && commit_sep ? 1u : 0u;
    const unsigned nred = gridDim.x - sep;
    const int64_t v0 = (sep && blockIdx.x == 0) ? n4 : (int64_t)(blockIdx.x - sep) * blockDim.x + threadIdx.x;
    uint2 eb0 = make_uint2(0, 0);
    if (v0 < n4) {  // first element's E0 chunk, ahead of the GEMM's completion
        const int64_t t = v0 * 4 / D;
        const uint32_t tok = __ldg(tokens + t);
        eb0 = __ldg(reinterpret_cast<const uint2*>(e0 + (int64_t)(tok < V0 ? tok : 0u) * D + (v0 * 4 - t * D)));
    }
    griddep_wait();  // PDL launch: the split-K GEMM has completed (no-op for a normal launch)
    if (commit_here) decode_commit_block(commit, err);  // fused decode-state commit
    const bool bad = *err != ~0ull;  // a token was out of range: no output (uniform)
    for (int64_t v = v0; !bad && v < n4; v += (int64_t)nred * blockDim.x) {
        const int64_t t = v * 4 / D;
        const int i = (int)(v * 4 - t * D);
        float4 acc;
        if (S <= kReduceMaxS) {
            float4 q[kReduceMaxS];
#pragma unroll
            for (int s = 0; s < kReduceMaxS; ++s)
                if (s < S) q[s] = __ldcg(reinterpret_cast<const float4*>(partial + (int64_t)s * T * D) + v);
            acc = q[0];
#pragma unroll
            for (int s = 1; s < kReduceMaxS; ++s)
                if (s < S) {
                    acc.x += q[s].x;
                    acc.y += q[s].y;
                    acc.z += q[s].z;
                    acc.w += q[s].w;
                }
        } else {
            acc = reinterpret_cast<const float4*>(partial)[v];
            for (int s = 1; s < S; ++s) {
                const float4 q = reinterpret_cast<const float4*>(partial + (int64_t)s * T * D)[v];
                acc.x += q.x;
                acc.y += q.y;
                acc.z += q.z;
                acc.w += q.w;
            }
        }
        const uint2 eb = v == v0 ? eb0 : *reinterpret_cast<const uint2*>(e0 + (int64_t)__ldg(tokens + t) * D + i);
        float m[4] = {__fmul_rn(__fadd_rn(bf16_bits_to_f32(eb.x & 0xffffu), acc.x), scale),
                      __fmul_rn(__fadd_rn(bf16_bits_to_f32(eb.x >> 16), acc.y), scale),
                      __fmul_rn(__fadd_rn(bf16_bits_to_f32(eb.y & 0xffffu), acc.z), scale),
                      __fmul_rn(__fadd_rn(bf16_bits_to_f32(eb.y >> 16), acc.w), scale)};
        auto put = [&](void* out, const float* x) {
            if (out_bf16)
                reinterpret_cast<uint2*>(out)[v] = make_uint2(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]));
            else
                reinterpret_cast<float4*>(out)[v] = make_float4(x[0], x[1], x[2], x[3]);
        };
        if (merged) put(merged, m);
        if (write_rows) {
            const float r[4] = {__fmul_rn(m[0], amp), __fmul_rn(m[1], amp), __fmul_rn(m[2], amp),
                                __fmul_rn(m[3], amp)};
            put(rows, r);
        }
    }
    if (commit.ticket) {  // decode step: the last block to finish releases the error word
        __syncthreads();  // the block's reads of the error word precede thread 0's release
        if (threadIdx.x == 0) {
            unsigned prev;
            asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(commit.ticket) : "memory");
            if (prev == gridDim.x - 1) {  // acquired every other block's release
                decode_release_err(commit, const_cast<unsigned long long*>(err));
                *commit.ticket = 0u;
            }
        }
    }
}

static int split_s1(int D, int num_sms, int mtiles = 1) {
    // BN = 128 tiles; split K until the m-tiles' grid covers the SMs (one wave)
    const int KB = D / BK;
    const int64_t nN = D / 128;
    int best = 1;
    for (int S = 1; S <= KB; ++S)
        if (KB % S == 0 && nN * mtiles * S <= num_sms) best = S;
    return best;
}

bool small_t_regime(int D, int64_t T, int num_sms) {
    // A verify-sized middle regime (256 < T <= 1024, fewer splits) was measured slower than
    // the pair kernel at D = 3072 (64 x 8 verify: 36.9 vs 34.9 us), so the split-K GEMM
    // serves T <= 256 only.
    (void)D;
    (void)num_sms;
    return T <= 256;
}

int splitk_factor(const FwdArgs& a, int num_sms) {
    // S depends only on D and the regime of T, so every row of a regime is computed
    // identically (batch-composition invariance within a regime).  Two sub-regimes: T <= 128
    // (one m-tile) and 128 < T <= 256 (two m-tiles: half the splits keep the grid at one wave).
    static const bool by_m = !(getenv("NGRAM_SPLITK_BY_M") && atoi(getenv("NGRAM_SPLITK_BY_M")) == 0);
    const int64_t rt = a.regime_T > 0 ? a.regime_T : a.T;
    return split_s1(a.s.D, num_sms, (by_m && rt > 128) ? 2 : 1);
}


int tc_variant() {  // 2 = cta_group::2 pair kernel (default when D % 256 == 0), 1 = single-CTA
    static int v = [] {
        const char* e = getenv("NGRAM_TC_VARIANT");
        return e ? atoi(e) : 2;
    }();
    return v;
}

// Programmatic dependent launch of the small-T chain (gather -> split-K GEMM -> reduce);
// NGRAM_PDL=0 launches them plainly (A/B).
static bool pdl_enabled() {
    static const bool v = !(getenv("NGRAM_PDL") && atoi(getenv("NGRAM_PDL")) == 0);
    return v;
}

size_t splitk_workspace_floats(const FwdArgs& a, int num_sms) {
    if (!small_t_regime(a.s.D, a.regime_T > 0 ? a.regime_T : a.T, num_sms) || (a.tmap_x == nullptr && a.seq_off == nullptr)) return 0;
    const int S = splitk_factor(a, num_sms);
    return S > 1 ? (size_t)S * (size_t)a.T * (size_t)a.s.D : 0;
}

void launch_forward_tc(const FwdArgs& a, int num_sms, cudaStream_t st, float* splitk_ws) {
    if (a.T <= 0) return;
    if (splitk_ws && small_t_regime(a.s.D, a.regime_T > 0 ? a.regime_T : a.T, num_sms) && (a.tmap_x != nullptr || a.seq_off != nullptr)) {
        const int S = splitk_factor(a, num_sms);
        if (S > 1) {
            const bool pdl = pdl_enabled();
            if (a.tmap_x) launch_cfg<128, 4, 0>(a, num_sms, st, S, splitk_ws, pdl);  // A from X
            else launch_cfg<128, 4, 2>(a, num_sms, st, S, splitk_ws);                // hash + gather4 in-kernel
            const float scale = 1.0f / (float)a.s.denom;
            const float amp = a.s.amp == kAmpSqrt ? (float)__builtin_sqrt((double)a.s.D) : 1.0f;
            const int64_t n4 = a.T * a.s.D / 4;
            DecodeCommit c{};
            if (a.commit) c = *a.commit;
            int64_t blocks = (n4 + kReduceThreads - 1) / kReduceThreads;
            if (blocks > num_sms * 16) blocks = num_sms * 16;
            static const int commit_sep = !(getenv("NGRAM_COMMIT_BLOCK") && atoi(getenv("NGRAM_COMMIT_BLOCK")) == 0);
            if (c.ring && commit_sep) ++blocks;
            const int wr = (a.rows_out != nullptr && a.s.amp != kAmpLN) ? 1 : 0;
            if (pdl) {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3((unsigned)blocks);
                cfg.blockDim = dim3(kReduceThreads);
                cfg.stream = st;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, splitk_reduce_kernel, (const float*)splitk_ws, S, a.T, a.s.D, a.tokens, a.e0,
                                   a.s.V0, scale, amp, wr, a.rows_out, a.merged_out, a.out_bf16, a.err, c, commit_sep);
            } else {
                splitk_reduce_kernel<<<(unsigned)blocks, kReduceThreads, 0, st>>>(
                    splitk_ws, S, a.T, a.s.D, a.tokens, a.e0, a.s.V0, scale, amp, wr, a.rows_out, a.merged_out,
                    a.out_bf16, a.err, c, commit_sep);
            }
            count_launch();
            return;
        }
    }
    const bool bn256 = a.s.D % 256 == 0;
    // Verify-sized T (past the split-K regime) whose 128 x 128 single-CTA tiles still fit one wave:
    // more SMs busy than the pair kernel's few 256 x 256 tiles (D = 3072, 64 streams x 8 drafts:
    // 96 CTAs vs 24 pairs), bit-identical results (same K order per element; tested).  Measured
    // at D = 3072, L2 flushed, verify + commit: T = 320..768 2.0-3.5 us faster; T = 1024 (two
    // waves) 10 us slower.  NGRAM_VERIFY_TILE=0 keeps the pair kernel (read per call: tests pin
    // the pair kernel's epilogue on small ragged batches with it).
    const char* vte = getenv("NGRAM_VERIFY_TILE");
    const bool vt = !(vte && atoi(vte) == 0);
    // Long K only: at D = 256 (config A, T = 2048) the 32 short tiles measured slower than the
    // 8 pair tiles (24.0 vs 23.2 us).
    if (vt && a.tmap_x && a.s.D % 128 == 0 && a.s.D >= 2048 && !small_t_regime(a.s.D, a.T, num_sms) &&
        ((a.T + 127) / 128) * (a.s.D / 128) <= num_sms && !a.wide) {
        // programmatic dependent launch: set-up overlaps the gather kernel's tail (it waits for X)
        launch_cfg<128, 4, 1>(a, num_sms, st, 1, nullptr, pdl_enabled());
        if (a.commit) launch_decode_commit_c(*a.commit, a.err, st);
        return;
    }
    if (a.wide && a.seq_off && !a.tmap_x && a.tmap_w32 != nullptr && wide_prefill_shape(a.s)) {
        launch_forward_wide(a, num_sms, st);
        if (a.commit) launch_decode_commit_c(*a.commit, a.err, st);
        return;
    }
    if (bn256 && tc_variant() == 2 && a.tmap_w2 != nullptr) {
        launch_tc2(a, num_sms, st);
        if (a.commit) launch_decode_commit_c(*a.commit, a.err, st);
        return;
    }
    if (producer_mode() == 0) {
        if (bn256) launch_cfg<256, 4, 0>(a, num_sms, st);
        else launch_cfg<128, 4, 0>(a, num_sms, st);
    } else {
        if (bn256) launch_cfg<256, 4, 1>(a, num_sms, st);
        else launch_cfg<128, 4, 1>(a, num_sms, st);
    }
    if (a.commit) launch_decode_commit_c(*a.commit, a.err, st);
}

}  // namespace ngk
