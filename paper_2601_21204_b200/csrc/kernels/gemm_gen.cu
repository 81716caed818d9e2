// gemm_gen.cu -- the dense GEMMs of the backward pass and of the per-layer N-gram FFN
// (PLNE), on the 5th-gen tensor cores with fp32-accurate products, plus a CUDA-core fp32
// GEMM for the pedantic mode.  No library GEMMs anywhere in the product.
//
//   C[M][N] (fp32, row-major) = (accumulate ? C : 0) + sum over term pairs (i, j) of A_i . B_j^T
//
// where the operands are bf16 "split terms" of fp32 matrices: x = x_1 + x_2 + x_3 with
// x_1 = bf16(x), x_2 = bf16(x - x_1), x_3 = bf16(x - x_1 - x_2) (24 mantissa bits), and an
// operand that is exact in bf16 (gathered table rows, W_cat) has one term.  With three terms
// on both sides the six products with i + j <= 2 (0-based) are kept; the dropped ones are
// below fp32 rounding.  References: embed_backward's dW_cat += u x^T and d(rows) = W^T u
// (embedding.hpp:342-376); ffn_plne / ffn_plne_backward (ple.hpp:174-196).
//
// Operand layouts: every operand is a logical [R][K] matrix (R = M for A, N for B) stored
// either K-major (element (r, k) at p[r * ld + k]) or MN-major (at p[k * ld + r]); both map
// onto tcgen05 shared-memory descriptors directly (MN-major = the descriptor's "transpose"
// bit), so no operand is ever transposed in memory.
//
// gemm2_kernel: CTA pairs (cta_group::2), 256 x 256 output tiles, BK = 64, persistent over
// tiles (n-fastest), warp-specialised as the forward projection (gemm_tc.cu):
//   warp 0      TMA producer (one elected lane; both CTAs load their own halves)
//   warps 1..8  epilogue, two per TMEM lane quadrant (128 columns each)
//   warp 9      MMA issuer (leader CTA), the highest warp id so the arbiter never starves it
//
// Accuracy: the tensor core's fp32 accumulation does not round to nearest on every update --
// measured, its error grows with the number of MMAs folded into a large accumulator (about
// 4e-8 x updates, relative; 4e-5 for six products over K = 3072).  So the K loop runs in
// chunks of chunk_kb() k-blocks, each into a FRESH TMEM accumulator (two 256-column buffers,
// alternating), the small products of a k-block are issued before the big one, and the
// epilogue warps fold every chunk into fp32 registers (IEEE adds) while the MMAs of the next
// chunk run: the error is that of one chunk, independent of K, and the hand-off is hidden
// behind the next chunk's MMAs (>= 12 MMAs of 256 x 256 x 16 per chunk).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "ptx.cuh"

namespace ngk {

namespace {

constexpr int GBM = 256;  // rows of C per pair tile (128 per CTA)
constexpr int GBN = 256;  // columns of C per pair tile (B: 128 rows per CTA)
constexpr int GBK = 64;
constexpr int kTileBytes = 128 * GBK * 2;  // one CTA's 128 x 64 bf16 slab of one term
constexpr int kEpiWarpsG = 8;
constexpr int kGemmThreads = (2 + kEpiWarpsG) * 32;
constexpr int kMmaWarpG = 1 + kEpiWarpsG;
// k-blocks per TMEM accumulation chunk: one k-block when there are six products (the five
// small ones are issued first, into a still-tiny accumulator, then the big a1 b1 -- so only its
// four MMAs meet a large accumulator), four with two or three, eight for a single product.
constexpr int chunk_kb(int pairs) { return pairs >= 6 ? 1 : pairs >= 2 ? 4 : 8; }
constexpr int kStageRowFloats = 33;  // epilogue transpose tile: 32 rows x 32 floats, padded (no bank conflicts)
constexpr int kEpiStageBytes = kEpiWarpsG * 32 * kStageRowFloats * 4;  // 33.8 KB
constexpr int kSmemBudget = 227 * 1024 - kEpiStageBytes - 2048;

constexpr int gstages(int na, int nb) {
    const int s = kSmemBudget / ((na + nb) * kTileBytes);
    return s > 6 ? 6 : s;
}
constexpr int gpairs(int na, int nb) { return (na == 3 && nb == 3) ? 6 : na * nb; }

// SWIZZLE_128B smem descriptor of an MN-major slab: 64-element (128 B) MN chunks of GBK K-rows,
// K-row stride 128 B, 8-row K groups 1024 B apart (SBO), MN chunks 8 KB apart (LBO).
__device__ __forceinline__ uint64_t smem_desc_sw128_mn(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
    d |= (uint64_t)((GBK * 128) >> 4) << 16;  // LBO: next 64-element MN chunk
    d |= (uint64_t)(1024 >> 4) << 32;         // SBO: next 8 K-rows
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

struct GemmParams {
    int64_t M, N, K;
    float* C;
    int64_t ldc;
    int accumulate;
    int staged_store;  // overwrite mode: coalesced stores through the smem transpose tile
};

// NGRAM_GEMM_STAGED_STORE=0 selects per-thread row stores in overwrite mode too (A/B switch)
int staged_store() {
    static const int v = getenv("NGRAM_GEMM_STAGED_STORE") ? atoi(getenv("NGRAM_GEMM_STAGED_STORE")) : 1;
    return v;
}

template <int NA, int NB, bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap ma0, const __grid_constant__ CUtensorMap ma1,
                 const __grid_constant__ CUtensorMap ma2, const __grid_constant__ CUtensorMap mb0,
                 const __grid_constant__ CUtensorMap mb1, const __grid_constant__ CUtensorMap mb2, GemmParams p) {
    constexpr int kStages = gstages(NA, NB);
    constexpr int kStageBytes = (NA + NB) * kTileBytes;
    constexpr int kPairs = gpairs(NA, NB);
    constexpr int kChunkKB = chunk_kb(kPairs);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* epi_stage = reinterpret_cast<float*>(smem + kStages * kStageBytes + 256);  // [8 warps][32][33]

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int64_t pair = cluster_id_x();
    const int64_t npairs = nclusters_x();
    const int64_t nN = (p.N + GBN - 1) / GBN;
    const int64_t nM = (p.M + GBM - 1) / GBM;
    const int64_t tiles = nM * nN;
    const int KB = (int)((p.K + GBK - 1) / GBK);

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 2 * kEpiWarpsG);  // the epilogue warps of both CTAs (leader's copy)
        }
        fence_mbar_init();
        tma_prefetch_desc(&ma0);
        tma_prefetch_desc(&mb0);
    }
    if (warp == kMmaWarpG) tmem_alloc_2cta<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer (both CTAs)
        if (lane == 0) {
            const CUtensorMap* mas[3] = {&ma0, &ma1, &ma2};
            const CUtensorMap* mbs[3] = {&mb0, &mb1, &mb2};
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t tile = pair; tile < tiles; tile += npairs) {
                const int64_t m = tile / nN;
                const int64_t n = tile - m * nN;
                const int32_t arow = (int32_t)(m * GBM + (int64_t)rank * 128);  // this CTA's A rows
                const int32_t brow = (int32_t)(n * GBN + (int64_t)rank * 128);  // this CTA's B rows
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* dst = smem + stage * kStageBytes;
                    const uint32_t bar = leader_bar(&full[stage]);
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
                    const int32_t k0 = kb * GBK;
#pragma unroll
                    for (int i = 0; i < NA; ++i) {
                        uint8_t* d = dst + i * kTileBytes;
                        if (A_MN) {
                            tma_load_2d_2cta(d, mas[i], bar, arow, k0, 0);
                            tma_load_2d_2cta(d + kTileBytes / 2, mas[i], bar, arow + 64, k0, 0);
                        } else {
                            tma_load_2d_2cta(d, mas[i], bar, k0, arow, 0);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        uint8_t* d = dst + (NA + j) * kTileBytes;
                        if (B_MN) {
                            tma_load_2d_2cta(d, mbs[j], bar, brow, k0, 0);
                            tma_load_2d_2cta(d + kTileBytes / 2, mbs[j], bar, brow + 64, k0, 0);
                        } else {
                            tma_load_2d_2cta(d, mbs[j], bar, k0, brow, 0);
                        }
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarpG) {
        // ------------------------------------------------------------ MMA issuer (leader only)
        if (leader) {
            constexpr uint32_t idesc =
                idesc_bf16_f32(GBM, GBN) | (A_MN ? (1u << 15) : 0u) | (B_MN ? (1u << 16) : 0u);
            // per-k16 descriptor advance (16-byte units): K-major +32 B inside the 128 B row,
            // MN-major +16 K-rows = 2048 B
            constexpr uint64_t kStepA = A_MN ? 128 : 2;
            constexpr uint64_t kStepB = B_MN ? 128 : 2;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t tile = pair; tile < tiles; tile += npairs) {
                for (int kc = 0; kc < KB; kc += kChunkKB) {
                    mbar_wait(&tempty[acc], acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + (uint32_t)(acc * GBN);
                    const int kend = kc + kChunkKB < KB ? kc + kChunkKB : KB;
                    for (int kb = kc; kb < kend; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        if (lane == 0) {
                            const uint32_t base = smem_u32(smem + stage * kStageBytes);
#pragma unroll
                            for (int pr = kPairs - 1; pr >= 0; --pr) {  // small products first
                                // pairs (i, j): NA x NB when one side has a single term, else i + j <= 2
                                const int i = (NA == 3 && NB == 3) ? (pr < 3 ? 0 : (pr < 5 ? 1 : 2)) : pr / NB;
                                const int j = (NA == 3 && NB == 3) ? (pr < 3 ? pr : (pr < 5 ? pr - 3 : 0)) : pr % NB;
                                const uint32_t aa = base + (uint32_t)(i * kTileBytes);
                                const uint32_t ba = base + (uint32_t)((NA + j) * kTileBytes);
                                const uint64_t adesc = A_MN ? smem_desc_sw128_mn(aa) : smem_desc_sw128(aa);
                                const uint64_t bdesc = B_MN ? smem_desc_sw128_mn(ba) : smem_desc_sw128(ba);
#pragma unroll
                                for (int k = 0; k < GBK / 16; ++k)
                                    tc_mma_bf16_2cta(d_tmem, adesc + (uint64_t)k * kStepA,
                                                     bdesc + (uint64_t)k * kStepB, idesc, ((kb - kc) | k | (kPairs - 1 - pr)) != 0);
                            }
                            tc_commit_2cta_mc(&empty[stage], 0x3);
                        }
                        __syncwarp();
                        if (++stage == kStages) {
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
        }
    } else {
        // ------------------------------------------------------------ epilogue (both CTAs)
        const int ew = warp - 1;       // 0..7
        const int q = warp & 3;        // TMEM lane quadrant this warp may access
        const int half = ew >> 2;      // column half (128 columns) of the tile this warp owns
        const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
        const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty[1]), 0);
        const bool vec = (p.ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(p.C) % 16) == 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t tile = pair; tile < tiles; tile += npairs) {
            const int64_t m = tile / nN;
            const int64_t n = tile - m * nN;
            const int64_t row = m * GBM + (int64_t)rank * 128 + q * 32 + lane;
            float sum[GBN / 2];
#pragma unroll
            for (int j = 0; j < GBN / 2; ++j) sum[j] = 0.0f;
            for (int kc = 0; kc < KB; kc += kChunkKB) {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < GBN / 2 / 32; c += 2) {  // two loads in flight per wait
                    uint32_t v[2][32];
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) +
                                               (uint32_t)(acc * GBN + half * (GBN / 2) + (c + h) * 32),
                                           v[h]);
                    tmem_ld_wait();
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int j = 0; j < 32; ++j) sum[(c + h) * 32 + j] += __uint_as_float(v[h][j]);
                }
                tc_fence_before();
                __syncwarp();
                // relaxed: the chunk's TMEM loads completed (tcgen05.wait::ld); a release arrive
                // would put a GPU-scope MEMBAR behind the warp's outstanding epilogue stores
                if (lane == 0) mbar_arrive_cluster_relaxed(acc == 0 ? tempty_leader0 : tempty_leader1);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
            const int64_t col0 = n * GBN + half * (GBN / 2);
            if (!p.accumulate && p.staged_store) {
                // overwrite: each 32 x 32 block goes through this warp's padded smem tile so every
                // store instruction writes one row's 32 consecutive floats (a 128-byte segment)
                // instead of 32 rows x 16 bytes (dX of the backward: 805 MB at config C)
                const int64_t row0 = row - lane;
                const int nr = p.M - row0 < 32 ? (p.M - row0 > 0 ? (int)(p.M - row0) : 0) : 32;
                float* stg = epi_stage + (warp - 1) * 32 * kStageRowFloats;
#pragma unroll
                for (int c = 0; c < GBN / 2 / 32; ++c) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) stg[lane * kStageRowFloats + j] = sum[c * 32 + j];
                    __syncwarp();
                    const int64_t col = col0 + c * 32 + lane;
                    if (col < p.N) {
                        float* dst = p.C + row0 * p.ldc + col;
#pragma unroll 4
                        for (int r = 0; r < nr; ++r) dst[r * p.ldc] = stg[r * kStageRowFloats + lane];
                    }
                    __syncwarp();
                }
            } else if (row < p.M && col0 < p.N) {
                float* dst = p.C + row * p.ldc + col0;
                if (vec && col0 + GBN / 2 <= p.N) {
#pragma unroll
                    for (int i = 0; i < GBN / 8; ++i) {
                        float4 o = make_float4(sum[4 * i], sum[4 * i + 1], sum[4 * i + 2], sum[4 * i + 3]);
                        if (p.accumulate) {
                            const float4 c4 = reinterpret_cast<const float4*>(dst)[i];
                            o.x += c4.x;
                            o.y += c4.y;
                            o.z += c4.z;
                            o.w += c4.w;
                        }
                        reinterpret_cast<float4*>(dst)[i] = o;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < GBN / 2; ++j)
                        if (col0 + j < p.N) dst[j] = sum[j] + (p.accumulate ? dst[j] : 0.0f);
                }
            }
        }
    }

    tc_fence_before();
    cluster_sync();  // every MMA retired and every remote arrive delivered before TMEM is freed
    if (warp == kMmaWarpG) {
        tc_fence_after();
        tmem_dealloc_2cta<512>(tmem_base);
    }
}

template <int NA, int NB, bool A_MN, bool B_MN>
void launch_g2(const CUtensorMap* ma, const CUtensorMap* mb, const GemmParams& p, int num_sms, cudaStream_t st) {
    constexpr int kStages = gstages(NA, NB);
    constexpr int smem = kStages * (NA + NB) * kTileBytes + 1024 + 256 + kEpiStageBytes;
    const int64_t tiles = ((p.M + GBM - 1) / GBM) * ((p.N + GBN - 1) / GBN);
    int64_t pairs = num_sms / 2;
    if (tiles < pairs) pairs = tiles;
    if (pairs < 1) pairs = 1;
    auto k = gemm2_kernel<NA, NB, A_MN, B_MN>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<(unsigned)(2 * pairs), kGemmThreads, smem, st>>>(ma[0], ma[NA > 1 ? 1 : 0], ma[NA > 2 ? 2 : 0], mb[0],
                                                       mb[NB > 1 ? 1 : 0], mb[NB > 2 ? 2 : 0], p);
    count_launch();
}

template <int NA, int NB>
void dispatch_major(const CUtensorMap* ma, const CUtensorMap* mb, bool a_mn, bool b_mn, const GemmParams& p,
                    int num_sms, cudaStream_t st) {
    if (a_mn && b_mn) launch_g2<NA, NB, true, true>(ma, mb, p, num_sms, st);
    else if (a_mn) launch_g2<NA, NB, true, false>(ma, mb, p, num_sms, st);
    else if (b_mn) launch_g2<NA, NB, false, true>(ma, mb, p, num_sms, st);
    else launch_g2<NA, NB, false, false>(ma, mb, p, num_sms, st);
}

// ---------------------------------------------------------------- fp32 CUDA-core GEMM
// Pedantic mode and shapes without a tensor-core tile: 64 x 64 tiles, 256 threads, 4 x 4
// outputs per thread, fp32 FMA in k order.  Operands in the same [R][K] convention.
constexpr int FB = 64, FK = 16;
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int64_t lda, int a_mn,
                                                       const float* __restrict__ B, int64_t ldb, int b_mn,
                                                       GemmParams p) {
    __shared__ float As[FK][FB + 4];
    __shared__ float Bs[FK][FB + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t m0 = (int64_t)blockIdx.y * FB, n0 = (int64_t)blockIdx.x * FB;
    float acc[4][4] = {};
    for (int64_t k0 = 0; k0 < p.K; k0 += FK) {
        for (int e = threadIdx.x; e < FB * FK; e += 256) {
            // MN-major operands: consecutive threads walk the contiguous MN index
            const int r = a_mn ? e % FB : e / FK, kk = a_mn ? e / FB : e % FK;
            const int64_t gr = m0 + r, gk = k0 + kk;
            As[kk][r] = (gr < p.M && gk < p.K) ? A[a_mn ? gk * lda + gr : gr * lda + gk] : 0.0f;
            const int rb = b_mn ? e % FB : e / FK, kb = b_mn ? e / FB : e % FK;
            const int64_t gn = n0 + rb, gkb = k0 + kb;
            Bs[kb][rb] = (gn < p.N && gkb < p.K) ? B[b_mn ? gkb * ldb + gn : gn * ldb + gkb] : 0.0f;
        }
        __syncthreads();
        // per-block partial sums (k order inside the block), then one add into the running sum:
        // the rounding error grows with sqrt(K / FK) block adds instead of sqrt(K) fmas
        float part[4][4] = {};
#pragma unroll
        for (int kk = 0; kk < FK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                a[i] = As[kk][ty * 4 + i];
                b[i] = Bs[kk][tx * 4 + i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) part[i][j] = fmaf(a[i], b[j], part[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] += part[i][j];
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = m0 + ty * 4 + i;
        if (r >= p.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t c = n0 + tx * 4 + j;
            if (c < p.N) {
                float* d = p.C + r * p.ldc + c;
                *d = p.accumulate ? *d + acc[i][j] : acc[i][j];
            }
        }
    }
}

// x -> (x1, x2, x3) bf16 with x = x1 + x2 + x3 to 24 bits; rows x cols with pitches
__global__ void split3_kernel(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                              __nv_bfloat16* __restrict__ t0, __nv_bfloat16* __restrict__ t1,
                              __nv_bfloat16* __restrict__ t2, int64_t ldt) {
    const int64_t n = rows * cols;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / cols, c = e - r * cols;
        const float v = x[r * ldx + c];
        const __nv_bfloat16 a = __float2bfloat16_rn(v);
        const float r1 = v - __bfloat162float(a);
        const __nv_bfloat16 b = __float2bfloat16_rn(r1);
        const __nv_bfloat16 cc = __float2bfloat16_rn(r1 - __bfloat162float(b));
        t0[r * ldt + c] = a;
        if (t1) t1[r * ldt + c] = b;
        if (t2) t2[r * ldt + c] = cc;
    }
}

}  // namespace

void launch_gemm_bf16_terms(const CUtensorMap* ma, int na, bool a_mn, const CUtensorMap* mb, int nb, bool b_mn,
                            int64_t M, int64_t N, int64_t K, float* C, int64_t ldc, bool accumulate, int num_sms,
                            cudaStream_t st) {
    const GemmParams p{M, N, K, C, ldc, accumulate ? 1 : 0, staged_store()};
    if (na == 1 && nb == 1) dispatch_major<1, 1>(ma, mb, a_mn, b_mn, p, num_sms, st);
    else if (na == 3 && nb == 1) dispatch_major<3, 1>(ma, mb, a_mn, b_mn, p, num_sms, st);
    else if (na == 2 && nb == 1) dispatch_major<2, 1>(ma, mb, a_mn, b_mn, p, num_sms, st);
    else if (na == 1 && nb == 3) dispatch_major<1, 3>(ma, mb, a_mn, b_mn, p, num_sms, st);
    else dispatch_major<3, 3>(ma, mb, a_mn, b_mn, p, num_sms, st);
}

void launch_gemm_f32(const float* A, int64_t lda, bool a_mn, const float* B, int64_t ldb, bool b_mn, int64_t M,
                     int64_t N, int64_t K, float* C, int64_t ldc, bool accumulate, cudaStream_t st) {
    if (M <= 0 || N <= 0) return;
    const GemmParams p{M, N, K, C, ldc, accumulate ? 1 : 0, 0};
    const dim3 grid((unsigned)((N + FB - 1) / FB), (unsigned)((M + FB - 1) / FB));
    gemm_f32_kernel<<<grid, 256, 0, st>>>(A, lda, a_mn ? 1 : 0, B, ldb, b_mn ? 1 : 0, p);
    count_launch();
}

void launch_split3(const float* x, int64_t rows, int64_t cols, int64_t ldx, __nv_bfloat16* t0, __nv_bfloat16* t1,
                   __nv_bfloat16* t2, int64_t ldt, cudaStream_t st) {
    const int64_t n = rows * cols;
    if (n <= 0) return;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    split3_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, rows, cols, ldx, t0, t1, t2, ldt);
    count_launch();
}

}  // namespace ngk
