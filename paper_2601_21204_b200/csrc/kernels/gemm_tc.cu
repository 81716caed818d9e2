// gemm_tc.cu -- K2+K3 fused: the sub-table gather and the projection GEMM on the 5th-gen
// tensor cores, with the base-row add, 1/denom scale and amplification in the epilogue.
//
//   Y[t, :] = amplify( (E0[tok_t, :] + X[t, :] . W_cat^T) * fp32(1/denom) )
//   X[t, b*d:(b+1)*d] = E_b[id_b(t)]   (never materialised: gathered straight into smem)
//
// This is embed_from_ids (embedding.hpp:163-201) + amplify (:239-287) for a tile of 128
// positions: the reference's per-token D x d matvec per branch (its >99% hot loop,
// embedding.hpp:189-195) becomes ONE bf16 GEMM with K = (N-1)K*d = D (branch-
// concatenated), fp32 accumulation in TMEM.
//
// Structure (persistent, 1 CTA per SM, 6 warps, warp-specialised):
//   warp 0      TMA producer.  Per K-block (64 columns = one 128-B swizzle atom): the 32
//               lanes each issue one tile::gather4 (4 gathered rows of the sub-table, row
//               coordinate = storage row of bucket id_b(t)) -> A tile 128 x 64; lane 0
//               issues the W_cat tile 256 x 64.  Both land SWIZZLE_128B, K-major.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16).
//   warps 2..5  epilogue: tcgen05.ld accumulator rows -> + E0 row -> * 1/denom -> * amp
//               -> fp32/bf16 stores.  TMEM is double-buffered (2 x BN columns) so the
//               epilogue of tile i overlaps the MMAs of tile i+1.
// Tiles are ordered n-fastest so the CTAs running concurrently share an m-block's
// gathered rows through L2; W_cat (2*D^2 bytes) stays L2-resident.
#include <cstdint>

#include "kernels.h"
#include "ptx.cuh"

namespace ngk {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one SWIZZLE_128B atom of bf16
constexpr int kStages = 4;
constexpr int kThreads = 192;

template <int BN>
struct Cfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

struct TcParams {
    Shape s;
    const uint32_t* tokens;
    const int32_t* grow;
    const __nv_bfloat16* e0;
    void* rows_out;
    void* merged_out;
    int out_bf16;
    int write_rows;  // amp != LN
    int64_t T, Tpad;  // rows of this call, grow row stride
    float scale, amp;
    const unsigned long long* err;
    int use_x;  // A operand from materialised X (tmap_a is X) instead of gathered sub-table rows
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    forward_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_w,
                      TcParams p) {
    using C = Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    if (*p.err != ~0ull) return;  // a token was out of range: produce no output (uniform)

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int D = p.s.D;
    const int nN = D / BN;
    const int64_t nM = (p.T + BM - 1) / BM;
    const int64_t tiles = nM * nN;
    const int KB = D / BK;        // K-blocks per tile
    const int KPB = p.s.d / BK;   // K-blocks per branch (gather mode)

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
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
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        int stage = 0;
        uint32_t phase = 0;
        const uint64_t pol_w = policy_evict_last();
        for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const int64_t m = tile / nN;
            const int n = (int)(tile - m * nN);
            const int64_t t0 = m * BM;
            if (!p.use_x) {
                int4 rows = *reinterpret_cast<const int4*>(p.grow + t0 + 4 * lane);
                for (int b = 0; b < p.s.B; ++b) {
                    int4 next = rows;
                    if (b + 1 < p.s.B)
                        next = *reinterpret_cast<const int4*>(p.grow + (int64_t)(b + 1) * p.Tpad + t0 + 4 * lane);
                    for (int c = 0; c < KPB; ++c) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (lane == 0) mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                        __syncwarp();
                        uint8_t* a_dst = smem + stage * C::kStageBytes;
                        tma_gather4(a_dst + lane * 4 * (BK * 2), &tmap_a, &full[stage], c * BK, rows.x, rows.y,
                                    rows.z, rows.w);
                        if (lane == 0)
                            tma_load_2d_hint(a_dst + C::kABytes, &tmap_w, &full[stage], (b * KPB + c) * BK, n * BN,
                                             pol_w);
                        if (++stage == kStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    rows = next;
                }
            } else {
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (lane == 0) {
                        uint8_t* a_dst = smem + stage * C::kStageBytes;
                        mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                        tma_load_2d(a_dst, &tmap_a, &full[stage], kb * BK, (int32_t)t0);
                        tma_load_2d_hint(a_dst + C::kABytes, &tmap_w, &full[stage], kb * BK, n * BN, pol_w);
                    }
                    __syncwarp();
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
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
            const int64_t m = tile / nN;
            const int n = (int)(tile - m * nN);
            const int64_t t = m * BM + r;
            const bool valid = t < p.T;
            const uint32_t tok = valid ? __ldg(p.tokens + t) : 0u;
            const __nv_bfloat16* e0row = p.e0 + (int64_t)tok * D + n * BN;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
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
                    if (p.merged_out) {
                        if (p.out_bf16) {
                            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.merged_out) + o);
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                dst[i] = make_uint4(pack_bf16x2(mv[8 * i], mv[8 * i + 1]),
                                                    pack_bf16x2(mv[8 * i + 2], mv[8 * i + 3]),
                                                    pack_bf16x2(mv[8 * i + 4], mv[8 * i + 5]),
                                                    pack_bf16x2(mv[8 * i + 6], mv[8 * i + 7]));
                        } else {
                            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.merged_out) + o);
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                dst[i] = make_float4(mv[4 * i], mv[4 * i + 1], mv[4 * i + 2], mv[4 * i + 3]);
                        }
                    }
                    if (p.write_rows) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) mv[j] = __fmul_rn(mv[j], p.amp);
                        if (p.out_bf16) {
                            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.rows_out) + o);
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                dst[i] = make_uint4(pack_bf16x2(mv[8 * i], mv[8 * i + 1]),
                                                    pack_bf16x2(mv[8 * i + 2], mv[8 * i + 3]),
                                                    pack_bf16x2(mv[8 * i + 4], mv[8 * i + 5]),
                                                    pack_bf16x2(mv[8 * i + 6], mv[8 * i + 7]));
                        } else {
                            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.rows_out) + o);
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                dst[i] = make_float4(mv[4 * i], mv[4 * i + 1], mv[4 * i + 2], mv[4 * i + 3]);
                        }
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
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

template <int BN>
void launch_bn(const FwdArgs& a, int num_sms, cudaStream_t st) {
    using C = Cfg<BN>;
    TcParams p;
    p.s = a.s;
    p.tokens = a.tokens;
    p.grow = a.grow;
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
    const int64_t tiles = ((a.T + BM - 1) / BM) * (a.s.D / BN);
    int grid = (int)(tiles < num_sms ? tiles : num_sms);
    if (grid < 1) grid = 1;
    cudaFuncSetAttribute(forward_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    forward_tc_kernel<BN><<<grid, kThreads, C::kSmemBytes, st>>>(a.tmap_x ? *a.tmap_x : *a.tmap_sub, *a.tmap_w, p);
    count_launch();
}

}  // namespace

void launch_forward_tc(const FwdArgs& a, int num_sms, cudaStream_t st) {
    if (a.T <= 0) return;
    if (a.s.D % 256 == 0) launch_bn<256>(a, num_sms, st);
    else launch_bn<128>(a, num_sms, st);
}

}  // namespace ngk
