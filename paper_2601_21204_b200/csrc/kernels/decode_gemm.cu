// decode_gemm.cu -- the small-batch projection (decode steps / verify blocks, T <= 256):
// Y = amplify((E0[tok] + X . W_cat^T) * 1/denom) in ONE kernel.
//
// W_cat (2*D^2 bytes, 18.9 MB at D=3072) dominates the bytes, so it is streamed exactly
// once: every CTA owns a 128-column slice of the output (a W_cat row block) and one of S
// K-ranges (split-K), and computes ALL T <= 256 tokens with two 128-row TMEM accumulators
// that share each W tile.  The S CTAs of an output slice form a thread-block cluster:
// each writes its fp32 partial tile, a cluster barrier orders them, and each CTA then
// reduces a 1/S share of the rows across the S partials (in split order: deterministic),
// adds the E0 row, scales and amplifies, and stores.  Optionally CTA 0 also commits the
// decode state (the ring update of sequence_cache::append, cache.cpp:49-55), so a decode
// step is: hash+gather kernel -> this kernel.
//
// Warps: 0 TMA producer, 1..4 epilogue / reduce (TMEM lane quadrants), 5 MMA issuer
// (highest id: first pick of the warp arbiter).
#include <cstdint>

#include "decodedev.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace ngk {

namespace {

constexpr int DBN = 128;  // output columns per cluster
constexpr int DBK = 64;
constexpr int kDStages = 4;
constexpr int kDThreads = 192;
constexpr int kAB = 128 * DBK * 2;  // one 128-row A (X) tile
constexpr int kBB = DBN * DBK * 2;  // W tile
constexpr int kDStage = 2 * kAB + kBB;
constexpr int kDSmem = kDStages * kDStage + 1024 + 256;

struct DecParams {
    int D;
    int S;    // split-K factor = cluster size
    int KBs;  // K-blocks per split
    int64_t T;
    const uint32_t* tokens;
    const __nv_bfloat16* e0;
    float* partial;  // [nN][S][256][DBN]
    void* rows;
    void* merged;
    int out_bf16;
    int write_rows;
    float scale, amp;
    const unsigned long long* err;
    DecodeCommit commit;
};

__global__ void __launch_bounds__(kDThreads, 1)
    decode_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                       DecParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kDStages * kDStage);
    uint64_t* empty = full + kDStages;
    uint64_t* tfull = empty + kDStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

    if (*p.err != ~0ull) return;  // uniform: a token was out of range, produce nothing

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int S = p.S;
    const int n = blockIdx.x / S;   // output column slice (= cluster id)
    const int ks = blockIdx.x % S;  // K split (= rank in the cluster)
    const bool two = p.T > 128;     // second 128-row accumulator in use

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kDStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmap_x);
        tma_prefetch_desc(&tmap_w);
    }
    if (warp == 5) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        const uint64_t pol_w = policy_evict_first();  // W is read exactly once per step
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = ks * p.KBs; kb < (ks + 1) * p.KBs; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (lane == 0) {
                uint8_t* dst = smem + stage * kDStage;
                mbar_arrive_expect_tx(&full[stage], (two ? 2 * kAB : kAB) + kBB);
                tma_load_2d(dst, &tmap_x, &full[stage], kb * DBK, 0);
                if (two) tma_load_2d(dst + kAB, &tmap_x, &full[stage], kb * DBK, 128);
                tma_load_2d_hint(dst + 2 * kAB, &tmap_w, &full[stage], kb * DBK, n * DBN, pol_w);
            }
            __syncwarp();
            if (++stage == kDStages) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = idesc_bf16_f32(128, DBN);
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < p.KBs; ++i) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t base = smem_u32(smem + stage * kDStage);
                const uint64_t a0 = smem_desc_sw128(base);
                const uint64_t a1 = smem_desc_sw128(base + kAB);
                const uint64_t bd = smem_desc_sw128(base + 2 * kAB);
#pragma unroll
                for (int k = 0; k < DBK / 16; ++k) {
                    tc_mma_bf16(tmem_base, a0 + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, (i | k) != 0);
                    if (two)
                        tc_mma_bf16(tmem_base + DBN, a1 + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc,
                                    (i | k) != 0);
                }
                tc_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == kDStages) {
                stage = 0;
                phase ^= 1;
            }
        }
        if (lane == 0) tc_commit(tfull);
        __syncwarp();
    } else {
        // ------------------------------------------------------------ partial tile -> global
        const int q = warp & 3;
        mbar_wait(tfull, 0);
        tc_fence_after();
        for (int a = 0; a < (two ? 2 : 1); ++a) {
            const int row = a * 128 + q * 32 + lane;
            float* dst = p.partial + (((int64_t)n * S + ks) * 256 + row) * DBN;
#pragma unroll 1
            for (int c = 0; c < DBN / 32; ++c) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * DBN + c * 32), v);
                tmem_ld_wait();
                if (row < p.T) {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        reinterpret_cast<float4*>(dst + c * 32)[i] =
                            make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                        __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                }
            }
        }
    }

    tc_fence_before();
    cluster_sync();  // every split's partial tile written (release/acquire at cluster scope)

    // ---------------------------------------------------------------- reduce + epilogue
    const int64_t R0 = (p.T + S - 1) / S;
    const int64_t r_lo = ks * R0, r_hi = (r_lo + R0 < p.T) ? r_lo + R0 : p.T;
    const int64_t items = (r_hi > r_lo ? r_hi - r_lo : 0) * (DBN / 4);
    for (int64_t it = threadIdx.x; it < items; it += kDThreads) {
        const int64_t row = r_lo + it / (DBN / 4);
        const int c4 = (int)(it % (DBN / 4)) * 4;
        const float* src = p.partial + ((int64_t)n * S * 256 + row) * DBN + c4;
        float4 acc = *reinterpret_cast<const float4*>(src);
        for (int s2 = 1; s2 < S; ++s2) {
            const float4 x = *reinterpret_cast<const float4*>(src + (int64_t)s2 * 256 * DBN);
            acc.x += x.x;
            acc.y += x.y;
            acc.z += x.z;
            acc.w += x.w;
        }
        const int col = n * DBN + c4;
        const uint2 eb = *reinterpret_cast<const uint2*>(p.e0 + (int64_t)__ldg(p.tokens + row) * p.D + col);
        const float m[4] = {__fmul_rn(__fadd_rn(bf16_bits_to_f32(eb.x & 0xffffu), acc.x), p.scale),
                            __fmul_rn(__fadd_rn(bf16_bits_to_f32(eb.x >> 16), acc.y), p.scale),
                            __fmul_rn(__fadd_rn(bf16_bits_to_f32(eb.y & 0xffffu), acc.z), p.scale),
                            __fmul_rn(__fadd_rn(bf16_bits_to_f32(eb.y >> 16), acc.w), p.scale)};
        const int64_t o = row * p.D + col;
        auto put = [&](void* out, const float* x) {
            if (p.out_bf16)
                *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(out) + o) =
                    make_uint2(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]));
            else
                *reinterpret_cast<float4*>(static_cast<float*>(out) + o) = make_float4(x[0], x[1], x[2], x[3]);
        };
        if (p.merged) put(p.merged, m);
        if (p.write_rows) {
            const float r[4] = {__fmul_rn(m[0], p.amp), __fmul_rn(m[1], p.amp), __fmul_rn(m[2], p.amp),
                                __fmul_rn(m[3], p.amp)};
            put(p.rows, r);
        }
    }

    // ---------------------------------------------------------------- fused decode commit
    if (p.commit.ring && blockIdx.x == 0) decode_commit_block(p.commit, p.err);

    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc<256>(tmem_base);
    }
}

}  // namespace

int decode_gemm_splits(int D, int num_sms) {
    const int KB = D / DBK, nN = D / DBN;
    int best = 1;
    for (int S = 1; S <= 8 && S <= KB; ++S)  // portable cluster size
        if (KB % S == 0 && nN * S <= num_sms) best = S;
    return best;
}

size_t decode_gemm_workspace_floats(int D, int num_sms) {
    return (size_t)(D / DBN) * decode_gemm_splits(D, num_sms) * 256 * DBN;
}

void launch_decode_gemm(const FwdArgs& a, int num_sms, float* partial, const DecodeCommit* commit, cudaStream_t st) {
    const int S = decode_gemm_splits(a.s.D, num_sms);
    DecParams p{};
    p.D = a.s.D;
    p.S = S;
    p.KBs = a.s.D / DBK / S;
    p.T = a.T;
    p.tokens = a.tokens;
    p.e0 = a.e0;
    p.partial = partial;
    p.rows = a.rows_out;
    p.merged = a.merged_out;
    p.out_bf16 = a.out_bf16;
    p.write_rows = (a.rows_out != nullptr && a.s.amp != kAmpLN) ? 1 : 0;
    p.scale = 1.0f / (float)a.s.denom;
    p.amp = a.s.amp == kAmpSqrt ? (float)__builtin_sqrt((double)a.s.D) : 1.0f;
    p.err = a.err;
    if (commit) p.commit = *commit;
    cudaFuncSetAttribute(decode_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDSmem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)((a.s.D / DBN) * S));
    cfg.blockDim = dim3(kDThreads);
    cfg.dynamicSmemBytes = kDSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, decode_gemm_kernel, *a.tmap_x, *a.tmap_w2, p);
    count_launch();
}

}  // namespace ngk
