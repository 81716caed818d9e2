// backward.cu -- the gradient of embed_sequence_cached w.r.t. the bank parameters
// (embedding.hpp:291-459), the irregular parts on CUDA cores:
//   * amp_backward_kernel: warp per row -- amplify_backward (embedding.hpp:291-336) from the
//     pre-amplification `merged` row and the upstream row, then u = fp32(1/denom) * d_pre
//     (embedding.hpp:350-357); u is written to U[t] (the GEMM operand) and scattered into the
//     E0 gradient row of the token; layer_norm accumulates the gain / bias gradients per
//     block in shared memory, one global atomic per column per block.
//   * gather_rows_f32_kernel: X[t] = the (bf16) sub-table rows of position t, widened to f32
//     (the right operand of dW_cat = U^T X).
//   * scatter_rows_kernel: the sub-table gradients, g_sub[row_b(t)] += dX[t, b*d:(b+1)*d]
//     (v2: dX = U W_cat) or += U[t] (v1: averaged rows, embedding.hpp:364-365).
// The two dense products (dW_cat += U^T X, dX = U W_cat) run in gemm_gen.cu; on tensor-core
// banks amp_backward writes u straight as its bf16 split terms (the GEMM operand).  Accumulation order differs from the reference's sequential loops (atomics),
// so parity is within a stated fp32 tolerance against the reference's double path.
#include <cuda_bf16.h>

#include <cstdint>

#include "kernels.h"

namespace ngk {

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int kBwdWarps = 8;

// u -> the GEMM operand: fp32 (U) and / or `nterms` bf16 split terms (u = t1 + t2 (+ t3), each
// the bf16 rounding of the remainder; terms[h * tstride + i])
__device__ __forceinline__ void put_u(float u, int64_t i, float* __restrict__ U, __nv_bfloat16* __restrict__ terms,
                                      int nterms, int64_t tstride) {
    if (U) U[i] = u;
    if (terms) {
        float r = u;
        for (int h = 0; h < nterms; ++h) {
            const __nv_bfloat16 b = __float2bfloat16_rn(r);
            terms[h * tstride + i] = b;
            r -= __bfloat162float(b);
        }
    }
}

__global__ void __launch_bounds__(kBwdWarps * 32) amp_backward_kernel(
    const float* __restrict__ up, const float* __restrict__ pre, const uint32_t* __restrict__ tokens, int64_t T,
    int D, int amp, float scale, float sqrt_d, const float* __restrict__ gain, float* __restrict__ U,
    __nv_bfloat16* __restrict__ terms, int nterms, int64_t tstride, float* __restrict__ g_e0,
    float* __restrict__ g_gain, float* __restrict__ g_bias, const unsigned long long* __restrict__ err) {
    extern __shared__ float s_ln[];  // [2][D] gain / bias partials (layer_norm only)
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (*err != ~0ull) {  // a bad token: no gradient is produced (hashing.cpp:49-54)
        // u = 0, so the dense products that follow (which do not read the error word) add exact
        // zeros to the W_cat gradient instead of stale workspace contents
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T * D; i += (int64_t)gridDim.x * blockDim.x)
            put_u(0.0f, i, U, terms, nterms, tstride);
        return;
    }
    if (amp == kAmpLN) {
        for (int i = threadIdx.x; i < 2 * D; i += blockDim.x) s_ln[i] = 0.0f;
        __syncthreads();
    }
    const bool vec = amp != kAmpLN && (D % 4) == 0;
    for (int64_t t = (int64_t)blockIdx.x * kBwdWarps + warp; t < T; t += (int64_t)gridDim.x * kBwdWarps) {
        const float* ur = up + t * D;
        float* g0 = g_e0 ? g_e0 + (int64_t)tokens[t] * D : nullptr;  // null: sparse E0 (U holds the pairs)
        if (vec) {
            // 16-byte loads, stores and vector atomics (red.global.add.v4.f32): a quarter of the
            // atomic operations of the scalar form
            const bool two = amp == kAmpSqrt;  // reference order: (up * sqrt(D)) * (1/denom)
            for (int i = 4 * lane; i < D; i += 128) {
                const float4 x = *reinterpret_cast<const float4*>(ur + i);
                float4 u;
                if (two) {
                    u = make_float4(scale * (x.x * sqrt_d), scale * (x.y * sqrt_d), scale * (x.z * sqrt_d),
                                    scale * (x.w * sqrt_d));
                } else {
                    u = make_float4(scale * x.x, scale * x.y, scale * x.z, scale * x.w);
                }
                const int64_t o = t * D + i;
                if (U) *reinterpret_cast<float4*>(U + o) = u;
                if (terms) {
                    float r[4] = {u.x, u.y, u.z, u.w};
                    for (int h = 0; h < nterms; ++h) {
                        __nv_bfloat162 lo = __floats2bfloat162_rn(r[0], r[1]);
                        __nv_bfloat162 hi = __floats2bfloat162_rn(r[2], r[3]);
                        uint2 pk;
                        pk.x = *reinterpret_cast<uint32_t*>(&lo);
                        pk.y = *reinterpret_cast<uint32_t*>(&hi);
                        *reinterpret_cast<uint2*>(terms + h * tstride + o) = pk;
                        r[0] -= __low2float(lo);
                        r[1] -= __high2float(lo);
                        r[2] -= __low2float(hi);
                        r[3] -= __high2float(hi);
                    }
                }
                if (g_e0) atomicAdd(reinterpret_cast<float4*>(g0 + i), u);
            }
        } else if (amp == kAmpLN) {
            const float* pr = pre + t * D;
            float sum = 0.0f;
            for (int i = lane; i < D; i += 32) sum += pr[i];
            const float mean = warp_sum(sum) / (float)D;
            float sq = 0.0f;
            for (int i = lane; i < D; i += 32) {
                const float c = pr[i] - mean;
                sq += c * c;
            }
            const float var = warp_sum(sq) / (float)D;
            const float inv_std = 1.0f / sqrtf(var + 1e-5f);
            float ms = 0.0f, msx = 0.0f;
            for (int i = lane; i < D; i += 32) {
                const float xhat = (pr[i] - mean) * inv_std;
                const float s = ur[i] * gain[i];
                atomicAdd(&s_ln[i], ur[i] * xhat);
                atomicAdd(&s_ln[D + i], ur[i]);
                ms += s;
                msx += s * xhat;
            }
            const float mean_s = warp_sum(ms) / (float)D;
            const float mean_sx = warp_sum(msx) / (float)D;
            for (int i = lane; i < D; i += 32) {
                const float xhat = (pr[i] - mean) * inv_std;
                const float s = ur[i] * gain[i];
                const float u = scale * ((s - mean_s - xhat * mean_sx) * inv_std);
                put_u(u, t * D + i, U, terms, nterms, tstride);
                if (g_e0) atomicAdd(&g0[i], u);
            }
        } else {
            for (int i = lane; i < D; i += 32) {
                const float u = scale * (amp == kAmpSqrt ? ur[i] * sqrt_d : ur[i]);
                put_u(u, t * D + i, U, terms, nterms, tstride);
                if (g_e0) atomicAdd(&g0[i], u);
            }
        }
    }
    if (amp == kAmpLN) {
        __syncthreads();
        for (int i = threadIdx.x; i < D; i += blockDim.x) {
            atomicAdd(&g_gain[i], s_ln[i]);
            atomicAdd(&g_bias[i], s_ln[D + i]);
        }
    }
}

// dense[tok[i]][:] += vals[i][:] (the sparse base-table gradient, densified on request)
__global__ void coo_densify_kernel(const int32_t* __restrict__ tok, const float* __restrict__ vals, int64_t n, int D,
                                   float* __restrict__ dense) {
    const int64_t total = n * D;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / D;
        atomicAdd(&dense[(int64_t)tok[i] * D + (e - i * D)], vals[e]);
    }
}

// one thread per (position, branch, column) -- any branch width
__global__ void gather_rows_f32_scalar_kernel(const int32_t* __restrict__ grow, int64_t Tpad, int64_t T, int B, int d,
                                              const __nv_bfloat16* __restrict__ sub, float* __restrict__ X,
                                              const unsigned long long* __restrict__ err) {
    const bool bad = *err != ~0ull;  // X = 0 then: the GEMMs after it must add exact zeros
    const int64_t n = T * B * d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i % d);
        const int64_t tb = i / d;
        const int b = (int)(tb % B);
        const int64_t t = tb / B;
        const int32_t row = bad ? -1 : grow[(int64_t)b * Tpad + t];
        X[i] = row >= 0 ? __bfloat162float(sub[(int64_t)row * d + j]) : 0.0f;
    }
}

// one thread per (position, branch, 8 columns), d % 8 == 0
__global__ void gather_rows_f32_kernel(const int32_t* __restrict__ grow, int64_t Tpad, int64_t T, int B, int d,
                                       const __nv_bfloat16* __restrict__ sub, float* __restrict__ X,
                                       const unsigned long long* __restrict__ err) {
    const bool bad = *err != ~0ull;  // X = 0 then: the GEMMs after it must add exact zeros
    const int per_row = d / 8;
    const int64_t n = T * B * per_row;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % per_row);
        const int64_t tb = i / per_row;
        const int b = (int)(tb % B);
        const int64_t t = tb / B;
        const int32_t row = bad ? -1 : grow[(int64_t)b * Tpad + t];
        const uint4 v = row >= 0 ? *reinterpret_cast<const uint4*>(sub + (int64_t)row * d + c * 8)
                                 : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        float* dst = X + t * (int64_t)B * d + (int64_t)b * d + c * 8;
        float4 lo, hi;
        lo.x = __uint_as_float(w[0] << 16);
        lo.y = __uint_as_float(w[0] & 0xffff0000u);
        lo.z = __uint_as_float(w[1] << 16);
        lo.w = __uint_as_float(w[1] & 0xffff0000u);
        hi.x = __uint_as_float(w[2] << 16);
        hi.y = __uint_as_float(w[2] & 0xffff0000u);
        hi.z = __uint_as_float(w[3] << 16);
        hi.w = __uint_as_float(w[3] & 0xffff0000u);
        reinterpret_cast<float4*>(dst)[0] = lo;
        reinterpret_cast<float4*>(dst)[1] = hi;
    }
}

// g_sub[row_b(t)][j] += src[t][b*width_src_off + j], one thread per (position, branch, column)
__global__ void scatter_rows_kernel(const int32_t* __restrict__ grow, int64_t Tpad, int64_t T, int B, int w,
                                    int src_stride, int src_branch_step, const float* __restrict__ src,
                                    float* __restrict__ g_sub, const unsigned long long* __restrict__ err) {
    if (*err != ~0ull) return;
    const int64_t n = T * B * w;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i % w);
        const int64_t tb = i / w;
        const int b = (int)(tb % B);
        const int64_t t = tb / B;
        const int32_t row = grow[(int64_t)b * Tpad + t];
        if (row < 0) continue;  // not stored on this shard
        atomicAdd(&g_sub[(int64_t)row * w + j], src[t * src_stride + (int64_t)b * src_branch_step + j]);
    }
}

// rows[t * B + b] = grow[b][t]: the storage rows of the appended sparse pairs, (t, b) order
__global__ void rows_to_coo_kernel(const int32_t* __restrict__ grow, int64_t Tpad, int64_t T, int B,
                                   int32_t* __restrict__ rows, const unsigned long long* __restrict__ err) {
    const bool bad = *err != ~0ull;  // a call with an out-of-range token appends no gradient
    const int64_t n = T * B;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / B;
        const int b = (int)(i - t * B);
        rows[i] = bad ? -1 : grow[(int64_t)b * Tpad + t];
    }
}

__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ src, float* __restrict__ dst, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __bfloat162float(src[i]);
}

// u -> (hi, lo): hi = u rounded to the nearest TF32 value (exact in a TF32 GEMM), lo = u - hi
// (exact in fp32).  hi is written over u.
__global__ void split_tf32_kernel(float* __restrict__ u, float* __restrict__ lo, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = u[i];
        uint32_t h;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
        const float hf = __uint_as_float(h);
        u[i] = hf;
        lo[i] = x - hf;
    }
}

__global__ void split_tf32_copy_kernel(const float* __restrict__ a, float* __restrict__ hi, float* __restrict__ lo,
                                       int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = a[i];
        uint32_t h;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
        hi[i] = __uint_as_float(h);
        lo[i] = x - __uint_as_float(h);
    }
}

// u -> u1 + u2 + u3, three bf16 terms (round to nearest each): 24 mantissa bits, |u - sum| ~2^-25 |u|
__global__ void split_bf16x3_kernel(const float* __restrict__ u, __nv_bfloat16* __restrict__ u1,
                                    __nv_bfloat16* __restrict__ u2, __nv_bfloat16* __restrict__ u3, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = u[i];
        const __nv_bfloat16 a = __float2bfloat16_rn(x);
        const float r1 = x - __bfloat162float(a);
        const __nv_bfloat16 b = __float2bfloat16_rn(r1);
        const float r2 = r1 - __bfloat162float(b);
        u1[i] = a;
        u2[i] = b;
        u3[i] = __float2bfloat16_rn(r2);
    }
}

int grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g > 148 * 16) g = 148 * 16;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

void launch_amp_backward(const Shape& s, const float* up, const float* pre, const uint32_t* tokens, int64_t T,
                         int amp, const float* gain, float* U, float* g_e0, float* g_gain, float* g_bias,
                         const unsigned long long* err, cudaStream_t st, __nv_bfloat16* terms, int nterms,
                         int64_t tstride) {
    if (T <= 0) return;
    const float scale = 1.0f / (float)s.denom;  // T(1) / T(denom), embedding.hpp:350
    const float sqrt_d = (float)__builtin_sqrt((double)s.D);
    int64_t blocks = (T + kBwdWarps - 1) / kBwdWarps;
    if (blocks > 148 * 4) blocks = 148 * 4;
    const size_t smem = amp == kAmpLN ? 2 * (size_t)s.D * sizeof(float) : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(amp_backward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    amp_backward_kernel<<<(unsigned)blocks, kBwdWarps * 32, smem, st>>>(up, pre, tokens, T, s.D, amp, scale, sqrt_d,
                                                                        gain, U, terms, nterms, tstride, g_e0, g_gain,
                                                                        g_bias, err);
    count_launch();
}

void launch_gather_rows_f32(const Shape& s, const int32_t* grow, int64_t Tpad, int64_t T, const __nv_bfloat16* sub,
                            float* X, const unsigned long long* err, cudaStream_t st) {
    if (T <= 0 || s.B == 0) return;
    if (s.d % 8 == 0)
        gather_rows_f32_kernel<<<grid_for(T * s.B * (s.d / 8), 256), 256, 0, st>>>(grow, Tpad, T, s.B, s.d, sub, X, err);
    else
        gather_rows_f32_scalar_kernel<<<grid_for(T * s.B * s.d, 256), 256, 0, st>>>(grow, Tpad, T, s.B, s.d, sub, X,
                                                                                    err);
    count_launch();
}

void launch_scatter_rows(const Shape& s, const int32_t* grow, int64_t Tpad, int64_t T, int width, int src_stride,
                         int src_branch_step, const float* src, float* g_sub, const unsigned long long* err,
                         cudaStream_t st) {
    if (T <= 0 || s.B == 0) return;
    scatter_rows_kernel<<<grid_for(T * s.B * width, 256), 256, 0, st>>>(grow, Tpad, T, s.B, width, src_stride,
                                                                       src_branch_step, src, g_sub, err);
    count_launch();
}

void launch_rows_to_coo(const Shape& s, const int32_t* grow, int64_t Tpad, int64_t T, int32_t* rows,
                        const unsigned long long* err, cudaStream_t st) {
    if (T <= 0 || s.B == 0) return;
    rows_to_coo_kernel<<<grid_for(T * s.B, 256), 256, 0, st>>>(grow, Tpad, T, s.B, rows, err);
    count_launch();
}

void launch_split_bf16x3(const float* u, __nv_bfloat16* u1, __nv_bfloat16* u2, __nv_bfloat16* u3, int64_t n,
                         cudaStream_t st) {
    if (n <= 0) return;
    split_bf16x3_kernel<<<grid_for(n, 256), 256, 0, st>>>(u, u1, u2, u3, n);
    count_launch();
}

void launch_split_tf32_copy(const float* a, float* hi, float* lo, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    split_tf32_copy_kernel<<<grid_for(n, 256), 256, 0, st>>>(a, hi, lo, n);
    count_launch();
}

void launch_split_tf32(float* u, float* lo, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    split_tf32_kernel<<<grid_for(n, 256), 256, 0, st>>>(u, lo, n);
    count_launch();
}

void launch_bf16_to_f32(const __nv_bfloat16* src, float* dst, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    bf16_to_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(src, dst, n);
    count_launch();
}

void launch_coo_densify(const int32_t* tok, const float* vals, int64_t n, int D, float* dense, cudaStream_t st) {
    if (n <= 0) return;
    coo_densify_kernel<<<grid_for(n * D, 256), 256, 0, st>>>(tok, vals, n, D, dense);
    count_launch();
}

}  // namespace ngk
