// simt.cu -- CUDA-core kernels of the forward path:
//   * forward_v1:  the averaged-variant gather-reduce (embedding.hpp:186-187): each token
//     sums E0(t) and its N-1 full-width rows in fp32, 16-byte vector loads, then scales and
//     amplifies.  HBM-bound; elementwise adds in the reference's order, so for amp none /
//     scale_sqrt_d it is bit-identical to the reference's float path.
//   * forward_v2_simt: the sub-table variant for shapes the tensor-core tile cannot take
//     (d % 64 != 0 or D % 128 != 0): one CTA per token, rows staged in shared memory, the
//     projection evaluated with the reference's float op order (embedding.hpp:189-200:
//     per-branch sequential-j accumulator, separate multiply and add, then out += acc), so
//     it too is bit-identical to the reference's float path.
//   * layernorm_rows: amplify(layer_norm) (embedding.hpp:257-278) over merged rows, one
//     warp per row, two-pass mean/variance in fp32 (tolerance-level vs the reference's
//     sequential sums).
#include <cstdint>

#include "kernels.h"
#include "ptx.cuh"

namespace ngk {

namespace {

__device__ __forceinline__ void store_out(void* out, int out_bf16, int64_t idx, float v) {
    if (out_bf16) static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
    else static_cast<float*>(out)[idx] = v;
}

// ---------------------------------------------------------------- v1 gather-reduce
template <bool VEC>
__global__ void __launch_bounds__(256) forward_v1_kernel(FwdArgs a, float scale, float amp) {
    if (*a.err != ~0ull) return;
    const Shape& s = a.s;
    const int D = s.D;
    const int B = s.B;
    const int64_t t = blockIdx.x;
    if (t >= a.T) return;
    const uint32_t tok = a.tokens[t];
    const __nv_bfloat16* e0 = a.e0 + (int64_t)tok * D;
    if (VEC) {
        for (int c = threadIdx.x * 8; c < D; c += blockDim.x * 8) {
            float acc[8];
            const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(e0 + c));
            const uint32_t w0[4] = {v0.x, v0.y, v0.z, v0.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc[2 * i] = bf16_bits_to_f32(w0[i] & 0xffffu);
                acc[2 * i + 1] = bf16_bits_to_f32(w0[i] >> 16);
            }
            for (int b = 0; b < B; ++b) {
                const int32_t row = a.grow[(int64_t)b * a.Tpad + t];
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.sub + (int64_t)row * D + c));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    acc[2 * i] = __fadd_rn(acc[2 * i], bf16_bits_to_f32(w[i] & 0xffffu));
                    acc[2 * i + 1] = __fadd_rn(acc[2 * i + 1], bf16_bits_to_f32(w[i] >> 16));
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float m = __fmul_rn(acc[i], scale);
                if (a.merged_out) store_out(a.merged_out, a.out_bf16, t * D + c + i, m);
                if (a.rows_out && s.amp != kAmpLN) store_out(a.rows_out, a.out_bf16, t * D + c + i, __fmul_rn(m, amp));
            }
        }
    } else {
        for (int c = threadIdx.x; c < D; c += blockDim.x) {
            float acc = __bfloat162float(e0[c]);
            for (int b = 0; b < B; ++b) {
                const int32_t row = a.grow[(int64_t)b * a.Tpad + t];
                acc = __fadd_rn(acc, __bfloat162float(a.sub[(int64_t)row * D + c]));
            }
            const float m = __fmul_rn(acc, scale);
            if (a.merged_out) store_out(a.merged_out, a.out_bf16, t * D + c, m);
            if (a.rows_out && s.amp != kAmpLN) store_out(a.rows_out, a.out_bf16, t * D + c, __fmul_rn(m, amp));
        }
    }
}

// ---------------------------------------------------------------- v2, generic shapes
__global__ void __launch_bounds__(128) forward_v2_simt_kernel(FwdArgs a, float scale, float amp) {
    extern __shared__ float rows[];  // B x d
    if (*a.err != ~0ull) return;
    const Shape& s = a.s;
    const int D = s.D, d = s.d, B = s.B;
    const int64_t t = blockIdx.x;
    if (t >= a.T) return;
    for (int k = threadIdx.x; k < B * d; k += blockDim.x) {
        const int b = k / d, j = k - b * d;
        const int32_t row = a.grow[(int64_t)b * a.Tpad + t];
        rows[k] = __bfloat162float(a.sub[(int64_t)row * d + j]);
    }
    __syncthreads();
    const uint32_t tok = a.tokens[t];
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
        float out = __bfloat162float(a.e0[(int64_t)tok * D + i]);
        const __nv_bfloat16* wrow = a.wcat + (int64_t)i * D;
        for (int b = 0; b < B; ++b) {
            float acc = 0.0f;
            const float* r = rows + b * d;
            for (int j = 0; j < d; ++j) acc = __fadd_rn(acc, __fmul_rn(__bfloat162float(wrow[b * d + j]), r[j]));
            out = __fadd_rn(out, acc);
        }
        const float m = __fmul_rn(out, scale);
        if (a.merged_out) store_out(a.merged_out, a.out_bf16, t * D + i, m);
        if (a.rows_out && s.amp != kAmpLN) store_out(a.rows_out, a.out_bf16, t * D + i, __fmul_rn(m, amp));
    }
}

// ---------------------------------------------------------------- K2 standalone gather
// X[t, b*d : (b+1)*d] = E_b[id_b(t)] (bf16, 16-byte vectors; one warp per (t, b) row group).
// Used when X must be materialised (multi-GPU home buffer) -- the single-GPU forward
// gathers straight into the GEMM's shared memory instead.
__global__ void __launch_bounds__(256) gather_rows_kernel(const int32_t* __restrict__ grow, int64_t Tpad, int64_t T,
                                                          int B, int d, const __nv_bfloat16* __restrict__ sub,
                                                          __nv_bfloat16* __restrict__ X, const unsigned long long* err) {
    if (*err != ~0ull) return;
    constexpr int U = 4;            // independent 16-B loads in flight per thread
    const int vec_per_row = d / 8;  // 16-byte vectors per sub-table row
    const int64_t total = T * B * vec_per_row;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < total; v0 += stride * U) {
        uint4 val[U];
        int64_t dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + u * stride;
            dst[u] = -1;
            if (v < total) {
                const int64_t rowv = v / vec_per_row;
                const int c = (int)(v - rowv * vec_per_row);
                const int64_t t = rowv / B;
                const int b = (int)(rowv - t * B);
                const int32_t row = __ldg(grow + (int64_t)b * Tpad + t);
                // row < 0: not stored on this shard -- a zero row, never an out-of-bounds read
                val[u] = row >= 0 ? __ldg(reinterpret_cast<const uint4*>(sub + (int64_t)row * d) + c)
                                  : make_uint4(0u, 0u, 0u, 0u);
                dst[u] = (t * (int64_t)B * d + (int64_t)b * d) / 8 + c;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (dst[u] >= 0) reinterpret_cast<uint4*>(X)[dst[u]] = val[u];
    }
}

// ---------------------------------------------------------------- LayerNorm amplification
__global__ void __launch_bounds__(256) layernorm_rows_kernel(int D, const float* __restrict__ merged,
                                                             const float* __restrict__ gain,
                                                             const float* __restrict__ bias, void* rows,
                                                             void* merged_copy, int out_bf16, int64_t T,
                                                             const unsigned long long* err) {
    if (*err != ~0ull) return;
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x / 32);
    if (r >= T) return;
    const float* e = merged + r * D;
    float sum = 0.f;
    for (int i = lane; i < D; i += 32) sum += e[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float mean = sum / (float)D;
    float var = 0.f;
    for (int i = lane; i < D; i += 32) {
        const float c = e[i] - mean;
        var += c * c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
    var /= (float)D;
    const float inv_std = 1.0f / sqrtf(var + 1e-5f);
    for (int i = lane; i < D; i += 32) {
        if (rows) store_out(rows, out_bf16, r * D + i, gain[i] * (e[i] - mean) * inv_std + bias[i]);
        if (merged_copy) store_out(merged_copy, out_bf16, r * D + i, e[i]);
    }
}

}  // namespace

void launch_forward_simt(const FwdArgs& a, cudaStream_t st) {
    if (a.T <= 0) return;
    const float scale = 1.0f / (float)a.s.denom;
    const float amp = a.s.amp == kAmpSqrt ? (float)__builtin_sqrt((double)a.s.D) : 1.0f;
    if (a.s.variant == 0) {
        if (a.s.D % 8 == 0)
            forward_v1_kernel<true><<<(unsigned)a.T, 128, 0, st>>>(a, scale, amp);
        else
            forward_v1_kernel<false><<<(unsigned)a.T, 128, 0, st>>>(a, scale, amp);
    } else {
        const size_t smem = sizeof(float) * (size_t)a.s.B * (size_t)a.s.d;
        if (smem > 48 * 1024) cudaFuncSetAttribute(forward_v2_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        forward_v2_simt_kernel<<<(unsigned)a.T, 128, smem, st>>>(a, scale, amp);
    }
    count_launch();
}

void launch_gather_rows(const Shape& s, const int32_t* grow, int64_t Tpad, int64_t T, const __nv_bfloat16* sub,
                        __nv_bfloat16* X, const unsigned long long* err, cudaStream_t st) {
    if (T <= 0) return;
    const int64_t total = T * s.B * (s.d / 8);
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    gather_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(grow, Tpad, T, s.B, s.d, sub, X, err);
    count_launch();
}

namespace {
__global__ void scale_rows_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n, float s) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i] * s;
}
}  // namespace

void launch_scale(const float* in, float* out, int64_t n, float s, cudaStream_t st) {
    if (n <= 0) return;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    scale_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(in, out, n, s);
    count_launch();
}

void launch_layernorm_rows(const Shape& s, const float* merged, const float* gain, const float* bias, void* rows,
                           void* merged_copy, int out_bf16, int64_t T, const unsigned long long* err,
                           cudaStream_t st) {
    if (T <= 0) return;
    const int rows_per_block = 8;
    layernorm_rows_kernel<<<(unsigned)((T + rows_per_block - 1) / rows_per_block), 32 * rows_per_block, 0, st>>>(
        s.D, merged, gain, bias, rows, merged_copy, out_bf16, T, err);
    count_launch();
}

}  // namespace ngk
