// f64.cu -- the reference's double-precision instantiations on the device: embed_window /
// embed_sequence (embedding.hpp:163-201, 383-436), amplify (:239-287), amplify_backward and
// embed_backward (:291-376), and the gated FFN body of ffn_ple / ffn_plne (ple.hpp:77-146).
// The reference uses them for its finite-difference gradient checks (tests/gradcases.hpp), so
// they follow the reference's operation order in double (no FMA contraction: __dmul_rn /
// __dadd_rn), one small problem per launch.  Tables in the device layout of a bank: sub-tables
// concatenated by branch (storage row = row_base[b] + bucket), projections [B][D][d].
#include <cstdint>

#include "hashdev.cuh"
#include "kernels.h"

namespace ngk {

namespace {

constexpr int kF64Threads = 128;

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// amplify of one row (block-wide; the layer-norm statistics are computed by thread 0 in the
// reference's sequential order)
__device__ void amplify_row(int amp, int D, const double* __restrict__ e, const double* __restrict__ gain,
                            const double* __restrict__ bias, double* __restrict__ out, double* sh) {
    if (amp == kAmpNone) {
        for (int i = threadIdx.x; i < D; i += blockDim.x) out[i] = e[i];
        return;
    }
    if (amp == kAmpSqrt) {
        const double s = sqrt((double)D);
        for (int i = threadIdx.x; i < D; i += blockDim.x) out[i] = dmul(e[i], s);
        return;
    }
    if (threadIdx.x == 0) {
        double mean = 0;
        for (int i = 0; i < D; ++i) mean = dadd(mean, e[i]);
        mean = __ddiv_rn(mean, (double)D);
        double var = 0;
        for (int i = 0; i < D; ++i) {
            const double c = e[i] - mean;
            var = dadd(var, dmul(c, c));
        }
        var = __ddiv_rn(var, (double)D);
        sh[0] = mean;
        sh[1] = __ddiv_rn(1.0, __dsqrt_rn(dadd(var, 1e-5)));
    }
    __syncthreads();
    const double mean = sh[0], inv_std = sh[1];
    for (int i = threadIdx.x; i < D; i += blockDim.x) out[i] = dadd(dmul(dmul(gain[i], e[i] - mean), inv_std), bias[i]);
}

// d(amplify)/d(pre) of one row; layer_norm accumulates the gain / bias gradients
__device__ void amplify_backward_row(int amp, int D, const double* __restrict__ pre, const double* __restrict__ up,
                                     const double* __restrict__ gain, double* __restrict__ d_pre,
                                     double* __restrict__ g_gain, double* __restrict__ g_bias, double* sh) {
    if (amp == kAmpNone) {
        for (int i = threadIdx.x; i < D; i += blockDim.x) d_pre[i] = up[i];
        return;
    }
    if (amp == kAmpSqrt) {
        const double s = sqrt((double)D);
        for (int i = threadIdx.x; i < D; i += blockDim.x) d_pre[i] = dmul(up[i], s);
        return;
    }
    if (threadIdx.x == 0) {
        double mean = 0;
        for (int i = 0; i < D; ++i) mean = dadd(mean, pre[i]);
        mean = __ddiv_rn(mean, (double)D);
        double var = 0;
        for (int i = 0; i < D; ++i) {
            const double c = pre[i] - mean;
            var = dadd(var, dmul(c, c));
        }
        var = __ddiv_rn(var, (double)D);
        const double inv_std = __ddiv_rn(1.0, __dsqrt_rn(dadd(var, 1e-5)));
        double ms = 0, msx = 0;
        for (int i = 0; i < D; ++i) {
            const double xhat = dmul(pre[i] - mean, inv_std);
            const double s = dmul(up[i], gain[i]);
            g_gain[i] = dadd(g_gain[i], dmul(up[i], xhat));
            g_bias[i] = dadd(g_bias[i], up[i]);
            ms = dadd(ms, s);
            msx = dadd(msx, dmul(s, xhat));
        }
        sh[0] = mean;
        sh[1] = inv_std;
        sh[2] = __ddiv_rn(ms, (double)D);
        sh[3] = __ddiv_rn(msx, (double)D);
    }
    __syncthreads();
    const double mean = sh[0], inv_std = sh[1], mean_s = sh[2], mean_sx = sh[3];
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
        const double xhat = dmul(pre[i] - mean, inv_std);
        const double s = dmul(up[i], gain[i]);
        d_pre[i] = dmul(s - mean_s - dmul(xhat, mean_sx), inv_std);
    }
}

// One block per position t of one sequence: window (zero pad / prior), ids, merged row
// (embed_from_ids order: E0 row, then branches in b order, each projected with a sequential
// j sum, then * T(1)/T(denom)), amplified row.
__global__ void __launch_bounds__(kF64Threads) f64_forward_kernel(Shape s, const HashTables* __restrict__ ht,
                                                                  const uint32_t* __restrict__ tokens,
                                                                  const int64_t* __restrict__ off,
                                                                  const uint32_t* __restrict__ prior,
                                                                  const double* __restrict__ base,
                                                                  const double* __restrict__ sub,
                                                                  const double* __restrict__ proj,
                                                                  const double* __restrict__ gain,
                                                                  const double* __restrict__ bias, int amp,
                                                                  double* __restrict__ merged,
                                                                  double* __restrict__ rows) {
    __shared__ int64_t srow[kMaxBranches];
    __shared__ double sh[4];
    const int64_t t = blockIdx.x;
    const int D = s.D, d = s.d;
    uint32_t w[kMaxOrder];
    load_window<kMaxOrder>(s, tokens, off, 1, prior, t, w);
    if (threadIdx.x < s.B) {
        const int b = threadIdx.x;
        srow[b] = __ldg(&ht->row_base[b]) + (int64_t)branch_hash<kMaxOrder>(s, ht, w, b);
    }
    __syncthreads();
    const uint32_t tok = w[s.N - 1];
    double* out = merged + t * D;
    const double scale = __ddiv_rn(1.0, (double)s.denom);
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
        double o = base[(int64_t)tok * D + i];
        for (int b = 0; b < s.B; ++b) {
            const double* row = sub + srow[b] * d;  // v1: d == D
            if (s.variant != 1) {
                o = dadd(o, row[i]);
            } else {
                const double* wr = proj + ((int64_t)b * D + i) * d;
                double acc = 0;
                for (int j = 0; j < d; ++j) acc = dadd(acc, dmul(wr[j], row[j]));
                o = dadd(o, acc);
            }
        }
        out[i] = dmul(o, scale);
    }
    __syncthreads();
    if (rows) amplify_row(amp, D, out, gain, bias, rows + t * D, sh);
}

// One block per position: amplify_backward (unless skip) then embed_backward, accumulated
// into the gradient tables with double atomics (positions may share rows).
__global__ void __launch_bounds__(kF64Threads) f64_backward_kernel(
    Shape s, const HashTables* __restrict__ ht, const uint32_t* __restrict__ tokens, const int64_t* __restrict__ off,
    const uint32_t* __restrict__ prior, const double* __restrict__ sub, const double* __restrict__ proj,
    const double* __restrict__ gain, int amp, const double* __restrict__ merged, const double* __restrict__ upstream,
    double* __restrict__ dpre_ws, double* __restrict__ g_base, double* __restrict__ g_sub,
    double* __restrict__ g_proj, double* __restrict__ g_gain, double* __restrict__ g_bias) {
    __shared__ int64_t srow[kMaxBranches];
    __shared__ double sh[4];
    const int64_t t = blockIdx.x;
    const int D = s.D, d = s.d;
    uint32_t w[kMaxOrder];
    load_window<kMaxOrder>(s, tokens, off, 1, prior, t, w);
    if (threadIdx.x < s.B) {
        const int b = threadIdx.x;
        srow[b] = __ldg(&ht->row_base[b]) + (int64_t)branch_hash<kMaxOrder>(s, ht, w, b);
    }
    double* dp = dpre_ws + t * D;
    if (merged) {
        // LN parameter gradients of this position go to a private (zeroed) pair of rows, then
        // into g_gain / g_bias with atomics (positions run concurrently)
        double* gg = dpre_ws + (int64_t)gridDim.x * D + t * 2 * D;  // [T][2][D]
        amplify_backward_row(amp, D, merged + t * D, upstream + t * D, gain, dp, gg, gg + D, sh);
        __syncthreads();
        if (amp == kAmpLN)
            for (int i = threadIdx.x; i < D; i += blockDim.x) {
                atomicAdd(&g_gain[i], gg[i]);
                atomicAdd(&g_bias[i], gg[D + i]);
            }
    } else {
        for (int i = threadIdx.x; i < D; i += blockDim.x) dp[i] = upstream[t * D + i];
    }
    __syncthreads();
    const uint32_t tok = w[s.N - 1];
    const double scale = __ddiv_rn(1.0, (double)s.denom);
    for (int i = threadIdx.x; i < D; i += blockDim.x) atomicAdd(&g_base[(int64_t)tok * D + i], dmul(scale, dp[i]));
    for (int b = 0; b < s.B; ++b) {
        if (s.variant != 1) {
            for (int i = threadIdx.x; i < D; i += blockDim.x)
                atomicAdd(&g_sub[srow[b] * d + i], dmul(scale, dp[i]));  // v1: d == D
            continue;
        }
        const double* row = sub + srow[b] * d;
        // g_proj[b][i][j] += u_i row[j] (thread per i); g_sub[row][j] += sum_i u_i W[i][j] (thread per j)
        for (int i = threadIdx.x; i < D; i += blockDim.x) {
            const double u = dmul(scale, dp[i]);
            double* gw = g_proj + ((int64_t)b * D + i) * d;
            for (int j = 0; j < d; ++j) atomicAdd(&gw[j], dmul(u, row[j]));
        }
        for (int j = threadIdx.x; j < d; j += blockDim.x) {
            double acc = 0;
            for (int i = 0; i < D; ++i) acc = dadd(acc, dmul(dmul(scale, dp[i]), proj[((int64_t)b * D + i) * d + j]));
            atomicAdd(&g_sub[srow[b] * d + j], acc);
        }
    }
}

__global__ void f64_amplify_kernel(int amp, int D, const double* gain, const double* bias, const double* in,
                                   double* out) {
    __shared__ double sh[4];
    amplify_row(amp, D, in, gain, bias, out, sh);
}

__global__ void f64_amplify_backward_kernel(int amp, int D, const double* pre, const double* up, const double* gain,
                                            double* d_pre, double* g_gain, double* g_bias) {
    __shared__ double sh[4];
    amplify_backward_row(amp, D, pre, up, gain, d_pre, g_gain, g_bias, sh);
}

__device__ __forceinline__ double silu_d(double x) { return __ddiv_rn(x, dadd(1.0, exp(-x))); }
__device__ __forceinline__ double silu_grad_d(double x) {
    const double s = __ddiv_rn(1.0, dadd(1.0, exp(-x)));
    return dmul(s, dadd(1.0, dmul(x, 1.0 - s)));
}

// gated FFN body (ple.hpp:77-101): h = SiLU(W_g x) (.) g, y = W_d h; one block.
__global__ void __launch_bounds__(kF64Threads) f64_gated_ffn_kernel(int Dm, int H, const double* __restrict__ gate,
                                                                    const double* __restrict__ down,
                                                                    const double* __restrict__ x,
                                                                    const double* __restrict__ g, double* h_ws,
                                                                    double* __restrict__ y) {
    for (int r = threadIdx.x; r < H; r += blockDim.x) {
        double acc = 0;
        for (int c = 0; c < Dm; ++c) acc = dadd(acc, dmul(gate[(int64_t)r * Dm + c], x[c]));
        h_ws[r] = dmul(silu_d(acc), g[r]);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < Dm; r += blockDim.x) {
        double acc = 0;
        for (int c = 0; c < H; ++c) acc = dadd(acc, dmul(down[(int64_t)r * H + c], h_ws[c]));
        y[r] = acc;
    }
}

// gated FFN backward (ple.hpp:103-146): accumulates g_gate, g_down, dx; writes dg.
__global__ void __launch_bounds__(kF64Threads) f64_gated_ffn_backward_kernel(
    int Dm, int H, const double* __restrict__ gate, const double* __restrict__ down, const double* __restrict__ x,
    const double* __restrict__ g, const double* __restrict__ up, double* ws /* [3][H] u, s, h + [H] dh */,
    double* __restrict__ g_gate, double* __restrict__ g_down, double* __restrict__ dx, double* __restrict__ dg) {
    double *u = ws, *sv = ws + H, *h = ws + 2 * H, *dh = ws + 3 * H;
    for (int r = threadIdx.x; r < H; r += blockDim.x) {
        double acc = 0;
        for (int c = 0; c < Dm; ++c) acc = dadd(acc, dmul(gate[(int64_t)r * Dm + c], x[c]));
        u[r] = acc;
        sv[r] = silu_d(acc);
        h[r] = dmul(sv[r], g[r]);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < H; c += blockDim.x) {  // dh[c] = sum_r up[r] W_d[r][c]; g_down[r][c] += up[r] h[c]
        double acc = 0;
        for (int r = 0; r < Dm; ++r) {
            g_down[(int64_t)r * H + c] = dadd(g_down[(int64_t)r * H + c], dmul(up[r], h[c]));
            acc = dadd(acc, dmul(up[r], down[(int64_t)r * H + c]));
        }
        dh[c] = acc;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < H; r += blockDim.x) {
        dg[r] = dadd(dg[r], dmul(dh[r], sv[r]));  // accumulated (a table-row gradient or a zeroed vector)
        const double du = dmul(dmul(dh[r], g[r]), silu_grad_d(u[r]));
        for (int c = 0; c < Dm; ++c)
            g_gate[(int64_t)r * Dm + c] = dadd(g_gate[(int64_t)r * Dm + c], dmul(du, x[c]));
        u[r] = du;  // reuse: du per row for the dx sum below
    }
    __syncthreads();
    for (int c = threadIdx.x; c < Dm; c += blockDim.x) {
        double acc = dx[c];
        for (int r = 0; r < H; ++r) acc = dadd(acc, dmul(u[r], gate[(int64_t)r * Dm + c]));
        dx[c] = acc;
    }
}

}  // namespace

void launch_f64_forward(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* off, int64_t T,
                        const uint32_t* prior, const double* base, const double* sub, const double* proj,
                        const double* gain, const double* bias, int amp, double* merged, double* rows,
                        cudaStream_t st) {
    if (T <= 0) return;
    f64_forward_kernel<<<(unsigned)T, kF64Threads, 0, st>>>(s, ht, tokens, off, prior, base, sub, proj, gain, bias,
                                                            amp, merged, rows);
    count_launch();
}

void launch_f64_backward(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* off, int64_t T,
                         const uint32_t* prior, const double* sub, const double* proj, const double* gain, int amp,
                         const double* merged, const double* upstream, double* ws, double* g_base, double* g_sub,
                         double* g_proj, double* g_gain, double* g_bias, cudaStream_t st) {
    if (T <= 0) return;
    f64_backward_kernel<<<(unsigned)T, kF64Threads, 0, st>>>(s, ht, tokens, off, prior, sub, proj, gain, amp, merged,
                                                             upstream, ws, g_base, g_sub, g_proj, g_gain, g_bias);
    count_launch();
}

void launch_f64_amplify(int amp, int D, const double* gain, const double* bias, const double* in, double* out,
                        cudaStream_t st) {
    f64_amplify_kernel<<<1, kF64Threads, 0, st>>>(amp, D, gain, bias, in, out);
    count_launch();
}

void launch_f64_amplify_backward(int amp, int D, const double* pre, const double* up, const double* gain,
                                 double* d_pre, double* g_gain, double* g_bias, cudaStream_t st) {
    f64_amplify_backward_kernel<<<1, kF64Threads, 0, st>>>(amp, D, pre, up, gain, d_pre, g_gain, g_bias);
    count_launch();
}

void launch_f64_gated_ffn(int Dm, int H, const double* gate, const double* down, const double* x, const double* g,
                          double* h_ws, double* y, cudaStream_t st) {
    f64_gated_ffn_kernel<<<1, kF64Threads, 0, st>>>(Dm, H, gate, down, x, g, h_ws, y);
    count_launch();
}

void launch_f64_gated_ffn_backward(int Dm, int H, const double* gate, const double* down, const double* x,
                                   const double* g, const double* up, double* ws, double* g_gate, double* g_down,
                                   double* dx, double* dg, cudaStream_t st) {
    f64_gated_ffn_backward_kernel<<<1, kF64Threads, 0, st>>>(Dm, H, gate, down, x, g, up, ws, g_gate, g_down, dx, dg);
    count_launch();
}

}  // namespace ngk
