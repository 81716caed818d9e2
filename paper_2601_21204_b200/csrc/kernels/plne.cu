// plne.cu -- elementwise parts of the per-layer N-gram FFN (PLNE, ple.hpp:76-196):
//   forward : Hh = SiLU(U) * G                       (detail::gated_ffn, ple.hpp:85-89)
//   backward: dG = dHh * SiLU(U); dU = dHh * G * SiLU'(U)   (ple.hpp:130-134)
// U = X W_g^T and the two down / gate products are plain fp32 GEMMs (cuBLAS, host side);
// G is the layer bank's merged embedding from the N-gram forward.  Reference op order
// per element (silu(x) = x / (1 + exp(-x)), silu'(x) = s (1 + x (1 - s))).
#include <cstdint>

#include "kernels.h"

namespace ngk {

namespace {

__global__ void silu_gate_kernel(const float* __restrict__ U, const float* __restrict__ G, float* __restrict__ Hh,
                                 int64_t n, const unsigned long long* __restrict__ err) {
    if (*err != ~0ull) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float u = U[i];
        Hh[i] = (u / (1.0f + expf(-u))) * G[i];
    }
}

__global__ void silu_gate_backward_kernel(const float* __restrict__ dHh, const float* __restrict__ U,
                                          const float* __restrict__ G, float* __restrict__ dG,
                                          float* __restrict__ dU, int64_t n,
                                          const unsigned long long* __restrict__ err) {
    if (*err != ~0ull) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float u = U[i];
        const float s = 1.0f / (1.0f + expf(-u));
        const float silu = u / (1.0f + expf(-u));
        dG[i] = dHh[i] * silu;
        dU[i] = dHh[i] * G[i] * (s * (1.0f + u * (1.0f - s)));
    }
}

int grid_of(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

void launch_silu_gate(const float* U, const float* G, float* Hh, int64_t n, const unsigned long long* err,
                      cudaStream_t st) {
    if (n <= 0) return;
    silu_gate_kernel<<<grid_of(n), 256, 0, st>>>(U, G, Hh, n, err);
    count_launch();
}

void launch_silu_gate_backward(const float* dHh, const float* U, const float* G, float* dG, float* dU, int64_t n,
                               const unsigned long long* err, cudaStream_t st) {
    if (n <= 0) return;
    silu_gate_backward_kernel<<<grid_of(n), 256, 0, st>>>(dHh, U, G, dG, dU, n, err);
    count_launch();
}

}  // namespace ngk
