// bank.cu -- device-side bank construction: the counter-based synthetic generator for
// LongCat-scale tables (defined in oracle/ngram_oracle.c, evaluated identically here), f32 -> bf16 conversion of uploaded reference banks,
// and W_b -> W_cat packing.  Pure HBM-write kernels, grid-stride, 16-byte stores.
#include <atomic>
#include <cstdint>

#include "kernels.h"
#include "ptx.cuh"

namespace ngk {

namespace {
std::atomic<uint64_t> g_launches{0};
}  // namespace

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
uint64_t launches() { return g_launches.load(std::memory_order_relaxed); }

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// Identical definition to oracle/ngram_oracle.c:or_synth_value (integer sum of four
// 16-bit uniforms, one exactly-rounded float multiply, RNE to bf16).
__device__ __forceinline__ uint16_t synth_bits(uint64_t key, uint64_t row, uint32_t col, float scale) {
    const uint64_t h = splitmix64(key + row * 65536ULL + (uint64_t)col);
    const int32_t sm =
        (int32_t)((h & 0xffffu) + ((h >> 16) & 0xffffu) + ((h >> 32) & 0xffffu) + ((h >> 48) & 0xffffu));
    const float v = __fmul_rn((float)(sm - 131070), scale);
    const uint32_t u = __float_as_uint(v);
    return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

__global__ void synth_fill_kernel(__nv_bfloat16* __restrict__ dst, uint64_t key, int64_t row0, int64_t nrows,
                                  int ncols, int64_t pitch, float scale) {
    // each thread writes 8 consecutive columns (16 B) of one row; ncols % 8 == 0 here
    const int64_t vec_per_row = ncols / 8;
    const int64_t total = nrows * vec_per_row;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = v / vec_per_row;
        const int c0 = (int)(v - r * vec_per_row) * 8;
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t lo = synth_bits(key, (uint64_t)(row0 + r), (uint32_t)(c0 + 2 * i), scale);
            const uint32_t hi = synth_bits(key, (uint64_t)(row0 + r), (uint32_t)(c0 + 2 * i + 1), scale);
            w[i] = lo | (hi << 16);
        }
        *reinterpret_cast<uint4*>(dst + r * pitch + c0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

__global__ void synth_fill_scalar_kernel(__nv_bfloat16* __restrict__ dst, uint64_t key, int64_t row0, int64_t nrows,
                                         int ncols, int64_t pitch, float scale) {
    const int64_t total = nrows * ncols;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = v / ncols;
        const int c = (int)(v - r * ncols);
        const uint16_t bits = synth_bits(key, (uint64_t)(row0 + r), (uint32_t)c, scale);
        reinterpret_cast<uint16_t*>(dst)[r * pitch + c] = bits;
    }
}

__global__ void synth_wcat_kernel(__nv_bfloat16* __restrict__ wcat, uint64_t seed, int D, int d, int B, float scale) {
    const int64_t total = (int64_t)D * D;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = v / D;
        const int k = (int)(v - i * D);
        const int b = k / d, j = k - b * d;
        const uint64_t key = splitmix64(seed ^ ((uint64_t)(100 + b) * 0xd1342543de82ef95ULL));
        reinterpret_cast<uint16_t*>(wcat)[v] = synth_bits(key, (uint64_t)i, (uint32_t)j, scale);
    }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __float2bfloat16_rn(src[i]);
}

__global__ void pack_wcat_kernel(const float* __restrict__ proj, __nv_bfloat16* __restrict__ wcat, int D, int d,
                                 int b) {
    const int64_t total = (int64_t)D * d;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = v / d;
        const int j = (int)(v - i * d);
        wcat[i * D + (int64_t)b * d + j] = __float2bfloat16_rn(proj[v]);
    }
}

__global__ void fill_f32_kernel(float* dst, float v, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = v;
}

inline unsigned grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b > 148 * 32) b = 148 * 32;
    if (b < 1) b = 1;
    return (unsigned)b;
}

uint64_t table_key(uint64_t seed, uint32_t table) {
    uint64_t x = seed ^ ((uint64_t)table * 0xd1342543de82ef95ULL);
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

}  // namespace

void launch_synth_fill_bf16(__nv_bfloat16* dst, uint64_t seed, uint32_t table, int64_t row0, int64_t nrows, int ncols,
                            int64_t pitch, float scale, cudaStream_t st) {
    if (nrows <= 0) return;
    const uint64_t key = table_key(seed, table);
    if (ncols % 8 == 0 && pitch % 8 == 0)
        synth_fill_kernel<<<grid_for(nrows * (ncols / 8), 256), 256, 0, st>>>(dst, key, row0, nrows, ncols, pitch,
                                                                              scale);
    else
        synth_fill_scalar_kernel<<<grid_for(nrows * ncols, 256), 256, 0, st>>>(dst, key, row0, nrows, ncols, pitch,
                                                                               scale);
    count_launch();
}

void launch_synth_wcat(__nv_bfloat16* wcat, uint64_t seed, int D, int d, int B, float scale, cudaStream_t st) {
    synth_wcat_kernel<<<grid_for((int64_t)D * D, 256), 256, 0, st>>>(wcat, seed, D, d, B, scale);
    count_launch();
}

void launch_f32_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    f32_to_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(src, dst, n);
    count_launch();
}

void launch_pack_wcat(const float* proj_b, __nv_bfloat16* wcat, int D, int d, int b, cudaStream_t st) {
    pack_wcat_kernel<<<grid_for((int64_t)D * d, 256), 256, 0, st>>>(proj_b, wcat, D, d, b);
    count_launch();
}

void launch_fill_f32(float* dst, float v, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    fill_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(dst, v, n);
    count_launch();
}

}  // namespace ngk
