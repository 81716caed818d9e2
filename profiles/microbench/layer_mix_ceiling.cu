// Access-pattern ceiling for config B's WHOLE layer (not only its row gather): the exact byte
// mix of one prefill step with the projection taken out.  65 536 tokens; per token 12 random
// 128-byte sub-table rows (out of config B's 4.4 GB of sub-tables), its random 1536-byte E0 row
// (128 000 x 768 bf16) and a 3072-byte fp32 output row:  out[t, c] = E0[tok_t, c] + X[t, c],
// X[t] = the 12 rows concatenated (768 bf16).  Row ids are precomputed (+3 MB of reads the
// fused kernel does not make: it hashes them).  One warp per token, 16-byte loads, 4 tokens in
// flight per warp, fp32 stores evict-first (st.global.cs), L2 flushed before every launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o layer_mix layer_mix_ceiling.cu
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include <cuda_bf16.h>

constexpr int D = 768, B = 12, d = 64, TOK = 4;

__device__ __forceinline__ void st_cs4(float4* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
// volatile and coherent (not .nc, which ptxas may sink below the stores): every load of an
// iteration is issued ahead of its stores (memory-level parallelism)
__device__ __forceinline__ uint4 ld16(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// MODE 0: full mix (rows + E0 read, fp32 written); 1: reads only; 2: writes only
template <int MODE>
__global__ void __launch_bounds__(256) layer_mix(const uint4* __restrict__ sub, const uint4* __restrict__ e0,
                                                 const int* __restrict__ ids, const int* __restrict__ tok,
                                                 int T, float4* __restrict__ out, unsigned* sink) {
    const int lane = threadIdx.x & 31;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    unsigned acc = 0;
    for (int t0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * TOK; t0 < T; t0 += nwarps * TOK) {
        uint4 x[TOK][3], e[TOK][3];
#pragma unroll
        for (int k = 0; k < TOK; ++k) {
            const int t = t0 + k;
            const int tk = MODE == 2 ? 0 : __ldg(tok + t);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int v = c * 32 + lane;  // 16-byte chunk of the 768-column row (96 per row)
                const int b = v >> 3;         // branch: 8 chunks per 128-byte sub-table row
                if (MODE != 2) {
                    x[k][c] = ld16(sub + (int64_t)__ldg(ids + t * B + b) * (d / 8) + (v & 7));
                    e[k][c] = ld16(e0 + (int64_t)tk * (D / 8) + v);
                } else {
                    x[k][c] = make_uint4(t, v, 0, 0);
                    e[k][c] = make_uint4(0, 0, t, v);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < TOK; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int v = c * 32 + lane;
                const uint4 a = x[k][c], q = e[k][c];
                if (MODE == 1) {
                    acc ^= a.x ^ a.w ^ q.y ^ q.z;
                    continue;
                }
                float4* o = out + ((int64_t)(t0 + k) * D + v * 8) / 4;
                st_cs4(o, make_float4(lo(q.x) + lo(a.x), hi(q.x) + hi(a.x), lo(q.y) + lo(a.y), hi(q.y) + hi(a.y)));
                st_cs4(o + 1, make_float4(lo(q.z) + lo(a.z), hi(q.z) + hi(a.z), lo(q.w) + lo(a.w), hi(q.w) + hi(a.w)));
            }
    }
    if (MODE == 1 && acc == 0x12345678u) *sink = acc;
}

int main() {
    const int T = 65536, V0 = 128000;
    const int64_t sub_rows = (4400LL << 20) / 128;
    uint4 *sub, *e0;
    cudaMalloc(&sub, sub_rows * 128);
    cudaMemset(sub, 1, sub_rows * 128);
    cudaMalloc(&e0, (int64_t)V0 * D * 2);
    cudaMemset(e0, 2, (int64_t)V0 * D * 2);
    int *ids, *tok;
    cudaMalloc(&ids, (int64_t)T * B * 4);
    cudaMalloc(&tok, (int64_t)T * 4);
    float4* out;
    cudaMalloc(&out, (int64_t)T * D * 4);
    char* flush;
    cudaMalloc(&flush, 512 << 20);
    unsigned* sink;
    cudaMalloc(&sink, 4);
    std::mt19937_64 g(7);
    std::vector<int> h_ids((size_t)T * B), h_tok(T);
    for (auto& x : h_ids) x = (int)(g() % sub_rows);
    for (auto& x : h_tok) x = (int)(g() % V0);
    cudaMemcpy(ids, h_ids.data(), h_ids.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(tok, h_tok.data(), h_tok.size() * 4, cudaMemcpyHostToDevice);
    const double rd = (double)T * (B * 128 + D * 2), wr = (double)T * D * 4;
    const char* names[3] = {"full mix (rows + E0 in, fp32 out)", "reads only (rows + E0)      ", "writes only (fp32 out)      "};
    for (int grid_mul : {4, 8, 16})
        for (int mode = 0; mode < 3; ++mode) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            float sum = 0;
            const int n = 10;
            for (int i = 0; i < n + 2; ++i) {
                cudaMemsetAsync(flush, i, 512 << 20);
                cudaEventRecord(a);
                const int grid = 148 * grid_mul;
                if (mode == 0) layer_mix<0><<<grid, 256>>>(sub, e0, ids, tok, T, out, sink);
                if (mode == 1) layer_mix<1><<<grid, 256>>>(sub, e0, ids, tok, T, out, sink);
                if (mode == 2) layer_mix<2><<<grid, 256>>>(sub, e0, ids, tok, T, out, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (i >= 2) sum += ms;
            }
            const double us = sum / n * 1e3;
            const double bytes = mode == 0 ? rd + wr : mode == 1 ? rd : wr;
            printf("grid 148x%-2d %s: %6.1f us = %.2f TB/s (%.0f MB)\n", grid_mul, names[mode], us, bytes / (us * 1e-6) / 1e12,
                   bytes / 1e6);
        }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
