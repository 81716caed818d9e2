// Access-pattern ceiling for config B's row gather: random 128-byte rows out of a large table,
// 16-byte loads (U in flight per thread, shifts only); 100 MB gathered per launch (config B's
// sub-table bytes per step).  (a) copy into a contiguous X (the K2 pattern), (b) read-only.
// Table 4.4 GB (config B's sub-tables) vs 128 MB; row widths 128 / 512 B; random vs sorted rows.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
template <int U, bool WRITE>
__global__ void gather(const uint4* __restrict__ tab, const int* __restrict__ rows, int lvpr, int nvec,
                       uint4* __restrict__ out, unsigned* sink) {
    unsigned acc = 0;
    const int stride = gridDim.x * blockDim.x;
    for (int v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < nvec; v0 += stride * U) {
        uint4 val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int v = v0 + u * stride;
            if (v < nvec) val[u] = __ldg(tab + ((long)__ldg(rows + (v >> lvpr)) << lvpr) + (v & ((1 << lvpr) - 1)));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int v = v0 + u * stride;
            if (v < nvec) { if (WRITE) out[v] = val[u]; else acc ^= val[u].x ^ val[u].w; }
        }
    }
    if (!WRITE && acc == 0x12345678u) *sink = acc;
}
int main() {
    const long big = 4400L << 20;
    uint4* tab; cudaMalloc(&tab, big); cudaMemset(tab, 1, big);
    char* flush; cudaMalloc(&flush, 512 << 20);
    unsigned* sink; cudaMalloc(&sink, 4);
    const long total = 100L << 20;
    uint4* out; cudaMalloc(&out, total);
    int* rows; cudaMalloc(&rows, (total / 128) * 4);
    for (long tb : {big, 128L << 20}) for (int rowb : {128, 512}) for (int sorted = 0; sorted < 2; ++sorted) {
        const long nrows_tab = tb / rowb, nrows = total / rowb;
        std::vector<int> h(nrows); std::mt19937_64 g(1);
        for (auto& x : h) x = (int)(g() % nrows_tab);
        if (sorted) std::sort(h.begin(), h.end());
        cudaMemcpy(rows, h.data(), nrows * 4, cudaMemcpyHostToDevice);
        const int lvpr = rowb == 128 ? 3 : 5; const int nvec = (int)(total / 16);
        for (int w = 0; w < 2; ++w) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            float sum = 0; int n = 10;
            for (int i = 0; i < n + 2; ++i) {
                cudaMemsetAsync(flush, i, 512 << 20);
                cudaEventRecord(a);
                if (w) gather<8, true><<<148 * 8, 256>>>(tab, rows, lvpr, nvec, out, sink);
                else gather<8, false><<<148 * 8, 256>>>(tab, rows, lvpr, nvec, out, sink);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (i >= 2) sum += ms;
            }
            const double bytes = total * (w ? 2.0 : 1.0);
            printf("table %5ld MB row %3d B %s %s: %6.1f us = %.2f TB/s (%s)\n", tb >> 20, rowb, sorted ? "sorted" : "random",
                   w ? "gather+store" : "gather-only ", sum / n * 1e3, bytes / (sum / n * 1e-3) / 1e12, w ? "read+write" : "read");
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
