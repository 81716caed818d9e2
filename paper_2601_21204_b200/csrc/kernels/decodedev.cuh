// decodedev.cuh -- the decode-state commit as a block-level device routine, shared by
// commit_kernel (decode.cu) and the fused tail of decode_gemm_kernel.
//   ring <- last N-1 tokens of (ring ++ draft[0..accept)), length += accept,
//   last <- draft[accept-1]  ==  `accept` sequential appends (cache.cpp:49-55).
// The whole batch is validated first (accept in [0, L], no out-of-range token recorded by
// K1): on any violation no stream changes, as the reference raises before mutating.
// Must be called by every thread of one block.
#pragma once
#include <cstdint>

#include "kernels.h"

namespace ngk {

__device__ inline void decode_commit_block(const DecodeCommit& c, const unsigned long long* err) {
    int bad = 0;
    for (int64_t s = threadIdx.x; s < c.batch; s += blockDim.x) {
        const int a = c.accept ? c.accept[s] : c.L;
        if (a < 0 || a > c.L) bad = 1;
    }
    bad = __syncthreads_or(bad);
    if (bad) {
        if (threadIdx.x == 0) atomicMin(c.derr, (1ull << 32) | 1ull);  // NGRAM_EINVAL
        return;
    }
    if (*err != ~0ull) return;  // a token of this block was out of range: state unchanged
    const int R = c.R;
    for (int64_t s = threadIdx.x; s < c.batch; s += blockDim.x) {
        const int a = c.accept ? c.accept[s] : c.L;
        if (a == 0) continue;
        uint32_t* rg = c.ring + s * R;
        const uint32_t* dr = c.draft + s * c.L;
        uint32_t nr[kMaxOrder];
        for (int j = 0; j < R; ++j) {  // new ring[j] = element (a + j) of ring ++ draft
            const int k = a + j;
            nr[j] = k < R ? rg[k] : dr[k - R];
        }
        for (int j = 0; j < R; ++j) rg[j] = nr[j];
        c.length[s] += (uint64_t)a;
        c.last[s] = dr[a - 1];
    }
}

// Decode-step tail, run once after every reader of the error word in the chain: a token error
// of this step moves to *c.err_reported, the error word is left clear for the next step.
__device__ inline void decode_release_err(const DecodeCommit& c, unsigned long long* err) {
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(err);
    if (e != ~0ull) atomicMin(c.err_reported, e);
    *err = ~0ull;
}

}  // namespace ngk
