// decode.cu -- device-resident sequence_cache state for a batch of decode streams
// (cache.hpp:38-80, cache.cpp:31-96).  The hashing of a decode step / verify block is
// K1 itself (the ring plays the role of prior_context), the projection is K3; these
// kernels only move the ring:
//   * commit: ring <- last N-1 tokens of (ring ++ draft[0..accept)), length += accept,
//     last <- draft[accept-1] -- exactly `accept` sequential appends (cache.cpp:49-55),
//     i.e. the state draft_verify leaves behind (cache.cpp:182-193).  The whole batch is
//     validated first (accept <= L for every stream, no out-of-range token recorded by
//     K1): on any violation no stream changes, as the reference raises before mutating.
//   * reset: seed every ring from a prior context (prefill hand-off) or zeros.
#include <cstdint>

#include <cstdlib>

#include "decodedev.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace ngk {

namespace {

__global__ void __launch_bounds__(1024) commit_kernel(DecodeCommit c, const unsigned long long* err) {
    griddep_wait();  // PDL launch: the preceding kernel (projection / gather) has completed
    decode_commit_block(c, err);
    if (c.err_reported) {
        __syncthreads();  // every thread's reads of the error word are done
        if (threadIdx.x == 0) decode_release_err(c, const_cast<unsigned long long*>(err));
    }
}

__global__ void reset_kernel(int R, uint32_t* __restrict__ ring, uint64_t* __restrict__ length,
                             uint32_t* __restrict__ last, const uint32_t* __restrict__ prior,
                             const uint64_t* __restrict__ lengths, int64_t batch) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= batch) return;
    for (int j = 0; j < R; ++j) ring[s * R + j] = prior ? prior[s * R + j] : 0u;
    length[s] = lengths ? lengths[s] : 0ull;
    last[s] = (prior && R > 0) ? prior[s * R + R - 1] : 0u;
}

// Commit kernels launch with programmatic stream serialization: the launch overlaps the tail
// of the projection before them, griddepcontrol.wait then waits for its completion (so the
// ring is updated only after every kernel that reads it).  NGRAM_PDL=0 launches plainly.
void launch_commit(const DecodeCommit& c, const unsigned long long* err, cudaStream_t st) {
    static const bool pdl = !(getenv("NGRAM_PDL") && atoi(getenv("NGRAM_PDL")) == 0);
    const int threads = c.batch >= 1024 ? 1024 : (int)((c.batch + 31) / 32 * 32);
    if (!pdl) {
        commit_kernel<<<1, threads, 0, st>>>(c, err);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, commit_kernel, c, err);
}

}  // namespace

void launch_decode_commit(const Shape& s, uint32_t* ring, uint64_t* length, uint32_t* last, const uint32_t* draft,
                          int L, const int32_t* accept, int64_t batch, unsigned long long* err,
                          unsigned long long* derr, cudaStream_t st, unsigned long long* err_reported) {
    if (batch <= 0) return;
    DecodeCommit c{s.N > 1 ? s.N - 1 : 0, ring, length, last, draft, L, accept, batch, derr, err_reported, nullptr};
    launch_commit(c, err, st);
    count_launch();
}

void launch_decode_commit_c(const DecodeCommit& c, const unsigned long long* err, cudaStream_t st) {
    if (c.batch <= 0) return;
    launch_commit(c, err, st);
    count_launch();
}

void launch_decode_reset(const Shape& s, uint32_t* ring, uint64_t* length, uint32_t* last, const uint32_t* prior,
                         const uint64_t* lengths, int64_t batch, cudaStream_t st) {
    if (batch <= 0) return;
    const int R = s.N > 1 ? s.N - 1 : 0;
    reset_kernel<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(R, ring, length, last, prior, lengths, batch);
    count_launch();
}

}  // namespace ngk
