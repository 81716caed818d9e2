// decode.cpp -- C-ABI of the incremental decode / speculative-verify path
// (sequence_cache, draft_verify: cache.hpp:38-136, cache.cpp:31-195) over a batch of
// device-resident streams.  No host round trip on the hot calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "api_util.hpp"
#include "bank.hpp"


using namespace ngh;

namespace {

// Hash + project T = batch * L block positions whose windows are ring ++ draft.  With
// `commit`, the state update is fused into the projection when possible; returns whether
// it was (otherwise the caller launches the commit kernel).
constexpr int64_t kReleaseMaxT = 256;  // the small-T (split-K + reduce) regime

bool decode_block(ngram_decode* d, const uint32_t* draft, int L, uint64_t* ids_out, void* merged_out, int out_dtype,
                  cudaStream_t st, const ngk::DecodeCommit* commit = nullptr) {
    ngram_bank* b = d->bank;
    if (b->shard_count != 1)
        throw Error(NGRAM_EINVAL, "decode steps on a row-sharded bank run through the shard group "
                                  "(ngram_shard_scatter_rows with the rings as prior + ngram_shard_project)");
    const int64_t T = d->batch * L;
    const int64_t Tpad = round_up(T, kRowPad);
    // A decode step whose commit runs in the chain's last kernel releases the error word there
    // (DecodeCommit::err_reported): back-to-back steps then need no reset node between them
    // (-1.4 to -1.6 us per step, profiles/README.md).
    const bool release = commit != nullptr && merged_out != nullptr && b->tc_path && T <= kReleaseMaxT;
    // A verify block (no commit here) leaves the word to the ngram_commit that follows it, which
    // releases it; so a verify needs no reset either when the word is known clear.
    const bool verify = commit == nullptr && merged_out != nullptr && ids_out == nullptr;
    if (!((release || verify) && b->err_clean)) reset_error_word(b, st);
    b->err_clean = false;
    ngk::DecodeCommit cr{};
    if (release) {
        cr = *commit;
        cr.err_reported = b->err_rep.p;
        cr.ticket = b->err_ticket.p;
        commit = &cr;
    }
    const int R = b->cfg.max_order - 1;
    const int64_t* off = d->seq_off.p + size_t(L - 1) * size_t(d->batch + 1);
    if (ids_out || !merged_out)
        ngk::launch_hash_ids(b->shape, b->ht.p, draft, off, d->batch, T, R > 0 ? d->ring.p : nullptr, ids_out, 1,
                             nullptr, Tpad, b->err.p, st);
    if (merged_out) {
        const bool fused = forward_tokens(b, draft, off, d->batch, T, R > 0 ? d->ring.p : nullptr, nullptr,
                                          merged_out, out_dtype == NGRAM_BF16, st, 0, &d->xbuf, d->grow.p, true,
                                          commit, L);
        if (release) {
            if (!fused) throw Error(NGRAM_ECUDA, "decode step: commit was not fused into the projection");
            b->err_clean = true;  // the chain's tail cleared the error word
        }
        return fused;
    }
    return false;
}

}  // namespace

extern "C" {

int ngram_decode_create(ngram_bank* b, int64_t batch, int max_draft, ngram_decode** out) {
    NGRAM_API_BEGIN
    if (!b || !out || batch < 1 || max_draft < 1) throw Error(NGRAM_EINVAL, "ngram_decode_create: bad argument");
    *out = nullptr;
    DeviceGuard g(b->device);
    auto d = std::make_unique<ngram_decode>();
    d->bank = b;
    d->batch = batch;
    d->max_draft = max_draft;
    const int R = std::max(b->cfg.max_order - 1, 1);
    d->ring.alloc(size_t(batch) * size_t(R));
    d->length.alloc(size_t(batch));
    d->last.alloc(size_t(batch));
    const int64_t Tmax = batch * max_draft;
    d->grow.alloc(size_t(std::max(b->shape.B, 1)) * size_t(round_up(Tmax, kRowPad)));
    d->derr.alloc(1);
    // per-L sequence offsets {0, L, 2L, ..., batch*L} for L = 1..max_draft
    std::vector<int64_t> off(size_t(max_draft) * size_t(batch + 1));
    for (int L = 1; L <= max_draft; ++L)
        for (int64_t s = 0; s <= batch; ++s) off[size_t(L - 1) * size_t(batch + 1) + size_t(s)] = s * L;
    d->seq_off.alloc(off.size());
    NGH_CUDA(cudaMemcpy(d->seq_off.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemset(d->derr.p, 0xff, 8));
    ngk::launch_decode_reset(b->shape, d->ring.p, d->length.p, d->last.p, nullptr, nullptr, batch, nullptr);
    NGH_CUDA(cudaDeviceSynchronize());
    ensure_workspace(b, Tmax);
    *out = d.release();
    NGRAM_API_END
}

int ngram_decode_destroy(ngram_decode* d) {
    NGRAM_API_BEGIN
    if (d) {
        DeviceGuard g(d->bank->device);
        delete d;
    }
    NGRAM_API_END
}

int ngram_decode_reset(ngram_decode* d, const uint32_t* prior, const uint64_t* lengths, void* stream) {
    NGRAM_API_BEGIN
    if (!d) throw Error(NGRAM_EINVAL, "null decode state");
    DeviceGuard g(d->bank->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ngk::launch_decode_reset(d->bank->shape, d->ring.p, d->length.p, d->last.p, prior, lengths, d->batch, st);
    NGH_CUDA(cudaMemsetAsync(d->derr.p, 0xff, 8, st));
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_decode_step(ngram_decode* d, const uint32_t* tokens, uint64_t* ids_out, void* merged_out, int out_dtype,
                      void* stream) {
    NGRAM_API_BEGIN
    if (!d || !tokens) throw Error(NGRAM_EINVAL, "ngram_decode_step: bad argument");
    if (out_dtype != NGRAM_F32 && out_dtype != NGRAM_BF16) throw Error(NGRAM_EINVAL, "bad out_dtype");
    DeviceGuard g(d->bank->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const ngk::DecodeCommit c{std::max(d->bank->cfg.max_order - 1, 0), d->ring.p, d->length.p, d->last.p,
                              tokens, 1, nullptr, d->batch, d->derr.p};
    if (!decode_block(d, tokens, 1, ids_out, merged_out, out_dtype, st, c.R > 0 ? &c : nullptr))
        ngk::launch_decode_commit(d->bank->shape, d->ring.p, d->length.p, d->last.p, tokens, 1, nullptr, d->batch,
                                  d->bank->err.p, d->derr.p, st);
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_verify_block(ngram_decode* d, const uint32_t* draft, int L, void* merged_out, int out_dtype, void* stream) {
    NGRAM_API_BEGIN
    if (!d || !draft || L < 1 || L > d->max_draft) throw Error(NGRAM_EINVAL, "ngram_verify_block: bad argument");
    if (out_dtype != NGRAM_F32 && out_dtype != NGRAM_BF16) throw Error(NGRAM_EINVAL, "bad out_dtype");
    DeviceGuard g(d->bank->device);
    decode_block(d, draft, L, nullptr, merged_out, out_dtype, static_cast<cudaStream_t>(stream));
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_commit(ngram_decode* d, const uint32_t* draft, int L, const int32_t* accept, void* stream) {
    NGRAM_API_BEGIN
    if (!d || !draft || !accept || L < 1 || L > d->max_draft) throw Error(NGRAM_EINVAL, "ngram_commit: bad argument");
    DeviceGuard g(d->bank->device);
    ngram_bank* b = d->bank;
    ngk::launch_decode_commit(b->shape, d->ring.p, d->length.p, d->last.p, draft, L, accept, d->batch, b->err.p,
                              d->derr.p, static_cast<cudaStream_t>(stream), b->err_rep.p);
    NGH_CUDA(cudaGetLastError());
    b->err_clean = true;  // this commit, the last reader of its verify's error word, released it
    NGRAM_API_END
}

int ngram_decode_ring(ngram_decode* d, uint32_t** ring) {
    NGRAM_API_BEGIN
    if (!d || !ring) throw Error(NGRAM_EINVAL, "ngram_decode_ring: bad argument");
    *ring = d->ring.p;
    NGRAM_API_END
}

int ngram_decode_copy_ring(ngram_decode* d, uint32_t* dst, void* stream) {
    NGRAM_API_BEGIN
    if (!d || !dst) throw Error(NGRAM_EINVAL, "ngram_decode_copy_ring: bad argument");
    DeviceGuard g(d->bank->device);
    const size_t R = size_t(std::max(d->bank->cfg.max_order - 1, 0));
    if (R) NGH_CUDA(cudaMemcpyAsync(dst, d->ring.p, size_t(d->batch) * R * 4, cudaMemcpyDefault,
                                    static_cast<cudaStream_t>(stream)));
    NGRAM_API_END
}

int ngram_decode_get_state(ngram_decode* d, uint32_t* ring, uint64_t* length, uint32_t* last) {
    NGRAM_API_BEGIN
    if (!d) throw Error(NGRAM_EINVAL, "null decode state");
    DeviceGuard g(d->bank->device);
    NGH_CUDA(cudaDeviceSynchronize());
    unsigned long long e = 0;
    NGH_CUDA(cudaMemcpy(&e, d->derr.p, 8, cudaMemcpyDeviceToHost));
    const int R = d->bank->cfg.max_order - 1;
    if (ring && R > 0) NGH_CUDA(cudaMemcpy(ring, d->ring.p, size_t(d->batch) * size_t(R) * 4, cudaMemcpyDeviceToHost));
    if (length) NGH_CUDA(cudaMemcpy(length, d->length.p, size_t(d->batch) * 8, cudaMemcpyDeviceToHost));
    if (last) NGH_CUDA(cudaMemcpy(last, d->last.p, size_t(d->batch) * 4, cudaMemcpyDeviceToHost));
    if (e != ~0ull) {
        NGH_CUDA(cudaMemset(d->derr.p, 0xff, 8));
        throw Error(int(e >> 32), "draft_verify: accept count exceeds draft length");
    }
    NGRAM_API_END
}


int ngram_decode_reset_host(ngram_decode* d, const uint32_t* prior, const uint64_t* lengths) {
    NGRAM_API_BEGIN
    if (!d) throw Error(NGRAM_EINVAL, "null decode state");
    std::lock_guard<std::mutex> host_lock(d->bank->host_mu);
    DeviceGuard g(d->bank->device);
    const int R = std::max(d->bank->cfg.max_order - 1, 0);
    DevBuf<uint32_t> pr;
    DevBuf<uint64_t> le;
    if (prior && R > 0) {
        pr.alloc(size_t(d->batch) * size_t(R));
        NGH_CUDA(cudaMemcpy(pr.p, prior, size_t(d->batch) * size_t(R) * 4, cudaMemcpyHostToDevice));
    }
    if (lengths) {
        le.alloc(size_t(d->batch));
        NGH_CUDA(cudaMemcpy(le.p, lengths, size_t(d->batch) * 8, cudaMemcpyHostToDevice));
    }
    int rc = ngram_decode_reset(d, pr.p, le.p, nullptr);
    if (rc) return rc;
    NGH_CUDA(cudaDeviceSynchronize());
    NGRAM_API_END
}

// Host-buffer path: stage the inputs in pinned memory, enqueue H2D -> step -> D2H of the
// error words and outputs on the state's own stream, one synchronisation, then copy out
// (the caller's buffers are written only on success, as the reference returns by value).
namespace {
struct HostIo {
    ngram_decode* d;
    unsigned long long* words;  // [0] token error, [1] released (reported) error
    unsigned char* ids;
    unsigned char* out;
    unsigned char* in;
};

HostIo host_io(ngram_decode* d, size_t ids_bytes, size_t out_bytes, size_t in_bytes) {
    if (!d->io_stream) NGH_CUDA(cudaStreamCreateWithFlags(&d->io_stream, cudaStreamNonBlocking));
    const size_t a = 16, b = a + round_up(int64_t(ids_bytes), 16), c = b + round_up(int64_t(out_bytes), 16);
    d->io_pin.ensure(c + in_bytes);
    return {d, reinterpret_cast<unsigned long long*>(d->io_pin.p), d->io_pin.p + a, d->io_pin.p + b,
            d->io_pin.p + c};
}

// Enqueue the error-word read, synchronise, and raise a token error like ngram_sync_errors.
void finish_host_io(const HostIo& io) {
    ngram_bank* b = io.d->bank;
    cudaStream_t st = io.d->io_stream;
    NGH_CUDA(cudaStreamSynchronize(st));
    const unsigned long long e = std::min(io.words[0], io.words[1]);
    b->err_clean = true;
    if (e != ~0ull) {
        NGH_CUDA(cudaMemsetAsync(b->err.p, 0xff, 8, st));
        NGH_CUDA(cudaMemsetAsync(b->err_rep.p, 0xff, 8, st));
        NGH_CUDA(cudaStreamSynchronize(st));
        throw Error(NGRAM_ERANGE, "embedding: token out of range for base vocabulary " +
                                      std::to_string(b->cfg.base_vocab) + " (first bad window at position " +
                                      std::to_string(e) + ")");
    }
}

// Page-locked host memory: the device-to-host copy can land in the caller's buffer directly.
bool host_pinned(const void* p) {
    cudaPointerAttributes pa{};
    if (!p || cudaPointerGetAttributes(&pa, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return pa.type == cudaMemoryTypeHost;
}

void read_words(const HostIo& io) {
    ngram_bank* b = io.d->bank;
    NGH_CUDA(cudaMemcpyAsync(&io.words[0], b->err.p, 8, cudaMemcpyDeviceToHost, io.d->io_stream));
    NGH_CUDA(cudaMemcpyAsync(&io.words[1], b->err_rep.p, 8, cudaMemcpyDeviceToHost, io.d->io_stream));
}
}  // namespace

int ngram_decode_set_state_host(ngram_decode* d, const uint32_t* ring, const uint64_t* length, const uint32_t* last) {
    NGRAM_API_BEGIN
    const int rc = ngram_decode_reset_host(d, ring, length);
    if (rc) return rc;
    if (last) {
        DeviceGuard g(d->bank->device);
        NGH_CUDA(cudaMemcpy(d->last.p, last, size_t(d->batch) * 4, cudaMemcpyHostToDevice));
    }
    NGRAM_API_END
}

int ngram_decode_step_host(ngram_decode* d, const uint32_t* tokens, uint64_t* ids_out, float* merged_out) {
    NGRAM_API_BEGIN
    if (!d || !tokens) throw Error(NGRAM_EINVAL, "ngram_decode_step_host: bad argument");
    std::lock_guard<std::mutex> host_lock(d->bank->host_mu);
    DeviceGuard g(d->bank->device);
    ngram_bank* b = d->bank;
    for (int64_t s = 0; s < d->batch; ++s)  // the reference validates before mutating (cache.cpp:39-42)
        if (tokens[s] >= b->cfg.base_vocab)
            throw Error(NGRAM_ERANGE, "sequence_cache: token " + std::to_string(tokens[s]) + " out of range");
    const size_t nb = size_t(std::max(b->shape.B, 0));
    const size_t tok_bytes = size_t(d->batch) * 4;
    const size_t ids_bytes = ids_out ? size_t(d->batch) * nb * 8 : 0;
    const size_t out_bytes = merged_out ? size_t(d->batch) * size_t(b->cfg.dim) * 4 : 0;
    d->io_tok.ensure(size_t(d->batch) * size_t(d->max_draft));
    if (ids_out) d->io_ids.ensure(std::max<size_t>(size_t(d->batch) * nb, 1));
    if (merged_out) d->io_out.ensure(size_t(d->batch) * size_t(d->max_draft) * size_t(b->cfg.dim));
    const HostIo io = host_io(d, ids_bytes, out_bytes, tok_bytes);
    cudaStream_t st = d->io_stream;
    std::memcpy(io.in, tokens, tok_bytes);
    // a pinned output buffer receives the copy directly (no staging memcpy of batch x D floats)
    unsigned char* out_dst = (out_bytes && host_pinned(merged_out)) ? reinterpret_cast<unsigned char*>(merged_out)
                                                                       : io.out;
    auto enqueue = [&]() {
        NGH_CUDA(cudaMemcpyAsync(d->io_tok.p, io.in, tok_bytes, cudaMemcpyHostToDevice, st));
        int rc = ngram_decode_step(d, d->io_tok.p, ids_out ? d->io_ids.p : nullptr,
                                   merged_out ? d->io_out.p : nullptr, NGRAM_F32, st);
        if (rc) return rc;
        read_words(io);
        if (ids_bytes) NGH_CUDA(cudaMemcpyAsync(io.ids, d->io_ids.p, ids_bytes, cudaMemcpyDeviceToHost, st));
        if (out_bytes) NGH_CUDA(cudaMemcpyAsync(out_dst, d->io_out.p, out_bytes, cudaMemcpyDeviceToHost, st));
        return 0;
    };
    // Steady state (the error word clean after the previous step): replay the captured sequence
    // -- the same copies and kernels, one graph launch instead of ~8 API calls.  The first call,
    // a different output variant or a moved buffer re-captures; a larger batch runs eagerly.
    // The graph holds raw pointers: it is re-captured whenever a buffer it uses was reallocated
    // (a workspace grown by another call), and only after one eager step has sized them all.
    const bool graphable = (merged_out || ids_out) && d->batch <= 256 && b->err_clean && d->host_steps > 0 &&
                           !(getenv("NGRAM_HOST_STEP_GRAPH") && atoi(getenv("NGRAM_HOST_STEP_GRAPH")) == 0);
    const void* key[9] = {io.in, out_dst, io.ids, d->io_tok.p, d->io_out.p, d->io_ids.p, d->xbuf.x.p,
                          b->ws.splitk.p,
                          reinterpret_cast<const void*>(uintptr_t((ids_out ? 1 : 0) | (merged_out ? 2 : 0)))};
    if (graphable && d->step_exec && !std::equal(key, key + 9, d->step_key)) {
        cudaGraphExecDestroy(d->step_exec);
        d->step_exec = nullptr;
    }
    if (graphable && !d->step_exec) {
        const uint64_t l0 = ngk::launches();
        cudaGraph_t graph = nullptr;
        NGH_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        const int rc = enqueue();
        const cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        NGH_CUDA(ce);
        const cudaError_t ie = cudaGraphInstantiate(&d->step_exec, graph, 0);
        cudaGraphDestroy(graph);
        NGH_CUDA(ie);
        std::copy(key, key + 9, d->step_key);
        d->step_launches = ngk::launches() - l0;
    }
    if (graphable) {
        NGH_CUDA(cudaGraphLaunch(d->step_exec, st));
        ngk::count_launch(int(d->step_launches));
    } else {
        const int rc = enqueue();
        if (rc) return rc;
        ++d->host_steps;
    }
    finish_host_io(io);
    if (ids_bytes) std::memcpy(ids_out, io.ids, ids_bytes);
    if (out_bytes && out_dst == io.out) std::memcpy(merged_out, io.out, out_bytes);
    NGRAM_API_END
}

int ngram_verify_commit_host(ngram_decode* d, const uint32_t* draft, int L, const int32_t* accept,
                             float* merged_out) {
    NGRAM_API_BEGIN
    if (!d || !draft || !accept || L < 1 || L > d->max_draft)
        throw Error(NGRAM_EINVAL, "ngram_verify_commit_host: bad argument");
    std::lock_guard<std::mutex> host_lock(d->bank->host_mu);
    ngram_bank* b = d->bank;
    for (int64_t s = 0; s < d->batch; ++s) {
        if (accept[s] < 0 || accept[s] > L) throw Error(NGRAM_EINVAL, "draft_verify: accept count exceeds draft length");
        for (int i = 0; i < L; ++i)
            if (draft[s * L + i] >= b->cfg.base_vocab)
                throw Error(NGRAM_ERANGE, "sequence_cache: token " + std::to_string(draft[s * L + i]) + " out of range");
    }
    DeviceGuard g(b->device);
    const size_t dr_bytes = size_t(d->batch) * size_t(L) * 4, ac_bytes = size_t(d->batch) * 4;
    const size_t out_bytes = merged_out ? size_t(d->batch) * size_t(L) * size_t(b->cfg.dim) * 4 : 0;
    d->io_tok.ensure(size_t(d->batch) * size_t(d->max_draft));
    d->io_acc.ensure(size_t(d->batch));
    d->io_out.ensure(size_t(d->batch) * size_t(d->max_draft) * size_t(b->cfg.dim));
    const HostIo io = host_io(d, 0, out_bytes, dr_bytes + ac_bytes);
    cudaStream_t st = d->io_stream;
    std::memcpy(io.in, draft, dr_bytes);
    std::memcpy(io.in + dr_bytes, accept, ac_bytes);
    NGH_CUDA(cudaMemcpyAsync(d->io_tok.p, io.in, dr_bytes, cudaMemcpyHostToDevice, st));
    NGH_CUDA(cudaMemcpyAsync(d->io_acc.p, io.in + dr_bytes, ac_bytes, cudaMemcpyHostToDevice, st));
    int rc = ngram_verify_block(d, d->io_tok.p, L, d->io_out.p, NGRAM_F32, st);
    if (rc) return rc;
    rc = ngram_commit(d, d->io_tok.p, L, d->io_acc.p, st);
    if (rc) return rc;
    read_words(io);
    unsigned char* out_dst = (out_bytes && host_pinned(merged_out)) ? reinterpret_cast<unsigned char*>(merged_out)
                                                                       : io.out;
    if (out_bytes) NGH_CUDA(cudaMemcpyAsync(out_dst, d->io_out.p, out_bytes, cudaMemcpyDeviceToHost, st));
    finish_host_io(io);
    if (out_bytes && out_dst == io.out) std::memcpy(merged_out, io.out, out_bytes);
    NGRAM_API_END
}

}  // extern "C"

