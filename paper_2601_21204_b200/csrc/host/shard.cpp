// shard.cpp -- C-ABI of the row-sharded multi-GPU path: double-buffered
// home X buffers shared over CUDA IPC, K1 over the gathered batch + the fused
// gather/peer-store scatter (kernels/shard.cu), then K3 on the local X.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <vector>

#include "api_util.hpp"
#include "bank.hpp"


using namespace ngh;

struct ngram_shard_group {
    ngram_bank* bank = nullptr;
    int rank = 0, nranks = 1;
    int64_t max_home = 0;
    XBuf x[2];
    __nv_bfloat16* peer[2][64] = {};
    std::vector<void*> ipc_mapped;
    DevBuf<int32_t> grow_all;
    int parity = 0;  // buffer the next scatter writes and the next project reads
    int64_t regime_T = 0;  // size of the gathered batch of the last scatter: the projection's kernel regime
    // NCCL exchange variants (ngram_shard_xchg_*): the prepared step
    DevBuf<uint64_t> ids_all;                 // [all_T][B] global bucket ids of the gathered batch
    DevBuf<int64_t> xtot, xchunk, xcoltot;    // scan scratch
    DevBuf<int64_t> xpref;                    // [1 + nranks][pref_stride] exclusive prefixes
    DevBuf<int64_t> xbounds;                  // [2 * nranks + 1]
    int64_t pref_stride = 0, xchg_T = -1;
    std::vector<int64_t> rank_tok, send_rows, recv_rows;
    ~ngram_shard_group() {
        for (void* p : ipc_mapped) cudaIpcCloseMemHandle(p);
    }
};

extern "C" {

int ngram_shard_group_create(ngram_bank* b, int64_t max_home_tokens, ngram_shard_group** out) {
    NGRAM_API_BEGIN
    if (!b || !out || max_home_tokens < 1) throw Error(NGRAM_EINVAL, "ngram_shard_group_create: bad argument");
    if (!b->tc_path) throw Error(NGRAM_EINVAL, "row-sharded exchange needs the tensor-core shape (d%64, D%128)");
    if (b->shard_count > 64) throw Error(NGRAM_EINVAL, "at most 64 ranks");
    *out = nullptr;
    DeviceGuard dg(b->device);
    auto g = std::make_unique<ngram_shard_group>();
    g->bank = b;
    g->rank = b->shard_rank;
    g->nranks = b->shard_count;
    g->max_home = max_home_tokens;
    for (int i = 0; i < 2; ++i) {
        g->x[i].ensure(round_up(max_home_tokens, kRowPad), b->shape.D);
        g->peer[i][g->rank] = g->x[i].x.p;
    }
    ensure_workspace(b, max_home_tokens);
    *out = g.release();
    NGRAM_API_END
}

int ngram_shard_group_destroy(ngram_shard_group* g) {
    NGRAM_API_BEGIN
    if (g) {
        DeviceGuard dg(g->bank->device);
        delete g;
    }
    NGRAM_API_END
}

int ngram_shard_export(ngram_shard_group* g, void* handle_out) {
    NGRAM_API_BEGIN
    if (!g || !handle_out) throw Error(NGRAM_EINVAL, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    DeviceGuard dg(g->bank->device);
    cudaIpcMemHandle_t h[2];
    for (int i = 0; i < 2; ++i) NGH_CUDA(cudaIpcGetMemHandle(&h[i], g->x[i].x.p));
    std::memcpy(handle_out, h, sizeof(h));
    NGRAM_API_END
}

int ngram_shard_open(ngram_shard_group* g, int peer_rank, const void* handle) {
    NGRAM_API_BEGIN
    if (!g || !handle || peer_rank < 0 || peer_rank >= g->nranks) throw Error(NGRAM_EINVAL, "bad peer");
    if (peer_rank == g->rank) NGRAM_API_RETURN_OK;
    DeviceGuard dg(g->bank->device);
    cudaIpcMemHandle_t h[2];
    std::memcpy(h, handle, sizeof(h));
    for (int i = 0; i < 2; ++i) {
        void* p = nullptr;
        NGH_CUDA(cudaIpcOpenMemHandle(&p, h[i], cudaIpcMemLazyEnablePeerAccess));
        g->ipc_mapped.push_back(p);
        g->peer[i][peer_rank] = static_cast<__nv_bfloat16*>(p);
    }
    NGRAM_API_END
}

int ngram_shard_local_buffers(ngram_shard_group* g, void** x0, void** x1) {
    NGRAM_API_BEGIN
    if (!g || !x0 || !x1) throw Error(NGRAM_EINVAL, "null argument");
    *x0 = g->x[0].x.p;
    *x1 = g->x[1].x.p;
    NGRAM_API_END
}

int ngram_shard_set_peer(ngram_shard_group* g, int peer_rank, void* x0, void* x1) {
    NGRAM_API_BEGIN
    if (!g || !x0 || !x1 || peer_rank < 0 || peer_rank >= g->nranks) throw Error(NGRAM_EINVAL, "bad peer");
    g->peer[0][peer_rank] = static_cast<__nv_bfloat16*>(x0);
    g->peer[1][peer_rank] = static_cast<__nv_bfloat16*>(x1);
    NGRAM_API_END
}

int ngram_shard_scatter_rows(ngram_shard_group* g, const uint32_t* all_tokens, const int64_t* all_seq_offsets,
                             int64_t all_nseq, int64_t all_T, const int64_t* rank_token_offsets,
                             const uint32_t* all_prior, void* stream) {
    NGRAM_API_BEGIN
    if (!g || !all_tokens || !all_seq_offsets || !rank_token_offsets || all_nseq < 1 || all_T < 0)
        throw Error(NGRAM_EINVAL, "ngram_shard_scatter_rows: bad argument");
    if (rank_token_offsets[0] != 0 || rank_token_offsets[g->nranks] != all_T)
        throw Error(NGRAM_EINVAL, "rank_token_offsets must span the gathered batch");
    for (int r = 0; r < g->nranks; ++r) {
        if (rank_token_offsets[r + 1] < rank_token_offsets[r] ||
            rank_token_offsets[r + 1] - rank_token_offsets[r] > g->max_home)
            throw Error(NGRAM_EINVAL, "a rank's home tokens exceed max_home_tokens");
        if (!g->peer[g->parity][r]) throw Error(NGRAM_EINVAL, "peer " + std::to_string(r) + " not opened");
    }
    ngram_bank* b = g->bank;
    DeviceGuard dg(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t Tpad = round_up(std::max<int64_t>(all_T, 1), kRowPad);
    g->grow_all.ensure(size_t(b->shape.B) * size_t(Tpad));
    reset_error_word(b, st);
    g->regime_T = all_T;
    if (all_T == 0) NGRAM_API_RETURN_OK;
    ngk::launch_hash_ids(b->shape, b->ht.p, all_tokens, all_seq_offsets, all_nseq, all_T, all_prior, nullptr, 0,
                         g->grow_all.p, Tpad, b->err.p, st);
    ngk::launch_shard_scatter(b->shape, g->grow_all.p, Tpad, rank_token_offsets, g->nranks, b->sub.p,
                              g->peer[g->parity], all_T, b->err.p, st);
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

// Shared argument checks of the calls that consume the gathered batch.
static void check_gathered(ngram_shard_group* g, const uint32_t* all_tokens, const int64_t* all_seq_offsets,
                           int64_t all_nseq, int64_t all_T, const int64_t* rank_token_offsets, bool peers) {
    if (!g || !all_tokens || !all_seq_offsets || !rank_token_offsets || all_nseq < 1 || all_T < 0)
        throw Error(NGRAM_EINVAL, "sharded exchange: bad argument");
    if (rank_token_offsets[0] != 0 || rank_token_offsets[g->nranks] != all_T)
        throw Error(NGRAM_EINVAL, "rank_token_offsets must span the gathered batch");
    for (int r = 0; r < g->nranks; ++r) {
        if (rank_token_offsets[r + 1] < rank_token_offsets[r] ||
            rank_token_offsets[r + 1] - rank_token_offsets[r] > g->max_home)
            throw Error(NGRAM_EINVAL, "a rank's home tokens exceed max_home_tokens");
        if (peers && !g->peer[g->parity][r]) throw Error(NGRAM_EINVAL, "peer " + std::to_string(r) + " not opened");
    }
}

int ngram_shard_xchg_prepare(ngram_shard_group* g, const uint32_t* all_tokens, const int64_t* all_seq_offsets,
                             int64_t all_nseq, int64_t all_T, const int64_t* rank_token_offsets,
                             const uint32_t* all_prior, int64_t* send_rows, int64_t* recv_rows, void* stream) {
    NGRAM_API_BEGIN
    check_gathered(g, all_tokens, all_seq_offsets, all_nseq, all_T, rank_token_offsets, false);
    if (!send_rows || !recv_rows) throw Error(NGRAM_EINVAL, "ngram_shard_xchg_prepare: null counts");
    ngram_bank* b = g->bank;
    DeviceGuard dg(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int P = g->nranks, B = b->shape.B;
    const int64_t Tpad = round_up(std::max<int64_t>(all_T, 1), kRowPad);
    g->grow_all.ensure(size_t(B) * size_t(Tpad));
    g->ids_all.ensure(size_t(std::max<int64_t>(all_T, 1)) * size_t(B));
    const int64_t nchunks = (all_T + ngk::kXchgChunkTokens - 1) / ngk::kXchgChunkTokens;
    g->xtot.ensure(size_t(std::max<int64_t>(nchunks, 1)) * size_t(P + 1));
    g->xchunk.ensure(size_t(std::max<int64_t>(nchunks, 1)) * size_t(P + 1));
    g->xcoltot.ensure(size_t(P + 1));
    g->pref_stride = std::max<int64_t>(all_T, 1);
    g->xpref.ensure(size_t(g->pref_stride) * size_t(P + 1));
    g->xbounds.ensure(size_t(2 * P + 1));
    g->rank_tok.assign(rank_token_offsets, rank_token_offsets + P + 1);
    g->send_rows.assign(size_t(P), 0);
    g->recv_rows.assign(size_t(P), 0);
    g->xchg_T = all_T;
    reset_error_word(b, st);
    g->regime_T = all_T;
    if (all_T > 0) {
        ngk::launch_hash_ids(b->shape, b->ht.p, all_tokens, all_seq_offsets, all_nseq, all_T, all_prior, g->ids_all.p,
                             1, g->grow_all.p, Tpad, b->err.p, st);
        ngk::launch_xchg_prepare(b->shape, b->cfg.sub_vocab.data(), g->rank, P, rank_token_offsets, all_T,
                                 g->ids_all.p, g->xtot.p, g->xchunk.p, g->xcoltot.p, g->xpref.p, g->pref_stride,
                                 g->xbounds.p, b->err.p, st);
        std::vector<int64_t> bounds(size_t(2 * P + 1));
        NGH_CUDA(cudaMemcpyAsync(bounds.data(), g->xbounds.p, bounds.size() * 8, cudaMemcpyDeviceToHost, st));
        NGH_CUDA(cudaStreamSynchronize(st));
        for (int p = 0; p < P; ++p) {
            g->send_rows[size_t(p)] = bounds[size_t(p + 1)] - bounds[size_t(p)];
            g->recv_rows[size_t(p)] = bounds[size_t(P + 1 + p)];
        }
    }
    std::copy(g->send_rows.begin(), g->send_rows.end(), send_rows);
    std::copy(g->recv_rows.begin(), g->recv_rows.end(), recv_rows);
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_shard_xchg_pack(ngram_shard_group* g, void* send, void* stream) {
    NGRAM_API_BEGIN
    if (!g || g->xchg_T < 0) throw Error(NGRAM_EINVAL, "ngram_shard_xchg_pack: no prepared exchange");
    ngram_bank* b = g->bank;
    int64_t total = 0;
    for (const int64_t n : g->send_rows) total += n;
    if (total > 0 && !send) throw Error(NGRAM_EINVAL, "ngram_shard_xchg_pack: null send buffer");
    DeviceGuard dg(b->device);
    const int64_t Tpad = round_up(std::max<int64_t>(g->xchg_T, 1), kRowPad);
    ngk::launch_xchg_pack(b->shape, b->cfg.sub_vocab.data(), g->rank, g->nranks, g->xchg_T, g->ids_all.p,
                          g->grow_all.p, Tpad, g->xpref.p, b->sub.p, static_cast<__nv_bfloat16*>(send), b->err.p,
                          static_cast<cudaStream_t>(stream));
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_shard_xchg_unpack(ngram_shard_group* g, const void* recv, void* stream) {
    NGRAM_API_BEGIN
    if (!g || g->xchg_T < 0) throw Error(NGRAM_EINVAL, "ngram_shard_xchg_unpack: no prepared exchange");
    int64_t total = 0;
    for (const int64_t n : g->recv_rows) total += n;
    if (total > 0 && !recv) throw Error(NGRAM_EINVAL, "ngram_shard_xchg_unpack: null receive buffer");
    ngram_bank* b = g->bank;
    DeviceGuard dg(b->device);
    ngk::launch_xchg_unpack(b->shape, b->cfg.sub_vocab.data(), g->rank, g->nranks, g->rank_tok.data(), g->ids_all.p,
                            g->xpref.p, g->pref_stride, g->recv_rows.data(),
                            static_cast<const __nv_bfloat16*>(recv), g->x[g->parity].x.p, b->err.p,
                            static_cast<cudaStream_t>(stream));
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_shard_pack_padded(ngram_shard_group* g, const uint32_t* all_tokens, const int64_t* all_seq_offsets,
                            int64_t all_nseq, int64_t all_T, const int64_t* rank_token_offsets,
                            const uint32_t* all_prior, void* send, void* stream) {
    NGRAM_API_BEGIN
    check_gathered(g, all_tokens, all_seq_offsets, all_nseq, all_T, rank_token_offsets, false);
    if (!send) throw Error(NGRAM_EINVAL, "ngram_shard_pack_padded: null send buffer");
    ngram_bank* b = g->bank;
    DeviceGuard dg(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t Tpad = round_up(std::max<int64_t>(all_T, 1), kRowPad);
    g->grow_all.ensure(size_t(b->shape.B) * size_t(Tpad));
    reset_error_word(b, st);
    g->regime_T = all_T;
    if (all_T > 0)
        ngk::launch_hash_ids(b->shape, b->ht.p, all_tokens, all_seq_offsets, all_nseq, all_T, all_prior, nullptr, 0,
                             g->grow_all.p, Tpad, b->err.p, st);
    ngk::launch_xchg_pack_padded(b->shape, g->grow_all.p, Tpad, rank_token_offsets, g->nranks, g->max_home, b->sub.p,
                                 static_cast<__nv_bfloat16*>(send), all_T, b->err.p, st);
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_shard_home_x(ngram_shard_group* g, void** x) {
    NGRAM_API_BEGIN
    if (!g || !x) throw Error(NGRAM_EINVAL, "null argument");
    *x = g->x[g->parity].x.p;
    NGRAM_API_END
}

int ngram_shard_project(ngram_shard_group* g, const uint32_t* home_tokens, int64_t home_T, void* rows_out,
                        void* merged_out, int out_dtype, void* stream) {
    NGRAM_API_BEGIN
    if (!g || home_T < 0 || home_T > g->max_home || (home_T > 0 && !home_tokens))
        throw Error(NGRAM_EINVAL, "ngram_shard_project: bad argument");
    if (out_dtype != NGRAM_F32 && out_dtype != NGRAM_BF16) throw Error(NGRAM_EINVAL, "bad out_dtype");
    ngram_bank* b = g->bank;
    DeviceGuard dg(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    XBuf& xb = g->x[g->parity];
    // The kernel regime (pair GEMM vs split-K, and the split-K sub-regime) follows the GATHERED
    // batch of the preceding scatter, not home_T: the 1-GPU call over the same streams sees that
    // T, so every row is computed with the same K split and summation order (bit-identical).
    const int64_t rT = g->regime_T > 0 ? g->regime_T : home_T;
    run_projection(b, home_tokens, nullptr, round_up(std::max<int64_t>(home_T, 1), kRowPad), home_T, rows_out,
                   merged_out, out_dtype == NGRAM_BF16, b->ws.merged_f32.p, &xb.map, st, -1, nullptr,
                   ngk::small_t_regime(b->shape.D, rT, b->num_sms), nullptr, nullptr, rT);
    g->parity ^= 1;
    NGRAM_API_END
}

}  // extern "C"
