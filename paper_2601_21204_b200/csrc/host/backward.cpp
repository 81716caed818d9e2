// backward.cpp -- C-ABI of the training-side gradient:
// embed_sequence_backward (embedding.hpp:438-459) over a batch of sequences on the device.
//
//   K1        storage rows of every (position, branch) (hash_ids_kernel, validates tokens)
//   amp_bwd   U = fp32(1/denom) * amplify_backward(merged, upstream); g_E0[tok] += U;
//             layer_norm: g_gain / g_bias                               (backward.cu)
//   v2:  X    = gathered sub-table rows (f32)                           (backward.cu)
//        g_W += U^T X            D x D x T   tcgen05 (gemm_gen.cu), U in bf16 split terms
//        dX   = U W_cat          T x D x D   tcgen05 (gemm_gen.cu), U in bf16 split terms
//        (pedantic mode / CUDA-core-shaped banks: the fp32 CUDA-core GEMM of gemm_gen.cu)
//        g_sub[row_b(t)] += dX[t, b]                                    (backward.cu)
//   v1:  g_sub[row_b(t)] += U[t]                                        (backward.cu)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "api_util.hpp"
#include "bank.hpp"
#include "gemm.hpp"

using namespace ngh;

struct ngram_grad {
    ngram_bank* bank = nullptr;
    DevBuf<float> e0, sub, w, gain, bias;  // gradients, device layout
    DevBuf<float> U, X, dX, wf;            // workspaces
    DevBuf<__nv_bfloat16> X16, Ub;         // bf16x3 mode: bf16 X and the three bf16 terms of U
    int gemm_mode = 0;                     // 0 split-bf16 (default), 1 single-term bf16, 2 pedantic fp32
    int terms = 2;                         // bf16 terms of U in mode 0 (NGRAM_GRAD_EXACT: 3)
    DevBuf<int32_t> grow;
    int64_t cap = 0;
    bool sparse = false;                 // NGRAM_GRAD_SPARSE_ROWS
    DevBuf<int32_t> sp_rows;             // [sp_cap] storage rows
    DevBuf<float> sp_vals;               // [sp_cap][d]
    int64_t sp_count = 0, sp_cap = 0;
    bool sparse_base = false;            // NGRAM_GRAD_SPARSE_BASE
    DevBuf<int32_t> sb_tok;              // [sb_cap] tokens
    DevBuf<float> sb_vals;               // [sb_cap][D] merged-row gradients u
    int64_t sb_count = 0, sb_cap = 0;
    bool e0_dense_stale = false;         // sparse base: g->e0 must be rebuilt from the pairs
    DevBuf<uint32_t> h_tokens, h_prior;  // host-buffer entry staging
    DevBuf<int64_t> h_off;
    DevBuf<float> h_merged, h_up;
};

namespace ngh {
ngram_bank* grad_bank(ngram_grad* g) { return g->bank; }
}  // namespace ngh

namespace {

void zero_all(ngram_grad* g, cudaStream_t st) {
    for (DevBuf<float>* b : {&g->e0, &g->sub, &g->w, &g->gain, &g->bias})
        if (b->n && !(b == &g->e0 && g->sparse_base))  // a sparse base is rebuilt from its pairs on request
            NGH_CUDA(cudaMemsetAsync(b->p, 0, b->n * sizeof(float), st));
    g->sp_count = 0;
    g->sb_count = 0;
    g->e0_dense_stale = g->sparse_base;
}

// sparse base-table gradient: room for `more` (token, D-wide row) pairs, keeping the held ones
void base_reserve(ngram_grad* g, int64_t more, int D, cudaStream_t st) {
    const int64_t need = g->sb_count + more;
    if (need <= g->sb_cap) return;
    const int64_t cap = std::max<int64_t>(need, g->sb_cap * 2);
    DevBuf<int32_t> r;
    DevBuf<float> v;
    r.alloc(size_t(cap));
    v.alloc(size_t(cap) * size_t(D));
    if (g->sb_count) {
        NGH_CUDA(cudaMemcpyAsync(r.p, g->sb_tok.p, size_t(g->sb_count) * 4, cudaMemcpyDeviceToDevice, st));
        NGH_CUDA(cudaMemcpyAsync(v.p, g->sb_vals.p, size_t(g->sb_count) * size_t(D) * 4, cudaMemcpyDeviceToDevice, st));
        NGH_CUDA(cudaStreamSynchronize(st));
    }
    std::swap(g->sb_tok.p, r.p);
    std::swap(g->sb_tok.n, r.n);
    std::swap(g->sb_vals.p, v.p);
    std::swap(g->sb_vals.n, v.n);
    g->sb_cap = cap;
}

// sparse base: rebuild the dense E0 gradient from the pairs (ngram_grad_tensor(0) / download)
void densify_base(ngram_grad* g, cudaStream_t st) {
    if (!g->sparse_base || !g->e0_dense_stale) return;
    const size_t n = size_t(g->bank->cfg.base_vocab) * size_t(g->bank->shape.D);
    if (g->e0.n != n) g->e0.alloc(n);
    NGH_CUDA(cudaMemsetAsync(g->e0.p, 0, n * sizeof(float), st));
    ngk::launch_coo_densify(g->sb_tok.p, g->sb_vals.p, g->sb_count, g->bank->shape.D, g->e0.p, st);
    NGH_CUDA(cudaGetLastError());
    g->e0_dense_stale = false;
}

// Make room for `more` sparse (row, gradient row) pairs, preserving the ones already held.
void sparse_reserve(ngram_grad* g, int64_t more, int d, cudaStream_t st) {
    const int64_t need = g->sp_count + more;
    if (need <= g->sp_cap) return;
    const int64_t cap = std::max<int64_t>(need, g->sp_cap * 2);
    DevBuf<int32_t> r;
    DevBuf<float> v;
    r.alloc(size_t(cap));
    v.alloc(size_t(cap) * size_t(d));
    if (g->sp_count) {
        NGH_CUDA(cudaMemcpyAsync(r.p, g->sp_rows.p, size_t(g->sp_count) * 4, cudaMemcpyDeviceToDevice, st));
        NGH_CUDA(cudaMemcpyAsync(v.p, g->sp_vals.p, size_t(g->sp_count) * size_t(d) * 4, cudaMemcpyDeviceToDevice, st));
        NGH_CUDA(cudaStreamSynchronize(st));
    }
    std::swap(g->sp_rows.p, r.p);
    std::swap(g->sp_rows.n, r.n);
    std::swap(g->sp_vals.p, v.p);
    std::swap(g->sp_vals.n, v.n);
    g->sp_cap = cap;
}

}  // namespace

extern "C" {

int ngram_grad_create(ngram_bank* b, ngram_grad** out) { return ngram_grad_create_ex(b, 0, out); }

int ngram_grad_create_ex(ngram_bank* b, int flags, ngram_grad** out) {
    NGRAM_API_BEGIN
    if (!b || !out ||
        (flags & ~(NGRAM_GRAD_SPARSE_ROWS | NGRAM_GRAD_TF32 | NGRAM_GRAD_PEDANTIC | NGRAM_GRAD_EXACT |
                   NGRAM_GRAD_SPARSE_BASE)) ||
        __builtin_popcount(unsigned(flags & (NGRAM_GRAD_TF32 | NGRAM_GRAD_PEDANTIC | NGRAM_GRAD_EXACT))) > 1)
        throw Error(NGRAM_EINVAL, "ngram_grad_create: bad argument");
    if (b->hash_only) throw Error(NGRAM_EINVAL, "bank was created hash-only (NGRAM_BANK_HASH_ONLY)");
    if (b->shard_count != 1) throw Error(NGRAM_EINVAL, "ngram_grad_create: row-sharded banks are not supported");
    DeviceGuard dg(b->device);
    auto g = std::make_unique<ngram_grad>();
    g->bank = b;
    const auto& s = b->shape;
    g->sparse = (flags & NGRAM_GRAD_SPARSE_ROWS) != 0;
    g->sparse_base = (flags & NGRAM_GRAD_SPARSE_BASE) != 0;
    if (!g->sparse_base) g->e0.alloc(size_t(b->cfg.base_vocab) * size_t(s.D));  // else densified on request
    if (!g->sparse) g->sub.alloc(size_t(b->local_rows) * size_t(s.d));
    if (s.variant == 1 && s.B > 0) g->w.alloc(size_t(s.D) * size_t(s.D));
    if (s.amp == ngk::kAmpLN) {
        g->gain.alloc(size_t(s.D));
        g->bias.alloc(size_t(s.D));
    }
    // 0: U in bf16 split terms on the tensor cores (tensor-core banks: X and W_cat are bf16) --
    //    two by default, three with NGRAM_GRAD_EXACT; 1 (NGRAM_GRAD_TF32): one bf16 term;
    // 2: the fp32 CUDA-core GEMM (pedantic; also every CUDA-core-shaped bank)
    g->gemm_mode = ((flags & NGRAM_GRAD_PEDANTIC) || !b->tc_path) ? 2 : (flags & NGRAM_GRAD_TF32) ? 1 : 0;
    g->terms = g->gemm_mode == 1 ? 1 : (flags & NGRAM_GRAD_EXACT) ? 3 : 2;
    zero_all(g.get(), nullptr);
    NGH_CUDA(cudaDeviceSynchronize());
    *out = g.release();
    NGRAM_API_END
}

int ngram_grad_destroy(ngram_grad* g) {
    NGRAM_API_BEGIN
    if (g) {
        DeviceGuard dg(g->bank->device);
        delete g;
    }
    NGRAM_API_END
}

int ngram_grad_zero(ngram_grad* g, void* stream) {
    NGRAM_API_BEGIN
    if (!g) throw Error(NGRAM_EINVAL, "null gradient bank");
    DeviceGuard dg(g->bank->device);
    zero_all(g, static_cast<cudaStream_t>(stream));
    NGRAM_API_END
}

int ngram_embed_backward(ngram_grad* g, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                         int64_t T, const uint32_t* prior, const float* merged, const float* upstream, int flags,
                         void* stream) {
    NGRAM_API_BEGIN
    if (!g || nseq < 1 || T < 0 || !seq_offsets || (T > 0 && (!tokens || !upstream)))
        throw Error(NGRAM_EINVAL, "ngram_embed_backward: bad argument");
    ngram_bank* b = g->bank;
    const auto& s = b->shape;
    const int amp = (flags & NGRAM_BWD_SKIP_AMPLIFY) ? ngk::kAmpNone : s.amp;
    if (amp == ngk::kAmpLN && T > 0 && !merged)
        throw Error(NGRAM_EINVAL, "ngram_embed_backward: layer_norm needs the pre-amplification rows (merged)");
    DeviceGuard dg(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    reset_error_word(b, st);
    if (T == 0) return NGRAM_OK;
    const int64_t Tpad = round_up(T, kRowPad);
    const int D = s.D, B = s.B, d = s.d;
    const bool tc_terms = B > 0 && s.variant == 1 && g->gemm_mode != 2;  // u goes out as bf16 terms only
    if (T > g->cap) {
        if (!tc_terms) g->U.alloc(size_t(Tpad) * size_t(D));
        if (s.variant == 1 && B > 0) {
            if (g->gemm_mode == 2) g->X.alloc(size_t(Tpad) * size_t(D));  // fp32 X: pedantic GEMMs only
            if (!(tc_terms && g->sparse)) g->dX.alloc(size_t(Tpad) * size_t(D));  // sparse: straight to COO
        }
        g->grow.alloc(size_t(std::max(B, 1)) * size_t(Tpad));
        g->cap = Tpad;
    }
    // K1: storage rows (and token validation: a bad token leaves every gradient untouched)
    ngk::launch_hash_ids(s, b->ht.p, tokens, seq_offsets, nseq, T, prior, nullptr, 0, g->grow.p, g->cap, b->err.p, st);
    const size_t n_td = size_t(T) * size_t(D);
    if (tc_terms) g->Ub.ensure(size_t(g->terms) * n_td);
    float* u_rows = tc_terms ? nullptr : g->U.p;
    if (g->sparse_base) {  // the E0 gradient is the (token, u) pairs: u lands in the COO values directly
        base_reserve(g, T, D, st);
        float* vals = g->sb_vals.p + size_t(g->sb_count) * size_t(D);
        if (u_rows) {  // v1 / pedantic paths read U later: keep writing it, then copy to the pairs
        } else {
            u_rows = vals;
        }
        NGH_CUDA(cudaMemcpyAsync(g->sb_tok.p + g->sb_count, tokens, size_t(T) * 4, cudaMemcpyDeviceToDevice, st));
    }
    ngk::launch_amp_backward(s, upstream, merged, tokens, T, amp, b->ln_gain.p, u_rows,
                             g->sparse_base ? nullptr : g->e0.p, g->gain.p, g->bias.p, b->err.p, st,
                             tc_terms ? g->Ub.p : nullptr, g->terms, int64_t(n_td));
    if (g->sparse_base) {
        float* vals = g->sb_vals.p + size_t(g->sb_count) * size_t(D);
        if (u_rows != vals) NGH_CUDA(cudaMemcpyAsync(vals, u_rows, n_td * 4, cudaMemcpyDeviceToDevice, st));
        g->sb_count += T;
        g->e0_dense_stale = true;
    }
    // Tensor-core banks: X (gathered rows) and W_cat are exact in bf16, so only U is split
    // (three bf16 terms = 24 mantissa bits, or one term in the single-term mode); the products
    // accumulate in fp32 TMEM.  Row-major views in the GEMM convention C[M][N] += A(m,k) B(n,k):
    //   g_W[i][k] += sum_t U[t][i] X[t][k]   A = U (MN-major), B = X (MN-major), K = T
    //   dX[t][k]   = sum_i U[t][i] W[i][k]   A = U (K-major),  B = W_cat (MN-major), K = D
    if (tc_terms) {
        const size_t n = n_td;
        const size_t had = g->X16.n;
        g->X16.ensure(n);
        // fresh workspace holds arbitrary bits: zero it once, so that after a bad token (u = 0,
        // the gather skipped) the products are exact zeros, never 0 * NaN
        if (g->X16.n != had) NGH_CUDA(cudaMemsetAsync(g->X16.p, 0, g->X16.n * sizeof(*g->X16.p), st));
        ngk::launch_gather_rows(s, g->grow.p, g->cap, T, b->sub.p, g->X16.p, b->err.p, st);
        Bf16Op u{};
        u.terms = g->terms;
        u.ld = D;
        for (int h = 0; h < g->terms; ++h) u.t[h] = g->Ub.p + size_t(h) * n;
        const Bf16Op x{{g->X16.p, nullptr, nullptr}, 1, true, D};
        const Bf16Op w{{b->wcat.p, nullptr, nullptr}, 1, true, D};
        u.mn = true;
        gemm_bf16_terms(u, x, D, D, T, g->w.p, D, true, b->num_sms, st);
        u.mn = false;
        if (g->sparse) {  // dX [T][B][d] is exactly the appended COO values: the GEMM writes them there
            sparse_reserve(g, T * B, d, st);
            gemm_bf16_terms(u, w, T, D, D, g->sp_vals.p + size_t(g->sp_count) * size_t(d), D, false, b->num_sms, st);
            ngk::launch_rows_to_coo(s, g->grow.p, g->cap, T, g->sp_rows.p + g->sp_count, b->err.p, st);
            g->sp_count += T * B;
        } else {
            gemm_bf16_terms(u, w, T, D, D, g->dX.p, D, false, b->num_sms, st);
            ngk::launch_scatter_rows(s, g->grow.p, g->cap, T, d, D, d, g->dX.p, g->sub.p, b->err.p, st);
        }
    } else if (B > 0 && s.variant == 1) {
        ngk::launch_gather_rows_f32(s, g->grow.p, g->cap, T, b->sub.p, g->X.p, b->err.p, st);
        // fp32 W_cat (re-widened every call: the bank may have been re-uploaded)
        g->wf.ensure(size_t(D) * size_t(D));
        ngk::launch_bf16_to_f32(b->wcat.p, g->wf.p, int64_t(D) * D, st);
        ngk::launch_gemm_f32(g->U.p, D, true, g->X.p, D, true, D, D, T, g->w.p, D, true, st);     // g_W += U^T X
        ngk::launch_gemm_f32(g->U.p, D, false, g->wf.p, D, true, T, D, D, g->dX.p, D, false, st);  // dX = U W_cat
        NGH_CUDA(cudaGetLastError());
        if (g->sparse) {  // dX is [T][B][d]: exactly the appended values, rows transposed from grow
            sparse_reserve(g, T * B, d, st);
            NGH_CUDA(cudaMemcpyAsync(g->sp_vals.p + size_t(g->sp_count) * size_t(d), g->dX.p,
                                     size_t(T) * size_t(D) * 4, cudaMemcpyDeviceToDevice, st));
            ngk::launch_rows_to_coo(s, g->grow.p, g->cap, T, g->sp_rows.p + g->sp_count, b->err.p, st);
            g->sp_count += T * B;
        } else {
            ngk::launch_scatter_rows(s, g->grow.p, g->cap, T, d, D, d, g->dX.p, g->sub.p, b->err.p, st);
        }
    } else if (B > 0) {  // averaged_v1: every branch row receives u (rows are D wide)
        if (g->sparse) {
            sparse_reserve(g, T * B, D, st);
            for (int i = 0; i < B; ++i)  // value of pair (t, b) = U[t]
                NGH_CUDA(cudaMemcpy2DAsync(g->sp_vals.p + (size_t(g->sp_count) + size_t(i)) * size_t(D),
                                           size_t(B) * size_t(D) * 4, g->U.p, size_t(D) * 4, size_t(D) * 4,
                                           size_t(T), cudaMemcpyDeviceToDevice, st));
            ngk::launch_rows_to_coo(s, g->grow.p, g->cap, T, g->sp_rows.p + g->sp_count, b->err.p, st);
            g->sp_count += T * B;
        } else {
            ngk::launch_scatter_rows(s, g->grow.p, g->cap, T, D, D, 0, g->U.p, g->sub.p, b->err.p, st);
        }
    }
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_embed_backward_host(ngram_grad* g, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                              const uint32_t* prior, const float* merged, const float* upstream, int flags) {
    NGRAM_API_BEGIN
    if (!g || nseq < 1 || !seq_offsets) throw Error(NGRAM_EINVAL, "ngram_embed_backward_host: bad argument");
    ngram_bank* b = g->bank;
    std::lock_guard<std::mutex> host_lock(g->bank->host_mu);
    const int64_t T = seq_offsets[nseq];
    if (seq_offsets[0] != 0 || T < 0) throw Error(NGRAM_EINVAL, "seq_offsets must start at 0");
    for (int64_t i = 0; i < nseq; ++i)
        if (seq_offsets[i + 1] < seq_offsets[i]) throw Error(NGRAM_EINVAL, "seq_offsets must be non-decreasing");
    if (T > 0 && (!tokens || !upstream)) throw Error(NGRAM_EINVAL, "ngram_embed_backward_host: bad argument");
    DeviceGuard dg(b->device);
    const size_t D = size_t(b->cfg.dim);
    const int N1 = std::max(b->cfg.max_order - 1, 0);
    g->h_tokens.ensure(size_t(std::max<int64_t>(T, 1)));
    g->h_off.ensure(size_t(nseq + 1));
    g->h_up.ensure(std::max<size_t>(size_t(T) * D, 1));
    if (merged) g->h_merged.ensure(std::max<size_t>(size_t(T) * D, 1));
    if (prior && N1 > 0) g->h_prior.ensure(size_t(nseq) * size_t(N1));
    if (T > 0) {
        NGH_CUDA(cudaMemcpy(g->h_tokens.p, tokens, size_t(T) * 4, cudaMemcpyHostToDevice));
        NGH_CUDA(cudaMemcpy(g->h_up.p, upstream, size_t(T) * D * 4, cudaMemcpyHostToDevice));
        if (merged) NGH_CUDA(cudaMemcpy(g->h_merged.p, merged, size_t(T) * D * 4, cudaMemcpyHostToDevice));
    }
    NGH_CUDA(cudaMemcpy(g->h_off.p, seq_offsets, size_t(nseq + 1) * 8, cudaMemcpyHostToDevice));
    if (prior && N1 > 0)
        NGH_CUDA(cudaMemcpy(g->h_prior.p, prior, size_t(nseq) * size_t(N1) * 4, cudaMemcpyHostToDevice));
    const int rc = ngram_embed_backward(g, g->h_tokens.p, g->h_off.p, nseq, T, (prior && N1 > 0) ? g->h_prior.p : nullptr,
                                        merged ? g->h_merged.p : nullptr, g->h_up.p, flags, nullptr);
    if (rc != NGRAM_OK) return rc;
    unsigned long long e = 0;
    NGH_CUDA(cudaMemcpy(&e, b->err.p, sizeof(e), cudaMemcpyDeviceToHost));
    if (e != ~0ull)
        throw Error(NGRAM_ERANGE, "embedding: token out of range for base vocabulary " +
                                      std::to_string(b->cfg.base_vocab) + " (first bad window at position " +
                                      std::to_string(e) + ")");
    NGRAM_API_END
}

int ngram_amplify_backward_host(ngram_bank* b, int64_t rows, const float* pre, const float* upstream, float* d_pre,
                                float* g_gain, float* g_bias) {
    NGRAM_API_BEGIN
    if (!b || rows < 0 || (rows > 0 && (!pre || !upstream || !d_pre)))
        throw Error(NGRAM_EINVAL, "ngram_amplify_backward_host: bad argument");
    if (b->hash_only) throw Error(NGRAM_EINVAL, "bank was created hash-only (NGRAM_BANK_HASH_ONLY)");
    if (rows == 0) return NGRAM_OK;
    std::lock_guard<std::mutex> host_lock(b->host_mu);
    DeviceGuard dg(b->device);
    ngk::Shape s = b->shape;
    s.denom = 1;  // d_pre itself: no 1/denom merge scale here (that is embed_backward's)
    const size_t D = size_t(s.D), n = size_t(rows) * D;
    const bool ln = s.amp == ngk::kAmpLN;
    DevBuf<float> dp, du, dd, ge0, gg, gb;
    DevBuf<uint32_t> tok;
    DevBuf<unsigned long long> err;
    dp.alloc(n);
    du.alloc(n);
    dd.alloc(n);
    ge0.alloc(D);  // the kernel's E0-row scatter lands here (token 0) and is discarded
    tok.alloc(size_t(rows));
    err.alloc(1);
    NGH_CUDA(cudaMemcpy(dp.p, pre, n * 4, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(du.p, upstream, n * 4, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemset(tok.p, 0, size_t(rows) * 4));
    NGH_CUDA(cudaMemset(err.p, 0xff, 8));
    if (ln) {
        gg.alloc(D);
        gb.alloc(D);
        if (g_gain) NGH_CUDA(cudaMemcpy(gg.p, g_gain, D * 4, cudaMemcpyHostToDevice));
        else NGH_CUDA(cudaMemset(gg.p, 0, D * 4));
        if (g_bias) NGH_CUDA(cudaMemcpy(gb.p, g_bias, D * 4, cudaMemcpyHostToDevice));
        else NGH_CUDA(cudaMemset(gb.p, 0, D * 4));
    }
    ngk::launch_amp_backward(s, du.p, dp.p, tok.p, rows, s.amp, b->ln_gain.p, dd.p, ge0.p, gg.p, gb.p, err.p, nullptr);
    NGH_CUDA(cudaMemcpy(d_pre, dd.p, n * 4, cudaMemcpyDeviceToHost));
    if (ln && g_gain) NGH_CUDA(cudaMemcpy(g_gain, gg.p, D * 4, cudaMemcpyDeviceToHost));
    if (ln && g_bias) NGH_CUDA(cudaMemcpy(g_bias, gb.p, D * 4, cudaMemcpyDeviceToHost));
    NGRAM_API_END
}

int ngram_grad_sparse_rows(ngram_grad* g, int32_t** rows, float** vals, int64_t* count) {
    NGRAM_API_BEGIN
    if (!g || !rows || !vals || !count) throw Error(NGRAM_EINVAL, "ngram_grad_sparse_rows: bad argument");
    if (!g->sparse) throw Error(NGRAM_EINVAL, "gradient bank was not created with NGRAM_GRAD_SPARSE_ROWS");
    *rows = g->sp_rows.p;
    *vals = g->sp_vals.p;
    *count = g->sp_count;
    NGRAM_API_END
}

int ngram_grad_sparse_read(ngram_grad* g, int64_t first, int64_t count, int32_t* rows, float* vals, void* stream) {
    NGRAM_API_BEGIN
    if (!g || first < 0 || count < 0 || first + count > g->sp_count)
        throw Error(NGRAM_EINVAL, "ngram_grad_sparse_read: bad range");
    if (!g->sparse) throw Error(NGRAM_EINVAL, "gradient bank was not created with NGRAM_GRAD_SPARSE_ROWS");
    DeviceGuard dg(g->bank->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t d = size_t(g->bank->shape.d);
    if (rows && count)
        NGH_CUDA(cudaMemcpyAsync(rows, g->sp_rows.p + first, size_t(count) * 4, cudaMemcpyDefault, st));
    if (vals && count)
        NGH_CUDA(cudaMemcpyAsync(vals, g->sp_vals.p + size_t(first) * d, size_t(count) * d * 4, cudaMemcpyDefault, st));
    NGRAM_API_END
}

int ngram_grad_sparse_base(ngram_grad* g, int32_t** tokens, float** vals, int64_t* count) {
    NGRAM_API_BEGIN
    if (!g || !tokens || !vals || !count) throw Error(NGRAM_EINVAL, "ngram_grad_sparse_base: bad argument");
    if (!g->sparse_base) throw Error(NGRAM_EINVAL, "gradient bank was not created with NGRAM_GRAD_SPARSE_BASE");
    *tokens = g->sb_tok.p;
    *vals = g->sb_vals.p;
    *count = g->sb_count;
    NGRAM_API_END
}

int ngram_grad_tensor(ngram_grad* g, int which, float** dev_ptr, int64_t* numel) {
    NGRAM_API_BEGIN
    if (!g || !dev_ptr || !numel) throw Error(NGRAM_EINVAL, "ngram_grad_tensor: bad argument");
    DevBuf<float>* t = nullptr;
    if (which == 0) densify_base(g, nullptr);
    switch (which) {
        case 0: t = &g->e0; break;
        case 1: t = &g->sub; break;
        case 2: t = &g->w; break;
        case 3: t = &g->gain; break;
        case 4: t = &g->bias; break;
        default: throw Error(NGRAM_EINVAL, "ngram_grad_tensor: which must be 0..4");
    }
    *dev_ptr = t->p;
    *numel = int64_t(t->n);
    NGRAM_API_END
}

int ngram_grad_download(ngram_grad* g, float* base, float* const* sub, float* const* proj, float* gain, float* bias) {
    NGRAM_API_BEGIN
    if (!g) throw Error(NGRAM_EINVAL, "null gradient bank");
    ngram_bank* b = g->bank;
    DeviceGuard dg(b->device);
    if (base) densify_base(g, nullptr);
    NGH_CUDA(cudaDeviceSynchronize());
    const auto& s = b->shape;
    if (base) NGH_CUDA(cudaMemcpy(base, g->e0.p, g->e0.n * sizeof(float), cudaMemcpyDeviceToHost));
    if (sub && g->sparse)
        throw Error(NGRAM_EINVAL, "row-sparse gradient bank: read sub-table gradients with ngram_grad_sparse_rows");
    if (sub)
        for (int i = 0; i < s.B; ++i)
            if (sub[i])
                NGH_CUDA(cudaMemcpy(sub[i], g->sub.p + size_t(b->row_base[size_t(i)]) * size_t(s.d),
                                    size_t(b->row_hi[size_t(i)] - b->row_lo[size_t(i)]) * size_t(s.d) * sizeof(float),
                                    cudaMemcpyDeviceToHost));
    if (proj && g->w.n) {  // W_cat[i][b*d + j] -> proj_b[i*d + j]
        const size_t D = size_t(s.D), d = size_t(s.d);
        for (int i = 0; i < s.B; ++i)
            if (proj[i])
                NGH_CUDA(cudaMemcpy2D(proj[i], d * sizeof(float), g->w.p + size_t(i) * d, D * sizeof(float),
                                      d * sizeof(float), D, cudaMemcpyDeviceToHost));
    }
    if (gain && g->gain.n) NGH_CUDA(cudaMemcpy(gain, g->gain.p, g->gain.n * sizeof(float), cudaMemcpyDeviceToHost));
    if (bias && g->bias.n) NGH_CUDA(cudaMemcpy(bias, g->bias.p, g->bias.n * sizeof(float), cudaMemcpyDeviceToHost));
    NGRAM_API_END
}

}  // extern "C"
