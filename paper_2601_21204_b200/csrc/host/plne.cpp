// plne.cpp -- C-ABI of the per-layer N-gram FFN (PLNE, ple.hpp:168-196):
//   y = W_d (SiLU(W_g x) (.) g),   g = the layer bank's merged embedding (no amplification).
// Batched over T positions: G from the N-gram forward (K1+K2 -> K3, amp none), U = X W_g^T and
// Y = Hh W_d^T as fp32 GEMMs (gemm_gen.cu: the fp32 CUDA-core GEMM by default, or -- with
// NGRAM_PLNE_FAST -- both operands split into three bf16 terms on the tensor cores), SiLU
// gating elementwise (plne.cu).  The plain
// per-layer form ffn_ple (a table row as the gate) is PLNE with a base-only layer bank
// (max_order 1, E0 = the table), as the reference's own test states (test_ple.cpp:150-172).
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <string>

#include "api_util.hpp"
#include "bank.hpp"
#include "gemm.hpp"

using namespace ngh;

struct ngram_plne {
    ngram_bank* bank = nullptr;
    int d_model = 0, hidden = 0;
    DevBuf<float> U, G, Hh, dHh, dG, dU;
    int64_t cap = 0;
    // host-buffer entry staging
    DevBuf<float> h_gate, h_down, h_x, h_y, h_up, h_dgate, h_ddown, h_dx;
    DevBuf<uint32_t> h_tok, h_prior;
    DevBuf<int64_t> h_off;
    bool three = true;                 // split-bf16 tensor-core GEMMs (default); false: NGRAM_PLNE_PEDANTIC
    SplitWs ws;                        // three bf16 terms of each GEMM operand
};

namespace {

// C[M][N] (+)= sum_k A(m, k) B(n, k) (gemm.hpp convention).  Default: the fp32 CUDA-core GEMM
// (pedantic).  NGRAM_PLNE_FAST: on the bf16 tensor cores -- A = a1 + a2 + a3 and B = b1 + b2 + b3
// in bf16, the six products a_i b_j with i + j <= 4 accumulated in fp32 TMEM
// (tests/test_gpu_plne.py: within 1e-5 relL2 of fp64 at d_model = hidden = 3072).
void gemm(ngram_plne* p, const F32Op& A, const F32Op& B, int64_t M, int64_t N, int64_t K, float* C, int64_t ldc,
          bool accumulate, cudaStream_t st) {
    gemm_f32(A, B, M, N, K, C, ldc, accumulate, p->three, p->ws, p->bank->num_sms, st);
}

void status_ok(int rc) {
    if (rc != NGRAM_OK) throw Error(rc, ngram_last_error());
}

void ensure(ngram_plne* p, int64_t T, bool backward) {
    if (T <= p->cap && (!backward || p->dHh.n)) return;
    const int64_t cap = std::max<int64_t>(T, p->cap);
    const size_t n = size_t(cap) * size_t(p->hidden);
    for (DevBuf<float>* b : {&p->U, &p->G, &p->Hh}) b->ensure(n);
    if (backward)
        for (DevBuf<float>* b : {&p->dHh, &p->dG, &p->dU}) b->ensure(n);
    p->cap = cap;
}

// G = merged layer-bank rows, U = X W_g^T, Hh = SiLU(U) * G.  Row-major M (r x c) is the
// column-major M^T with ld = c, so U^T (H x T) = gate_cm^T X_cm etc.
void forward_common(ngram_plne* p, const float* gate, const float* x, const uint32_t* tokens, const int64_t* off,
                    int64_t nseq, int64_t T, const uint32_t* prior, cudaStream_t st) {
    status_ok(ngram_embed_forward(p->bank, tokens, off, nseq, T, prior, nullptr, p->G.p, NGRAM_F32, st));
    const int H = p->hidden, Dm = p->d_model;
    // U[t][h] = sum_dm X[t][dm] W_g[h][dm]
    gemm(p, {x, false, Dm}, {gate, false, Dm}, T, H, Dm, p->U.p, H, false, st);
    ngk::launch_silu_gate(p->U.p, p->G.p, p->Hh.p, T * H, p->bank->err.p, st);
}

}  // namespace

extern "C" {

int ngram_plne_create(ngram_bank* b, int d_model, ngram_plne** out) { return ngram_plne_create_ex(b, d_model, 0, out); }

int ngram_plne_create_ex(ngram_bank* b, int d_model, int flags, ngram_plne** out) {
    NGRAM_API_BEGIN
    if (flags & ~(NGRAM_PLNE_FAST | NGRAM_PLNE_PEDANTIC) || flags == (NGRAM_PLNE_FAST | NGRAM_PLNE_PEDANTIC))
        throw Error(NGRAM_EINVAL, "ngram_plne_create_ex: unknown flags");
    if (!b || !out) throw Error(NGRAM_EINVAL, "ngram_plne_create: bad argument");
    if (d_model < 1) throw Error(NGRAM_EINVAL, "ple: d_model and hidden must be >= 1");
    if (b->hash_only) throw Error(NGRAM_EINVAL, "bank was created hash-only (NGRAM_BANK_HASH_ONLY)");
    if (b->shard_count != 1) throw Error(NGRAM_EINVAL, "ngram_plne_create: row-sharded layer banks are not supported");
    if (b->shape.amp != ngk::kAmpNone) throw Error(NGRAM_EINVAL, "ffn_plne: layer banks use no amplification");
    DeviceGuard dg(b->device);
    auto p = std::make_unique<ngram_plne>();
    p->bank = b;
    p->d_model = d_model;
    p->hidden = b->shape.D;
    p->three = (flags & NGRAM_PLNE_PEDANTIC) == 0;  // tensor-core split GEMMs unless pedantic
    *out = p.release();
    NGRAM_API_END
}

int ngram_plne_destroy(ngram_plne* p) {
    NGRAM_API_BEGIN
    if (p) {
        DeviceGuard dg(p->bank->device);
        delete p;
    }
    NGRAM_API_END
}

int ngram_plne_forward(ngram_plne* p, const float* gate, const float* down, const float* x, const uint32_t* tokens,
                       const int64_t* seq_offsets, int64_t nseq, int64_t T, const uint32_t* prior, float* y,
                       void* stream) {
    NGRAM_API_BEGIN
    if (!p || !seq_offsets || nseq < 1 || T < 0 || (T > 0 && (!gate || !down || !x || !tokens || !y)))
        throw Error(NGRAM_EINVAL, "ngram_plne_forward: bad argument");
    DeviceGuard dg(p->bank->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (T == 0) return NGRAM_OK;
    ensure(p, T, false);
    forward_common(p, gate, x, tokens, seq_offsets, nseq, T, prior, st);
    const int H = p->hidden, Dm = p->d_model;
    // Y[t][dm] = sum_h Hh[t][h] W_d[dm][h]
    gemm(p, {p->Hh.p, false, H}, {down, false, H}, T, Dm, H, y, Dm, false, st);
    NGRAM_API_END
}

int ngram_plne_backward(ngram_plne* p, ngram_grad* bank_grads, const float* gate, const float* down, const float* x,
                        const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq, int64_t T,
                        const uint32_t* prior, const float* upstream, float* d_gate, float* d_down, float* dx,
                        void* stream) {
    NGRAM_API_BEGIN
    if (!p || !seq_offsets || nseq < 1 || T < 0 ||
        (T > 0 && (!gate || !down || !x || !tokens || !upstream || !d_gate || !d_down || !dx)))
        throw Error(NGRAM_EINVAL, "ngram_plne_backward: bad argument");
    if (bank_grads && grad_bank(bank_grads) != p->bank)
        throw Error(NGRAM_EINVAL, "ngram_plne_backward: gradient bank belongs to another bank");
    DeviceGuard dg(p->bank->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (T == 0) return NGRAM_OK;
    ensure(p, T, true);
    forward_common(p, gate, x, tokens, seq_offsets, nseq, T, prior, st);  // recompute, as the reference
    const int H = p->hidden, Dm = p->d_model;
    // g_down[dm][h] += sum_t dY[t][dm] Hh[t][h]
    gemm(p, {upstream, true, Dm}, {p->Hh.p, true, H}, Dm, H, T, d_down, H, true, st);
    // dHh[t][h] = sum_dm dY[t][dm] W_d[dm][h]
    gemm(p, {upstream, false, Dm}, {down, true, H}, T, H, Dm, p->dHh.p, H, false, st);
    ngk::launch_silu_gate_backward(p->dHh.p, p->U.p, p->G.p, p->dG.p, p->dU.p, T * H, p->bank->err.p, st);
    if (bank_grads)  // embed_backward of dL/dg (ple.hpp:195)
        status_ok(ngram_embed_backward(bank_grads, tokens, seq_offsets, nseq, T, prior, nullptr, p->dG.p,
                                       NGRAM_BWD_SKIP_AMPLIFY, st));
    // g_gate[h][dm] += sum_t dU[t][h] X[t][dm]
    gemm(p, {p->dU.p, true, H}, {x, true, Dm}, H, Dm, T, d_gate, Dm, true, st);
    // dx[t][dm] += sum_h dU[t][h] W_g[h][dm]
    gemm(p, {p->dU.p, false, H}, {gate, true, Dm}, T, Dm, H, dx, Dm, true, st);
    NGRAM_API_END
}

// Host-buffer variants (synchronous): stage through device buffers, accumulate on the device.
static void stage_common(ngram_plne* p, const float* gate, const float* down, const float* x, const uint32_t* tokens,
                         const int64_t* off, int64_t nseq, int64_t T, const uint32_t* prior) {
    const size_t H = size_t(p->hidden), Dm = size_t(p->d_model);
    const int N1 = std::max(p->bank->cfg.max_order - 1, 0);
    p->h_gate.ensure(H * Dm);
    p->h_down.ensure(H * Dm);
    p->h_x.ensure(std::max<size_t>(size_t(T) * Dm, 1));
    p->h_tok.ensure(size_t(std::max<int64_t>(T, 1)));
    p->h_off.ensure(size_t(nseq + 1));
    NGH_CUDA(cudaMemcpy(p->h_gate.p, gate, H * Dm * 4, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(p->h_down.p, down, H * Dm * 4, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(p->h_x.p, x, size_t(T) * Dm * 4, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(p->h_tok.p, tokens, size_t(T) * 4, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(p->h_off.p, off, size_t(nseq + 1) * 8, cudaMemcpyHostToDevice));
    if (prior && N1 > 0) {
        p->h_prior.ensure(size_t(nseq) * size_t(N1));
        NGH_CUDA(cudaMemcpy(p->h_prior.p, prior, size_t(nseq) * size_t(N1) * 4, cudaMemcpyHostToDevice));
    }
}

static void check_host_offsets(const int64_t* off, int64_t nseq) {
    if (off[0] != 0) throw Error(NGRAM_EINVAL, "seq_offsets must start at 0");
    for (int64_t i = 0; i < nseq; ++i)
        if (off[i + 1] < off[i]) throw Error(NGRAM_EINVAL, "seq_offsets must be non-decreasing");
}

static void raise_token_error(ngram_bank* b) {
    unsigned long long e = 0;
    NGH_CUDA(cudaMemcpy(&e, b->err.p, sizeof(e), cudaMemcpyDeviceToHost));
    if (e != ~0ull)
        throw Error(NGRAM_ERANGE, "embedding: token out of range for base vocabulary " +
                                      std::to_string(b->cfg.base_vocab) + " (first bad window at position " +
                                      std::to_string(e) + ")");
}

int ngram_plne_forward_host(ngram_plne* p, const float* gate, const float* down, const float* x,
                            const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq, const uint32_t* prior,
                            float* y) {
    NGRAM_API_BEGIN
    if (!p || !seq_offsets || nseq < 1) throw Error(NGRAM_EINVAL, "ngram_plne_forward_host: bad argument");
    check_host_offsets(seq_offsets, nseq);
    std::lock_guard<std::mutex> host_lock(p->bank->host_mu);
    const int64_t T = seq_offsets[nseq];
    if (T == 0) return NGRAM_OK;
    if (!gate || !down || !x || !tokens || !y) throw Error(NGRAM_EINVAL, "ngram_plne_forward_host: bad argument");
    DeviceGuard dg(p->bank->device);
    stage_common(p, gate, down, x, tokens, seq_offsets, nseq, T, prior);
    const size_t Dm = size_t(p->d_model);
    p->h_y.ensure(size_t(T) * Dm);
    const int N1 = std::max(p->bank->cfg.max_order - 1, 0);
    status_ok(ngram_plne_forward(p, p->h_gate.p, p->h_down.p, p->h_x.p, p->h_tok.p, p->h_off.p, nseq, T,
                                 (prior && N1 > 0) ? p->h_prior.p : nullptr, p->h_y.p, nullptr));
    raise_token_error(p->bank);
    NGH_CUDA(cudaMemcpy(y, p->h_y.p, size_t(T) * Dm * 4, cudaMemcpyDeviceToHost));
    NGRAM_API_END
}

int ngram_plne_backward_host(ngram_plne* p, ngram_grad* bank_grads, const float* gate, const float* down,
                             const float* x, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                             const uint32_t* prior, const float* upstream, float* d_gate, float* d_down, float* dx) {
    NGRAM_API_BEGIN
    if (!p || !seq_offsets || nseq < 1) throw Error(NGRAM_EINVAL, "ngram_plne_backward_host: bad argument");
    check_host_offsets(seq_offsets, nseq);
    std::lock_guard<std::mutex> host_lock(p->bank->host_mu);
    const int64_t T = seq_offsets[nseq];
    if (T == 0) return NGRAM_OK;
    if (!gate || !down || !x || !tokens || !upstream || !d_gate || !d_down || !dx)
        throw Error(NGRAM_EINVAL, "ngram_plne_backward_host: bad argument");
    DeviceGuard dg(p->bank->device);
    stage_common(p, gate, down, x, tokens, seq_offsets, nseq, T, prior);
    const size_t H = size_t(p->hidden), Dm = size_t(p->d_model), n = size_t(T) * Dm;
    p->h_up.ensure(n);
    p->h_dx.ensure(n);
    p->h_dgate.ensure(H * Dm);
    p->h_ddown.ensure(H * Dm);
    NGH_CUDA(cudaMemcpy(p->h_up.p, upstream, n * 4, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(p->h_dx.p, dx, n * 4, cudaMemcpyHostToDevice));  // accumulated on the device
    NGH_CUDA(cudaMemcpy(p->h_dgate.p, d_gate, H * Dm * 4, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(p->h_ddown.p, d_down, H * Dm * 4, cudaMemcpyHostToDevice));
    const int N1 = std::max(p->bank->cfg.max_order - 1, 0);
    status_ok(ngram_plne_backward(p, bank_grads, p->h_gate.p, p->h_down.p, p->h_x.p, p->h_tok.p, p->h_off.p, nseq, T,
                                  (prior && N1 > 0) ? p->h_prior.p : nullptr, p->h_up.p, p->h_dgate.p, p->h_ddown.p,
                                  p->h_dx.p, nullptr));
    raise_token_error(p->bank);
    NGH_CUDA(cudaMemcpy(dx, p->h_dx.p, n * 4, cudaMemcpyDeviceToHost));
    NGH_CUDA(cudaMemcpy(d_gate, p->h_dgate.p, H * Dm * 4, cudaMemcpyDeviceToHost));
    NGH_CUDA(cudaMemcpy(d_down, p->h_ddown.p, H * Dm * 4, cudaMemcpyDeviceToHost));
    NGRAM_API_END
}

}  // extern "C"
