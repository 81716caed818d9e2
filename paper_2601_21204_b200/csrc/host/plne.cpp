// plne.cpp -- C-ABI of the per-layer N-gram FFN (PLNE, ple.hpp:168-196):
//   y = W_d (SiLU(W_g x) (.) g),   g = the layer bank's merged embedding (no amplification).
// Batched over T positions: G from the N-gram forward (K1+K2 -> K3, amp none), U = X W_g^T and
// Y = Hh W_d^T as fp32 GEMMs (cuBLAS, no TF32), SiLU gating elementwise (plne.cu).  The plain
// per-layer form ffn_ple (a table row as the gate) is PLNE with a base-only layer bank
// (max_order 1, E0 = the table), as the reference's own test states (test_ple.cpp:150-172).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <string>

#include "api_util.hpp"
#include "bank.hpp"

using namespace ngh;

struct ngram_plne {
    ngram_bank* bank = nullptr;
    int d_model = 0, hidden = 0;
    cublasHandle_t blas = nullptr;
    DevBuf<float> U, G, Hh, dHh, dG, dU;
    int64_t cap = 0;
    // host-buffer entry staging
    DevBuf<float> h_gate, h_down, h_x, h_y, h_up, h_dgate, h_ddown, h_dx;
    DevBuf<uint32_t> h_tok, h_prior;
    DevBuf<int64_t> h_off;
    bool three = false;                // NGRAM_PLNE_FAST: split-bf16 tensor-core GEMMs
    DevBuf<__nv_bfloat16> as, bs;      // three bf16 terms of each GEMM operand
    ~ngram_plne() {
        if (blas) cublasDestroy(blas);
    }
};

namespace {

void blas_ok(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS)
        throw Error(NGRAM_ECUDA, std::string(what) + " failed (cublas status " + std::to_string(int(s)) + ")");
}

// C = A op B (+ beta C).  Default: one pedantic fp32 GEMM (CUDA cores; relL2 6e-7 vs fp64 at
// K = 3072).  NGRAM_PLNE_FAST: on the bf16 tensor cores -- A = a1 + a2 + a3 and B = b1 + b2 + b3
// in bf16, the six products a_i b_j with i + j <= 4 accumulated in fp32: 2.9x faster, relL2 7e-6
// vs fp64 at K = 3072 (a three-term TF32 split measured 1.5e-5; tests/test_gpu_plne.py).
// nA / nB: element counts of the stored operands (split elementwise, whatever the op).
void gemm(ngram_plne* p, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, const float* A, size_t nA,
          int lda, const float* B, size_t nB, int ldb, float beta, float* C, int ldc, cudaStream_t st,
          const char* what) {
    const float one = 1.0f;
    if (!p->three) {
        blas_ok(cublasSgemm(p->blas, ta, tb, m, n, k, &one, A, lda, B, ldb, &beta, C, ldc), what);
        return;
    }
    p->as.ensure(3 * nA);
    p->bs.ensure(3 * nB);
    ngk::launch_split_bf16x3(A, p->as.p, p->as.p + nA, p->as.p + 2 * nA, int64_t(nA), st);
    ngk::launch_split_bf16x3(B, p->bs.p, p->bs.p + nB, p->bs.p + 2 * nB, int64_t(nB), st);
    static const int pairs[6][2] = {{2, 0}, {1, 1}, {0, 2}, {1, 0}, {0, 1}, {0, 0}};  // small terms first
    for (int q = 0; q < 6; ++q) {
        const float* bt = &beta;
        blas_ok(cublasGemmEx(p->blas, ta, tb, m, n, k, &one, p->as.p + size_t(pairs[q][0]) * nA, CUDA_R_16BF, lda,
                             p->bs.p + size_t(pairs[q][1]) * nB, CUDA_R_16BF, ldb, q ? &one : bt, C, CUDA_R_32F, ldc,
                             CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT),
                what);
    }
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
    const float one = 1.0f, zero = 0.0f;
    const int H = p->hidden, Dm = p->d_model;
    blas_ok(cublasSetStream(p->blas, st), "cublasSetStream");
    (void)one;
    gemm(p, CUBLAS_OP_T, CUBLAS_OP_N, H, int(T), Dm, gate, size_t(H) * Dm, Dm, x, size_t(T) * Dm, Dm, zero, p->U.p, H,
         st, "cublasSgemm(U = X W_g^T)");
    ngk::launch_silu_gate(p->U.p, p->G.p, p->Hh.p, T * H, p->bank->err.p, st);
}

}  // namespace

extern "C" {

int ngram_plne_create(ngram_bank* b, int d_model, ngram_plne** out) { return ngram_plne_create_ex(b, d_model, 0, out); }

int ngram_plne_create_ex(ngram_bank* b, int d_model, int flags, ngram_plne** out) {
    NGRAM_API_BEGIN
    if (flags & ~NGRAM_PLNE_FAST) throw Error(NGRAM_EINVAL, "ngram_plne_create_ex: unknown flags");
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
    blas_ok(cublasCreate(&p->blas), "cublasCreate");
    p->three = (flags & NGRAM_PLNE_FAST) != 0;
    blas_ok(cublasSetMathMode(p->blas, p->three ? CUBLAS_DEFAULT_MATH : CUBLAS_PEDANTIC_MATH), "cublasSetMathMode");
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
    const float one = 1.0f, zero = 0.0f;
    const int H = p->hidden, Dm = p->d_model;
    (void)one;
    gemm(p, CUBLAS_OP_T, CUBLAS_OP_N, Dm, int(T), H, down, size_t(H) * Dm, H, p->Hh.p, size_t(T) * H, H, zero, y, Dm,
         st, "cublasSgemm(Y = Hh W_d^T)");
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
    const float one = 1.0f, zero = 0.0f;
    const int H = p->hidden, Dm = p->d_model;
    const int n = int(T);
    // g_down (Dm x H) += dY^T Hh  <=>  col-major g_down^T (H x Dm) += Hh_cm dY_cm^T
    gemm(p, CUBLAS_OP_N, CUBLAS_OP_T, H, Dm, n, p->Hh.p, size_t(n) * H, H, upstream, size_t(n) * Dm, Dm, one, d_down,
         H, st, "cublasSgemm(dW_d)");
    // dHh (T x H) = dY W_d  <=>  col-major dHh^T = down_cm dY_cm
    gemm(p, CUBLAS_OP_N, CUBLAS_OP_N, H, n, Dm, down, size_t(H) * Dm, H, upstream, size_t(n) * Dm, Dm, zero, p->dHh.p,
         H, st, "cublasSgemm(dHh)");
    ngk::launch_silu_gate_backward(p->dHh.p, p->U.p, p->G.p, p->dG.p, p->dU.p, T * H, p->bank->err.p, st);
    if (bank_grads)  // embed_backward of dL/dg (ple.hpp:195)
        status_ok(ngram_embed_backward(bank_grads, tokens, seq_offsets, nseq, T, prior, nullptr, p->dG.p,
                                       NGRAM_BWD_SKIP_AMPLIFY, st));
    // g_gate (H x Dm) += dU^T X  <=>  col-major g_gate^T (Dm x H) += X_cm dU_cm^T
    gemm(p, CUBLAS_OP_N, CUBLAS_OP_T, Dm, H, n, x, size_t(n) * Dm, Dm, p->dU.p, size_t(n) * H, H, one, d_gate, Dm, st,
         "cublasSgemm(dW_g)");
    // dx (T x Dm) += dU W_g  <=>  col-major dx^T += gate_cm dU_cm
    gemm(p, CUBLAS_OP_N, CUBLAS_OP_N, Dm, n, H, gate, size_t(H) * Dm, Dm, p->dU.p, size_t(n) * H, H, one, dx, Dm, st,
         "cublasSgemm(dx)");
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
