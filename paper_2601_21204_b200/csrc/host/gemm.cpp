// gemm.cpp -- host side of gemm_gen.cu (see gemm.hpp).
#include "gemm.hpp"

#include <algorithm>
#include <map>
#include <memory>
#include <mutex>

#include "api_util.hpp"
#include "../kernels/kernels.h"

namespace ngh {

namespace {
void operand_maps(const Bf16Op& X, int64_t R, int64_t K, CUtensorMap (&maps)[3]) {
    for (int i = 0; i < X.terms; ++i) {
        if ((X.ld % 8) != 0 || (reinterpret_cast<uintptr_t>(X.t[i]) % 16) != 0)
            throw Error(NGRAM_EINVAL, "gemm: bf16 operand pitch must be a multiple of 8 elements, 16-byte aligned");
        if (X.mn)  // inner = R (contiguous), rows = K; box 64 x 64
            make_tensor_map_2d(&maps[i], X.t[i], uint64_t(R), uint64_t(K), uint64_t(X.ld) * 2, 64, 64);
        else  // inner = K, rows = R; box 64 x 128
            make_tensor_map_2d(&maps[i], X.t[i], uint64_t(K), uint64_t(R), uint64_t(X.ld) * 2, 64, 128);
    }
}
}  // namespace

void gemm_bf16_terms(const Bf16Op& A, const Bf16Op& B, int64_t M, int64_t N, int64_t K, float* C, int64_t ldc,
                     bool accumulate, int num_sms, cudaStream_t st) {
    if (M <= 0 || N <= 0) return;
    if (!((A.terms == 1 || A.terms == 3) && (B.terms == 1 || B.terms == 3)) && !(A.terms == 2 && B.terms == 1))
        throw Error(NGRAM_EINVAL, "gemm: operand terms (1 or 3 each, or 2 x 1)");
    if (K <= 0) {
        if (!accumulate) NGH_CUDA(cudaMemset2DAsync(C, size_t(ldc) * 4, 0, size_t(N) * 4, size_t(M), st));
        return;
    }
    CUtensorMap ma[3], mb[3];
    operand_maps(A, M, K, ma);
    operand_maps(B, N, K, mb);
    ngk::launch_gemm_bf16_terms(ma, A.terms, A.mn, mb, B.terms, B.mn, M, N, K, C, ldc, accumulate, num_sms, st);
    NGH_CUDA(cudaGetLastError());
}

Bf16Op split_operand(const F32Op& X, int64_t R, int64_t K, int terms, DevBuf<__nv_bfloat16>& buf, cudaStream_t st) {
    // stored matrix: rows x cols (K-major: R x K; MN-major: K x R)
    const int64_t rows = X.mn ? K : R, cols = X.mn ? R : K;
    const int64_t ldt = round_up(std::max<int64_t>(cols, 1), 8);
    const size_t n = size_t(rows) * size_t(ldt);
    buf.ensure(size_t(terms) * n);
    Bf16Op o{};
    o.terms = terms;
    o.mn = X.mn;
    o.ld = ldt;
    for (int i = 0; i < terms; ++i) o.t[i] = buf.p + size_t(i) * n;
    ngk::launch_split3(X.p, rows, cols, X.ld, buf.p, terms > 1 ? buf.p + n : nullptr, terms > 2 ? buf.p + 2 * n : nullptr,
                       ldt, st);
    return o;
}

void gemm_f32(const F32Op& A, const F32Op& B, int64_t M, int64_t N, int64_t K, float* C, int64_t ldc,
              bool accumulate, bool split3, SplitWs& ws, int num_sms, cudaStream_t st) {
    if (M <= 0 || N <= 0) return;
    if (!split3) {
        if (K <= 0) {
            if (!accumulate) NGH_CUDA(cudaMemset2DAsync(C, size_t(ldc) * 4, 0, size_t(N) * 4, size_t(M), st));
            return;
        }
        ngk::launch_gemm_f32(A.p, A.ld, A.mn, B.p, B.ld, B.mn, M, N, K, C, ldc, accumulate, st);
        NGH_CUDA(cudaGetLastError());
        return;
    }
    const Bf16Op a = split_operand(A, M, K, 3, ws.a, st);
    const Bf16Op b = split_operand(B, N, K, 3, ws.b, st);
    gemm_bf16_terms(a, b, M, N, K, C, ldc, accumulate, num_sms, st);
}

}  // namespace ngh

using namespace ngh;

extern "C" int ngram_gemm_f32(int device, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int a_mn,
                              const float* B, int64_t ldb, int b_mn, float* C, int64_t ldc, int accumulate,
                              int a_terms, int b_terms, void* stream) {
    NGRAM_API_BEGIN
    if (M < 0 || N < 0 || K < 0 || (M && N && (!C || ldc < N)) || (M && N && K && (!A || !B)))
        throw Error(NGRAM_EINVAL, "ngram_gemm_f32: bad argument");
    if (a_terms != 0 && !(((a_terms == 1 || a_terms == 3) && (b_terms == 1 || b_terms == 3)) ||
                          (a_terms == 2 && b_terms == 1)))
        throw Error(NGRAM_EINVAL, "ngram_gemm_f32: terms 1 or 3 each, or 2 x 1 (or a_terms = 0: fp32 CUDA cores)");
    if (lda < (a_mn ? M : K) || ldb < (b_mn ? N : K)) throw Error(NGRAM_EINVAL, "ngram_gemm_f32: bad pitch");
    DeviceGuard g(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    static std::mutex mu;
    static auto& wss = *new std::map<int, std::unique_ptr<SplitWs>>();  // per device, never destroyed
    std::lock_guard<std::mutex> lk(mu);
    auto& ws = wss[device];
    if (!ws) ws = std::make_unique<SplitWs>();
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (a_terms == 0) {
        gemm_f32({A, a_mn != 0, lda}, {B, b_mn != 0, ldb}, M, N, K, C, ldc, accumulate != 0, false, *ws, sms, st);
    } else {
        if (M <= 0 || N <= 0) return NGRAM_OK;
        const Bf16Op a = split_operand({A, a_mn != 0, lda}, M, K, a_terms, ws->a, st);
        const Bf16Op b = split_operand({B, b_mn != 0, ldb}, N, K, b_terms, ws->b, st);
        gemm_bf16_terms(a, b, M, N, K, C, ldc, accumulate != 0, sms, st);
    }
    NGRAM_API_END
}
