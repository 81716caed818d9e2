// gemm.hpp -- the host side of the dense GEMMs of the backward pass and PLNE (gemm_gen.cu):
// tensor maps for bf16 term operands, the fp32 -> bf16 three-term split, and the fp32
// CUDA-core path.  Convention: C[M][N] (+)= sum_k A(m, k) B(n, k); an operand is a logical
// [R][K] matrix stored K-major (element (r, k) at p[r * ld + k]) or MN-major (at p[k * ld + r]).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "bank.hpp"

namespace ngh {

struct F32Op {
    const float* p;
    bool mn;
    int64_t ld;
};

// Up to three bf16 terms sharing one layout (an exact bf16 operand has one term).
struct Bf16Op {
    const __nv_bfloat16* t[3];
    int terms;
    bool mn;
    int64_t ld;
};

// Workspace of the fp32 -> three-term split (grown on demand, owned by the caller).
struct SplitWs {
    DevBuf<__nv_bfloat16> a, b;
};

// Tensor-core GEMM over pre-split (or exact) bf16 terms.
void gemm_bf16_terms(const Bf16Op& A, const Bf16Op& B, int64_t M, int64_t N, int64_t K, float* C, int64_t ldc,
                     bool accumulate, int num_sms, cudaStream_t st);

// fp32 operands.  split3 = true: both operands split into three bf16 terms on the device, six
// tensor-core products in fp32 (fp32-accurate); false: the CUDA-core fp32 GEMM (pedantic).
void gemm_f32(const F32Op& A, const F32Op& B, int64_t M, int64_t N, int64_t K, float* C, int64_t ldc,
              bool accumulate, bool split3, SplitWs& ws, int num_sms, cudaStream_t st);

// Split an fp32 operand (logical [R][K], layout as given) into `terms` bf16 terms stored in the
// same orientation with a TMA-friendly pitch; returns the bf16 operand.
Bf16Op split_operand(const F32Op& X, int64_t R, int64_t K, int terms, DevBuf<__nv_bfloat16>& buf, cudaStream_t st);

}  // namespace ngh
