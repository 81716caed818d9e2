"""The dense GEMM building block of the backward pass and PLNE (gemm_gen.cu) through the
C-ABI (ngram_gemm_f32): every operand layout (K-major / MN-major), term count (three bf16
terms = fp32-accurate, one term) and the fp32 CUDA-core path, against an fp64 torch product;
ragged shapes exercise the TMA out-of-bounds fill and the masked epilogue."""
import ctypes as C

import pytest
import torch

from paper_2601_21204_b200 import abi

pytestmark = pytest.mark.gpu


def _gemm(A, a_mn, B, b_mn, M, N, K, Cm, acc, at, bt):
    lda = A.shape[1]
    ldb = B.shape[1]
    abi.check(abi.lib().ngram_gemm_f32(0, M, N, K, C.c_void_p(A.data_ptr()), lda, int(a_mn), C.c_void_p(B.data_ptr()),
                                       ldb, int(b_mn), C.c_void_p(Cm.data_ptr()), Cm.shape[1], int(acc), at, bt,
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))


def _operand(R, K, mn, gen, bf16_exact=False):
    x = torch.randn((K, R) if mn else (R, K), generator=gen, device="cuda", dtype=torch.float32)
    if bf16_exact:
        x = x.bfloat16().float()
    logical = x.t() if mn else x  # [R][K]
    return x, logical.double()


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("terms", [(3, 1), (2, 1), (3, 3), (1, 3), (1, 1), (0, 0)])
def test_gemm_layouts_and_terms(cuda, a_mn, b_mn, terms):
    gen = torch.Generator(device="cuda").manual_seed(7)
    M, N, K = 520, 264, 392  # ragged in every dimension (tiles 256 x 256 x 64)
    at, bt = terms
    A, Ad = _operand(M, K, a_mn, gen, bf16_exact=(at == 1))
    B, Bd = _operand(N, K, b_mn, gen, bf16_exact=(bt == 1))
    C0 = torch.randn((M, N + 8), generator=gen, device="cuda")  # ldc > N
    Cm = C0.clone()
    _gemm(A, a_mn, B, b_mn, M, N, K, Cm, True, at, bt)
    torch.cuda.synchronize()
    ref = C0[:, :N].double() + Ad @ Bd.t()
    err = float((Cm[:, :N].double() - ref).norm() / ref.norm())
    assert err < (5e-6 if at == 2 else 1e-6), err  # two terms: a 17-bit operand
    assert torch.equal(Cm[:, N:], C0[:, N:]), "wrote past N"


@pytest.mark.parametrize("shape", [(3072, 3072, 8192), (8192, 3072, 3072)])
def test_gemm_backward_shapes(cuda, shape):
    """The config C backward shapes (dW: D x D x T with both operands MN-major, dX: T x D x D)
    at reduced T, U in three terms, X / W exact in bf16: fp32-accurate."""
    gen = torch.Generator(device="cuda").manual_seed(11)
    M, N, K = shape
    dw = M == N
    A, Ad = _operand(M, K, dw, gen)                     # U (MN-major for dW, K-major for dX)
    B, Bd = _operand(N, K, True, gen, bf16_exact=True)  # X / W_cat (MN-major)
    Cm = torch.zeros((M, N), device="cuda")
    _gemm(A, dw, B, True, M, N, K, Cm, False, 3, 1)
    torch.cuda.synchronize()
    ref = Ad @ Bd.t()
    err = float((Cm.double() - ref).norm() / ref.norm())
    assert err < 1e-6, err


def test_gemm_overwrite_and_empty(cuda):
    gen = torch.Generator(device="cuda").manual_seed(3)
    A, Ad = _operand(64, 0, False, gen)
    B, Bd = _operand(48, 0, False, gen)
    Cm = torch.full((64, 48), 5.0, device="cuda")
    _gemm(A, False, B, False, 64, 48, 0, Cm, False, 3, 3)  # K = 0, overwrite: zeros
    torch.cuda.synchronize()
    assert float(Cm.abs().max()) == 0.0
