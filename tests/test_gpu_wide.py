"""The fused wide-tile prefill kernel (gemm_wide.cu: hash + tile::gather4 into resident A
slots + every N-tile of an m-block on one CTA pair, direct-register epilogue), the opt-in
prefill path for D <= 768 on tensor-core banks (NGRAM_PREFILL_PATH=wide).

Checked (a) against the oracle's double path (the reference's arithmetic, embedding.hpp:163-201
+ amplify :239-287) within the tensor-core tolerance of tests/helpers.py, and (b) bit for bit
against the X path (K1+K2 kernel -> X -> pair kernel; NGRAM_PREFILL_PATH, read per call).  Covers D = 256 / 512 / 768, d = 64 / 128, ragged T
(partial m-blocks, rows past T never stored), several m-blocks per CTA pair, carried prior
context, every amplification, bf16 output, rows + merged, and an out-of-range token."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import assert_rows_close, dev_i64, dev_u32
from paper_2601_21204_b200 import ngram as G
from paper_2601_21204_b200.abi import OutOfRange

pytestmark = pytest.mark.gpu

# (V0, D, N, K, amplification, seq lengths, seed)
CASES = {
    "d768_sqrt": (3000, 768, 4, 4, "scale_sqrt_d", [1001, 2900, 7, 513], 3),
    "d512_d128_none": (2000, 512, 3, 2, "none", [600, 1700], 5),
    "d256_ln": (1500, 256, 3, 2, "layer_norm", [300, 1029], 7),
    "d768_n5_k3": (2500, 768, 5, 3, "scale_sqrt_d", [700, 333], 9),   # order-5 windows, 12 branches
    "d512_n2_k8": (1200, 512, 2, 8, "none", [900, 41], 11),           # bigrams only, 8 sub-tables
}


@pytest.fixture
def path(monkeypatch):
    """Select the prefill path for the calls of one test (the library reads
    NGRAM_PREFILL_PATH per call)."""
    def use(name):
        monkeypatch.setenv("NGRAM_PREFILL_PATH", name)
    use("wide")
    return use


def _case(case, cuda):
    V0, D, N, K, amp, lens, seed = CASES[case]
    cfg = O.make_default_config(V0, D, N, K)
    cfg["amplification"] = amp
    hb = O.make_bank(cfg, seed, round_bf16=True)
    ln = amp == "layer_norm"
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj, hb.gain if ln else None, hb.bias if ln else None)
    seqs = [O.uniform_tokens(seed * 10 + i, V0, n) for i, n in enumerate(lens)]
    toks = np.concatenate(seqs)
    off = np.concatenate([[0], np.cumsum(lens)])
    prior = np.zeros((len(lens), N - 1), np.uint32)
    prior[1] = np.arange(1, N) * 7
    args = (dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda))
    return hb, db, seqs, prior, args


@pytest.mark.parametrize("case", list(CASES))
def test_wide_kernel_matches_oracle(cuda, path, case):
    hb, db, seqs, prior, (t, o) = _case(case, cuda)
    rows, merged = G.embed_forward(db, t, o, merged=True, prior=dev_u32(torch, prior, cuda))
    db.sync_errors()
    refs = [O.embed_sequence(hb, s, double=True, prior=prior[i] if i == 1 else None) for i, s in enumerate(seqs)]
    assert_rows_close(rows.cpu().numpy(), np.concatenate([r for r, _ in refs]))
    assert_rows_close(merged.cpu().numpy(), np.concatenate([m for _, m in refs]))
    db.close()


@pytest.mark.parametrize("case,dtype", [("d768_sqrt", torch.float32), ("d768_sqrt", torch.bfloat16),
                                        ("d512_d128_none", torch.float32), ("d256_ln", torch.float32),
                                        ("d768_n5_k3", torch.float32), ("d512_n2_k8", torch.bfloat16)])
def test_wide_kernel_bit_identical_to_x_path(cuda, path, case, dtype):
    _, db, _, prior, (t, o) = _case(case, cuda)
    pr = dev_u32(torch, prior, cuda)
    outs = []
    for name in ("wide", "x"):
        path(name)
        r, m = G.embed_forward(db, t, o, merged=True, prior=pr, out_dtype=dtype)
        db.sync_errors()
        outs.append(torch.stack([r, m]))
    assert torch.equal(outs[0], outs[1])
    path("wide")
    r1, _ = G.embed_forward(db, t, o, merged=False, prior=pr, out_dtype=dtype)  # rows-only kernel form
    db.sync_errors()
    assert torch.equal(r1, outs[0][0])
    db.close()


def test_wide_kernel_many_m_blocks_per_pair(cuda, path):
    """T = 40 000 at D = 768: 157 m-blocks over 74 CTA pairs (every pair refills its resident A
    slots at least twice); rows compared with the X path's bits on a sample and against the
    oracle on sampled rows."""
    V0, D = 5000, 768
    cfg = O.make_default_config(V0, D, 4, 4)
    hb = O.make_bank(cfg, 41, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    toks = O.uniform_tokens(77, V0, 40000)
    rows, _ = G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, [0, 40000], cuda))
    db.sync_errors()
    path("x")
    xrows, _ = G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, [0, 40000], cuda))
    db.sync_errors()
    assert torch.equal(rows, xrows)
    path("wide")
    for a, b in [(0, 300), (19900, 20300), (39700, 40000)]:
        ref, _ = O.embed_sequence(hb, toks[max(0, a - 3):b], double=True)
        assert_rows_close(rows[a:b].cpu().numpy(), ref[a - max(0, a - 3):])
    # same rows computed as separate sequences with their prior carried: identical bits
    prior = dev_u32(torch, toks[19997:20000].reshape(1, 3), cuda)
    part, _ = G.embed_forward(db, dev_u32(torch, toks[20000:], cuda), dev_i64(torch, [0, 20000], cuda), prior=prior)
    db.sync_errors()
    assert torch.equal(part, rows[20000:])
    db.close()


def test_wide_kernel_out_of_range_token_writes_nothing(cuda, path):
    cfg = O.make_default_config(3000, 768, 4, 4)
    hb = O.make_bank(cfg, 3, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    toks = O.uniform_tokens(5, 3000, 2000)
    toks[1777] = 3000
    out = torch.full((2000, 768), 3.0, device=cuda)
    G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, [0, 1000, 2000], cuda), out_rows=out)
    with pytest.raises(OutOfRange):
        db.sync_errors()
    assert (out == 3.0).all()
    toks[1777] = 2999  # the bank is usable afterwards
    G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, [0, 1000, 2000], cuda), out_rows=out)
    db.sync_errors()
    assert not (out == 3.0).all()
    db.close()
