"""Seeded random sweep over the forward's shape space against the oracle's double path
(embed_sequence_cached, embedding.hpp:383-436): model widths on and off the tensor-core tiles,
orders 2..5, 1..4 sub-tables per order, every amplification, ragged multi-sequence batches of
1..3000 tokens (so every path selection -- split-K small T, the one-wave 128 x 128 tiles, the
pair kernel, the CUDA-core kernels -- is crossed), a carried prior on one sequence, and bf16 as
well as fp32 output.  Tolerance: tests/helpers.py (bit-exact where the CUDA-core kernels keep
the reference's float order is covered elsewhere)."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import assert_rows_close, dev_i64, dev_u32
from paper_2601_21204_b200 import ngram as G

pytestmark = pytest.mark.gpu

_rng = np.random.default_rng(20261019)
CASES = []
for i in range(14):
    N = int(_rng.integers(2, 6))
    K = int(_rng.integers(1, 5))
    B = (N - 1) * K
    d = int(_rng.choice([16, 32, 64, 128, 256]))
    D = B * d
    if D > 3072:
        d = max(16, (3072 // B) // 16 * 16)
        D = B * d
    V0 = int(_rng.integers(50, 4000))
    amp = str(_rng.choice(["none", "scale_sqrt_d", "layer_norm"]))
    nseq = int(_rng.integers(1, 5))
    lens = [int(x) for x in _rng.integers(1, 3000 // nseq + 1, size=nseq)]
    bf16 = bool(_rng.integers(0, 2))
    CASES.append((i, V0, D, N, K, amp, lens, bf16))
# wide models across the regime boundaries (T = 200 / 700 / 1100 / 2600 around 256, 768, 1024)
CASES += [(14, 900, 3072, 4, 4, "scale_sqrt_d", [150, 50], False), (15, 700, 3072, 4, 4, "none", [400, 300], True),
          (16, 1100, 1536, 5, 3, "layer_norm", [600, 500], False), (17, 500, 2048, 3, 4, "scale_sqrt_d", [2000, 600], False)]


@pytest.mark.parametrize("case", CASES, ids=[f"c{c[0]}_D{c[2]}_N{c[3]}_K{c[4]}_T{sum(c[6])}" for c in CASES])
def test_random_shape_matches_oracle(cuda, case):
    i, V0, D, N, K, amp, lens, bf16 = case
    cfg = O.make_default_config(V0, D, N, K)
    cfg["amplification"] = amp
    hb = O.make_bank(cfg, 100 + i, round_bf16=True)
    ln = amp == "layer_norm"
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj, hb.gain if ln else None, hb.bias if ln else None)
    seqs = [O.uniform_tokens(1000 * i + j, V0, n) for j, n in enumerate(lens)]
    toks = np.concatenate(seqs)
    off = np.concatenate([[0], np.cumsum(lens)])
    prior = np.zeros((len(lens), max(N - 1, 1)), np.uint32)
    prior[-1] = (np.arange(max(N - 1, 1)) * 13 + 5) % V0
    out_dtype = torch.bfloat16 if bf16 else torch.float32
    rows, merged = G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda), merged=True,
                                   prior=dev_u32(torch, prior, cuda), out_dtype=out_dtype)
    db.sync_errors()
    refs = [O.embed_sequence(hb, s, double=True, prior=prior[j] if j == len(lens) - 1 else None)
            for j, s in enumerate(seqs)]
    assert_rows_close(rows.float().cpu().numpy(), np.concatenate([r for r, _ in refs]), bf16=bf16)
    assert_rows_close(merged.float().cpu().numpy(), np.concatenate([m for _, m in refs]), bf16=bf16)
    db.close()
