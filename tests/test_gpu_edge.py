"""Edge cases of the reference semantics on the device path: the degenerate base-only
config (max_order == 1, config.hpp:21-24), empty and ragged sequences in one batch,
N=2 / K=1 shapes, the averaged variant with LayerNorm, and orders up to 8."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import assert_rows_close, dev_i64, dev_u32
from paper_2601_21204_b200 import ngram as G

pytestmark = pytest.mark.gpu


def _run(cfg, seed, seqs, cuda, priors=None):
    N = cfg["max_order"]
    hb = O.make_bank(cfg, seed, round_bf16=True)
    ln = cfg["amplification"] == "layer_norm"
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj, hb.gain if ln else None, hb.bias if ln else None)
    allt = np.concatenate([np.asarray(s, np.uint32) for s in seqs]) if sum(map(len, seqs)) else np.zeros(0, np.uint32)
    off = np.concatenate([[0], np.cumsum([len(s) for s in seqs])])
    prior = None
    if priors is not None and N > 1:
        pm = np.zeros((len(seqs), N - 1), np.uint32)
        for i, p in enumerate(priors):
            if len(p):
                pm[i, N - 1 - len(p[-(N - 1):]):] = p[-(N - 1):]
        prior = dev_u32(torch, pm, cuda)
    t = dev_u32(torch, allt if len(allt) else np.zeros(1, np.uint32), cuda)[:len(allt)]
    rows, merged = G.embed_forward(db, t, dev_i64(torch, off, cuda), prior=prior, merged=True)
    db.sync_errors()
    ref_r, ref_m = [], []
    for i, s in enumerate(seqs):
        if len(s) == 0:
            continue
        r, m = O.embed_sequence(hb, s, prior=None if priors is None else priors[i], double=True)
        ref_r.append(r)
        ref_m.append(m)
    return db, rows.cpu().numpy(), merged.cpu().numpy(), np.concatenate(ref_r), np.concatenate(ref_m)


def test_base_only_config(cuda):  # max_order == 1: E0 only, merge scale 1
    cfg = O.make_config(64, 16, 1, 1, [], "subtable_v2", "scale_sqrt_d")
    db, rows, merged, rr, rm = _run(cfg, 3, [[1, 2, 3], [63, 0]], cuda)
    assert db.B == 0
    assert np.array_equal(merged, rm.astype(np.float32))  # E0 rows exactly
    assert_rows_close(rows, rr)


def test_empty_and_ragged_sequences(cuda):
    cfg = O.make_default_config(300, 256, 3, 2)
    seqs = [[], O.uniform_tokens(1, 300, 5), [], O.uniform_tokens(2, 300, 1), O.uniform_tokens(3, 300, 333), []]
    priors = [[], [7], [], [1, 2], [5, 6, 7, 8], []]
    db, rows, merged, rr, rm = _run(cfg, 4, seqs, cuda, priors)
    assert rows.shape[0] == 339
    assert_rows_close(rows, rr)
    assert_rows_close(merged, rm)


def test_zero_tokens_is_a_no_op(cuda):
    cfg = O.make_default_config(300, 256, 3, 2)
    db = G.DeviceBank(cfg).generate(1)
    t = torch.zeros(0, dtype=torch.int32, device=cuda)
    rows, _ = G.embed_forward(db, t, dev_i64(torch, [0, 0], cuda))
    db.sync_errors()
    assert rows.shape == (0, 256)


@pytest.mark.parametrize("N,K,D", [(2, 1, 128), (2, 2, 256), (5, 2, 512), (8, 1, 448)])
def test_orders_and_sub_tables(cuda, N, K, D):
    cfg = O.make_default_config(200, D, N, K)
    seqs = [O.uniform_tokens(10 + N, 200, 400), O.uniform_tokens(20 + K, 200, 77)]
    db, rows, merged, rr, rm = _run(cfg, N * 10 + K, seqs, cuda)
    assert_rows_close(rows, rr)
    assert_rows_close(merged, rm)


def test_averaged_variant_with_layer_norm(cuda):
    cfg = O.make_config(100, 384, 3, 1, [1101, 1303], "averaged_v1", "layer_norm")
    db, rows, merged, rr, rm = _run(cfg, 5, [O.uniform_tokens(4, 100, 300)], cuda)
    assert_rows_close(merged, rm)
    assert_rows_close(rows, rr)


def test_decode_with_two_token_windows(cuda):  # N=2: the ring holds one token
    cfg = O.make_default_config(50, 128, 2, 1)
    hb = O.make_bank(cfg, 8, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    st = G.SequenceCache(db)
    seq = [3, 49, 0, 7, 7]
    for i, t in enumerate(seq):
        ids = st.append(t)
        assert ids == [int(x) for x in O.hash_sequence(cfg, seq[:i + 1])[-1]]
    assert list(st.ring()) == [7]
