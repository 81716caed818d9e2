"""Row-sharded multi-GPU data path, emulated in one process on one GPU:
P shard banks (each holding only its row block of every sub-table) scatter their owned
rows into every rank's home X through the same kernel the multi-process path runs over
NVLink, then each rank projects its home tokens.  The sharded output must be
bit-identical to the single-GPU forward (rows are exchanged raw)."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import dev_i64, dev_u32
from paper_2601_21204_b200 import ngram as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("amp", ["scale_sqrt_d", "layer_norm"])
def test_sharded_forward_bit_identical_to_single_gpu(cuda, P, amp):
    cfg = O.make_default_config(4000, 768, 4, 4)  # config B shape, reduced vocabulary
    cfg["amplification"] = amp
    full = G.DeviceBank(cfg).generate(99)
    nseq, L = 8, 700
    toks = np.random.default_rng(P).integers(0, 4000, size=nseq * L).astype(np.uint32)
    prior = np.random.default_rng(7).integers(0, 4000, size=(nseq, 3)).astype(np.uint32)
    off = np.arange(0, nseq * L + 1, L)
    t_all, off_all, pr_all = dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda), dev_u32(torch, prior, cuda)
    ref_rows, ref_merged = G.embed_forward(full, t_all, off_all, prior=pr_all, merged=True)
    per = nseq // P
    rank_tok = [r * per * L for r in range(P + 1)]
    banks = [G.DeviceBank(cfg, shard_rank=r, shard_count=P).generate(99) for r in range(P)]
    groups = [G.ShardGroup(b, per * L) for b in banks]
    G.emulate_shards_single_process(groups)
    for step in range(2):  # two steps exercise both halves of the double-buffered X
        for g in groups:
            g.scatter(t_all, off_all, rank_tok, pr_all)
        torch.cuda.synchronize()  # stands in for the cross-rank barrier
        for r, g in enumerate(groups):
            rows, merged = g.project(t_all[rank_tok[r]:rank_tok[r + 1]], merged=True)
            assert torch.equal(rows, ref_rows[rank_tok[r]:rank_tok[r + 1]]), (P, r, step)
            assert torch.equal(merged, ref_merged[rank_tok[r]:rank_tok[r + 1]])
        banks[0].sync_errors()
