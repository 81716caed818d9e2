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


@pytest.mark.parametrize("P,home", [(2, 96), (4, 80), (2, 40)])
def test_sharded_small_batch_follows_the_gathered_batch_regime(cuda, P, home):
    """A sharded projection of home_T rows runs the kernel regime of the GATHERED batch (the
    T the 1-GPU call sees): global 192 -> split-K sub-regime 2 although home 96 <= 128; global
    320 -> the pair GEMM although home 80 <= 256; global 80 -> sub-regime 1.  At D = 3072 the
    regimes split K differently, so only this choice keeps the result bit-identical."""
    cfg = O.make_default_config(1000, 3072, 4, 4)
    full = G.DeviceBank(cfg).generate(5)
    T = P * home
    toks = np.random.default_rng(T).integers(0, 1000, size=T).astype(np.uint32)
    prior = np.random.default_rng(8).integers(0, 1000, size=(T, 3)).astype(np.uint32)
    off = np.arange(0, T + 1)  # one token per stream (a decode step of T streams)
    t_all, off_all, pr_all = dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda), dev_u32(torch, prior, cuda)
    ref_rows, _ = G.embed_forward(full, t_all, off_all, prior=pr_all)
    rank_tok = [r * home for r in range(P + 1)]
    banks = [G.DeviceBank(cfg, shard_rank=r, shard_count=P).generate(5) for r in range(P)]
    groups = [G.ShardGroup(b, home) for b in banks]
    G.emulate_shards_single_process(groups)
    for g in groups:
        g.scatter(t_all, off_all, rank_tok, pr_all)
    torch.cuda.synchronize()
    for r, g in enumerate(groups):
        rows, _ = g.project(t_all[rank_tok[r]:rank_tok[r + 1]])
        assert torch.equal(rows, ref_rows[rank_tok[r]:rank_tok[r + 1]]), (P, home, r)
    banks[0].sync_errors()


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("mode", ["a2a", "rs"])
def test_nccl_exchange_variants_bit_identical_to_single_gpu(cuda, P, mode):
    """The NCCL forms of the exchange (include/ngram_b200.h): all-to-all of the owned rows
    (compact, slots derived from the receiver's own ids) and reduce-scatter of the -0.0-padded X.
    The collective is emulated in-process (slices / an fp32 sum of the chunks, which is what NCCL's
    bf16 sum computes for one real value plus -0.0 pads); ranks hold unequal numbers of tokens."""
    cfg = O.make_default_config(4000, 768, 4, 4)
    full = G.DeviceBank(cfg).generate(13)
    rng = np.random.default_rng(P)
    lens = [int(x) for x in rng.integers(1, 400, size=2 * P)]
    toks = rng.integers(0, 4000, size=sum(lens)).astype(np.uint32)
    off = np.concatenate([[0], np.cumsum(lens)])
    prior = rng.integers(0, 4000, size=(len(lens), 3)).astype(np.uint32)
    t_all, off_all, pr_all = dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda), dev_u32(torch, prior, cuda)
    ref_rows, _ = G.embed_forward(full, t_all, off_all, prior=pr_all)
    rank_tok = [int(off[2 * r]) for r in range(P)] + [int(off[-1])]  # two sequences per rank
    max_home = max(rank_tok[r + 1] - rank_tok[r] for r in range(P))
    banks = [G.DeviceBank(cfg, shard_rank=r, shard_count=P).generate(13) for r in range(P)]
    groups = [G.ShardGroup(b, max_home) for b in banks]
    for step in range(2):  # both halves of the double-buffered X
        if mode == "a2a":
            counts = [g.xchg_prepare(t_all, off_all, rank_tok, pr_all) for g in groups]
            sends = []
            for g, (snd, rcv) in zip(groups, counts):
                s = torch.empty((int(snd.sum()), 64), dtype=torch.bfloat16, device=cuda)
                g.xchg_pack(s)
                sends.append(s)
            for p, g in enumerate(groups):
                parts = []
                for r in range(P):
                    snd = counts[r][0]
                    assert snd[p] == counts[p][1][r]  # what r sends p is what p expects from r
                    a = int(snd[:p].sum())
                    parts.append(sends[r][a:a + int(snd[p])])
                g.xchg_unpack(torch.cat(parts).contiguous())
        else:
            sends = []
            for g in groups:
                s = torch.empty((P * max_home, 768), dtype=torch.bfloat16, device=cuda)
                g.pack_padded(t_all, off_all, rank_tok, s, pr_all)
                sends.append(s)
            for p, g in enumerate(groups):
                chunk = torch.stack([s[p * max_home:(p + 1) * max_home].float() for s in sends]).sum(0)
                g.home_x().copy_(chunk.to(torch.bfloat16))
        torch.cuda.synchronize()
        for r, g in enumerate(groups):
            rows, _ = g.project(t_all[rank_tok[r]:rank_tok[r + 1]])
            assert torch.equal(rows, ref_rows[rank_tok[r]:rank_tok[r + 1]]), (mode, P, r, step)
    banks[0].sync_errors()
