"""Bank ingest: the reference's on-disk bank (save_bank, embedding.cpp:77-98)
streamed straight into the device bank (ngram_bank_load_file), and the row-sharded
bank layout.  The file is written by the reference itself when oracle/_ref is built,
and by a writer of the same byte format otherwise."""
import json
import os
import struct

import numpy as np
import pytest
import torch

import oracle as O
from helpers import dev_i64, dev_u32
from paper_2601_21204_b200 import ngram as G
from paper_2601_21204_b200.abi import ConfigError, IoError, ParseError

pytestmark = pytest.mark.gpu


def write_bank_file(path, cfg, hb):
    """u32 LE header length, config JSON, then raw LE f32 tensors (embedding.hpp:486-491)."""
    header = json.dumps(cfg, indent=2).encode()
    with open(path, "wb") as f:
        f.write(struct.pack("<I", len(header)))
        f.write(header)
        for a in [hb.base] + hb.sub + hb.proj:
            f.write(np.ascontiguousarray(a, "<f4").tobytes())
        if cfg["amplification"] == "layer_norm":
            f.write(hb.gain.astype("<f4").tobytes())
            f.write(hb.bias.astype("<f4").tobytes())


@pytest.fixture
def small(cuda, tmp_path):
    cfg = O.make_default_config(700, 256, 3, 2)
    cfg["amplification"] = "layer_norm"
    hb = O.make_bank(cfg, 77, round_bf16=True)
    path = str(tmp_path / "bank.bin")
    if O.ref_available():  # the reference's own save_bank
        R = O.ref()
        h = R.ref_bank_create(json.dumps(cfg).encode(), 77, 1)
        assert R.ref_bank_save(h, path.encode()) == 0
        R.ref_bank_destroy(h)
    else:
        write_bank_file(path, cfg, hb)
    return cfg, hb, path


def test_load_file_equals_upload(small, cuda):
    cfg, hb, path = small
    a = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj, hb.gain, hb.bias)
    b = G.DeviceBank(cfg).load_file(path)
    toks = dev_u32(torch, O.uniform_tokens(1, 700, 500), cuda)
    off = dev_i64(torch, [0, 200, 500], cuda)
    ra, ma = G.embed_forward(a, toks, off, merged=True)
    rb, mb = G.embed_forward(b, toks, off, merged=True)
    assert torch.equal(ra, rb) and torch.equal(ma, mb)


def test_load_file_errors(small, tmp_path):  # embedding.cpp:100-140 error behaviour
    cfg, hb, path = small
    data = open(path, "rb").read()
    bank = G.DeviceBank(cfg)
    with pytest.raises(IoError):
        bank.load_file(str(tmp_path / "missing.bin"))
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(data[:-64])
    with pytest.raises(ParseError):
        bank.load_file(str(trunc))
    longer = tmp_path / "long.bin"
    longer.write_bytes(data + b"\0")
    with pytest.raises(ParseError):
        bank.load_file(str(longer))
    short = tmp_path / "short.bin"
    short.write_bytes(data[:3])
    with pytest.raises(ParseError):
        bank.load_file(str(short))
    other = dict(cfg)
    other["amplification"] = "none"
    with pytest.raises(ConfigError):
        G.DeviceBank(other).load_file(path)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_row_shards_partition_every_table(cuda, P):
    """owner(b, h) = floor(h * P / V_b): the shards' row blocks tile [0, V_b) exactly."""
    cfg = O.make_default_config(300, 256, 4, 4)
    cfg["dim"] = 768
    V = [e["vocab"] for e in cfg["sub_vocab"]]
    los, his = [], []
    for r in range(P):
        info = G.DeviceBank(cfg, shard_rank=r, shard_count=P).info
        los.append([info.row_lo[b] for b in range(12)])
        his.append([info.row_hi[b] for b in range(12)])
    for b in range(12):
        assert los[0][b] == 0 and his[P - 1][b] == V[b]
        for r in range(1, P):
            assert los[r][b] == his[r - 1][b]
        for r in range(P):
            for h in (los[r][b], his[r][b] - 1):
                assert h * P // V[b] == r


def test_load_file_into_row_shards(small, cuda):  # ingest sliced per shard
    """Each shard bank streams only its row block of every sub-table from the same file; the
    sharded forward over those banks equals the unsharded forward bit for bit."""
    cfg, hb, path = small
    full = G.DeviceBank(cfg).load_file(path)
    P, nseq, L = 2, 4, 300  # T = 1200 > 1024: both sides in the prefill regime
    toks = O.uniform_tokens(9, cfg["base_vocab"], nseq * L)
    t_all, off_all = dev_u32(torch, toks, cuda), dev_i64(torch, np.arange(0, nseq * L + 1, L), cuda)
    ref, _ = G.embed_forward(full, t_all, off_all)
    per = nseq // P
    rank_tok = [r * per * L for r in range(P + 1)]
    banks = [G.DeviceBank(cfg, shard_rank=r, shard_count=P).load_file(path) for r in range(P)]
    groups = [G.ShardGroup(b, per * L) for b in banks]
    G.emulate_shards_single_process(groups)
    for g in groups:
        g.scatter(t_all, off_all, rank_tok)
    torch.cuda.synchronize()
    for r, g in enumerate(groups):
        rows, _ = g.project(t_all[rank_tok[r]:rank_tok[r + 1]])
        assert torch.equal(rows, ref[rank_tok[r]:rank_tok[r + 1]])
