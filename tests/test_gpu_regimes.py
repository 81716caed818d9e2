"""Parity on the regimes and banks the first golden set did not reach (tests/golden/make_golden.py
sections 12-17, all produced by the reference itself through oracle/_ref):

* the split-K small-T GEMM's second sub-regime (128 < T <= 256) at D = 3072: prefill calls of
  T = 129 / 200 / 256, a 64 x 4 verify block + commit (config E's shape) and a 256-stream decode
  step (config D's largest batch), against embed_sequence<double> and the reference's
  sequence_cache + draft_verify;
* config A's and config B's ACTUAL banks (make_bank(make_default_config(...), 1234)), not
  reduced-vocabulary stand-ins: config A over its full 4 x 512 batch, config B at 128 sampled
  positions of its full 16 x 4096 prefill;
* the Barrett fast path of K1 at its edge: V0 = 2^32 - 5 and moduli in (2^31, 2^32], where the
  modular products approach 2^64.

Tolerance: tests/helpers.py (per-row max |err| <= 1e-5 * max|row|, relL2 <= 1e-6, fp32 out).
Ids and rings: bit-exact."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
from helpers import assert_rows_close, dev_i64, dev_u32, gold, gold_config, u64
from paper_2601_21204_b200 import ngram as G

pytestmark = pytest.mark.gpu


def _bank(cfg, seed):
    hb = O.make_bank(cfg, seed, round_bf16=True)
    return hb, G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)


def _rings(pref, lens, n1):
    """The ring a sequence_cache holds after appending each stream's prefix (cache.cpp:49-52)."""
    ring = np.zeros((len(lens), n1), np.uint32)
    for s, l in enumerate(lens):
        tail = pref[s, :l][-n1:]
        if len(tail):
            ring[s, n1 - len(tail):] = tail
    return ring


# ---------------------------------------------------------------------------------- section 12
def test_split_k_second_sub_regime_d3072_prefix_calls(cuda):
    g = gold("regime2_d3072.npz")
    cfg = gold_config(g)
    hb, db = _bank(cfg, int(g["seed"]))
    assert O.bank_checksum(hb) == int(g["bank_checksum"])  # the reference's bank, value for value
    toks = g["tokens"]
    for T in (129, 200, 256):  # 128 < T <= 256: two m-tiles, half the splits
        rows, _ = G.embed_forward(db, dev_u32(torch, toks[:T], cuda), dev_i64(torch, [0, T], cuda))
        db.sync_errors()
        assert_rows_close(rows.cpu().numpy(), g["rows_f64_f32"][:T])
    # and the same rows out of one T = 256 call split into ragged sequences with carried context
    cut = [0, 1, 100, 129, 256]
    prior = np.zeros((4, 3), np.uint32)
    for i in range(1, 4):
        a = cut[i]
        prior[i, 3 - min(3, a):] = toks[max(0, a - 3):a]
    rows, _ = G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, cut, cuda),
                              prior=dev_u32(torch, prior, cuda))
    db.sync_errors()
    assert_rows_close(rows.cpu().numpy(), g["rows_f64_f32"])


# ---------------------------------------------------------------------------------- section 13
def test_verify_commit_64x4_d3072_matches_reference_draft_verify(cuda):
    g = gold("verify_d3072_64x4.npz")
    cfg = gold_config(g)
    hb, db = _bank(cfg, int(g["seed"]))
    n, L = g["draft"].shape
    st = G.DecodeState(db, n, max_draft=L)
    st.reset(dev_u32(torch, _rings(g["prefix"], g["prefix_len"], 3), cuda),
             dev_i64(torch, g["prefix_len"], cuda))
    draft = dev_u32(torch, g["draft"], cuda)
    out = st.verify(draft)
    st.commit(draft, torch.from_numpy(g["accept"].astype(np.int32)).to(cuda))
    db.sync_errors()
    acc = g["accept"]
    got = np.concatenate([out[s, :acc[s]].cpu().numpy() for s in range(n)])
    assert got.shape == g["accepted"].shape
    assert_rows_close(got, g["accepted"])  # the reference's float path
    ring, length, last = st.state()
    assert np.array_equal(ring, g["ring"])
    assert np.array_equal(length, g["length"]) and np.array_equal(last, g["last"])
    # the accepted rows are the memo hits: recomputing them as decode steps gives the same bits
    st.close()


# ---------------------------------------------------------------------------------- section 14
def test_decode_step_256_streams_d3072_matches_reference(cuda):
    g = gold("decode_d3072_b256.npz")
    cfg = gold_config(g)
    hb, db = _bank(cfg, int(g["seed"]))
    n = len(g["token"])
    st = G.DecodeState(db, n, max_draft=1)
    st.reset(dev_u32(torch, _rings(g["prefix"], g["prefix_len"], 3), cuda), dev_i64(torch, g["prefix_len"], cuda))
    ids, merged = st.step(dev_u32(torch, g["token"], cuda))
    db.sync_errors()
    assert_rows_close(merged.cpu().numpy(), g["merged"])
    ring, length, last = st.state()
    assert np.array_equal(ring, g["ring"])
    assert np.array_equal(length, g["length"]) and np.array_equal(last, g["last"])
    # ids == the reference hash of each stream's window (prefix ++ token)
    want = np.stack([O.hash_sequence(cfg, list(g["prefix"][s, :g["prefix_len"][s]]) + [int(g["token"][s])])[-1]
                     for s in range(0, n, 17)])
    assert np.array_equal(u64(ids)[::17], want)
    st.close()


# ---------------------------------------------------------------------------------- section 15
def test_config_a_actual_bank_full_batch(cuda):
    g = gold("cfgA_bank_embed.npz")
    cfg = gold_config(g)
    hb, db = _bank(cfg, int(g["seed"]))
    assert O.bank_checksum(hb) == int(g["bank_checksum"])
    toks = g["tokens"]
    L = int(g["seq_len"])
    rows, _ = G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, np.arange(0, len(toks) + 1, L), cuda))
    db.sync_errors()
    assert_rows_close(rows.cpu().numpy(), g["rows_f64_f32"])
    # host-buffer entry (the drop-in embed_sequence path) gives the same bits
    host, _ = G.embed_batch_host(db, [toks[i:i + L] for i in range(0, len(toks), L)])
    assert np.array_equal(host, rows.cpu().numpy())


# ---------------------------------------------------------------------------------- section 16
def _cudart():
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            lib = C.CDLL(name)
            lib.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
            return lib
        except OSError:
            continue
    import glob
    import os
    for p in glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                    "libcudart.so*")):
        lib = C.CDLL(p)
        lib.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
        return lib
    pytest.fail("libcudart not found")


def _write(rt, dst, src_u16):
    """Device bytes at `dst` <- the bf16 bit patterns (host, contiguous)."""
    a = np.ascontiguousarray(src_u16, np.uint16)
    assert rt.cudaMemcpy(C.c_void_p(dst), a.ctypes.data, a.nbytes, 1) == 0  # cudaMemcpyHostToDevice


def test_config_b_actual_bank_sampled_positions(cuda):
    """Config B's own bank (2.31 B params; 9.2 GB as the reference's float bank) cannot be rebuilt
    in a test, so the device bank is generated and then every row the sampled positions read --
    their E0 rows, their 12 sub-table rows and the full projections -- is overwritten with the
    reference bank's values.  The forward then runs the real config-B prefill (16 x 4096 tokens
    in one launch, the production K1+K2 -> K3 path) and the sampled rows are compared."""
    g = gold("cfgB_sampled.npz")
    cfg = gold_config(g)
    db = G.DeviceBank(cfg).generate(99)
    assert db.tensor_core_path
    info = db.info
    D, B = db.D, db.B
    d = D // B
    rt = _cudart()
    torch.cuda.synchronize()
    toks, pos, ids = g["tokens"], g["positions"], g["ids"]
    e0 = g["e0_rows_bf16"]
    for i, p in enumerate(pos):
        _write(rt, info.e0_ptr + int(toks[p]) * D * 2, e0[i])
    row_base = np.concatenate([[0], np.cumsum([info.sub_vocab[b] for b in range(B)])])
    for i in range(len(pos)):
        for b in range(B):
            _write(rt, info.sub_ptr + (int(row_base[b]) + int(ids[i, b])) * d * 2, g["sub_rows_bf16"][i, b])
    proj = g["proj_bf16"].reshape(B, D, d)  # W_b[i][j] -> W_cat[i][b*d + j]
    _write(rt, info.wcat_ptr, np.ascontiguousarray(proj.transpose(1, 0, 2)).reshape(D, D))
    # the ids the device computes are the reference's (bit-exact), so the patched rows are the ones read
    off = g["seq_offsets"]
    dids = G.hash_ids(db, dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda))
    assert np.array_equal(u64(dids)[pos], ids)
    rows, merged = G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda), merged=True)
    db.sync_errors()
    assert_rows_close(rows[torch.from_numpy(pos).to(cuda)].cpu().numpy(), g["rows_f64_f32"])
    assert_rows_close(merged[torch.from_numpy(pos).to(cuda)].cpu().numpy(), g["merged_f64_f32"])


# ---------------------------------------------------------------------------------- section 17
def test_barrett_fast_path_at_the_2pow32_edge(cuda):
    g = gold("barrett_edge_ids.npz")
    cfg = gold_config(g)
    assert max(e["vocab"] for e in cfg["sub_vocab"]) == 1 << 32  # fast path: every modulus <= 2^32
    db = G.DeviceBank(cfg, tables=False)
    ids = G.hash_ids(db, dev_u32(torch, g["tokens"], cuda), dev_i64(torch, g["seq_offsets"], cuda))
    db.sync_errors()
    assert np.array_equal(u64(ids), g["ids"])
    # the host-buffer entry (the drop-in hash_all_orders path) agrees
    from paper_2601_21204_b200 import abi
    toks, off = np.ascontiguousarray(g["tokens"]), np.ascontiguousarray(g["seq_offsets"])
    host = np.zeros_like(g["ids"])
    abi.check(abi.lib().ngram_hash_ids_host(db.handle, toks.ctypes.data, off.ctypes.data, len(off) - 1, None,
                                            host.ctypes.data))
    assert np.array_equal(host, g["ids"])
