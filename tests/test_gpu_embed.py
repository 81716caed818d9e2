"""Forward parity (K1 + K2 + K3 / CUDA-core paths) through the C-ABI against the
reference's own outputs (tests/golden, produced by oracle/_ref) and the pinned oracle.
Mirrors proj/tests/test_embedding.cpp where a case has a device analogue.

Tolerance (tensor-core path, stated in tests/helpers.py): vs the reference's double
path on the same bf16-representable bank, per-row max |err| <= 1e-5 * max|row| and
relL2 <= 1e-6 (fp32 out); bf16 out additionally 2^-8 relative per element.  The
CUDA-core paths keep the reference's float operation order and are checked bit-exact."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import assert_rows_close, bf16_to_f32, dev_i64, dev_u32, gold, gold_config
from paper_2601_21204_b200 import ngram as G
from paper_2601_21204_b200.abi import InvalidArgument, OutOfRange

pytestmark = pytest.mark.gpu


def _bank(g, cuda, cfg=None):
    cfg = cfg or gold_config(g)
    hb = O.make_bank(cfg, int(g["seed"]), round_bf16=True)
    if "ln_gain" in g.files:
        hb.gain[:] = g["ln_gain"]
        hb.bias[:] = g["ln_bias"]
    ln = cfg["amplification"] == "layer_norm"
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj, hb.gain if ln else None, hb.bias if ln else None)
    return hb, db


def _forward(db, g, cuda, out_dtype=torch.float32):
    toks = g["tokens"]
    off = g["seq_offsets"]
    prior = None
    if "prior1" in g.files:
        p = np.zeros((len(off) - 1, db.N - 1), np.uint32)
        p[1, -len(g["prior1"]):] = g["prior1"]
        prior = dev_u32(torch, p, cuda)
    rows, merged = G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda), prior=prior,
                                   rows=True, merged=True, out_dtype=out_dtype)
    db.sync_errors()
    cv = (lambda t: t.float().cpu().numpy()) if out_dtype == torch.bfloat16 else (lambda t: t.cpu().numpy())
    return cv(rows), cv(merged)


@pytest.mark.parametrize("amp", ["none", "scale_sqrt_d", "layer_norm"])
def test_tensor_core_path_matches_reference(cuda, amp):  # embed_sequence_cached, every amplification
    g = gold(f"embed_tc_{amp}.npz")
    hb, db = _bank(g, cuda)
    assert db.tensor_core_path
    rows, merged = _forward(db, g, cuda)
    assert_rows_close(merged, g["merged_f64"])
    assert_rows_close(rows, g["rows_f64"])
    # and against the reference's own float path (it differs from double by ~1e-7)
    assert_rows_close(rows, g["rows_f32"])


@pytest.mark.parametrize("amp", ["none", "scale_sqrt_d", "layer_norm"])
def test_tensor_core_path_bf16_out(cuda, amp):
    g = gold(f"embed_tc_{amp}.npz")
    hb, db = _bank(g, cuda)
    rows, merged = _forward(db, g, cuda, torch.bfloat16)
    assert_rows_close(rows, g["rows_f64"], bf16=True)
    assert_rows_close(merged, g["merged_f64"], bf16=True)


@pytest.mark.parametrize("name", ["embed_simt_v2.npz", "embed_simt_v2_k1.npz", "embed_v1.npz", "embed_v1_wide.npz"])
def test_cuda_core_paths_bitexact_vs_reference_float(cuda, name):
    g = gold(name)
    hb, db = _bank(g, cuda)
    assert not db.tensor_core_path
    rows, merged = _forward(db, g, cuda)
    assert np.array_equal(merged, g["merged_f32"])
    assert np.array_equal(rows, g["rows_f32"])


def test_longcat_width_d3072_matches_reference(cuda):  # D=3072, N=4, K=4: the full K=3072 contraction
    g = gold("embed_d3072.npz")
    hb, db = _bank(g, cuda)
    rows, merged = _forward(db, g, cuda)
    assert_rows_close(merged, g["merged_f64"])
    assert_rows_close(rows, g["rows_f64"])


def test_first_row_uses_zero_padded_window(cuda):  # test_embedding.cpp:143-153
    cfg = O.make_default_config(1000, 256, 4, 2)
    cfg["dim"] = 384  # (N-1)K = 6 -> d = 64, tensor-core shape with a 128-wide N tile
    hb = O.make_bank(cfg, 7, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    rows, _ = G.embed_forward(db, dev_u32(torch, [9], cuda), dev_i64(torch, [0, 1], cuda))
    padded, _ = G.embed_forward(db, dev_u32(torch, [9], cuda), dev_i64(torch, [0, 1], cuda),
                                prior=dev_u32(torch, np.zeros((1, 3), np.uint32), cuda))
    assert torch.equal(rows, padded)
    ref, _ = O.embed_sequence(hb, [9], double=True)
    assert_rows_close(rows.cpu().numpy(), ref)


def test_split_with_carried_context_equals_whole_sequence(cuda):  # test_embedding.cpp:155-174, bit-exact
    g = gold("embed_tc_scale_sqrt_d.npz")
    hb, db = _bank(g, cuda)
    seq = O.uniform_tokens(5, 1000, 700)
    whole, _ = G.embed_forward(db, dev_u32(torch, seq, cuda), dev_i64(torch, [0, 700], cuda))
    for cut in (1, 7, 255, 256, 513):
        prior = np.zeros((2, 2), np.uint32)
        prior[1, -min(2, cut):] = seq[max(0, cut - 2):cut]
        parts, _ = G.embed_forward(db, dev_u32(torch, seq, cuda), dev_i64(torch, [0, cut, 700], cuda),
                                   prior=dev_u32(torch, prior, cuda))
        assert torch.equal(whole, parts), cut


def test_row_results_independent_of_batch_composition(cuda):
    """Each row's arithmetic depends only on its own ids within a regime: bit-identical for
    T > 256 (prefill GEMM) and within T <= 256 (split-K small-batch GEMM); across the two
    regimes the K summation order differs and results agree within the stated tolerance."""
    g = gold("embed_tc_none.npz")
    hb, db = _bank(g, cuda)
    seqs = [O.uniform_tokens(s, 1000, n) for s, n in [(1, 300), (2, 17), (3, 512), (4, 1)]]
    allt = np.concatenate(seqs)
    off = np.concatenate([[0], np.cumsum([len(s) for s in seqs])])
    batch, _ = G.embed_forward(db, dev_u32(torch, allt, cuda), dev_i64(torch, off, cuda))
    small = []
    for i, s in enumerate(seqs):
        alone, _ = G.embed_forward(db, dev_u32(torch, s, cuda), dev_i64(torch, [0, len(s)], cuda))
        if len(s) > 256:
            assert torch.equal(alone, batch[off[i]:off[i + 1]])
        else:
            assert_rows_close(alone.cpu().numpy(), batch[off[i]:off[i + 1]].cpu().numpy())
            small.append(alone)
    # both small sequences in one small call == each alone (same regime)
    both, _ = G.embed_forward(db, dev_u32(torch, np.concatenate([seqs[1], seqs[3]]), cuda),
                              dev_i64(torch, [0, 17, 18], cuda))
    assert torch.equal(both, torch.cat(small))
    again, _ = G.embed_forward(db, dev_u32(torch, allt, cuda), dev_i64(torch, off, cuda))
    assert torch.equal(batch, again)  # deterministic


def test_split_k_sub_regimes_are_batch_composition_invariant(cuda):
    """The split-K small-batch GEMM has two sub-regimes (T <= 128 and 128 < T <= 256: the split
    count depends on D and the sub-regime only).  Within each, a row's result does not depend on
    the batch; across them, the K summation order differs (tolerance)."""
    g = gold("embed_tc_none.npz")
    hb, db = _bank(g, cuda)
    a, b, c = (O.uniform_tokens(s, 1000, n) for s, n in [(11, 140), (12, 60), (13, 30)])

    def fwd(*parts):
        toks = np.concatenate(parts)
        o = np.concatenate([[0], np.cumsum([len(q) for q in parts])])
        out, _ = G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, o, cuda))
        return out

    alone_a = fwd(a)                                       # T = 140
    assert torch.equal(fwd(a, b)[:140], alone_a)           # T = 200, same sub-regime
    alone_c = fwd(c)                                       # T = 30
    assert torch.equal(fwd(c, b)[:30], alone_c)            # T = 90, same sub-regime
    assert_rows_close(fwd(c, a)[:30].cpu().numpy(), alone_c.cpu().numpy())  # T = 170: other sub-regime


def test_zero_bank_embeds_to_zero(cuda):  # test_embedding.cpp:176-181
    cfg = O.make_default_config(64, 256, 3, 2)
    cfg["amplification"] = "none"
    hb = O.make_bank(cfg, 1)
    for a in [hb.base] + hb.sub + hb.proj:
        a[:] = 0
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    rows, _ = G.embed_forward(db, dev_u32(torch, [1, 2, 3, 4], cuda), dev_i64(torch, [0, 4], cuda))
    assert (rows == 0).all()


def test_linearity_in_tables(cuda):  # test_embedding.cpp:283-299 (scale tables x2: exact in bf16)
    cfg = O.make_default_config(500, 256, 3, 2)
    cfg["amplification"] = "none"
    hb = O.make_bank(cfg, 31)
    db1 = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    db2 = G.DeviceBank(cfg).upload(hb.base * 2, [s * 2 for s in hb.sub], hb.proj)
    t = dev_u32(torch, O.uniform_tokens(3, 500, 300), cuda)
    off = dev_i64(torch, [0, 300], cuda)
    a, _ = G.embed_forward(db1, t, off)
    b, _ = G.embed_forward(db2, t, off)
    assert torch.equal(a * 2, b)


def test_embed_from_ids_equals_forward_merged(cuda):  # embedding.hpp:163-201 (the decode-cache entry)
    g = gold("embed_tc_scale_sqrt_d.npz")
    hb, db = _bank(g, cuda)
    toks = dev_u32(torch, g["tokens"][:100], cuda)
    off = dev_i64(torch, [0, 100], cuda)
    ids = G.hash_ids(db, toks, off)
    m = G.embed_from_ids(db, toks, ids)
    _, merged = G.embed_forward(db, toks, off, rows=False, merged=True)
    assert torch.equal(m, merged)


def test_out_of_range_token_produces_no_output(cuda):  # hashing.cpp:49-54 / embedding.hpp:41-44
    g = gold("embed_tc_none.npz")
    hb, db = _bank(g, cuda)
    toks = O.uniform_tokens(9, 1000, 256)
    toks[200] = 5000
    out = torch.full((256, 256), 7.0, device=cuda)
    G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, [0, 256], cuda), out_rows=out)
    with pytest.raises(OutOfRange):
        db.sync_errors()
    assert (out == 7.0).all()  # nothing written, as the reference throws before writing
    with pytest.raises(OutOfRange):  # host-buffer entry raises before copying anything back
        G.embed_sequence(db, toks)


def test_host_buffer_entry_equals_device_entry(cuda):  # the drop-in embed_sequence(_cached) path
    g = gold("embed_tc_layer_norm.npz")
    hb, db = _bank(g, cuda)
    seqs = [g["tokens"][:100], g["tokens"][100:]]
    rows_h, merged_h = G.embed_batch_host(db, seqs, [[], g["prior1"]], want_rows=True, want_merged=True)
    rows_d, merged_d = _forward(db, g, cuda)
    assert np.array_equal(rows_h, rows_d) and np.array_equal(merged_h, merged_d)
    r1, m1 = G.embed_sequence_cached(db, seqs[1], g["prior1"])  # T=200 alone: small-T regime
    assert_rows_close(r1, rows_d[100:])
    # long batch: crosses the host pipeline's 8192-token chunking, pinned output
    big = O.uniform_tokens(11, 1000, 20000)
    pin = torch.empty((20000, 256), dtype=torch.float32).pin_memory()
    G.embed_batch_host(db, [big], want_rows=True, out_rows=pin.numpy())
    dev, _ = G.embed_forward(db, dev_u32(torch, big, cuda), dev_i64(torch, [0, 20000], cuda))
    assert torch.equal(pin, dev.cpu())


def test_longcat_scale_bank_sampled_tokens(cuda):
    """Full config C bank (31.9B params, device-generated) and the 8 x 8192 headline batch:
    sampled rows against the oracle's double evaluation of the same synthetic bank."""
    g = gold("cfgC_ids.npz")
    cfg = gold_config(g)
    db = G.DeviceBank(cfg)
    db.generate(1234)
    T = 8 * 8192
    toks = np.random.default_rng(42).integers(0, 128000, size=T).astype(np.uint32)
    off = np.arange(0, T + 1, 8192)
    rows, merged = G.embed_forward(db, dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda), merged=True)
    db.sync_errors()
    ids = G.hash_ids(db, dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda)).cpu().numpy().view(np.uint64)
    pick = [0, 1, 2, 8191, 8192, 40000, 65535]
    ref = np.stack([O.synth_embed_merged_f64(1234, toks[t], ids[t], 4, 4, 3072) for t in pick])
    got = merged[pick].cpu().numpy()
    assert_rows_close(got, ref)
    assert_rows_close(rows[pick].cpu().numpy(), ref * np.sqrt(3072.0))
    # size-independent properties of the whole output: finite, amplification = sqrt(D) * merged
    assert torch.isfinite(rows).all()
    assert torch.allclose(rows, merged * np.float32(np.sqrt(3072.0)), rtol=0, atol=0)
    db.close()


def test_fused_k1_k2_k3_kernel_matches_oracle(cuda):
    """D > 1024, T > 256: the fused K1+K2 kernel writes X and the pair kernel projects it:
    vs the oracle's double path and bit-identical across batch compositions in that regime."""
    cfg = O.make_default_config(500, 1536, 4, 4)  # d = 128
    cfg["amplification"] = "scale_sqrt_d"
    hb = O.make_bank(cfg, 21, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    seqs = [O.uniform_tokens(s, 500, n) for s, n in [(1, 1100), (2, 300), (3, 1200)]]
    allt = np.concatenate(seqs)
    off = np.concatenate([[0], np.cumsum([len(s) for s in seqs])])
    rows, merged = G.embed_forward(db, dev_u32(torch, allt, cuda), dev_i64(torch, off, cuda), merged=True)
    db.sync_errors()
    ref = np.concatenate([O.embed_sequence(hb, s, double=True)[1] for s in seqs])
    assert_rows_close(merged.cpu().numpy(), ref)
    for i, s in enumerate(seqs):
        alone, _ = G.embed_forward(db, dev_u32(torch, s, cuda), dev_i64(torch, [0, len(s)], cuda))
        if len(s) > 256:
            assert torch.equal(alone, rows[off[i]:off[i + 1]])
        else:
            assert_rows_close(alone.cpu().numpy(), rows[off[i]:off[i + 1]].cpu().numpy())
    bad = allt.copy()
    bad[1500] = 500  # inside the second sequence
    out = torch.full((len(bad), 1536), 3.0, device=cuda)
    G.embed_forward(db, dev_u32(torch, bad, cuda), dev_i64(torch, off, cuda), out_rows=out)
    with pytest.raises(OutOfRange):
        db.sync_errors()
    assert (out == 3.0).all()


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_pair_kernel_tma_epilogue_edges(cuda, out_dtype, monkeypatch):
    """The 2-CTA projection's TMA epilogue (E0 rows by tile::gather4, outputs by bulk tensor
    stores clipped at T): ragged T (not a multiple of 32 / 128 / 256), rows + merged; the
    direct-store epilogue and the 32-column E0 gather variant (NGRAM_TMA_EPI=0 / 1 in a
    subprocess are the A/B switches) compute the same bits.  Output buffers that are not 16-byte aligned are rejected up front."""
    monkeypatch.setenv("NGRAM_VERIFY_TILE", "0")  # pin the pair kernel whatever the verify-tile rule says
    cfg = O.make_default_config(3000, 512, 3, 2)
    hb = O.make_bank(cfg, 17, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    seqs = [O.uniform_tokens(40, 3000, 1001), O.uniform_tokens(41, 3000, 290), O.uniform_tokens(42, 3000, 7)]
    allt = np.concatenate(seqs)
    off = np.concatenate([[0], np.cumsum([len(s) for s in seqs])])
    T = len(allt)
    t, o = dev_u32(torch, allt, cuda), dev_i64(torch, off, cuda)
    rows, merged = G.embed_forward(db, t, o, merged=True, out_dtype=out_dtype)
    db.sync_errors()
    ref_r, ref_m = zip(*[O.embed_sequence(hb, s, double=True) for s in seqs])
    bf = out_dtype == torch.bfloat16
    assert_rows_close(rows.float().cpu().numpy(), np.concatenate(ref_r), bf16=bf)
    assert_rows_close(merged.float().cpu().numpy(), np.concatenate(ref_m), bf16=bf)
    buf = torch.empty(T * 512 + 8, dtype=out_dtype, device=cuda)
    with pytest.raises(InvalidArgument):
        G.embed_forward(db, t, o, out_dtype=out_dtype, out_rows=buf[1:1 + T * 512].view(T, 512))
    # the direct-store epilogue (selected once per process) must produce identical bits
    import os, subprocess, sys, tempfile
    code = f"""
import sys, numpy as np, torch
sys.path[:0] = {[os.path.join(os.path.dirname(__file__)), os.path.dirname(os.path.dirname(__file__)),
                 os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle")]!r}
import oracle as O
from helpers import dev_i64, dev_u32
from paper_2601_21204_b200 import ngram as G
cfg = O.make_default_config(3000, 512, 3, 2)
hb = O.make_bank(cfg, 17, round_bf16=True)
db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
seqs = [O.uniform_tokens(40, 3000, 1001), O.uniform_tokens(41, 3000, 290), O.uniform_tokens(42, 3000, 7)]
allt = np.concatenate(seqs)
off = np.concatenate([[0], np.cumsum([len(s) for s in seqs])])
r, m = G.embed_forward(db, dev_u32(torch, allt, "cuda:0"), dev_i64(torch, off, "cuda:0"), merged=True,
                       out_dtype=torch.{'bfloat16' if bf else 'float32'})
db.sync_errors()
np.save(sys.argv[1], torch.stack([r, m]).view(torch.int16 if r.dtype == torch.bfloat16 else torch.int32).cpu().numpy())
"""
    ours = torch.stack([rows, merged]).view(torch.int16 if bf else torch.int32).cpu().numpy()
    for mode in ("0", "1"):  # direct stores; TMA epilogue with 32-column E0 gathers
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "other.npy")
            subprocess.run([sys.executable, "-c", code, path], check=True, timeout=300,
                           env={**os.environ, "NGRAM_TMA_EPI": mode, "NGRAM_VERIFY_TILE": "0"})
            other = np.load(path)
        assert np.array_equal(ours, other), mode


def test_small_t_hash_in_gemm_variant_is_bit_identical(cuda):
    """The opt-in small-T GEMM that hashes and gathers in its producers (MODE 2,
    NGRAM_DECODE_HASH_IN_GEMM=1, selected once per process) computes the same split-K sums
    as the default gather-kernel + X path: bit-identical outputs, incl. a carried prior."""
    import os, subprocess, sys, tempfile
    code = f"""
import sys, numpy as np, torch
sys.path[:0] = {[os.path.dirname(__file__), os.path.dirname(os.path.dirname(__file__)),
                 os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle")]!r}
import oracle as O
from helpers import dev_i64, dev_u32
from paper_2601_21204_b200 import ngram as G
cfg = O.make_default_config(3000, 768, 4, 2)
hb = O.make_bank(cfg, 23, round_bf16=True)
db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
toks = O.uniform_tokens(81, 3000, 200)
prior = np.zeros((4, 3), np.uint32); prior[2] = [5, 6, 7]
r, m = G.embed_forward(db, dev_u32(torch, toks, "cuda:0"), dev_i64(torch, [0, 50, 120, 190, 200], "cuda:0"),
                       prior=dev_u32(torch, prior, "cuda:0"), merged=True)
db.sync_errors()
np.save(sys.argv[1], torch.stack([r, m]).view(torch.int32).cpu().numpy())
"""
    outs = []
    with tempfile.TemporaryDirectory() as td:
        for v in ("0", "1"):
            path = os.path.join(td, f"o{v}.npy")
            subprocess.run([sys.executable, "-c", code, path], check=True, timeout=300,
                           env={**os.environ, "NGRAM_DECODE_HASH_IN_GEMM": v})
            outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


def test_verify_sized_regime_at_longcat_width(cuda, monkeypatch):
    """D = 3072, verify-sized T (500 / 600): the one-wave 128 x 128 single-CTA tiles at LongCat
    width match the reference within tolerance, are batch-composition invariant, and compute the
    same bits as the pair kernel (NGRAM_VERIFY_TILE=0, read per call)."""
    cfg = O.make_default_config(1000, 3072, 4, 4)
    hb = O.make_bank(cfg, 31, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    seqs = [O.uniform_tokens(90 + i, 1000, n) for i, n in enumerate([300, 200, 100])]
    allt = np.concatenate(seqs)
    off = np.concatenate([[0], np.cumsum([len(s) for s in seqs])])
    rows, merged = G.embed_forward(db, dev_u32(torch, allt, cuda), dev_i64(torch, off, cuda), merged=True)
    db.sync_errors()
    ref_r, ref_m = zip(*[O.embed_sequence(hb, s, double=True) for s in seqs])
    assert_rows_close(rows.cpu().numpy(), np.concatenate(ref_r))
    assert_rows_close(merged.cpu().numpy(), np.concatenate(ref_m))
    a01, _ = G.embed_forward(db, dev_u32(torch, np.concatenate(seqs[:2]), cuda), dev_i64(torch, off[:3], cuda))
    assert torch.equal(a01, rows[:500])  # T = 500 and T = 600: same regime, same bits
    monkeypatch.setenv("NGRAM_VERIFY_TILE", "0")
    pr, pm = G.embed_forward(db, dev_u32(torch, allt, cuda), dev_i64(torch, off, cuda), merged=True)
    db.sync_errors()
    assert torch.equal(pr, rows) and torch.equal(pm, merged)


@pytest.mark.parametrize("env", [{"NGRAM_FUSED_GATHER": "1"}, {"NGRAM_PREFILL_PATH": "lsu"},
                                 {"NGRAM_PREFILL_PATH": "x"}])
def test_fused_gather_variant_is_bit_identical(cuda, env):
    """Every prefill producer variant -- A rows gathered by tile::gather4 straight into shared
    memory (NGRAM_FUSED_GATHER=1), hashed and cp.async-copied by the projection's own producers
    (NGRAM_PREFILL_PATH=lsu), or materialised as X by the K1+K2 kernel (x) -- feeds the tensor
    cores the same bf16 rows in the same K order: identical bits (D = 768, T = 900, with a
    carried prior context).  Selected once per process, hence the subprocesses."""
    import os, subprocess, sys, tempfile
    code = f"""
import sys, numpy as np, torch
sys.path[:0] = {[os.path.dirname(__file__), os.path.dirname(os.path.dirname(__file__)),
                 os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle")]!r}
import oracle as O
from helpers import dev_i64, dev_u32
from paper_2601_21204_b200 import ngram as G
cfg = O.make_default_config(3000, 768, 4, 4)
hb = O.make_bank(cfg, 29, round_bf16=True)
db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
toks = O.uniform_tokens(83, 3000, 900)
prior = dev_u32(torch, np.array([[5, 6, 7], [2900, 1, 17]], np.uint32), "cuda:0")
r, m = G.embed_forward(db, dev_u32(torch, toks, "cuda:0"), dev_i64(torch, [0, 400, 900], "cuda:0"), merged=True,
                       prior=prior)
db.sync_errors()
np.save(sys.argv[1], torch.stack([r, m]).view(torch.int32).cpu().numpy())
"""
    outs = []
    with tempfile.TemporaryDirectory() as td:
        for i, e in enumerate(({"NGRAM_FUSED_GATHER": "0", "NGRAM_PREFILL_PATH": "x"}, env)):
            path = os.path.join(td, f"o{i}.npy")
            subprocess.run([sys.executable, "-c", code, path], check=True, timeout=300, env={**os.environ, **e})
            outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])
