#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libngram_ref.so, the
unmodified reference sources compiled by oracle/Makefile).  Run here, where
/root/reference exists:  python tests/golden/make_golden.py

Every fixture records which reference entry point produced it.  Seeds follow SURVEY.md
8(d) / the reference tests (test_hashing.cpp:40-57 seed 0x5eed0001, tokens seed 42,
banks seed 1234, bf16-rounded so the bf16 device bank and the float bank are equal).
"""
import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

R = O.ref()


def ref_default_config(v0, dim, N, K):
    buf = C.create_string_buffer(1 << 16)
    assert R.ref_make_default_config_json(v0, dim, N, K, buf, len(buf)) == 0
    return json.loads(buf.value)


def ref_hash_sequences(cfg, seqs, priors=None):
    out = []
    for i, s in enumerate(seqs):
        s = np.ascontiguousarray(s, np.uint32)
        B = (cfg["max_order"] - 1) * cfg["sub_tables"]
        ids = np.zeros((len(s), max(B, 1)), np.uint64)
        pr = None if priors is None else np.ascontiguousarray(priors[i], np.uint32)
        rc = R.ref_hash_sequence(json.dumps(cfg).encode(), s, len(s), None if pr is None else pr.ctypes.data,
                                 0 if pr is None else len(pr), ids)
        assert rc == 0, R.ref_last_error()
        out.append(ids[:, :B])
    return np.concatenate(out)


def ref_bank(cfg, seed):
    h = R.ref_bank_create(json.dumps(cfg).encode(), seed, 1)
    assert h, R.ref_last_error()
    return h


def ref_tensor(h, which, b=0):
    n = C.c_int64()
    p = R.ref_bank_tensor(h, which, b, C.byref(n))
    return np.ctypeslib.as_array(p, (n.value,)).copy()


def bank_checksum_ref(h, cfg):
    N, K, D, B, d, v, denom = O.shape(cfg)
    hb = O.HostBank(cfg, ref_tensor(h, 0), [ref_tensor(h, 1, b) for b in range(B)],
                    [ref_tensor(h, 2, b) for b in range(B)] if v == 1 else [],
                    ref_tensor(h, 3) if cfg["amplification"] == "layer_norm" else np.zeros(0, np.float32),
                    ref_tensor(h, 4) if cfg["amplification"] == "layer_norm" else np.zeros(0, np.float32))
    return O.bank_checksum(hb)


def ref_embed(h, seqs, priors=None, D=None):
    rows32, merged32, rows64, merged64 = [], [], [], []
    for i, s in enumerate(seqs):
        s = np.ascontiguousarray(s, np.uint32)
        pr = None if priors is None else np.ascontiguousarray(priors[i], np.uint32)
        a = [np.zeros((len(s), D), np.float32) for _ in range(2)]
        b = [np.zeros((len(s), D), np.float64) for _ in range(2)]
        args = (s, len(s), None if pr is None else pr.ctypes.data, 0 if pr is None else len(pr))
        assert R.ref_embed_sequence_f32(h, *args, a[0].ctypes.data, a[1].ctypes.data) == 0
        assert R.ref_embed_sequence_f64(h, *args, b[0].ctypes.data, b[1].ctypes.data) == 0
        rows32.append(a[0]), merged32.append(a[1]), rows64.append(b[0]), merged64.append(b[1])
    return tuple(np.concatenate(x) for x in (rows32, merged32, rows64, merged64))


def save(name, **kw):
    np.savez_compressed(os.path.join(HERE, name), **kw)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in kw.items() if hasattr(v, "shape")})


def v2_config(v0, dim, order, k, amp="none"):
    """tests/test_embedding.cpp:28-44 v2_config."""
    sv = [13 + 8 * n + 3 * kk for n in range(2, order + 1) for kk in range(1, k + 1)]
    return O.make_config(v0, dim, order, k, sv, "subtable_v2", amp)


def v1_config(v0, dim, order):
    """tests/test_embedding.cpp:15-26 v1_config."""
    return O.make_config(v0, dim, order, 1, [17 + 10 * n for n in range(2, order + 1)], "averaged_v1", "none")


def main():
    # 1. rolling_hash: reference's own randomized case stream (test_hashing.cpp:40-57)
    cnt = 20000
    n = np.zeros(cnt, np.int32)
    base = np.zeros(cnt, np.uint64)
    mod = np.zeros(cnt, np.uint64)
    win = np.zeros((cnt, 8), np.uint32)
    h = np.zeros(cnt, np.uint64)
    assert R.ref_rolling_hash_cases(0x5EED0001, cnt, n, base, mod, win.reshape(-1), h) == 0
    save("rolling_hash_20k.npz", n=n, base=base, modulus=mod, windows=win, hash=h,
         source="ref_rolling_hash_cases -> ngram::rolling_hash (hashing.cpp:33-59)")

    # 2. config A ids: make_default_config(32000, 256, 3, 2), 4 x 512 tokens, seed 42
    cfgA = ref_default_config(32000, 256, 3, 2)
    toksA = O.uniform_tokens(42, 32000, 4 * 512)
    idsA = ref_hash_sequences(cfgA, [toksA[i * 512:(i + 1) * 512] for i in range(4)])
    save("cfgA_ids.npz", config=json.dumps(cfgA), tokens=toksA, ids=idsA, seq_len=512)

    # 3. LongCat-scale (config C) ids, 2 sequences x 1024 with a carried prior on the second
    sv = [(2 * (74 + b) + 1) * 64000 for b in range(12)]
    cfgC = O.make_config(128000, 3072, 4, 4, sv, "subtable_v2", "scale_sqrt_d")
    toksC = O.uniform_tokens(43, 128000, 2048)
    priorC = O.uniform_tokens(44, 128000, 3)
    idsC = np.concatenate([ref_hash_sequences(cfgC, [toksC[:1024]]),
                           ref_hash_sequences(cfgC, [toksC[1024:]], [priorC])])
    save("cfgC_ids.npz", config=json.dumps(cfgC), tokens=toksC, prior=priorC, ids=idsC)

    # 4. moduli above 2^32 (general 128-bit path): N=5, K=2
    svb = [(1 << 40) + 12345 * (i + 1) for i in range(8)]
    cfgBig = O.make_config(1 << 20, 16, 5, 2, svb, "subtable_v2", "none")
    toksB = O.uniform_tokens(45, 1 << 20, 600)
    save("bigmod_ids.npz", config=json.dumps(cfgBig), tokens=toksB,
         ids=ref_hash_sequences(cfgBig, [toksB[:300], toksB[300:]]))

    # 5. embeddings on the tensor-core shape (D=256, d=64), every amplification mode
    for amp in ["none", "scale_sqrt_d", "layer_norm"]:
        cfg = ref_default_config(1000, 256, 3, 2)
        cfg["amplification"] = amp
        hb = ref_bank(cfg, 1234)
        if amp == "layer_norm":  # non-trivial gain / bias, as test_embedding.cpp:211-214
            g = np.random.default_rng(5)
            gain = (1.0 + 0.1 * g.standard_normal(256)).astype(np.float32)
            bias = (0.05 * g.standard_normal(256)).astype(np.float32)
            O.lib().or_round_bf16(gain, gain.size)
            O.lib().or_round_bf16(bias, bias.size)
            R.ref_bank_set_ln(hb, gain, bias)
        toks = O.uniform_tokens(7, 1000, 300)
        prior = O.uniform_tokens(8, 1000, 2)
        seqs = [toks[:100], toks[100:300]]
        r32, m32, r64, m64 = ref_embed(hb, seqs, [np.zeros(0, np.uint32), prior], D=256)
        extra = {}
        if amp == "layer_norm":
            extra = {"ln_gain": ref_tensor(hb, 3), "ln_bias": ref_tensor(hb, 4)}
        save(f"embed_tc_{amp}.npz", config=json.dumps(cfg), seed=1234, tokens=toks, seq_offsets=np.array([0, 100, 300]),
             prior1=prior, rows_f32=r32, merged_f32=m32, rows_f64=r64, merged_f64=m64,
             bank_checksum=np.uint64(bank_checksum_ref(hb, cfg)), **extra)
        R.ref_bank_destroy(hb)

    # 6. generic shapes (CUDA-core path): the reference tests' v2_config / v1_config banks
    for name, cfg, seed in [("simt_v2", v2_config(16, 12, 4, 2, "scale_sqrt_d"), 7),
                            ("simt_v2_k1", v2_config(32, 12, 3, 2, "none"), 11),
                            ("v1", v1_config(8, 4, 3), 17),
                            ("v1_wide", O.make_config(500, 512, 4, 1, [3001, 3011, 3019], "averaged_v1",
                                                      "scale_sqrt_d"), 19)]:
        hb = ref_bank(cfg, seed)
        toks = O.uniform_tokens(13, cfg["base_vocab"], 64)
        r32, m32, r64, m64 = ref_embed(hb, [toks[:20], toks[20:]], None, D=cfg["dim"])
        save(f"embed_{name}.npz", config=json.dumps(cfg), seed=seed, tokens=toks, seq_offsets=np.array([0, 20, 64]),
             rows_f32=r32, merged_f32=m32, rows_f64=r64, merged_f64=m64,
             bank_checksum=np.uint64(bank_checksum_ref(hb, cfg)))
        R.ref_bank_destroy(hb)

    # 7. full LongCat width D=3072, N=4, K=4 (reduced vocabulary bank), 48 tokens
    cfgW = ref_default_config(1000, 3072, 4, 4)
    hb = ref_bank(cfgW, 1234)
    toks = O.uniform_tokens(21, 1000, 48)
    r32, m32, r64, m64 = ref_embed(hb, [toks], None, D=3072)
    save("embed_d3072.npz", config=json.dumps(cfgW), seed=1234, tokens=toks, seq_offsets=np.array([0, 48]),
         rows_f32=r32, merged_f64=m64, rows_f64=r64, bank_checksum=np.uint64(bank_checksum_ref(hb, cfgW)))
    R.ref_bank_destroy(hb)

    # 8. decode: draft_verify through the reference (cache.cpp:152-195) after a warm-up append
    cfgD = ref_default_config(64, 384, 4, 2)  # TC shape (d=64), BN=128 tile
    cfgD["amplification"] = "none"
    hb = ref_bank(cfgD, 99)
    rng = np.random.default_rng(3)
    cases = {}
    for trial in range(6):
        ch = R.ref_cache_create(json.dumps(cfgD).encode())
        prefix = rng.integers(0, 64, size=int(rng.integers(0, 6)), dtype=np.uint32)
        pid = np.zeros(16, np.uint64)
        for t in prefix:
            assert R.ref_cache_append(ch, int(t), pid) == 0
        L = int(rng.integers(1, 9))
        draft = rng.integers(0, 64, size=L, dtype=np.uint32)
        accept = int(rng.integers(0, L + 1))
        acc = np.zeros((max(accept, 1), 384), np.float32)
        cnt8 = np.zeros(8, np.uint64)
        assert R.ref_draft_verify(ch, hb, draft, L, accept, 256, 0, acc, cnt8) == 0
        ring = np.zeros(3, np.uint32)
        length = C.c_uint64()
        last = C.c_uint32()
        R.ref_cache_ring(ch, ring, C.byref(length), C.byref(last))
        i = trial
        cases.update({f"c{i}_prefix": prefix, f"c{i}_draft": draft, f"c{i}_accept": np.int64(accept),
                      f"c{i}_accepted": acc[:accept], f"c{i}_ring": ring.copy(), f"c{i}_length": np.uint64(length.value),
                      f"c{i}_last": np.uint32(last.value), f"c{i}_counters": cnt8})
        R.ref_cache_destroy(ch)
    save("draft_verify.npz", config=json.dumps(cfgD), seed=99, ncases=6, **cases)
    R.ref_bank_destroy(hb)
    backward_goldens()
    plne_goldens()
    analysis_goldens()


def backward_goldens():
    # 9. backward: embed_sequence_backward<double> (embedding.hpp:438-459), two sequences
    #    (the second with a carried prior), gradients summed over the two calls.  Sparse
    #    storage of the touched E0 / sub-table rows; projections and LN dense.
    for name, cfg, seed in [("tc_none", dict(ref_default_config(1000, 256, 3, 2), amplification="none"), 1234),
                            ("tc_scale_sqrt_d", ref_default_config(1000, 256, 3, 2), 1234),
                            ("tc_layer_norm", dict(ref_default_config(1000, 256, 3, 2), amplification="layer_norm"),
                             1234),
                            ("simt_v2", v2_config(16, 12, 4, 2, "scale_sqrt_d"), 7),
                            ("v1_wide", O.make_config(500, 512, 4, 1, [3001, 3011, 3019], "averaged_v1",
                                                      "layer_norm"), 19)]:
        hb = ref_bank(cfg, seed)
        D = cfg["dim"]
        extra = {}
        if cfg["amplification"] == "layer_norm":
            g = np.random.default_rng(6)
            gain = (1.0 + 0.1 * g.standard_normal(D)).astype(np.float32)
            bias = (0.05 * g.standard_normal(D)).astype(np.float32)
            O.lib().or_round_bf16(gain, gain.size)
            O.lib().or_round_bf16(bias, bias.size)
            R.ref_bank_set_ln(hb, gain, bias)
            extra = {"ln_gain": gain, "ln_bias": bias}
        toks = O.uniform_tokens(31, cfg["base_vocab"], 120)
        prior = O.uniform_tokens(32, cfg["base_vocab"], cfg["max_order"] - 1)
        seqs, priors = [toks[:40], toks[40:]], [np.zeros(0, np.uint32), prior]
        _, _, _, m64 = ref_embed(hb, seqs, priors, D=D)
        up = np.random.default_rng(9).standard_normal((len(toks), D)).astype(np.float32).astype(np.float64)
        acc = O.zero_grads(cfg)
        for (a, b), pr in zip([(0, 40), (40, 120)], priors):
            gr = O.zero_grads(cfg)
            sp = (C.c_void_p * max(len(gr["sub"]), 1))(*[x.ctypes.data for x in gr["sub"]])
            pp = (C.c_void_p * max(len(gr["proj"]), 1))(*[x.ctypes.data for x in gr["proj"]])
            mm = np.ascontiguousarray(m64[a:b])
            uu = np.ascontiguousarray(up[a:b])
            assert R.ref_embed_sequence_backward_f64(hb, toks[a:b], b - a, pr.ctypes.data if len(pr) else None, len(pr),
                                                     mm.ctypes.data, uu.ctypes.data, gr["base"].ctypes.data, sp, pp,
                                                     gr["gain"].ctypes.data, gr["bias"].ctypes.data) == 0
            for k in ("base", "gain", "bias"):
                acc[k] += gr[k]
            for k in ("sub", "proj"):
                for x, y in zip(acc[k], gr[k]):
                    x += y
        out = {}
        nz = np.nonzero(np.any(acc["base"] != 0, axis=1))[0]
        out["g_base_idx"], out["g_base_val"] = nz, acc["base"][nz]
        for b, x in enumerate(acc["sub"]):
            nz = np.nonzero(np.any(x != 0, axis=1))[0]
            out[f"g_sub{b}_idx"], out[f"g_sub{b}_val"] = nz, x[nz]
        if acc["proj"]:
            out["g_proj"] = np.stack(acc["proj"])
        if cfg["amplification"] == "layer_norm":
            out["g_gain"], out["g_bias"] = acc["gain"], acc["bias"]
        save(f"backward_{name}.npz", config=json.dumps(cfg), seed=seed, tokens=toks, seq_offsets=np.array([0, 40, 120]),
             prior1=prior, merged_f64=m64, upstream=up, bank_checksum=np.uint64(bank_checksum_ref(hb, cfg)),
             **extra, **out)
        R.ref_bank_destroy(hb)


def plne_goldens():
    # 10. PLNE (ple.hpp:168-196): ffn_plne<double> / ffn_plne_backward<double> per position of
    #     two sequences (the second with a carried prior); params are float-representable.
    for name, cfg, seed, dm in [("tc", dict(ref_default_config(1000, 256, 3, 2), amplification="none"), 77, 128),
                                ("small", O.make_config(10, 6, 3, 1, [25, 31], "subtable_v2", "none"), 21, 4)]:
        hb = ref_bank(cfg, seed)
        H, N = cfg["dim"], cfg["max_order"]
        r = np.random.default_rng(seed)
        gate = (0.02 * r.standard_normal((H, dm))).astype(np.float32).astype(np.float64)
        down = (0.02 * r.standard_normal((dm, H))).astype(np.float32).astype(np.float64)
        toks = O.uniform_tokens(61, cfg["base_vocab"], 48)
        prior = O.uniform_tokens(62, cfg["base_vocab"], N - 1)
        T = len(toks)
        x = r.standard_normal((T, dm)).astype(np.float32).astype(np.float64)
        up = r.standard_normal((T, dm)).astype(np.float32).astype(np.float64)
        y = np.zeros((T, dm))
        dx = np.zeros((T, dm))
        g_gate, g_down = np.zeros((H, dm)), np.zeros((dm, H))
        acc = O.zero_grads(cfg)
        for (a, b), pr in zip([(0, 16), (16, T)], [None, prior]):
            for pos in range(b - a):
                ctx = O.window(toks[a:b], pos, N, pr)
                t = a + pos
                assert R.ref_ffn_plne_f64(hb, gate.ctypes.data, down.ctypes.data, dm, x[t].ctypes.data, ctx,
                                          y[t].ctypes.data) == 0
                gg, gd, d1 = np.zeros((H, dm)), np.zeros((dm, H)), np.zeros(dm)
                gr = O.zero_grads(cfg)
                sp = (C.c_void_p * max(len(gr["sub"]), 1))(*[q.ctypes.data for q in gr["sub"]])
                pp = (C.c_void_p * max(len(gr["proj"]), 1))(*[q.ctypes.data for q in gr["proj"]])
                uu = np.ascontiguousarray(up[t])
                assert R.ref_ffn_plne_backward_f64(hb, gate.ctypes.data, down.ctypes.data, dm, x[t].ctypes.data,
                                                   ctx, uu.ctypes.data, gg.ctypes.data, gd.ctypes.data,
                                                   gr["base"].ctypes.data, sp, pp, d1.ctypes.data) == 0
                g_gate += gg
                g_down += gd
                dx[t] = d1
                acc["base"] += gr["base"]
                for k in ("sub", "proj"):
                    for q1, q2 in zip(acc[k], gr[k]):
                        q1 += q2
        out = {}
        nz = np.nonzero(np.any(acc["base"] != 0, axis=1))[0]
        out["g_base_idx"], out["g_base_val"] = nz, acc["base"][nz]
        for b, q in enumerate(acc["sub"]):
            nz = np.nonzero(np.any(q != 0, axis=1))[0]
            out[f"g_sub{b}_idx"], out[f"g_sub{b}_val"] = nz, q[nz]
        if acc["proj"]:
            out["g_proj"] = np.stack(acc["proj"])
        save(f"plne_{name}.npz", config=json.dumps(cfg), seed=seed, d_model=dm, gate=gate, down=down, tokens=toks,
             seq_offsets=np.array([0, 16, T]), prior1=prior, x=x, y=y, upstream=up, g_gate=g_gate, g_down=g_down,
             dx=dx, bank_checksum=np.uint64(bank_checksum_ref(hb, cfg)), **out)
        R.ref_bank_destroy(hb)


def analysis_goldens():
    # 11. corpus_analyzer (analysis.cpp:44-176) on the reference itself: the worked examples of
    #     test_analysis.cpp, its Zipf-Markov corpora, random corpora, a bad token (partial
    #     counts), moduli above 2^32 and near 2^64, order-100 windows over V0 = 2 (128-bit keys).
    r = np.random.default_rng(2026)
    cases = [
        ("worked20", 10, [2], [20, 23], [[1, 5], [3, 5], [5, 5]]),
        ("single", 10, [2], [100], [[5]]),
        ("allpairs", 7, [2], [49, 30], [[a, b] for a in range(7) for b in range(7)]),
        ("zipf1000", 1000, [2, 3, 4], [4999, 2000, 2500, 30000, 30500],
         O.ref_zipf_markov(1000, 16, 4096, 99, 1.1, 0.85)),
        ("random", 120, [2, 3], [37, 240, 4000], [r.integers(0, 120, size=int(r.integers(1, 101))) for _ in range(9)]),
        ("badtoken", 10, [2, 3], [5, 7], [[1, 2, 3], [3, 11, 4], [5]]),
        ("bigmod", 128000, [2, 3], [(1 << 40) + 15, (1 << 33) + 1, 10944000, 1],
         O.ref_zipf_markov(128000, 8, 2048, 20260809)),
        ("wide_v0", 4000000000, [2, 3], [1 << 32, (1 << 32) + 1, (1 << 64) - 59, 3],
         [r.integers(3999990000, 4000000000, size=400) for _ in range(3)]),
        ("order100", 2, [2, 64, 100], [97, 1 << 35], [r.integers(0, 2, size=300) for _ in range(4)]),
        ("empty_seqs", 50, [2], [40], [[], [3, 4], [], [4, 3, 4]]),
    ]
    for name, v0, orders, moduli, seqs in cases:
        seqs = [np.asarray(q, np.uint32) for q in seqs]
        rc, st = O.ref_corpus_analyze(v0, orders, moduli, seqs)
        toks, off = O._flat(seqs)
        save(f"analysis_{name}.npz", v0=np.uint64(v0), orders=np.array(orders, np.int32),
             moduli=np.array(moduli, np.uint64), tokens=toks[:off[-1]], seq_offsets=off, status=rc,
             meta=np.array([st["sequences_seen"], st["tokens_seen"]], np.uint64),
             seen=np.array([st["ngrams_seen"][o] for o in orders], np.uint64),
             distinct=np.array([st["distinct_ngrams"][o] for o in orders], np.uint64),
             buckets=np.array([st["distinct_buckets"][(o, m)] for o in orders for m in moduli], np.uint64))


def _bf16_bits(a):
    """float32 values that are bf16-exact -> their uint16 bf16 bit patterns."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32)
    assert not (u & 0xFFFF).any()
    return (u >> 16).astype(np.uint16)


def _prefixed_streams(rng, n, v0, max_prefix=6):
    """n decode streams, each primed by 0..max_prefix appended tokens: (prefix matrix, lengths)."""
    lens = rng.integers(0, max_prefix + 1, size=n)
    pref = np.zeros((n, max_prefix), np.uint32)
    for s in range(n):
        pref[s, :lens[s]] = rng.integers(0, v0, size=lens[s])
    return pref, lens.astype(np.int64)


def _ref_stream_cases(cfg, hb, pref, lens, draft, accept):
    """Per stream: reference sequence_cache fed the prefix (cache.cpp:37-57), then draft_verify
    (cache.cpp:152-195) with a fresh memo.  Returns accepted rows (concatenated in stream order),
    and the rings / lengths / last tokens afterwards."""
    n, L = draft.shape
    D = cfg["dim"]
    acc_rows, rings, lengths, lasts = [], [], [], []
    pid = np.zeros(64, np.uint64)
    for s in range(n):
        ch = R.ref_cache_create(json.dumps(cfg).encode())
        for t in pref[s, :lens[s]]:
            assert R.ref_cache_append(ch, int(t), pid) == 0
        out = np.zeros((max(int(accept[s]), 1), D), np.float32)
        cnt8 = np.zeros(8, np.uint64)
        assert R.ref_draft_verify(ch, hb, np.ascontiguousarray(draft[s]), L, int(accept[s]), 4096, 0, out, cnt8) == 0
        acc_rows.append(out[:int(accept[s])])
        ring = np.zeros(cfg["max_order"] - 1, np.uint32)
        length, last = C.c_uint64(), C.c_uint32()
        R.ref_cache_ring(ch, ring, C.byref(length), C.byref(last))
        rings.append(ring)
        lengths.append(length.value)
        lasts.append(last.value)
        R.ref_cache_destroy(ch)
    return (np.concatenate(acc_rows), np.stack(rings), np.array(lengths, np.uint64), np.array(lasts, np.uint32))


def r2_goldens():
    """Round-2 fixtures: the regimes and banks the round-1 goldens did not reach.
    12. D=3072 prefix calls of T = 129 / 200 / 256 (the split-K GEMM's second sub-regime).
    13. verify block + commit at D=3072, 64 streams x 4 drafts (config E shape; T = 256).
    14. decode step at D=3072 with 256 streams (config D's largest batch; T = 256).
    15. config A's actual bank make_bank(make_default_config(32000, 256, 3, 2), 1234), full 4 x 512.
    16. config B's actual bank make_bank(make_default_config(128000, 768, 4, 4), 1234), 16 x 4096
        tokens, 128 sampled positions (with the bank rows they touch).
    17. Barrett fast-path edge: V0 = 2^32 - 5, moduli in (2^31, 2^32]."""
    # 12
    cfgW = ref_default_config(1000, 3072, 4, 4)
    hb = ref_bank(cfgW, 1234)
    toks = O.uniform_tokens(23, 1000, 256)
    _, _, r64, m64 = ref_embed(hb, [toks], None, D=3072)
    save("regime2_d3072.npz", config=json.dumps(cfgW), seed=1234, tokens=toks, rows_f64_f32=r64.astype(np.float32),
         bank_checksum=np.uint64(bank_checksum_ref(hb, cfgW)),
         source="embed_sequence_cached<double> (embedding.hpp:409-429), rows rounded to f32")
    R.ref_bank_destroy(hb)

    # 13 / 14: the cache path (amplification none: merged vectors, cache.hpp:122-124)
    cfgE = dict(ref_default_config(1000, 3072, 4, 4), amplification="none")
    hb = ref_bank(cfgE, 1234)
    rng = np.random.default_rng(2027)
    pref, lens = _prefixed_streams(rng, 64, 1000)
    draft = rng.integers(0, 1000, size=(64, 4), dtype=np.uint32)
    accept = rng.integers(0, 5, size=64)
    accept[:3] = [0, 4, 4]
    acc, rings, lengths, lasts = _ref_stream_cases(cfgE, hb, pref, lens, draft, accept)
    save("verify_d3072_64x4.npz", config=json.dumps(cfgE), seed=1234, prefix=pref, prefix_len=lens, draft=draft,
         accept=accept.astype(np.int64), accepted=acc, ring=rings, length=lengths, last=lasts,
         source="sequence_cache::append + draft_verify (cache.cpp:37-57, 152-195), float path")
    pref, lens = _prefixed_streams(rng, 256, 1000)
    step = rng.integers(0, 1000, size=(256, 1), dtype=np.uint32)
    acc, rings, lengths, lasts = _ref_stream_cases(cfgE, hb, pref, lens, step, np.ones(256, np.int64))
    save("decode_d3072_b256.npz", config=json.dumps(cfgE), seed=1234, prefix=pref, prefix_len=lens, token=step[:, 0],
         merged=acc, ring=rings, length=lengths, last=lasts,
         source="sequence_cache::append + draft_verify(accept = L = 1) (cache.cpp:152-195), float path")
    R.ref_bank_destroy(hb)

    # 15
    cfgA = ref_default_config(32000, 256, 3, 2)
    hb = ref_bank(cfgA, 1234)
    toksA = O.uniform_tokens(42, 32000, 4 * 512)
    _, _, r64, m64 = ref_embed(hb, [toksA[i * 512:(i + 1) * 512] for i in range(4)], None, D=256)
    save("cfgA_bank_embed.npz", config=json.dumps(cfgA), seed=1234, tokens=toksA, seq_len=512,
         rows_f64_f32=r64.astype(np.float32), bank_checksum=np.uint64(bank_checksum_ref(hb, cfgA)),
         source="make_bank<float>(config A, 1234) bf16-rounded; embed_sequence_cached<double>")
    R.ref_bank_destroy(hb)

    # 16
    cfgB = ref_default_config(128000, 768, 4, 4)
    hb = ref_bank(cfgB, 1234)
    N, K, D, B, d, v, denom = O.shape(cfgB)
    toksB = O.uniform_tokens(42, 128000, 16 * 4096)
    off = np.arange(0, 16 * 4096 + 1, 4096, dtype=np.int64)
    rs = np.random.default_rng(16)
    pos = np.unique(np.concatenate([[0, 1, 2, 3, 4095, 4096, 4097, 4098, 65535],
                                    rs.choice(65536, size=119, replace=False)]))[:128].astype(np.int64)
    rows = np.zeros((len(pos), D), np.float64)
    merged = np.zeros((len(pos), D), np.float64)
    assert R.ref_embed_positions_f64(hb, toksB, off, 16, pos, len(pos), rows.ctypes.data, merged.ctypes.data) == 0, \
        R.ref_last_error()
    ids = np.concatenate([ref_hash_sequences(cfgB, [toksB[off[s]:off[s + 1]]]) for s in range(16)])[pos]
    base = ref_tensor(hb, 0).reshape(-1, D)
    sub_rows = np.stack([ref_tensor(hb, 1, b).reshape(-1, d)[ids[:, b].astype(np.int64)] for b in range(B)], axis=1)
    proj = np.stack([ref_tensor(hb, 2, b) for b in range(B)])
    save("cfgB_sampled.npz", config=json.dumps(cfgB), seed=1234, tokens=toksB, seq_offsets=off, positions=pos,
         ids=ids, e0_rows_bf16=_bf16_bits(base[toksB[pos]]), sub_rows_bf16=_bf16_bits(sub_rows),
         proj_bf16=_bf16_bits(proj), rows_f64_f32=rows.astype(np.float32), merged_f64_f32=merged.astype(np.float32),
         bank_checksum=np.uint64(bank_checksum_ref(hb, cfgB)),
         source="make_bank<float>(config B, 1234) bf16-rounded; embed_sequence_cached<double> at sampled positions")
    R.ref_bank_destroy(hb)

    # 17: products up to (2^32-1)^2 -- the Barrett quotient's worst case (hashdev.cuh barrett_mod)
    v0 = (1 << 32) - 5
    moduli = [(1 << 31) + 1, 3000000019, (1 << 32) - 5, (1 << 32) - 1, 1 << 32, (1 << 32) - 65,
              (1 << 31) + 11, 4000000007, 3 * (1 << 30)]
    cfgX = O.make_config(v0, 18, 4, 3, moduli, "subtable_v2", "none")
    rx = np.random.default_rng(17)
    edge = np.array([0, 1, v0 - 1, v0 - 2, (1 << 31), (1 << 31) + 1, (1 << 31) - 1, 3000000018, 3000000019,
                     (1 << 32) - 6, (1 << 32) - 66, (1 << 32) - 65, 4000000006], np.uint64)
    seqs = [rx.integers(0, v0, size=700, dtype=np.uint64).astype(np.uint32),
            rx.choice(edge, size=500).astype(np.uint32),
            rx.integers(v0 - 1000, v0, size=300, dtype=np.uint64).astype(np.uint32),
            np.concatenate([rx.choice(edge, size=100), rx.integers(0, v0, size=100, dtype=np.uint64)]).astype(np.uint32)]
    tk = np.concatenate(seqs)
    so = np.concatenate([[0], np.cumsum([len(q) for q in seqs])]).astype(np.int64)
    save("barrett_edge_ids.npz", config=json.dumps(cfgX), tokens=tk, seq_offsets=so, ids=ref_hash_sequences(cfgX, seqs),
         source="hash_all_orders (hashing.cpp:61-81) over fill_context windows")


if __name__ == "__main__":
    if sys.argv[1:] == ["r2"]:  # regenerate only sections 12-17
        r2_goldens()
    elif sys.argv[1:] == ["backward"]:  # regenerate only section 9
        backward_goldens()
    elif sys.argv[1:] == ["plne"]:  # regenerate only section 10
        plne_goldens()
    elif sys.argv[1:] == ["analysis"]:  # regenerate only section 11
        analysis_goldens()
    else:
        main()
