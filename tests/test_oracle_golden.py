"""Pin the CPU restatement (oracle/ngram_oracle.c) against the REFERENCE.

Every expected value here comes either from a literal in the reference's own tests
(proj/tests/test_hashing.cpp, test_embedding.cpp, test_cache.cpp -- cited per case) or
from tests/golden/*.npz, which tests/golden/make_golden.py produced by running the
unmodified reference (oracle/_ref).  Once pinned, the restatement is the checker the
GPU parity tests use for cases no fixture covers (e.g. full LongCat-scale sampling).
"""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


import helpers  # noqa: E402
from helpers import gold, gold_config  # noqa: E402


# ---------------------------------------------------------------- hashing (test_hashing.cpp)
def test_rolling_hash_worked_examples():  # test_hashing.cpp:12-26
    assert O.rolling_hash([3, 5], 2, 10, 7) == (0, 0)
    assert O.rolling_hash([0] * 5, 5, 1000, 12345) == (0, 0)
    assert O.rolling_hash([0, 0], 2, 7, 3) == (0, 0)
    assert O.rolling_hash([0, 0, 7], 3, 128000, 13) == (0, 7)


def test_rolling_hash_input_validation():  # test_hashing.cpp:28-38
    assert O.rolling_hash([1, 2, 3], 2, 10, 7)[0] == -1
    assert O.rolling_hash([1, 2, 3], 4, 10, 7)[0] == -1
    assert O.rolling_hash([1, 12], 2, 10, 7)[0] == -2
    assert O.rolling_hash([1, 2, 3], 3, 1, 7)[0] == -1
    assert O.rolling_hash([1, 2, 3], 3, 10, 0)[0] == -1
    assert O.rolling_hash([5], 1, 10, 7)[0] == -1


def test_rolling_hash_matches_reference_and_bigint():  # test_hashing.cpp:40-57 (seed 0x5eed0001)
    g = gold("rolling_hash_20k.npz")
    for i in range(len(g["n"])):
        n = int(g["n"][i])
        w = [int(x) for x in g["windows"][i, :n]]
        base, mod = int(g["base"][i]), int(g["modulus"][i])
        rc, h = O.rolling_hash(w, n, base, mod)
        assert rc == 0 and h == int(g["hash"][i]) and h < mod
        if i % 10 == 0:  # the reference's arbitrary-precision oracle (tests/oracles.hpp:20-30)
            val = sum(w[n - 1 - j] * base ** j for j in range(n))
            assert val % mod == h


def test_prefix_pad_identity():  # test_hashing.cpp:59-74, same rng stream
    rng = O.Rng64(0x5EED0002)
    for _ in range(2000):
        n = 2 + rng.below(5)
        base = 2 + rng.below(100000)
        mod = 1 + rng.below(1 << 20)
        w = [rng.below(base) for _ in range(n)]
        assert O.rolling_hash(w, n, base, mod) == O.rolling_hash([0] + w, n + 1, base, mod)


def test_hash_all_orders_worked_example():  # test_hashing.cpp:83-101
    cfg = O.make_config(16, 4, 3, 1, [101, 103], "averaged_v1", "none")
    ids = O.hash_sequence(cfg, [9], prior=[0, 4])
    assert ids.tolist() == [[73, 73]]
    assert O.hash_sequence(cfg, [0], prior=[0, 0]).tolist() == [[0, 0]]


def test_equal_moduli_equal_ids():  # test_hashing.cpp:103-120
    cfg = O.make_config(32, 8, 2, 2, [77, 77], "subtable_v2", "none")
    rng = O.Rng64(7)
    toks = [rng.below(32) for _ in range(400)]
    ids = O.hash_sequence(cfg, toks)
    assert (ids[:, 0] == ids[:, 1]).all()


@pytest.mark.parametrize("name,nseq", [("cfgA_ids.npz", 4)])
def test_config_a_ids_match_reference(name, nseq):
    g = gold(name)
    cfg = json.loads(str(g["config"]))
    toks = g["tokens"]
    L = len(toks) // nseq
    ids = np.concatenate([O.hash_sequence(cfg, toks[i * L:(i + 1) * L]) for i in range(nseq)])
    assert (ids == g["ids"]).all()
    assert cfg == O.make_default_config(32000, 256, 3, 2)  # config.cpp:163-183 restated exactly


def test_config_c_ids_match_reference():
    g = gold("cfgC_ids.npz")
    cfg = json.loads(str(g["config"]))
    toks = g["tokens"]
    ids = np.concatenate([O.hash_sequence(cfg, toks[:1024]), O.hash_sequence(cfg, toks[1024:], prior=g["prior"])])
    assert (ids == g["ids"]).all()


def test_moduli_above_2_32_match_reference():
    g = gold("bigmod_ids.npz")
    cfg = json.loads(str(g["config"]))
    toks = g["tokens"]
    ids = np.concatenate([O.hash_sequence(cfg, toks[:300]), O.hash_sequence(cfg, toks[300:])])
    assert (ids == g["ids"]).all()


# ---------------------------------------------------------------- banks and embeddings
EMBED = ["embed_tc_none.npz", "embed_tc_scale_sqrt_d.npz", "embed_tc_layer_norm.npz", "embed_simt_v2.npz",
         "embed_simt_v2_k1.npz", "embed_v1.npz", "embed_v1_wide.npz"]


def _bank_for(g):
    cfg = json.loads(str(g["config"]))
    bank = O.make_bank(cfg, int(g["seed"]), round_bf16=True)
    if "ln_gain" in g.files:
        bank.gain[:] = g["ln_gain"]
        bank.bias[:] = g["ln_bias"]
    return cfg, bank


def _run(bank, g, double):
    toks = g["tokens"]
    off = g["seq_offsets"]
    rows, merged = [], []
    for s in range(len(off) - 1):
        prior = g["prior1"] if (s == 1 and "prior1" in g.files) else None
        r, m = O.embed_sequence(bank, toks[off[s]:off[s + 1]], prior=prior, double=double)
        rows.append(r)
        merged.append(m)
    return np.concatenate(rows), np.concatenate(merged)


@pytest.mark.parametrize("name", EMBED)
def test_make_bank_matches_reference(name):  # embedding.hpp:76-110 incl. RNG order
    g = gold(name)
    cfg, bank = _bank_for(g)
    if "ln_gain" in g.files:
        pytest.skip("LN gain/bias overridden after make_bank")
    assert O.bank_checksum(bank) == int(g["bank_checksum"])


@pytest.mark.parametrize("name", EMBED)
def test_embed_float_bitexact_vs_reference(name):  # embedding.hpp:163-201, 239-287, 409-429
    g = gold(name)
    cfg, bank = _bank_for(g)
    rows, merged = _run(bank, g, double=False)
    assert np.array_equal(rows, g["rows_f32"])
    assert np.array_equal(merged, g["merged_f32"])


@pytest.mark.parametrize("name", EMBED)
def test_embed_double_vs_reference(name):  # the reference's own double path at 1e-12 (test_embedding.cpp:72-85)
    g = gold(name)
    cfg, bank = _bank_for(g)
    rows, merged = _run(bank, g, double=True)
    scale = max(1.0, np.abs(g["rows_f64"]).max())
    assert np.abs(rows - g["rows_f64"]).max() <= 1e-12 * scale
    assert np.abs(merged - g["merged_f64"]).max() <= 1e-12 * max(1.0, np.abs(g["merged_f64"]).max())


def test_embed_d3072_vs_reference():
    g = gold("embed_d3072.npz")
    cfg, bank = _bank_for(g)
    assert O.bank_checksum(bank) == int(g["bank_checksum"])
    rows, merged = O.embed_sequence(bank, g["tokens"], double=True)
    assert np.abs(merged - g["merged_f64"]).max() <= 1e-12
    r32, _ = O.embed_sequence(bank, g["tokens"], double=False)
    assert np.array_equal(r32, g["rows_f32"])


def test_split_with_carried_context_equals_whole():  # test_embedding.cpp:155-174
    cfg = O.make_config(32, 12, 3, 2, [13 + 8 * n + 3 * k for n in (2, 3) for k in (1, 2)], "subtable_v2",
                        "scale_sqrt_d")
    bank = O.make_bank(cfg, 11, round_bf16=False)
    rng = O.Rng64(13)
    seq = [rng.below(32) for _ in range(20)]
    whole, _ = O.embed_sequence(bank, seq)
    p1, _ = O.embed_sequence(bank, seq[:7])
    p2, _ = O.embed_sequence(bank, seq[7:], prior=seq[:7])
    assert np.array_equal(whole, np.concatenate([p1, p2]))


# ---------------------------------------------------------------- cache (test_cache.cpp)
def test_append_stream_equals_batch_and_replay_schedules():  # test_cache.cpp:54-65, 128-153
    cfg = O.make_config(32, 8, 3, 2, [23 + 12 * n + 5 * k for n in (2, 3) for k in (1, 2)], "subtable_v2", "none")
    sv = O.sub_vocab_array(cfg)
    rng = O.Rng64(0xCAFE)
    for _ in range(100):
        ring = np.zeros(2, np.uint32)
        confirmed, snaps = [], []
        for _ in range(40):
            r = rng.below(10)
            if r < 6:
                t = rng.below(32)
                ids = np.zeros(4, np.uint64)
                assert O.lib().or_cache_append(ring, 3, 2, 32, sv, t, ids) == 0
                confirmed.append(t)
                want = O.hash_sequence(cfg, confirmed)[-1]
                assert (ids == want).all()
            elif r < 8:
                snaps.append((ring.copy(), len(confirmed)))
            elif snaps:
                pick = rng.below(len(snaps))
                ring = snaps[pick][0].copy()
                confirmed = confirmed[:snaps[pick][1]]
                snaps = snaps[:pick + 1]


def test_draft_verify_golden_is_sequential_appends():  # test_cache.cpp:221-243 semantics, via the oracle
    g = gold("draft_verify.npz")
    cfg = json.loads(str(g["config"]))
    bank = O.make_bank(cfg, int(g["seed"]), round_bf16=True)
    for i in range(int(g["ncases"])):
        prefix, draft, acc = g[f"c{i}_prefix"], g[f"c{i}_draft"], int(g[f"c{i}_accept"])
        seq = np.concatenate([prefix, draft[:acc]]).astype(np.uint32)
        if acc:
            _, merged = O.embed_sequence(bank, seq)
            assert np.array_equal(merged[len(prefix):], g[f"c{i}_accepted"])
        assert int(g[f"c{i}_length"]) == len(prefix) + acc


# ---------------------------------------------------------------- synthetic generator
def test_synthetic_generator_statistics():
    v = O.synth_rows(1234, 5, 1000, 200, 256, 0.02).reshape(-1).astype(np.float64)
    assert abs(v.mean()) < 2e-4 and abs(v.std() - 0.02) < 5e-4
    w = O.synth_rows(1234, 105, 0, 64, 256, 0.02 / 16)
    assert abs(w.std() - 0.02 / 16) < 1e-4


@pytest.mark.parametrize("name", helpers.BACKWARD)
def test_backward_restatement_matches_reference(name):  # embedding.hpp:291-459 in double
    g = gold(name)
    cfg = json.loads(str(g["config"]))
    bank = O.make_bank(cfg, int(g["seed"]), round_bf16=True)
    assert O.bank_checksum(bank) == int(g["bank_checksum"]) or "ln_gain" in g.files
    if "ln_gain" in g.files:
        bank.gain[:], bank.bias[:] = g["ln_gain"], g["ln_bias"]
    off = g["seq_offsets"]
    acc = O.zero_grads(cfg)
    for s, prior in enumerate([None, g["prior1"]]):
        a, b = int(off[s]), int(off[s + 1])
        part = O.embed_sequence_backward(bank, g["tokens"][a:b], g["merged_f64"][a:b], g["upstream"][a:b], prior)
        for k in ("base", "gain", "bias"):
            acc[k] += part[k]
        for k in ("sub", "proj"):
            for x, y in zip(acc[k], part[k]):
                x += y
    ref = helpers.golden_grads(g, O.zero_grads(cfg))
    ln = cfg["amplification"] == "layer_norm"
    for (n, a), (_, b) in zip(helpers.grad_items(acc, ln), helpers.grad_items(ref, ln)):
        assert np.array_equal(a, b), n  # same double operation order as the reference


@pytest.mark.parametrize("name", ["plne_tc.npz", "plne_small.npz"])
def test_plne_restatement_matches_reference(name):  # ple.hpp:76-196 in double
    g = gold(name)
    cfg = json.loads(str(g["config"]))
    bank = O.make_bank(cfg, int(g["seed"]), round_bf16=True)
    assert O.bank_checksum(bank) == int(g["bank_checksum"])
    N, off, toks = cfg["max_order"], g["seq_offsets"], g["tokens"]
    H, dm = g["gate"].shape
    y = np.zeros_like(g["y"])
    dx = np.zeros_like(g["dx"])
    g_gate, g_down = np.zeros((H, dm)), np.zeros((dm, H))
    acc = O.zero_grads(cfg)
    for s, prior in enumerate([None, g["prior1"]]):
        a, b = int(off[s]), int(off[s + 1])
        for pos in range(b - a):
            ctx = O.window(toks[a:b], pos, N, prior)
            y[a + pos] = O.ffn_plne(bank, g["gate"], g["down"], g["x"][a + pos], ctx)
            O.ffn_plne_backward(bank, g["gate"], g["down"], g["x"][a + pos], ctx, g["upstream"][a + pos], g_gate,
                                g_down, acc, dx[a + pos])
    close = lambda a, b: np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max())  # noqa: E731
    assert close(y, g["y"]) and close(dx, g["dx"]) and close(g_gate, g["g_gate"]) and close(g_down, g["g_down"])
    ref = helpers.golden_grads(g, O.zero_grads(cfg))
    for (n, a), (_, b) in zip(helpers.grad_items(acc, False), helpers.grad_items(ref, False)):
        assert close(a, b), n


@pytest.mark.parametrize("name", helpers.ANALYSIS)
def test_analysis_restatement_matches_reference(name):  # analysis.cpp:44-176
    v0, orders, moduli, seqs, (status, meta, seen, distinct, buckets) = helpers.analysis_case(name)
    rc, st = O.corpus_analyze(v0, orders, moduli, seqs)
    assert rc == status
    got = helpers.stats_arrays(st, orders, moduli)
    for a, b in zip(got, (meta, seen, distinct, buckets)):
        np.testing.assert_array_equal(a, b)


def test_analysis_reference_worked_examples():  # test_analysis.cpp:50-113
    def hit(corpus, order, v0, m):
        _, st = O.corpus_analyze(v0, [order], [m], corpus)
        return st["distinct_buckets"][(order, m)] / m

    def coll(corpus, order, v0, m):
        _, st = O.corpus_analyze(v0, [order], [m], corpus)
        return st["distinct_ngrams"][order] - st["distinct_buckets"][(order, m)]

    assert hit([[5]], 2, 10, 100) == pytest.approx(0.01)
    pairs = [[a, b] for a in range(7) for b in range(7)]
    assert hit(pairs, 2, 7, 49) == pytest.approx(1.0) and hit(pairs, 2, 7, 30) == pytest.approx(1.0)
    assert coll([[1, 5], [3, 5], [5, 5]], 2, 10, 20) == 2 and coll([[1, 5], [3, 5], [5, 5]], 2, 10, 23) == 0
    assert coll([list(range(1, 10))], 2, 10, 1000000) == 0
    assert O.corpus_analyze(1 << 17, [8], [100], [[1]])[0] == -1  # V0^order beyond 128 bits


def test_oracle_hash_matches_reference_at_barrett_edge():  # make_golden.py section 17
    g = gold("barrett_edge_ids.npz")
    cfg = gold_config(g)
    off = g["seq_offsets"]
    got = np.concatenate([O.hash_sequence(cfg, g["tokens"][off[i]:off[i + 1]]) for i in range(len(off) - 1)])
    assert np.array_equal(got, g["ids"])


def test_oracle_embed_matches_reference_d3072_regime2_rows():  # make_golden.py section 12 (first rows)
    g = gold("regime2_d3072.npz")
    cfg = gold_config(g)
    hb = O.make_bank(cfg, int(g["seed"]), round_bf16=True)
    assert O.bank_checksum(hb) == int(g["bank_checksum"])
    rows, _ = O.embed_sequence(hb, g["tokens"][:12], double=True)
    assert np.allclose(rows, g["rows_f64_f32"][:12], rtol=0, atol=1e-7 * np.abs(rows).max())
