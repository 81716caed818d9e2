"""Device backward (embed_sequence_backward, embedding.hpp:291-459) vs
the reference's double path: the golden fixtures (tests/golden/backward_*.npz, produced by the
reference itself) and the pinned oracle.  fp32 atomics + fp32 GEMMs: per-tensor relL2 and
max-error bounds in tests/helpers.py (GRAD_REL_L2, GRAD_MAX_RTOL)."""
import json

import numpy as np
import pytest
import torch

import oracle as O
from helpers import BACKWARD, assert_grads_close, dev_i64, dev_u32, gold, golden_grads
from paper_2601_21204_b200 import ngram as G
from paper_2601_21204_b200.abi import OutOfRange

pytestmark = pytest.mark.gpu


def _setup(name, cuda):
    g = gold(name)
    cfg = json.loads(str(g["config"]))
    hb = O.make_bank(cfg, int(g["seed"]), round_bf16=True)
    ln = cfg["amplification"] == "layer_norm"
    if ln:
        hb.gain[:], hb.bias[:] = g["ln_gain"], g["ln_bias"]
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj, hb.gain if ln else None, hb.bias if ln else None)
    prior = np.zeros((2, cfg["max_order"] - 1), np.uint32)
    prior[1] = g["prior1"]
    args = dict(tokens=dev_u32(torch, g["tokens"], cuda), seq_offsets=dev_i64(torch, g["seq_offsets"], cuda),
                upstream=torch.from_numpy(g["upstream"].astype(np.float32)).to(cuda),
                merged=torch.from_numpy(g["merged_f64"].astype(np.float32)).to(cuda),
                prior=dev_u32(torch, prior, cuda) if cfg["max_order"] > 1 else None)
    return g, cfg, hb, db, args, ln


@pytest.mark.parametrize("name", BACKWARD)
def test_backward_matches_reference(cuda, name):
    g, cfg, hb, db, args, ln = _setup(name, cuda)
    gb = G.GradBank(db)
    gb.backward(**args)
    db.sync_errors()
    assert_grads_close(gb.download(), golden_grads(g, O.zero_grads(cfg)), ln)


def test_backward_accumulates_and_zeroes(cuda):
    g, cfg, hb, db, args, ln = _setup("backward_tc_scale_sqrt_d.npz", cuda)
    gb = G.GradBank(db)
    gb.backward(**args)
    gb.backward(**args)
    db.sync_errors()
    ref = golden_grads(g, O.zero_grads(cfg))
    twice = {k: ([2 * x for x in v] if isinstance(v, list) else 2 * v) for k, v in ref.items()}
    assert_grads_close(gb.download(), twice, ln)
    gb.zero()
    torch.cuda.synchronize()
    got = gb.download()
    assert not got["base"].any() and not any(x.any() for x in got["sub"]) and not any(x.any() for x in got["proj"])


def test_skip_amplify_takes_d_merged(cuda):  # embed_backward alone (embedding.hpp:338-376)
    g, cfg, hb, db, args, ln = _setup("backward_tc_scale_sqrt_d.npz", cuda)
    a = G.GradBank(db)
    a.backward(**args)
    b = G.GradBank(db)
    d_pre = args["upstream"] * np.float32(np.sqrt(np.float64(db.D)))  # amplify_backward of scale_sqrt_d
    b.backward(**dict(args, upstream=d_pre), skip_amplify=True)
    db.sync_errors()
    assert_grads_close(b.download(), a.download(), ln)


@pytest.mark.parametrize("mode", [{}, {"exact": True}, {"tf32": True}, {"pedantic": True}])
def test_out_of_range_token_leaves_gradients_untouched(cuda, mode):  # hashing.cpp:49-54
    """A bad call leaves EVERY gradient -- E0, sub-tables and the projection (W_cat) -- exactly as
    it was, including after a good call filled the GEMM workspaces with that call's operands."""
    g, cfg, hb, db, args, ln = _setup("backward_tc_none.npz", cuda)
    gb = G.GradBank(db, **mode)
    bad = args["tokens"].clone()
    bad[77] = cfg["base_vocab"]
    gb.backward(**dict(args, tokens=bad))  # first call: fresh (uninitialised) workspaces
    with pytest.raises(OutOfRange):
        db.sync_errors()
    got = gb.download()
    assert not got["base"].any() and not any(x.any() for x in got["sub"])
    assert not any(x.any() for x in got["proj"])
    gb.backward(**args)  # a good call, then a bad one: the gradients stay those of the good call
    db.sync_errors()
    good = gb.download()
    gb.backward(**dict(args, tokens=bad))
    with pytest.raises(OutOfRange):
        db.sync_errors()
    after = gb.download()
    for k in ("base", "sub", "proj"):
        for x, y in zip(good[k] if isinstance(good[k], list) else [good[k]],
                        after[k] if isinstance(after[k], list) else [after[k]]):
            assert np.array_equal(x, y), k


def test_forward_then_backward_at_longcat_width(cuda):
    """D = 3072, N = 4, K = 4 (12 branches, d = 256): merged from the device forward, then the
    device backward vs the oracle's double backward on the same inputs."""
    cfg = O.make_default_config(1000, 3072, 4, 4)
    hb = O.make_bank(cfg, 5, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    toks = O.uniform_tokens(51, 1000, 48)
    t, off = dev_u32(torch, toks, cuda), dev_i64(torch, [0, 48], cuda)
    _, merged = G.embed_forward(db, t, off, rows=False, merged=True)
    up = torch.from_numpy(np.random.default_rng(4).standard_normal((48, 3072)).astype(np.float32)).to(cuda)
    gb = G.GradBank(db)
    gb.backward(t, off, up, merged=merged)
    db.sync_errors()
    ref = O.embed_sequence_backward(hb, toks, merged.cpu().numpy().astype(np.float64),
                                    up.cpu().numpy().astype(np.float64))
    assert_grads_close(gb.download(), ref, False)


def _densify(rows, vals, cfg):
    """Row-sparse pairs (device storage rows) -> dense per-branch sub-table gradients."""
    sv = O.sub_vocab_array(cfg)
    base = np.concatenate([[0], np.cumsum(sv)]).astype(np.int64)
    d = vals.shape[1]
    dense = [np.zeros((int(v), d)) for v in sv]
    rows = rows.astype(np.int64)
    keep = rows >= 0
    rows, vals = rows[keep], vals[keep].astype(np.float64)
    b = np.searchsorted(base, rows, side="right") - 1
    for i in range(len(sv)):
        m = b == i
        np.add.at(dense[i], rows[m] - base[i], vals[m])
    return dense


@pytest.mark.parametrize("name", ["backward_tc_layer_norm.npz", "backward_v1_wide.npz"])
def test_row_sparse_gradients_sum_to_the_dense_ones(cuda, name):
    g, cfg, hb, db, args, ln = _setup(name, cuda)
    gb = G.GradBank(db, sparse_rows=True)
    gb.backward(**args)
    gb.backward(**args)  # appends: every (position, branch) pair twice
    db.sync_errors()
    rows, vals = gb.sparse()
    assert rows.numel() == 2 * len(g["tokens"]) * db.B
    got = gb.download()
    got["base"] = got["base"] / 2
    got["gain"], got["bias"] = got["gain"] / 2, got["bias"] / 2
    got["proj"] = [p / 2 for p in got["proj"]]
    got["sub"] = [x / 2 for x in _densify(rows.cpu().numpy(), vals.cpu().numpy(), cfg)]
    assert_grads_close(got, golden_grads(g, O.zero_grads(cfg)), ln)
    gb.zero()
    bad = args["tokens"].clone()
    bad[5] = cfg["base_vocab"]
    gb.backward(**dict(args, tokens=bad))
    with pytest.raises(OutOfRange):
        db.sync_errors()
    rows, _ = gb.sparse()
    assert (rows.cpu().numpy() == -1).all()


def test_tf32_backward_within_training_precision(cuda):  # NGRAM_GRAD_TF32
    g, cfg, hb, db, args, ln = _setup("backward_tc_scale_sqrt_d.npz", cuda)
    gb = G.GradBank(db, tf32=True)
    gb.backward(**args)
    db.sync_errors()
    assert_grads_close(gb.download(), golden_grads(g, O.zero_grads(cfg)), ln, rel_l2=3e-3, max_rtol=1e-2)


@pytest.mark.parametrize("name", ["backward_tc_scale_sqrt_d.npz", "backward_tc_layer_norm.npz"])
def test_pedantic_fp32_backward(cuda, name):  # NGRAM_GRAD_PEDANTIC: CUDA-core fp32 GEMMs
    g, cfg, hb, db, args, ln = _setup(name, cuda)
    gb = G.GradBank(db, pedantic=True)
    gb.backward(**args)
    db.sync_errors()
    assert_grads_close(gb.download(), golden_grads(g, O.zero_grads(cfg)), ln)


def test_longcat_scale_sparse_backward_sampled(cuda):
    """Full LongCat width and table scale (D = 3072, N = 4, K = 4, ~19 M sub-table rows,
    counter-based device tables): the row-sparse backward of a 64-token sequence, checked
    entry by entry against double-precision sums over the generator's table values."""
    cfg = O.make_default_config(128000, 3072, 4, 4)  # amplification scale_sqrt_d
    seed, T, D, d, B = 77, 64, 3072, 256, 12
    db = G.DeviceBank(cfg).generate(seed)
    toks = O.uniform_tokens(5, 128000, T)
    up = np.random.default_rng(6).standard_normal((T, D)).astype(np.float32)
    gb = G.GradBank(db, sparse_rows=True)
    t_dev = dev_u32(torch, toks, cuda)
    gb.backward(t_dev, dev_i64(torch, [0, T], cuda), torch.from_numpy(up).to(cuda))
    db.sync_errors()
    rows, vals = (x.cpu().numpy() for x in gb.sparse())
    ids = O.hash_sequence(cfg, toks).astype(np.int64)  # [T][B] bucket ids
    base = np.concatenate([[0], np.cumsum(O.sub_vocab_array(cfg))]).astype(np.int64)
    assert np.array_equal(rows.reshape(T, B), ids + base[:B])  # storage rows, (t, b) order
    # u_t = fp32(1/denom) * (upstream * fp32(sqrt D)) -- amplify_backward then the merge scale
    u = (np.float32(1.0 / 13.0) * (up * np.float32(np.sqrt(D)))).astype(np.float64)
    for t, b in [(0, 0), (17, 5), (63, 11)]:
        w_b = O.synth_rows(seed, 100 + b, 0, D, d, 0.02 / np.sqrt(d)).astype(np.float64)  # W_b [D][d]
        want = u[t] @ w_b
        got = vals[t * B + b]
        assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max()
    g = gb.download()
    for t in (3, 40):  # E0 gradient row of the token: u_t (tokens are distinct here)
        assert np.allclose(g["base"][toks[t]], u[t], rtol=1e-6, atol=1e-12)
    # projection gradient entries: dW_b[i][j] = sum_t u_t[i] * E_b[id_b(t)][j]
    for b, i, j in [(2, 100, 7), (9, 3000, 255)]:
        x = np.stack([O.synth_rows(seed, 1 + b, int(ids[t, b]), 1, d, 0.02)[0] for t in range(T)]).astype(np.float64)
        want = float(u[:, i] @ x[:, j])
        assert abs(g["proj"][b][i, j] - want) <= 1e-5 * max(abs(want), np.abs(u[:, i]).max() * 1e-2)


def test_default_gemms_match_pedantic_at_width(cuda):
    """At D = 3072 (K = 3072 / T = 1024 accumulations) the default tensor-core GEMMs (U in two
    bf16 terms) give the pedantic fp32 gradients to within 1e-5 relL2, and NGRAM_GRAD_EXACT
    (three terms) to within 2e-6; the single-term mode is ~1e-3 (why it is opt-in)."""
    cfg = O.make_default_config(2000, 3072, 4, 4)
    db = G.DeviceBank(cfg).generate(3)
    T = 1024
    gen = torch.Generator(device=cuda).manual_seed(1)
    toks = torch.randint(0, 2000, (T,), dtype=torch.int32, device=cuda, generator=gen)
    off = torch.tensor([0, 512, T], dtype=torch.int64, device=cuda)
    up = torch.randn((T, 3072), device=cuda, generator=gen)
    res = {}
    for name, kw in (("default", {}), ("exact", {"exact": True}), ("pedantic", {"pedantic": True})):
        gb = G.GradBank(db, **kw)
        gb.backward(toks, off, up)
        db.sync_errors()
        d = gb.download()
        res[name] = (np.stack(d["proj"]).astype(np.float64), np.concatenate(d["sub"]).astype(np.float64))
        gb.close()
    errs = {k: [np.linalg.norm(a - b) / np.linalg.norm(b) for a, b in zip(res[k], res["pedantic"])]
            for k in ("default", "exact")}
    print("relL2 vs pedantic (W_cat, sub rows):", errs)
    assert max(errs["default"]) < 1e-5 and max(errs["exact"]) < 2e-6, errs


@pytest.mark.parametrize("name", ["backward_tc_scale_sqrt_d.npz", "backward_tc_layer_norm.npz", "backward_simt_v2.npz"])
def test_sparse_base_equals_dense(cuda, name):
    """NGRAM_GRAD_SPARSE_BASE keeps the E0 gradient as (token, u) pairs: the pairs sum to the dense
    gradient (densified on request), two accumulating calls append, zero() clears."""
    g, cfg, hb, db, args, ln = _setup(name, cuda)
    dense = G.GradBank(db)
    sparse = G.GradBank(db, sparse_base=True)
    for gb in (dense, sparse):
        gb.backward(**args)
        gb.backward(**args)
    db.sync_errors()
    toks, vals = sparse.sparse_base()
    assert toks.numel() == 2 * args["tokens"].numel() and vals.shape[1] == db.D
    a, b = dense.download(), sparse.download()
    # both sums are fp32 atomics in no fixed order: equal to fp32 rounding of the largest terms
    for x, y in zip([a["base"]] + a["sub"] + a["proj"], [b["base"]] + b["sub"] + b["proj"]):
        assert np.abs(x - y).max() <= 1e-5 * max(float(np.abs(x).max()), 1e-30)
    sparse.zero()
    t2, _ = sparse.sparse_base()
    assert t2.numel() == 0 and float(np.abs(sparse.download()["base"]).max()) == 0.0
