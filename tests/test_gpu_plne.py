"""Per-layer N-gram FFN (PLNE, ple.hpp:168-196) on the device vs the
reference's double path (tests/golden/plne_*.npz, produced by the reference) and the pinned
oracle.  fp32 GEMMs: outputs within the forward tolerance contract, gradients within the
backward one (tests/helpers.py)."""
import json

import numpy as np
import pytest
import torch

import oracle as O
from helpers import assert_grads_close, assert_rows_close, dev_i64, dev_u32, gold, golden_grads
from paper_2601_21204_b200 import ngram as G
from paper_2601_21204_b200.abi import InvalidArgument, OutOfRange

pytestmark = pytest.mark.gpu


def _f32(a, cuda):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(cuda)


def _setup(name, cuda):
    g = gold(name)
    cfg = json.loads(str(g["config"]))
    hb = O.make_bank(cfg, int(g["seed"]), round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    N = cfg["max_order"]
    prior = np.zeros((2, N - 1), np.uint32)
    prior[1] = g["prior1"]
    a = dict(gate=_f32(g["gate"], cuda), down=_f32(g["down"], cuda), x=_f32(g["x"], cuda),
             tokens=dev_u32(torch, g["tokens"], cuda), seq_offsets=dev_i64(torch, g["seq_offsets"], cuda),
             prior=dev_u32(torch, prior, cuda))
    return g, cfg, hb, db, a


@pytest.mark.parametrize("fast", [False, True])  # pedantic fp32 / split-bf16 tensor cores (default)
@pytest.mark.parametrize("name", ["plne_tc.npz", "plne_small.npz"])
def test_plne_forward_matches_reference(cuda, name, fast):
    g, cfg, hb, db, a = _setup(name, cuda)
    layer = G.PlneLayer(db, int(g["d_model"]), fast=fast)
    y = layer.forward(**a)
    db.sync_errors()
    assert_rows_close(y.cpu().numpy(), g["y"])


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("name", ["plne_tc.npz", "plne_small.npz"])
def test_plne_backward_matches_reference(cuda, name, fast):
    g, cfg, hb, db, a = _setup(name, cuda)
    layer = G.PlneLayer(db, int(g["d_model"]), fast=fast)
    gb = G.GradBank(db)
    d_gate = torch.zeros_like(a["gate"])
    d_down = torch.zeros_like(a["down"])
    dx = torch.zeros_like(a["x"])
    layer.backward(a["gate"], a["down"], a["x"], a["tokens"], a["seq_offsets"], _f32(g["upstream"], cuda), d_gate,
                   d_down, dx, bank_grads=gb, prior=a["prior"])
    db.sync_errors()
    assert_grads_close({"base": d_gate.cpu().numpy(), "sub": [d_down.cpu().numpy(), dx.cpu().numpy()], "proj": []},
                       {"base": g["g_gate"], "sub": [g["g_down"], g["dx"]], "proj": []}, False)
    assert_grads_close(gb.download(), golden_grads(g, O.zero_grads(cfg)), False)


def test_ple_is_plne_with_a_base_only_bank(cuda):  # test_ple.cpp:150-172
    cfg = O.make_config(300, 256, 1, 1, [], "subtable_v2", "none")
    hb = O.make_bank(cfg, 3, round_bf16=True)  # E0 plays the PLE table
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    r = np.random.default_rng(5)
    dm = 64
    gate = (0.02 * r.standard_normal((256, dm))).astype(np.float32)
    down = (0.02 * r.standard_normal((dm, 256))).astype(np.float32)
    toks = O.uniform_tokens(71, 300, 40)
    x = r.standard_normal((40, dm)).astype(np.float32)
    layer = G.PlneLayer(db, dm)
    y = layer.forward(_f32(gate, cuda), _f32(down, cuda), _f32(x, cuda), dev_u32(torch, toks, cuda),
                      dev_i64(torch, [0, 40], cuda)).cpu().numpy()
    want = np.stack([O.ffn_plne(hb, gate, down, x[i], toks[i:i + 1]) for i in range(40)])
    assert_rows_close(y, want)


def test_plne_validates_the_layer_bank_and_tokens(cuda):  # test_ple.cpp:174-181, hashing.cpp:49-54
    with pytest.raises(InvalidArgument):
        G.PlneLayer(G.DeviceBank(O.make_default_config(100, 256, 3, 2)).generate(1), 64)  # amp scale_sqrt_d
    g, cfg, hb, db, a = _setup("plne_small.npz", cuda)
    layer = G.PlneLayer(db, int(g["d_model"]))
    bad = a["tokens"].clone()
    bad[3] = cfg["base_vocab"]
    layer.forward(**dict(a, tokens=bad))
    with pytest.raises(OutOfRange):
        db.sync_errors()


def test_split_bf16_gemms_match_fp64_at_width(cuda):
    """At a LongCat-like width (d_model = hidden = 3072, K = 3072 accumulations), vs an fp64
    evaluation: the default split-bf16 tensor-core GEMMs within 2e-6 relL2 and the pedantic
    CUDA-core fp32 ones (NGRAM_PLNE_PEDANTIC) within 1e-6 (forward and the gate / down / x
    gradients).  (A three-term
    TF32 split measured 1.5e-5 here and was dropped.)"""
    cfg = O.make_default_config(500, 3072, 3, 2)
    cfg["amplification"] = "none"
    db = G.DeviceBank(cfg).generate(11)
    T, Dm, H = 256, 3072, 3072
    gen = torch.Generator(device=cuda).manual_seed(5)
    toks = torch.randint(0, 500, (T,), dtype=torch.int32, device=cuda, generator=gen)
    off = torch.tensor([0, 100, T], dtype=torch.int64, device=cuda)
    gate = 0.02 * torch.randn((H, Dm), device=cuda, generator=gen)
    down = 0.02 * torch.randn((Dm, H), device=cuda, generator=gen)
    x = torch.randn((T, Dm), device=cuda, generator=gen)
    up = torch.randn((T, Dm), device=cuda, generator=gen)
    _, g = G.embed_forward(db, toks, off, rows=False, merged=True)  # the layer bank's g (fp32)
    # fp64 reference of ple.hpp:168-196 on the same fp32 inputs
    gd, dn, xd, ud, g64 = (t.double() for t in (gate, down, x, up, g))
    u = xd @ gd.T
    sg = torch.sigmoid(u)
    hh = u * sg * g64
    y_ref = hh @ dn.T
    dhh = ud @ dn
    dd_ref = ud.T @ hh
    du = dhh * g64 * (sg * (1 + u * (1 - sg)))
    dg_ref = du.T @ xd
    dx_ref = du @ gd
    refs = (y_ref, dg_ref, dd_ref, dx_ref)
    errs = {}
    for fast in (True, False):
        layer = G.PlneLayer(db, Dm, fast=fast)
        y = layer.forward(gate, down, x, toks, off)
        dg, dd, dx = torch.zeros_like(gate), torch.zeros_like(down), torch.zeros_like(x)
        layer.backward(gate, down, x, toks, off, up, dg, dd, dx)
        db.sync_errors()
        errs[fast] = [float((a.double() - r).norm() / r.norm()) for a, r in zip((y, dg, dd, dx), refs)]
    print("relL2 vs fp64 (split-bf16, pedantic):", errs[True], errs[False])
    for ef, ep in zip(errs[True], errs[False]):
        assert ef < 2e-6 and ep < 1e-6, errs
