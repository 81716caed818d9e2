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


@pytest.mark.parametrize("pedantic", [False, True])  # three-term TF32 (default) / CUDA-core fp32
@pytest.mark.parametrize("name", ["plne_tc.npz", "plne_small.npz"])
def test_plne_forward_matches_reference(cuda, name, pedantic):
    g, cfg, hb, db, a = _setup(name, cuda)
    layer = G.PlneLayer(db, int(g["d_model"]), pedantic=pedantic)
    y = layer.forward(**a)
    db.sync_errors()
    assert_rows_close(y.cpu().numpy(), g["y"])


@pytest.mark.parametrize("pedantic", [False, True])
@pytest.mark.parametrize("name", ["plne_tc.npz", "plne_small.npz"])
def test_plne_backward_matches_reference(cuda, name, pedantic):
    g, cfg, hb, db, a = _setup(name, cuda)
    layer = G.PlneLayer(db, int(g["d_model"]), pedantic=pedantic)
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
