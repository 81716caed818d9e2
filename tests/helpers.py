"""Shared test helpers: fixture loading, device buffers, the stated tolerances."""
import json
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# ---------------------------------------------------------------- tolerance contract
# Tensor-core path (bf16 tables, fp32 TMEM accumulation, different summation order than the
# reference's sequential float loop), compared with the reference's double path on the same
# bf16-representable bank:
ROW_RTOL = 1e-5   # per row: max |err| <= ROW_RTOL * max |ref row|
REL_L2 = 1e-6     # whole output: ||err||_2 <= REL_L2 * ||ref||_2
BF16_REL = 2.0 ** -8  # bf16 output: additionally |err| <= 2^-8 |ref| per element


class Gold(dict):
    """An .npz fixture fully loaded (NpzFile re-decompresses on every key access)."""

    @property
    def files(self):
        return list(self.keys())


def gold(name):
    with np.load(os.path.join(GOLD, name), allow_pickle=False) as z:
        return Gold({k: z[k] for k in z.files})


def gold_config(g):
    return json.loads(str(g["config"]))


def assert_rows_close(got, ref, bf16=False, row_rtol=ROW_RTOL, rel_l2=REL_L2):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape
    err = np.abs(got - ref)
    rowmax = np.abs(ref).max(axis=1, keepdims=True) + 1e-30
    if bf16:
        bound = BF16_REL * np.abs(ref) + row_rtol * rowmax
        assert (err <= bound).all(), f"bf16 max excess {(err - bound).max()}"
    else:
        worst = (err / rowmax).max()
        assert worst <= row_rtol, f"per-row max err {worst:.3e} > {row_rtol}"
        rel = np.linalg.norm(got - ref) / (np.linalg.norm(ref) + 1e-30)
        assert rel <= rel_l2, f"relL2 {rel:.3e} > {rel_l2}"


def bf16_to_f32(u16):
    return (np.asarray(u16, np.uint16).astype(np.uint32) << 16).view(np.float32)


def dev_u32(torch, a, device):
    """uint32 host array -> int32 device tensor with the same bits."""
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(device)


def dev_i64(torch, a, device):
    return torch.from_numpy(np.ascontiguousarray(a, np.int64)).to(device)


def u64(t):
    """int64 device/host tensor holding u64 bits -> numpy uint64."""
    return t.cpu().numpy().view(np.uint64) if hasattr(t, "cpu") else np.asarray(t).view(np.uint64)


# ---------------------------------------------------------------- backward (gradients)
# Device backward: fp32 atomics + fp32 GEMMs vs the reference's double path.  Per gradient
# tensor: ||err||_2 <= GRAD_REL_L2 * ||ref||_2 and max |err| <= GRAD_MAX_RTOL * max |ref|.
GRAD_REL_L2 = 1e-5
GRAD_MAX_RTOL = 1e-5
BACKWARD = ["backward_tc_none.npz", "backward_tc_scale_sqrt_d.npz", "backward_tc_layer_norm.npz",
            "backward_simt_v2.npz", "backward_v1_wide.npz"]


def golden_grads(g, zero):
    """Dense gradients (reference layout) from a backward fixture's sparse storage."""
    out = {k: ([x.copy() for x in v] if isinstance(v, list) else v.copy()) for k, v in zero.items()}
    out["base"][g["g_base_idx"]] = g["g_base_val"]
    for b in range(len(out["sub"])):
        out["sub"][b][g[f"g_sub{b}_idx"]] = g[f"g_sub{b}_val"]
    if "g_proj" in g.files:
        for b in range(len(out["proj"])):
            out["proj"][b][:] = g["g_proj"][b]
    if "g_gain" in g.files:
        out["gain"][:], out["bias"][:] = g["g_gain"], g["g_bias"]
    return out


def grad_items(gr, ln):
    yield "base", gr["base"]
    for b, x in enumerate(gr["sub"]):
        yield f"sub{b}", x
    for b, x in enumerate(gr["proj"]):
        yield f"proj{b}", x
    if ln:
        yield "gain", gr["gain"]
        yield "bias", gr["bias"]


def assert_grads_close(got, ref, ln, rel_l2=GRAD_REL_L2, max_rtol=GRAD_MAX_RTOL):
    for (name, a), (_, b) in zip(grad_items(got, ln), grad_items(ref, ln)):
        a = np.asarray(a, np.float64)
        b = np.asarray(b, np.float64)
        assert a.shape == b.shape, name
        err = np.abs(a - b)
        scale = np.abs(b).max() + 1e-30
        assert err.max() <= max_rtol * scale, f"{name}: max err {err.max() / scale:.3e} of max|ref|"
        rel = np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30)
        assert rel <= rel_l2, f"{name}: relL2 {rel:.3e}"


ANALYSIS = ["worked20", "single", "allpairs", "zipf1000", "random", "badtoken", "bigmod", "wide_v0", "order100",
            "empty_seqs"]


def analysis_case(name):
    """(v0, orders, moduli, sequences, expected (status, meta, seen, distinct, buckets)) of a
    tests/golden/analysis_*.npz made by the reference corpus_analyzer."""
    g = gold(f"analysis_{name}.npz")
    off = g["seq_offsets"]
    seqs = [g["tokens"][off[i]:off[i + 1]] for i in range(len(off) - 1)]
    return (int(g["v0"]), [int(o) for o in g["orders"]], [int(m) for m in g["moduli"]], seqs,
            (int(g["status"]), g["meta"], g["seen"], g["distinct"], g["buckets"]))


def stats_arrays(st, orders, moduli):
    return (np.array([st["sequences_seen"], st["tokens_seen"]], np.uint64),
            np.array([st["ngrams_seen"][o] for o in orders], np.uint64),
            np.array([st["distinct_ngrams"][o] for o in orders], np.uint64),
            np.array([st["distinct_buckets"][(o, m)] for o in orders for m in moduli], np.uint64))
