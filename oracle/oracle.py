"""ctypes bindings for the TEST-ONLY checkers under oracle/.

* ``liboracle.so``       -- oracle/ngram_oracle.c, the C restatement of the reference path.
* ``_ref/libngram_ref.so`` -- the unmodified reference sources + oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this module.
The product (paper_2601_21204_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libngram_ref.so")

VARIANTS = {"averaged_v1": 0, "subtable_v2": 1}
AMPS = {"none": 0, "scale_sqrt_d": 1, "layer_norm": 2}

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile liboracle.so (and _ref/ when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_ORACLE = None
_REF = None


def lib():
    global _ORACLE
    if _ORACLE is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.or_rolling_hash.argtypes = [_u32p, C.c_int64, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
        L.or_hash_sequence.argtypes = [_u32p, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_uint64, _u64p,
                                       _u64p]
        L.or_default_sub_vocab.argtypes = [C.c_uint32, C.c_int, C.c_int, _u64p]
        L.or_make_bank_f32.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_int, _u64p, C.c_uint64,
                                       _f32p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p]
        L.or_round_bf16.argtypes = [_f32p, C.c_int64]
        seq_args = [_u32p, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_int,
                    _u64p, _f32p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p]
        L.or_embed_sequence_f32.argtypes = seq_args + [C.c_void_p, _f32p]
        L.or_embed_sequence_f64.argtypes = seq_args + [C.c_void_p, _f64p]
        L.or_embed_sequence_backward_f64.argtypes = [
            _u32p, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_int, _u64p,
            C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
            C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p]
        plne = [C.c_void_p, _u32p, C.c_int, C.c_int, C.c_uint32, C.c_int, C.c_int, _u64p, _f32p,
                C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p, C.c_int]
        L.or_ffn_plne_f64.argtypes = plne + [C.c_void_p]
        L.or_ffn_plne_backward_f64.argtypes = plne + [C.c_void_p] * 4 + [C.POINTER(C.c_void_p)] * 2 + [C.c_void_p]
        an = [C.c_uint64, C.c_void_p, C.c_int, C.c_void_p, C.c_int, _u32p, C.c_void_p, C.c_int64, _u64p, _u64p,
              _u64p, _u64p]
        L.or_corpus_analyze.argtypes = an
        L.or_synth_value.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_float]
        L.or_synth_value.restype = C.c_float
        L.or_synth_scale.argtypes = [C.c_double]
        L.or_synth_scale.restype = C.c_float
        L.or_synth_fill.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32, C.c_float, _f32p]
        L.or_synth_embed_from_ids_f64.argtypes = [C.c_uint64, C.c_uint32, _u64p, C.c_int, C.c_int, C.c_int, _f64p]
        L.or_uniform_below_fill.argtypes = [C.c_uint64, C.c_uint64, _u32p, C.c_int64]
        L.or_cache_append.argtypes = [_u32p, C.c_int, C.c_int, C.c_uint64, _u64p, C.c_uint32, _u64p]
        L.or_hash_throughput_probe.argtypes = [_u32p, C.c_int64, C.c_int, C.c_int, C.c_uint64, _u64p]
        L.or_hash_throughput_probe.restype = C.c_int64
        L.or_rng_new.argtypes = [C.c_uint64]
        L.or_rng_new.restype = C.c_void_p
        L.or_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        L.or_rng_below.restype = C.c_uint64
        L.or_rng_next.argtypes = [C.c_void_p]
        L.or_rng_next.restype = C.c_uint64
        L.or_rng_gaussian.argtypes = [C.c_void_p]
        L.or_rng_gaussian.restype = C.c_double
        L.or_rng_free.argtypes = [C.c_void_p]
        _ORACLE = L
    return _ORACLE


class Rng64:
    """rng64 (std::mt19937_64) + uniform_below / gaussian (rng.hpp:14-40), call by call."""

    def __init__(self, seed):
        self.h = lib().or_rng_new(seed)

    def below(self, bound):
        return int(lib().or_rng_below(self.h, bound))

    def __call__(self):
        return int(lib().or_rng_next(self.h))

    def gaussian(self):
        return float(lib().or_rng_gaussian(self.h))

    def __del__(self):
        try:
            lib().or_rng_free(self.h)
        except Exception:
            pass


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The compiled reference (None-safe callers should check ref_available())."""
    global _REF
    if _REF is None:
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_make_default_config_json.argtypes = [C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int64]
        L.ref_config_validate_json.argtypes = [C.c_char_p]
        L.ref_rolling_hash.argtypes = [_u32p, C.c_int64, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_rolling_hash_cases.argtypes = [C.c_uint64, C.c_int, np.ctypeslib.ndpointer(np.int32), _u64p, _u64p,
                                             _u32p, _u64p]
        L.ref_hash_sequence.argtypes = [C.c_char_p, _u32p, C.c_int64, C.c_void_p, C.c_int64, _u64p]
        L.ref_bank_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int]
        L.ref_bank_create.restype = C.c_void_p
        L.ref_bank_load.argtypes = [C.c_char_p]
        L.ref_bank_load.restype = C.c_void_p
        L.ref_bank_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_bank_destroy.argtypes = [C.c_void_p]
        L.ref_bank_tensor.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int64)]
        L.ref_bank_tensor.restype = C.POINTER(C.c_float)
        L.ref_bank_set_ln.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ref_embed_sequence_f32.argtypes = [C.c_void_p, _u32p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                             C.c_void_p]
        L.ref_embed_sequence_f64.argtypes = [C.c_void_p, _u32p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                             C.c_void_p]
        L.ref_embed_batch_mt.argtypes = [C.c_void_p, _u32p, np.ctypeslib.ndpointer(np.int64), C.c_int, C.c_int,
                                         _f32p]
        L.ref_embed_sequence_backward_f64.argtypes = [C.c_void_p, _u32p, C.c_int64, C.c_void_p, C.c_int64,
                                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                      C.c_void_p, C.c_void_p]
        L.ref_ffn_plne_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, _u32p, C.c_void_p]
        L.ref_ffn_plne_backward_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, _u32p,
                                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_void_p, C.c_void_p]
        L.ref_corpus_analyze.argtypes = [C.c_uint64, C.c_void_p, C.c_int, C.c_void_p, C.c_int, _u32p, C.c_void_p,
                                         C.c_int64, _u64p, _u64p, _u64p, _u64p]
        L.ref_generate_zipf_markov.argtypes = [C.c_uint32, C.c_int64, C.c_int64, C.c_uint64, C.c_double, C.c_double,
                                               _u32p]
        L.ref_cache_create.argtypes = [C.c_char_p]
        L.ref_cache_create.restype = C.c_void_p
        L.ref_cache_destroy.argtypes = [C.c_void_p]
        L.ref_cache_append.argtypes = [C.c_void_p, C.c_uint32, _u64p]
        L.ref_cache_ring.argtypes = [C.c_void_p, _u32p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.ref_draft_verify.argtypes = [C.c_void_p, C.c_void_p, _u32p, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                       _f32p, _u64p]
        L.ref_embed_positions_f64.argtypes = [C.c_void_p, _u32p, np.ctypeslib.ndpointer(np.int64), C.c_int64,
                                              np.ctypeslib.ndpointer(np.int64), C.c_int64, C.c_void_p, C.c_void_p]
        L.ref_decode_mt.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _u32p, C.c_int, _u32p, C.c_int, C.c_int,
                                    C.c_void_p, C.c_int64, _f32p]
        L.ref_hash_all_orders_mt.argtypes = [C.c_char_p, _u32p, C.c_int64, C.c_int, _u64p]
        L.ref_time_calls.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double)]
        _REF = L
    return _REF


# ----------------------------------------------------------------------------- config
def make_config(base_vocab, dim, max_order, sub_tables, sub_vocab, variant="subtable_v2", amplification="none"):
    """ngram_config as the reference's JSON dict (config.cpp:109-122). sub_vocab in branch order."""
    sv = []
    i = 0
    for n in range(2, max_order + 1):
        for k in range(1, sub_tables + 1):
            sv.append({"n": n, "k": k, "vocab": int(sub_vocab[i])})
            i += 1
    return {"max_order": max_order, "sub_tables": sub_tables, "base_vocab": int(base_vocab), "dim": dim,
            "variant": variant, "amplification": amplification, "sub_vocab": sv}


def make_default_config(base_vocab, dim, max_order=4, sub_tables=2):
    """config.cpp:163-183 (restated in ngram_oracle.c:or_default_sub_vocab)."""
    nb = (max_order - 1) * sub_tables
    sv = np.zeros(max(nb, 1), np.uint64)
    lib().or_default_sub_vocab(base_vocab, max_order, sub_tables, sv)
    return make_config(base_vocab, dim, max_order, sub_tables, sv[:nb], "subtable_v2", "scale_sqrt_d")


def sub_vocab_array(cfg):
    """V_{n,k} in branch order b=(n-2)K+(k-1) (config.hpp:48-50)."""
    K = cfg["sub_tables"]
    nb = max((cfg["max_order"] - 1) * K, 0)
    out = np.zeros(max(nb, 1), np.uint64)
    for e in cfg["sub_vocab"]:
        out[(e["n"] - 2) * K + (e["k"] - 1)] = e["vocab"]
    return out


def shape(cfg):
    N, K, D = cfg["max_order"], cfg["sub_tables"], cfg["dim"]
    B = (N - 1) * K if N >= 2 else 0
    v = VARIANTS[cfg["variant"]]
    d = D if (v == 0 or B == 0) else D // B
    denom = N if v == 0 else B + 1
    return N, K, D, B, d, v, denom


def cfg_json(cfg) -> bytes:
    return json.dumps(cfg).encode()


# ----------------------------------------------------------------------------- hashing
def rolling_hash(window, order, base, modulus):
    w = np.ascontiguousarray(window, np.uint32)
    out = C.c_uint64(0)
    rc = lib().or_rolling_hash(w, len(w), order, base, modulus, C.byref(out))
    return rc, out.value


def hash_sequence(cfg, tokens, prior=None):
    N, K, D, B, d, v, denom = shape(cfg)
    t = np.ascontiguousarray(tokens, np.uint32)
    ids = np.zeros((len(t), max(B, 1)), np.uint64)
    pr = None if prior is None else np.ascontiguousarray(prior, np.uint32)
    rc = lib().or_hash_sequence(t, len(t), None if pr is None else pr.ctypes.data, 0 if pr is None else len(pr), N, K,
                                cfg["base_vocab"], sub_vocab_array(cfg), ids)
    if rc:
        raise (IndexError if rc == -2 else ValueError)(f"or_hash_sequence rc={rc}")
    return ids[:, :B]


# ----------------------------------------------------------------------------- banks
class HostBank:
    """Reference-layout float bank (embedding.hpp:31-38) held as numpy arrays."""

    def __init__(self, cfg, base, sub, proj, gain, bias):
        self.cfg, self.base, self.sub, self.proj, self.gain, self.bias = cfg, base, sub, proj, gain, bias

    def _ptrs(self, arrs):
        return (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])


def make_bank(cfg, seed, round_bf16=True):
    """make_bank<float> restated (embedding.hpp:76-110), optionally bf16-rounded."""
    N, K, D, B, d, v, denom = shape(cfg)
    sv = sub_vocab_array(cfg)
    base = np.zeros(cfg["base_vocab"] * D, np.float32)
    sub = [np.zeros(int(sv[b]) * d, np.float32) for b in range(B)]
    proj = [np.zeros(D * d, np.float32) for b in range(B)] if v == 1 else []
    amp = AMPS[cfg["amplification"]]
    gain = np.zeros(D, np.float32) if amp == 2 else np.zeros(0, np.float32)
    bias = np.zeros(D, np.float32) if amp == 2 else np.zeros(0, np.float32)
    sp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in sub])
    pp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in proj])
    lib().or_make_bank_f32(N, K, cfg["base_vocab"], D, v, amp, sv, seed, base, sp, pp,
                           gain.ctypes.data if amp == 2 else None, bias.ctypes.data if amp == 2 else None)
    if round_bf16:
        for a in [base] + sub + proj + [gain, bias]:
            if a.size:
                lib().or_round_bf16(a, a.size)
    return HostBank(cfg, base, sub, proj, gain, bias)


def embed_sequence(bank: HostBank, tokens, prior=None, double=False):
    """embed_sequence_cached restated (embedding.hpp:409-429): (rows, merged), each len x D."""
    cfg = bank.cfg
    N, K, D, B, d, v, denom = shape(cfg)
    t = np.ascontiguousarray(tokens, np.uint32)
    dt = np.float64 if double else np.float32
    rows = np.zeros((len(t), D), dt)
    merged = np.zeros((len(t), D), dt)
    pr = None if prior is None else np.ascontiguousarray(prior, np.uint32)
    sp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in bank.sub])
    pp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in bank.proj])
    fn = lib().or_embed_sequence_f64 if double else lib().or_embed_sequence_f32
    amp = AMPS[cfg["amplification"]]
    rc = fn(t, len(t), None if pr is None else pr.ctypes.data, 0 if pr is None else len(pr), N, K, cfg["base_vocab"],
            D, v, amp, sub_vocab_array(cfg), bank.base, sp, pp, bank.gain.ctypes.data if amp == 2 else None,
            bank.bias.ctypes.data if amp == 2 else None, rows.ctypes.data, merged)
    if rc:
        raise (IndexError if rc == -2 else ValueError)(f"or_embed_sequence rc={rc}")
    return rows, merged


def zero_grads(cfg):
    """zeros_like(bank) in double (embedding.hpp:123-134): the gradient accumulator."""
    N, K, D, B, d, v, denom = shape(cfg)
    sv = sub_vocab_array(cfg)
    return {"base": np.zeros((cfg["base_vocab"], D)), "sub": [np.zeros((int(sv[b]), d)) for b in range(B)],
            "proj": [np.zeros((D, d)) for _ in range(B)] if v == 1 else [], "gain": np.zeros(D), "bias": np.zeros(D)}


def embed_sequence_backward(bank: HostBank, tokens, merged, upstream, prior=None, grads=None):
    """embed_sequence_backward<double> restated (embedding.hpp:438-459) over the float bank:
    amplify_backward then embed_backward per position, accumulated into `grads` (double)."""
    cfg = bank.cfg
    N, K, D, B, d, v, denom = shape(cfg)
    g = grads if grads is not None else zero_grads(cfg)
    t = np.ascontiguousarray(tokens, np.uint32)
    m = np.ascontiguousarray(merged, np.float64)
    u = np.ascontiguousarray(upstream, np.float64)
    pr = None if prior is None else np.ascontiguousarray(prior, np.uint32)
    sp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in bank.sub])
    pp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in bank.proj])
    gsp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in g["sub"]])
    gpp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in g["proj"]])
    amp = AMPS[cfg["amplification"]]
    rc = lib().or_embed_sequence_backward_f64(
        t, len(t), None if pr is None else pr.ctypes.data, 0 if pr is None else len(pr), N, K, cfg["base_vocab"], D, v,
        amp, sub_vocab_array(cfg), sp, pp, bank.gain.ctypes.data if amp == 2 else None, m.ctypes.data, u.ctypes.data,
        g["base"].ctypes.data, gsp, gpp, g["gain"].ctypes.data, g["bias"].ctypes.data)
    if rc:
        raise (IndexError if rc == -2 else ValueError)(f"or_embed_sequence_backward rc={rc}")
    return g


def window(tokens, pos, N, prior=None):
    """detail::fill_context (embedding.hpp:391-405): the N-token window ending at pos."""
    pr = [] if prior is None else list(prior)
    out = []
    for j in range(N):
        i = pos - (N - 1) + j
        if i >= 0:
            out.append(int(tokens[i]))
        else:
            k = len(pr) + i
            out.append(int(pr[k]) if k >= 0 else 0)
    return np.array(out, np.uint32)


def ffn_plne(bank: HostBank, gate, down, x, ctx):
    """ffn_plne<double> restated (ple.hpp:168-181, 76-100): one position."""
    cfg = bank.cfg
    N, K, D, B, d, v, denom = shape(cfg)
    Dm = gate.shape[1]
    y = np.zeros(Dm)
    sp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in bank.sub])
    pp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in bank.proj])
    g64, d64, x64 = (np.ascontiguousarray(a, np.float64) for a in (gate, down, x))
    rc = lib().or_ffn_plne_f64(x64.ctypes.data, np.ascontiguousarray(ctx, np.uint32), N, K, cfg["base_vocab"], D, v,
                               sub_vocab_array(cfg), bank.base, sp, pp, g64.ctypes.data, d64.ctypes.data, Dm,
                               y.ctypes.data)
    if rc:
        raise (IndexError if rc == -2 else ValueError)(f"or_ffn_plne rc={rc}")
    return y


def ffn_plne_backward(bank: HostBank, gate, down, x, ctx, up, g_gate, g_down, grads, dx):
    """ffn_plne_backward<double> restated (ple.hpp:183-196, 102-142); accumulates."""
    cfg = bank.cfg
    N, K, D, B, d, v, denom = shape(cfg)
    Dm = gate.shape[1]
    sp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in bank.sub])
    pp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in bank.proj])
    gsp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in grads["sub"]])
    gpp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in grads["proj"]])
    g64, d64, x64, u64_ = (np.ascontiguousarray(a, np.float64) for a in (gate, down, x, up))
    rc = lib().or_ffn_plne_backward_f64(x64.ctypes.data, np.ascontiguousarray(ctx, np.uint32), N, K,
                                        cfg["base_vocab"], D, v, sub_vocab_array(cfg), bank.base, sp, pp,
                                        g64.ctypes.data, d64.ctypes.data, Dm, u64_.ctypes.data, g_gate.ctypes.data,
                                        g_down.ctypes.data, grads["base"].ctypes.data, gsp, gpp, dx.ctypes.data)
    if rc:
        raise (IndexError if rc == -2 else ValueError)(f"or_ffn_plne_backward rc={rc}")


def bank_checksum(bank: HostBank) -> int:
    """Order-sensitive 64-bit checksum over every tensor's float bits."""
    h = np.uint64(1469598103934665603)
    acc = 0
    for a in [bank.base] + bank.sub + bank.proj + [bank.gain, bank.bias]:
        u = a.view(np.uint32).astype(np.uint64)
        w = np.arange(1, u.size + 1, dtype=np.uint64)
        acc = (acc * 1000003 + int((u * w).sum(dtype=np.uint64))) & 0xFFFFFFFFFFFFFFFF
    del h
    return acc


def uniform_tokens(seed, bound, n):
    """uniform_below(rng64(seed), bound) stream (rng.hpp:26-33)."""
    out = np.zeros(n, np.uint32)
    lib().or_uniform_below_fill(seed, bound, out, n)
    return out


# ----------------------------------------------------------------------------- synthetic bank
def synth_scale(sigma):
    return lib().or_synth_scale(sigma)


def synth_rows(seed, table, row0, nrows, ncols, sigma):
    out = np.zeros(nrows * ncols, np.float32)
    lib().or_synth_fill(seed, table, row0, nrows, ncols, synth_scale(sigma), out)
    return out.reshape(nrows, ncols)


def synth_embed_merged_f64(seed, token, ids, N, K, D):
    out = np.zeros(D, np.float64)
    lib().or_synth_embed_from_ids_f64(seed, int(token), np.ascontiguousarray(ids, np.uint64), N, K, D, out)
    return out


def synth_host_bank(cfg, seed):
    """Materialise the synthetic bank for a SMALL config as a HostBank (reference layout)."""
    N, K, D, B, d, v, denom = shape(cfg)
    sv = sub_vocab_array(cfg)
    base = synth_rows(seed, 0, 0, cfg["base_vocab"], D, 0.02).reshape(-1)
    sub = [synth_rows(seed, 1 + b, 0, int(sv[b]), d, 0.02).reshape(-1) for b in range(B)]
    proj = [synth_rows(seed, 100 + b, 0, D, d, 0.02 / np.sqrt(d)).reshape(-1) for b in range(B)] if v == 1 else []
    amp = AMPS[cfg["amplification"]]
    gain = np.ones(D, np.float32) if amp == 2 else np.zeros(0, np.float32)
    bias = np.zeros(D, np.float32) if amp == 2 else np.zeros(0, np.float32)
    return HostBank(cfg, base, sub, proj, gain, bias)


# ----------------------------------------------------------------------------- analysis
def _flat(seqs):
    off = np.zeros(len(seqs) + 1, np.int64)
    off[1:] = np.cumsum([len(q) for q in seqs])
    toks = np.ascontiguousarray(np.concatenate([np.asarray(q, np.uint32) for q in seqs])
                                if seqs and off[-1] else np.zeros(1, np.uint32), np.uint32)
    return toks, off


def _analyze(fn, v0, orders, moduli, seqs):
    toks, off = _flat(seqs)
    o = (C.c_int * len(orders))(*orders)
    m = (C.c_uint64 * len(moduli))(*moduli)
    meta, seen, dist = np.zeros(2, np.uint64), np.zeros(len(orders), np.uint64), np.zeros(len(orders), np.uint64)
    bk = np.zeros(len(orders) * len(moduli), np.uint64)
    rc = fn(v0, o, len(orders), m, len(moduli), toks, off.ctypes.data, len(seqs), meta, seen, dist, bk)
    return rc, {"sequences_seen": int(meta[0]), "tokens_seen": int(meta[1]),
                "ngrams_seen": {o_: int(seen[i]) for i, o_ in enumerate(orders)},
                "distinct_ngrams": {o_: int(dist[i]) for i, o_ in enumerate(orders)},
                "distinct_buckets": {(o_, m_): int(bk[i * len(moduli) + j]) for i, o_ in enumerate(orders)
                                     for j, m_ in enumerate(moduli)}}


def corpus_analyze(v0, orders, moduli, seqs):
    """corpus_analyzer restated (analysis.cpp:44-176): (status, stats) -- status -2 = a token
    out of range (stats then hold the reference's partial counts)."""
    return _analyze(lib().or_corpus_analyze, v0, orders, moduli, seqs)


def ref_corpus_analyze(v0, orders, moduli, seqs):
    """The reference corpus_analyzer itself (oracle/_ref)."""
    return _analyze(ref().ref_corpus_analyze, v0, orders, moduli, seqs)


def ref_zipf_markov(vocab, sequences, seq_len, seed, exponent=1.1, markov_prob=0.35):
    out = np.zeros(sequences * seq_len, np.uint32)
    assert ref().ref_generate_zipf_markov(vocab, sequences, seq_len, seed, exponent, markov_prob, out) == 0
    return [out[i * seq_len:(i + 1) * seq_len] for i in range(sequences)]
