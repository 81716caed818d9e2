"""Python mirror of the reference's hot-path API, backed by the C-ABI.

Names and argument meaning follow proj/include/ngram/*.hpp so the parity tests read
like the reference's own doctest suites:

    reference (C++)                          here
    ---------------------------------------  ------------------------------------------
    make_default_config (config.cpp:163)     make_default_config
    ngram_config::validate (config.cpp:32)   validate_config
    rolling_hash (hashing.cpp:33)            rolling_hash / rolling_hash_batch
    hash_all_orders (hashing.cpp:61)         hash_all_orders / hash_ids (batched)
    embedding_bank_t (embedding.hpp:31)      DeviceBank (device-resident, bf16)
    embed_from_ids (embedding.hpp:163)       embed_from_ids
    embed_sequence(_cached) (:409-436)       embed_sequence / embed_sequence_cached (host
                                             buffers) and embed_forward (device buffers)
    sequence_cache (cache.hpp:38)            SequenceCache (one stream) / DecodeState (batch)
    draft_verify (cache.cpp:152)             draft_verify / DecodeState.verify + commit

Exceptions: InvalidArgument (std::invalid_argument), OutOfRange (std::out_of_range),
IoError, ParseError, ConfigError -- see abi.py.  torch is used only to own device
memory and streams; every computation is a CUDA kernel behind the C-ABI.
"""
from __future__ import annotations

import ctypes as C
import json
from typing import Optional, Sequence

import numpy as np
import torch

from . import abi
from .abi import InvalidArgument, OutOfRange, check

VARIANTS = {"averaged_v1": 0, "subtable_v2": 1}
AMPS = {"none": 0, "scale_sqrt_d": 1, "layer_norm": 2}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


# ----------------------------------------------------------------------------- config
def make_default_config(base_vocab: int, dim: int, max_order: int = 4, sub_tables: int = 2) -> dict:
    buf = C.create_string_buffer(1 << 16)
    check(abi.lib().ngram_make_default_config(base_vocab, dim, max_order, sub_tables, buf, len(buf)))
    return json.loads(buf.value)


def validate_config(cfg: dict) -> None:
    check(abi.lib().ngram_config_validate(json.dumps(cfg).encode()))


def branch_count(cfg) -> int:
    return 0 if cfg["max_order"] < 2 else (cfg["max_order"] - 1) * cfg["sub_tables"]


def branch_dim(cfg) -> int:
    B = branch_count(cfg)
    return cfg["dim"] if (cfg["variant"] == "averaged_v1" or B == 0) else cfg["dim"] // B


# ----------------------------------------------------------------------------- bank
class DeviceBank:
    """Device-resident embedding bank (bf16 tables, W_cat, E0)."""

    def __init__(self, cfg: dict, device: int = 0, shard_rank: int = 0, shard_count: int = 1, tables: bool = True):
        self.cfg = cfg
        self.device = device
        h = C.c_void_p()
        flags = 0 if tables else abi.NGRAM_BANK_HASH_ONLY
        check(abi.lib().ngram_bank_create_ex(json.dumps(cfg).encode(), device, shard_rank, shard_count, flags,
                                             C.byref(h)))
        self.handle = h
        self.info = abi.BankInfo()
        check(abi.lib().ngram_bank_get_info(self.handle, C.byref(self.info)))
        self.D = self.info.dim
        self.B = self.info.branch_count
        self.N = self.info.max_order

    def close(self):
        if self.handle:
            abi.lib().ngram_bank_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def tensor_core_path(self) -> bool:
        return bool(self.info.tensor_core_path)

    def upload(self, base: np.ndarray, sub: Sequence[np.ndarray], proj: Sequence[np.ndarray] = (),
               ln_gain: Optional[np.ndarray] = None, ln_bias: Optional[np.ndarray] = None) -> "DeviceBank":
        """Upload a reference-layout float bank (make_bank / load_bank) from host memory."""
        keep = [np.ascontiguousarray(a, np.float32) for a in [base] + list(sub) + list(proj)]
        base_a, sub_a, proj_a = keep[0], keep[1:1 + len(sub)], keep[1 + len(sub):]
        sp = (C.c_void_p * max(len(sub_a), 1))(*[a.ctypes.data for a in sub_a])
        pp = (C.c_void_p * max(len(proj_a), 1))(*[a.ctypes.data for a in proj_a])
        g = None if ln_gain is None else np.ascontiguousarray(ln_gain, np.float32)
        b = None if ln_bias is None else np.ascontiguousarray(ln_bias, np.float32)
        check(abi.lib().ngram_bank_upload_f32(self.handle, base_a.ctypes.data, sp, pp if proj_a else None,
                                              None if g is None else g.ctypes.data,
                                              None if b is None else b.ctypes.data))
        return self

    def generate(self, seed: int, stream=None) -> "DeviceBank":
        """Synthetic counter-based bank, generated on the device (LongCat-scale)."""
        check(abi.lib().ngram_bank_generate(self.handle, seed, _stream(stream)))
        return self

    def load_file(self, path: str) -> "DeviceBank":
        check(abi.lib().ngram_bank_load_file(self.handle, path.encode()))
        return self

    def reserve(self, max_tokens: int) -> None:
        check(abi.lib().ngram_bank_reserve(self.handle, max_tokens))

    def sync_errors(self, stream=None) -> None:
        check(abi.lib().ngram_sync_errors(self.handle, _stream(stream)))


# ----------------------------------------------------------------------------- hashing
def rolling_hash_batch(windows: torch.Tensor, orders: torch.Tensor, bases: torch.Tensor, moduli: torch.Tensor,
                       lengths: Optional[torch.Tensor] = None, stream=None):
    """Batched rolling_hash on device. windows: [count, stride] uint32 (int32 storage)."""
    count, stride = windows.shape
    out = torch.empty(count, dtype=torch.int64, device=windows.device)
    status = torch.empty(count, dtype=torch.int32, device=windows.device)
    check(abi.lib().ngram_rolling_hash_batch(_ptr(windows), stride, _ptr(lengths), _ptr(orders), _ptr(bases),
                                             _ptr(moduli), count, _ptr(out), _ptr(status), _stream(stream)))
    return out, status


def rolling_hash(window: Sequence[int], spec: tuple, device: int = 0) -> int:
    """rolling_hash(window, hash_spec{order, base, modulus}) with the reference's exceptions."""
    order, base, modulus = spec
    w = list(window)
    dev = torch.device("cuda", device)
    wt = torch.tensor([w + [0] * (max(len(w), 1) - len(w))], dtype=torch.int64).to(torch.int32).to(dev)
    if len(w) == 0:
        wt = torch.zeros((1, 1), dtype=torch.int32, device=dev)
    lens = torch.tensor([len(w)], dtype=torch.int32, device=dev)
    orders = torch.tensor([order], dtype=torch.int32, device=dev)
    bases = torch.tensor([np.uint64(base).astype(np.int64)], dtype=torch.int64, device=dev)
    mods = torch.tensor([np.uint64(modulus).astype(np.int64)], dtype=torch.int64, device=dev)
    out, status = rolling_hash_batch(wt, orders, bases, mods, lens)
    st = int(status.item())
    if st == abi.NGRAM_EINVAL:
        raise InvalidArgument("rolling_hash: invalid hash_spec or window length")
    if st == abi.NGRAM_ERANGE:
        raise OutOfRange("rolling_hash: token out of range for base vocabulary")
    return int(np.int64(out.item()).astype(np.uint64))


def hash_ids(bank: DeviceBank, tokens: torch.Tensor, seq_offsets: torch.Tensor, prior: Optional[torch.Tensor] = None,
             u64: bool = True, stream=None) -> torch.Tensor:
    """hash_all_orders at every position of a batch (device tensors). -> [T, B] ids."""
    T = tokens.numel()
    nseq = seq_offsets.numel() - 1
    out = torch.empty((T, bank.B), dtype=torch.int64 if u64 else torch.int32, device=tokens.device)
    check(abi.lib().ngram_hash_ids(bank.handle, _ptr(tokens), _ptr(seq_offsets), nseq, T, _ptr(prior), _ptr(out),
                                   1 if u64 else 0, _stream(stream)))
    return out


def hash_all_orders(context: Sequence[int], bank: DeviceBank) -> list:
    """hash_all_orders(context, cfg) for one N-token context (reference signature)."""
    N = bank.N
    if len(context) != N:
        raise InvalidArgument(f"hash_all_orders: context length {len(context)} does not match max order {N}")
    dev = torch.device("cuda", bank.device)
    toks = torch.tensor([context[-1]], dtype=torch.int64).to(torch.int32).to(dev)
    prior = torch.tensor([list(context[:-1])], dtype=torch.int64).to(torch.int32).to(dev) if N > 1 else None
    off = torch.tensor([0, 1], dtype=torch.int64, device=dev)
    ids = hash_ids(bank, toks, off, prior)
    bank.sync_errors()
    return [int(x) for x in ids[0].cpu().numpy().astype(np.uint64)]


# ----------------------------------------------------------------------------- forward
_DT = {torch.float32: abi.NGRAM_F32, torch.bfloat16: abi.NGRAM_BF16}


def embed_forward(bank: DeviceBank, tokens: torch.Tensor, seq_offsets: torch.Tensor,
                  prior: Optional[torch.Tensor] = None, rows: bool = True, merged: bool = False,
                  out_dtype=torch.float32, stream=None, out_rows: Optional[torch.Tensor] = None,
                  out_merged: Optional[torch.Tensor] = None):
    """Batched embed_sequence_cached on device tensors. Returns (rows, merged) (None if not requested)."""
    T = tokens.numel()
    nseq = seq_offsets.numel() - 1
    dev = tokens.device
    if rows and out_rows is None:
        out_rows = torch.empty((T, bank.D), dtype=out_dtype, device=dev)
    if merged and out_merged is None:
        out_merged = torch.empty((T, bank.D), dtype=out_dtype, device=dev)
    check(abi.lib().ngram_embed_forward(bank.handle, _ptr(tokens), _ptr(seq_offsets), nseq, T, _ptr(prior),
                                        _ptr(out_rows if rows else None), _ptr(out_merged if merged else None),
                                        _DT[out_dtype], _stream(stream)))
    return (out_rows if rows else None), (out_merged if merged else None)


def embed_from_ids(bank: DeviceBank, tokens: torch.Tensor, ids: torch.Tensor, out_dtype=torch.float32,
                   stream=None) -> torch.Tensor:
    """embed_from_ids for T tokens (device): ids [T, B] int64 (u64 bits) -> merged [T, D]."""
    T = tokens.numel()
    out = torch.empty((T, bank.D), dtype=out_dtype, device=tokens.device)
    check(abi.lib().ngram_embed_from_ids(bank.handle, _ptr(tokens), _ptr(ids), T, _ptr(out), _DT[out_dtype],
                                         _stream(stream)))
    return out


def embed_sequence_cached(bank: DeviceBank, tokens: Sequence[int], prior_context: Sequence[int] = (),
                          out_dtype=np.float32):
    """embed_sequence_cached (host buffers in and out): (rows, merged), each len x D."""
    return embed_batch_host(bank, [tokens], [prior_context], want_rows=True, want_merged=True, out_dtype=out_dtype)


def embed_sequence(bank: DeviceBank, tokens: Sequence[int], prior_context: Sequence[int] = ()) -> np.ndarray:
    return embed_batch_host(bank, [tokens], [prior_context], want_rows=True, want_merged=False)[0]


def _prior_matrix(N1: int, priors) -> Optional[np.ndarray]:
    if N1 <= 0 or priors is None or all(len(p) == 0 for p in priors):
        return None
    m = np.zeros((len(priors), N1), np.uint32)
    for i, p in enumerate(priors):
        tail = list(p)[-N1:]
        if tail:
            m[i, N1 - len(tail):] = np.asarray(tail, np.uint32)
    return m


def embed_batch_host(bank: DeviceBank, seqs, priors=None, want_rows=True, want_merged=False, out_dtype=np.float32,
                     out_rows: Optional[np.ndarray] = None, out_merged: Optional[np.ndarray] = None):
    """The host-buffer C-ABI entry (ngram_embed_sequence_host) over a list of sequences."""
    lens = [len(s) for s in seqs]
    off = np.zeros(len(seqs) + 1, np.int64)
    off[1:] = np.cumsum(lens)
    T = int(off[-1])
    toks = np.ascontiguousarray(np.concatenate([np.asarray(s, np.uint32) for s in seqs]) if T else
                                np.zeros(1, np.uint32))
    pm = _prior_matrix(bank.N - 1, priors)
    odt = abi.NGRAM_F32 if out_dtype == np.float32 else abi.NGRAM_BF16
    npdt = np.float32 if odt == abi.NGRAM_F32 else np.uint16
    rows = out_rows if out_rows is not None else (np.empty((T, bank.D), npdt) if want_rows else None)
    merged = out_merged if out_merged is not None else (np.empty((T, bank.D), npdt) if want_merged else None)
    check(abi.lib().ngram_embed_sequence_host(bank.handle, toks.ctypes.data, off.ctypes.data, len(seqs),
                                              None if pm is None else pm.ctypes.data,
                                              None if rows is None else rows.ctypes.data,
                                              None if merged is None else merged.ctypes.data, odt))
    return rows, merged


# ----------------------------------------------------------------------------- decode
class DecodeState:
    """A batch of device-resident sequence_cache streams (cache.hpp:38-80)."""

    def __init__(self, bank: DeviceBank, batch: int, max_draft: int = 8):
        self.bank, self.batch, self.max_draft = bank, batch, max_draft
        h = C.c_void_p()
        check(abi.lib().ngram_decode_create(bank.handle, batch, max_draft, C.byref(h)))
        self.handle = h
        self.dev = torch.device("cuda", bank.device)

    def close(self):
        if self.handle:
            abi.lib().ngram_decode_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self, prior: Optional[torch.Tensor] = None, lengths: Optional[torch.Tensor] = None, stream=None):
        check(abi.lib().ngram_decode_reset(self.handle, _ptr(prior), _ptr(lengths), _stream(stream)))

    def step(self, tokens: torch.Tensor, want_ids=True, want_merged=True, out_dtype=torch.float32, stream=None,
             out: Optional[torch.Tensor] = None):
        ids = torch.empty((self.batch, self.bank.B), dtype=torch.int64, device=self.dev) if want_ids else None
        if want_merged and out is None:
            out = torch.empty((self.batch, self.bank.D), dtype=out_dtype, device=self.dev)
        check(abi.lib().ngram_decode_step(self.handle, _ptr(tokens), _ptr(ids), _ptr(out if want_merged else None),
                                          _DT[out_dtype], _stream(stream)))
        return ids, (out if want_merged else None)

    def verify(self, draft: torch.Tensor, out_dtype=torch.float32, stream=None, out: Optional[torch.Tensor] = None):
        L = draft.shape[1]
        if out is None:
            out = torch.empty((self.batch, L, self.bank.D), dtype=out_dtype, device=self.dev)
        check(abi.lib().ngram_verify_block(self.handle, _ptr(draft), L, _ptr(out), _DT[out_dtype], _stream(stream)))
        return out

    def commit(self, draft: torch.Tensor, accept: torch.Tensor, stream=None):
        check(abi.lib().ngram_commit(self.handle, _ptr(draft), draft.shape[1], _ptr(accept), _stream(stream)))

    def rings(self, stream=None) -> torch.Tensor:
        """Device copy of the rings [batch, N-1] (int32 storage): the decode windows' prior."""
        R = max(self.bank.N - 1, 0)
        out = torch.empty((self.batch, max(R, 1)), dtype=torch.int32, device=self.dev)[:, :R]
        check(abi.lib().ngram_decode_copy_ring(self.handle, _ptr(out), _stream(stream)))
        return out

    def state(self):
        R = max(self.bank.N - 1, 0)
        ring = np.zeros((self.batch, max(R, 1)), np.uint32)
        length = np.zeros(self.batch, np.uint64)
        last = np.zeros(self.batch, np.uint32)
        check(abi.lib().ngram_decode_get_state(self.handle, ring.ctypes.data, length.ctypes.data, last.ctypes.data))
        return ring[:, :R], length, last


class SequenceCache:
    """sequence_cache (cache.hpp:38-80) for one stream, state resident on the device.

    snapshot/rollback/discard keep the reference's handle semantics (cache.cpp:59-96);
    a snapshot is a copy of the device ring state."""

    _uid = 0

    def __init__(self, bank: DeviceBank, max_draft: int = 8):
        self.bank = bank
        self.st = DecodeState(bank, 1, max_draft)
        SequenceCache._uid += 1
        self.uid = SequenceCache._uid
        self.snaps = []
        self.next_serial = 1

    def append(self, token: int) -> list:
        if int(token) >= self.bank.info.base_vocab:
            raise OutOfRange(f"sequence_cache: token {token} out of range")
        t = torch.tensor([int(token)], dtype=torch.int64).to(torch.int32).to(self.st.dev)
        ids, _ = self.st.step(t, want_ids=True, want_merged=False)
        self.bank.sync_errors()
        return [int(x) for x in ids[0].cpu().numpy().astype(np.uint64)]

    def ring(self):
        return self.st.state()[0][0]

    def length(self) -> int:
        return int(self.st.state()[1][0])

    def last_token(self) -> int:
        return int(self.st.state()[2][0])

    def snapshot_depth(self) -> int:
        return len(self.snaps)

    def snapshot(self):
        ring, length, last = self.st.state()
        serial = self.next_serial
        self.next_serial += 1
        self.snaps.append((serial, ring.copy(), length.copy()))
        return (self.uid, serial, len(self.snaps) - 1)

    def _check(self, h):
        owner, serial, slot = h
        if owner != self.uid:
            raise InvalidArgument("sequence_cache: handle belongs to another state")
        if slot >= len(self.snaps) or self.snaps[slot][0] != serial:
            raise InvalidArgument("sequence_cache: stale snapshot handle")

    def rollback(self, h):
        self._check(h)
        _, ring, length = self.snaps[h[2]]
        R = self.bank.N - 1
        prior = torch.from_numpy(ring.astype(np.int64)).to(torch.int32).to(self.st.dev) if R > 0 else None
        lens = torch.from_numpy(length.astype(np.int64)).to(self.st.dev)
        self.st.reset(prior, lens)
        del self.snaps[h[2] + 1:]

    def discard(self, h):
        self._check(h)
        if h[2] + 1 != len(self.snaps):
            raise InvalidArgument("sequence_cache: only the top snapshot can be discarded")
        self.snaps.pop()


def draft_verify(state: SequenceCache, bank: DeviceBank, draft: Sequence[int], accept_count: int) -> list:
    """draft_verify (cache.cpp:152-195) for one stream: merged embeddings of the accepted prefix.

    The verify block computes every draft position's embedding from ring ++ draft in one
    batched call (the memo's warm-up), then commit() advances the state by accept_count."""
    if accept_count > len(draft):
        raise InvalidArgument("draft_verify: accept count exceeds draft length")
    if len(draft) == 0:
        return []
    for t in draft:
        if int(t) >= bank.info.base_vocab:
            raise OutOfRange(f"sequence_cache: token {t} out of range")
    d = torch.tensor([list(draft)], dtype=torch.int64).to(torch.int32).to(state.st.dev)
    out = state.st.verify(d)
    acc = torch.tensor([accept_count], dtype=torch.int32, device=state.st.dev)
    state.st.commit(d, acc)
    bank.sync_errors()
    res = out[0, :accept_count].cpu().numpy()
    return [res[i] for i in range(accept_count)]


# ----------------------------------------------------------------------------- backward
class GradBank:
    """fp32 gradient accumulator of a DeviceBank (embedding_bank_t<T>& grads of
    embed_sequence_backward, embedding.hpp:438-459), zero-initialised, device layout."""

    def __init__(self, bank: DeviceBank, sparse_rows: bool = False, tf32: bool = False, pedantic: bool = False,
                 exact: bool = False, sparse_base: bool = False):
        self.bank = bank
        self.sparse_rows = sparse_rows
        h = C.c_void_p()
        flags = ((abi.NGRAM_GRAD_SPARSE_ROWS if sparse_rows else 0) | (abi.NGRAM_GRAD_TF32 if tf32 else 0) |
                 (abi.NGRAM_GRAD_PEDANTIC if pedantic else 0) | (abi.NGRAM_GRAD_EXACT if exact else 0) |
                 (abi.NGRAM_GRAD_SPARSE_BASE if sparse_base else 0))
        check(abi.lib().ngram_grad_create_ex(bank.handle, flags, C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            abi.lib().ngram_grad_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def zero(self, stream=None) -> "GradBank":
        check(abi.lib().ngram_grad_zero(self.handle, _stream(stream)))
        return self

    def backward(self, tokens: torch.Tensor, seq_offsets: torch.Tensor, upstream: torch.Tensor,
                 merged: Optional[torch.Tensor] = None, prior: Optional[torch.Tensor] = None,
                 skip_amplify: bool = False, stream=None) -> None:
        """embed_sequence_backward on device tensors: upstream = dL/d(rows) f32 [T, D],
        merged = the forward's pre-amplification rows (layer_norm only)."""
        T = tokens.numel()
        flags = abi.NGRAM_BWD_SKIP_AMPLIFY if skip_amplify else 0
        check(abi.lib().ngram_embed_backward(self.handle, _ptr(tokens), _ptr(seq_offsets), seq_offsets.numel() - 1, T,
                                             _ptr(prior), _ptr(merged), _ptr(upstream), flags, _stream(stream)))

    def sparse(self, device=None):
        """Row-sparse sub-table gradient (sparse_rows=True): (rows int32 [n], vals f32 [n, d])
        on the device, duplicates not merged (their sum is the dense gradient)."""
        p_r, p_v, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(abi.lib().ngram_grad_sparse_rows(self.handle, C.byref(p_r), C.byref(p_v), C.byref(n)))
        dev = device or torch.device("cuda", self.bank.device)
        d = branch_dim(self.bank.cfg)
        rows = torch.empty(n.value, dtype=torch.int32, device=dev)
        vals = torch.empty((n.value, d), dtype=torch.float32, device=dev)
        check(abi.lib().ngram_grad_sparse_read(self.handle, 0, n.value, _ptr(rows), _ptr(vals), _stream()))
        return rows, vals

    def sparse_base(self, device=None):
        """Base-table gradient pairs (sparse_base=True): (tokens int32 [n], vals f32 [n, D]) on the
        device, a view of the bank's buffers (valid until the next backward / zero)."""
        p_t, p_v, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(abi.lib().ngram_grad_sparse_base(self.handle, C.byref(p_t), C.byref(p_v), C.byref(n)))
        if n.value == 0:
            dev = device or torch.device("cuda", self.bank.device)
            return (torch.empty(0, dtype=torch.int32, device=dev),
                    torch.empty((0, self.bank.D), dtype=torch.float32, device=dev))
        return (_device_view(p_t.value, (n.value,), torch.int32, self.bank.device),
                _device_view(p_v.value, (n.value, self.bank.D), torch.float32, self.bank.device))

    def tensor(self, which: int) -> tuple:
        """(device pointer, numel) of 0 E0, 1 sub-tables, 2 W_cat, 3 ln_gain, 4 ln_bias."""
        p, n = C.c_void_p(), C.c_int64()
        check(abi.lib().ngram_grad_tensor(self.handle, which, C.byref(p), C.byref(n)))
        return p.value, n.value

    def download(self) -> dict:
        """Host copy in the reference layout: base, sub[b], proj[b] (v2), gain, bias (LN)."""
        cfg = self.bank.cfg
        D, B = self.bank.D, self.bank.B
        V0 = cfg["base_vocab"]
        v2 = cfg["variant"] == "subtable_v2"
        d = D // B if (v2 and B) else D
        sv = [0] * B  # branch b = (n-2)K + (k-1) (config.hpp:41-44)
        for e in cfg.get("sub_vocab", []):
            sv[(e["n"] - 2) * cfg["sub_tables"] + e["k"] - 1] = int(e["vocab"])
        out = {"base": np.zeros((V0, D), np.float32), "sub": [np.zeros((v, d), np.float32) for v in sv],
               "proj": [np.zeros((D, d), np.float32) for _ in range(B)] if v2 else [],
               "gain": np.zeros(D, np.float32), "bias": np.zeros(D, np.float32)}
        sp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in out["sub"]])
        pp = (C.c_void_p * max(B, 1))(*[a.ctypes.data for a in out["proj"]])
        ln = cfg["amplification"] == "layer_norm"
        check(abi.lib().ngram_grad_download(self.handle, out["base"].ctypes.data,
                                            sp if (B and not self.sparse_rows) else None,
                                            pp if (v2 and B) else None, out["gain"].ctypes.data if ln else None,
                                            out["bias"].ctypes.data if ln else None))
        return out


# ----------------------------------------------------------------------------- PLNE
class PlneLayer:
    """Per-layer N-gram FFN (ffn_plne / ffn_plne_backward, ple.hpp:168-196) over a device
    layer bank (amplification none, dim = hidden): y = W_d (SiLU(W_g x) * g).  gate:
    [hidden, d_model] f32, down: [d_model, hidden] f32, x / y: [T, d_model] f32 (device).
    ffn_ple (table-row gate) = a base-only layer bank (max_order 1, E0 = the table)."""

    def __init__(self, layer_bank: DeviceBank, d_model: int, fast: bool = True):
        """fast (default): split-bf16 tensor-core GEMMs; fast=False: CUDA-core fp32
        (NGRAM_PLNE_PEDANTIC)."""
        self.bank, self.d_model, self.hidden = layer_bank, d_model, layer_bank.D
        h = C.c_void_p()
        check(abi.lib().ngram_plne_create_ex(layer_bank.handle, d_model, 0 if fast else abi.NGRAM_PLNE_PEDANTIC,
                                             C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            abi.lib().ngram_plne_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, gate: torch.Tensor, down: torch.Tensor, x: torch.Tensor, tokens: torch.Tensor,
                seq_offsets: torch.Tensor, prior: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                stream=None) -> torch.Tensor:
        T = tokens.numel()
        y = out if out is not None else torch.empty((T, self.d_model), dtype=torch.float32, device=x.device)
        check(abi.lib().ngram_plne_forward(self.handle, _ptr(gate), _ptr(down), _ptr(x), _ptr(tokens),
                                           _ptr(seq_offsets), seq_offsets.numel() - 1, T, _ptr(prior), _ptr(y),
                                           _stream(stream)))
        return y

    def backward(self, gate, down, x, tokens, seq_offsets, upstream, d_gate, d_down, dx,
                 bank_grads: Optional["GradBank"] = None, prior=None, stream=None) -> None:
        """Accumulates d_gate, d_down, dx and (optionally) the layer bank's gradients."""
        check(abi.lib().ngram_plne_backward(self.handle, bank_grads.handle if bank_grads else None, _ptr(gate),
                                            _ptr(down), _ptr(x), _ptr(tokens), _ptr(seq_offsets),
                                            seq_offsets.numel() - 1, tokens.numel(), _ptr(prior), _ptr(upstream),
                                            _ptr(d_gate), _ptr(d_down), _ptr(dx), _stream(stream)))


# ----------------------------------------------------------------------------- corpus analysis
class CorpusAnalyzer:
    """corpus_analyzer (analysis.hpp:45-93) on the device: windows seen, exact distinct windows
    and distinct buckets per (order, modulus) over every position of every sequence.  add()
    takes device tensors (tokens u32/i32 [T], offsets i64 [nseq+1]); add_host() numpy arrays
    or a list of sequences.  stats() / reports() mirror the reference's structs."""

    def __init__(self, base_vocab: int, orders: Sequence[int], moduli: Sequence[int], device: int = 0):
        self.base_vocab, self.orders, self.moduli = int(base_vocab), [int(o) for o in orders], [int(m) for m in moduli]
        o = (C.c_int * max(len(self.orders), 1))(*self.orders)
        m = (C.c_uint64 * max(len(self.moduli), 1))(*self.moduli)
        h = C.c_void_p()
        check(abi.lib().ngram_analyzer_create(device, self.base_vocab, o, len(self.orders), m, len(self.moduli),
                                              C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            abi.lib().ngram_analyzer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def add(self, tokens: torch.Tensor, seq_offsets: torch.Tensor, stream=None) -> None:
        check(abi.lib().ngram_analyzer_add(self.handle, _ptr(tokens), _ptr(seq_offsets), seq_offsets.numel() - 1,
                                           tokens.numel(), _stream(stream)))

    def add_host(self, seqs) -> None:
        """seqs: a list of token sequences, or (flat u32 tokens, i64 offsets)."""
        if isinstance(seqs, tuple):
            toks, off = np.ascontiguousarray(seqs[0], np.uint32), np.ascontiguousarray(seqs[1], np.int64)
        else:
            lens = [len(q) for q in seqs]
            off = np.zeros(len(seqs) + 1, np.int64)
            off[1:] = np.cumsum(lens)
            toks = np.ascontiguousarray(np.concatenate([np.asarray(q, np.uint64) for q in seqs])
                                        if seqs and off[-1] else np.zeros(0, np.uint64))
            if toks.size and int(toks.max()) > 0xFFFFFFFF:
                raise OverflowError("token ids are u32")
            toks = toks.astype(np.uint32)
        check(abi.lib().ngram_analyzer_add_host(self.handle, toks.ctypes.data if toks.size else None,
                                                off.ctypes.data, off.size - 1))

    def add_sequence(self, seq) -> None:
        self.add_host([seq])

    def merge(self, other: "CorpusAnalyzer", stream=None) -> None:
        check(abi.lib().ngram_analyzer_merge(self.handle, other.handle, _stream(stream)))

    def sync_errors(self) -> None:
        check(abi.lib().ngram_analyzer_sync_errors(self.handle))

    def reserve(self, windows: int) -> None:
        """Pre-size the sets for `windows` more positions (no rehash inside the next adds)."""
        check(abi.lib().ngram_analyzer_reserve(self.handle, int(windows)))

    def stats(self) -> dict:
        no, nm = len(self.orders), len(self.moduli)
        sq, tk = C.c_uint64(), C.c_uint64()
        seen, dist = (C.c_uint64 * no)(), (C.c_uint64 * no)()
        bk = (C.c_uint64 * (no * nm))()
        check(abi.lib().ngram_analyzer_stats(self.handle, C.byref(sq), C.byref(tk), seen, dist, bk))
        return {"sequences_seen": sq.value, "tokens_seen": tk.value,
                "ngrams_seen": {o: seen[i] for i, o in enumerate(self.orders)},
                "distinct_ngrams": {o: dist[i] for i, o in enumerate(self.orders)},
                "distinct_buckets": {(o, m): bk[i * nm + j] for i, o in enumerate(self.orders)
                                     for j, m in enumerate(self.moduli)}}

    def reports(self, corpus_id: str = "") -> list:
        """collision_report per (order, modulus), order-major (analysis.cpp:158-181)."""
        s = self.stats()
        if s["tokens_seen"] == 0:
            raise ValueError("corpus_analyzer: empty corpus")
        out = []
        for o in self.orders:
            for m in self.moduli:
                b = s["distinct_buckets"][(o, m)]
                out.append({"order": o, "modulus": m, "hit_rate": float(b) / float(m),
                            "collision_count": s["distinct_ngrams"][o] - b, "corpus_id": corpus_id,
                            "tokens_processed": s["tokens_seen"]})
        return out


class _CudaArray:
    """__cuda_array_interface__ of library-owned device memory (so torch can alias it)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _device_view(ptr: int, shape, dtype, device: int) -> torch.Tensor:
    """A torch tensor aliasing `ptr` (no copy); bf16 goes through its int16 bit pattern."""
    typestr = {torch.bfloat16: "<i2", torch.float32: "<f4", torch.int32: "<i4", torch.int64: "<i8"}[dtype]
    t = torch.as_tensor(_CudaArray(ptr, shape, typestr), device=torch.device("cuda", device))
    return t.view(dtype) if dtype == torch.bfloat16 else t


# ----------------------------------------------------------------------------- row shards
class ShardGroup:
    """Row-sharded exchange of one rank: double-buffered home X, peer buffers
    mapped over CUDA IPC (multi-process) or by pointer (single-process emulation)."""

    def __init__(self, bank: DeviceBank, max_home_tokens: int):
        self.bank = bank
        self.rank, self.nranks = bank.info.shard_rank, bank.info.shard_count
        h = C.c_void_p()
        check(abi.lib().ngram_shard_group_create(bank.handle, max_home_tokens, C.byref(h)))
        self.handle = h
        self.max_home = max_home_tokens

    def close(self):
        if self.handle:
            abi.lib().ngram_shard_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export_handle(self) -> bytes:
        buf = C.create_string_buffer(abi.NGRAM_SHARD_HANDLE_BYTES)
        check(abi.lib().ngram_shard_export(self.handle, buf))
        return buf.raw

    def open_peer(self, peer_rank: int, handle: bytes) -> None:
        check(abi.lib().ngram_shard_open(self.handle, peer_rank, handle))

    def local_buffers(self):
        a, b = C.c_void_p(), C.c_void_p()
        check(abi.lib().ngram_shard_local_buffers(self.handle, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_peer(self, peer_rank: int, bufs) -> None:
        check(abi.lib().ngram_shard_set_peer(self.handle, peer_rank, C.c_void_p(bufs[0]), C.c_void_p(bufs[1])))

    # ---- NCCL exchange variants (include/ngram_b200.h): the caller runs the collective
    def xchg_prepare(self, all_tokens: torch.Tensor, all_seq_offsets: torch.Tensor, rank_token_offsets,
                     all_prior: Optional[torch.Tensor] = None, stream=None):
        """K1 over the gathered batch + the all-to-all counts -> (send_rows, recv_rows) per rank."""
        rto = np.ascontiguousarray(rank_token_offsets, np.int64)
        snd = np.zeros(self.nranks, np.int64)
        rcv = np.zeros(self.nranks, np.int64)
        check(abi.lib().ngram_shard_xchg_prepare(self.handle, _ptr(all_tokens), _ptr(all_seq_offsets),
                                                 all_seq_offsets.numel() - 1, all_tokens.numel(), rto.ctypes.data,
                                                 _ptr(all_prior), snd.ctypes.data, rcv.ctypes.data, _stream(stream)))
        return snd, rcv

    def xchg_pack(self, send: torch.Tensor, stream=None) -> None:
        check(abi.lib().ngram_shard_xchg_pack(self.handle, _ptr(send), _stream(stream)))

    def xchg_unpack(self, recv: torch.Tensor, stream=None) -> None:
        check(abi.lib().ngram_shard_xchg_unpack(self.handle, _ptr(recv), _stream(stream)))

    def pack_padded(self, all_tokens: torch.Tensor, all_seq_offsets: torch.Tensor, rank_token_offsets, send: torch.Tensor,
                    all_prior: Optional[torch.Tensor] = None, stream=None) -> None:
        rto = np.ascontiguousarray(rank_token_offsets, np.int64)
        check(abi.lib().ngram_shard_pack_padded(self.handle, _ptr(all_tokens), _ptr(all_seq_offsets),
                                                all_seq_offsets.numel() - 1, all_tokens.numel(), rto.ctypes.data,
                                                _ptr(all_prior), _ptr(send), _stream(stream)))

    def home_x(self) -> torch.Tensor:
        """The home X the next project() reads, as a [max_home, D] bf16 tensor aliasing it."""
        p = C.c_void_p()
        check(abi.lib().ngram_shard_home_x(self.handle, C.byref(p)))
        return _device_view(p.value, (self.max_home, self.bank.D), torch.bfloat16, self.bank.device)

    def exchange(self, mode: str, all_tokens: torch.Tensor, all_seq_offsets: torch.Tensor, rank_token_offsets,
                 all_prior: Optional[torch.Tensor] = None, pg=None) -> None:
        """Step 2 of the row-sharded forward through an NCCL collective (torch.distributed):
        mode "a2a" -- all-to-all of the owned rows (compact); "rs" -- reduce-scatter of the
        -0.0-padded X.  Leaves this rank's home X as scatter() would (bit-identical)."""
        import torch.distributed as dist
        dev = all_tokens.device
        D, d = self.bank.D, self.bank.D // max(self.bank.B, 1)
        # gloo (functional runs with every rank on one device) moves host tensors only
        host = dist.get_backend(pg) == "gloo"
        if mode == "a2a":
            snd, rcv = self.xchg_prepare(all_tokens, all_seq_offsets, rank_token_offsets, all_prior)
            send = torch.empty((int(snd.sum()), d), dtype=torch.bfloat16, device=dev)
            recv = torch.empty((int(rcv.sum()), d), dtype=torch.bfloat16, device=dev)
            self.xchg_pack(send)
            if host:  # fp32 staging (gloo has no 16-bit types; bf16 -> fp32 -> bf16 is exact)
                r = torch.empty((int(rcv.sum()), d), dtype=torch.float32)
                dist.all_to_all_single(r, send.float().cpu(), output_split_sizes=[int(x) for x in rcv],
                                       input_split_sizes=[int(x) for x in snd], group=pg)
                recv.copy_(r.to(torch.bfloat16))
            else:
                dist.all_to_all_single(recv, send, output_split_sizes=[int(x) for x in rcv],
                                       input_split_sizes=[int(x) for x in snd], group=pg)
            self.xchg_unpack(recv)
        elif mode == "rs":
            send = torch.empty((self.nranks * self.max_home, D), dtype=torch.bfloat16, device=dev)
            self.pack_padded(all_tokens, all_seq_offsets, rank_token_offsets, send, all_prior)
            if host:  # all-reduce of the padded batch, then this rank's slice (same sum)
                h = send.float().cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=pg)
                self.home_x().copy_(h[self.rank * self.max_home:(self.rank + 1) * self.max_home].to(torch.bfloat16))
            else:
                dist.reduce_scatter_tensor(self.home_x(), send, op=dist.ReduceOp.SUM, group=pg)
        else:
            raise ValueError(f"unknown exchange {mode!r}")

    def scatter(self, all_tokens: torch.Tensor, all_seq_offsets: torch.Tensor, rank_token_offsets,
                all_prior: Optional[torch.Tensor] = None, stream=None) -> None:
        rto = np.ascontiguousarray(rank_token_offsets, np.int64)
        check(abi.lib().ngram_shard_scatter_rows(self.handle, _ptr(all_tokens), _ptr(all_seq_offsets),
                                                 all_seq_offsets.numel() - 1, all_tokens.numel(), rto.ctypes.data,
                                                 _ptr(all_prior), _stream(stream)))

    def project(self, home_tokens: torch.Tensor, rows: bool = True, merged: bool = False, out_dtype=torch.float32,
                stream=None, out_rows: Optional[torch.Tensor] = None, out_merged: Optional[torch.Tensor] = None):
        T = home_tokens.numel()
        dev = home_tokens.device
        if rows and out_rows is None:
            out_rows = torch.empty((T, self.bank.D), dtype=out_dtype, device=dev)
        if merged and out_merged is None:
            out_merged = torch.empty((T, self.bank.D), dtype=out_dtype, device=dev)
        check(abi.lib().ngram_shard_project(self.handle, _ptr(home_tokens), T, _ptr(out_rows if rows else None),
                                            _ptr(out_merged if merged else None), _DT[out_dtype], _stream(stream)))
        return (out_rows if rows else None), (out_merged if merged else None)


def sharded_verify_block(group: ShardGroup, state: DecodeState, draft: torch.Tensor, out_dtype=torch.bfloat16,
                         pg=None, barrier=None, exchange: str = "peer") -> torch.Tensor:
    """A verify block (L = 1: a decode step) of this rank's home streams on row-sharded tables
    (DESIGN.md 7): all-gather the drafts and the decode rings (the windows' prior), scatter the
    owned rows into every home X, barrier, project the home rows (merged, pre-amplification,
    cache.hpp:122-124).  `state` is this rank's DecodeState on its shard bank; commit with
    state.commit(draft, accept) afterwards.  Every rank must hold the same number of streams.
    exchange: "peer" (NVLink peer stores + a barrier), or the NCCL forms "rs" (reduce-scatter of
    the padded X) / "a2a" (all-to-all of the owned rows); all bit-identical."""
    import torch.distributed as dist
    world = dist.get_world_size(pg)
    Bh, L = draft.shape
    R = max(state.bank.N - 1, 0)
    all_draft = torch.empty((world * Bh, L), dtype=torch.int32, device=draft.device)
    dist.all_gather_into_tensor(all_draft, draft.contiguous().to(torch.int32), group=pg)
    all_ring = None
    if R:
        all_ring = torch.empty((world * Bh, R), dtype=torch.int32, device=draft.device)
        dist.all_gather_into_tensor(all_ring, state.rings().contiguous(), group=pg)
    all_off = torch.arange(0, world * Bh * L + 1, L, dtype=torch.int64, device=draft.device)
    rank_tok = [r * Bh * L for r in range(world + 1)]
    if exchange != "peer":
        group.exchange(exchange, all_draft.view(-1), all_off, rank_tok, all_ring, pg=pg)
    else:
        group.scatter(all_draft.view(-1), all_off, rank_tok, all_ring)
        if barrier is not None:
            barrier()
        else:
            one = torch.ones(1, device=draft.device)
            dist.all_reduce(one, group=pg)  # stream-ordered (NCCL): every rank's rows have landed
    _, merged = group.project(draft.contiguous().view(-1).to(torch.int32), rows=False, merged=True,
                              out_dtype=out_dtype)
    return merged.view(Bh, L, -1)


def connect_shard_groups(group: ShardGroup, pg=None) -> None:
    """Exchange IPC handles across the torch.distributed process group and map every peer."""
    import torch.distributed as dist
    mine = group.export_handle()
    allh = [None] * dist.get_world_size(pg)
    dist.all_gather_object(allh, (group.rank, mine), group=pg)
    for r, h in allh:
        if r != group.rank:
            group.open_peer(r, h)


def emulate_shards_single_process(groups) -> None:
    """Map every group's buffers into every other group (all ranks in one process)."""
    bufs = [g.local_buffers() for g in groups]
    for g in groups:
        for r, bb in enumerate(bufs):
            if r != g.rank:
                g.set_peer(r, bb)
