"""Drive every kernel family of libngram_b200.so once, at small sizes, with canary-guarded
outputs: every output buffer the caller owns is the middle of a larger allocation filled with
a sentinel, and the sentinel must survive the call (no write outside the declared output).
Meant to run under compute-sanitizer (memcheck / racecheck / synccheck) as well:

    compute-sanitizer --tool memcheck python tests/sanitize_paths.py

but the GPU pool refuses compute-sanitizer (profiles/r02_sanitizer.txt), so the canaries and the
per-step invariants are the evidence.  Not a pytest module (no test_ prefix); run as one
process.  Each step checks its result against a cheap invariant.
Paths: fused K1+K2 + the pair tcgen05 projection (every amplification, fp32 / bf16 out), the
fused wide-tile prefill kernel (D <= 768), the
1-CTA tile and the split-K small-T GEMM + reduce, the CUDA-core kernels, decode step / verify /
commit (fused error-word release), the backward (gather, amp_backward, both tcgen05 GEMM
layouts, COO append), the generic GEMM in every layout / term count, PLNE (both modes), the
corpus analyzer, and the row-sharded scatter (P = 2 emulated in one process).
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ctypes as C  # noqa: E402

import oracle as O  # noqa: E402  (checker only)
from paper_2601_21204_b200 import abi  # noqa: E402
from paper_2601_21204_b200 import ngram as G  # noqa: E402

dev = torch.device("cuda", 0)


def u32(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(dev)


def i64(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.int64)).to(dev)


def step(name):
    print("--", name, flush=True)


SENTINEL = -7.77e30


def guarded(shape, dtype=torch.float32, pad=4096):
    """(view, check): `view` is a contiguous tensor of `shape` inside a sentinel-filled buffer."""
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * pad,), SENTINEL, dtype=dtype, device=dev)
    view = buf[pad:pad + n].view(*shape)

    def check(what):
        torch.cuda.synchronize()
        s = torch.tensor(SENTINEL, dtype=dtype, device=dev)
        assert bool((buf[:pad] == s).all()) and bool((buf[pad + n:] == s).all()), f"{what}: write outside the output"
    return view, check


def forward_paths():
    for D, amp in ((256, "scale_sqrt_d"), (256, "layer_norm"), (384, "none")):
        cfg = O.make_default_config(1000, D, 3, 2)
        cfg["amplification"] = amp
        bank = G.DeviceBank(cfg).generate(3)
        for T in (40, 300, 700, 20000 if D == 256 else 900):  # split-K, one-wave 1-CTA tiles, pair tiles, ragged
            step(f"forward D={D} amp={amp} T={T}")
            toks = np.random.default_rng(T).integers(0, 1000, size=T)
            off = [0, T // 3, T]
            rows, merged = G.embed_forward(bank, u32(toks), i64(off), merged=True)
            rbv, chk = guarded((T, D), torch.bfloat16)
            rb, _ = G.embed_forward(bank, u32(toks), i64(off), out_dtype=torch.bfloat16, out_rows=rbv)
            bank.sync_errors()
            chk(f"forward bf16 D={D} T={T}")
            assert torch.isfinite(rows).all() and rows.shape == (T, D)
            assert float((rb.float() - rows).abs().max()) <= 0.02 * float(rows.abs().max()) + 1e-6
            ids = G.hash_ids(bank, u32(toks), i64(off))
            assert ids.shape == (T, 4)
    step("CUDA-core shape (d = 6)")
    cfg = O.make_config(50, 12, 3, 1, [37, 47])
    hb = O.make_bank(cfg, 5, round_bf16=True)
    bank = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    rows, _ = G.embed_forward(bank, u32(np.arange(20) % 50), i64([0, 20]))
    bank.sync_errors()
    assert torch.isfinite(rows).all()


def wide_paths():
    # the fused wide-tile prefill kernel (gemm_wide.cu; NGRAM_PREFILL_PATH is read per call):
    # canary-guarded rows-only fp32 (the OUT = 1 instance) and rows + merged bf16, ragged T,
    # every width it takes; bits equal to the X path
    for D in (256, 512, 768):
        cfg = O.make_default_config(1000, D, 4 if D == 768 else 3, 4 if D == 768 else 2)
        bank = G.DeviceBank(cfg).generate(9)
        for T in (300, 1029):
            step(f"wide prefill D={D} T={T}")
            toks = u32(np.random.default_rng(T + D).integers(0, 1000, size=T))
            off = i64([0, T // 2, T])
            os.environ["NGRAM_PREFILL_PATH"] = "x"
            ref, refm = G.embed_forward(bank, toks, off, merged=True, out_dtype=torch.bfloat16)
            os.environ["NGRAM_PREFILL_PATH"] = "wide"
            rv, chk = guarded((T, D))
            G.embed_forward(bank, toks, off, out_rows=rv)
            mv, chkm = guarded((T, D), torch.bfloat16)
            rbv, chkr = guarded((T, D), torch.bfloat16)
            G.embed_forward(bank, toks, off, merged=True, out_dtype=torch.bfloat16, out_rows=rbv, out_merged=mv)
            bank.sync_errors()
            chk(f"wide fp32 D={D} T={T}")
            chkm(f"wide merged D={D} T={T}")
            chkr(f"wide bf16 D={D} T={T}")
            assert torch.equal(rbv, ref) and torch.equal(mv, refm)
            os.environ.pop("NGRAM_PREFILL_PATH")
            assert torch.isfinite(rv).all()


def decode_paths():
    cfg = O.make_default_config(1000, 768, 4, 2)
    bank = G.DeviceBank(cfg).generate(4)
    for B, L in ((3, 1), (40, 4), (70, 2)):
        step(f"decode B={B} L={L}")
        st = G.DecodeState(bank, B, max_draft=4)
        rng = np.random.default_rng(B)
        st.reset(u32(rng.integers(0, 1000, size=(B, 3))), i64(np.full(B, 9)))
        st.step(u32(rng.integers(0, 1000, size=B)))
        d = u32(rng.integers(0, 1000, size=(B, L)))
        ov, chk = guarded((B, L, 768))
        out = st.verify(d, out=ov)
        st.commit(d, torch.from_numpy(rng.integers(0, L + 1, size=B).astype(np.int32)).to(dev))
        bank.sync_errors()
        chk(f"verify B={B} L={L}")
        ring, length, last = st.state()
        assert torch.isfinite(out).all() and (length >= 10).all()
        st.close()


def backward_paths():
    cfg = O.make_default_config(600, 256, 3, 2)
    bank = G.DeviceBank(cfg).generate(6)
    T = 200
    toks = u32(np.random.default_rng(1).integers(0, 600, size=T))
    off = i64([0, 77, T])
    up = torch.randn((T, 256), device=dev)
    for kw in ({}, {"exact": True}, {"tf32": True}, {"pedantic": True}, {"sparse_rows": True}):
        step(f"backward {kw}")
        gb = G.GradBank(bank, **kw)
        gb.backward(toks, off, up)
        bank.sync_errors()
        d = gb.download() if not kw.get("sparse_rows") else None
        if d is not None:
            assert np.isfinite(d["base"]).all()
        gb.close()


def gemm_paths():
    gen = torch.Generator(device=dev).manual_seed(2)
    M, N, K = 300, 200, 130
    for a_mn in (False, True):
        for b_mn in (False, True):
            for at, bt in ((3, 1), (2, 1), (3, 3), (1, 3), (1, 1), (0, 0)):
                step(f"gemm a_mn={a_mn} b_mn={b_mn} terms={at}x{bt}")
                A = torch.randn((K, M) if a_mn else (M, K), generator=gen, device=dev).bfloat16().float()
                B = torch.randn((K, N) if b_mn else (N, K), generator=gen, device=dev).bfloat16().float()
                Cv, chk = guarded((M, N + 4))  # ldc = N + 4: the pad columns must stay untouched too
                Cv[:, N:] = SENTINEL
                abi.check(abi.lib().ngram_gemm_f32(0, M, N, K, C.c_void_p(A.data_ptr()), A.shape[1], int(a_mn),
                                                   C.c_void_p(B.data_ptr()), B.shape[1], int(b_mn),
                                                   C.c_void_p(Cv.data_ptr()), N + 4, 0, at, bt, None))
                chk(f"gemm {a_mn} {b_mn} {at}x{bt}")
                assert bool((Cv[:, N:] == SENTINEL).all()), "gemm wrote past N"
                Cm = Cv[:, :N]
                ref = (A.t() if a_mn else A).double() @ (B.t() if b_mn else B).double().t()
                assert float((Cm.double() - ref).norm() / ref.norm()) < 1e-5


def plne_paths():
    cfg = O.make_default_config(300, 256, 3, 2)
    cfg["amplification"] = "none"  # PLNE layer banks (ple.hpp:177-182)
    bank = G.DeviceBank(cfg).generate(8)
    T, Dm = 50, 96
    gen = torch.Generator(device=dev).manual_seed(5)
    gate = torch.randn((256, Dm), generator=gen, device=dev) * 0.05
    down = torch.randn((Dm, 256), generator=gen, device=dev) * 0.05
    x = torch.randn((T, Dm), generator=gen, device=dev)
    toks, off = u32(np.arange(T) % 300), i64([0, T])
    for fast in (False, True):
        step(f"plne fast={fast}")
        layer = G.PlneLayer(bank, Dm, fast=fast)
        y = layer.forward(gate, down, x, toks, off)
        dg, dd, dx = torch.zeros_like(gate), torch.zeros_like(down), torch.zeros_like(x)
        layer.backward(gate, down, x, toks, off, torch.ones_like(y), dg, dd, dx)
        bank.sync_errors()
        assert torch.isfinite(y).all() and torch.isfinite(dg).all()
        layer.close()


def analysis_paths():
    step("corpus analyzer")
    an = G.CorpusAnalyzer(500, [2, 3], [97, 5000003])
    toks = np.random.default_rng(3).integers(0, 500, size=3000)
    an.add(u32(toks), i64([0, 1000, 3000]))
    an.sync_errors()
    s = an.stats()
    assert s["tokens_seen"] == 3000


def shard_paths():
    step("row-sharded scatter, P = 2 (one process)")
    cfg = O.make_default_config(800, 256, 3, 2)
    full = G.DeviceBank(cfg).generate(9)
    nseq, L = 4, 150
    toks = u32(np.random.default_rng(4).integers(0, 800, size=nseq * L))
    off = i64(np.arange(0, nseq * L + 1, L))
    ref, _ = G.embed_forward(full, toks, off)
    banks = [G.DeviceBank(cfg, shard_rank=r, shard_count=2).generate(9) for r in range(2)]
    groups = [G.ShardGroup(b, nseq * L // 2) for b in banks]
    G.emulate_shards_single_process(groups)
    rank_tok = [0, nseq * L // 2, nseq * L]
    for g in groups:
        g.scatter(toks, off, rank_tok)
    torch.cuda.synchronize()
    for r, g in enumerate(groups):
        rows, _ = g.project(toks[rank_tok[r]:rank_tok[r + 1]])
        assert torch.equal(rows, ref[rank_tok[r]:rank_tok[r + 1]])


if __name__ == "__main__":
    which = sys.argv[1:] or ["forward", "wide", "decode", "backward", "gemm", "plne", "analysis", "shard"]
    for w in which:
        globals()[w + "_paths"]()
    torch.cuda.synchronize()
    print("sanitize_paths: all paths ran,", abi.lib().ngram_kernel_launches(), "kernel launches")
