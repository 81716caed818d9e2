"""Incremental decode / speculative verification (device-resident sequence_cache state)
against the reference's semantics -- mirrors proj/tests/test_cache.cpp, plus the
reference's own draft_verify outputs (tests/golden/draft_verify.npz)."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import assert_rows_close, dev_i64, dev_u32, gold, gold_config, u64
from paper_2601_21204_b200 import ngram as G
from paper_2601_21204_b200.abi import InvalidArgument, OutOfRange

pytestmark = pytest.mark.gpu


def small_config(v0=32, dim=384, order=4, k=2, amp="none"):  # test_cache.cpp:15-29, widened to a TC shape
    sv = [23 + 12 * n + 5 * kk for n in range(2, order + 1) for kk in range(1, k + 1)]
    return O.make_config(v0, dim, order, k, sv, "subtable_v2", amp)


def scratch_ids(cfg, confirmed):  # test_cache.cpp:33-38, via the pinned oracle
    return O.hash_sequence(cfg, confirmed)[-1]


@pytest.fixture
def bank(cuda):
    cfg = small_config()
    hb = O.make_bank(cfg, 5, round_bf16=True)
    return cfg, hb, G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)


def test_first_append_hashes_zero_padded_windows(bank):  # test_cache.cpp:40-52
    cfg, hb, db = bank
    st = G.SequenceCache(db)
    ids = st.append(7)
    assert ids == [int(x) for x in scratch_ids(cfg, [7])]
    assert st.length() == 1 and st.last_token() == 7


def test_append_stream_equals_batch(bank):  # test_cache.cpp:54-65
    cfg, hb, db = bank
    st = G.SequenceCache(db)
    rng = O.Rng64(1)
    confirmed = []
    for _ in range(60):
        t = rng.below(32)
        ids = st.append(t)
        confirmed.append(t)
        assert ids == [int(x) for x in scratch_ids(cfg, confirmed)]


def test_snapshot_rollback_and_stale_handles(bank):  # test_cache.cpp:81-126
    cfg, hb, db = bank
    st = G.SequenceCache(db)
    st.append(5)
    st.append(9)
    h = st.snapshot()
    first = [st.append(t) for t in (1, 2, 3)]
    st.rollback(h)
    assert [st.append(t) for t in (1, 2, 3)] == first
    other = G.SequenceCache(db)
    with pytest.raises(InvalidArgument):
        other.rollback(h)
    h1 = st.snapshot()
    st.append(1)
    h2 = st.snapshot()
    st.append(2)
    st.rollback(h1)
    with pytest.raises(InvalidArgument):
        st.rollback(h2)
    st.rollback(h)
    assert st.length() == 2


def test_randomized_schedules_match_replay_oracle(bank):  # test_cache.cpp:128-153 (fewer schedules)
    cfg, hb, db = bank
    rng = O.Rng64(0xCAFE)
    for _ in range(8):
        st = G.SequenceCache(db)
        confirmed, snaps = [], []
        for _ in range(25):
            r = rng.below(10)
            if r < 6:
                t = rng.below(32)
                ids = st.append(t)
                confirmed.append(t)
                assert ids == [int(x) for x in scratch_ids(cfg, confirmed)]
            elif r < 8:
                snaps.append((st.snapshot(), len(confirmed)))
            elif snaps:
                pick = rng.below(len(snaps))
                st.rollback(snaps[pick][0])
                confirmed = confirmed[:snaps[pick][1]]
                snaps = snaps[:pick + 1]
            assert st.length() == len(confirmed)


def test_draft_verify_matches_reference_outputs(cuda):  # cache.cpp:152-195 via the reference itself
    g = gold("draft_verify.npz")
    cfg = gold_config(g)
    hb = O.make_bank(cfg, int(g["seed"]), round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    for i in range(int(g["ncases"])):
        st = G.SequenceCache(db)
        for t in g[f"c{i}_prefix"]:
            st.append(int(t))
        acc = int(g[f"c{i}_accept"])
        out = G.draft_verify(st, db, [int(t) for t in g[f"c{i}_draft"]], acc)
        assert len(out) == acc
        if acc:
            assert_rows_close(np.stack(out), g[f"c{i}_accepted"])
        assert np.array_equal(st.ring(), g[f"c{i}_ring"])
        assert st.length() == int(g[f"c{i}_length"]) and st.last_token() == int(g[f"c{i}_last"])


def test_draft_verify_accept_all_equals_sequential(bank):  # test_cache.cpp:221-243
    cfg, hb, db = bank
    st = G.SequenceCache(db)
    st.append(11)
    draft = [3, 1, 4, 1, 5]
    res = G.draft_verify(st, db, draft, len(draft))
    _, merged = O.embed_sequence(hb, [11] + draft, double=True)
    assert_rows_close(np.stack(res), merged[1:])
    assert st.length() == 6 and st.last_token() == 5 and st.snapshot_depth() == 0


def test_draft_verify_accept_none_leaves_state(bank):  # test_cache.cpp:245-262
    cfg, hb, db = bank
    st = G.SequenceCache(db)
    st.append(2)
    st.append(8)
    assert G.draft_verify(st, db, [9, 9, 9], 0) == []
    assert st.length() == 2 and st.last_token() == 8
    with pytest.raises(InvalidArgument):
        G.draft_verify(st, db, [9, 9, 9], 4)
    with pytest.raises(OutOfRange):
        G.draft_verify(st, db, [9, 99], 1)


def test_batched_decode_steps_equal_prefill(bank, cuda):
    """B streams decoded token by token == the same sequences run through the prefill
    forward (ids bit-identical, merged rows within tolerance)."""
    cfg, hb, db = bank
    B, L = 16, 24
    rng = np.random.default_rng(1)
    seqs = rng.integers(0, 32, size=(B, L)).astype(np.uint32)
    st = G.DecodeState(db, B, max_draft=8)
    outs, idss = [], []
    for i in range(L):
        ids, m = st.step(dev_u32(torch, seqs[:, i], cuda))
        outs.append(m.clone())
        idss.append(u64(ids))
    db.sync_errors()
    dec = torch.stack(outs, 1).reshape(B * L, -1)
    off = np.arange(0, B * L + 1, L)
    _, pre = G.embed_forward(db, dev_u32(torch, seqs.reshape(-1), cuda), dev_i64(torch, off, cuda), rows=False,
                             merged=True)
    # decode steps run the small-T split-K GEMM, the prefill the full-K GEMM: tolerance
    assert_rows_close(dec.cpu().numpy(), pre.cpu().numpy())
    ring, length, last = st.state()
    assert (length == L).all() and np.array_equal(last, seqs[:, -1]) and np.array_equal(ring, seqs[:, -3:])
    for s in range(B):
        want = O.hash_sequence(cfg, seqs[s])
        assert np.array_equal(np.stack([x[s] for x in idss]), want)


def test_batched_verify_and_commit(bank, cuda):
    """batch 64, draft length 4..8 (config E shape): verify-block rows == prefill rows of
    confirmed ++ draft; commit(accept) == accept sequential appends (ring, length, last)."""
    cfg, hb, db = bank
    B = 64
    rng = np.random.default_rng(2)
    hist = [list(rng.integers(0, 32, size=5)) for _ in range(B)]
    st = G.DecodeState(db, B, max_draft=8)
    for i in range(5):
        st.step(dev_u32(torch, [h[i] for h in hist], cuda), want_ids=False, want_merged=False)
    for L in (4, 8, 6):
        draft = rng.integers(0, 32, size=(B, L)).astype(np.uint32)
        out = st.verify(dev_u32(torch, draft, cuda))
        accept = rng.integers(0, L + 1, size=B).astype(np.int32)
        st.commit(dev_u32(torch, draft, cuda), torch.from_numpy(accept).to(cuda))
        db.sync_errors()
        full = [np.array(h + list(draft[s]), np.uint32) for s, h in enumerate(hist)]
        off = np.concatenate([[0], np.cumsum([len(f) for f in full])])
        _, pre = G.embed_forward(db, dev_u32(torch, np.concatenate(full), cuda), dev_i64(torch, off, cuda),
                                 rows=False, merged=True)
        got = out.cpu().numpy()
        want = pre.cpu().numpy()
        for s in range(B):
            assert_rows_close(got[s], want[off[s] + len(hist[s]):off[s + 1]])
        hist = [h + [int(x) for x in draft[s, :accept[s]]] for s, h in enumerate(hist)]
        ring, length, last = st.state()
        for s in range(B):
            assert list(ring[s]) == hist[s][-3:] and int(length[s]) == len(hist[s]) and int(last[s]) == hist[s][-1]


def test_commit_rejects_accept_above_draft_length(bank, cuda):
    cfg, hb, db = bank
    st = G.DecodeState(db, 4, max_draft=4)
    draft = dev_u32(torch, np.ones((4, 3), np.uint32), cuda)
    st.commit(draft, torch.tensor([0, 1, 4, 2], dtype=torch.int32, device=cuda))
    with pytest.raises(InvalidArgument):
        st.state()
    ring, length, last = st.state()
    assert (length == 0).all()  # whole batch left untouched


@pytest.mark.parametrize("order,k", [(2, 2), (7, 1)])
def test_decode_and_verify_other_orders(cuda, order, k):
    """Ring sizes 1 and 6 (N = 2 / 7): decode steps and a verify block + commit equal the
    prefill of the same sequences (ids bit-exact, rows within tolerance, ring = last N-1)."""
    cfg = small_config(v0=50, dim=384, order=order, k=k)
    hb = O.make_bank(cfg, 9, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    B, L, Ld = 8, 10, 5
    rng = np.random.default_rng(order)
    seqs = rng.integers(0, 50, size=(B, L)).astype(np.uint32)
    st = G.DecodeState(db, B, max_draft=Ld)
    outs = []
    for i in range(L):
        ids, m = st.step(dev_u32(torch, seqs[:, i], cuda))
        outs.append(m.clone())
        for s in range(B):
            assert np.array_equal(u64(ids)[s], O.hash_sequence(cfg, seqs[s, :i + 1])[-1])
    draft = rng.integers(0, 50, size=(B, Ld)).astype(np.uint32)
    ver = st.verify(dev_u32(torch, draft, cuda))
    accept = rng.integers(0, Ld + 1, size=B).astype(np.int32)
    st.commit(dev_u32(torch, draft, cuda), torch.from_numpy(accept).to(cuda))
    db.sync_errors()
    full = np.concatenate([seqs, draft], 1)
    off = np.arange(0, B * (L + Ld) + 1, L + Ld)
    _, pre = G.embed_forward(db, dev_u32(torch, full.reshape(-1), cuda), dev_i64(torch, off, cuda), rows=False,
                             merged=True)
    pre = pre.cpu().numpy().reshape(B, L + Ld, -1)
    assert_rows_close(torch.stack(outs, 1).cpu().numpy().reshape(B * L, -1), pre[:, :L].reshape(B * L, -1))
    assert_rows_close(ver.cpu().numpy().reshape(B * Ld, -1), pre[:, L:].reshape(B * Ld, -1))
    ring, length, last = st.state()
    R = order - 1
    for s in range(B):
        hist = list(seqs[s]) + list(draft[s, :accept[s]])
        assert list(ring[s]) == [int(x) for x in hist[-R:]] and int(length[s]) == len(hist)
        assert int(last[s]) == int(hist[-1])


def test_decode_step_and_verify_replay_in_cuda_graph(bank, cuda):
    """A decode step and a verify block + commit are capturable in a CUDA graph (the serving
    pattern of bench.py --workload D/E): replays advance the device state exactly like eager
    calls do."""
    cfg, hb, db = bank
    B = 8
    rng = np.random.default_rng(5)
    toks = dev_u32(torch, rng.integers(0, 32, size=B), cuda)
    draft = dev_u32(torch, rng.integers(0, 32, size=(B, 4)), cuda)
    acc = torch.from_numpy(rng.integers(0, 5, size=B).astype(np.int32)).to(cuda)
    eager, graph = G.DecodeState(db, B, max_draft=4), G.DecodeState(db, B, max_draft=4)
    out_e = torch.empty((B, 4, db.D), dtype=torch.float32, device=cuda)
    out_g = torch.empty_like(out_e)
    step_e = torch.empty((B, db.D), dtype=torch.float32, device=cuda)
    step_g = torch.empty_like(step_e)

    def one(st, so, vo):
        st.step(toks, want_ids=False, out=so, out_dtype=torch.float32)
        st.verify(draft, out=vo, out_dtype=torch.float32)
        st.commit(draft, acc)

    one(graph, step_g, out_g)  # warm-up (allocations happen outside the capture)
    torch.cuda.synchronize()
    one(eager, step_e, out_e)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        one(graph, step_g, out_g)
    for _ in range(3):
        g.replay()
        one(eager, step_e, out_e)
    torch.cuda.synchronize()
    db.sync_errors()
    assert torch.equal(step_e, step_g) and torch.equal(out_e, out_g)
    for a, b in zip(eager.state(), graph.state()):
        assert np.array_equal(a, b)


def test_bad_token_step_between_good_steps(bank, cuda):
    """A decode step with a token >= V0 leaves every stream untouched and is reported (once) at
    the next sync, while the steps around it -- which run without a per-step error reset --
    advance the state and produce the same rows as a clean run."""
    cfg, hb, db = bank
    B = 4
    good1, good2 = np.array([1, 2, 3, 4], np.uint32), np.array([5, 6, 7, 8], np.uint32)
    bad = np.array([1, 32, 3, 4], np.uint32)  # V0 = 32
    ref = G.DecodeState(db, B)
    _, r1 = ref.step(dev_u32(torch, good1, cuda))
    _, r2 = ref.step(dev_u32(torch, good2, cuda))
    db.sync_errors()
    st = G.DecodeState(db, B)
    _, m1 = st.step(dev_u32(torch, good1, cuda))
    st.step(dev_u32(torch, bad, cuda), want_ids=False, want_merged=True)
    _, m2 = st.step(dev_u32(torch, good2, cuda))
    with pytest.raises(OutOfRange):
        db.sync_errors()
    db.sync_errors()  # reported once
    assert torch.equal(m1, r1) and torch.equal(m2, r2)
    for a, b in zip(st.state(), ref.state()):
        assert np.array_equal(a, b)


def test_bad_token_verify_then_commit_is_refused_and_reported(bank, cuda):
    """verify + commit without a per-call reset: a draft holding a token >= V0 makes the commit
    leave every stream untouched and is reported once at the next sync; the next verify +
    commit works normally."""
    cfg, hb, db = bank
    B, L = 4, 3
    st = G.DecodeState(db, B, max_draft=L)
    good = dev_u32(torch, np.array([[1, 2, 3]] * B, np.uint32), cuda)
    bad = dev_u32(torch, np.array([[1, 2, 3], [4, 40, 6], [7, 8, 9], [1, 1, 1]], np.uint32), cuda)
    acc = torch.full((B,), L, dtype=torch.int32, device=cuda)
    st.verify(good)
    st.commit(good, acc)
    db.sync_errors()
    before = st.state()
    st.verify(bad)
    st.commit(bad, acc)
    with pytest.raises(OutOfRange):
        db.sync_errors()
    for a, b in zip(st.state(), before):
        assert np.array_equal(a, b)
    st.verify(good)
    st.commit(good, acc)
    db.sync_errors()
    assert (st.state()[1] == 2 * L).all()


def test_host_decode_step_graph_replay_equals_device_steps(cuda, monkeypatch):
    """ngram_decode_step_host in steady state replays a captured H2D -> kernels -> D2H graph:
    over several steps it returns the device entry's bits (a twin state stepped on the device),
    a bad token raises and leaves the state untouched, a verify block in between (which grows the
    X workspace, forcing a re-capture) keeps both in step, and the eager form
    (NGRAM_HOST_STEP_GRAPH=0) agrees."""
    import ctypes as C
    from paper_2601_21204_b200 import abi
    cfg = O.make_default_config(1000, 768, 4, 2)
    hb = O.make_bank(cfg, 13, round_bf16=True)
    db = G.DeviceBank(cfg).upload(hb.base, hb.sub, hb.proj)
    B = 6
    host, dev = G.DecodeState(db, B, max_draft=3), G.DecodeState(db, B, max_draft=3)
    rng = np.random.default_rng(3)
    out = np.zeros((B, 768), np.float32)

    def host_step(tok):
        t = np.ascontiguousarray(tok, np.uint32)
        abi.check(abi.lib().ngram_decode_step_host(host.handle, t.ctypes.data, None, out.ctypes.data))
        return out.copy()

    for i in range(8):
        if i == 5:  # a verify block + commit on both: grows the workspace, the graph is re-captured
            draft = dev_u32(torch, rng.integers(0, 1000, size=(B, 3)), cuda)
            acc = torch.tensor(rng.integers(0, 4, size=B).astype(np.int32), device=cuda)
            for s in (host, dev):
                s.verify(draft)
                s.commit(draft, acc)
            db.sync_errors()
        if i == 3:  # a bad token: raises, nothing changes
            bad = rng.integers(0, 1000, size=B).astype(np.uint32)
            bad[2] = 1000
            with pytest.raises(OutOfRange):
                host_step(bad)
        tok = rng.integers(0, 1000, size=B).astype(np.uint32)
        got = host_step(tok)
        _, want = dev.step(dev_u32(torch, tok, cuda), want_ids=False)
        db.sync_errors()
        assert np.array_equal(got, want.cpu().numpy()), i
    # a page-locked output buffer receives the device-to-host copy directly (graph re-captured)
    pinned = torch.zeros((B, 768), dtype=torch.float32).pin_memory().numpy()
    for _ in range(2):
        tok = np.ascontiguousarray(rng.integers(0, 1000, size=B).astype(np.uint32))
        abi.check(abi.lib().ngram_decode_step_host(host.handle, tok.ctypes.data, None, pinned.ctypes.data))
        _, want = dev.step(dev_u32(torch, tok, cuda), want_ids=False)
        db.sync_errors()
        assert np.array_equal(pinned, want.cpu().numpy())
    # the ids-only variant (the drop-in's sequence_cache::append) is captured too: ids equal the
    # device entry's
    ids_h = np.zeros((B, db.B), np.uint64)
    for _ in range(3):
        tok = np.ascontiguousarray(rng.integers(0, 1000, size=B).astype(np.uint32))
        abi.check(abi.lib().ngram_decode_step_host(host.handle, tok.ctypes.data, ids_h.ctypes.data, None))
        ids_d, _ = dev.step(dev_u32(torch, tok, cuda), want_ids=True, want_merged=False)
        db.sync_errors()
        assert np.array_equal(ids_h, ids_d.cpu().numpy().view(np.uint64).reshape(B, -1))
    monkeypatch.setenv("NGRAM_HOST_STEP_GRAPH", "0")
    tok = rng.integers(0, 1000, size=B).astype(np.uint32)
    got = host_step(tok)
    _, want = dev.step(dev_u32(torch, tok, cuda), want_ids=False)
    db.sync_errors()
    assert np.array_equal(got, want.cpu().numpy())
    host.close()
    dev.close()
    db.close()
