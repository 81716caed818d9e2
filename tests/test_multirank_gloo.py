"""Multi-rank host logic of the row-sharded exchange on CPU (gloo, world_size 2 and 4).

What runs here is everything except the CUDA kernels: the partition every shard bank
uses (ngram_shard_rows, the C-ABI's own host code), the routing rule of the scatter
kernel (each (token, branch) row goes from its owner to the token's home rank at
[t_home][b*d:(b+1)*d]), the handle exchange protocol of connect_shard_groups, and the
claim the design rests on: the owners' contributions tile every home X exactly once, so
the sharded X is bit-identical to the unsharded gather.  Row values come from the
oracle's synthetic generator (test infrastructure)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2601_21204_b200 import abi
    from paper_2601_21204_b200 import ngram as G
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = O.make_default_config(300, 256, 3, 2)
        N, K, D, B, d, v, denom = O.shape(cfg)
        V = O.sub_vocab_array(cfg)[:B]
        # 1. partition from the C-ABI host code
        lo, hi = C.c_int64(), C.c_int64()
        blocks = []
        for b in range(B):
            assert abi.lib().ngram_shard_rows(int(V[b]), rank, world, C.byref(lo), C.byref(hi)) == 0
            blocks.append((lo.value, hi.value))
        allb = [None] * world
        dist.all_gather_object(allb, blocks)
        for b in range(B):
            assert allb[0][b][0] == 0 and allb[-1][b][1] == V[b]
            for r in range(1, world):
                assert allb[r][b][0] == allb[r - 1][b][1]
        # 2. every rank holds the all-gathered batch; sequences split evenly by home rank
        nseq, L = 4, 96
        toks = np.random.default_rng(5).integers(0, 300, size=nseq * L).astype(np.uint32)
        per = nseq // world * L
        ids = np.concatenate([O.hash_sequence(cfg, toks[s * L:(s + 1) * L]) for s in range(nseq)])
        seed = 99
        # 3. owner-side scatter: contributions[home] = list of (t_home, b, row values)
        X_parts = [np.zeros((per, D), np.float32) for _ in range(world)]
        cover = [np.zeros((per, B), np.int32) for _ in range(world)]
        for t in range(nseq * L):
            home, th = t // per, t % per
            for b in range(B):
                h = int(ids[t, b])
                if blocks[b][0] <= h < blocks[b][1]:  # this rank owns the bucket row
                    X_parts[home][th, b * d:(b + 1) * d] = O.synth_rows(seed, 1 + b, h, 1, d, 0.02)[0]
                    cover[home][th, b] += 1
        # 4. the exchange itself (NVLink peer stores on the GPU; a gloo all-reduce of disjoint
        #    contributions here -- exact because every slice has exactly one non-zero owner)
        X = torch.from_numpy(np.stack(X_parts))
        cv = torch.from_numpy(np.stack(cover))
        dist.all_reduce(X)
        dist.all_reduce(cv)
        assert (cv.numpy() == 1).all(), "every (token, branch) row must have exactly one owner"
        mine = X[rank].numpy()
        want = np.zeros((per, D), np.float32)
        for th in range(per):
            t = rank * per + th
            for b in range(B):
                want[th, b * d:(b + 1) * d] = O.synth_rows(seed, 1 + b, int(ids[t, b]), 1, d, 0.02)[0]
        assert np.array_equal(mine, want)

        # 5. handle exchange protocol of connect_shard_groups (fake groups on CPU)
        class FakeGroup:
            def __init__(self):
                self.rank, self.opened = rank, {}

            def export_handle(self):
                return bytes([rank]) * 128

            def open_peer(self, r, h):
                self.opened[r] = h

        fg = FakeGroup()
        G.connect_shard_groups(fg)
        assert sorted(fg.opened) == [r for r in range(world) if r != rank]
        assert all(h == bytes([r]) * 128 for r, h in fg.opened.items())
        q.put((rank, "ok"))
    except Exception as e:  # surface to the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_row_sharded_exchange_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(v == "ok" for v in res.values()), res
    assert all(p.exitcode == 0 for p in procs)
