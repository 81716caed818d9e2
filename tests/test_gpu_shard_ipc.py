"""Row-sharded exchange across PROCESSES: two ranks, each its own process with its
own shard bank, map each other's home X buffers through CUDA IPC handles exchanged over
torch.distributed (gloo, 127.0.0.1), scatter their owned rows into the peers' X, meet at a
host barrier, and project their home tokens.  The pool has one GPU, so both processes use
cuda:0 (CUDA IPC between processes on one device is the same mechanism as across NVLink
peers); the kernels never wait on each other -- the barrier is a host collective after a
device synchronize.  Output must be bit-identical to the unsharded forward."""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

WORKER = r"""
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path[:0] = [{root!r}, {tests!r}, os.path.join({root!r}, "oracle")]
import oracle as O
from helpers import dev_i64, dev_u32
from paper_2601_21204_b200 import ngram as G
rank, world = int(sys.argv[1]), 2
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=world)
torch.cuda.set_device(0)
cfg = O.make_default_config(4000, 768, 4, 4)
nseq, L = 4, 500
toks = np.random.default_rng(3).integers(0, 4000, size=nseq * L).astype(np.uint32)
prior = np.random.default_rng(4).integers(0, 4000, size=(nseq, 3)).astype(np.uint32)
off = np.arange(0, nseq * L + 1, L)
t_all, off_all, pr_all = dev_u32(torch, toks, "cuda:0"), dev_i64(torch, off, "cuda:0"), dev_u32(torch, prior, "cuda:0")
per = nseq // world
rank_tok = [r * per * L for r in range(world + 1)]
bank = G.DeviceBank(cfg, shard_rank=rank, shard_count=world).generate(5)
group = G.ShardGroup(bank, per * L)
G.connect_shard_groups(group)  # IPC handles all-gathered over gloo, peers opened
home = t_all[rank_tok[rank]:rank_tok[rank + 1]]
outs = []
for step in range(3):  # both halves of the double-buffered X, then the first again
    group.scatter(t_all, off_all, rank_tok, pr_all)
    torch.cuda.synchronize()
    dist.barrier()  # every rank's rows have landed in every home X
    rows, merged = group.project(home, merged=True)
    torch.cuda.synchronize()
    dist.barrier()  # nobody scatters into a buffer a peer is still projecting from
    outs.append(torch.stack([rows, merged]).cpu().numpy())
bank.sync_errors()
full = G.DeviceBank(cfg).generate(5)
ref_rows, ref_merged = G.embed_forward(full, t_all, off_all, prior=pr_all, merged=True)
ref = torch.stack([ref_rows, ref_merged])[:, rank_tok[rank]:rank_tok[rank + 1]].cpu().numpy()
ok = all(np.array_equal(o, ref) for o in outs)
np.save(sys.argv[2], np.array([1 if ok else 0]))
dist.barrier()
dist.destroy_process_group()
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_process_ipc_exchange_bit_identical(cuda):
    code = WORKER.format(root=ROOT, tests=HERE, port=_free_port())
    with tempfile.TemporaryDirectory() as td:
        procs, outs = [], []
        for r in range(2):
            out = os.path.join(td, f"r{r}.npy")
            outs.append(out)
            procs.append(subprocess.Popen([sys.executable, "-c", code, str(r), out]))
        for p in procs:
            assert p.wait(timeout=300) == 0
        assert all(int(np.load(o)[0]) == 1 for o in outs)


VERIFY_WORKER = r"""
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path[:0] = [{root!r}, {tests!r}, os.path.join({root!r}, "oracle")]
import oracle as O
from paper_2601_21204_b200 import ngram as G
rank, world = int(sys.argv[1]), 2
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=world)
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
cfg = O.make_default_config(4000, 768, 4, 4)
cfg["amplification"] = "none"  # the cache path returns merged vectors
Bh, L = 6, int(sys.argv[3])
rng = np.random.default_rng(11)
prior = torch.from_numpy(rng.integers(0, 4000, size=(world * Bh, 3)).astype(np.int32)).to(dev)
lengths = torch.full((world * Bh,), 100, dtype=torch.int64, device=dev)
draft = torch.from_numpy(rng.integers(0, 4000, size=(world * Bh, L)).astype(np.int32)).to(dev)
accept = torch.from_numpy(rng.integers(0, L + 1, size=world * Bh).astype(np.int32)).to(dev)
# single-GPU reference: every stream on the full bank
full = G.DeviceBank(cfg).generate(5)
ref_state = G.DecodeState(full, world * Bh, max_draft=L)
ref_state.reset(prior, lengths)
ref = ref_state.verify(draft, out_dtype=torch.float32)
ref_state.commit(draft, accept)
ref_ring = ref_state.state()[0]
# this rank: its home streams on its shard bank
home = slice(rank * Bh, (rank + 1) * Bh)
bank = G.DeviceBank(cfg, shard_rank=rank, shard_count=world).generate(5)
group = G.ShardGroup(bank, Bh * L)
G.connect_shard_groups(group)
st = G.DecodeState(bank, Bh, max_draft=L)
st.reset(prior[home].contiguous(), lengths[home].contiguous())

def barrier():
    torch.cuda.synchronize()
    dist.barrier()

ok = True
for step in range(2):  # both halves of the double-buffered X
    merged = G.sharded_verify_block(group, st, draft[home], out_dtype=torch.float32, barrier=barrier,
                                    exchange=sys.argv[4])
    torch.cuda.synchronize()
    dist.barrier()  # nobody scatters into a buffer a peer still projects from
    ok = ok and torch.equal(merged, ref[home])
st.commit(draft[home].contiguous(), accept[home].contiguous())
ok = ok and np.array_equal(st.state()[0], ref_ring[home])
np.save(sys.argv[2], np.array([1 if ok else 0]))
dist.barrier()
dist.destroy_process_group()
"""


@pytest.mark.parametrize("L,exchange", [(1, "peer"), (4, "peer"), (4, "rs"), (4, "a2a"), (1, "a2a")])
def test_two_process_sharded_verify_and_commit(cuda, L, exchange):
    """Config E on row-sharded tables, two ranks: all-gathered drafts + rings, owned rows
    moved to their home rank -- scattered over CUDA IPC ("peer"), or by the collective forms
    (reduce-scatter of the -0.0-padded X, all-to-all of the owned rows; gloo here, NCCL on a
    multi-GPU node) -- split-K projection of the home block, local commit: identical to the
    single-GPU verify + commit of the same streams.  L = 1 is a sharded decode step."""
    code = VERIFY_WORKER.format(root=ROOT, tests=HERE, port=_free_port())
    with tempfile.TemporaryDirectory() as td:
        procs, outs = [], []
        for r in range(2):
            out = os.path.join(td, f"r{r}.npy")
            outs.append(out)
            procs.append(subprocess.Popen([sys.executable, "-c", code, str(r), out, str(L), exchange]))
        for p in procs:
            assert p.wait(timeout=300) == 0
        assert all(int(np.load(o)[0]) == 1 for o in outs)
