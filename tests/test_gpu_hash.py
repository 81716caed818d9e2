"""K1 hash-index kernel parity (bit-exact) through the C-ABI -- mirrors
proj/tests/test_hashing.cpp case by case, plus batch-scale checks vs reference goldens."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import dev_i64, dev_u32, gold, gold_config, u64
from paper_2601_21204_b200 import ngram as G
from paper_2601_21204_b200.abi import InvalidArgument, OutOfRange

pytestmark = pytest.mark.gpu


def test_rolling_hash_worked_examples(cuda):  # test_hashing.cpp:12-26
    assert G.rolling_hash([3, 5], (2, 10, 7)) == 0
    assert G.rolling_hash([0] * 5, (5, 1000, 12345)) == 0
    assert G.rolling_hash([0, 0], (2, 7, 3)) == 0
    assert G.rolling_hash([0, 0, 7], (3, 128000, 13)) == 7


def test_rolling_hash_input_validation(cuda):  # test_hashing.cpp:28-38
    with pytest.raises(InvalidArgument):
        G.rolling_hash([1, 2, 3], (2, 10, 7))
    with pytest.raises(InvalidArgument):
        G.rolling_hash([1, 2, 3], (4, 10, 7))
    with pytest.raises(OutOfRange):
        G.rolling_hash([1, 12], (2, 10, 7))
    with pytest.raises(InvalidArgument):
        G.rolling_hash([1, 2, 3], (3, 1, 7))
    with pytest.raises(InvalidArgument):
        G.rolling_hash([1, 2, 3], (3, 10, 0))
    with pytest.raises(InvalidArgument):
        G.rolling_hash([5], (1, 10, 7))


def test_rolling_hash_20k_reference_cases(cuda):  # test_hashing.cpp:40-57, reference outputs
    g = gold("rolling_hash_20k.npz")
    win = dev_u32(torch, g["windows"], cuda)
    out, status = G.rolling_hash_batch(win, torch.from_numpy(g["n"]).to(cuda),
                                       torch.from_numpy(g["base"].view(np.int64)).to(cuda),
                                       torch.from_numpy(g["modulus"].view(np.int64)).to(cuda))
    assert (status.cpu().numpy() == 0).all()
    got = u64(out)
    assert np.array_equal(got, g["hash"])
    assert (got < g["modulus"]).all()


def test_prefix_pad_identity(cuda):  # test_hashing.cpp:59-74, same rng stream
    rng = O.Rng64(0x5EED0002)
    rows, orders, bases, mods = [], [], [], []
    for _ in range(2000):
        n = 2 + rng.below(5)
        base = 2 + rng.below(100000)
        mod = 1 + rng.below(1 << 20)
        w = [rng.below(base) for _ in range(n)]
        rows += [w + [0] * (8 - n), [0] + w + [0] * (7 - n)]
        orders += [n, n + 1]
        bases += [base, base]
        mods += [mod, mod]
    out, status = G.rolling_hash_batch(dev_u32(torch, np.array(rows), cuda),
                                       torch.tensor(orders, dtype=torch.int32, device=cuda),
                                       torch.tensor(bases, dtype=torch.int64, device=cuda),
                                       torch.tensor(mods, dtype=torch.int64, device=cuda))
    got = u64(out)
    assert (status.cpu().numpy() == 0).all()
    assert np.array_equal(got[0::2], got[1::2])


def test_rolling_hash_is_deterministic(cuda):  # test_hashing.cpp:76-81
    first = G.rolling_hash([11, 3, 0, 42], (4, 64, 999983))
    for _ in range(10):
        assert G.rolling_hash([11, 3, 0, 42], (4, 64, 999983)) == first


def test_hash_all_orders_worked_example(cuda):  # test_hashing.cpp:83-101
    cfg = O.make_config(16, 4, 3, 1, [101, 103], "averaged_v1", "none")
    bank = G.DeviceBank(cfg)
    assert G.hash_all_orders([0, 4, 9], bank) == [73, 73]
    assert G.hash_all_orders([0, 0, 0], bank) == [0, 0]


def test_equal_moduli_imply_equal_ids(cuda):  # test_hashing.cpp:103-120
    cfg = O.make_config(32, 8, 2, 2, [77, 77], "subtable_v2", "none")
    bank = G.DeviceBank(cfg)
    rng = O.Rng64(7)
    toks = np.array([rng.below(32) for _ in range(400)], np.uint32)
    ids = u64(G.hash_ids(bank, dev_u32(torch, toks, cuda), dev_i64(torch, [0, 400], cuda)))
    assert np.array_equal(ids[:, 0], ids[:, 1])


def test_hash_all_orders_matches_per_window_rolling_hash(cuda):  # test_hashing.cpp:122-138
    cfg = O.make_default_config(50, 24, 4, 2)
    bank = G.DeviceBank(cfg)
    rng = O.Rng64(99)
    for _ in range(20):
        ctx = [rng.below(50) for _ in range(4)]
        ids = G.hash_all_orders(ctx, bank)
        for n in range(2, 5):
            for k in (1, 2):
                b = (n - 2) * 2 + (k - 1)
                assert ids[b] == G.rolling_hash(ctx[-n:], (n, 50, cfg["sub_vocab"][b]["vocab"]))


def test_hash_all_orders_propagates_range_errors(cuda):  # test_hashing.cpp:140-146
    bank = G.DeviceBank(O.make_default_config(10, 12, 3, 2))
    with pytest.raises(OutOfRange):
        G.hash_all_orders([0, 3, 10], bank)
    with pytest.raises(InvalidArgument):
        G.hash_all_orders([3, 4], bank)


@pytest.mark.parametrize("u64_out", [True, False])
def test_config_a_batch_ids_bitexact(cuda, u64_out):  # SURVEY 8(d) config A, 4 x 512
    g = gold("cfgA_ids.npz")
    bank = G.DeviceBank(gold_config(g))
    ids = G.hash_ids(bank, dev_u32(torch, g["tokens"], cuda), dev_i64(torch, [0, 512, 1024, 1536, 2048], cuda),
                     u64=u64_out)
    got = u64(ids) if u64_out else ids.cpu().numpy().view(np.uint32).astype(np.uint64)
    assert np.array_equal(got, g["ids"])


def test_config_c_ids_with_prior_bitexact(cuda):
    g = gold("cfgC_ids.npz")
    cfg = gold_config(g)
    bank = G.DeviceBank(cfg, tables=False)
    prior = np.zeros((2, 3), np.uint32)
    prior[1] = g["prior"]
    ids = G.hash_ids(bank, dev_u32(torch, g["tokens"], cuda), dev_i64(torch, [0, 1024, 2048], cuda),
                     prior=dev_u32(torch, prior, cuda))
    assert np.array_equal(u64(ids), g["ids"])


def test_moduli_above_2_32_bitexact(cuda):  # the 128-bit general path
    g = gold("bigmod_ids.npz")
    bank = G.DeviceBank(gold_config(g), tables=False)
    ids = G.hash_ids(bank, dev_u32(torch, g["tokens"], cuda), dev_i64(torch, [0, 300, 600], cuda))
    assert np.array_equal(u64(ids), g["ids"])


def test_config_c_full_batch_vs_oracle(cuda):  # all 65536 positions of the headline workload
    g = gold("cfgC_ids.npz")
    cfg = gold_config(g)
    bank = G.DeviceBank(cfg, tables=False)
    toks = np.random.default_rng(42).integers(0, 128000, size=8 * 8192).astype(np.uint32)
    off = np.arange(0, 8 * 8192 + 1, 8192)
    ids = u64(G.hash_ids(bank, dev_u32(torch, toks, cuda), dev_i64(torch, off, cuda)))
    want = np.concatenate([O.hash_sequence(cfg, toks[off[i]:off[i + 1]]) for i in range(8)])
    assert np.array_equal(ids, want)


def test_out_of_range_token_reported_at_sync(cuda):  # hashing.cpp:49-54
    bank = G.DeviceBank(O.make_default_config(1000, 256, 3, 2))
    toks = np.arange(100, dtype=np.uint32)
    toks[57] = 1000
    G.hash_ids(bank, dev_u32(torch, toks, cuda), dev_i64(torch, [0, 100], cuda))
    with pytest.raises(OutOfRange, match="position 57"):
        bank.sync_errors()
    bank.sync_errors()  # cleared
