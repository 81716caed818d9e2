"""Device corpus analyzer (corpus_analyzer, analysis.cpp:44-176) against the reference: the
golden fixtures tests/golden/analysis_*.npz (made by the reference itself), the reference's own
test cases (test_analysis.cpp), streaming / merge / growth invariants, and larger corpora
against the pinned oracle.  Counts are integers: every comparison is exact."""
import numpy as np
import pytest
import torch

import helpers
import oracle as O
from paper_2601_21204_b200 import ngram as G
from paper_2601_21204_b200.abi import NgramError

pytestmark = pytest.mark.gpu


def run(v0, orders, moduli, seqs, mode="host"):
    an = G.CorpusAnalyzer(v0, orders, moduli)
    status = 0
    try:
        if mode == "host":
            an.add_host(seqs)
        elif mode == "per_sequence":  # add_sequence one at a time (analysis.cpp:96)
            for q in seqs:
                an.add_sequence(q)
        else:  # device tensors, error at the sync
            toks, off = O._flat(seqs)
            t = torch.from_numpy(toks.astype(np.int32)).cuda()
            o = torch.from_numpy(off).cuda()
            an.add(t, o)
            an.sync_errors()
    except NgramError as e:
        status = -2 if e.status == 2 else -e.status
    return status, an


@pytest.mark.parametrize("mode", ["host", "per_sequence", "device"])
@pytest.mark.parametrize("name", helpers.ANALYSIS)
def test_matches_reference_goldens(cuda, name, mode):
    v0, orders, moduli, seqs, (status, meta, seen, distinct, buckets) = helpers.analysis_case(name)
    rc, an = run(v0, orders, moduli, seqs, mode)
    assert rc == status
    got = helpers.stats_arrays(an.stats(), orders, moduli)
    for a, b in zip(got, (meta, seen, distinct, buckets)):
        np.testing.assert_array_equal(a, b)


def test_reference_test_cases(cuda):  # test_analysis.cpp:50-113, 166-183
    def rep(corpus, order, v0, m):
        _, an = run(v0, [order], [m], corpus)
        return an.reports("")[0]

    assert rep([[5]], 2, 10, 100)["hit_rate"] == pytest.approx(0.01)
    pairs = [[a, b] for a in range(7) for b in range(7)]
    assert rep(pairs, 2, 7, 49)["hit_rate"] == pytest.approx(1.0)
    assert rep(pairs, 2, 7, 30)["hit_rate"] == pytest.approx(1.0)
    ex = [[1, 5], [3, 5], [5, 5]]
    assert rep(ex, 2, 10, 20)["collision_count"] == 2 and rep(ex, 2, 10, 23)["collision_count"] == 0
    assert rep([list(range(1, 10))], 2, 10, 1000000)["collision_count"] == 0
    z = O.ref_zipf_markov(1000, 16, 4096, 99, 1.1, 0.85)
    assert rep(z, 4, 1000, 4999)["hit_rate"] > rep(z, 2, 1000, 4999)["hit_rate"]
    z = O.ref_zipf_markov(1000, 24, 4096, 20260809, 1.1, 0.85)
    _, an = run(1000, [2], [2000, 2500, 30000, 30500], z)
    r = an.reports("c")
    assert r[0]["collision_count"] > r[1]["collision_count"] and r[3]["collision_count"] <= r[2]["collision_count"]
    assert all(x["corpus_id"] == "c" and x["tokens_processed"] == 24 * 4096 for x in r)
    rng = np.random.default_rng(42)  # injective regime (test_analysis.cpp:105-113)
    for _ in range(5):
        c = [rng.integers(0, 6, size=int(rng.integers(1, 51))) for _ in range(4)]
        _, an = run(6, [2, 3], [36, 216], c)
        st = an.stats()
        assert st["distinct_buckets"][(2, 36)] == st["distinct_ngrams"][2]
        assert st["distinct_buckets"][(3, 216)] == st["distinct_ngrams"][3]


def test_create_errors(cuda):  # analysis.cpp:47-85, test_analysis.cpp:241-250
    for args in [(1, [2], [5]), (10, [], [5]), (10, [2], []), (10, [1], [5]), (10, [2], [0]), (1 << 17, [8], [100])]:
        with pytest.raises(NgramError) as e:
            G.CorpusAnalyzer(*args)
        assert e.value.status == 1
    _, an = run(10, [2], [5], [[], []])
    with pytest.raises(ValueError):
        an.reports("")  # empty corpus


def test_merge_equals_single_pass(cuda):  # test_analysis.cpp:197-222
    rng = np.random.default_rng(0x5eed)
    corpus = [rng.integers(0, 120, size=int(rng.integers(1, 101))) for _ in range(9)]
    orders, moduli = [2, 3], [37, 240, 4000, (1 << 33) + 7]
    _, whole = run(120, orders, moduli, corpus)
    parts = [G.CorpusAnalyzer(120, orders, moduli) for _ in range(3)]
    for i, q in enumerate(corpus):
        parts[i % 3].add_sequence(q)
    parts[2].merge(parts[0])
    parts[2].merge(parts[1])
    assert parts[2].stats() == whole.stats()
    other = G.CorpusAnalyzer(120, [2], moduli)
    with pytest.raises(NgramError):
        parts[2].merge(other)


def test_streaming_growth_and_monotonicity(cuda):
    """Many distinct windows (sets grow several times), added in uneven device chunks, equal the
    oracle's single pass; the counters never decrease along the way."""
    rng = np.random.default_rng(7)
    v0, orders, moduli = 128000, [2, 3, 4], [10944000, 9536000, (1 << 36) + 3, 4999]
    seqs = [rng.integers(0, v0, size=int(rng.integers(1, 40000))).astype(np.uint32) for _ in range(12)]
    an = G.CorpusAnalyzer(v0, orders, moduli)
    prev = None
    for a, b in [(0, 1), (1, 4), (4, 5), (5, 12)]:
        toks, off = O._flat(seqs[a:b])
        an.add(torch.from_numpy(toks.astype(np.int32)).cuda(), torch.from_numpy(off).cuda())
        cur = helpers.stats_arrays(an.stats(), orders, moduli)
        if prev is not None:
            assert all((c >= p).all() for c, p in zip(cur, prev))
        prev = cur
    rc, ref = O.corpus_analyze(v0, orders, moduli, seqs)
    assert rc == 0 and an.stats() == ref


def test_longcat_moduli_on_zipf_stream(cuda):
    """Config C's twelve sub-table moduli over a 65 536-token Zipf-Markov stream (V0 = 128000),
    orders 2..4 -- the collision table of the production configuration, vs the oracle."""
    sv = [(2 * (74 + b) + 1) * 64000 for b in range(12)]
    seqs = O.ref_zipf_markov(128000, 8, 8192, 20260809)
    rc, ref = O.corpus_analyze(128000, [2, 3, 4], sv, seqs)
    _, an = run(128000, [2, 3, 4], sv, seqs, mode="device")
    assert rc == 0 and an.stats() == ref


def test_reserve_then_add_equals_growth(cuda):
    rng = np.random.default_rng(9)
    seqs = [rng.integers(0, 50000, size=30000).astype(np.uint32) for _ in range(4)]
    a, b = G.CorpusAnalyzer(50000, [2, 3], [40009, (1 << 34) + 1]), G.CorpusAnalyzer(50000, [2, 3], [40009, (1 << 34) + 1])
    b.reserve(120000)
    for q in seqs:
        a.add_sequence(q)
        b.add_sequence(q)
    assert a.stats() == b.stats()
    rc, ref = O.corpus_analyze(50000, [2, 3], [40009, (1 << 34) + 1], seqs)
    assert rc == 0 and a.stats() == ref
