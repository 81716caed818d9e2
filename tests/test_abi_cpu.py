"""C-ABI checks that need no GPU: the library loads, exports every symbol the header
declares, and its host-side config logic (shape algebra, validation, JSON) matches the
reference (config.cpp:23-183) -- compared with oracle/_ref when it is built, else with
the reference behaviour the tests state explicitly."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2601_21204_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "ngram_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ngram_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = abi.lib()
    declared = header_functions()
    assert len(declared) >= 30
    missing = [f for f in declared if not hasattr(L, f)]
    assert not missing, missing
    assert set(declared) == set(abi.SYMBOLS)  # the ctypes binding covers the whole header


def test_version_and_launch_counter():
    assert b"sm_100a" in abi.lib().ngram_version()
    assert abi.lib().ngram_kernel_launches() >= 0


def _ours_validate(cfg) -> int:
    return abi.lib().ngram_config_validate(json.dumps(cfg).encode())


def _ref_validate(cfg):
    if not O.ref_available():
        return None
    return O.ref().ref_config_validate_json(json.dumps(cfg).encode())


def _v2(v0, dim, order, k, amp="none"):
    return O.make_config(v0, dim, order, k, [13 + 8 * n + 3 * kk for n in range(2, order + 1)
                                             for kk in range(1, k + 1)], "subtable_v2", amp)


def _bad_configs():  # test_embedding.cpp:424-444 plus the other validate() branches (config.cpp:32-77)
    c = []
    x = _v2(16, 8, 3, 2)
    x["dim"] = 9
    c.append(("dim not divisible", x))
    x = _v2(16, 8, 3, 2)
    x["sub_vocab"] = x["sub_vocab"][:-1]
    c.append(("missing (3,2)", x))
    x = O.make_config(16, 8, 3, 1, [37, 47], "averaged_v1", "none")
    x["sub_tables"] = 2
    c.append(("v1 with K=2", x))
    c.append(("base_vocab 1", _v2(1, 8, 3, 2)))
    x = _v2(16, 8, 3, 2)
    x["max_order"] = 0
    c.append(("max_order 0", x))
    x = _v2(16, 8, 3, 2)
    x["sub_vocab"][0]["vocab"] = 0
    c.append(("V_nk 0", x))
    x = _v2(16, 8, 3, 2)
    x["sub_vocab"].append({"n": 5, "k": 1, "vocab": 9})
    c.append(("extra branch", x))
    x = _v2(16, 8, 3, 2)
    x["variant"] = "bogus"
    c.append(("unknown variant", x))
    x = _v2(16, 8, 3, 2)
    x["amplification"] = "bogus"
    c.append(("unknown amplification", x))
    base_only = O.make_config(16, 8, 1, 1, [], "subtable_v2", "none")
    base_only["sub_vocab"] = [{"n": 2, "k": 1, "vocab": 5}]
    c.append(("base-only with sub vocab", base_only))
    return c


@pytest.mark.parametrize("name,cfg", _bad_configs())
def test_config_validation_rejects_like_reference(name, cfg):
    assert _ours_validate(cfg) == abi.NGRAM_EINVAL  # std::invalid_argument
    r = _ref_validate(cfg)
    if r is not None:
        assert r == -1, f"reference accepted {name}"


def test_config_validation_accepts_like_reference():
    for cfg in [_v2(16, 8, 3, 2), _v2(128, 24, 4, 2, "layer_norm"), O.make_default_config(32000, 256, 3, 2),
                O.make_config(16, 8, 1, 1, [], "subtable_v2", "none")]:
        assert _ours_validate(cfg) == abi.NGRAM_OK
        r = _ref_validate(cfg)
        assert r in (None, 0)


def test_bad_json_is_a_parse_error():
    assert abi.lib().ngram_config_validate(b"{not json") == abi.NGRAM_EPARSE
    assert abi.lib().ngram_config_validate(b'{"max_order": 3}') == abi.NGRAM_EPARSE
    assert b"JSON" in abi.lib().ngram_last_error()


@pytest.mark.parametrize("v0,dim,N,K", [(32000, 256, 3, 2), (128000, 768, 4, 4), (128000, 3072, 4, 4), (50, 24, 4, 2)])
def test_make_default_config_matches_reference(v0, dim, N, K):  # config.cpp:163-183
    buf = C.create_string_buffer(1 << 16)
    assert abi.lib().ngram_make_default_config(v0, dim, N, K, buf, len(buf)) == 0
    ours = json.loads(buf.value)
    assert ours == O.make_default_config(v0, dim, N, K)
    if O.ref_available():
        rb = C.create_string_buffer(1 << 16)
        assert O.ref().ref_make_default_config_json(v0, dim, N, K, rb, len(rb)) == 0
        assert json.loads(rb.value) == ours


def test_no_cpu_fallback_without_gpu():
    """Creating a device bank on a host without a usable GPU fails loudly (ECUDA/ENOMEM)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = abi.lib().ngram_bank_create(json.dumps(_v2(16, 8, 3, 2)).encode(), 0, 0, 1, C.byref(h))
    assert rc in (abi.NGRAM_ECUDA, abi.NGRAM_ENOMEM)
    assert not h.value


@pytest.mark.skipif(not O.ref_available(), reason="reference not built here")
def test_bench_zipf_markov_stream_is_the_reference_generator():  # corpus.cpp:211-271
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for vocab, nseq, n, seed in [(1000, 3, 400, 20260809), (128000, 2, 2000, 7)]:
        ours = bench.zipf_markov_tokens(vocab, nseq, n, seed)
        ref = np.zeros((nseq, n), np.uint32)
        assert O.ref().ref_generate_zipf_markov(vocab, nseq, n, seed, 1.1, 0.35, ref.reshape(-1)) == 0
        assert np.array_equal(ours, ref)


@pytest.mark.skipif(not O.ref_available(), reason="reference not built here")
def test_bench_reference_arm_json_contract():
    import subprocess, sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--workload", "A"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["warmup"] >= 3
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "reference" and line["config"]["workload"]


def test_analyzer_argument_checks_and_no_gpu():
    """corpus_analyzer's constructor checks (analysis.cpp:47-85) run on the host before any
    device work, with the reference's messages; a valid analyzer needs a GPU (fails loudly)."""
    import torch
    L = abi.lib()

    def create(v0, orders, moduli):
        o = (C.c_int * max(len(orders), 1))(*orders)
        m = (C.c_uint64 * max(len(moduli), 1))(*moduli)
        h = C.c_void_p()
        rc = L.ngram_analyzer_create(0, v0, o, len(orders), m, len(moduli), C.byref(h))
        return rc, h, L.ngram_last_error().decode()

    for args, msg in [((1, [2], [5]), "base vocabulary must be >= 2"),
                      ((10, [], [5]), "need at least one order and one modulus"),
                      ((10, [2], []), "need at least one order and one modulus"),
                      ((10, [1], [5]), "orders must be >= 2"),
                      ((10, [2], [0]), "moduli must be >= 1"),
                      ((1 << 17, [8], [100]), "V0^order exceeds 128 bits")]:
        rc, h, err = create(*args)
        assert rc == abi.NGRAM_EINVAL and not h.value and msg in err
    if not torch.cuda.is_available():
        rc, h, _ = create(10, [2], [5])
        assert rc in (abi.NGRAM_ECUDA, abi.NGRAM_ENOMEM) and not h.value
