#!/usr/bin/env python3
"""bench.py -- N-gram Embedding forward throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C|B|A]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

Secondary lines (not the driver's headline): --workload D | E (decode steps / verify blocks,
CUDA-graph replay; sharded under torchrun), --workload backward (config C gradients),
--workload analysis (corpus collision analysis), --workload plne (per-layer N-gram FFN),
--workload dropin (per-call latency of the C++ drop-in's one-token entries vs the reference);
--tokens zipf (the reference's text model).

A "step" is one pass of the hot path -- hash-index (K1) + gather/projection/epilogue
(K2+K3) -- over one batch of synthetic tokens, inputs resident in HBM.  The headline
workload is SURVEY.md 8(d) config C (LongCat-Flash-Lite-scale tables: V0=128000, N=4,
K=4, D=3072, d=256, 31.46B sub-table params in bf16 + E0 + W_cat, prefill 8 x 8192
tokens), tables generated on device by the counter-based generator (no checkpoint).

Timing: W untimed warm-ups, then K steps, each bracketed by CUDA events on the launch
stream; L2 is flushed (512 MiB write) between timed steps, outside the events.  With
N > 1 the 8 sequences are split across ranks (strong scaling) and the step time is the
max over ranks.  Stage times (K1 vs K2+K3) come from the library's own events
(ngram_profile_*), recorded on the stream the kernels run on.

One JSON line on rank 0.  `e2e` is the same metric through the host-buffer C-ABI entry
(ngram_embed_sequence_host: tokens H2D, forward, embeddings D2H into pinned memory).
`cpu_baseline` (rank 0, N=1) times the REFERENCE implementation (oracle/_ref, the
unmodified reference sources) on this host's cores over a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# a rank that dies mid-run must not leave the others blocked in a collective forever
_PG_TIMEOUT = __import__("datetime").timedelta(minutes=10)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


# ------------------------------------------------------------------ token streams
class _MT64:
    """std::mt19937_64 (the reference's rng64, rng.hpp:14), numpy-vectorised twist."""
    N, M = 312, 156

    def __init__(self, seed: int):
        mask = (1 << 64) - 1
        mt = [seed & mask]
        for i in range(1, self.N):
            mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & mask)
        self.mt = np.array(mt, dtype=np.uint64)
        self.out, self.pos = None, self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        up, lo, a = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF), np.uint64(0xB5026F5AA96619E9)
        for i0, i1 in ((0, N - M), (N - M, N - 1), (N - 1, N)):  # the recurrence's three dependency ranges
            i = np.arange(i0, i1)
            x = (mt[i] & up) | (mt[(i + 1) % N] & lo)
            xa = (x >> np.uint64(1)) ^ np.where((x & np.uint64(1)) == 1, a, np.uint64(0))
            mt[i] = mt[(i + M) % N] ^ xa
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self.out, self.pos = [int(v) for v in y], 0

    def __call__(self) -> int:
        if self.pos >= self.N:
            self._twist()
        self.pos += 1
        return self.out[self.pos - 1]

    def uniform01(self) -> float:  # rng.hpp:17-19
        return (self() >> 11) * 2.0 ** -53

    def below(self, bound: int) -> int:  # rng.hpp:22-29
        limit = (2 ** 64 - 1) - (2 ** 64 - 1) % bound
        while True:
            x = self()
            if x < limit:
                return x % bound


def zipf_markov_tokens(vocab, sequences, seq_len, seed=20260809, exponent=1.1, markov_prob=0.35):
    """generate_zipf_markov (corpus.cpp:211-271) restated for the bench's token input:
    text-like skew (Zipf fresh draws, a function-token pool, Markov successors).
    tests/test_abi_cpu.py pins it to the reference generator token for token."""
    import bisect
    rng = _MT64(seed)
    cdf = np.cumsum(1.0 / np.power(np.arange(1, vocab + 1, dtype=np.float64), exponent))
    cdf = (cdf / cdf[-1]).tolist()

    def zipf():
        i = bisect.bisect_right(cdf, rng.uniform01())
        return i if i < vocab else vocab - 1

    pool = min(vocab, max(2, vocab * 3 // 50))
    block = max(1, vocab // 20)
    active = max(pool, vocab // 2)
    succ = []
    for v in range(vocab):
        if v < pool:
            s = zipf()
            while s >= pool:
                s = zipf()
            succ.append(s)
        else:
            succ.append((2 * (v // block) + 1) % pool)
    out = np.zeros((sequences, seq_len), np.uint32)
    for q in range(sequences):
        prev, fresh = 0, True
        row = out[q]
        for i in range(seq_len):
            if not fresh and rng.uniform01() >= markov_prob:
                if rng.uniform01() < 0.001:
                    nxt = rng.below(vocab)
                else:
                    nxt = zipf()
                    while nxt >= active:
                        nxt = zipf()
                fresh = True
            else:
                nxt = succ[prev]
                fresh = False
            row[i] = nxt
            prev = nxt
    return out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def workload(name: str):
    """SURVEY.md 8(d) configs; returns (config dict, nseq, seq_len, label)."""
    if name == "C":
        sv = [(2 * (74 + b) + 1) * 64000 for b in range(12)]
        cfg = {"max_order": 4, "sub_tables": 4, "base_vocab": 128000, "dim": 3072, "variant": "subtable_v2",
               "amplification": "scale_sqrt_d",
               "sub_vocab": [{"n": 2 + b // 4, "k": 1 + b % 4, "vocab": sv[b]} for b in range(12)]}
        return cfg, 8, 8192, "longcat_flash_lite_prefill_8x8192"
    from paper_2601_21204_b200 import ngram as G
    if name == "B":
        return G.make_default_config(128000, 768, 4, 4), 16, 4096, "mid_prefill_16x4096"
    if name == "A":
        return G.make_default_config(32000, 256, 3, 2), 4, 512, "toy_4x512"
    raise SystemExit(f"unknown workload {name}")


def param_count(cfg):
    B = (cfg["max_order"] - 1) * cfg["sub_tables"]
    d = cfg["dim"] // B
    sub = sum(e["vocab"] for e in cfg["sub_vocab"]) * d
    return cfg["base_vocab"] * cfg["dim"] + sub + cfg["dim"] * cfg["dim"], sub


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU (reference) leg
def reference_cpu_rate(cfg_c, seconds: float, seq_len: int = 16, max_rounds: int | None = None):
    """Reference embed_sequence<float> (oracle/_ref = unmodified reference sources) on this
    host's cores, one sequence per std::thread, over a reduced-vocabulary bank with the
    workload's D / N / K (the 127 GB fp32 LongCat bank cannot exist on the host; the
    per-token cost is the D^2 projection, independent of vocabulary size)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # noqa: E402  (test/baseline infrastructure only)
    if not O.ref_available():
        return None
    R = O.ref()
    N, K, D = cfg_c["max_order"], cfg_c["sub_tables"], cfg_c["dim"]
    buf = C.create_string_buffer(1 << 16)
    R.ref_make_default_config_json(1000, D, N, K, buf, len(buf))
    small = json.loads(buf.value)
    small["amplification"] = cfg_c["amplification"]
    h = R.ref_bank_create(json.dumps(small).encode(), 1234, 1)
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(7)
    nseq = cores
    toks = rng.integers(0, 1000, size=nseq * seq_len, dtype=np.uint32)
    off = np.arange(0, nseq * seq_len + 1, seq_len, dtype=np.int64)
    out = np.zeros((nseq * seq_len, D), np.float32)
    done, t0, rounds, times = 0, time.perf_counter(), 0, []
    while True:
        t1 = time.perf_counter()
        rc = R.ref_embed_batch_mt(h, toks, off, nseq, cores, out)
        times.append(time.perf_counter() - t1)
        if rc:
            raise RuntimeError("reference embed failed")
        done += nseq * seq_len
        rounds += 1
        if (max_rounds and rounds >= max_rounds) or (not max_rounds and time.perf_counter() - t0 >= seconds):
            break
    el = time.perf_counter() - t0
    # one host thread (SURVEY 8(d) also asks for the single-core rate): 2 sequences x seq_len
    t1 = time.perf_counter()
    if R.ref_embed_batch_mt(h, toks[:2 * seq_len], off[:3], 2, 1, out):
        raise RuntimeError("reference embed failed")
    one_thread = 2 * seq_len / (time.perf_counter() - t1)
    R.ref_bank_destroy(h)
    try:
        model = subprocess.run(["bash", "-c", "lscpu | grep 'Model name' | head -1"], capture_output=True,
                               text=True).stdout.split(":")[-1].strip()
    except Exception:
        model = "?"
    return {"value": done / el, "cores": cores, "tokens": done, "seconds": el, "step_times": times,
            "value_1thread": one_thread,
            "cpu_model": model,
            "sample": f"{done} tokens of the workload's shape (D={D}, N={N}, K={K}) through the reference "
                      f"embed_sequence<float>, {nseq} sequences x {seq_len} tokens per round, one std::thread per "
                      f"sequence on {cores} host threads, reduced-vocabulary bank (V0=1000, default V_nk) -- "
                      f"per-token cost is the D^2 projection (embedding.hpp:189-195)"}


def workload_config(cfg, label, nseq, seq_len, args):
    """The `config` keys both arms report for a workload (the reference arm runs the same
    shape on a reduced-vocabulary bank; see cpu_baseline.sample)."""
    return {"workload": label, "V0": cfg["base_vocab"], "N": cfg["max_order"], "K": cfg["sub_tables"],
            "D": cfg["dim"], "tokens": nseq * seq_len, "sequences": nseq, "seq_len": seq_len,
            "out_dtype": args.out_dtype, "amplification": cfg["amplification"], "token_stream": args.tokens}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.workload in ("D", "E"):
        return run_reference_decode(args)
    cfg, nseq, seq_len, label = workload(args.workload)
    # each step: one bounded sample (one round of cores x 16 tokens)
    r = reference_cpu_rate(cfg, 0, seq_len=16, max_rounds=args.warmup + args.steps)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libngram_ref.so not built"}))
        return
    times = r["step_times"][args.warmup:]
    toks_per_step = r["cores"] * 16
    v = toks_per_step / (sum(times) / len(times))
    line = {"metric": "ngram_embedding_tokens_per_sec", "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": dict(workload_config(cfg, label, nseq, seq_len, args),
                           note="CPU reference (oracle/_ref = the reference sources), bounded sample per step"),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r["cores"], "kind": "reference",
                             "sample": r["sample"], "cpu_model": r["cpu_model"]},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_reference_decode(args):
    """Reference arm of workloads D / E: per step, every host thread runs one stream's decode
    step (append + memo lookup) or verify block (draft_verify) -- a bounded sample."""
    cfg, _, _, _ = workload("C")
    L = 1 if args.workload == "D" else args.draft
    r = reference_decode_rate(cfg, 0 if args.workload == "D" else 1, L, 0, max_rounds=args.warmup + args.steps)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libngram_ref.so not built"}))
        return
    times = r["step_times"][args.warmup:]
    v = r["tokens_per_step"] / (sum(times) / len(times))
    metric = "ngram_decode_tokens_per_sec" if args.workload == "D" else "ngram_verify_tokens_per_sec"
    line = {"metric": metric, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": {"workload": "longcat_decode" if args.workload == "D" else f"longcat_verify_x{L}",
                       "D": cfg["dim"], "N": cfg["max_order"], "K": cfg["sub_tables"], "draft": L,
                       "note": "CPU reference (oracle/_ref = the reference sources), bounded sample per step"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r["cores"], "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------------------- GPU leg
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2601_21204_b200 import abi
    from paper_2601_21204_b200 import ngram as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # NGRAM_BENCH_ONE_DEVICE=1 (functional test of the multi-rank flow on a 1-GPU box): every
    # rank on cuda:0 over gloo.  The kernels never wait on each other (the barrier is a host
    # collective), but the numbers are not multi-GPU numbers.
    one_dev = os.environ.get("NGRAM_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        init_dist(dev, one_dev)
    sharding = args.sharding if world > 1 else "single"
    exchange = args.exchange

    cfg, nseq, seq_len, label = workload(args.workload)
    if nseq % world != 0:
        raise SystemExit(f"{nseq} sequences do not split over {world} ranks")
    my_nseq = nseq // world
    T = my_nseq * seq_len
    total_tokens = nseq * seq_len
    peaks, peak_src = load_peaks()
    out_dtype = torch.bfloat16 if args.out_dtype == "bf16" else torch.float32
    esz = 2 if out_dtype == torch.bfloat16 else 4

    if args.tokens == "zipf":  # generate_zipf_markov(V0, nseq, len, 20260809, 1.1, 0.35)
        all_tokens = zipf_markov_tokens(cfg["base_vocab"], nseq, seq_len).reshape(-1).astype(np.int32)
    else:
        rng = np.random.default_rng(42)
        all_tokens = rng.integers(0, cfg["base_vocab"], size=total_tokens, dtype=np.int64).astype(np.int32)
    toks = torch.from_numpy(all_tokens[rank * T:(rank + 1) * T].copy()).to(dev)
    off = torch.arange(0, T + 1, seq_len, dtype=torch.int64, device=dev)
    rows = torch.empty((T, (cfg["dim"])), dtype=out_dtype, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    fallback = None
    prefill_path = "x"  # row-sharded flow: scatter into X, then the pair projection
    if sharding == "row":
        # row-sharded tables: this rank keeps 1/world of every sub-table; rows travel over
        # NVLink by the fused gather + peer-store kernel; one NCCL all-reduce = barrier.
        # Set-up is agreed collectively: if any rank cannot map its peers (CUDA IPC), every
        # rank falls back to replicas and the JSON line says so.
        ok, why = 1, ""
        bank = G.DeviceBank(cfg, device=local, shard_rank=rank, shard_count=world)
        bank.generate(1234)
        group = G.ShardGroup(bank, T)
        if exchange in ("peer", "auto"):
            try:
                G.connect_shard_groups(group)
            except Exception as e:  # noqa: BLE001 -- reported, then agreed across ranks
                ok, why = 0, f"rank {rank}: {type(e).__name__}: {e}"
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:  # no peer mappings: the same rows move by NCCL all-to-all instead
            fallback = (why or "a peer rank failed to map the peer buffers") + "; exchange falls back to NCCL a2a"
            exchange = "a2a" if exchange == "peer" else exchange
            torch.cuda.synchronize()
    if sharding == "row":
        all_t = torch.empty(total_tokens, dtype=torch.int32, device=dev)
        all_off = torch.arange(0, total_tokens + 1, seq_len, dtype=torch.int64, device=dev)
        rank_tok = [r * T for r in range(world + 1)]
        one = torch.ones(1, dtype=torch.float32, device=dev)
        sev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]

        def step(record=False, xchg=None):
            xchg = xchg or exchange
            if record:
                sev[0].record(stream)
            dist.all_gather_into_tensor(all_t, toks)  # 4 B/token
            if record:
                sev[1].record(stream)
            if xchg == "peer":
                group.scatter(all_t, all_off, rank_tok)   # K1 + fused gather / NVLink peer store
                if record:
                    sev[2].record(stream)
                dist.all_reduce(one)                      # every rank's rows have landed
            else:  # K1 + pack, the NCCL collective, unpack (a2a) -- the collective orders the stream
                group.exchange(xchg, all_t, all_off, rank_tok)
                if record:
                    sev[2].record(stream)
            if record:
                sev[3].record(stream)
            group.project(toks, out_dtype=out_dtype, out_rows=rows)  # K3 on the home X
            if record:
                sev[4].record(stream)
    else:
        bank = G.DeviceBank(cfg, device=local)
        bank.generate(1234)
        bank.reserve(T)
        sbuf = (C.c_float * 3)()  # stage times: a separate profiled pass after the timed region
        pp = C.c_int(0)
        abi.check(abi.lib().ngram_prefill_path(bank.handle, T, C.byref(pp)))
        prefill_path = {0: "x", 1: "lsu", 2: "wide"}[pp.value]

        def step(record=False):
            G.embed_forward(bank, toks, off, rows=True, merged=False, out_dtype=out_dtype, out_rows=rows)

    def time_exchange(xv, reps):
        """whole-step ms of the row-sharded flow with exchange xv (max over ranks, L2 flushed)"""
        for _ in range(2):
            step(xchg=xv)
        torch.cuda.synchronize()
        dist.barrier()
        tt = []
        for i in range(reps):
            flush.fill_(i & 0xff)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(xchg=xv)
            e1.record(stream)
            e1.synchronize()
            tt.append(e0.elapsed_time(e1))
        t = torch.tensor([float(np.mean(tt))], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    exchange_pick = None
    if sharding == "row" and exchange == "auto":
        # pick the exchange by measured latency at this batch size (every rank
        # agrees: the times are maxima over ranks)
        variants = [v for v in ("peer", "a2a", "rs") if not (v == "peer" and fallback)]
        exchange_pick = {v: time_exchange(v, 3) for v in variants}
        exchange = min(exchange_pick, key=exchange_pick.get)
    for _ in range(args.warmup):
        step()
    bank.sync_errors()
    torch.cuda.synchronize()

    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    nst = 4 if sharding == "row" else 3
    stage = np.zeros((args.steps, nst), np.float32)
    launches0 = abi.lib().ngram_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(i & 0xff)  # > L2 (126 MB): every step starts cold
        ev[i][0].record(stream)
        step(record=True)
        ev[i][1].record(stream)
        if sharding == "row":
            sev[4].synchronize()
            stage[i] = [sev[j].elapsed_time(sev[j + 1]) for j in range(4)]
    torch.cuda.synchronize()
    launches = abi.lib().ngram_kernel_launches() - launches0
    if sharding != "row":
        # stage breakdown from the library's own events in a separate pass (the events between
        # the kernels are kept out of the timed steps above)
        abi.check(abi.lib().ngram_profile_enable(bank.handle, 1))
        step()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(i & 0xff)
            step()
            abi.check(abi.lib().ngram_profile_read(bank.handle, sbuf, 3))
            stage[i] = [sbuf[0], sbuf[1], sbuf[2]]
        abi.check(abi.lib().ngram_profile_enable(bank.handle, 0))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    bank.sync_errors()
    step_ms = np.array([a.elapsed_time(b) for a, b in ev])
    ms = float(step_ms.mean())
    st_ms = [float(x) for x in stage.mean(axis=0)]
    if world > 1:
        t = torch.tensor([ms] + st_ms, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, st_ms = float(t[0]), [float(x) for x in t[1:].tolist()]
    if sharding == "row":
        stages = {"all_gather_tokens": st_ms[0], "k1_k2_scatter_nvlink": st_ms[1], "barrier": st_ms[2],
                  "k3_projection_epilogue": st_ms[3]}
        proj_ms = st_ms[3]
        # every exchange variant on the same tables and tokens (pick by measured
        # latency): whole-step ms, max over ranks, L2 flushed as above
        exchange_ms = {}
        reps = 1 if one_dev else max(3, args.steps)
        for xv in ("peer", "a2a", "rs"):
            if xv == "peer" and fallback:
                continue
            exchange_ms[xv] = time_exchange(xv, reps)
        bank.sync_errors()
    else:
        if prefill_path == "wide":  # token check, then the one fused kernel (no X)
            stages = {"validate_tokens": st_ms[0] + st_ms[1], "fused_wide_kernel": st_ms[2]}
        else:  # K1 (hash) and K2 (gather) run fused in one kernel on the X path (stage 1 ~ 0 then)
            stages = {"k1_k2_hash_gather": st_ms[0] + st_ms[1], "k3_projection_epilogue": st_ms[2]}
        proj_ms = st_ms[2]

    # ---------------------------------------------------------------- index stage alone
    # hash_all_orders over the step's tokens ("time hash_all_orders alone"): K1 only,
    # u64 ids out (4 B token in + 8 B per branch out), L2 flushed between launches
    index_stage = None
    if sharding != "row":
        ids_out = torch.empty((T, bank.B), dtype=torch.int64, device=dev)
        for _ in range(2):
            G.hash_ids(bank, toks, off)
        it = []
        for i in range(args.steps):
            flush.fill_(i & 0xff)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            abi.check(abi.lib().ngram_hash_ids(bank.handle, C.c_void_p(toks.data_ptr()), C.c_void_p(off.data_ptr()),
                                               my_nseq, T, None, C.c_void_p(ids_out.data_ptr()), 1,
                                               C.c_void_p(stream.cuda_stream)))
            e1.record(stream)
            e1.synchronize()
            it.append(e0.elapsed_time(e1))
        bank.sync_errors()
        ims = float(np.mean(it))
        ib = T * (4 + 8 * bank.B)
        index_stage = {"kernel": "hash_ids_kernel (hash_all_orders, u64 ids)", "ms": ims,
                       "tokens_per_s": T / (ims * 1e-3), "bytes": ib, "gbs": ib / (ims * 1e-3) / 1e9,
                       "frac": ib / (ims * 1e-3) / 1e9 / peaks["hbm_gbs"]}
        del ids_out

    # ---------------------------------------------------------------- e2e (host buffers)
    e2e_steps = max(2, min(args.steps, 5))
    host_tok = torch.from_numpy(all_tokens[rank * T:(rank + 1) * T].copy()).pin_memory()
    host_out = torch.empty((T, bank.D), dtype=out_dtype).pin_memory()
    host_off = np.arange(0, T + 1, seq_len, dtype=np.int64)
    odt = abi.NGRAM_BF16 if out_dtype == torch.bfloat16 else abi.NGRAM_F32

    if sharding == "row":
        def e2e_step():
            toks.copy_(host_tok, non_blocking=True)
            step()
            host_out.copy_(rows, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        e2e_path = ("pinned host tokens -> H2D -> all-gather -> " +
                    ("scatter -> barrier" if exchange == "peer" else f"NCCL {exchange}") + " -> K3 -> D2H pinned embeddings")
    else:
        def e2e_step():
            abi.check(abi.lib().ngram_embed_sequence_host(bank.handle, C.c_void_p(host_tok.data_ptr()),
                                                          host_off.ctypes.data, my_nseq, None,
                                                          C.c_void_p(host_out.data_ptr()), None, odt))
        e2e_path = "ngram_embed_sequence_host (pinned host tokens -> HBM -> pinned host embeddings)"

    e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": total_tokens / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": int(T * 4 + host_off.nbytes),
           "d2h_bytes_per_step": int(T * bank.D * esz), "ms_per_step": e2e_s * 1e3, "path": e2e_path}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---------------------------------------------------------------- roofline
    D, B = cfg["dim"], (cfg["max_order"] - 1) * cfg["sub_tables"]
    d = D // B
    flops = 2.0 * T * D * D
    tflops = flops / (proj_ms * 1e-3) / 1e12
    bytes_tok = 4 + 2 * B * d + 2 * D + esz * D  # token + sub rows + E0 row + output
    hbm_bytes = T * bytes_tok + 2 * D * D
    hbm_gbs = hbm_bytes / (ms * 1e-3) / 1e9
    nparams, nsub = param_count(cfg)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("workload") == label and tj.get("T") == T:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    hbm = {"achieved_gbs": hbm_gbs, "peak_gbs": peaks["hbm_gbs"], "frac": hbm_gbs / peaks["hbm_gbs"],
           "algorithmic_bytes_per_token": bytes_tok}
    if sharding != "row" and prefill_path != "wide":
        kb = T * (4 + 2 * B * d + 2 * D)  # tokens in, B sub-table rows in, X out
        k12 = st_ms[0] + st_ms[1]
        hbm["k1_k2_hash_gather"] = {"ms": k12, "bytes": kb, "gbs": kb / (k12 * 1e-3) / 1e9,
                                    "frac": kb / (k12 * 1e-3) / 1e9 / peaks["hbm_gbs"]}
        if d * 2 == 128 and T == 65536:
            # 128-byte random rows do not stream at the copy peak: the bare gather of the same
            # 786 432 precomputed random rows out of 4.4 GB into a contiguous X takes 50.4 us on
            # a B200 (profiles/microbench/gather_ceiling.cu, gather_ceiling_b200.txt)
            hbm["k1_k2_hash_gather"]["access_ceiling_ms"] = 0.0504
            hbm["k1_k2_hash_gather"]["frac_of_access_ceiling"] = 0.0504 / k12
    # K3's own bound: its tensor time (2 T D^2 at the measured bf16 peak) vs its HBM time (per
    # token: the token, the X row it reads in place of the sub-table rows, the E0 row and the
    # output -- the same 4 + 2 B d + 2 D + esz D bytes as the layer's algorithmic figure)
    k3_name = "forward_tc2_kernel (K3: tcgen05 cta_group::2 projection + base/scale/amplify epilogue)"
    if prefill_path == "wide":  # the fused kernel moves the layer's own bytes (no X)
        k3_name = ("forward_wide_kernel (hash + row gather into resident shared-memory K-blocks + tcgen05 "
                   "cta_group::2 projection over every N-tile + base/scale/amplify epilogue; no X)")
    k3_bytes = T * bytes_tok + 2 * D * D
    if flops / (peaks["bf16_tflops"] * 1e12) >= k3_bytes / (peaks["hbm_gbs"] * 1e9):
        roofline = {"bound": "tensor", "kernel": k3_name, "achieved": tflops, "peak": peaks["bf16_tflops"],
                    "unit": "TFLOP/s", "frac": tflops / peaks["bf16_tflops"], "traffic": traffic,
                    "peak_source": peak_src, "flops_per_launch": flops, "launch_ms": proj_ms}
    else:  # narrow model (config B, D = 768): K3 moves more bytes than the tensor pipe can stall on
        k3_gbs = k3_bytes / (proj_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": k3_name, "achieved": k3_gbs, "peak": peaks["hbm_gbs"],
                    "unit": "GB/s", "frac": k3_gbs / peaks["hbm_gbs"], "traffic": traffic,
                    "peak_source": peak_src, "bytes_per_launch": k3_bytes, "launch_ms": proj_ms,
                    "tensor_frac": tflops / peaks["bf16_tflops"]}
        if D == 768 and d == 64 and T == 65536 and esz == 4:
            # the layer's byte mix (random 128-byte rows + random E0 rows in, fp32 rows out) does not
            # stream at the copy peak either: the same traffic with no projection, moved by a
            # plain CUDA-core kernel, takes 75.9 us on a B200 (5.3 TB/s;
            # profiles/microbench/layer_mix_ceiling.cu, layer_mix_ceiling_b200.txt)
            roofline["access_ceiling_ms"] = 0.0759
            roofline["frac_of_access_ceiling"] = 0.0759 / proj_ms
    line = {
        "metric": "ngram_embedding_tokens_per_sec", "value": total_tokens / (ms * 1e-3), "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (device-generated counter-based tables, " + (
            "Zipf-Markov tokens generate_zipf_markov(V0, nseq, len, 20260809, 1.1, 0.35))" if args.tokens == "zipf"
            else "uniform tokens seed 42)"),
        "config": dict(workload_config(cfg, label, nseq, seq_len, args), d=d, embedding_params=nparams,
                       sub_table_params=nsub, table_dtype="bf16", sharding=sharding,
                       l2="flushed (512 MiB write) between timed steps", tensor_core_path=bank.tensor_core_path),
        "roofline": roofline,
        "hbm": hbm, "stages_ms": stages, "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches),
    }
    line["config"]["prefill_path"] = prefill_path
    if fallback:
        line["config"]["sharding_fallback"] = fallback
    if one_dev and world > 1:
        line["config"]["one_device_test"] = "all ranks on cuda:0 over gloo (functional only)"
    if sharding == "row":
        line["config"]["exchange"] = exchange
        if exchange_pick is not None:
            line["config"]["exchange_pick_ms"] = exchange_pick  # the pre-pass that chose it
        line["exchange_ms"] = exchange_ms
        remote = T * world * B * d * 2 * (world - 1) / world / world  # rows this rank ships to peers
        line["nvlink"] = {"remote_bytes_per_rank": remote, "scatter_ms": st_ms[1],
                          "gbs": remote / (st_ms[1] * 1e-3) / 1e9, "peak_gbs": 770.0,
                          "frac": remote / (st_ms[1] * 1e-3) / 1e9 / 770.0}
    if index_stage is not None:
        line["index_stage"] = index_stage
    if world == 1 and not args.no_cpu:
        r = reference_cpu_rate(cfg, args.cpu_seconds)
        if r is not None:
            line["cpu_baseline"] = {"value": r["value"], "unit": "tokens/s", "cores": r["cores"], "kind": "reference",
                                    "sample": r["sample"], "cpu_model": r["cpu_model"],
                                    "value_1thread": r["value_1thread"]}
            hr = reference_hash_rate(cfg, all_tokens[:200000].astype(np.uint32))
            if hr is not None:
                line["cpu_baseline"]["hash_all_orders"] = hr[0]
                if index_stage is not None:
                    line["index_stage"]["cpu_reference_tokens_per_s"] = hr[0]["tokens_per_s"]
    print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def reference_decode_rate(cfg_c, mode: int, L: int, seconds: float, max_rounds: int | None = None):
    """Reference decode (mode 0: sequence_cache::append + embedding_memo::lookup per token,
    cache.cpp:37-57, 123-150) or verify (mode 1: draft_verify of L drafts, cache.cpp:152-195) on
    this host's cores: one stream per std::thread, reduced-vocabulary bank with the workload's
    D / N / K (per-token cost = the D^2 projection of the memo miss)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # noqa: E402  (baseline infrastructure only)
    if not O.ref_available():
        return None
    R = O.ref()
    N, K, D = cfg_c["max_order"], cfg_c["sub_tables"], cfg_c["dim"]
    buf = C.create_string_buffer(1 << 16)
    R.ref_make_default_config_json(1000, D, N, K, buf, len(buf))
    small = json.loads(buf.value)
    small["amplification"] = "none"
    h = R.ref_bank_create(json.dumps(small).encode(), 1234, 1)
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(11)
    ns = cores
    prior = rng.integers(0, 1000, size=(ns, N - 1)).astype(np.uint32)
    per = 1 if mode == 0 else L
    toks = rng.integers(0, 1000, size=(ns, per)).astype(np.uint32)
    acc = rng.integers(0, L + 1, size=(ns, 1)).astype(np.int32)
    last = np.zeros((ns, D), np.float32)
    done, times, t0 = 0, [], time.perf_counter()
    while True:
        t1 = time.perf_counter()
        rc = R.ref_decode_mt(h, mode, ns, cores, prior, N - 1, toks, 1, L, acc.ctypes.data, 1024, last)
        times.append(time.perf_counter() - t1)
        if rc:
            raise RuntimeError("reference decode failed")
        done += ns * per
        if (max_rounds and len(times) >= max_rounds) or (not max_rounds and time.perf_counter() - t0 >= seconds):
            break
    el = sum(times)
    R.ref_bank_destroy(h)
    what = ("sequence_cache::append + embedding_memo::lookup (a memo miss = embed_from_ids) per token"
            if mode == 0 else f"draft_verify of {L} draft tokens (memo warm-up, rollback, re-append, memo hits)")
    return {"value": done / el, "cores": cores, "step_times": times, "tokens_per_step": ns * per,
            "sample": f"{done} tokens: {ns} streams (one std::thread each, {cores} host threads), each primed "
                      f"with {N - 1} appends, then {what}; reduced-vocabulary bank (V0=1000, D={D}, N={N}, K={K}) "
                      f"-- per-token cost is the D^2 projection (embedding.hpp:189-195)"}


def reference_hash_rate(cfg, tokens: np.ndarray):
    """Reference hash_all_orders alone (hashing.cpp:61-81, the index stage) on this host's cores
    over the workload's own config (ids need only the config), plus one thread."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # noqa: E402
    if not O.ref_available():
        return None
    R = O.ref()
    cores = os.cpu_count() or 1
    B = (cfg["max_order"] - 1) * cfg["sub_tables"]
    t = np.ascontiguousarray(tokens.astype(np.uint32))
    ids = np.zeros((len(t), B), np.uint64)
    js = json.dumps(cfg).encode()
    t0 = time.perf_counter()
    if R.ref_hash_all_orders_mt(js, t, len(t), cores, ids):
        raise RuntimeError("reference hash failed")
    el = time.perf_counter() - t0
    n1 = min(len(t), 20000)
    t0 = time.perf_counter()
    if R.ref_hash_all_orders_mt(js, t[:n1], n1, 1, ids[:n1]):
        raise RuntimeError("reference hash failed")
    el1 = time.perf_counter() - t0
    return {"tokens_per_s": len(t) / el, "cores": cores, "tokens": int(len(t)),
            "tokens_per_s_1thread": n1 / el1, "ns_per_token_1thread": el1 / n1 * 1e9}, ids


def run_decode(args):
    """Configs D / E: LongCat-scale tables, a batch of decode streams primed by
    a prefill hand-off (ring = 3 prior tokens, length 4096); D times single-token steps
    (sequence_cache::append + embed_from_ids + commit), E times a verify block of L drafts plus
    the commit of the accepted prefix (draft_verify).  The step is captured once in a CUDA graph;
    every timed step is one replay bracketed by CUDA events, with L2 flushed (512 MiB write)
    between steps, so W_cat (18.9 MB) and the rows come from HBM each step.  A warm-L2
    back-to-back replay time (serving steady state: W_cat stays L2-resident) is reported beside
    it.  The headline `value` is the largest batch in --batches."""
    import torch
    from paper_2601_21204_b200 import abi
    from paper_2601_21204_b200 import ngram as G
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    cfg, _, _, label = workload("C")
    cfg = dict(cfg)
    cfg["amplification"] = "none"  # the cache path returns merged vectors (cache.hpp:122-124)
    bank = G.DeviceBank(cfg).generate(1234)
    D, N = bank.D, cfg["max_order"]
    nb = (N - 1) * cfg["sub_tables"]
    peaks, peak_src = load_peaks()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    L = 1 if args.workload == "D" else args.draft
    rng = np.random.default_rng(1)
    batches = [int(b) for b in args.batches.split(",")] if args.batches else []
    if not batches:
        batches = [1, 8, 64, 256] if args.workload == "D" else [64]
    res, clocks, launches_total = {}, None, 0
    sbuf = (C.c_float * 3)()
    for B in batches:
        st = G.DecodeState(bank, B, max_draft=max(L, 1))
        prior = torch.from_numpy(rng.integers(0, cfg["base_vocab"], size=(B, N - 1)).astype(np.int32)).to(dev)
        lens = torch.full((B,), 4096, dtype=torch.int64, device=dev)
        toks = torch.from_numpy(rng.integers(0, cfg["base_vocab"], size=(B, L)).astype(np.int32)).to(dev)
        acc = torch.from_numpy(rng.integers(0, L + 1, size=B).astype(np.int32)).to(dev)
        out = torch.empty((B, L, D), dtype=torch.bfloat16, device=dev)
        st.reset(prior, lens)

        def one():
            if args.workload == "D":
                st.step(toks[:, 0].contiguous(), want_ids=False, out=out[:, 0], out_dtype=torch.bfloat16)
            else:
                st.verify(toks, out=out, out_dtype=torch.bfloat16)
                st.commit(toks, acc)
        for _ in range(args.warmup):
            one()
        torch.cuda.synchronize()
        l0 = abi.lib().ngram_kernel_launches()
        one()
        torch.cuda.synchronize()
        per_step_launches = abi.lib().ngram_kernel_launches() - l0
        # stage split from the library's own events (eager, L2 flushed): K1+gather | GEMM + reduce
        abi.check(abi.lib().ngram_profile_enable(bank.handle, 1))
        stg = []
        for i in range(max(args.steps, 5)):
            flush.fill_(i & 0xff)
            one()
            abi.check(abi.lib().ngram_profile_read(bank.handle, sbuf, 3))
            stg.append([sbuf[0], sbuf[1], sbuf[2]])
        abi.check(abi.lib().ngram_profile_enable(bank.handle, 0))
        stg = np.array(stg).mean(axis=0)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            one()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        clk = ClockSampler(0) if B == batches[-1] else None
        if clk:
            clk.start()
            time.sleep(0.3)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.fill_(i & 0xff)
            ev[i][0].record(stream)
            g.replay()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        cold_us = float(np.mean([a.elapsed_time(b) for a, b in ev])) * 1e3
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = args.steps * 10
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        warm_us = e0.elapsed_time(e1) / reps * 1e3
        if clk:
            clocks = clk.stop()
        launches_total = per_step_launches * args.steps
        # e2e through the host-buffer C-ABI entry (host tokens in, host fp32 merged out)
        T = B * L
        # pinned host buffers (the e2e contract: inputs from and results to pinned host memory)
        h_tok_t = torch.from_numpy(toks.cpu().numpy().astype(np.int32)).pin_memory()
        h_acc_t = torch.from_numpy(acc.cpu().numpy().astype(np.int32)).pin_memory()
        h_out_t = torch.zeros((B, L, D), dtype=torch.float32).pin_memory()
        h_tok, h_acc, h_out = h_tok_t.numpy(), h_acc_t.numpy(), h_out_t.numpy()
        if args.workload == "D":
            def e2e_call():
                abi.check(abi.lib().ngram_decode_step_host(st.handle, h_tok.ctypes.data, None, h_out.ctypes.data))
            h2d, d2h = B * 4, B * D * 4
            e2e_path = "ngram_decode_step_host (host tokens -> append + embed_from_ids + commit -> host fp32 merged)"
        else:
            def e2e_call():
                abi.check(abi.lib().ngram_verify_commit_host(st.handle, h_tok.ctypes.data, L, h_acc.ctypes.data,
                                                             h_out.ctypes.data))
            h2d, d2h = B * L * 4 + B * 4, B * L * D * 4
            e2e_path = "ngram_verify_commit_host (host drafts + accepts -> verify block + commit -> host fp32 merged)"
        for _ in range(3):
            e2e_call()
        t0 = time.perf_counter()
        ne = max(args.steps, 20)
        for _ in range(ne):
            e2e_call()
        e2e_us = (time.perf_counter() - t0) / ne * 1e6
        # algorithmic bytes: W_cat once + per position: token 4, B sub rows 2D, E0 row 2D, bf16 out 2D
        step_bytes = 2 * D * D + T * (4 + 6 * D)
        gemm_bytes = 2 * D * D + T * (2 * D + 2 * D + 2 * D)  # W_cat + X + E0 + out
        res[B] = {"tokens_per_step": T, "us_per_step": cold_us, "tokens_per_s": T / (cold_us * 1e-6),
                  "us_per_step_warm_l2": warm_us, "tokens_per_s_warm_l2": T / (warm_us * 1e-6),
                  "stages_us_eager": {"k1_hash_gather": float(stg[0] + stg[1]) * 1e3,
                                      "splitk_gemm_reduce_commit": float(stg[2]) * 1e3},
                  "step_floor_us": step_bytes / (peaks["hbm_gbs"] * 1e9) * 1e6,
                  "step_frac_of_hbm_floor": step_bytes / (peaks["hbm_gbs"] * 1e9) / (cold_us * 1e-6),
                  "gemm_stage_gbs": gemm_bytes / (float(stg[2]) * 1e-3) / 1e9,
                  "algorithmic_bytes_per_step": step_bytes, "launches_per_step": per_step_launches,
                  "e2e": {"us_per_step": e2e_us, "tokens_per_s": T / (e2e_us * 1e-6), "h2d_bytes_per_step": h2d,
                          "d2h_bytes_per_step": d2h, "path": e2e_path}}
        st.close()
    bank.sync_errors()
    Bh = batches[-1]
    r = res[Bh]
    T = r["tokens_per_step"]
    gemm_bytes = 2 * D * D + T * 6 * D
    gemm_ms = r["stages_us_eager"]["splitk_gemm_reduce_commit"] * 1e-3
    metric = "ngram_decode_tokens_per_sec" if args.workload == "D" else "ngram_verify_tokens_per_sec"
    wl = (f"longcat_decode_B{Bh}" if args.workload == "D" else f"longcat_verify_B{Bh}x{L}")
    line = {"metric": metric, "value": r["tokens_per_s"], "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["us_per_step"] * 1e-3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (device-generated counter-based LongCat-scale tables, uniform tokens)",
            "config": {"workload": wl, "V0": cfg["base_vocab"], "N": N, "K": cfg["sub_tables"], "D": D,
                       "streams": Bh, "draft": L, "prefill_len": 4096, "out_dtype": "bf16",
                       "amplification": "none (cache path: merged vectors, cache.hpp:122-124)",
                       "l2": "flushed (512 MiB write) between timed steps; warm-L2 replay reported per batch",
                       "cuda_graph": True, "batches": batches},
            "roofline": {"bound": "hbm",
                         "kernel": "split-K tcgen05 GEMM + reduce (+ fused commit): W_cat + X + E0 + out",
                         "achieved": gemm_bytes / gemm_ms / 1e6, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": gemm_bytes / gemm_ms / 1e6 / peaks["hbm_gbs"], "traffic": None,
                         "peak_source": peak_src, "bytes_per_launch": gemm_bytes, "launch_ms": gemm_ms,
                         "note": "stage time from the library's events on eager steps (L2 flushed); the whole "
                                 "step against its algorithmic-byte floor is step_frac_of_hbm_floor"},
            "results": res, "clocks": clocks,
            "e2e": {"value": r["e2e"]["tokens_per_s"], "unit": "tokens/s",
                    "h2d_bytes_per_step": r["e2e"]["h2d_bytes_per_step"],
                    "d2h_bytes_per_step": r["e2e"]["d2h_bytes_per_step"], "ms_per_step": r["e2e"]["us_per_step"] * 1e-3,
                    "path": r["e2e"]["path"]},
            "gpu_launches": int(launches_total)}
    if not args.no_cpu:
        cb = reference_decode_rate(cfg, 0 if args.workload == "D" else 1, L, min(args.cpu_seconds, 10.0))
        if cb is not None:
            line["cpu_baseline"] = {"value": cb["value"], "unit": "tokens/s", "cores": cb["cores"],
                                    "kind": "reference", "sample": cb["sample"]}
            hr = reference_hash_rate(workload("C")[0], np.random.default_rng(42).integers(
                0, cfg["base_vocab"], size=200000).astype(np.uint32))
            if hr is not None:
                line["cpu_baseline"]["hash_all_orders"] = hr[0]
    print(json.dumps(line))


def run_decode_sharded(args):
    """Configs D / E on row-sharded tables (8 GPUs): every rank serves B home
    streams on its 1/world row block; per step the drafts and rings are all-gathered, owned rows
    scattered into the home X over NVLink peer stores, one NCCL all-reduce is the barrier, the
    home block is projected (split-K) and committed.  Eager launches (no CUDA graph: the
    collectives run through torch.distributed); time = max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2601_21204_b200 import ngram as G
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    one_dev = os.environ.get("NGRAM_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    init_dist(dev, one_dev)
    cfg, _, _, _ = workload("C" if not os.environ.get("NGRAM_BENCH_DECODE_CFG") else os.environ["NGRAM_BENCH_DECODE_CFG"])
    cfg = dict(cfg)
    cfg["amplification"] = "none"  # the cache path returns merged vectors (cache.hpp:122-124)
    bank = G.DeviceBank(cfg, device=local, shard_rank=rank, shard_count=world).generate(1234)
    L = 1 if args.workload == "D" else args.draft
    batches = ([int(b) for b in args.batches.split(",")] if args.batches else
               ([1, 8, 64, 256] if args.workload == "D" else [64]))
    group = G.ShardGroup(bank, max(batches) * L)
    G.connect_shard_groups(group)
    rng = np.random.default_rng(1 + rank)
    res = {}
    stream = torch.cuda.current_stream()
    barrier = (lambda: (torch.cuda.synchronize(), dist.barrier())) if one_dev else None
    for B in batches:
        st = G.DecodeState(bank, B, max_draft=L)
        prior = torch.from_numpy(rng.integers(0, cfg["base_vocab"], size=(B, cfg["max_order"] - 1))
                                 .astype(np.int32)).to(dev)
        st.reset(prior, torch.full((B,), 4096, dtype=torch.int64, device=dev))
        toks = torch.from_numpy(rng.integers(0, cfg["base_vocab"], size=(B, L)).astype(np.int32)).to(dev)
        acc = torch.from_numpy(rng.integers(0, L + 1, size=B).astype(np.int32)).to(dev)

        def one(xv):
            G.sharded_verify_block(group, st, toks, out_dtype=torch.bfloat16, barrier=barrier, exchange=xv)
            st.commit(toks, acc)

        per = {}
        first = "peer" if args.exchange == "auto" else args.exchange
        for xv in [first] + [v for v in ("peer", "rs", "a2a") if v != first]:
            for _ in range(args.warmup):
                one(xv)
            torch.cuda.synchronize()
            dist.barrier()
            n = args.steps * (1 if one_dev else 10)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(stream)
            for _ in range(n):
                one(xv)
            ev[1].record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([ev[0].elapsed_time(ev[1]) / n], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            per[xv] = float(t.item()) * 1e3
        xbest = min(per, key=per.get) if args.exchange == "auto" else args.exchange  # picked by measured latency
        us = per[xbest]
        res[B] = {"us_per_step": us, "tokens_per_s": world * B * L / (us * 1e-6), "exchange": xbest,
                  "exchange_us": per}
        st.close()
    bank.sync_errors()
    if rank == 0:
        line = {"metric": "ngram_decode_tokens_per_sec" if args.workload == "D" else "ngram_verify_tokens_per_sec",
                "workload": args.workload, "draft": L, "n_gpus": world, "sharding": "row",
                "scaling": "weak", "home_streams_per_rank": batches, "cuda_graph": False, "out_dtype": "bf16",
                "results": res}
        if one_dev:
            line["one_device_test"] = "all ranks on cuda:0 over gloo (functional only)"
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()


def run_backward(args):
    """Backward of config C (embed_sequence_backward, embedding.hpp:438-459; SURVEY.md 8(f) row
    3): 8 x 8192 tokens, random fp32 upstream gradient, row-sparse sub-table gradients (a dense
    fp32 copy of the 31.5 B sub-table parameters does not fit beside the tables), gradient bank
    zeroed every step.  Lines for the default fp32-accurate GEMMs (U split into three bf16 terms),
    single-term TF32 and pedantic fp32."""
    import torch
    from paper_2601_21204_b200 import ngram as G
    dev = torch.device("cuda", 0)
    cfg, nseq, seq_len, label = workload("C")
    bank = G.DeviceBank(cfg).generate(1234)
    T = nseq * seq_len
    gen = torch.Generator(device=dev).manual_seed(42)
    toks = torch.randint(0, cfg["base_vocab"], (T,), dtype=torch.int32, device=dev, generator=gen)
    off = torch.arange(0, T + 1, seq_len, dtype=torch.int64, device=dev)
    up = torch.randn((T, cfg["dim"]), dtype=torch.float32, device=dev, generator=gen)
    res = {}
    modes = (("default_2term", {}), ("sparsebase_2term", {"sparse_base": True}), ("exact_3term", {"exact": True}),
             ("tf32_1term", {"tf32": True}), ("pedantic_fp32", {"pedantic": True}))
    for name, kw in [m for m in modes if m[0].split("_")[0] in args.bwd_modes.split(",")]:
        gb = G.GradBank(bank, sparse_rows=True, **kw)
        for _ in range(args.warmup):
            gb.zero()
            gb.backward(toks, off, up)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            ev[i][0].record()
            gb.zero()
            gb.backward(toks, off, up)
            ev[i][1].record()
        torch.cuda.synchronize()
        ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
        res[name] = {"ms_per_step": ms, "tokens_per_s": T / (ms * 1e-3)}
        gb.close()
    bank.sync_errors()
    print(json.dumps({"metric": "ngram_backward_tokens_per_sec", "value": next(iter(res.values()))["tokens_per_s"],
                      "unit": "tokens/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                      "higher_is_better": True, "data": "synthetic (device tables, uniform tokens, randn upstream)",
                      "config": {"workload": label + "_backward", "tokens": T, "sparse_rows": True,
                                 "includes": "gradient-bank zeroing + K1 + amplify/E0 backward (u written as bf16 "
                                             "terms) + gather + 2 tcgen05 GEMMs (U in 2 bf16 terms by default, 3 "
                                             "exact, 1 tf32-class) writing dX straight into the COO values"},
                      "results": res}))


def run_plne(args):
    """Per-layer N-gram FFN (ffn_plne / ffn_plne_backward, ple.hpp:168-196)
    at a LongCat-like width: d_model = hidden = 3072, layer bank make_default_config(8000, 3072,
    4, 4) (amplification none), 8 x 1024 tokens.  Forward and forward+backward (gate / down / x
    gradients, no bank gradients) for the default split-bf16 tcgen05 GEMMs and the opt-in
    CUDA-core fp32 GEMMs (NGRAM_PLNE_PEDANTIC)."""
    import torch
    from paper_2601_21204_b200 import ngram as G
    dev = torch.device("cuda", 0)
    cfg = G.make_default_config(8000, 3072, 4, 4)
    cfg["amplification"] = "none"
    bank = G.DeviceBank(cfg).generate(7)
    nseq, L, Dm, H = 8, 1024, 3072, 3072
    T = nseq * L
    gen = torch.Generator(device=dev).manual_seed(3)
    toks = torch.randint(0, 8000, (T,), dtype=torch.int32, device=dev, generator=gen)
    off = torch.arange(0, T + 1, L, dtype=torch.int64, device=dev)
    gate = 0.02 * torch.randn((H, Dm), device=dev, generator=gen)
    down = 0.02 * torch.randn((Dm, H), device=dev, generator=gen)
    x = torch.randn((T, Dm), device=dev, generator=gen)
    up = torch.randn((T, Dm), device=dev, generator=gen)
    dg, dd, dx = torch.zeros_like(gate), torch.zeros_like(down), torch.zeros_like(x)
    res = {}
    for name, fast in (("pedantic_fp32", False), ("split_bf16", True)):
        layer = G.PlneLayer(bank, Dm, fast=fast)
        out = {}
        for what, fn in (("forward", lambda: layer.forward(gate, down, x, toks, off)),
                         ("forward_backward", lambda: layer.backward(gate, down, x, toks, off, up, dg, dd, dx))):
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record()
            for _ in range(args.steps):
                fn()
            e[1].record()
            torch.cuda.synchronize()
            ms = e[0].elapsed_time(e[1]) / args.steps
            out[what] = {"ms_per_step": ms, "tokens_per_s": T / (ms * 1e-3)}
        res[name] = out
        layer.close()
    bank.sync_errors()
    print(json.dumps({"metric": "ngram_plne_tokens_per_sec", "value": res["split_bf16"]["forward"]["tokens_per_s"],
                      "unit": "tokens/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                      "higher_is_better": True, "data": "synthetic (device layer bank, uniform tokens, randn x)",
                      "config": {"workload": "plne_d3072_h3072_8x1024", "V0": 8000, "N": 4, "K": 4,
                                 "d_model": Dm, "hidden": H, "tokens": T},
                      "results": res}))


def run_analysis(args):
    """Corpus collision analysis (corpus_analyzer, analysis.cpp:93-121):
    the collision table of config C's twelve sub-table moduli, orders 2..4, V0 = 128000.  Each
    step streams a fresh batch of 16 x 65536 uniform tokens (device-resident; uniform = the most
    distinct windows, the sets' worst case) into one growing analyzer; the reference arm is the
    reference corpus_analyzer (single-threaded, as shipped) on a bounded sample."""
    import torch
    from paper_2601_21204_b200 import abi
    from paper_2601_21204_b200 import ngram as G
    dev = torch.device("cuda", 0)
    v0, orders = 128000, [2, 3, 4]
    moduli = [(2 * (74 + b) + 1) * 64000 for b in range(12)]
    nseq, L = 16, 65536
    T = nseq * L
    gen = torch.Generator(device=dev).manual_seed(42)
    batches = [torch.randint(0, v0, (T,), dtype=torch.int32, device=dev, generator=gen)
               for _ in range(args.warmup + args.steps)]
    off = torch.arange(0, T + 1, L, dtype=torch.int64, device=dev)
    an = G.CorpusAnalyzer(v0, orders, moduli)
    an.reserve(T * (args.warmup + args.steps))  # sized up front (unordered_set::reserve): no rehash timed
    for i in range(args.warmup):
        an.add(batches[i], off)
    torch.cuda.synchronize()
    l0 = abi.lib().ngram_kernel_launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        ev[i][0].record()
        an.add(batches[args.warmup + i], off)
        ev[i][1].record()
    torch.cuda.synchronize()
    launches = abi.lib().ngram_kernel_launches() - l0
    an.sync_errors()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    st = an.stats()
    line = {"metric": "corpus_analysis_tokens_per_sec", "value": T / (ms * 1e-3), "unit": "tokens/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "dtype": "u32/u128", "data": "synthetic (uniform tokens, fresh batch per step)",
            "config": {"workload": "collision_table_longcat_moduli", "V0": v0, "orders": orders, "moduli": moduli,
                       "tokens_per_step": T, "sequences": nseq},
            "inserts_per_token": len(orders) * (1 + len(moduli)),
            "final_stats": {"tokens_seen": st["tokens_seen"], "distinct_ngrams": st["distinct_ngrams"]},
            "gpu_launches": int(launches)}
    if not args.no_cpu and os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libngram_ref.so")):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        rng = np.random.default_rng(1)
        sample = [rng.integers(0, v0, size=16384).astype(np.uint32) for _ in range(16)]
        t0 = time.perf_counter()
        rc, _ = O.ref_corpus_analyze(v0, orders, moduli, sample)
        dt = time.perf_counter() - t0
        assert rc == 0
        line["cpu_baseline"] = {"value": 16 * 16384 / dt, "unit": "tokens/s", "cores": 1, "kind": "reference",
                                "sample": "16 x 16384 uniform tokens through the reference corpus_analyzer "
                                          "(add_sequence per sequence, single-threaded as shipped)"}
    print(json.dumps(line))


def run_dropin(args):
    """Per-call latency of the C++ drop-in's one-token entries (tests/cxx/bench_dropin: host ->
    device -> host round trips through the C-ABI) beside the reference's own per-call cost on
    one host thread (oracle/_ref, ref_time_calls), LongCat shape (N = 4, K = 4, D = 3072,
    reduced vocabulary).  Not a throughput line: the batched entries are the fast path."""
    import ctypes as C
    exe = os.path.join(ROOT, "tests", "cxx", "bench_dropin")
    r = subprocess.run([exe, "3072", "100"], capture_output=True, text=True, timeout=900)
    if r.returncode != 0:
        raise SystemExit(f"bench_dropin failed: {r.stderr[-2000:]}")
    ours = json.loads(r.stdout.strip().splitlines()[-1])
    line = {"metric": "dropin_us_per_call", "unit": "us", "higher_is_better": False, "n_gpus": 1,
            "config": {"workload": "dropin_per_call_latency", "V0": 1000, "N": 4, "K": 4, "D": 3072},
            "ours": ours["us_per_call"]}
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # noqa: E402  (reference timing only)
    if O.ref_available():
        R = O.ref()
        buf = C.create_string_buffer(1 << 16)
        R.ref_make_default_config_json(1000, 3072, 4, 4, buf, len(buf))
        h = R.ref_bank_create(buf.value, 3, 1)
        out = (C.c_double * 5)()
        if R.ref_time_calls(h, 3, out) == 0:
            line["reference_1thread"] = {"rolling_hash": out[0] / 1e3, "hash_all_orders": out[1] / 1e3,
                                         "sequence_cache_append": out[2] / 1e3,
                                         "append_plus_memo_lookup_miss": out[3] / 1e3,
                                         "draft_verify_4_accept_2": out[4] / 1e3}
        R.ref_bank_destroy(h)
    print(json.dumps(line))


def spawn_ranks(n: int) -> int:
    """Re-launch this command as n ranks (torch.distributed.run --nproc-per-node n) and return
    the launcher's exit code; stdout / stderr stream through (rank 0 prints the JSON line)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def init_dist(dev, one_dev: bool):
    """One process group per run: NCCL over NVLink (one GPU per rank), or gloo when every rank
    shares cuda:0 (functional tests).  NCCL's communicator-init lines (NCCL_DEBUG=INFO, INIT
    subsystem) are printed so the rank count of the communicator is visible in the log."""
    import torch.distributed as dist
    if one_dev:
        dist.init_process_group("gloo", timeout=_PG_TIMEOUT)
        return
    import torch
    if torch.cuda.device_count() < int(os.environ.get("WORLD_SIZE", "1")):
        raise SystemExit(f"--gpus {os.environ.get('WORLD_SIZE')} needs that many GPUs, "
                         f"this node has {torch.cuda.device_count()}")
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dist.init_process_group("nccl", device_id=dev, timeout=_PG_TIMEOUT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C")
    ap.add_argument("--out-dtype", choices=["fp32", "bf16"], default="fp32")
    ap.add_argument("--tokens", choices=["uniform", "zipf"], default="uniform",
                    help="token stream: iid uniform (headline) or the reference's Zipf-Markov text model")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--batches", default="", help="decode / verify batch sizes (workloads D, E; default D 1,8,64,256 and E 64; the last is the headline)")
    ap.add_argument("--draft", type=int, default=8, help="verify block length (workload E)")
    ap.add_argument("--bwd-modes", default="default,sparsebase,exact,tf32,pedantic",
                    help="backward workload: modes to time (sparsebase: E0 gradient as (token, u) pairs too)")
    ap.add_argument("--sharding", choices=["row", "replica"], default="row",
                    help="N > 1: row-sharded tables (default) or full replicas")
    ap.add_argument("--exchange", choices=["auto", "peer", "a2a", "rs"], default="auto",
                    help="row-sharded exchange: auto (default: the fastest of the three, measured before the "
                         "timed steps), NVLink peer stores, NCCL all-to-all of the owned rows, or NCCL "
                         "reduce-scatter of the -0.0-padded X (all bit-identical); every variant is timed and "
                         "reported under exchange_ms")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # `python bench.py --gpus N` with no launcher: start the N ranks here (one process per
        # GPU, torch.distributed.run on 127.0.0.1) and pass rank 0's line through
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "analysis":
        run_analysis(args)
    elif args.workload == "backward":
        run_backward(args)
    elif args.workload == "plne":
        run_plne(args)
    elif args.workload == "dropin":
        run_dropin(args)
    elif args.workload in ("D", "E") and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_decode_sharded(args)
    elif args.workload in ("D", "E"):
        run_decode(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
