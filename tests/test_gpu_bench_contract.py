"""bench.py's JSON line (the driver's contract) on a small workload: every required key,
the roofline / e2e / clocks objects and a non-zero count of this library's kernel launches."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract(cuda):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--no-cpu",
                          "--workload", "A"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["value"] > 0 and line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] >= 3
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in line["roofline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in line["e2e"], k
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in line["clocks"], k
    assert line["gpu_launches"] > 0 and line["config"]["workload"]


def _contract_keys(line):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in line, k
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in line["roofline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in line["e2e"], k
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0 and line["value"] > 0


@pytest.mark.parametrize("wl,extra", [("D", ["--batches", "1,8"]), ("E", ["--batches", "4", "--draft", "4"])])
def test_bench_decode_verify_contract(cuda, wl, extra):
    """The decode (D) and verify (E) lines carry the same keys as the prefill line, plus the
    reference CPU baseline (sequence_cache::append + memo / draft_verify, hash_all_orders)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                          "--workload", wl, "--cpu-seconds", "0.5"] + extra,
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    _contract_keys(line)
    assert line["roofline"]["bound"] == "hbm"
    if "cpu_baseline" in line:  # oracle/_ref travels with the snapshot when it was built
        cb = line["cpu_baseline"]
        assert cb["kind"] == "reference" and cb["value"] > 0 and cb["cores"] >= 1
        assert cb["hash_all_orders"]["tokens_per_s"] > 0
    for r in line["results"].values():
        assert r["us_per_step"] > 0 and r["e2e"]["us_per_step"] > 0


@pytest.mark.parametrize("sharding", ["row", "replica"])
def test_bench_two_ranks_one_device(cuda, sharding):
    """The N > 1 flow of bench.py (torchrun, row-sharded exchange over CUDA IPC or replicas,
    max-over-ranks timing, rank-0 JSON line) run functionally with both ranks on cuda:0 over
    gloo -- the pool has one GPU, so this is the only way to execute it before the driver's
    multi-GPU run."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, NGRAM_BENCH_ONE_DEVICE="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "B", "--sharding", sharding],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["sharding"] == sharding and "sharding_fallback" not in line["config"]
    assert line["e2e"]["value"] > 0 and "cpu_baseline" not in line
    if sharding == "row":
        assert set(line["stages_ms"]) == {"all_gather_tokens", "k1_k2_scatter_nvlink", "barrier",
                                          "k3_projection_epilogue"}
        # --exchange auto (default): the variant with the lowest pre-measured step time is timed
        pick = line["config"]["exchange_pick_ms"]
        assert line["config"]["exchange"] == min(pick, key=pick.get)
        assert set(line["exchange_ms"]) == set(pick)


def test_bench_gpus_flag_launches_the_ranks_itself(cuda):
    """`python bench.py --gpus 2` with no torchrun wrapper (the driver's command line) starts the
    two ranks itself: the line reports n_gpus = 2 and the row-sharded stages."""
    env = dict(os.environ, NGRAM_BENCH_ONE_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup",
                          "3", "--workload", "B"], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["sharding"] == "row"
    assert set(line["stages_ms"]) == {"all_gather_tokens", "k1_k2_scatter_nvlink", "barrier", "k3_projection_epilogue"}


def test_bench_sharded_verify_two_ranks_one_device(cuda):
    """bench.py --workload E at N = 2 (row-sharded verify + commit), functional, one device."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, NGRAM_BENCH_ONE_DEVICE="1", NGRAM_BENCH_DECODE_CFG="B")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "1", "--warmup", "3", "--workload", "E", "--batches", "1,8",
                          "--draft", "4"], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and set(line["results"]) == {"1", "8"}
    assert all(v["tokens_per_s"] > 0 for v in line["results"].values())
