"""Build libngram_b200.so in-tree with nvcc for sm_100a (no torch involvement).

    python -m paper_2601_21204_b200.build          # incremental
    python -m paper_2601_21204_b200.build --clean

Every .cu/.cpp under csrc/ is compiled with
    nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++20
and linked (static cudart) into paper_2601_21204_b200/libngram_b200.so.  Plain
`-arch=sm_100a` would also embed compute_100 PTX, which ptxas rejects for tcgen05 /
tile::gather4 -- hence the explicit -gencode.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "ngram_b200")
LIB = os.path.join(PKG, "libngram_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
JSON_DIR = os.environ.get(
    "NGRAM_JSON_DIR",
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")

GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
          "-isystem", JSON_DIR, "--expt-relaxed-constexpr"]


def _sources():
    """Sources of libngram_b200.so (kernels + C-ABI host layer); csrc/cxx is the C++ drop-in."""
    srcs = glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True) + \
        glob.glob(os.path.join(CSRC, "**", "*.cpp"), recursive=True)
    return sorted(s for s in srcs if os.sep + "cxx" + os.sep not in s)


def _headers():
    return (glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True) +
            glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True) +
            glob.glob(os.path.join(ROOT, "include", "*.h")))


def _obj(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(BUILD, rel + ".o")


def _compile(src, verbose=False):
    obj = _obj(src)
    cmd = [NVCC] + GENCODE + COMMON + ["-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    else:
        cmd += ["-x", "cu"] if False else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(clean: bool = False, verbose: bool = False) -> str:
    if clean and os.path.isdir(BUILD):
        shutil.rmtree(BUILD)
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    newest_hdr = max((os.path.getmtime(h) for h in _headers()), default=0)
    todo = [s for s in srcs if not os.path.exists(_obj(s)) or
            os.path.getmtime(_obj(s)) < max(os.path.getmtime(s), newest_hdr)]
    logs = []
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            for obj, log in ex.map(lambda s: _compile(s, verbose), todo):
                logs.append(log)
    objs = [_obj(s) for s in srcs]
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        # no library GEMMs: every dense product runs in gemm_tc.cu / gemm_gen.cu
        cmd = [NVCC] + GENCODE + ["-shared", "-o", LIB] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        for l in logs:
            if l.strip():
                print(l)
    build_cxx()
    return LIB


CXX_LIB = os.path.join(PKG, "libngram.so")
CXX_TEST = os.path.join(ROOT, "tests", "cxx", "test_dropin")  # git-ignored, travels with the snapshot


def build_cxx() -> None:
    """libngram.so: the C++ drop-in API (include/ngram/*.hpp) over the C-ABI, plus the
    C++ parity test program tests/cxx/test_dropin.cpp linked against it."""
    srcs = sorted(glob.glob(os.path.join(CSRC, "cxx", "*.cpp")))
    hdrs = glob.glob(os.path.join(ROOT, "include", "**", "*.h*"), recursive=True)
    newest = max(os.path.getmtime(f) for f in srcs + hdrs + [LIB])
    flags = ["-std=c++20", "-O2", "-fPIC", "-I" + os.path.join(ROOT, "include"), "-isystem", JSON_DIR]
    if not os.path.exists(CXX_LIB) or os.path.getmtime(CXX_LIB) < newest:
        cmd = ["g++"] + flags + ["-shared", "-o", CXX_LIB] + srcs + ["-L" + PKG, "-lngram_b200",
                                                                    "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed for libngram.so:\n{r.stderr}")
    for name in ("test_dropin", "bench_dropin"):  # C++ parity test program, per-call latency bench
        src = os.path.join(ROOT, "tests", "cxx", name + ".cpp")
        exe = os.path.join(ROOT, "tests", "cxx", name)
        if os.path.exists(src) and (not os.path.exists(exe) or os.path.getmtime(exe) <
                                    max(newest, os.path.getmtime(src), os.path.getmtime(CXX_LIB))):
            os.makedirs(os.path.dirname(exe), exist_ok=True)
            cmd = ["g++"] + flags + ["-o", exe, src, "-L" + PKG, "-lngram", "-lngram_b200",
                                     "-Wl,-rpath,$ORIGIN/../../paper_2601_21204_b200"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"g++ failed for {name}:\n{r.stderr}")


if __name__ == "__main__":
    build(clean="--clean" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
