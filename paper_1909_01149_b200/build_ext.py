"""Build libnncp_b200.so in-tree with nvcc for sm_100a (no torch JIT cache).

    python -m paper_1909_01149_b200.build_ext
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libnncp_b200.so")
BUILD = os.path.join(HERE, "csrc", "build")
SOURCES = ["abi.cu", "mttkrp_gemm.cu", "mttkrp_sliced.cu", "ttv.cu", "nnls.cu", "nnls_iter.cu", "synth.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _compile(src: str, extra=(), tag: str = "") -> tuple[str, str]:
    obj = os.path.join(BUILD, src.replace(".cu", tag + ".o"))
    cmd = [nvcc(), *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    return obj, res.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    if os.path.exists(OUT):
        os.remove(OUT)  # a failed build must not leave a stale library behind
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    cmd = [nvcc(), *ARCH, "-shared", "-o", OUT, *objs, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    return OUT


def build_variant(name: str, defines) -> str:
    """A tools-only variant of the library (loaded through NNCP_LIB_PATH), e.g. with extra -D flags."""
    out = os.path.join(HERE, f"libnncp_b200_{name}.so")
    os.makedirs(BUILD, exist_ok=True)
    extra = tuple(f"-D{d}" for d in defines)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = [o for o, _ in ex.map(lambda s: _compile(s, extra, "_" + name), SOURCES)]
    res = subprocess.run([nvcc(), *ARCH, "-shared", "-o", out, *objs, "-lcudart"], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    return out


def build_stats() -> str:
    """Instrumented variant (barrier wait counters in the sliced GEMM) for tools/sliced_stats.py."""
    return build_variant("stats", ["NNCP_SLICED_STATS"])


if __name__ == "__main__":
    if "--stats" in sys.argv:
        print(build_stats())
    elif "--variant" in sys.argv:   # --variant NAME DEFINE [DEFINE ...]
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        print(build(verbose="-v" in sys.argv))
