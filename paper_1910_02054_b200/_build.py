"""Build the in-tree shared libraries for sm_100a with nvcc (no JIT cache).

  paper_1910_02054_b200/libzero_b200.so   the C-ABI library (include/zero_b200.h)
  synth/libzero_synth.so                  the GPU side of the seeded input generator

Both are built IN-TREE so that they travel with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libzero_b200.so")
SYNTH_SRC = os.path.join(ROOT, "synth", "synth_fill.cu")
SYNTH_LIB = os.path.join(ROOT, "synth", "libzero_synth.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]


def nccl_root() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        cand = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    raise RuntimeError("NCCL headers (nvidia/nccl) not found next to torch")


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def _stale(out: str, srcs) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False) -> list:
    built = []
    nccl = nccl_root()
    srcs = [os.path.join(CSRC, "kernels.cu"), os.path.join(CSRC, "engine.cpp"), os.path.join(CSRC, "activation.cu")]
    deps = srcs + [os.path.join(CSRC, "zero_internal.h"), os.path.join(ROOT, "include", "zero_b200.h")]
    if force or _stale(LIB, deps):
        cmd = [_nvcc()] + COMMON + ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
                                    "-Xptxas", "-v"] + srcs + [
            "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + os.path.join(nccl, "lib"), "-o", LIB]
        _run(cmd, verbose)
        built.append(LIB)
    if force or _stale(SYNTH_LIB, [SYNTH_SRC]):
        _run([_nvcc()] + COMMON + [SYNTH_SRC, "-o", SYNTH_LIB], verbose)
        built.append(SYNTH_LIB)
    return built


def _run(cmd, verbose):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode})")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
