"""Build the in-tree C-ABI library paper_2511_02132_b200/lib/libattnnuma.so.

    python -m paper_2511_02132_b200.build [--force] [--verbose]

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, cudart linked
statically so the .so depends only on the CUDA driver.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libattnnuma.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared", "-cudart", "static",
    "--expt-relaxed-constexpr",
]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "attn_numa.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Compile api.cu (which includes every kernel) into `out`.  `defines` are
    extra -D flags for experiment variants (the default build uses none)."""
    if not force and not defines and out == LIB and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [NVCC, *NVCC_FLAGS] + [f"-D{d}" for d in defines]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += [os.path.join(CSRC, "api.cu"), "-o", out + ".tmp"]
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--out", default=LIB)
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, defines=a.defines, out=a.out))
