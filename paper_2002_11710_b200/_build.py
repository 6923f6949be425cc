"""Build the sm_100a C-ABI library in-tree (libairsched.so) with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libairsched.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(PKG, "csrc", "*.h")) + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + \
        [os.path.join(ROOT, "include", "airsched.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def nccl_dir() -> str:
    """torch's bundled NCCL (one NCCL per process: the same library torch loads)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("torch-bundled NCCL (nvidia/nccl) not found")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    nd = nccl_dir()
    cmd = [nvcc, ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O2",
           "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(nd, "include"), "-o", LIB + ".tmp"] + sources() + \
          ["-L" + os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
