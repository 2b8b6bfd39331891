"""Build libspecbranch.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2506_01979_b200.build [--verbose]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libspecbranch.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    """NCCL shipped with the venv's torch (nvidia/nccl: nccl.h + libnccl.so.2)."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers not found (expected site-packages/nvidia/nccl)")


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(HERE, "csrc", "*.h")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [
        os.path.join(ROOT, "include", "specbranch.h")]


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(f) <= t for f in deps())


def nvcc_cmd(verbose: bool = False):
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    nccl = nccl_dir()
    cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
           "-o", SO + ".tmp", *sources(), "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    return cmd


def build(force: bool = False, verbose: bool = False, extra=(), out: str = SO) -> str:
    """Compile libspecbranch.so (``extra`` nvcc flags and ``out`` only for A/B experiment
    builds, loaded through SB_LIB_PATH)."""
    if out == SO and not extra and not force and up_to_date():
        return SO
    import fcntl

    # several ranks of one torchrun job may get here at once: one builds, the others
    # wait on the lock and then find the library up to date
    with open(out + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if out == SO and not extra and not force and up_to_date():
            return SO
        tmp = f"{out}.{os.getpid()}.tmp"
        cmd = nvcc_cmd(verbose)
        cmd[cmd.index(SO + ".tmp")] = tmp
        cmd[1:1] = list(extra)
        subprocess.check_call(cmd)
        os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python -m paper_2506_01979_b200.build [--verbose] [--out PATH] [-- nvcc flags...]
    args = sys.argv[1:]
    extra = args[args.index("--") + 1:] if "--" in args else []
    out = args[args.index("--out") + 1] if "--out" in args else SO
    print(build(force=True, verbose="--verbose" in args, extra=extra, out=out))
