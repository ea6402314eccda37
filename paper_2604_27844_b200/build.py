"""Build libzipccl_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2604_27844_b200.build

The shared library is the product's only compute path; it is git-ignored but
travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libzipccl_b200.so"
SOURCES = ["zc_abi.cu", "zc_encode.cu", "zc_decode.cu", "zc_stats.cu", "zc_p2p.cu",
           "zc_reduce.cu", "zc_coll.cu", "zc_estimate.cu",
           "zc_small.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def nccl_paths():
    """Headers + library of the NCCL torch loads (pip nvidia-nccl), so the
    collective C-ABI links against the same libnccl.so.2 soname that torch
    has already mapped; the system copy otherwise."""
    import sysconfig
    for base in (sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]):
        d = Path(base) / "nvidia" / "nccl"
        if (d / "include" / "nccl.h").exists() and (d / "lib" / "libnccl.so.2").exists():
            return str(d / "include"), str(d / "lib")
    for inc, lib in (("/usr/include", "/usr/lib/x86_64-linux-gnu"),):
        if Path(inc, "nccl.h").exists():
            return inc, lib
    raise RuntimeError("nccl.h not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh"))
    return any(p.exists() and p.stat().st_mtime > mtime for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    srcs = [str(CSRC / s) for s in SOURCES if (CSRC / s).exists()]
    inc, libdir = nccl_paths()
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
           "-I", inc, "-shared", "-o", str(LIB) + ".tmp", *srcs,
           "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}", "-lpthread"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
