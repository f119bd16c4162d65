"""In-tree build of libnlse2shoc.so (nvcc, sm_100a) — used by __graft_entry__.build().

The library links the NCCL that ships with the torch wheel (nvidia/nccl/lib) so that one
process never holds two NCCLs.  CUDA runtime is linked statically.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libnlse2shoc.so")
SO_CHECKED = os.path.join(HERE, "libnlse2shoc_checked.so")  # -DNLSE_CHECKED: range-checked stores
SRC = os.path.join(HERE, "csrc", "nlse2shoc.cu")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir():
    for p in sys.path:
        d = os.path.join(p, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    return None


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*"))) + [os.path.join(ROOT, "include", "nlse2shoc.h")]


def needs_build():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libnlse2shoc.so (or `out`, with extra -D `defines`, for experiments)."""
    target = out or SO
    if not force and out is None and not needs_build():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(ROOT, "include")]
    nd = nccl_dir()
    if nd:
        cmd += ["-I", os.path.join(nd, "include"), "-DNLSE_WITH_NCCL"]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += [f"-D{d}" for d in defines]
    cmd += ["-o", target + ".tmp", SRC]
    if nd:
        cmd += ["-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nd, "lib")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    os.replace(target + ".tmp", target)
    if verbose:
        sys.stdout.write(r.stdout + r.stderr)
    return target


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(SO)
