"""Build libzk.so (sm_100a) in-tree with nvcc.  No torch in the build: the library is a plain
C-ABI shared object (include/zk.h) linked against the static CUDA runtime and NCCL."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libzk.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("NCCL (nvidia.nccl) not found")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h")) + [__file__]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in deps())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile csrc/*.cu into libzk.so (or `out` with extra -D defines, for A/B variants)."""
    so = out or SO
    if not force and out is None and not stale():
        return SO
    inc, lib = nccl_dirs()
    objdir = os.path.join(PKG, "build", "obj_" + os.path.basename(so).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    flags = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-I", inc,
                    "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]
    if verbose:
        flags += ["-Xptxas", "-v"]
    flags += [f"-D{d}" for d in defines]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen(["nvcc", "-c", src, "-o", obj] + flags))
    rc = [p.wait() for p in procs]
    if any(rc):
        raise RuntimeError(f"nvcc failed: {rc}")
    link = ["nvcc", "-shared", "-o", so] + objs + ARCH + [
        "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}"]
    subprocess.check_call(link)
    return so


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out")
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=a.out, defines=a.D))
