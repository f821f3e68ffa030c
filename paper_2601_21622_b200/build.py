"""Build libstarsd.so in-tree with nvcc for sm_100a (no JIT cache; the .so ships with the repo
snapshot to the GPU box)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libstarsd.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nccl_paths():
    """The pip NCCL that torch loads (2.28.x), not the system copy."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        return None, None
    base = list(spec.submodule_search_locations)[0]
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return None, None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps.append(os.path.join(ROOT, "include", "starsd.h"))
    return max(os.path.getmtime(d) for d in deps) > os.path.getmtime(LIB)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    inc, libdir = nccl_paths()
    cmd = ["nvcc", ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(ROOT, "include")]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    if os.environ.get("STARSD_BUILD_DEBUG"):
        cmd += ["-DSD_STREAM_DEBUG=1"]
    if inc:
        cmd += ["-DSD_WITH_NCCL=1", "-I", inc]
    tmp = LIB + f".tmp{os.getpid()}"
    cmd += ["-o", tmp] + sources()
    if libdir:
        cmd += ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
