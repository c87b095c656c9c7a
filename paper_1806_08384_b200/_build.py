"""Builds libsel.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo
snapshot to the GPU box). Host code (canon.cpp and the context/plan/probe/synopsis/graph units) and kernels (kernels.cu) link into one
shared library with a static CUDA runtime; NCCL is dlopen'd at run time."""

from __future__ import annotations

import os
import subprocess
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsel.so")
SOURCES = [os.path.join(CSRC, f) for f in ("kernels.cu", "canon.cpp", "context.cpp", "plan.cpp",
                                            "probe.cpp", "synopsis.cpp", "graph.cpp")]
HEADERS = [os.path.join(CSRC, f) for f in ("sel_internal.h", "canon.h", "host.h")] + \
          [os.path.join(ROOT, "include", "sel.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc = os.path.join(base, "include")
    lib = os.path.join(base, "lib", "libnccl.so.2")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        inc = "/usr/include"
    return inc, lib


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Build libsel.so. `out`/`defines` (-DNAME=VALUE tuning macros, e.g. SEL_GATHER_BATCH) build
    an A/B variant elsewhere; load it with SEL_LIB=<path>. The product is the default build."""
    if out == LIB and not defines and not force and not _stale():
        return LIB
    nccl_inc, nccl_lib = _nccl_dirs()
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-cudart", "static",
           "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", nccl_inc, *[f"-D{d}" for d in defines],
           f'-DSEL_NCCL_FALLBACK="{nccl_lib}"', *SOURCES, "-o", out + ".tmp", "-ldl"]
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import sys
    args = sys.argv[1:]
    defs = [a[2:] for a in args if a.startswith("-D")]
    outs = [a[6:] for a in args if a.startswith("--out=")]
    print(build(force="--force" in args, verbose="-v" in args, out=outs[0] if outs else LIB,
                defines=defs))
