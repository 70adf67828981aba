"""In-tree build of the CUDA library (sm_100a) with plain nvcc.

The shared object lands next to this file (``libpatfft_b200.so``) so it
travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpatfft_b200.so")
SOURCES = ["capi.cu", "spread.cu", "spread_tc.cu", "lateral.cu", "ner.cu", "ner_api.cu", "reflen.cu", "util.cu", "window.cpp", "hoststage.cpp"]
HEADERS = ["patfft_internal.h", "fft_smem.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-Xptxas", "-O3"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "patfft_b200.h"),
                                                                  __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra: list[str] | None = None) -> str:
    """Compile every source to an object in parallel, then link the .so.

    ``out``/``extra`` build an experimental variant (e.g. ``-DPATFFT_SPREAD_MINB=3``)
    next to the default library; the default path and flags are what the
    package loads.
    """
    lib = out or LIB
    extra = list(extra or []) + os.environ.get("PATFFT_NVCC_FLAGS", "").split()
    if not force and not extra and out is None and not _stale():
        return lib
    import concurrent.futures as cf
    import hashlib

    tag = hashlib.sha1(" ".join(extra).encode()).hexdigest()[:8]
    objdir = os.path.join(HERE, "_obj", tag)
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", "-o", obj, os.path.join(CSRC, src), "-I", os.path.join(ROOT, "include")]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [NVCC, *ARCH, "-shared", "-o", lib + ".tmp", *objs, "-lcufft", "-lpthread", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    import sys

    args = sys.argv[1:]
    out = None
    if "--out" in args:
        out = args[args.index("--out") + 1]
    extra = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose=True, out=out, extra=extra))
