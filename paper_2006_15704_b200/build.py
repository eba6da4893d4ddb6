"""In-tree build of the native libraries (sm_100a only).

    python -m paper_2006_15704_b200.build          # builds lib/libb200ddp.so

The shared library is linked against the SAME libnccl.so.2 that torch loads
(pip ``nvidia-nccl``, 2.28.x) via an rpath, and against the static CUDA
runtime.  Objects are compiled in parallel; a rebuild happens only when a
source or header is newer than the library.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(LIBDIR, "libb200ddp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    import nvidia.nccl  # the pip wheel torch itself loads
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True) +
                  glob.glob(os.path.join(CSRC, "**", "*.cpp"), recursive=True))


def _headers():
    return (glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True) +
            glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True) +
            glob.glob(os.path.join(ROOT, "include", "*.h")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    nccl_inc, nccl_lib = nccl_paths()
    srcs = _sources()
    deps = srcs + _headers() + [os.path.abspath(__file__)]
    if not force and not _stale(LIB, deps):
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(BUILD, exist_ok=True)
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                     "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_inc]

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.relpath(src, CSRC).replace(os.sep, "_") + ".o")
        cmd = [NVCC] + common + ["-Xptxas", "-v"] * (src.endswith(".cu") and verbose) + ["-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, "-x", "cu"] + cmd[1:]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    link = [NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + [
        "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nccl_lib}", "-cudart", "static"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


SYNTH_SRC = os.path.join(ROOT, "synth", "csrc", "synth.cu")
SYNTH_LIB = os.path.join(ROOT, "synth", "lib", "libb200synth.so")


def build_synth(force: bool = False) -> str:
    """Test/bench input generator (synth/csrc/synth.cu); not part of the product."""
    if not force and not _stale(SYNTH_LIB, [SYNTH_SRC, os.path.abspath(__file__)]):
        return SYNTH_LIB
    os.makedirs(os.path.dirname(SYNTH_LIB), exist_ok=True)
    cmd = [NVCC] + ARCH + ["-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
                           SYNTH_SRC, "-o", SYNTH_LIB + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {SYNTH_SRC}:\n{r.stdout}\n{r.stderr}")
    os.replace(SYNTH_LIB + ".tmp", SYNTH_LIB)
    return SYNTH_LIB


def build_all(verbose: bool = False, force: bool = False):
    return build(verbose, force), build_synth(force)


if __name__ == "__main__":
    print(build_all(verbose="-v" in sys.argv, force="-f" in sys.argv))
