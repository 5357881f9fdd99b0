"""Build libsmconv.so in-tree for sm_100a (nvcc -gencode arch=compute_100a,code=sm_100a).

The .so lands next to this file so gpurun snapshots carry it to the GPU box.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libsmconv.so")
STAMP = LIB + ".srchash"

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _hash():
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(INCLUDE, "*.h"))):
        with open(f, "rb") as fh:
            h.update(f.encode())
            h.update(fh.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu into one shared library (skipped when sources are unchanged)."""
    h = _hash()
    if not force and os.path.exists(LIB) and os.path.exists(STAMP) and open(STAMP).read() == h:
        return LIB
    tmp = LIB + ".tmp%d" % os.getpid()
    # one object per source, compiled in parallel, then one link (the single-command build was ~90 s)
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build", "obj%d" % os.getpid())
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]

    def one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc()] + cflags + ["-I" + INCLUDE, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd, cwd=CSRC)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(one, _sources()))
    subprocess.check_call([nvcc()] + NVCC_FLAGS + objs + ["-o", tmp], cwd=CSRC)
    for o in objs:
        os.remove(o)
    os.rmdir(objdir)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(h)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
