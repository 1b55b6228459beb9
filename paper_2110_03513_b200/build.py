"""Build libcwb.so in-tree with nvcc for sm_100a (B200)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libcwb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-shared", "-Xcompiler", "-fPIC", "-ldl", "-gencode", "arch=compute_100a,code=sm_100a",
         "-lineinfo", "-O3", "-std=c++17", "--expt-relaxed-constexpr"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps() -> list[str]:
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
        os.path.join(ROOT, "include", "cwb.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compiles every csrc/*.cu to an object in parallel (objects of unchanged sources are
    reused), then links libcwb.so."""
    if force or not up_to_date():
        from concurrent.futures import ThreadPoolExecutor
        odir = os.path.join(HERE, "build")
        os.makedirs(odir, exist_ok=True)
        hdrs = [p for p in deps() if not p.endswith(".cu")]
        newest_hdr = max(os.path.getmtime(p) for p in hdrs)
        comp = [f for f in FLAGS if f not in ("-shared", "-ldl")]

        def obj(src):
            o = os.path.join(odir, os.path.basename(src)[:-3] + ".o")
            if not force and os.path.exists(o) and os.path.getmtime(o) >= max(os.path.getmtime(src), newest_hdr):
                return o
            cmd = [NVCC, *comp, "-c", "-o", o + ".tmp", src]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
            os.replace(o + ".tmp", o)
            return o

        with ThreadPoolExecutor(max_workers=len(sources())) as ex:
            objs = list(ex.map(obj, sources()))
        cmd = [NVCC, "-shared", "-ldl", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB + ".tmp", *objs]
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
