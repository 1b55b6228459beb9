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


LIB_JITTER = os.path.join(HERE, "libcwb_jitter.so")
JITTER_SEED = 0x5EED


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(p) <= t for p in deps())


def _build(lib: str, odir: str, extra: list[str], force: bool, verbose: bool) -> str:
    """Compiles every csrc/*.cu to an object in parallel (objects of unchanged sources are reused), then
    links `lib`."""
    if force or not up_to_date(lib):
        from concurrent.futures import ThreadPoolExecutor
        os.makedirs(odir, exist_ok=True)
        hdrs = [p for p in deps() if not p.endswith(".cu")]
        newest_hdr = max(os.path.getmtime(p) for p in hdrs)
        comp = [f for f in FLAGS if f not in ("-shared", "-ldl")] + extra

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
        cmd = [NVCC, "-shared", "-ldl", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib + ".tmp", *objs]
        subprocess.run(cmd, check=True)
        os.replace(lib + ".tmp", lib)
    return lib


def build(force: bool = False, verbose: bool = False, jitter: bool = True) -> str:
    """libcwb.so, and (jitter=True) libcwb_jitter.so: the same sources with -DCWB_JITTER, the schedule-
    perturbation build of tests/test_gpu_jitter.py (race hunting; compute-sanitizer is closed on the pool)."""
    from concurrent.futures import ThreadPoolExecutor
    jobs = [(LIB, os.path.join(HERE, "build"), [])]
    if jitter:
        jobs.append((LIB_JITTER, os.path.join(HERE, "build", "jitter"), [f"-DCWB_JITTER={JITTER_SEED}"]))
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        list(ex.map(lambda j: _build(j[0], j[1], j[2], force, verbose), jobs))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
