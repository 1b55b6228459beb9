"""Schedule perturbation in place of compute-sanitizer (closed on this GPU pool; profiles/r2_sanitizer_closed.log):
libcwb_jitter.so is the same sources built with -DCWB_JITTER, which delays about a quarter of the warps by a
pseudo-random 0-2 us at every phase boundary of the persistent kernels (fused CWB / ACC / HC / BERN modes, the
cross-Gram kernel) and of the streaming findBest (per item, before the fit tail).  Every kernel is deterministic
by construction (fixed summation orders, no floating-point atomics), so the perturbed run must reproduce the
normal build's outputs BIT FOR BIT; a missing barrier or a read of a value before its writer finished shows up
as a difference."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2110_03513_b200")


def _run(lib, out):
    env = dict(os.environ, CWB_LIB=os.path.join(LIBDIR, lib), PYTHONPATH=ROOT)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "det_run.py"), out], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    assert lib in p.stdout, p.stdout   # the requested library was the one loaded
    return np.load(out)


def test_jitter_build_reproduces_normal_build_bitwise(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libcwb_jitter.so")):
        from paper_2110_03513_b200 import build
        build.build()
    a = _run("libcwb.so", str(tmp_path / "a.npz"))
    b = _run("libcwb_jitter.so", str(tmp_path / "b.npz"))
    assert sorted(a.files) == sorted(b.files) and len(a.files) > 40
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    assert not bad, f"outputs that depend on the warp schedule: {bad}"
