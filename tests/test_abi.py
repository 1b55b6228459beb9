"""The C-ABI library loads on a CPU-only host and exports every function that
include/cwb.h declares (no compute call is made here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cwb.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*[A-Za-z_][\w\s\*]*?\b(cwb_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ["cwb_init", "cwb_bin", "cwb_bin_mat_mat", "cwb_bin_mat_vec", "cwb_find_best", "cwb_train",
              "cwb_predict", "cwb_free", "cwb_fit_host", "cwb_status", "cwb_last_error"]:
        assert f in fns


def test_library_exports_every_declared_symbol():
    from paper_2110_03513_b200 import build, cwb
    build.build()
    lib = ctypes.CDLL(cwb.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert sorted(cwb.SYMBOLS) == declared_functions()


def test_host_side_validation_without_gpu():
    # argument checks happen on the host before any device work
    from paper_2110_03513_b200 import cwb
    lib = cwb.load()
    h = ctypes.c_void_p()
    assert lib.cwb_init(ctypes.byref(h), None, 10, 0, None, None) == -5       # CWB_EEMPTY
    assert lib.cwb_init(ctypes.byref(h), None, 10, 3, None, None) == -1       # CWB_EINVAL
    assert lib.cwb_bin(None, 10, 3, None, None, None, 1, None) == -1
    assert lib.cwb_bin(ctypes.c_void_p(16), 10, 300, ctypes.c_void_p(16), None, ctypes.c_void_p(16), 1, None) == -1
    cfg = cwb.cwb_config()
    lib.cwb_default_config(ctypes.byref(cfg))
    assert (cfg.n_star_rule, cfg.degree, cfg.n_knots, cfg.df, cfg.df_kind) == (0, 3, 20, 5.0, 1)
    assert (cfg.batch_hint, cfg.unbinned, cfg.train_hint) == (0, 0, 0)
    bad = cwb.cwb_config()
    lib.cwb_default_config(ctypes.byref(bad))
    bad.train_hint = 4  # out of range: rejected on the host before any device work
    assert lib.cwb_init(ctypes.byref(h), ctypes.c_void_p(16), 10, 3, ctypes.byref(bad), None) == -1
    assert lib.cwb_version() >= 100
    assert b"empty" in lib.cwb_last_error(None) or lib.cwb_last_error(None)


def test_product_package_does_not_import_oracle():
    import ast
    pkg = os.path.join(ROOT, "paper_2110_03513_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dp, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, (ast.Import, ast.ImportFrom)):
                        names = [a.name for a in node.names] + [getattr(node, "module", "") or ""]
                        assert not any(n.startswith("oracle") for n in names), (f, names)
            if f.endswith((".cu", ".cuh", ".h")):
                assert "oracle" not in open(os.path.join(dp, f)).read().lower().replace("oracle/", ""), f


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2110_03513_b200 import cwb
    monkeypatch.setattr(cwb, "_lib", None)
    monkeypatch.setattr(cwb, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError):
        cwb.load()
