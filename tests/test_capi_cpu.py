"""CPU-side checks of the C-ABI boundary: libmgpbd.so builds for sm_100a, loads, exports every symbol
include/mgpbd.h declares, and its host-only entry points validate arguments (no GPU compute)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2505_13390_b200 import build
    return build.build()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "mgpbd.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(mgpbd_[a-z_0-9]+)\s*\(", hdr)))


def test_header_symbols_exported(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mgpbd_\w+)", out))
    decl = declared_symbols()
    assert len(decl) >= 19
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    # nothing but the C-ABI is exported (C++ internals hidden)
    assert all(s.startswith("mgpbd_") for s in exported)


def test_binding_names_match_header():
    from paper_2505_13390_b200 import mgpbd
    assert sorted(mgpbd.SYMBOLS) == declared_symbols()


def test_sm100a_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_config_default_and_create_validation(libpath):
    from paper_2505_13390_b200 import mgpbd
    cfg = mgpbd.config_default()
    assert cfg.theta == 0.1 and cfg.min_coarse == 400 and cfg.pcg_iters == 10 and cfg.smoother_sweeps == 2
    assert cfg.setup_interval == 20 and cfg.bootstrap_sweeps == 20 and cfg.power_iters == 100
    assert abs(cfg.lambda_min_est - 0.1) < 1e-15 and list(cfg.gravity) == [0.0, -9.8, 0.0]
    L = mgpbd.lib()
    # argument errors are detected on the host before any device work
    X = np.zeros((2, 3)); X[1, 0] = 1
    bad = np.array([[0, 5]], np.int32)
    with pytest.raises(mgpbd.MgpbdError) as e:
        mgpbd.Context(2, bad, X, np.ones(2), np.ones(1))
    assert e.value.status == mgpbd.E_ARG and "out of range" in str(e.value)
    with pytest.raises(mgpbd.MgpbdError):
        mgpbd.Context(2, np.array([[1, 1]], np.int32), X, np.ones(2), np.ones(1))
    with pytest.raises(mgpbd.MgpbdError):
        mgpbd.Context(2, np.array([[0, 1]], np.int32), X, -np.ones(2), np.ones(1))
    with pytest.raises(mgpbd.MgpbdError):                           # negative compliance
        mgpbd.Context(2, np.array([[0, 1]], np.int32), X, np.ones(2), -np.ones(1))
    with pytest.raises(mgpbd.MgpbdError):                           # empty constraint set
        mgpbd.Context(2, np.zeros((0, 2), np.int32), X, np.ones(2), np.ones(0))
    for kw in (dict(smoother=3), dict(level0_operator=2), dict(pcg_tol=-1.0), dict(pcg_iters=5000),
               dict(k_nullspace=9), dict(k_nullspace=0), dict(precision=2), dict(smoother_sweeps=0)):
        with pytest.raises(mgpbd.MgpbdError) as e:
            mgpbd.Context(2, np.array([[0, 1]], np.int32), X, np.ones(2), np.ones(1), **kw)
        assert e.value.status == mgpbd.E_ARG, kw                     # host validation, no device work
    out = C.c_void_p()
    assert L.mgpbd_create(None, None, None, None, None, C.byref(out)) == mgpbd.E_ARG


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2505_13390_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|\borc_\w+\(|oracle\.h)", src), f
