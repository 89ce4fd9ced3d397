"""The C-ABI library loads on a CPU host and exports exactly the entry points declared in
include/scvt_b200.h (no compute calls: there is no GPU here)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "scvt_b200.h")
LIB = os.path.join(ROOT, "paper_1709_06924_b200", "libscvtb200.so")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(scvt_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__

        __graft_entry__.build()
    from paper_1709_06924_b200 import _lib

    return _lib.load()


def test_header_declares_the_abi():
    names = _declared()
    for must in ("scvt_create", "scvt_destroy", "scvt_evaluate", "scvt_triangulate",
                 "scvt_lbfgs_direction", "scvt_history_push", "scvt_last_error"):
        assert must in names


def test_exports_match_header(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines() if " T scvt_" in ln})
    assert exported == _declared()


def test_python_binding_covers_every_symbol(lib):
    from paper_1709_06924_b200 import _lib

    assert sorted(_lib.SIGNATURES) == _declared()


def test_version_string(lib):
    assert b"sm_100a" in lib.scvt_version()


def test_config_validation_without_gpu(lib):
    """Invalid configurations are rejected before any device work (SCVT_ERR_CONFIG = 9)."""
    import numpy as np

    from paper_1709_06924_b200 import _lib, density

    l1 = np.array([1 / 3]); l2 = np.array([1 / 3]); w = np.array([1.0])
    cfg, keep = _lib.make_config(density.device_params(density.density_preset("const")), "flat",
                                 l1, l2, w, 7)
    ctx = ctypes.c_void_p()
    assert lib.scvt_create(ctypes.byref(ctx), 0, 2, ctypes.byref(cfg)) == 9     # n_max < 4
    assert b"n_max" in lib.scvt_last_error(ctx)
    lib.scvt_destroy(ctx)
    cfg.lbfgs_m = 0
    ctx = ctypes.c_void_p()
    assert lib.scvt_create(ctypes.byref(ctx), 0, 100, ctypes.byref(cfg)) == 9
    lib.scvt_destroy(ctx)
    cfg.lbfgs_m = 7
    cfg.density_kind = 42
    ctx = ctypes.c_void_p()
    assert lib.scvt_create(ctypes.byref(ctx), 0, 100, ctypes.byref(cfg)) == 9
    lib.scvt_destroy(ctx)
    del keep


def test_status_codes_map_to_reference_exceptions():
    from paper_1709_06924_b200 import errors

    text = open(HEADER).read()
    codes = dict((name, int(v)) for name, v in re.findall(r"(SCVT_ERR_\w+)\s*=\s*(\d+)", text))
    assert errors.STATUS_ERRORS[codes["SCVT_ERR_INSUFFICIENT_POINTS"]] is errors.InsufficientPointsError
    assert errors.STATUS_ERRORS[codes["SCVT_ERR_COVERAGE"]] is errors.CoverageError
    assert errors.STATUS_ERRORS[codes["SCVT_ERR_CENTROID_AT_ORIGIN"]] is errors.CentroidAtOriginError
    assert errors.STATUS_ERRORS[codes["SCVT_ERR_NONPOSITIVE_DIAGONAL"]] is errors.NonpositiveDiagonalError
    assert errors.STATUS_ERRORS[codes["SCVT_ERR_POLE_AMBIGUITY"]] is errors.PoleAmbiguityError


def test_row_width_matches_header():
    """The host's neighbour-row width (Laplacian rows) is the header's SCVT_MAX_DEGREE."""
    from paper_1709_06924_b200 import _lib

    m = re.search(r"#define\s+SCVT_MAX_DEGREE\s+(\d+)", open(HEADER).read())
    assert m and int(m.group(1)) == _lib.MAX_DEGREE


def test_no_cpu_fallback_without_gpu():
    """The product path refuses to run without CUDA instead of computing on the host."""
    import torch

    import paper_1709_06924_b200 as P

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with P.MeshEvaluator(P.density_preset("const"), "4pt") as ev, pytest.raises(P.DeviceError):
        ev.evaluate(P.random_sphere_points(100, 0))
