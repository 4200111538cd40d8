"""The C-ABI library builds, loads and exports every symbol include/semflow_b200.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2207_07098_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "semflow_b200.h")).read()
    return sorted(set(re.findall(r"\b(sf_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2207_07098_b200 import build

    build.build()
    return _lib.load()


def test_header_and_binding_agree():
    assert set(header_symbols()) == set(_lib.EXPORTED)


def test_library_exports_every_header_symbol(lib):
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.sf_version()
    assert lib.sf_red_workspace_doubles() > 0


def test_library_targets_sm100a():
    path = _lib.LIB_PATH
    data = open(path, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_error_path_without_gpu(lib):
    # an argument error is reported through the status code and sf_last_error,
    # before any device work is attempted
    st = lib.sf_dssum_f64(None, None, None, 5, 7, None, None, 0, None)
    assert st == 1
    assert b"bad mode" in lib.sf_last_error()
    st = lib.sf_ax_helm_f64((ctypes.c_double * 1)(), 13, None, None, None, None, 4, 1.0, 0.0, 0, None)
    assert st == 3
