"""The C-ABI library: builds for sm_100a, loads, and exports exactly what
include/ivhd_b200.h declares.  No compute calls (CPU container)."""

import ctypes
import os
import re

import pytest

from paper_2303_05455_b200 import _lib
from paper_2303_05455_b200.errors import DeviceError

from .conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ivhd_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ivhd_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2303_05455_b200 import build

        build.build()
    return _lib.load()


def test_header_and_binding_agree():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    from paper_2303_05455_b200._lib import ABI_VERSION
    assert lib.ivhd_abi_version() == ABI_VERSION
    assert f"#define IVHD_ABI_VERSION {ABI_VERSION}" in open(HEADER).read()


def test_library_is_sm100a():
    from paper_2303_05455_b200 import build

    assert "arch=compute_100a,code=sm_100a" in " ".join(build.FLAGS)


def test_create_without_device_fails_loudly(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    code = lib.ivhd_create(ctypes.byref(h), 0, 100, 2, 0)
    assert code == _lib.ERR_CUDA
    assert b"CUDA" in lib.ivhd_global_error() or b"device" in lib.ivhd_global_error()


def test_invalid_arguments_are_rejected_before_cuda(lib):
    h = ctypes.c_void_p()
    assert lib.ivhd_create(ctypes.byref(h), 0, 0, 2, 0) == _lib.ERR_INVALID_ARG
    assert lib.ivhd_create(ctypes.byref(h), 0, 10, 4, 0) == _lib.ERR_INVALID_ARG


def test_product_path_has_no_cpu_fallback(monkeypatch):
    """With the library missing, the public API raises instead of computing."""
    import paper_2303_05455_b200 as P

    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libivhd_b200.so")
    monkeypatch.setattr(_lib, "_lib", None)
    graph = P.KnnGraph([[1], [2], [0], [0]])
    with pytest.raises(DeviceError):
        P.run_embedding(graph=graph, config=P.EmbeddingConfig(nn=1, rn=1, iterations=3))
