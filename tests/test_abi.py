"""The C ABI: the built library loads and exports every symbol the header
declares; the ctypes prototypes cover exactly that set.  No GPU needed."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fednl_b200.h")


def declared_symbols() -> set[str]:
    text = open(HEADER).read()
    return set(re.findall(r"^\s*(?:int|void|const char\*)\s+(fb_\w+)\s*\(", text, flags=re.M))


def test_header_declares_expected_surface():
    syms = declared_symbols()
    for must in ("fb_create", "fb_destroy", "fb_upload_shards", "fb_init_state", "fb_run_rounds",
                 "fb_compress", "fb_oracle_eval", "fb_shifted_solve", "fb_prg_u64", "fb_fp64_peak"):
        assert must in syms


def test_ctypes_prototypes_match_header():
    from paper_2410_08760_b200 import _lib

    assert set(_lib.PROTOTYPES) == declared_symbols()


def test_library_loads_and_exports_every_symbol():
    import __graft_entry__ as g

    g.build()
    lib = ctypes.CDLL(g.LIB)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_struct_layouts():
    """The ctypes mirrors have the sizes the library was compiled with."""
    import numpy as np

    from paper_2410_08760_b200 import _lib

    lib = _lib.load()
    sizes = np.zeros(3, dtype=np.int32)
    assert lib.fb_abi_sizes(_lib.ptr(sizes, ctypes.c_int32)) == 0
    assert sizes.tolist() == [ctypes.sizeof(_lib.FbConfig), ctypes.sizeof(_lib.FbStatus),
                              ctypes.sizeof(_lib.FbProfile)]
    # fb_config: 10 int32 + 4 double + u64 + 61 double + mu + topk_path + reserved
    assert ctypes.sizeof(_lib.FbConfig) == 10 * 4 + 4 * 8 + 8 + 61 * 8 + 8 + 2 * 4


def test_no_cpu_fallback_when_library_missing(monkeypatch):
    from paper_2410_08760_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libfednl_b200.so")
    with pytest.raises(_lib.LibraryMissing):
        _lib.load()


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2410_08760_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "fednl_oracle" not in src and "from oracle" not in src, f
