"""The C-ABI library loads without a GPU and exports every symbol the public
header declares; workspace sizing is pure host arithmetic."""

import ctypes
import os
import re

import pytest

from paper_2010_06654_b200 import _native as nat

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "lloydkit_b200.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(lk_\w+)\s*\(", src, re.M)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(nat.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = nat.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.lk_version() >= 1


def test_workspace_sizing_without_gpu():
    lib = nat.load()
    cfg = nat.LkConfig(n_local=1000, n_total=1000, d=16, k=10, strategy=1, groups=0, t_max=5,
                       kernel=0, has_x64=0, device=0)
    b = ctypes.c_uint64()
    assert lib.lk_workspace_bytes(ctypes.byref(cfg), ctypes.byref(b)) == nat.LK_OK
    # X32 alone is 64 KB; bounds and worklists add more
    assert b.value > 1000 * 16 * 4
    bad = nat.LkConfig(n_local=-1, n_total=0, d=0, k=0, strategy=0, groups=0, t_max=1,
                       kernel=0, has_x64=0, device=0)
    assert lib.lk_workspace_bytes(ctypes.byref(bad), ctypes.byref(b)) == nat.LK_ERR_ARG
    assert "invalid" in lib.lk_last_error().decode()


def test_cfg5_fits_one_b200():
    lib = nat.load()
    cfg = nat.LkConfig(n_local=50_000_000, n_total=50_000_000, d=32, k=4096, strategy=1,
                       groups=0, t_max=20, kernel=0, has_x64=0, device=0)
    b = ctypes.c_uint64()
    assert lib.lk_workspace_bytes(ctypes.byref(cfg), ctypes.byref(b)) == nat.LK_OK
    assert b.value < 40 * 2**30
