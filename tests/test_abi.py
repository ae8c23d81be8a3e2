"""Host-side checks of the C ABI that need no GPU: the library loads, exports every symbol
include/fgf.h declares, and validates arguments before touching the device."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

from tests.conftest import ROOT

import paper_1505_00996_b200 as fgf


def header_functions():
    txt = open(os.path.join(ROOT, "include", "fgf.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fgf_[a-z_]+)\s*\(", txt)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(fgf.LIB_PATH)
    names = header_functions()
    assert len(names) >= 9
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(fgf.EXPORTS)


def test_status_strings():
    assert fgf.fgf_status_str(0) == "ok"
    for s in range(1, 11):
        assert fgf.fgf_status_str(s) != "unknown status"
    assert "sm_100a" in fgf.fgf_version()


def test_library_is_sm100a_only():
    # the fat binary carries sm_100a SASS only (no PTX, no other arch)
    out = os.popen(f"cuobjdump --list-elf {fgf.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90", "sm_89"):
        assert other + "." not in out


BAD = 0x1000  # a fake, 16-byte aligned address; validation must fail before it is used


@pytest.mark.parametrize("args,code", [
    ((1, 64, 64, 1, 1, 0, 0.01, 4, 0), fgf.FGF_ERR_PARAM),     # r < 1
    ((1, 64, 64, 1, 1, 8, 0.0, 4, 0), fgf.FGF_ERR_PARAM),      # eps <= 0
    ((1, 64, 64, 1, 1, 8, float("nan"), 4, 0), fgf.FGF_ERR_PARAM),
    ((1, 64, 64, 1, 1, 8, float("inf"), 4, 0), fgf.FGF_ERR_PARAM),
    ((1, 64, 64, 1, 1, 8, 0.01, 0, 0), fgf.FGF_ERR_PARAM),     # s < 1
    ((1, 64, 64, 1, 1, 8, 0.01, 4, 2), fgf.FGF_ERR_PARAM),     # sub_mode
    ((1, 64, 4, 1, 1, 8, 0.01, 4, 0), fgf.FGF_ERR_PARAM),      # s >= min(H, W)
    ((0, 64, 64, 1, 1, 8, 0.01, 4, 0), fgf.FGF_ERR_SHAPE),
    ((1, 0, 64, 1, 1, 8, 0.01, 4, 0), fgf.FGF_ERR_SHAPE),
    ((1, 64, 64, 2, 1, 8, 0.01, 4, 0), fgf.FGF_ERR_SHAPE),     # C_I not in {1,3}
    ((1, 64, 64, 1, 5, 8, 0.01, 4, 0), fgf.FGF_ERR_SHAPE),     # C_p > 4
    ((1, 64, 64, 1, 0, 8, 0.01, 4, 0), fgf.FGF_ERR_SHAPE),
    ((1, 65536, 32768, 1, 1, 8, 0.01, 4, 0), fgf.FGF_ERR_UNSUPPORTED),  # 2^31 in-image elements
])
def test_validation_before_launch(args, code):
    a = 0x100000
    assert fgf.fgf_filter(a, a + 0x10000000, a + 0x20000000, *args, check=False) == code
    assert fgf.fgf_filter_ws(a, a + 0x10000000, a + 0x20000000, *args, BAD, 1 << 30, None,
                             check=False) == code
    assert fgf.fgf_filter_ex_ws(a, a + 0x10000000, a + 0x20000000, *args, fgf.FGF_F16, BAD,
                                1 << 30, None, check=False) == code


def test_extended_entry_point_validation():
    a = 0x100000
    geo = (1, 64, 64, 1, 1, 8, 0.01, 4, 0)
    # unknown element type; 16-bit types are not offered for C_I / C_p = 1 / 2
    assert fgf.fgf_filter_ex_ws(a, a + 0x100000, a + 0x200000, *geo, 7, BAD, 1 << 30, None,
                                check=False) == fgf.FGF_ERR_PARAM
    assert fgf.fgf_filter_ex_ws(a, a + 0x100000, a + 0x200000, 1, 64, 64, 1, 2, 8, 0.01, 4, 0,
                                fgf.FGF_F16, BAD, 1 << 30, None,
                                check=False) == fgf.FGF_ERR_UNSUPPORTED
    assert fgf.fgf_workspace_bytes_ex(1, 64, 64, 1, 1, 8, 4, 9) == 0
    assert fgf.fgf_workspace_bytes_ex(1, 64, 64, 1, 1, 8, 4, fgf.FGF_F16) > 0
    # enhancement: negative gain; band path: bad exchange mode, thin band, bad rank
    assert fgf.fgf_enhance_ws(a, a + 0x100000, 1, 64, 64, 1, 8, 0.01, 4, 0, -1.0, BAD, 1 << 30,
                              None, check=False) == fgf.FGF_ERR_PARAM
    assert fgf.fgf_filter_band_ex(a, a, a + 0x100000, 1024, 64, 0, 64, 1, 1, 8, 0.01, 4, 0, 5,
                                  None, 0, 1, BAD, 1 << 30, None,
                                  check=False) == fgf.FGF_ERR_PARAM
    assert fgf.fgf_filter_band(a, a, a + 0x100000, 1024, 64, 0, 64, 1, 1, 32, 0.01, 4, 0,
                               None, 0, 4, BAD, 1 << 30, None, check=False) == fgf.FGF_ERR_PARAM
    assert fgf.fgf_filter_band(a, a, a + 0x100000, 1024, 64, 0, 64, 1, 1, 8, 0.01, 4, 0,
                               None, 4, 4, BAD, 1 << 30, None, check=False) == fgf.FGF_ERR_PARAM
    assert fgf.fgf_band_workspace_bytes(1024, 64, 0, 256, 1, 1, 8, 4, 4) > 0


def test_pointer_errors():
    geo = (1, 64, 64, 1, 1, 8, 0.01, 4, 0)
    a = 0x100000
    assert fgf.fgf_filter(None, a, a + 0x100000, *geo, check=False) == fgf.FGF_ERR_NULL
    assert fgf.fgf_filter(a + 2, a + 0x100000, a + 0x200000, *geo, check=False) == fgf.FGF_ERR_ALIGN
    # q overlapping I or p
    assert fgf.fgf_filter(a, a + 0x100000, a + 0x100, *geo, check=False) == fgf.FGF_ERR_ALIAS
    assert fgf.fgf_filter(a, a + 0x100000, a + 0x100000 + 64, *geo, check=False) == fgf.FGF_ERR_ALIAS
    # s = 1 on a 1-pixel-high image is valid (R7): fails only at the pointer check
    rc = fgf.fgf_filter(a, a + 0x100000, a + 0x200000, 1, 1, 64, 1, 1, 2, 0.01, 1, 0, check=False)
    assert rc == fgf.FGF_ERR_DEVICE


def test_host_pointers_rejected_by_device_entry():
    import numpy as np
    I = np.zeros((64, 64), np.float32)
    p = np.zeros((64, 64), np.float32)
    q = np.zeros((64, 64), np.float32)
    rc = fgf.fgf_filter(I, p, q, 1, 64, 64, 1, 1, 8, 0.01, 4, 0, check=False)
    assert rc == fgf.FGF_ERR_DEVICE


def test_workspace_bytes():
    assert fgf.fgf_workspace_bytes(1, 64, 64, 1, 1, 8, 0) == 0
    small = fgf.fgf_workspace_bytes(1, 256, 256, 1, 1, 8, 4)
    assert small > 0 and small % 256 == 0
    # chunking keeps the workspace bounded for a large batch (L2-resident chunk)
    big = fgf.fgf_workspace_bytes(256, 4096, 4096, 1, 1, 32, 4)
    assert 0 < big <= 8 << 30
    # unsupported strip geometry (r' > 240 with w > 512)
    assert fgf.fgf_workspace_bytes(1, 2048, 2048, 1, 1, 300, 1) == 0
    assert fgf.fgf_workspace_bytes(1, 512, 512, 1, 1, 300, 1) > 0


def header_arities():
    """{name: number of parameters} for every prototype in include/fgf.h."""
    txt = open(os.path.join(ROOT, "include", "fgf.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(fgf_[a-z_]+)\s*\(([^)]*)\)\s*;", txt):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    return out


def test_binding_argtypes_match_header():
    lib = fgf._lib
    for name, n in header_arities().items():
        assert len(getattr(lib, name).argtypes) == n, name
