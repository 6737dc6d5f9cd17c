"""CPU: the C-ABI library loads without a GPU and exports every entry point
declared in include/*.h; host-side logic that needs no device."""
import ctypes
import os
import re

import pytest

from paper_2005_10445_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    syms = set()
    for h in ("tagdsp_gpu.h",):
        src = open(os.path.join(ROOT, "include", h)).read()
        syms |= set(re.findall(r"\b(tdg_[a-z0-9_]+)\s*\(", src))
    return syms


def test_library_loads_and_exports_all_declared_symbols():
    L = ctypes.CDLL(capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in sorted(syms) if not hasattr(L, s)]
    assert not missing, missing
    assert set(capi.EXPORTED_SYMBOLS) <= syms


def test_pad_length_matches_reference_rule():
    assert capi.pad_length(1) == 1 and capi.pad_length(1000) == 1000 and capi.pad_length(101) == 105
    assert capi.pad_length(865743) == 870912
    with pytest.raises(capi.InvalidArgument):
        capi.pad_length(0)


def test_corr_len_choice_is_linear_and_supported():
    # any N >= W + n - 1 keeps lags [0, W) free of circular wrap
    for W, n in [(800000, 65741), (96000, 65741), (4096, 64), (2048, 100), (100000, 65741)]:
        N = capi.corr_len(W, n)
        assert N >= W + n - 1, (W, n, N)
    assert capi.corr_len(800000, 65741) == 884736       # 1024 x 864
    assert capi.corr_len(1 << 30, 10) == 0              # beyond the largest transform


def test_version_and_launch_counter():
    assert b"sm_100a" in capi.lib().tdg_version()
    assert capi.kernel_launches() >= 0
