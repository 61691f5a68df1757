"""The C-ABI library loads and exports every symbol include/b2k.h declares;
argument validation works without a GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2605_13864_b200 import _lib


def header_symbols():
    with open(os.path.join(ROOT, "include", "b2k.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"B2_API\s+[\w\s\*]+?\b(b2_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 14
    L = _lib.lib()
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_abi_version_and_dtype_sizes():
    L = _lib.lib()
    assert L.b2_abi_version() == 1
    sizes = {_lib.BF16: 2, _lib.F16: 2, _lib.F32: 4, _lib.F64: 8, _lib.I32: 4, _lib.I64: 8,
             _lib.U8: 1, _lib.U16: 2, _lib.U32: 4, _lib.U64: 8, 99: 0}
    for d, s in sizes.items():
        assert L.b2_dtype_size(d) == s


@pytest.mark.parametrize("args,code", [
    ((None, None, 4, 4, 4, 4, _lib.F32, 0, None), _lib.B2_ERR_INVALID),
    ((1, 1, -1, 4, 4, 4, _lib.F32, 0, None), _lib.B2_ERR_INVALID),
    ((1, 1, 4, 4, 2, 4, _lib.F32, 0, None), _lib.B2_ERR_INVALID),
    ((1, 1, 4, 4, 4, 4, 99, 0, None), _lib.B2_ERR_UNSUPPORTED),
])
def test_transpose_argument_validation(args, code):
    L = _lib.lib()
    assert L.b2_transpose(*args) == code
    assert L.b2_last_error()


def test_zero_extent_is_a_noop():
    assert _lib.lib().b2_transpose(None, None, 0, 5, 5, 0, _lib.F32, 0, None) == 0


def test_reduce_argument_validation():
    L = _lib.lib()
    out = ctypes.c_double()
    assert L.b2_reduce_sum(None, -1, _lib.F32, ctypes.addressof(out), None, 0, 0, None) == _lib.B2_ERR_INVALID
    assert L.b2_reduce_sum_host(None, 4, 99, ctypes.addressof(out), 0) == _lib.B2_ERR_UNSUPPORTED
    f = ctypes.c_float()
    buf = (ctypes.c_float * 513)()
    assert L.b2_reduce_tree512_host(buf, 513, ctypes.byref(f), 0) == _lib.B2_ERR_INVALID
    assert b"exact_div(513, 512)" in L.b2_last_error()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.lib()


def test_multi_argument_validation():
    """b2_transpose_multi / b2_reduce_sum_multi reject bad shard arrays before
    touching a device."""
    L = _lib.lib()
    vp2 = (ctypes.c_void_p * 2)(None, None)
    i2 = (ctypes.c_int64 * 2)(4, 4)
    out = ctypes.c_double()
    assert L.b2_transpose_multi(vp2, vp2, i2, 4, i2, i2, _lib.F32, 0) == _lib.B2_ERR_INVALID
    assert L.b2_transpose_multi(vp2, vp2, i2, 4, i2, i2, 99, 2) == _lib.B2_ERR_UNSUPPORTED
    assert L.b2_transpose_multi(vp2, vp2, i2, 4, i2, i2, _lib.F32, 2) == _lib.B2_ERR_INVALID  # NULL shard
    neg = (ctypes.c_int64 * 2)(4, -1)
    assert L.b2_transpose_multi(vp2, vp2, neg, 4, i2, i2, _lib.F32, 2) == _lib.B2_ERR_INVALID
    assert L.b2_reduce_sum_multi(vp2, i2, 0, _lib.F32, ctypes.addressof(out)) == _lib.B2_ERR_INVALID
    assert L.b2_reduce_sum_multi(vp2, i2, 2, _lib.U8, ctypes.addressof(out)) == _lib.B2_ERR_UNSUPPORTED
    assert L.b2_reduce_sum_multi(vp2, neg, 2, _lib.I32, ctypes.addressof(out)) == _lib.B2_ERR_INVALID
    assert L.b2_reduce_sum_multi(vp2, i2, 2, _lib.I32, None) == _lib.B2_ERR_INVALID
    assert L.b2_peer_access(-1, 0) == 0


def test_build_id_matches_sources():
    """freshness is decided by content, not mtimes. The
    loaded library embeds the sha256 prefix of csrc/ + include/b2k.h + flags."""
    from paper_2605_13864_b200 import _build, _lib
    L = _lib.lib()
    assert L.b2_build_id().decode() == "b2k-build-" + _build.source_id()
    assert _build.lib_is_current()
