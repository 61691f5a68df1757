"""ctypes binding of libb200k.so (include/b2k.h).

There is deliberately no CPU fallback: if the library cannot be loaded, every
product entry point raises. The .so is built in-tree by `_build.build()`
(`__graft_entry__.build()` on the driver) so it travels with the repo snapshot.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# B2K_LIB overrides the in-tree library (A/B measurements of two builds, tools/ab_*.py)
LIB_PATH = os.environ.get("B2K_LIB") or os.path.join(PKG, "libb200k.so")

# enum b2_dtype (include/b2k.h)
BF16, F16, F32, F64, I32, I64, U8, U16, U32, U64 = 1, 2, 3, 4, 5, 6, 7, 8, 9, 10
DTYPE_NAMES = {BF16: "bf16", F16: "f16", F32: "f32", F64: "f64", I32: "i32", I64: "i64",
               U8: "u8", U16: "u16", U32: "u32", U64: "u64"}
B2_OK, B2_ERR_INVALID, B2_ERR_UNSUPPORTED, B2_ERR_CUDA, B2_ERR_NOMEM = 0, 1, 2, 3, 4

# every symbol include/b2k.h declares: (name, restype, argtypes)
_i64, _vp, _int, _sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
SIGNATURES = {
    "b2_abi_version": (_int, []),
    "b2_build_id": (ctypes.c_char_p, []),
    "b2_last_error": (ctypes.c_char_p, []),
    "b2_device_count": (_int, [ctypes.POINTER(_int)]),
    "b2_launch_count": (ctypes.c_uint64, []),
    "b2_dtype_size": (_sz, [_int]),
    "b2_tune_set": (_int, [ctypes.c_char_p, _i64]),
    "b2_tune_get": (_i64, [ctypes.c_char_p]),
    "b2_transpose": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, _int, _int, _vp]),
    "b2_transpose_host": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, _int, _int]),
    "b2_reduce_ws_bytes": (_sz, [_i64, _int]),
    "b2_reduce_sum": (_int, [_vp, _i64, _int, _vp, _vp, _sz, _int, _vp]),
    "b2_reduce_sum_host": (_int, [_vp, _i64, _int, _vp, _int]),
    "b2_reduce_sum_seq_f32": (_int, [_vp, _i64, _vp, _int, _vp]),
    "b2_reduce_sum_seq_f32_host": (_int, [_vp, _i64, _vp, _int]),
    "b2_mailbox_create": (_int, [_int, ctypes.POINTER(_vp), _vp]),
    "b2_mailbox_open": (_int, [_vp, _int, ctypes.POINTER(_vp)]),
    "b2_mailbox_close": (_int, [_vp, _int, _int]),
    "b2_mailbox_status": (_int, [_vp, _int, ctypes.POINTER(ctypes.c_uint64)]),
    "b2_reduce_sum_fused": (_int, [_vp, _i64, _int, _vp, _vp, _sz, _vp, _int, _int, ctypes.c_uint64,
                                   _int, _vp]),
    "b2_reduce_tree512_partials": (_int, [_vp, _i64, _vp, _int, _vp]),
    "b2_reduce_tree512": (_int, [_vp, _i64, _vp, _int, _vp]),
    "b2_reduce_tree512_host": (_int, [_vp, _i64, _vp, _int]),
    "b2_reduce_tree_partials": (_int, [_vp, _i64, _int, _vp, _int, _vp]),
    "b2_reduce_tree": (_int, [_vp, _i64, _int, _vp, _int, _vp]),
    "b2_reduce_tree_host": (_int, [_vp, _i64, _int, _vp, _int]),
    "b2_sync": (_int, [_int, _vp]),
    "b2_init": (_int, [_int]),
    "b2_peer_access": (_int, [_int, _int]),
    "b2_transpose_multi": (_int, [ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_i64), _i64,
                                  ctypes.POINTER(_i64), ctypes.POINTER(_i64), _int, _int]),
    "b2_reduce_sum_multi": (_int, [ctypes.POINTER(_vp), ctypes.POINTER(_i64), _int, _int, _vp]),
    "b2_copy_h2d": (_int, [_vp, _vp, _sz, _int]),
    "b2_copy_d2h": (_int, [_vp, _vp, _sz, _int]),
    "b2_device_alloc": (_int, [_sz, _int, ctypes.POINTER(_vp)]),
    "b2_device_free": (_int, [_vp, _int]),
    "b2_pipe_run": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _int]),
}


class B2Error(RuntimeError):
    """A libb200k call failed (code + the library's thread-local message)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"libb200k error {code}: {msg}")
        self.code = code
        self.msg = msg


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                "(there is no CPU fallback)")
        if not os.environ.get("B2K_LIB"):
            # the in-tree build must match the sources it ships with (content hash,
            # not mtimes): rebuild when nvcc is here, else refuse the stale library
            from . import _build
            if not _build.lib_is_current(LIB_PATH):
                try:
                    _build.build(force=True)
                except Exception as e:  # noqa: BLE001
                    raise ImportError(f"{LIB_PATH} was not built from this tree's csrc/ "
                                      f"(build id mismatch) and rebuilding failed: {e}") from None
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("B2K_LIB") and not hasattr(L, name):
                continue  # an older build under A/B measurement (tools/ab_*.py)
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.b2_abi_version() != 1:
            raise ImportError("libb200k ABI version mismatch")
        if not os.environ.get("B2K_LIB"):
            from . import _build
            want = "b2k-build-" + _build.source_id()
            if L.b2_build_id().decode() != want:
                raise ImportError(f"libb200k build id {L.b2_build_id().decode()} != {want}")
        _lib = L
        # B2K_TUNE="key=value,key=value": knob settings for measurement runs
        for kv in filter(None, os.environ.get("B2K_TUNE", "").split(",")):
            k, _, v = kv.partition("=")
            check(L.b2_tune_set(k.strip().encode(), int(v)))
    return _lib


def check(rc: int) -> None:
    if rc != B2_OK:
        msg = lib().b2_last_error().decode(errors="replace")
        raise B2Error(rc, msg)


def tune(key: str, value: int) -> None:
    """Set a performance knob (include/b2k.h b2_tune_set); results never depend on it."""
    check(lib().b2_tune_set(key.encode(), int(value)))


def tuning(key: str) -> int:
    return int(lib().b2_tune_get(key.encode()))


def launch_count() -> int:
    return int(lib().b2_launch_count())


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib().b2_device_count(ctypes.byref(n))
    return n.value if rc == B2_OK else 0
