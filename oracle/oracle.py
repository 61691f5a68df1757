"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product).

Python face of the oracle: ctypes bindings to `oracle/liboracle.so` (the C
restatement in oracle.c) plus an independent numpy restatement of the same
reference semantics, so the two restatements can be cross-checked against each
other and against the golden vectors the reference interpreter produced
(tests/golden/). Allowed importers: tests/, __graft_entry__.smoke(), bench.py
(cpu_baseline leg and `--impl reference`).

Reference semantics restated (file:line in /root/reference/pkg/src/minigpu):
  transpose      interp.py:282-300 (loop nest), :259-277 (Assign), :61-70 (row-major)
  reduce fp32    interp.py:262-270 (`sum += arr[i]`, f32() on every store, :43-44)
  reduce int     interp.py:262-270 (unbounded Python int; int32 cells, intrinsics.py:35)
  reduce tree    SURVEY Appendix A.5 executed by interp.py:282-300 / :320-323 / :215-219
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        L.or_max_threads.restype = ctypes.c_int
        L.or_transpose.argtypes = [vp, vp, i64, i64, i64, i64, ctypes.c_int, ctypes.c_int]
        L.or_transpose.restype = ctypes.c_int
        L.or_reduce_f32_seq.argtypes = [vp, i64]
        L.or_reduce_f32_seq.restype = ctypes.c_float
        L.or_reduce_i32.argtypes = [vp, i64, ctypes.c_int]
        L.or_reduce_i32.restype = ctypes.c_int64
        L.or_reduce_f32_tree512.argtypes = [vp, i64, vp, vp]
        L.or_reduce_f32_tree512.restype = ctypes.c_int
        L.or_sum_f64.argtypes = [vp, i64, vp, vp]
        L.or_fill_u32.argtypes = [vp, i64, ctypes.c_uint64, ctypes.c_int]
        L.or_seg_f32_fold.argtypes = [vp, vp, i64, vp]
        L.or_seg_f32_fold.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().or_max_threads())


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ----------------------------------------------------------------------------- C restatement

def transpose(a: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """out[x][y] = in[y][x]; `a` is H x W (any 1/2/4/8-byte dtype)."""
    a = np.ascontiguousarray(a)
    H, W = a.shape
    out = np.empty((W, H), dtype=a.dtype)
    rc = lib().or_transpose(_ptr(a), _ptr(out), H, W, W, H, a.dtype.itemsize, nthreads)
    if rc:
        raise ValueError(f"unsupported element size {a.dtype.itemsize}")
    return out


def transpose_into(a: np.ndarray, out: np.ndarray, nthreads: int = 0) -> None:
    H, W = a.shape
    lib().or_transpose(_ptr(a), _ptr(out), H, W, W, H, a.dtype.itemsize, nthreads)


def reduce_f32_seq(x: np.ndarray) -> float:
    """Reference A.2 result: sequential binary32 sum (returns a binary32 value)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    return float(np.float32(lib().or_reduce_f32_seq(_ptr(x), x.size)))


def reduce_i32(x: np.ndarray, nthreads: int = 0) -> int:
    """Reference A.3 result: exact (unbounded) sum of int32 cells."""
    x = np.ascontiguousarray(x, dtype=np.int32)
    return int(lib().or_reduce_i32(_ptr(x), x.size, nthreads))


def reduce_f32_tree512(x: np.ndarray) -> tuple[float, np.ndarray]:
    """Reference A.5 result and its per-512 partials. Raises if 512 does not divide N."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    parts = np.empty(max(x.size // 512, 1), dtype=np.float32)
    res = np.zeros(1, dtype=np.float32)
    if lib().or_reduce_f32_tree512(_ptr(x), x.size, _ptr(parts), _ptr(res)):
        raise ValueError(f"exact_div({x.size}, 512) is not exact")
    return float(res[0]), parts[: x.size // 512]


def sum_f64(x: np.ndarray) -> tuple[float, float]:
    """(compensated binary64 sum, sum of |x|) — the yardstick for fp32 tolerances."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    s = np.zeros(1, dtype=np.float64)
    a = np.zeros(1, dtype=np.float64)
    lib().or_sum_f64(_ptr(x), x.size, _ptr(s), _ptr(a))
    return float(s[0]), float(a[0])


def seg_f32_fold(v: np.ndarray, ends: np.ndarray, acc: np.ndarray) -> bool:
    """In place: acc[g] = f32(... f32(acc[g] + v[b]) ... + v[e-1]) per segment
    [ends[g-1], ends[g]); v, acc float64; returns True on binary32 overflow."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    ends = np.ascontiguousarray(ends, dtype=np.int64)
    assert acc.dtype == np.float64 and acc.flags.c_contiguous and acc.size == ends.size
    return bool(lib().or_seg_f32_fold(_ptr(v), _ptr(ends), ends.size, _ptr(acc)))


def fill_u32(x: np.ndarray, seed: int, nthreads: int = 0) -> None:
    lib().or_fill_u32(_ptr(x), x.size, seed, nthreads)


# ----------------------------------------------------------------------------- numpy restatement

def np_transpose(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).T)


def np_reduce_f32_seq(x: np.ndarray) -> float:
    # cumsum in float32 accumulates strictly left to right in binary32.
    x = np.asarray(x, dtype=np.float32)
    if x.size == 0:
        return 0.0
    return float(np.cumsum(x, dtype=np.float32)[-1])


def np_reduce_i32(x: np.ndarray) -> int:
    return int(np.asarray(x, dtype=np.int32).sum(dtype=np.int64))


def np_reduce_f32_tree512(x: np.ndarray) -> tuple[float, np.ndarray]:
    x = np.asarray(x, dtype=np.float32)
    if x.size % 512:
        raise ValueError(f"exact_div({x.size}, 512) is not exact")
    b = x.reshape(-1, 512)
    s = b[:, 0::2] + b[:, 1::2]
    h = 128
    while h >= 1:
        s = s.copy()
        s[:, :h] = s[:, :h] + s[:, h:2 * h]
        h //= 2
    parts = s[:, 0].copy()
    return np_reduce_f32_seq(parts), parts


# ----------------------------------------------------------------------------- tolerances

def f32_tolerance(n: int, exact: float, abssum: float) -> float:
    """North-star fp32 tolerance (BASELINE.json): relative 1e-6*log2(N), or the
    order-independent forward bound 2*log2(N)*2^-24*sum|x| when cancellation makes
    the relative form meaningless."""
    lg = max(math.log2(max(n, 2)), 1.0)
    return max(1e-6 * lg * abs(exact), 2.0 * lg * 2.0 ** -24 * abssum)


def f32_seq_error_bound(n: int, abssum: float) -> float:
    """Worst-case error of the reference's own sequential binary32 sum: (N-1)*u*sum|x|.
    Only a sanity bound on the reference value itself (tests/test_oracle.py); far too
    loose to compare a GPU result with."""
    return max(n - 1, 0) * 2.0 ** -24 * abssum


def ref_consistency_bound(ref: float, exact: float, tol: float) -> float:
    """|g - r_ref| <= |r_ref - exact| + tol: the GPU value g (within tol of the exact
    sum) may differ from the reference's sequential binary32 value r_ref by no more
    than r_ref's own measured error plus tol (r_ref is pinned, so its error is known)."""
    return abs(ref - exact) + tol


def f32_gpu_bound(n: int, exact: float, abssum: float) -> float:
    """Error bound of the B200 fp32 sum (binary64 accumulation, one rounding to
    binary32, csrc/reduce.cu AccOf<float>): |t - exact| <= n 2^-53 sum|x| for the
    binary64 total t, then <= half an ulp of binary32 at |t| for the final rounding.
    Much tighter than f32_tolerance on well-conditioned data (~1 ulp of the result)."""
    acc = n * 2.0 ** -53 * abssum
    return acc + 0.5 * float(np.spacing(np.float32(min(abs(exact) + acc, 3.0e38))))
