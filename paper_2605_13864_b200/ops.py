"""Typed, zero-copy entries on device tensors and host arrays.

These are the buffers-in / buffers-out faces of the two programs, named after
the DSL entries the reference interprets (`transpose(in, out, W, H)`,
`reduce(arr, N)`). `run_program` (interp.py in this package)
recognises a Program and lands here.

Device arguments are torch CUDA tensors (or anything exposing
`__cuda_array_interface__`): the work is enqueued on the current torch stream
and the call returns without synchronising. Host arguments are numpy arrays:
the library pipelines H2D / kernel / D2H through its own device buffers and
returns when the result is in host memory (pinned buffers make this fastest).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check, lib

try:  # torch is plumbing only (device memory, streams); optional for host calls
    import torch
except Exception:  # pragma: no cover
    torch = None

_NP_DTYPES = {
    np.dtype(np.float32): _lib.F32, np.dtype(np.float64): _lib.F64,
    np.dtype(np.int32): _lib.I32, np.dtype(np.int64): _lib.I64,
    np.dtype(np.uint8): _lib.U8, np.dtype(np.int8): _lib.U8,
    np.dtype(np.uint16): _lib.U16, np.dtype(np.int16): _lib.U16,
    np.dtype(np.float16): _lib.F16, np.dtype(np.uint32): _lib.U32,
    np.dtype(np.uint64): _lib.U64,
}


def _torch_dtypes():
    return {
        torch.float32: _lib.F32, torch.float64: _lib.F64, torch.bfloat16: _lib.BF16,
        torch.float16: _lib.F16, torch.int32: _lib.I32, torch.int64: _lib.I64,
        torch.uint8: _lib.U8, torch.int8: _lib.U8, torch.int16: _lib.U16,
        torch.uint16: _lib.U16, torch.uint32: _lib.U32, torch.uint64: _lib.U64,
    }


def _is_torch_cuda(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _as_device(x):
    """CUDA arrays from other libraries (`__cuda_array_interface__`, e.g. CuPy,
    Numba) become zero-copy torch views; everything else passes through."""
    if x is not None and torch is not None and not isinstance(x, torch.Tensor) \
            and hasattr(x, "__cuda_array_interface__"):
        return torch.as_tensor(x, device="cuda")
    return x


def b2_dtype(x) -> int:
    if torch is not None and isinstance(x, torch.Tensor):
        d = _torch_dtypes().get(x.dtype)
    else:
        d = _NP_DTYPES.get(np.asarray(x).dtype)
    if d is None:
        raise TypeError(f"unsupported dtype {getattr(x, 'dtype', type(x))}")
    return d


def _stream_ptr(t, stream=None) -> int:
    if stream is not None:
        return int(getattr(stream, "cuda_stream", stream))
    return int(torch.cuda.current_stream(t.device).cuda_stream)


# ----------------------------------------------------------------------------- transpose

def transpose(inp, out=None, *, stream=None):
    """out = inp^T (bit-exact). `inp` is rows x cols with unit column stride.

    Device tensors: returns `out` (allocated if None), asynchronous on the stream.
    Host numpy arrays: returns `out` after the host pipeline completes.
    """
    inp, out = _as_device(inp), _as_device(out)
    if _is_torch_cuda(inp):
        if inp.dim() != 2 or (inp.numel() and inp.stride(1) != 1):
            raise ValueError("transpose: input must be 2-D with unit column stride")
        rows, cols = inp.shape
        if out is None:
            out = torch.empty((cols, rows), dtype=inp.dtype, device=inp.device)
        if not _is_torch_cuda(out) or out.dtype != inp.dtype or tuple(out.shape) != (cols, rows):
            raise ValueError("transpose: out must be a (cols, rows) CUDA tensor of the same dtype")
        if out.numel() and out.stride(1) != 1:
            raise ValueError("transpose: out must have unit column stride")
        if inp.numel() == 0:
            return out
        check(lib().b2_transpose(inp.data_ptr(), out.data_ptr(), rows, cols, inp.stride(0),
                                 out.stride(0), b2_dtype(inp), inp.device.index,
                                 _stream_ptr(inp, stream)))
        return out
    a = np.asarray(inp)
    if a.ndim != 2 or (a.size and a.strides[1] != a.itemsize):
        raise ValueError("transpose: input must be 2-D with unit column stride")
    rows, cols = a.shape
    if out is None:
        out = np.empty((cols, rows), dtype=a.dtype)
    if out.shape != (cols, rows) or out.dtype != a.dtype or (out.size and out.strides[1] != out.itemsize):
        raise ValueError("transpose: out must be a (cols, rows) array of the same dtype")
    if a.size == 0:
        return out
    check(lib().b2_transpose_host(a.ctypes.data, out.ctypes.data, rows, cols,
                                  a.strides[0] // a.itemsize, out.strides[0] // out.itemsize,
                                  b2_dtype(a), _host_device()))
    return out


# ----------------------------------------------------------------------------- reduction

_ACC = {_lib.F32: (np.float32, "float32"), _lib.I32: (np.int64, "int64"),
        _lib.F64: (np.float64, "float64"), _lib.I64: (np.int64, "int64")}


def _int128(words) -> int:
    """(lo, hi) int64 words of a B2_I64 result -> Python int."""
    lo, hi = int(words[0]), int(words[1])
    return (lo & ((1 << 64) - 1)) + (hi << 64)


def reduce_sum(arr, *, out=None, ws=None, stream=None):
    """Sum of a 1-D float32 / int32 / int64 / float64 array (int32 accumulates in
    int64, int64 in 128 bits: exact like the reference's unbounded ints).

    Device: returns a 1-element CUDA tensor (float32 / int64 / float64), async;
    for int64 input a 2-element int64 tensor (lo, hi words; see `int128`).
    Host: returns a Python float / int.
    """
    arr, out = _as_device(arr), _as_device(out)
    d = b2_dtype(arr)
    if d not in _ACC:
        raise TypeError("reduce: dtype must be float32, int32, int64 or float64")
    npacc, tacc = _ACC[d]
    words = 2 if d == _lib.I64 else 1
    if _is_torch_cuda(arr):
        if arr.dim() != 1 or (arr.numel() and arr.stride(0) != 1):
            raise ValueError("reduce: input must be a contiguous 1-D tensor")
        if out is None:
            out = torch.empty(words, dtype=getattr(torch, tacc), device=arr.device)
        wsp, wsb = (0, 0) if ws is None else (ws.data_ptr(), ws.numel() * ws.element_size())
        check(lib().b2_reduce_sum(arr.data_ptr(), arr.numel(), d, out.data_ptr(), wsp or None, wsb,
                                  arr.device.index, _stream_ptr(arr, stream)))
        return out
    a = np.ascontiguousarray(arr).reshape(-1)
    res = np.zeros(words, dtype=npacc)
    check(lib().b2_reduce_sum_host(a.ctypes.data, a.size, d, res.ctypes.data, _host_device()))
    return _int128(res) if words == 2 else res[0].item()


def reduce_sum_sequential(arr, *, out=None, stream=None):
    """The naive fp32 program A.2 in the reference's own order (interp.py:262-270:
    `sum += arr[i]`, one binary32 rounding per cell, i ascending) — bit-identical with
    the reference interpreter, where `reduce_sum` returns the correctly rounded sum.
    Inherently sequential (one warp, ~4 cycles per cell). float32 1-D input.

    Device: returns a 1-element float32 CUDA tensor (async; `out`, if given, is
    overwritten with the sum). Host: returns a Python float."""
    arr, out = _as_device(arr), _as_device(out)
    if b2_dtype(arr) != _lib.F32:
        raise TypeError("sequential sum: dtype must be float32")
    if _is_torch_cuda(arr):
        if arr.dim() != 1 or (arr.numel() and arr.stride(0) != 1):
            raise ValueError("sequential sum: input must be a contiguous 1-D tensor")
        if out is None:
            out = torch.zeros(1, dtype=torch.float32, device=arr.device)
        else:
            out.zero_()
        check(lib().b2_reduce_sum_seq_f32(arr.data_ptr(), arr.numel(), out.data_ptr(), arr.device.index,
                                          _stream_ptr(arr, stream)))
        return out
    a = np.ascontiguousarray(arr, dtype=np.float32).reshape(-1)
    res = np.zeros(1, dtype=np.float32)
    check(lib().b2_reduce_sum_seq_f32_host(a.ctypes.data, a.size, res.ctypes.data, _host_device()))
    return float(res[0])


def int128(t) -> int:
    """Python int of a device int64-sum result tensor (lo, hi words)."""
    return _int128(t.cpu().numpy() if hasattr(t, "cpu") else t)


def reduce_tree(arr, block: int = 512, *, stream=None) -> float:
    """The A.5 tree-form program and its block-size family
    (programs.reduce_tree_family), bit-identical with the reference interpreter:
    per-`block` halving tree on the device, sequential binary32 host sum.
    `block` is a power of two in 64..2048 (A.5: 512)."""
    res = ctypes.c_float(0.0)
    if not _is_torch_cuda(arr):
        a = np.ascontiguousarray(arr, dtype=np.float32).reshape(-1)
        check(lib().b2_reduce_tree_host(a.ctypes.data, a.size, int(block), ctypes.byref(res), _host_device()))
        return float(res.value)
    if arr.dtype != torch.float32 or arr.dim() != 1 or (arr.numel() and arr.stride(0) != 1):
        raise ValueError("reduce_tree: input must be a contiguous 1-D float32 tensor")
    check(lib().b2_reduce_tree(arr.data_ptr(), arr.numel(), int(block), ctypes.byref(res),
                               arr.device.index, _stream_ptr(arr, stream)))
    return float(res.value)


def reduce_tree_partials(arr, block: int = 512, partials=None, *, stream=None):
    if partials is None:
        partials = torch.empty(arr.numel() // block, dtype=torch.float32, device=arr.device)
    check(lib().b2_reduce_tree_partials(arr.data_ptr(), arr.numel(), int(block), partials.data_ptr(),
                                        arr.device.index, _stream_ptr(arr, stream)))
    return partials


def reduce_tree512(arr, *, stream=None) -> float:
    """A.5: reduce_tree with 512-element blocks."""
    return reduce_tree(arr, 512, stream=stream)


def reduce_tree512_partials(arr, partials=None, *, stream=None):
    return reduce_tree_partials(arr, 512, partials, stream=stream)


def reduce_ws_bytes(n: int, dtype: int) -> int:
    return int(lib().b2_reduce_ws_bytes(n, dtype))


# ----------------------------------------------------------------------------- multi-GPU (one process)

def _ptr_array(ptrs):
    return (ctypes.c_void_p * len(ptrs))(*ptrs)


def _i64_array(vals):
    return (ctypes.c_int64 * len(vals))(*vals)


def transpose_multi(shards, outs=None):
    """Row-block sharded transpose driven from one process (b2_transpose_multi).

    `shards[g]` is a rows_g x cols CUDA tensor (any device); `outs[g]` receives
    its cols x rows_g transpose — by default a new tensor on the shard's device
    (the output stays sharded); pass column-slab views of one full
    matrix (e.g. `full[:, r0:r1]`, possibly on another GPU) to assemble it with
    the kernels' own peer stores. Synchronous; returns `outs`."""
    shards = [_as_device(t) for t in shards]
    if not shards:
        raise ValueError("transpose_multi: no shards")
    cols = shards[0].shape[1] if shards[0].dim() == 2 else -1
    dt = b2_dtype(shards[0])
    for t in shards:
        if not _is_torch_cuda(t) or t.dim() != 2 or t.shape[1] != cols or b2_dtype(t) != dt:
            raise ValueError("transpose_multi: shards must be 2-D CUDA tensors with equal cols and dtype")
        if t.numel() and t.stride(1) != 1:
            raise ValueError("transpose_multi: shards must have unit column stride")
    if outs is None:
        outs = [torch.empty((cols, t.shape[0]), dtype=t.dtype, device=t.device) for t in shards]
    outs = [_as_device(o) for o in outs]
    if len(outs) != len(shards):
        raise ValueError("transpose_multi: one output per shard")
    for t, o in zip(shards, outs):
        if not _is_torch_cuda(o) or tuple(o.shape) != (cols, t.shape[0]) or o.dtype != t.dtype \
                or (o.numel() and o.stride(1) != 1):
            raise ValueError("transpose_multi: outs[g] must be a (cols, rows_g) CUDA tensor, unit column stride")
    check(lib().b2_transpose_multi(
        _ptr_array([t.data_ptr() or None for t in shards]), _ptr_array([o.data_ptr() or None for o in outs]),
        _i64_array([t.shape[0] for t in shards]), cols,
        _i64_array([max(t.stride(0), cols) for t in shards]),
        _i64_array([max(o.stride(0), t.shape[0]) for t, o in zip(shards, outs)]), dt, len(shards)))
    return outs


def reduce_sum_multi(shards):
    """Sum over contiguous 1-D CUDA shards (any devices) with the cross-GPU
    combine fused into the kernels (b2_reduce_sum_multi). Synchronous; returns a
    Python float (fp32 / fp64) or int (int32 inputs, exact int64 sum)."""
    shards = [_as_device(t) for t in shards]
    if not shards:
        raise ValueError("reduce_sum_multi: no shards")
    d = b2_dtype(shards[0])
    if d not in _ACC:
        raise TypeError("reduce: dtype must be float32, int32 or float64")
    for t in shards:
        if not _is_torch_cuda(t) or t.dim() != 1 or b2_dtype(t) != d or (t.numel() and t.stride(0) != 1):
            raise ValueError("reduce_sum_multi: shards must be contiguous 1-D CUDA tensors of one dtype")
    res = np.zeros(1, dtype=_ACC[d][0])
    check(lib().b2_reduce_sum_multi(_ptr_array([t.data_ptr() or None for t in shards]),
                                    _i64_array([t.numel() for t in shards]), len(shards), d,
                                    res.ctypes.data))
    return res[0].item()


def init_devices(ndev: int = 0) -> None:
    """Create the library's per-device contexts and enable peer access between
    every pair of devices 0..ndev-1 (all devices when ndev <= 0)."""
    check(lib().b2_init(int(ndev)))


# ----------------------------------------------------------------------------- device choice

_HOST_DEVICE = None


def set_host_device(dev: int) -> None:
    """Device used by host-buffer calls (default: torch's current device, else 0)."""
    global _HOST_DEVICE
    _HOST_DEVICE = int(dev)


def _host_device() -> int:
    if _HOST_DEVICE is not None:
        return _HOST_DEVICE
    if torch is not None and torch.cuda.is_available():
        return torch.cuda.current_device()
    return 0
