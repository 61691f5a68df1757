"""Drop-in for the reference interpreter's entry points (minigpu/interp.py),
executing the OptiGPU transpose and reduce programs on a B200.

    run_program(program, entry, inputs) -> (ret, {param: flat data})   interp.py:380-387
    Interp(program).run(fn_name, inputs) -> (("ret", v) | None, {param: Array})  :106-128
    Array(dims, data, ctype="float", freed=False)                        :47-85
    InterpError, f32                                                     :39-44

How a call executes: parameters are marshalled exactly as Interp.run does
(missing input -> InterpError; Array arguments are used by reference and
mutated in place; other iterables become a fresh 1-D Array, f32-rounded for
`float*` parameters), the entry function is recognised (recognize.py) as one of
the hot-path programs, the program's own preconditions are checked with the
reference's error messages (bounds, rank, uninitialised cells, use after free,
exact_div), and the work runs through libb200k.so's host-buffer pipelines
(H2D / sm_100a kernel / D2H). Unrecognised programs raise UnsupportedProgram
(an InterpError): there is no CPU fallback.

Results: transposes are bit-identical to the reference; integer sums are exact
(the reference's unbounded ints; int cells are 4 bytes, intrinsics.py:35); the
A.5 tree-form fp32 sum is bit-identical; the naive fp32 sum (sequential order in
the reference) is returned correctly rounded from a parallel sum by default, within
the north-star tolerance, and bit-identical with the reference
with run_program(..., fp_order="reference") (its own sequential order, one warp).

Extensions (documented deviations):
  * `Array.data` may be a numpy array (zero-copy host buffer); results are then
    written into it and `run_program` returns that array instead of a list.
  * Rank-2 transpose parameters given as flat 1-D data are rejected; the
    reference would silently apply its 1-D pointer-offset rule (interp.py:239-240).
  * Errors are raised before any output cell is written (the reference leaves
    the cells it wrote before failing).
"""
from __future__ import annotations

import contextvars
import struct
from dataclasses import dataclass

import numpy as np

from . import ops
from .errors import InterpError, UnsupportedProgram
from .recognize import Plan, recognize


# fp_order of the Interp currently dispatching (run_program(..., fp_order=...))
_FP_ORDER: contextvars.ContextVar = contextvars.ContextVar("b2_fp_order", default="tree")


def f32(x: float) -> float:
    """Round to IEEE binary32 (interp.py:43-44)."""
    return struct.unpack("f", struct.pack("f", float(x)))[0]


@dataclass
class Array:
    """Row-major cells; `None` marks an uninitialised cell (interp.py:47-85).

    `data` is a Python list (reference layout) or a numpy array (zero-copy)."""

    dims: list
    data: object
    ctype: str = "float"
    freed: bool = False

    @staticmethod
    def alloc(dims, ctype):
        n = 1
        for d in dims:
            n *= d
        return Array(list(dims), [None] * n, ctype)

    @staticmethod
    def from_numpy(a: np.ndarray, ctype: str | None = None) -> "Array":
        """Zero-copy Array over a C-contiguous numpy buffer."""
        if not a.flags.c_contiguous:
            raise ValueError("Array.from_numpy needs a C-contiguous array")
        if ctype is None:
            ctype = "float" if a.dtype.kind == "f" and a.dtype.itemsize == 4 else "int"
        return Array(list(a.shape), a.reshape(-1), ctype)

    def offset(self, idxs) -> int:
        if len(idxs) != len(self.dims):
            raise InterpError(f"rank mismatch: {len(idxs)} indices into {len(self.dims)}-d array")
        off = 0
        for ix, d in zip(idxs, self.dims):
            if not (0 <= ix < d):
                raise InterpError(f"index {ix} out of bounds 0..{d}")
            off = off * d + ix
        return off

    def get(self, idxs):
        if self.freed:
            raise InterpError("use after free")
        v = self.data[self.offset(idxs)]
        if v is None:
            raise InterpError("read of uninitialized cell")
        return v

    def set(self, idxs, v):
        if self.freed:
            raise InterpError("use after free")
        if self.ctype == "float":
            v = f32(v)
        self.data[self.offset(idxs)] = v


def _is_array(v) -> bool:
    # this package's Array or the reference's (same fields)
    return all(hasattr(v, a) for a in ("dims", "data", "ctype", "freed"))


# ----------------------------------------------------------------------------- cell marshalling

def _cells(arr, n: int, want: str) -> np.ndarray:
    """First n cells of `arr` as a numpy vector: float32 for want == "float",
    the narrowest exact integer type for want == "int". Raises the reference's
    errors for freed arrays and uninitialised cells."""
    if arr.freed:
        raise InterpError("use after free")
    data = arr.data
    if isinstance(data, np.ndarray):
        v = data.reshape(-1)[:n]
        if v.size < n:
            raise IndexError("list index out of range")
        if want == "float" and v.dtype != np.float32:
            return _to_f32(v.astype(np.float64))
        return v
    if len(data) < n:
        raise IndexError("list index out of range")
    part = data[:n] if n != len(data) else data
    if any(x is None for x in part):
        raise InterpError("read of uninitialized cell")
    if want == "float":
        return _to_f32(np.fromiter(part, dtype=np.float64, count=n))
    return _ints(part)


def _struct_f_overflow_raises() -> bool:
    """struct.pack("f", x) for |x| beyond binary32 raises OverflowError on older
    CPythons and rounds to +-inf on 3.12+; f32() (interp.py:43-44) inherits
    whichever this interpreter does, so the drop-in follows the same rule."""
    try:
        struct.pack("f", 1e300)
        return False
    except OverflowError:
        return True


_F32_OVERFLOW_RAISES = _struct_f_overflow_raises()


def _to_f32(v: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        r = v.astype(np.float32)
    if _F32_OVERFLOW_RAISES and (np.isinf(r) & np.isfinite(v)).any():
        raise OverflowError("float too large to pack with f format")
    return r


def _ints(part) -> np.ndarray:
    """Exact integer cells: int32 when every value fits, else int64, else uint64
    (64-bit bit patterns such as fp64 bits). Values the reference would keep as
    non-integers (floats in an int cell) or beyond 64 bits are refused rather than
    silently converted."""
    if not all(isinstance(x, (int, np.integer)) for x in part):
        raise InterpError("int cell holds a non-integer value (not representable on the device)")
    try:
        v = np.array(part, dtype=np.int64)
        return v.astype(np.int32) if v.size == 0 or (
            v.min() >= -2**31 and v.max() < 2**31) else v
    except OverflowError:
        pass
    try:
        return np.array(part, dtype=np.uint64)
    except OverflowError:
        raise InterpError("int cell value outside the 64-bit range") from None


def _store(arr, values2d: np.ndarray, row_pitch: int):
    """Write a (rows x cols) block into arr.data, row r at offset r*row_pitch."""
    data = arr.data
    rows, cols = values2d.shape
    if isinstance(data, np.ndarray):
        dst = data.reshape(-1)
        view = np.lib.stride_tricks.as_strided(
            dst, shape=(rows, cols), strides=(row_pitch * dst.itemsize, dst.itemsize))
        view[...] = values2d.astype(dst.dtype, copy=False)
        return
    if row_pitch == cols:
        data[:rows * cols] = values2d.reshape(-1).tolist()
        return
    for r in range(rows):
        data[r * row_pitch:r * row_pitch + cols] = values2d[r].tolist()


# ----------------------------------------------------------------------------- interpreter

class Interp:
    """run(fn_name, inputs) mirrors minigpu.interp.Interp.run (interp.py:106-128)."""

    BACKENDS = ("auto", "kernels", "codegen")
    FP_ORDERS = ("tree", "reference")

    def __init__(self, program, backend: str = "auto", check=None, fp_order: str = "tree"):
        """backend: "kernels" = only the hand-written kernels (recognised
        programs); "codegen" = compile any GPU-form program (codegen.py);
        "auto" = kernels when the program is recognised, else codegen.
        check: pre-dispatch gate (gate.py): None (the reference's behaviour),
        "kernels" (device-side checker rules for this launch) or a callable
        such as minigpu.checker.check_program."""
        if backend not in self.BACKENDS:
            raise ValueError(f"backend must be one of {self.BACKENDS}")
        if fp_order not in self.FP_ORDERS:
            raise ValueError(f"fp_order must be one of {self.FP_ORDERS}")
        self.fp_order = fp_order
        self.program = program
        self.backend = backend
        self.check = check
        self.launch: list = []
        self.ctx_width: list = []

    def _dispatch(self, fn, fn_name, env, arrays):
        if self.backend != "codegen":
            try:
                plan = recognize(self.program, fn_name)
                token = _FP_ORDER.set(self.fp_order)
                try:
                    return _EXEC[(plan.kind, plan.form)](plan, env)
                finally:
                    _FP_ORDER.reset(token)
            except UnsupportedProgram:
                if self.backend == "kernels":
                    raise
        from . import codegen
        if not codegen.has_kernel(fn):
            # not one of the recognised programs and not a GPU program either
            recognize(self.program, fn_name)  # raises with the recogniser's diagnosis
        return codegen.run_compiled(codegen.compile_fn(fn), env, arrays)

    def run(self, fn_name: str, inputs: dict):
        fn = self.program.fn(fn_name)
        env: dict = {}
        arrays: dict = {}
        for pname, ptype in fn.params:
            if pname not in inputs:
                raise InterpError(f"missing input {pname!r}")
            v = inputs[pname]
            if ptype.endswith("*"):
                if _is_array(v):
                    arr = v
                    if isinstance(v.data, np.ndarray) and not v.data.flags.c_contiguous:
                        raise InterpError(f"{pname!r}: numpy-backed Array data must be C-contiguous "
                                          "(results are written in place)")
                elif isinstance(v, np.ndarray):
                    flat = np.ascontiguousarray(v).reshape(-1)
                    if ptype.startswith("float") and flat.dtype != np.float32:
                        flat = _to_f32(flat.astype(np.float64))
                    arr = Array([flat.size], flat, "float" if ptype.startswith("float") else "int")
                else:
                    data = list(v)
                    if ptype.startswith("float"):
                        data = _cells(Array([len(data)], data, "float"), len(data), "float").tolist()
                    arr = Array([len(data)], data, "float" if ptype.startswith("float") else "int")
                arrays[pname] = arr
                env[pname] = arr
            else:
                env[pname] = v
        if self.check is not None:
            from .gate import run_check
            run_check(self.check, self.program, fn_name, env)
        return self._dispatch(fn, fn_name, env, arrays), arrays


def run_program(program, entry: str, inputs: dict, backend: str = "auto", check=None,
                fp_order: str = "tree"):
    """Returns (return value, {param name: flat final array data}) (interp.py:380-387).

    List-backed arrays come back as fresh lists; numpy-backed arrays come back
    as the (mutated) numpy buffer itself. `backend` selects hand-written kernels
    and/or generated code, `check` an optional pre-dispatch gate (see Interp).
    `fp_order` for the naive fp32 sum (A.2): "tree" (default) returns the correctly
    rounded sum computed in parallel (binary64 accumulation; within the north-star
    tolerance of the reference's value), "reference" the reference's own sequential
    binary32 order, bit-identical with its result (one warp on the device)."""
    it = Interp(program, backend, check, fp_order)
    ret, arrays = it.run(entry, dict(inputs))
    out = {k: (a.data if isinstance(a.data, np.ndarray) else list(a.data))
           for k, a in arrays.items()}
    if isinstance(ret, tuple) and ret and ret[0] == "ret":
        ret = ret[1]
    return ret, out


# ----------------------------------------------------------------------------- program executors

def _int_arg(env, name):
    v = env[name]
    if isinstance(v, (bool, np.bool_)) or not isinstance(v, (int, np.integer)):
        raise InterpError(f"{name!r} must be an int")
    return int(v)


def _first_none(arr, n_rows, n_cols, pitch, yx):
    """(y, x) of the first uninitialised cell of arr[0:n_rows][0:n_cols] in the
    loop order (x outer unless yx), or None. numpy-backed data has none."""
    data = arr.data
    if isinstance(data, np.ndarray) or n_rows <= 0 or n_cols <= 0:
        return None
    best = None
    for pos, v in enumerate(data):
        if v is None:
            y, x = divmod(pos, pitch)
            if y < n_rows and x < n_cols:
                key = (y, x) if yx else (x, y)
                if best is None or key < best[0]:
                    best = (key, y, x)
    return None if best is None else best[1:]


def _transpose_naive_error(src, dst, sname, dname, W, H, yx):
    """The error the reference raises first walking `out[x][y] = in[y][x]` (x outer,
    or y outer for the swapped nest), or None. Per iteration it reads in[y][x]
    (freed, rank, bounds in index order, uninitialised: Array.get, interp.py:72-78)
    and then writes out[x][y] (freed, rank, bounds: Array.set, :80-85)."""
    cands = []  # (iteration key, 0 = read of in / 1 = write of out, exception)

    def key(x, y):
        return (y, x) if yx else (x, y)

    for which, arr, name, rows_need, cols_need in ((0, src, sname, H, W), (1, dst, dname, W, H)):
        # in[y][x] has (row, col) = (y, x); out[x][y] has (row, col) = (x, y)
        def at(r, c, which=which):
            return key(c, r) if which == 0 else key(r, c)
        if arr.freed:
            cands.append((key(0, 0), which, InterpError("use after free")))
            continue
        if len(arr.dims) == 1:
            cands.append((key(0, 0), which, InterpError(
                f"rank mismatch on {list(arr.dims)}: {name!r} is indexed as a 2-d array; flat "
                "data is not reinterpreted (the reference's 1-d pointer-offset rule, "
                "interp.py:239-240, is not supported)")))
            continue
        if len(arr.dims) != 2:
            cands.append((key(0, 0), which, InterpError(f"rank mismatch on {list(arr.dims)}￨[0, 0]")))
            continue
        R, C = arr.dims
        if rows_need > R:
            cands.append((at(R, 0), which, InterpError(f"index {R} out of bounds 0..{R}")))
        if cols_need > C:
            cands.append((at(0, C), which, InterpError(f"index {C} out of bounds 0..{C}")))
        if which == 0:
            hit = _first_none(arr, min(rows_need, R), min(cols_need, C), C, yx)
            if hit is not None:
                cands.append((at(*hit), 0, InterpError("read of uninitialized cell")))
    if not cands:
        return None
    return min(cands, key=lambda c: (c[0], c[1]))[2]


def _memcpy_cells(arr, n: int, want: str) -> np.ndarray:
    """memcpy_host_to_device of the first n cells (interp.py:353-365): flat, no
    freed check; the first missing cell raises IndexError, the first None cell
    InterpError, whichever comes first."""
    data = arr.data
    if n <= 0:
        return np.zeros(0, np.float32 if want == "float" else np.int32)
    if not isinstance(data, np.ndarray):
        for v in data[:n]:
            if v is None:
                raise InterpError("memcpy of uninitialized data")
        if len(data) < n:
            raise IndexError("list index out of range")
    return _cells(Array(list(arr.dims), data, arr.ctype), n, want)


def _exec_transpose_naive(plan: Plan, env):
    src, dst = env[plan.params["in"]], env[plan.params["out"]]
    W, H = _int_arg(env, plan.params["W"]), _int_arg(env, plan.params["H"])
    if W <= 0 or H <= 0:
        return None
    # in[y][x] for y < H, x < W; out[x][y] (interp.py:159-164, :271-276, Array.offset :61-70):
    # every error the walk could hit is decided up front, the earliest one raised
    err = _transpose_naive_error(src, dst, plan.params["in"], plan.params["out"], W, H,
                                 "_yx_" in plan.template.name)
    if err is not None:
        raise err
    R, C = src.dims
    Ro, Co = dst.dims
    want = "float" if dst.ctype == "float" else "int"
    a = _read_block(src, H, W, C, want)
    if isinstance(dst.data, np.ndarray) and dst.data.dtype == a.dtype and dst.data.flags.c_contiguous:
        out2d = np.lib.stride_tricks.as_strided(
            dst.data, shape=(W, H), strides=(Co * a.itemsize, a.itemsize))
        ops.transpose(a, out2d)
    else:
        out = ops.transpose(a)
        _store(dst, out, Co)
    return None


def _read_block(arr, rows, cols, pitch, want) -> np.ndarray:
    """arr.data as a (rows x cols) view/array with row pitch `pitch`."""
    data = arr.data
    if isinstance(data, np.ndarray) and (want == "int" or data.dtype == np.float32):
        flat = data.reshape(-1)
        return np.lib.stride_tricks.as_strided(flat, shape=(rows, cols),
                                               strides=(pitch * flat.itemsize, flat.itemsize))
    if pitch == cols:
        return _cells(arr, rows * cols, want).reshape(rows, cols)
    full = _cells(Array([len(data)], data, arr.ctype), (rows - 1) * pitch + cols, want)
    return np.lib.stride_tricks.as_strided(full, shape=(rows, cols),
                                           strides=(pitch * full.itemsize, full.itemsize)).copy()


def _exec_transpose_gpu(plan: Plan, env):
    """A.4 and its tile-size family (T x T tiles; A.4 is T = 32): memcpy_host_to_device2
    (flat copy of H*W cells), kernel, flat copy back. Any tile shape computes the
    same permutation, so every member runs on the hand-written transpose."""
    src, dst = env[plan.params["in"]], env[plan.params["out"]]
    W, H = _int_arg(env, plan.params["W"]), _int_arg(env, plan.params["H"])
    T = plan.consts.get("T", 32)
    n = H * W
    # host arrays are only touched by the flat memcpys (no freed check there)
    a = _memcpy_cells(src, n, "float")
    for v in (W, H):  # kernel_launch((W/T)*(H/T), ...): exact_div, interp.py:209-214
        if v % T != 0:
            raise InterpError(f"exact_div({v}, {T}) is not exact")
    if n <= 0:
        return None
    if (len(dst.data) if not isinstance(dst.data, np.ndarray) else dst.data.size) < n:
        raise IndexError("list assignment index out of range")
    a2d = np.ascontiguousarray(a).reshape(H, W)
    if isinstance(dst.data, np.ndarray) and dst.data.dtype == np.float32 and dst.data.flags.c_contiguous:
        # memcpy_device_to_host2 of the W x H result straight into the caller's buffer
        ops.transpose(a2d, dst.data.reshape(-1)[:n].reshape(W, H))
        return None
    out = ops.transpose(a2d)
    _store(dst, out.reshape(1, n), n)
    return None


def _exec_reduce_naive(plan: Plan, env):
    arr = env[plan.params["arr"]]
    N = _int_arg(env, plan.params["N"])
    cell = plan.cell
    if N <= 0:
        return ("ret", 0.0 if cell == "float" else 0)
    if arr.freed:
        raise InterpError("use after free")
    if len(arr.dims) != 1:
        raise InterpError(f"rank mismatch on {list(arr.dims)}￨[0]")
    # iteration i reads arr[i]: an uninitialised cell before dims[0] fails first
    if not isinstance(arr.data, np.ndarray) and any(v is None for v in arr.data[:min(N, arr.dims[0])]):
        raise InterpError("read of uninitialized cell")
    if N > arr.dims[0]:
        raise InterpError(f"index {arr.dims[0]} out of bounds 0..{arr.dims[0]}")
    x = _cells(arr, N, cell)
    if cell == "float":
        if _FP_ORDER.get() == "reference":  # the interpreter's own order, bit for bit
            return ("ret", ops.reduce_sum_sequential(np.ascontiguousarray(x)))
        return ("ret", float(np.float32(ops.reduce_sum(np.ascontiguousarray(x)))))
    if x.dtype not in (np.int32, np.int64):
        raise InterpError("int cell value outside the 64-bit range (cells beyond int64 are "
                          "not representable on the device)")
    # int32 cells: int64 accumulation; int64 cells: 128-bit (exact like Python ints)
    return ("ret", int(ops.reduce_sum(np.ascontiguousarray(x))))


def _exec_reduce_tree(plan: Plan, env):
    """A.5 and its block-size family (B-element blocks; A.5 is B = 512, float):
    flat copy of N cells, per-B tree on the device, sequential host sum. Int cells
    sum exactly in any order (the plain reduction kernel); float cells need the
    tree's own association (tree_kernel<B>, B = 64 .. 2048; other B -> codegen)."""
    B = plan.consts.get("B", 512)
    cell = plan.cell
    if cell == "float" and not (64 <= B <= 2048):
        raise UnsupportedProgram(f"no hand-written tree kernel for {B}-element blocks")
    arr = env[plan.params["arr"]]
    N = _int_arg(env, plan.params["N"])
    x = _memcpy_cells(arr, N, cell)  # memcpy_host_to_device1: no freed check
    if N % B != 0:
        raise InterpError(f"exact_div({N}, {B}) is not exact")
    if N <= 0:
        return ("ret", 0.0 if cell == "float" else 0)
    if cell == "int":
        if x.dtype not in (np.int32, np.int64):
            raise InterpError("int cell value outside the 64-bit range (cells beyond int64 are "
                              "not representable on the device)")
        return ("ret", int(ops.reduce_sum(np.ascontiguousarray(x))))
    return ("ret", ops.reduce_tree(np.ascontiguousarray(x), B))


_EXEC = {
    ("transpose", "naive"): _exec_transpose_naive,
    ("transpose", "gpu"): _exec_transpose_gpu,
    ("reduce", "naive"): _exec_reduce_naive,
    ("reduce", "tree512"): _exec_reduce_tree,
    ("reduce", "tree"): _exec_reduce_tree,
}

__all__ = ["Array", "Interp", "InterpError", "UnsupportedProgram", "f32", "run_program"]
