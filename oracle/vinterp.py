"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product).

Vectorised restatement of the reference interpreter (minigpu/interp.py) for the
program language: SURVEY §8(f) rank 4, "makes the reference CPU path measurable
at C3/C4". Same entry (`run_program(program, entry, inputs)`, interp.py:380-387),
same semantics, but loop nests run as numpy operations over *lanes* (one lane
per iteration) instead of one Python call chain per element.

Semantics restated (file:line in /root/reference/pkg/src/minigpu/interp.py):
  values       Python ints (unbounded) and floats (binary64); float literals and
               float stores round to binary32 (:43-44, :83-84, :152-153, :262-270)
  arrays       row-major, bounds / rank / uninitialised / use-after-free checks
               (:47-85), 1-D pointer-offset rule (:232-241), pointer params by
               reference, iterables copied with f32() for float* (:106-128)
  operators    :179-206 (`/` and `%` truncate via int(a / b), 0 for b == 0),
               exact_div / pow2 / DMINDEXk (:208-230)
  statements   :248-309; loops ascending; `thread for` narrows ctx_width
               (:282-300); declarations / allocations (:311-328); kernel_launch,
               barriers, frees, memcpy, user calls (:330-377)

Why vectorising is exact. The reference runs every loop sequentially. A loop is
executed lock-step (statement by statement for all its iterations at once) only
when that cannot change any result:
  * statically, its body has no return / allocation / launch / memcpy / free /
    user call, and assigns no cell declared outside the body, except the
    reduction pattern `c += e` (one such statement, `c` never read in the body);
  * dynamically, every address of an array that the loop writes is touched by
    at most one iteration (checked per execution from logged read / write
    addresses). If two iterations touch it, the whole program restarts from its
    original inputs with that loop run sequentially (its inner loops may still
    vectorise) — so a conflicting program gets exactly the sequential answer.
  * reductions fold in iteration order: integer sums exactly (int64, with an
    overflow guard), float cells with the binary64-add-then-binary32-round of
    :262-270 in sequence (oracle.c or_seg_f32_fold). A float reduction whose
    lanes would not be in sequential order (a sequential loop between the cell
    and a vectorised loop) demotes that loop instead.
Loops with one parent lane are cut into chunks of ~LANE_BUDGET lanes, executed
in order (chunks preserve sequential order because iterations of different
chunks never run interleaved).

Limitations (raise VUnsupported instead of guessing): int values beyond int64,
floats stored into int arrays, lambdas, allocations inside vectorised contexts.
Error messages are the reference's; when several iterations fail, the lane that
fails at the earliest statement is reported (the reference reports the earliest
iteration).
"""
from __future__ import annotations

import struct

import numpy as np

from . import oracle

LANE_BUDGET = 1 << 21


class InterpError(Exception):
    """Same name and messages as minigpu.interp.InterpError (interp.py:39)."""


class VUnsupported(Exception):
    """The program leaves the fragment this restatement reproduces exactly."""


class _Restart(Exception):
    def __init__(self, nid):
        super().__init__(f"restart: loop {nid} must run sequentially")
        self.nid = nid


def f32(x):
    """interp.py:43-44 (the same struct round trip as the reference)."""
    return struct.unpack("f", struct.pack("f", float(x)))[0]


def _overflow_raises():
    try:
        struct.pack("f", 1e300)
        return False
    except OverflowError:  # older CPythons; 3.12+ rounds to +-inf
        return True


F32_OVERFLOW_RAISES = _overflow_raises()


def _f32_arr(v):
    v = np.asarray(v, dtype=np.float64)
    with np.errstate(over="ignore"):
        r = v.astype(np.float32)
    if F32_OVERFLOW_RAISES and np.any(np.isinf(r) & ~np.isinf(v)):
        raise OverflowError("float too large to pack with f format")
    return r


# ----------------------------------------------------------------------------- lanes and values

class _Level:
    """A set of lanes; `pmap[i]` is lane i's lane in the parent level."""
    __slots__ = ("n", "parent", "pmap", "cache")

    def __init__(self, n, parent=None, pmap=None):
        self.n = int(n)
        self.parent = parent
        self.pmap = pmap
        self.cache = {}


def _amap(cur: _Level, target: _Level):
    """Index array mapping cur's lanes to target's (an ancestor); None = identity."""
    if cur is target:
        return None
    key = id(target)
    m = cur.cache.get(key)
    if m is not None:
        return m
    L, m = cur, None
    while L is not target:
        if L.parent is None:
            raise RuntimeError("vinterp: value from a non-ancestor lane level")
        m = L.pmap if m is None else L.pmap[m]
        L = L.parent
    cur.cache[key] = m
    return m


class _LV:
    """A per-lane value attached to the level it was computed at."""
    __slots__ = ("arr", "level")

    def __init__(self, arr, level):
        self.arr = arr
        self.level = level


def _at(v, cur):
    if isinstance(v, _LV):
        m = _amap(cur, v.level)
        return v.arr if m is None else v.arr[m]
    return v


def _wrap(v, cur):
    return _LV(v, cur) if isinstance(v, np.ndarray) else v


class _Cell:
    __slots__ = ("v", "init", "t", "level", "depth", "name")

    def __init__(self, v, init, t, level, depth, name):
        self.v, self.init, self.t, self.level, self.depth, self.name = v, init, t, level, depth, name


class _Arr:
    __slots__ = ("dims", "data", "init", "ctype", "freed")

    def __init__(self, dims, ctype, data=None, init=None):
        self.dims = [int(d) for d in dims]
        n = 1
        for d in self.dims:
            n *= d
        self.ctype = ctype
        self.data = data if data is not None else np.zeros(n, np.float32 if ctype == "float" else np.int64)
        self.init = init if init is not None else np.zeros(n, bool)
        self.freed = False


class _Ptr:
    __slots__ = ("arr", "prefix")

    def __init__(self, arr, prefix=()):
        self.arr = arr
        self.prefix = tuple(prefix)


class _Frame:
    __slots__ = ("vars", "level")

    def __init__(self, level):
        self.vars = {}
        self.level = level


class _VecLoop:
    """One lock-step execution (chunk) of a loop: its lanes and access logs."""

    def __init__(self, nid, level, parent, maybe_written):
        self.nid = nid
        self.level = level
        self.parent = parent
        self.maybe_written = maybe_written  # set of _Arr ids, or None = any
        self.log = {}  # arr id -> list of (addr, iter, parent, is_write)
        self.written = set()

    def record(self, arr, addrs, cur, is_write):
        k = id(arr)
        if is_write:
            self.written.add(k)
        elif self.maybe_written is not None and k not in self.maybe_written:
            return
        it = _amap(cur, self.level)
        if it is None:
            it = np.arange(cur.n, dtype=np.int64)
        a = np.broadcast_to(np.asarray(addrs, dtype=np.int64), (cur.n,))
        self.log.setdefault(k, []).append((a, it, is_write))

    def conflict(self) -> bool:
        """Does an address written in this chunk get touched by two iterations
        (lanes of self.level) with the same parent lane?"""
        pm = _amap(self.level, self.parent) if self.parent.n > 1 else None
        for k in self.written:
            ents = self.log.get(k, [])
            addr = np.concatenate([e[0] for e in ents])
            it = np.concatenate([e[1] for e in ents])
            waddr = np.concatenate([e[0] for e in ents if e[2]])
            base = int(addr.min())
            span = int(addr.max()) - base + 1
            if span <= 4 * addr.size + 4096:
                # dense owner map: the last lane to touch each address
                rel = addr - base
                owner = np.full(span, -1, np.int64)
                owner[rel] = it
                other = owner[rel]
                mism = other != it
                if not mism.any():
                    continue
                if pm is not None:
                    mism &= pm[other] == pm[it]
                wflag = np.zeros(span, bool)
                wflag[waddr - base] = True
                if np.any(mism & wflag[rel]):
                    return True
                continue
            # sparse: sort by (parent, address), compare iteration ranges per group
            key = addr if pm is None else addr * np.int64(self.parent.n) + pm[it]
            order = np.argsort(key, kind="stable")
            sk, si = key[order], it[order]
            w = np.isin(addr, waddr)[order]
            starts = np.concatenate(([0], np.flatnonzero(np.diff(sk)) + 1))
            gmin = np.minimum.reduceat(si, starts)
            gmax = np.maximum.reduceat(si, starts)
            gw = np.add.reduceat(w.astype(np.int64), starts) > 0
            if np.any(gw & (gmin != gmax)):
                return True
        return False


# ----------------------------------------------------------------------------- static loop analysis

_NOOP_CALLS = {"kernel_setup_end", "kernel_teardown_begin", "blocksync", "magic_barrier",
               "kernel_teardown_sync"}


def _expr_vars(e, out):
    t = type(e).__name__
    if t == "Var":
        out.add(e.name)
    elif t == "BinOp":
        _expr_vars(e.lhs, out)
        _expr_vars(e.rhs, out)
    elif t == "Call":
        for a in e.args:
            _expr_vars(a, out)
    elif t in ("Access", "Ptr"):
        out.add(e.base)
        for i in e.idxs:
            _expr_vars(i, out)
    elif t == "Lam":
        _expr_vars(e.body, out)


def _analyse(loop):
    """(vectorisable, reduction Assign nids, names assigned with indices)."""
    declared = {loop.index}
    reads = set()
    cell_assigns = {}  # name -> [(assign, nested_in_for)]
    arr_targets = set()
    ok = [True]

    def walk(s, in_for):
        t = type(s).__name__
        if t == "Seq":
            for c in s.stmts:
                walk(c, in_for)
        elif t == "Decl":
            if s.alloc is not None:
                ok[0] = False
            declared.add(s.name)
            if s.init is not None:
                _expr_vars(s.init, reads)
            for d in s.dims:
                _expr_vars(d, reads)
        elif t == "Assign":
            _expr_vars(s.value, reads)
            for i in s.target.idxs:
                _expr_vars(i, reads)
            if s.target.idxs:
                arr_targets.add(s.target.base)
            else:
                cell_assigns.setdefault(s.target.base, []).append((s, in_for))
        elif t == "CallStmt":
            if s.ghost or s.fn in _NOOP_CALLS:
                return
            ok[0] = False
        elif t == "For":
            declared.add(s.index)
            _expr_vars(s.range.start, reads)
            _expr_vars(s.range.stop, reads)
            walk(s.body, True)
        elif t == "If":
            _expr_vars(s.cond, reads)
            walk(s.then, in_for)
            if s.els is not None:
                walk(s.els, in_for)
        elif t == "Return":
            ok[0] = False
        else:
            ok[0] = False

    walk(loop.body, False)
    if arr_targets & declared:  # writes through pointers declared in the body
        arr_targets = None
    reductions = set()
    for name, lst in cell_assigns.items():
        if name in declared:
            continue
        if len(lst) != 1 or lst[0][0].op != "+=" or name in reads:
            ok[0] = False
            continue
        reductions.add(lst[0][0].nid)
    return ok[0], reductions, arr_targets


# ----------------------------------------------------------------------------- interpreter

class VInterp:
    def __init__(self, program, lane_budget: int = LANE_BUDGET):
        self.program = program
        self.budget = int(lane_budget)
        self.seq_nids = set()
        self.analysis = {}
        self.restarts = 0

    # -- entry ------------------------------------------------------------------------
    def run(self, fn_name: str, inputs: dict):
        while True:
            try:
                return self._run_once(fn_name, inputs)
            except _Restart as r:
                if r.nid in self.seq_nids:
                    raise RuntimeError("vinterp: restart loop")  # pragma: no cover
                self.seq_nids.add(r.nid)
                self.restarts += 1

    def _run_once(self, fn_name, inputs):
        try:
            fn = self.program.fn(fn_name)
        except KeyError:
            raise InterpError(f"unknown function {fn_name!r}")
        self.launch = []
        self.ctx_width = []
        self.vstack = []
        self.loops = []  # ("vec"|"seq", nid) of the loops being executed
        self.root = _Level(1)
        frame = _Frame(self.root)
        arrays = {}
        for pname, ptype in fn.params:
            if pname not in inputs:
                raise InterpError(f"missing input {pname!r}")
            v = inputs[pname]
            if ptype.endswith("*"):
                arr = self._marshal(v, ptype)
                arrays[pname] = (arr, v)
                frame.vars[pname] = _Ptr(arr)
            else:
                frame.vars[pname] = v
        ret = self.exec_seq(fn.body, [frame], self.root)
        return ret, arrays

    @staticmethod
    def _marshal(v, ptype):
        is_float = ptype.startswith("float")
        if hasattr(v, "dims") and hasattr(v, "data") and hasattr(v, "ctype"):
            ctype = v.ctype
            if isinstance(v.data, np.ndarray):
                raw = np.ascontiguousarray(v.data).reshape(-1)
                init = np.ones(raw.size, bool)
            else:
                lst = list(v.data)
                init = np.array([x is not None for x in lst], bool)
                raw = [0 if x is None else x for x in lst]
            arr = _Arr(v.dims, ctype, init=init)
            if getattr(v, "freed", False):
                arr.freed = True
        else:
            raw = list(v)
            ctype = "float" if is_float else "int"
            arr = _Arr([len(raw)], ctype, init=np.ones(len(raw), bool))
            if is_float:
                raw = [f32(x) for x in raw]
        if ctype == "float":
            arr.data = _f32_arr(np.asarray(raw, dtype=np.float64)) if not isinstance(raw, np.ndarray) \
                else raw.astype(np.float32)
        else:
            a = np.asarray(raw)
            if a.dtype.kind == "u" and a.size and int(a.max()) >= 2 ** 63:
                raise VUnsupported("int cells beyond int64")
            if a.dtype.kind not in "iub":
                if any(not isinstance(x, (int, np.integer)) for x in raw):
                    raise VUnsupported("non-integer cells in an int array")
                raise VUnsupported("int cells beyond int64")
            arr.data = a.astype(np.int64)
        return arr

    # -- environment ----------------------------------------------------------------
    @staticmethod
    def lookup(env, name):
        for frame in reversed(env):
            if name in frame.vars:
                return frame.vars[name]
        raise InterpError(f"unbound variable {name!r}")

    # -- expressions ----------------------------------------------------------------
    def eval(self, e, env, cur):
        t = type(e).__name__
        if t == "IntLit":
            return e.value
        if t == "FloatLit":
            return f32(e.value)
        if t == "Var":
            v = self.lookup(env, e.name)
            if isinstance(v, _Cell):
                init = _at(v.init, cur)
                if init is False or (isinstance(init, np.ndarray) and not init.all()):
                    raise InterpError(f"read of uninitialized {e.name!r}")
                return _at(v.v, cur)
            return _at(v, cur)
        if t == "Access":
            tgt = self.lookup(env, e.base)
            idxs = [self.eval(i, env, cur) for i in e.idxs]
            if not isinstance(tgt, _Ptr):
                raise InterpError(f"{e.base!r} is not an array")
            return self._get(tgt, idxs, cur)
        if t == "BinOp":
            return self._binop(e.op, self.eval(e.lhs, env, cur), self.eval(e.rhs, env, cur))
        if t == "Call":
            return self._call_expr(e, env, cur)
        if t == "Ptr":
            v = self.lookup(env, e.base)
            if not isinstance(v, _Ptr):
                raise InterpError(f"{e.base!r} is not an array")
            idxs = [_wrap(self.eval(i, env, cur), cur) for i in e.idxs]
            return _Ptr(v.arr, v.prefix + tuple(idxs))
        if t == "Lam":
            raise VUnsupported("lambda in an executed expression")
        raise InterpError(f"cannot evaluate {e!r}")

    @staticmethod
    def _int_guard(op, a, b, r):
        """Python ints never wrap: refuse int64 results that might have."""
        if isinstance(r, np.ndarray) and r.dtype.kind == "i":
            fa = float(np.abs(np.asarray(a, dtype=np.float64)).max(initial=0))
            fb = float(np.abs(np.asarray(b, dtype=np.float64)).max(initial=0))
            if (fa * fb if op == "*" else fa + fb) >= 2.0 ** 62:
                raise VUnsupported("int arithmetic beyond int64")
        return r

    def _binop(self, op, a, b):
        scalar = not isinstance(a, np.ndarray) and not isinstance(b, np.ndarray)
        if scalar:  # exactly the reference's Python arithmetic
            if op == "+":
                return a + b
            if op == "-":
                return a - b
            if op == "*":
                return a * b
            if op == "/":
                return int(a / b) if b else 0
            if op == "%":
                if b == 0:
                    return 0
                return a - int(a / b) * b
            return {"==": lambda: a == b, "!=": lambda: a != b, "<": lambda: a < b,
                    "<=": lambda: a <= b, ">": lambda: a > b, ">=": lambda: a >= b}.get(
                op, lambda: self._bad_op(op))()
        a = self._num(a)
        b = self._num(b)
        if op == "+":
            return self._int_guard(op, a, b, a + b)
        if op == "-":
            return self._int_guard(op, a, b, a - b)
        if op == "*":
            return self._int_guard(op, a, b, a * b)
        if op in ("/", "%"):
            bz = np.asarray(b) == 0
            with np.errstate(divide="ignore", invalid="ignore"):
                q = np.trunc(np.asarray(a, dtype=np.float64) / np.where(bz, 1, b))
            q = np.where(bz, 0, q).astype(np.int64)
            if op == "/":
                return q
            return np.where(bz, 0, a - q * np.asarray(b))
        if op == "==":
            return np.equal(a, b)
        if op == "!=":
            return np.not_equal(a, b)
        if op == "<":
            return np.less(a, b)
        if op == "<=":
            return np.less_equal(a, b)
        if op == ">":
            return np.greater(a, b)
        if op == ">=":
            return np.greater_equal(a, b)
        return self._bad_op(op)

    @staticmethod
    def _bad_op(op):
        raise InterpError(f"unknown operator {op}")

    @staticmethod
    def _num(x):
        if isinstance(x, np.ndarray):
            return x.astype(np.int64) if x.dtype == bool else x
        if isinstance(x, bool):
            return int(x)
        if isinstance(x, int) and not -(2 ** 63) <= x < 2 ** 63:
            raise VUnsupported("int beyond int64 in a vectorised expression")
        return x

    def _call_expr(self, e, env, cur):
        if e.fn == "exact_div":
            a = self.eval(e.args[0], env, cur)
            b = self.eval(e.args[1], env, cur)
            if not isinstance(a, np.ndarray) and not isinstance(b, np.ndarray):
                if b == 0 or a % b != 0:
                    raise InterpError(f"exact_div({a}, {b}) is not exact")
                return a // b
            a, b = np.broadcast_arrays(self._num(a), self._num(b))
            bad = (b == 0) | (np.mod(a, np.where(b == 0, 1, b)) != 0)
            if bad.any():
                i = int(np.argmax(bad))
                raise InterpError(f"exact_div({a[i].item()}, {b[i].item()}) is not exact")
            return np.floor_divide(a, b)
        if e.fn == "pow2":
            k = self.eval(e.args[0], env, cur)
            if not isinstance(k, np.ndarray):
                return 0 if k < 0 else 1 << k
            k = self._num(k)
            return np.where(k < 0, 0, np.left_shift(1, np.maximum(k, 0)))
        if e.fn.startswith("DMINDEX"):
            k = len(e.args) // 2
            dims = [self.eval(a, env, cur) for a in e.args[:k]]
            idxs = [self.eval(a, env, cur) for a in e.args[k:]]
            off = 0
            for d, ix in zip(dims, idxs):
                off = off * d + ix
            return off
        if e.fn.startswith("MINDEX") or e.fn.startswith("MSIZE"):
            raise InterpError(f"{e.fn} only appears in generated CUDA")
        raise InterpError(f"cannot call {e.fn!r} in an expression")

    # -- array access ---------------------------------------------------------------
    def _flat(self, p: _Ptr, idxs, cur):
        """interp.py:61-70 + :232-241 over lanes: flat offsets (scalar or array)."""
        full = [_at(x, cur) for x in p.prefix] + list(idxs)
        dims = p.arr.dims
        if len(full) == len(dims) or (len(full) == 1 and len(dims) == 1):
            pass
        elif len(full) == len(dims) + 1 and len(dims) == 1:
            full = [self._binop("+", full[0], full[1])]
        else:
            raise InterpError(f"rank mismatch on {dims}￨{self._show(full)}")
        off = 0
        for ix, d in zip(full, dims):
            if isinstance(ix, np.ndarray):
                ix = self._num(ix)
                if ix.dtype.kind == "f":
                    raise VUnsupported("float array index")
                bad = (ix < 0) | (ix >= d)
                if bad.any():
                    raise InterpError(f"index {ix[int(np.argmax(bad))].item()} out of bounds 0..{d}")
            elif not (0 <= ix < d):
                raise InterpError(f"index {ix} out of bounds 0..{d}")
            off = off * d + ix
        return off

    @staticmethod
    def _show(full):
        return [x.tolist()[:1] if isinstance(x, np.ndarray) else x for x in full]

    def _get(self, p: _Ptr, idxs, cur):
        arr = p.arr
        if arr.freed:
            raise InterpError("use after free")
        off = self._flat(p, idxs, cur)
        init = arr.init[off]
        if not np.all(init):
            raise InterpError("read of uninitialized cell")
        for v in self.vstack:
            v.record(arr, off, cur, False)
        val = arr.data[off]
        if arr.ctype == "float":
            return val.astype(np.float64) if isinstance(val, np.ndarray) else float(val)
        return val if isinstance(val, np.ndarray) else int(val)

    def _set(self, p: _Ptr, idxs, val, op, cur):
        arr = p.arr
        if op == "+=":
            val = self._binop("+", self._get(p, idxs, cur), val)
        if arr.freed:
            raise InterpError("use after free")
        off = self._flat(p, idxs, cur)
        for v in self.vstack:
            v.record(arr, off, cur, True)
        if arr.ctype == "float":
            val = _f32_arr(val) if isinstance(val, np.ndarray) else np.float32(f32(val))
        else:
            if isinstance(val, np.ndarray):
                if val.dtype.kind == "f":
                    raise VUnsupported("float stored into an int array")
                val = val.astype(np.int64)
            elif isinstance(val, float):
                raise VUnsupported("float stored into an int array")
            else:
                val = int(val)
                if not -(2 ** 63) <= val < 2 ** 63:
                    raise VUnsupported("int cell beyond int64")
        if isinstance(off, np.ndarray):
            arr.data[off] = np.broadcast_to(val, off.shape) if np.ndim(val) == 0 else val
        else:
            if isinstance(val, np.ndarray):  # uniform address written by several lanes: last wins
                val = val[-1]
            arr.data[off] = val
        arr.init[off] = True

    # -- statements -----------------------------------------------------------------
    def exec_seq(self, seq, env, cur):
        env = env + [_Frame(cur)]
        for s in seq.stmts:
            r = self.exec(s, env, cur)
            if r is not None:
                return r
        return None

    def exec(self, s, env, cur):
        t = type(s).__name__
        if t == "Decl":
            return self._decl(s, env, cur)
        if t == "Assign":
            return self._assign(s, env, cur)
        if t == "CallStmt":
            return self._call(s, env, cur)
        if t == "Seq":
            return self.exec_seq(s, env, cur)
        if t == "For":
            return self._for(s, env, cur)
        if t == "If":
            c = self.eval(s.cond, env, cur)
            if not isinstance(c, np.ndarray):
                if c:
                    return self.exec_seq(s.then, env, cur)
                return self.exec_seq(s.els, env, cur) if s.els is not None else None
            c = c.astype(bool)
            for branch, mask in ((s.then, c), (s.els, ~c)):
                if branch is None or not mask.any():
                    continue
                sub = cur if mask.all() else _Level(int(mask.sum()), cur, np.flatnonzero(mask))
                r = self.exec_seq(branch, env, sub)
                if r is not None:  # pragma: no cover - returns only run on one lane
                    return r
            return None
        if t == "Return":
            v = self.eval(s.value, env, cur)
            if isinstance(v, np.ndarray):
                if v.size != 1:
                    raise VUnsupported("return from several lanes")
                v = v.reshape(-1)[0].item()
            return ("ret", v)
        raise InterpError(f"cannot execute {t}")

    def _decl(self, d, env, cur):
        frame = env[-1]
        if d.alloc is None:
            val = self.eval(d.init, env, cur) if d.init is not None else None
            if val is not None and d.ctype == "float":
                val = _f32_arr(val).astype(np.float64) if isinstance(val, np.ndarray) else f32(val)
            if isinstance(val, _Ptr):
                frame.vars[d.name] = val
                return None
            frame.vars[d.name] = _Cell(_wrap(val, cur), val is not None, d.ctype, cur, len(self.loops),
                                       d.name)
            return None
        if cur.n != 1:
            raise VUnsupported("allocation in a vectorised context")
        dims = [self.eval(x, env, cur) for x in d.dims]
        if d.alloc == "__smem_malloc":
            if not self.launch:
                raise InterpError("__smem_malloc outside a kernel launch")
            dims = [self.launch[-1][0]] + dims
        elif d.alloc == "__treg_malloc":
            width = self.ctx_width[-1] if self.ctx_width else 1
            dims = [width] + dims
        frame.vars[d.name] = _Ptr(_Arr(dims, d.ctype))
        return None

    def _assign(self, s, env, cur):
        tgt = self.lookup(env, s.target.base)
        val = self.eval(s.value, env, cur)
        if isinstance(tgt, _Cell):
            if s.op == "+=" and tgt.level is not cur and self._is_reduction(s.nid):
                return self._fold(tgt, val, cur)
            if s.op == "+=":
                init = _at(tgt.init, cur)
                if init is False or (isinstance(init, np.ndarray) and not init.all()):
                    raise InterpError(f"read of uninitialized {s.target.base!r}")
                val = self._binop("+", _at(tgt.v, cur), val)
            if tgt.t == "float":
                val = _f32_arr(val).astype(np.float64) if isinstance(val, np.ndarray) else f32(val)
            self._cell_store(tgt, val, cur)
            return None
        if not isinstance(tgt, _Ptr):
            raise InterpError(f"{s.target.base!r} is not assignable")
        idxs = [self.eval(i, env, cur) for i in s.target.idxs]
        self._set(tgt, idxs, val, s.op, cur)
        return None

    @staticmethod
    def _cell_store(cell, val, cur):
        m = _amap(cur, cell.level)
        if m is None:
            cell.v = _wrap(val, cur)
            cell.init = True
            return
        # a subset of the cell's lanes (if-branches): scatter
        if len(np.unique(m)) != len(m):
            raise RuntimeError("vinterp: non-reduction cell write from several iterations")
        Lc = cell.level
        old = cell.v.arr if isinstance(cell.v, _LV) else np.full(Lc.n, 0 if cell.v is None else cell.v)
        new = old.astype(np.result_type(old, np.asarray(val)), copy=True)
        new[m] = val
        init = cell.init.copy() if isinstance(cell.init, np.ndarray) else np.full(Lc.n, bool(cell.init))
        init[m] = True
        cell.v = _LV(new, Lc)
        cell.init = init

    def _is_reduction(self, nid):
        for v in reversed(self.vstack):
            if nid in self.analysis[v.nid][1]:
                return True
        return False

    def _fold(self, cell, val, cur):
        """`cell += val` from many iterations: fold in lane (= iteration) order."""
        Lc = cell.level
        m = _amap(cur, Lc)
        vals = np.broadcast_to(np.asarray(val), (cur.n,))
        if m is None:
            m = np.arange(cur.n)
        init = cell.init
        if (isinstance(init, np.ndarray) and not init[np.unique(m)].all()) or init is False:
            raise InterpError(f"read of uninitialized {cell.name!r}")
        ends = np.flatnonzero(np.diff(m)) + 1
        ends = np.concatenate((ends, [m.size])).astype(np.int64)
        groups = m[ends - 1]
        old = cell.v.arr if isinstance(cell.v, _LV) else np.full(Lc.n, cell.v)
        fvals = vals.dtype.kind == "f" or (old.dtype.kind == "f")
        if cell.t == "float":
            # lanes must be in sequential order: no sequential loop below a vectorised one
            seen_vec = None
            for kind, nid in self.loops[cell.depth:]:
                if kind == "vec" and seen_vec is None:
                    seen_vec = nid
                elif kind == "seq" and seen_vec is not None:
                    raise _Restart(seen_vec)
            acc = old[groups].astype(np.float64)
            if oracle.seg_f32_fold(vals.astype(np.float64), ends, acc) and F32_OVERFLOW_RAISES:
                raise OverflowError("float too large to pack with f format")
            new = old.astype(np.float64, copy=True)
            new[groups] = acc
        else:
            if fvals:
                raise VUnsupported("float accumulated into an int cell")
            v64 = vals.astype(np.int64)
            mx = float(np.abs(v64).max(initial=0))
            starts = np.concatenate(([0], ends[:-1]))
            if mx * (np.diff(np.concatenate(([0], ends))).max(initial=1) + 1) < 2.0 ** 62:
                sums = np.add.reduceat(v64, starts) if v64.size else np.zeros(0, np.int64)
            else:
                sums = np.array([sum(int(x) for x in v64[b:e]) for b, e in zip(starts, ends)], dtype=object)
            new = old.astype(object if sums.dtype == object else np.int64, copy=True)
            new[groups] = new[groups] + sums
            if new.dtype == object:
                if any(not -(2 ** 63) <= int(x) < 2 ** 63 for x in new):
                    raise VUnsupported("int cell beyond int64")
                new = new.astype(np.int64)
        cell.v = new[0].item() if Lc.n == 1 else _LV(new, Lc)
        return None

    def _call(self, s, env, cur):
        if s.ghost:
            return None
        fn = s.fn
        if fn == "kernel_launch":
            bpg, tpb, smem = (self.eval(a, env, cur) for a in s.args[:3])
            self.launch.append((bpg, tpb, smem))
            self.ctx_width.append(bpg * tpb)
            return None
        if fn in _NOOP_CALLS:
            return None
        if fn == "kernel_kill":
            self.launch.pop()
            self.ctx_width.pop()
            return None
        if fn in ("free", "gmem_free") or fn.startswith("__smem_free"):
            p = self.eval(s.args[0], env, cur)
            if isinstance(p, _Ptr):
                p.arr.freed = True
            return None
        if fn.startswith("memcpy_host_to_device") or fn.startswith("memcpy_device_to_host"):
            dest = self.eval(s.args[0], env, cur)
            src = self.eval(s.args[1], env, cur)
            n = 1
            for a in s.args[2:]:
                n *= self.eval(a, env, cur)
            if n > src.arr.data.size or n > dest.arr.data.size:
                raise IndexError("list index out of range")
            if n > 0 and not src.arr.init[:n].all():
                raise InterpError("memcpy of uninitialized data")
            if src.arr.ctype != dest.arr.ctype:
                raise VUnsupported("memcpy between float and int arrays")
            dest.arr.data[:n] = src.arr.data[:n]
            dest.arr.init[:n] = True
            return None
        try:
            callee = self.program.fn(fn)
        except KeyError:
            raise InterpError(f"unknown function {fn!r}")
        if callee.body is None:
            raise InterpError(f"cannot interpret admitted function {fn!r}")
        if cur.n != 1:
            raise VUnsupported("user call in a vectorised context")
        frame = _Frame(cur)
        for (pname, _), a in zip(callee.params, s.args):
            frame.vars[pname] = _wrap(self.eval(a, env, cur), cur)
        self.exec_seq(callee.body, [frame], cur)
        return None

    # -- loops ------------------------------------------------------------------------
    def _for(self, s, env, cur):
        start = self.eval(s.range.start, env, cur)
        stop = self.eval(s.range.stop, env, cur)
        thread = s.mode in ("thread", "magic_thread")
        pushed = False
        if thread and self.ctx_width:
            outer = self.ctx_width[-1]
            n = stop - start
            if isinstance(n, np.ndarray):
                n = int(n.max(initial=0))
            n = max(n, 1)
            self.ctx_width.append(outer // n if n and outer % n == 0 else outer)
            pushed = True
        try:
            if s.nid not in self.analysis:
                self.analysis[s.nid] = _analyse(s)
            vec = self.analysis[s.nid][0] and s.nid not in self.seq_nids
            if vec:
                return self._for_vec(s, env, cur, start, stop)
            return self._for_seq(s, env, cur, start, stop)
        finally:
            if pushed:
                self.ctx_width.pop()

    def _for_seq(self, s, env, cur, start, stop):
        self.loops.append(("seq", s.nid))
        try:
            if not isinstance(start, np.ndarray) and not isinstance(stop, np.ndarray):
                for i in range(start, stop):
                    frame = _Frame(cur)
                    frame.vars[s.index] = i
                    r = self.exec_seq(s.body, env + [frame], cur)
                    if r is not None:
                        return r
                return None
            start = np.broadcast_to(self._num(start), (cur.n,))
            stop = np.broadcast_to(self._num(stop), (cur.n,))
            cnt = np.maximum(stop - start, 0)
            for k in range(int(cnt.max(initial=0))):
                act = cnt > k
                sub = cur if act.all() else _Level(int(act.sum()), cur, np.flatnonzero(act))
                frame = _Frame(sub)
                frame.vars[s.index] = _LV((start + k) if sub is cur else (start + k)[act], sub)
                r = self.exec_seq(s.body, env + [frame], sub)
                if r is not None:  # pragma: no cover
                    return r
            return None
        finally:
            self.loops.pop()

    def _maybe_written(self, s, env):
        names = self.analysis[s.nid][2]
        if names is None:
            return None
        ids = set()
        for nm in names:
            try:
                v = self.lookup(env, nm)
            except InterpError:
                return None
            if not isinstance(v, _Ptr):
                return None
            ids.add(id(v.arr))
        return ids

    def _for_vec(self, s, env, cur, start, stop):
        P = cur.n
        mw = self._maybe_written(s, env)
        self.loops.append(("vec", s.nid))
        try:
            if P == 1:
                a = int(_at(start, cur).reshape(-1)[0]) if isinstance(start, np.ndarray) else start
                b = int(_at(stop, cur).reshape(-1)[0]) if isinstance(stop, np.ndarray) else stop
                i, chunk = a, 1
                while i < b:
                    c = min(chunk, b - i)
                    saved = getattr(self, "_peak", 0)
                    self._peak = 0
                    self._vec_chunk(s, env, cur, np.arange(i, i + c, dtype=np.int64),
                                    np.zeros(c, np.int64), mw)
                    per = max(self._peak, c) / c
                    self._peak = max(saved, self._peak)
                    chunk = max(1, int(self.budget // max(per, 1)))
                    i += c
                return None
            st = np.broadcast_to(self._num(start), (P,)).astype(np.int64)
            sp = np.broadcast_to(self._num(stop), (P,)).astype(np.int64)
            cnt = np.maximum(sp - st, 0)
            total = int(cnt.sum())
            if total == 0:
                return None
            pmap = np.repeat(np.arange(P, dtype=np.int64), cnt)
            offs = np.arange(total, dtype=np.int64) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            self._vec_chunk(s, env, cur, st[pmap] + offs, pmap, mw)
            return None
        finally:
            self.loops.pop()

    def _vec_chunk(self, s, env, cur, idx, pmap, mw):
        L = _Level(idx.size, cur, pmap)
        self._peak = max(getattr(self, "_peak", 0), L.n)
        v = _VecLoop(s.nid, L, cur, mw)
        self.vstack.append(v)
        try:
            frame = _Frame(L)
            frame.vars[s.index] = _LV(idx, L)
            self.exec_seq(s.body, env + [frame], L)
        finally:
            self.vstack.pop()
        if v.conflict():
            raise _Restart(s.nid)


def run_program(program, entry: str, inputs: dict, as_numpy: bool = False, lane_budget: int = LANE_BUDGET):
    """interp.py:380-387 restated: (return value, {param: final array data}).

    Array inputs are updated in place like the reference's (list-backed ones
    cell by cell, numpy-backed ones by copy). With as_numpy=True the returned
    arrays are numpy buffers (float32 / int64) instead of Python lists, and
    uninitialised cells read 0."""
    it = VInterp(program, lane_budget)
    ret, arrays = it.run(entry, dict(inputs))
    out = {}
    for name, (arr, src) in arrays.items():
        if as_numpy:
            data = arr.data
        else:
            vals = arr.data.tolist()
            data = [v if ok else None for v, ok in zip(vals, arr.init.tolist())]
        out[name] = data
        if hasattr(src, "dims") and hasattr(src, "data"):
            if isinstance(src.data, np.ndarray):
                src.data.reshape(-1)[...] = arr.data.astype(src.data.dtype, copy=False)
            elif isinstance(src.data, list):
                src.data[:] = data if not as_numpy else \
                    [v if ok else None for v, ok in zip(arr.data.tolist(), arr.init.tolist())]
            src.freed = arr.freed
    if isinstance(ret, tuple) and ret and ret[0] == "ret":
        ret = ret[1]
        if isinstance(ret, np.generic):
            ret = ret.item()
    return ret, out
