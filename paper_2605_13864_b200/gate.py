"""Pre-dispatch gate for GPU-form programs.

The reference proves a derived program safe with its separation-logic checker
(`check_program`, minigpu/checker.py:927) before anything runs; the paper's
kernels are "verified" in that sense. `run_program(..., check=...)` restores
that gate in front of the B200 dispatch:

  * check=<callable>  — called as check(program) first; pass the reference's own
    `minigpu.checker.check_program` to gate on the full proof (it raises
    CheckError; nothing is launched);
  * check="kernels"   — this module: the checker's *device-side* rules, decided
    for the concrete launch (the parameters are known at dispatch time), with the
    checker's error codes:
      E-SMEM         the launch's shared-memory size is exactly what the
                     kernel's __smem_malloc calls allocate (checker.py:298-318);
      E-THREADS-CTX  `blocksync()` must run in a block-wide thread context of
                     exactly tpb threads, outside thread-dependent branches
                     (checker.py:779-789); global memory is only accessed from a
                     single-thread context (checker.py:405-422);
      E-DESYNC       no shared-memory cell written by one thread is read or
                     written by another thread of the block without a barrier in
                     between (checker.py:447-452) — decided exactly per barrier
                     interval over every thread of the analysed blocks;
                     likewise no global cell is written by one thread and touched
                     by another thread of the same launch (no grid barrier).
    Blocks analysed: all, one by one, when the launch has <= MAX_BLOCKS blocks.
    Larger launches are analysed ONCE with every block-level `thread for` index
    kept symbolic (an affine form base + sum c_j B_j over the block indices B_j):
    shared-memory indices, branch conditions and loop bounds must not depend on
    the block indices at all (then every block has the analysed block's exact
    intra-block pattern), and every global index must be affine in them with one
    coefficient vector per array (checked); two blocks can then only collide in a
    written array if some nonzero block offset delta keeps every dimension's
    offset sum_j c_kj delta_j within that dimension's per-block span — refused
    unless each block index owns a dimension whose coefficient exceeds the span
    (the tiling shape of every derived program). Anything else (a non-affine use
    of a block index, e.g. `b % 7`, a product of two block indices) is refused
    with E-GATE-UNSUPPORTED instead of being sampled.
    Indices and branch conditions must not depend on array contents; such a
    program is refused with E-GATE-DATA rather than waved through.
  * check=None (default) — no gate, exactly like the reference's run_program.
"""
from __future__ import annotations

import numpy as np

from .errors import InterpError

MAX_BLOCKS = 64


class GateError(Exception):
    """A kernel the gate refuses; `code` follows minigpu.errors (E-THREADS-CTX,
    E-DESYNC) plus E-GATE-DATA / E-GATE-UNSUPPORTED for what it cannot decide."""

    def __init__(self, code: str, message: str):
        self.code = code
        self.message = message
        super().__init__(f"{code}: {message}")


DATA = object()  # an array-content value: known to exist, never inspected


class Aff:
    """base + sum(coef[j] * B_j): a value affine in the symbolic block indices B_j
    (large launches, see the module doc). `base` is an int or a lane array."""

    __slots__ = ("base", "coef")

    def __init__(self, base, coef):
        self.base = base
        self.coef = {k: v for k, v in coef.items() if v}

    @staticmethod
    def of(v):
        return v if isinstance(v, Aff) else Aff(v, {})


def _aff_op(op, a, b):
    """Affine arithmetic; anything that would make a block index appear
    non-affinely is refused."""
    A, B = Aff.of(a), Aff.of(b)
    if op in ("+", "-"):
        sg = 1 if op == "+" else -1
        coef = dict(A.coef)
        for k, v in B.coef.items():
            coef[k] = coef.get(k, 0) + sg * v
        r = Aff(_binop(op, A.base, B.base), coef)
        return r if r.coef else r.base
    if op == "*":
        for X, Y in ((A, B), (B, A)):
            if not X.coef and not isinstance(X.base, np.ndarray):
                k = int(X.base)
                r = Aff(_binop("*", Y.base, k), {j: c * k for j, c in Y.coef.items()})
                return r if r.coef else r.base
    raise GateError("E-GATE-UNSUPPORTED", f"block index used non-affinely (operator {op!r}) in a large "
                                          "launch: the per-block analysis cannot cover every block")


def _cls(x):
    return type(x).__name__


def _stmts(s):
    return list(s.stmts) if s is not None else []


def _is_kernel_scope(s):
    st = [x for x in _stmts(s) if not (_cls(x) == "CallStmt" and x.ghost)]
    return bool(st) and _cls(st[0]) == "CallStmt" and st[0].fn == "kernel_launch"


class _Lanes:
    """Threads of one block being analysed: env values are scalars or arrays
    over the lanes; `tid` is each lane's thread index within the block — the
    first thread of the range the context-width narrowing gives it
    (interp.py:285-299: iteration i of a `thread for` over n in a context of
    width w owns threads [base + i*w/n, base + (i+1)*w/n))."""

    def __init__(self, tid):
        self.tid = tid

    @property
    def n(self):
        return self.tid.size


class _KernelGate:
    def __init__(self, env, arrays, bpg, tpb, dims):
        self.env0 = env          # host scalars
        self.arrays = arrays     # name -> "global" | "smem" | "treg"
        self.bpg, self.tpb = bpg, tpb
        self.dims = dims         # name -> dims (per-block dims for smem), when known
        self.glog = []           # (name, addr, global thread id, is_write) over the launch
        self.blocks = 0
        self.assigned = set()    # cells assigned in the kernel: their values are not tracked

    # ------------------------------------------------------------ values
    def eval(self, e, env, lanes):
        c = _cls(e)
        if c == "IntLit":
            return e.value
        if c == "FloatLit":
            return DATA
        if c == "Var":
            if e.name in self.assigned:
                return DATA
            if e.name in env:
                return env[e.name]
            raise GateError("E-GATE-UNSUPPORTED", f"unbound variable {e.name!r} in a kernel")
        if c == "Access":
            self.access(e.base, e.idxs, env, lanes, False)
            return DATA
        if c == "BinOp":
            a, b = self.eval(e.lhs, env, lanes), self.eval(e.rhs, env, lanes)
            if a is DATA or b is DATA:
                return DATA
            if isinstance(a, Aff) or isinstance(b, Aff):
                return _aff_op(e.op, a, b)
            return _binop(e.op, a, b)
        if c == "Call":
            args = [self.eval(a, env, lanes) for a in e.args]
            if any(a is DATA for a in args):
                return DATA
            if e.fn.startswith("DMINDEX"):
                return 0  # the block's own slot of a per-block array
            if any(isinstance(a, Aff) for a in args):
                raise GateError("E-GATE-UNSUPPORTED", f"block index inside {e.fn}() in a large launch")
            if e.fn == "exact_div":
                a, b = args
                if np.any(np.asarray(b) == 0) or np.any(np.mod(a, np.where(np.asarray(b) == 0, 1, b)) != 0):
                    raise InterpError(f"exact_div({_first(a)}, {_first(b)}) is not exact")
                return np.floor_divide(a, b) if isinstance(a, np.ndarray) or isinstance(b, np.ndarray) else a // b
            if e.fn == "pow2":
                k = args[0]
                if isinstance(k, np.ndarray):
                    return np.where(k < 0, 0, np.left_shift(1, np.maximum(k, 0)))
                return 0 if k < 0 else 1 << k
            if e.fn.startswith("DMINDEX"):
                return 0  # the block's own slot of a per-block array
            raise GateError("E-GATE-UNSUPPORTED", f"call to {e.fn!r} in a kernel expression")
        raise GateError("E-GATE-UNSUPPORTED", f"{c} in a kernel expression")

    def index(self, e, env, lanes, affine=False):
        v = self.eval(e, env, lanes)
        if v is DATA:
            raise GateError("E-GATE-DATA", "an index or condition depends on array contents")
        if isinstance(v, Aff) and not affine:
            raise GateError("E-GATE-UNSUPPORTED", "a loop bound, branch condition or shared-memory index "
                                                  "depends on the block index in a large launch")
        return v

    # ------------------------------------------------------------ memory
    def access(self, base, idxs, env, lanes, is_write):
        if lanes is None:
            raise GateError("E-GATE-DATA", "a launch parameter depends on array contents")
        kind = self.arrays.get(base)
        if kind is None:
            raise GateError("E-GATE-UNSUPPORTED", f"{base!r} is not an array the kernel can reach")
        ix = [self.index(i, env, lanes, affine=(kind == "global")) for i in idxs]
        if kind in ("smem", "treg"):
            ix = ix[1:]  # per-block (per-thread) storage: drop the DMINDEX slot
        if kind == "treg":
            return  # registers are private to their thread
        dims = self.dims.get(base)
        if dims is not None and len(dims) == 1 and len(ix) == 2:
            # the 1-D pointer-offset rule &a[k][j] -> a[k + j] (interp.py:239-240): one cell
            ix = [_aff_op("+", ix[0], ix[1]) if isinstance(ix[0], Aff) or isinstance(ix[1], Aff)
                  else _binop("+", ix[0], ix[1])]
        if kind == "global":
            self._affine_record(base, ix, is_write, lanes)
            ix = [v.base if isinstance(v, Aff) else v for v in ix]
        addr = np.zeros(lanes.n, np.int64)
        for k, v in enumerate(ix):  # row-major; any injective encoding serves the check
            stride = int(dims[k]) if dims is not None and k < len(dims) else 1 << 31
            addr = addr * stride + np.asarray(v, dtype=np.int64)
        if kind == "smem":
            self.seg.append((base, np.broadcast_to(addr, (lanes.n,)), lanes.tid, is_write))
            return
        if self.width != 1:
            raise GateError("E-THREADS-CTX", f"global memory access requires a single-thread context, "
                                             f"have ThreadsCtx of width {self.width}")
        gid = lanes.tid + np.int64(self.block_id) * self.tpb
        self.glog.append((base, np.broadcast_to(addr, (lanes.n,)), gid, is_write))

    # ------------------------------------------------------------ statements
    def run(self, body):
        """Walk the kernel body from the grid-wide context (width bpg * tpb)."""
        self.width = self.bpg * self.tpb
        self.block_id = -1
        self.seg = []
        self.symbolic = self.bpg > MAX_BLOCKS
        self.affine, self.block_vars = {}, {}
        self._walk_grid(body, dict(self.env0))
        _check_conflicts(self.glog, "global memory", per_block=False)
        if self.symbolic:
            self._cross_block_check()

    def _walk_grid(self, stmts, env):
        for pos, s in enumerate(stmts):
            c = _cls(s)
            if c == "CallStmt" and (s.ghost or s.fn in ("kernel_setup_end", "kernel_teardown_begin")):
                continue
            if self.width == self.tpb:  # one block: the rest of this sequence is per-block code
                self._block(stmts[pos:], env)
                return
            if c == "For" and s.mode in ("thread", "magic_thread"):
                a, b = self.index(s.range.start, env, None), self.index(s.range.stop, env, None)
                n = max(b - a, 1)
                outer = self.width
                self.width = outer // n if outer % n == 0 else outer
                if self.symbolic:  # one pass with the block index symbolic: B_j in [a, b)
                    if b > a:
                        self.block_vars[s.index] = (a, b - 1)
                        env2 = dict(env)
                        env2[s.index] = Aff(a, {s.index: 1})
                        self._walk_grid(_stmts(s.body), env2)
                else:
                    for v in range(a, b):
                        env2 = dict(env)
                        env2[s.index] = v
                        self._walk_grid(_stmts(s.body), env2)
                self.width = outer
                continue
            if c == "CallStmt" and s.fn == "blocksync":
                raise GateError("E-THREADS-CTX", f"blocksync requires a block-wide ThreadsCtx of {self.tpb} "
                                                 f"threads, have width {self.width}")
            raise GateError("E-GATE-UNSUPPORTED", f"{c} at grid level of a kernel")

    def _affine_record(self, base, ix, is_write, lanes):
        """Per global array: the block-index coefficient vector of every dimension
        (must agree between accesses) and the per-dimension range of the bases."""
        coefs = tuple(tuple(sorted(Aff.of(v).coef.items())) for v in ix)
        rec = self.affine.setdefault(base, {"coef": coefs, "lo": [None] * len(ix), "hi": [None] * len(ix),
                                            "write": False})
        if rec["coef"] != coefs:
            raise GateError("E-GATE-UNSUPPORTED", f"global array {base!r} indexed with different block-index "
                                                  "coefficients in one large launch")
        rec["write"] |= is_write
        for k, v in enumerate(ix):
            b = np.asarray(Aff.of(v).base, dtype=np.int64)
            if b.size == 0:
                continue
            lo, hi = int(b.min()), int(b.max())
            rec["lo"][k] = lo if rec["lo"][k] is None else min(rec["lo"][k], lo)
            rec["hi"][k] = hi if rec["hi"][k] is None else max(rec["hi"][k], hi)

    def _cross_block_check(self):
        """Large launches: no cell of a written global array is reached from two
        different blocks. Sufficient (and the tiling shape of the derived programs):
        every block index j varying over >1 value owns a dimension k whose index
        depends on B_j alone with |c_kj| > span_k (the per-block extent of that
        dimension), so any nonzero block offset separates the footprints there."""
        for name, rec in self.affine.items():
            if not rec["write"]:
                continue
            coefs = [dict(c) for c in rec["coef"]]
            for j, (lo_j, hi_j) in self.block_vars.items():
                if hi_j <= lo_j:
                    continue  # a block loop with one iteration
                ok = False
                for k, c in enumerate(coefs):
                    if set(c) == {j} and rec["lo"][k] is not None and abs(c[j]) > rec["hi"][k] - rec["lo"][k]:
                        ok = True
                        break
                if not ok:
                    raise GateError("E-GATE-UNSUPPORTED", f"cannot prove that blocks write disjoint cells of "
                                                          f"{name!r} (block index {j!r}) in a large launch")

    def _block(self, stmts, env):
        self.block_id += 1
        self.blocks += 1
        self.seg = []
        lanes = _Lanes(np.zeros(1, np.int64))
        self._walk(stmts, env, lanes, branch=False)
        _check_conflicts(self.seg, "shared memory", per_block=True)
        self.seg = []

    def _walk(self, stmts, env, lanes, branch):
        for s in stmts:
            self._stmt(s, env, lanes, branch)

    def _stmt(self, s, env, lanes, branch):
        c = _cls(s)
        if c == "Seq":
            self._walk(_stmts(s), dict(env), lanes, branch)
        elif c == "CallStmt":
            if s.ghost or s.fn in ("kernel_setup_end", "kernel_teardown_begin", "magic_barrier"):
                return
            if s.fn == "blocksync":
                if self.width != self.tpb:
                    raise GateError("E-THREADS-CTX", f"blocksync requires a block-wide ThreadsCtx of "
                                                     f"{self.tpb} threads, have width {self.width}")
                if branch:
                    raise GateError("E-THREADS-CTX", "blocksync under a thread-dependent branch")
                _check_conflicts(self.seg, "shared memory", per_block=True)
                self.seg = []
                return
            raise GateError("E-GATE-UNSUPPORTED", f"call to {s.fn!r} inside a kernel")
        elif c == "Decl":
            if s.alloc is not None:
                raise GateError("E-GATE-UNSUPPORTED", "allocation inside a kernel body")
            env[s.name] = self.eval(s.init, env, lanes) if s.init is not None else DATA
        elif c == "Assign":
            self.eval(s.value, env, lanes)
            if s.target.idxs:
                if s.op == "+=":
                    self.access(s.target.base, s.target.idxs, env, lanes, False)
                self.access(s.target.base, s.target.idxs, env, lanes, True)
            else:
                self.assigned.add(s.target.base)
        elif c == "For":
            a, b = self.index(s.range.start, env, lanes), self.index(s.range.stop, env, lanes)
            if isinstance(a, np.ndarray) or isinstance(b, np.ndarray):
                if not (np.all(a == _first(a)) and np.all(b == _first(b))):
                    raise GateError("E-GATE-UNSUPPORTED", "thread-dependent loop bounds")
                a, b = _first(a), _first(b)
            if s.mode in ("thread", "magic_thread"):
                n = max(b - a, 1)
                outer = self.width
                if outer % n:
                    raise GateError("E-GATE-UNSUPPORTED", f"thread for over {n} iterations in a context of "
                                                          f"width {outer}")
                self.width = outer // n
                k = max(b - a, 0)
                step = np.int64(self.width)
                sub = _Lanes(np.repeat(lanes.tid, k) + np.tile(np.arange(k, dtype=np.int64) * step, lanes.n))
                env2 = {kk: (np.repeat(v, k) if isinstance(v, np.ndarray) else v) for kk, v in env.items()}
                env2[s.index] = np.tile(np.arange(a, b, dtype=np.int64), lanes.n)
                if k:
                    self._walk(_stmts(s.body), env2, sub, branch)
                self.width = outer
            else:
                for i in range(a, b):
                    env2 = dict(env)
                    env2[s.index] = i
                    self._walk(_stmts(s.body), env2, lanes, branch)
        elif c == "If":
            cond = self.index(s.cond, env, lanes)
            if not isinstance(cond, np.ndarray):
                self._walk(_stmts(s.then) if cond else _stmts(s.els), dict(env), lanes, branch)
                return
            cond = cond.astype(bool)
            for body, m in ((s.then, cond), (s.els, ~cond)):
                if body is None or not m.any():
                    continue
                sub = _Lanes(lanes.tid[m])
                env2 = {kk: (v[m] if isinstance(v, np.ndarray) else v) for kk, v in env.items()}
                self._walk(_stmts(body), env2, sub, branch or not m.all())
        elif c == "Return":
            raise GateError("E-GATE-UNSUPPORTED", "return inside a kernel")
        else:
            raise GateError("E-GATE-UNSUPPORTED", f"{c} inside a kernel")


def _first(v):
    return int(np.asarray(v).reshape(-1)[0])


def _binop(op, a, b):
    if not isinstance(a, np.ndarray) and not isinstance(b, np.ndarray):
        if op == "/":
            return int(a / b) if b else 0
        if op == "%":
            return 0 if b == 0 else a - int(a / b) * b
    a = np.asarray(a)
    b = np.asarray(b)
    if op == "+":
        return a + b
    if op == "-":
        return a - b
    if op == "*":
        return a * b
    if op in ("/", "%"):
        bz = b == 0
        q = np.where(bz, 0, np.trunc(a / np.where(bz, 1, b))).astype(np.int64)
        return q if op == "/" else np.where(bz, 0, a - q * b)
    return {"==": np.equal, "!=": np.not_equal, "<": np.less, "<=": np.less_equal,
            ">": np.greater, ">=": np.greater_equal}[op](a, b)


def _check_conflicts(log, what, per_block):
    """E-DESYNC if an address written by one thread is touched by another."""
    by = {}
    for ent in log:
        by.setdefault(ent[0], []).append(ent)
    for name, ents in by.items():
        if not any(e[3] for e in ents):
            continue
        addr = np.concatenate([e[1] for e in ents])
        tid = np.concatenate([np.broadcast_to(e[2], e[1].shape) for e in ents])
        w = np.concatenate([np.full(e[1].shape, e[3]) for e in ents])
        order = np.argsort(addr, kind="stable")
        sa, st, sw = addr[order], tid[order], w[order]
        starts = np.concatenate(([0], np.flatnonzero(np.diff(sa)) + 1))
        tmin = np.minimum.reduceat(st, starts)
        tmax = np.maximum.reduceat(st, starts)
        wr = np.add.reduceat(sw.astype(np.int64), starts) > 0
        bad = wr & (tmin != tmax)
        if bad.any():
            g = int(np.flatnonzero(bad)[0])
            scope = "thread of the block without a barrier in between" if per_block else \
                "thread of the same launch (there is no grid-wide barrier)"
            raise GateError("E-DESYNC", f"{what} cell of {name!r} written by thread {int(tmin[g])} is "
                                        f"accessed by thread {int(tmax[g])}: another {scope}")


def check_kernels(program, entry: str, inputs: dict) -> dict:
    """Run the device-side gate on every kernel scope of `entry` for these inputs.
    Returns {"kernels": k, "blocks": analysed blocks}; raises GateError."""
    fn = program.fn(entry)
    env = {}
    arrays = {}
    dims = {}
    for pname, ptype in fn.params:
        if ptype.endswith("*"):
            arrays[pname] = "global"
            v = inputs.get(pname)
            if hasattr(v, "dims"):
                dims[pname] = list(v.dims)
            elif v is not None and hasattr(v, "__len__"):
                dims[pname] = [len(v)]
        elif pname in inputs:
            env[pname] = inputs[pname]
    report = {"kernels": 0, "blocks": 0}

    def host(stmts, env):
        for s in stmts:
            c = _cls(s)
            if c == "Seq":
                if _is_kernel_scope(s):
                    kernel(s, env)
                else:
                    host(_stmts(s), dict(env))
            elif c == "Decl":
                if s.alloc is not None:
                    arrays[s.name] = "global"
                    try:
                        dims[s.name] = [_host_eval(d, env) for d in s.dims]
                    except GateError:
                        dims.pop(s.name, None)
                elif s.init is not None:
                    try:
                        env[s.name] = _host_eval(s.init, env)
                    except GateError:
                        env.pop(s.name, None)
            elif c in ("For", "If"):
                if _has_kernel(s):
                    raise GateError("E-GATE-UNSUPPORTED", "kernel launch under host control flow")

    def kernel(seq, env):
        st = [x for x in _stmts(seq) if not (_cls(x) == "CallStmt" and x.ghost)]
        bpg, tpb = _host_eval(st[0].args[0], env), _host_eval(st[0].args[1], env)
        # shared-memory accounting (checker.py:298-318, intrinsics.py:70-84): the
        # launch's smem_sz is an allowance each __smem_malloc consumes (4-byte
        # cells, intrinsics.py:35); kernel_setup_end needs it used up exactly
        allowance = _host_eval(st[0].args[2], env) if len(st[0].args) > 2 else 0
        arr = dict(arrays)
        kd = dict(dims)
        body = []
        for x in st[1:]:
            if _cls(x) == "CallStmt" and x.fn == "kernel_setup_end" and allowance != 0:
                raise GateError("E-SMEM", f"kernel_setup_end needs the whole shared-memory allowance "
                                          f"allocated: {allowance} bytes left")
            if _cls(x) == "Decl" and x.alloc in ("__smem_malloc", "__treg_malloc"):
                arr[x.name] = "smem" if x.alloc == "__smem_malloc" else "treg"
                kd[x.name] = [_host_eval(d, env) for d in x.dims]
                if x.alloc == "__smem_malloc":
                    nbytes = 4
                    for d in kd[x.name]:
                        nbytes *= d
                    allowance -= nbytes
                    if allowance < 0:
                        raise GateError("E-SMEM", f"shared memory over-allocation: remaining allowance "
                                                  f"{allowance} is negative")
            elif _cls(x) == "CallStmt" and (x.fn.startswith("__smem_free") or x.fn in ("kernel_kill",)):
                continue
            else:
                body.append(x)
        g = _KernelGate(env, arr, bpg, tpb, kd)
        g.run(body)
        report["kernels"] += 1
        report["blocks"] += g.blocks

    host(_stmts(fn.body), env)
    return report


def _has_kernel(s):
    c = _cls(s)
    if c == "Seq":
        return _is_kernel_scope(s) or any(_has_kernel(x) for x in _stmts(s))
    if c == "For":
        return _has_kernel(s.body)
    if c == "If":
        return _has_kernel(s.then) or (s.els is not None and _has_kernel(s.els))
    return False


def _host_eval(e, env):
    g = _KernelGate(env, {}, 1, 1, {})
    v = g.eval(e, env, None)
    if v is DATA or isinstance(v, np.ndarray):
        raise GateError("E-GATE-DATA", "a launch parameter depends on array contents")
    return v


def run_check(check, program, entry, inputs):
    """The `check=` argument of run_program."""
    if check is None:
        return None
    if callable(check):
        return check(program)
    if check == "kernels":
        return check_kernels(program, entry, inputs)
    raise ValueError(f"check must be None, 'kernels' or a callable, not {check!r}")


__all__ = ["GateError", "check_kernels", "run_check", "MAX_BLOCKS"]
