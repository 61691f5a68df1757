"""CUDA code generation for GPU-form OptiGPU programs.

The reference specifies this module but does not ship it (
PAPER.md:1017-1084 describe it): every `kernel_launch ... kernel_kill` scope
becomes a `__global__` function, `thread for` nests become index arithmetic on
the global thread id, `__smem_malloc` becomes (dynamic) shared memory, the
`DMINDEX` block index of shared/thread-register arrays becomes 0, `blocksync()`
becomes `__syncthreads()`, and the host part (gmem_malloc / memcpy / host
loops / return) becomes native host code. The translation unit is compiled with
nvcc for sm_100a into a shared object and called through a tiny C ABI.

Semantics kept identical to the reference interpreter (minigpu/interp.py):
  * float cells are binary32; every expression is evaluated in binary64 and
    rounded to binary32 only when stored into a float cell (interp.py:43-44,
    :262-270, :83-84); FMA contraction is disabled (host and device), so the
    arithmetic is the interpreter's bit for bit;
  * int cells and int scalars are int64 (the reference's Python ints never wrap;
    programs whose values leave the int64 range diverge);
  * `/` is exact_div (raises unless exact), raw `/` `%` truncate (interp.py:187-214),
    pow2, DMINDEX (interp.py:215-227);
  * `thread for` narrows the context width like interp.py:285-299; a statement
    that writes memory in a context wider than one thread runs once (thread 0 of
    the context), as the interpreter runs it once;
  * array accesses are bounds- and rank-checked on host and device (violations
    raise InterpError after the kernel instead of faulting); host arrays track
    initialisation (reads / memcpys of uninitialised cells raise) and
    use-after-free.
Device-side gmem cells are not tracked for initialisation (documented deviation).

Only programs that contain at least one kernel scope are compiled: host code is
part of such a program (e.g. A.5's final host loop), while a program with no
kernel is not a GPU program and is refused (no CPU fallback).
"""
from __future__ import annotations

import contextlib
import ctypes
import hashlib
import os
import struct
import subprocess
import threading

import numpy as np

from .errors import InterpError, UnsupportedProgram

PKG = os.path.dirname(os.path.abspath(__file__))
GEN_DIR = os.path.join(PKG, "progcache")  # compiled generated programs (git-ignored)
MAX_RANK = 8

# ----------------------------------------------------------------------------- helpers


def _cls(x) -> str:
    return type(x).__name__


def _is_const(e) -> bool:
    """Integer expression built from literals only."""
    c = _cls(e)
    if c == "IntLit":
        return True
    if c == "BinOp":
        return _is_const(e.lhs) and _is_const(e.rhs)
    return False


def _ast_eq(a, b) -> bool:
    """Structural equality of index expressions (works for either parser's nodes)."""
    ca, cb = _cls(a), _cls(b)
    if ca != cb:
        return False
    if ca in ("IntLit", "FloatLit"):
        return a.value == b.value
    if ca == "Var":
        return a.name == b.name
    if ca == "BinOp":
        return a.op == b.op and _ast_eq(a.lhs, b.lhs) and _ast_eq(a.rhs, b.rhs)
    if ca == "Call":
        return a.fn == b.fn and len(a.args) == len(b.args) and all(_ast_eq(x, y) for x, y in zip(a.args, b.args))
    if ca in ("Access", "Ptr"):
        return a.base == b.base and len(a.idxs) == len(b.idxs) and all(_ast_eq(x, y) for x, y in zip(a.idxs, b.idxs))
    return False


def _even(e) -> bool:
    """The integer expression is even for every value of its variables: an even
    literal, a product with an even factor, a sum / difference of even terms."""
    c = _cls(e)
    if c == "IntLit":
        return int(e.value) % 2 == 0
    if c == "BinOp":
        if e.op == "*":
            return _even(e.lhs) or _even(e.rhs)
        if e.op in ("+", "-"):
            return _even(e.lhs) and _even(e.rhs)
    return False


def _plus_one(hi, lo) -> bool:
    """hi is literally `lo + 1`."""
    return (_cls(hi) == "BinOp" and hi.op == "+" and _cls(hi.rhs) == "IntLit" and int(hi.rhs.value) == 1
            and _ast_eq(hi.lhs, lo))


def _is_ghost(s) -> bool:
    return _cls(s) == "CallStmt" and getattr(s, "ghost", False)


def _stmts(seq):
    return [s for s in seq.stmts if not _is_ghost(s)]


def _f32_literal(v: float) -> str:
    f = struct.unpack("f", struct.pack("f", float(v)))[0]
    if f != f or f in (float("inf"), float("-inf")):
        raise UnsupportedProgram(f"non-finite float literal {v}")
    return f"({f.hex()})"


def _is_kernel_scope(s) -> bool:
    if _cls(s) != "Seq":
        return False
    st = _stmts(s)
    return bool(st) and _cls(st[0]) == "CallStmt" and st[0].fn == "kernel_launch"


def has_kernel(fn) -> bool:
    def walk(s):
        if _is_kernel_scope(s):
            return True
        c = _cls(s)
        if c == "Seq":
            return any(walk(t) for t in s.stmts)
        if c == "For":
            return walk(s.body)
        if c == "If":
            return walk(s.then) or (s.els is not None and walk(s.els))
        return False
    return fn.body is not None and walk(fn.body)


# kernel instantiations: <B2CK, B2CO (program threads per CUDA thread), B2PK (program
# blocks per CUDA block), B2IX (index type)>. Packing (B2PK = 2, with twice the base
# coarsening factor) only exists in 32-bit index arithmetic.
_VARIANTS = {"int32_t": ((1, 1), (2, 1), (4, 1), (4, 2), (8, 2)),
             "int64_t": ((1, 1), (2, 1), (4, 1))}
_INSTANCES = ("true, 1, 1, int64_t",) + tuple(f"false, {c}, {p}, {ity}" for ity, vs in _VARIANTS.items()
                                             for c, p in vs)


def _launch_switch(name, pv, ix32, co, pk, grid, t, smem, stream, args):
    """Host lines launching the instantiation chosen at run time: the checked one
    unless proved; proved launches coarsened by `co`, `pk` program blocks per CUDA
    block (when the launch's block count divides by it; else unpacked at the base
    factor co / pk) and in 32-bit
    index arithmetic when `ix32` (the proof bounded every integer below 2^31)."""
    L = [f"{{ const unsigned _gb = {grid};",
         f"  const int _pk = (_gb % (unsigned){pk} == 0u) ? {pk} : 1;",
         f"  const int _co = (_pk == {pk}) ? {co} : {co} / {pk};"]
    first = True
    for ity, vs in _VARIANTS.items():
        for c, p in vs:
            cond = f"{pv} && _co == {c} && _pk == {p} && {'' if ity == 'int32_t' else '!'}{ix32}"
            L.append(f"  {'if' if first else 'else if'} ({cond}) {name}<false, {c}, {p}, {ity}><<<_gb / {p}u, "
                     f"(unsigned)({p} * {t} / {c}), (size_t)({p} * {smem}), {stream}>>>({args});")
            first = False
    L.append(f"  else {name}<true, 1, 1, int64_t><<<_gb, (unsigned){t}, (size_t){smem}, {stream}>>>({args}); }}")
    return L


class Seq_like:
    """A statement list viewed as a Seq (for _rw_sets)."""

    def __init__(self, stmts):
        self.stmts = list(stmts)


def _block_level(kbody):
    """(For node, depth) of the kernel's block level: follow the chain of thread-fors
    that are the only statement of their enclosing body, from the kernel body down;
    the last one is where the program's blocks are (None if the kernel does not open
    with such a chain)."""
    stmts = [x for x in kbody if not _is_ghost(x)]
    node, depth = None, 0
    while len(stmts) == 1 and _cls(stmts[0]) == "For" and stmts[0].mode in ("thread", "magic_thread"):
        node, depth = stmts[0], depth + 1
        stmts = [x for x in node.body.stmts if not _is_ghost(x)]
    return node, depth


def _rw_sets(scope):
    """Names read / assigned (as arrays or scalars) anywhere inside a statement tree."""
    reads, writes = set(), set()

    def ex(e):
        c = _cls(e)
        if c == "Var":
            reads.add(e.name)
        elif c == "Access":
            reads.add(e.base)
            for x in e.idxs:
                ex(x)
        elif c == "BinOp":
            ex(e.lhs)
            ex(e.rhs)
        elif c == "Call":
            for x in e.args:
                ex(x)
        elif c == "Ptr":
            for x in getattr(e, "idxs", []):
                ex(x)

    def walk(st):
        c = _cls(st)
        if c == "Seq":
            for x in st.stmts:
                walk(x)
        elif c == "Assign":
            writes.add(st.target.base)
            if st.op == "+=":
                reads.add(st.target.base)
            for x in st.target.idxs:
                ex(x)
            ex(st.value)
        elif c == "Decl":
            if getattr(st, "init", None) is not None:
                ex(st.init)
            for x in getattr(st, "dims", None) or []:
                ex(x)
        elif c == "For":
            ex(st.range.start)
            ex(st.range.stop)
            walk(st.body)
        elif c == "If":
            ex(st.cond)
            walk(st.then)
            if st.els is not None:
                walk(st.els)
        elif c == "CallStmt":
            for x in st.args:
                ex(x)
        elif c == "Return":
            ex(st.value)
    walk(scope)
    return reads, writes


class Sym:
    """A named thing in the program: scalar or array, where it lives."""

    def __init__(self, name, kind, ctype, rank=0, index=None):
        self.name = name
        self.kind = kind        # param_arr | param_int | param_float | scalar | host_arr | dev_arr | smem_arr | treg_arr
        self.ctype = ctype      # "float" | "int"
        self.rank = rank        # declared rank (arrays; smem/treg without the block dim)
        self.index = index      # parameter position for params
        self.cname = "v_" + name
        self.loop = False       # a for / thread-for index: not assignable (interp.py:271-272)

    @property
    def is_array(self):
        return self.kind.endswith("arr")

    @property
    def elem(self):
        # int cells hold the reference's unbounded Python ints: int64 (not the
        # 4-byte CELL_BYTES of the proof model) so in-kernel sums never wrap
        return "float" if self.ctype == "float" else "int64_t"


# ----------------------------------------------------------------------------- C++ prelude

PRELUDE = r"""
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <string>
#include <vector>

struct B2Arr { void *data; int64_t n; int64_t rank; int64_t dims[8]; uint8_t *init; int64_t freed; };
struct B2Err { std::string msg; };
static inline void b2_throw(const std::string &m) { throw B2Err{m}; }

// device-side error flags (first error wins)
enum { B2E_OOB = 1, B2E_RANK = 2, B2E_DIV = 3, B2E_WIDTH = 4 };
__device__ __forceinline__ void b2_flag(int *f, int code, int64_t a, int64_t b) {
    if (atomicCAS(f, 0, code) == 0) { f[1] = (int)a; f[2] = (int)b; f[3] = (int)(a >> 32); f[4] = (int)(b >> 32); }
}
// integer helpers in the operands' common type: int64_t on the host and in checked
// kernels, int32_t in check-free kernels whose launch-time proof bounded every
// integer expression below 2^31 (then no intermediate can overflow)
template <typename A, typename B> __host__ __device__ __forceinline__ auto b2_div(A a, B b) -> decltype(a / b) {
    return b ? a / b : 0;
}
template <typename A, typename B> __host__ __device__ __forceinline__ auto b2_mod(A a, B b) -> decltype(a % b) {
    return b ? a - (a / b) * b : 0;
}
template <typename I> __host__ __device__ __forceinline__ I b2_pow2(I k) { return k < 0 ? 0 : ((I)1 << k); }
static inline int64_t b2_exact_div_h(int64_t a, int64_t b) {
    if (b == 0 || a % b != 0) b2_throw("exact_div(" + std::to_string(a) + ", " + std::to_string(b) + ") is not exact");
    return a / b;
}
template <typename A, typename B> __device__ __forceinline__ auto b2_exact_div_d(A a, B b, int *f) -> decltype(a / b) {
    if (b == 0 || a % b != 0) { b2_flag(f, B2E_DIV, a, b); return 0; }
    return a / b;
}
// host element offset with the interpreter's checks (Array.offset, interp.py:61-70)
static inline int64_t b2_off_h(const int64_t *dims, int64_t rank, int64_t nidx, const int64_t *idx) {
    if (nidx == rank + 1 && rank == 1) {  // pointer-offset rule (interp.py:239-240)
        int64_t ix = idx[0] + idx[1];
        if (ix < 0 || ix >= dims[0]) b2_throw("index " + std::to_string(ix) + " out of bounds 0.." + std::to_string(dims[0]));
        return ix;
    }
    if (nidx != rank) b2_throw("rank mismatch: " + std::to_string(nidx) + " indices into " + std::to_string(rank) + "-d array");
    int64_t off = 0;
    for (int64_t i = 0; i < rank; ++i) {
        if (idx[i] < 0 || idx[i] >= dims[i]) b2_throw("index " + std::to_string(idx[i]) + " out of bounds 0.." + std::to_string(dims[i]));
        off = off * dims[i] + idx[i];
    }
    return off;
}
__device__ __forceinline__ bool b2_chk(int64_t ix, int64_t d, int *f) {
    if (ix < 0 || ix >= d) { b2_flag(f, B2E_OOB, ix, d); return false; }
    return true;
}
// kernels are templates on B2CK: the checked instantiation is the interpreter's
// semantics; the unchecked one is launched only when the host has proved, for this
// concrete launch, that every access is in bounds (b2i_* below), so the checks
// could never fire
#define B2_CHK(ix, d) (!B2CK || b2_chk((ix), (d), b2_err))
// launch-time bounds proofs: interval evaluation of a kernel's index expressions
// over its loop ranges (values kept within +-2^62 so the arithmetic cannot wrap);
// anything not provable (data-dependent indices, reassigned locals, inexact
// exact_div, non-constant divisors) abandons the proof -> checked kernel
struct B2NoProof {};
struct B2I { int64_t lo, hi; };
static const int64_t B2I_BIG = (int64_t)1 << 62;
// largest |bound| of any interval the current proof produced: < 2^31 lets the
// check-free kernel run with 32-bit integer arithmetic (B2IX = int32_t)
static int64_t b2i_maxabs = 0;
static inline B2I b2i_t(B2I x) {
    const int64_t m = std::max(x.lo < 0 ? -x.lo : x.lo, x.hi < 0 ? -x.hi : x.hi);
    if (m > b2i_maxabs) b2i_maxabs = m;
    return x;
}
static inline B2I b2i_fit(__int128 lo, __int128 hi) {
    if (lo < -(__int128)B2I_BIG || hi > (__int128)B2I_BIG) throw B2NoProof{};
    return b2i_t(B2I{(int64_t)lo, (int64_t)hi});
}
static inline B2I b2i_c(int64_t v) { return b2i_fit(v, v); }
static inline B2I b2i_unknown() { throw B2NoProof{}; }
static inline B2I b2i_add(B2I a, B2I b) { return b2i_fit((__int128)a.lo + b.lo, (__int128)a.hi + b.hi); }
static inline B2I b2i_sub(B2I a, B2I b) { return b2i_fit((__int128)a.lo - b.hi, (__int128)a.hi - b.lo); }
static inline B2I b2i_mul(B2I a, B2I b) {
    __int128 c[4] = {(__int128)a.lo * b.lo, (__int128)a.lo * b.hi, (__int128)a.hi * b.lo, (__int128)a.hi * b.hi};
    __int128 lo = c[0], hi = c[0];
    for (int i = 1; i < 4; ++i) { lo = c[i] < lo ? c[i] : lo; hi = c[i] > hi ? c[i] : hi; }
    return b2i_fit(lo, hi);
}
static inline B2I b2i_div(B2I a, B2I b) {  // truncating, non-negative dividend, constant positive divisor
    if (b.lo != b.hi || b.lo <= 0 || a.lo < 0) throw B2NoProof{};
    return b2i_t(B2I{a.lo / b.lo, a.hi / b.lo});
}
static inline B2I b2i_mod(B2I a, B2I b) {
    if (b.lo != b.hi || b.lo <= 0 || a.lo < 0) throw B2NoProof{};
    return b2i_t(a.hi < b.lo ? a : B2I{0, b.lo - 1});
}
static inline B2I b2i_exact_div(B2I a, B2I b) {
    if (b.lo != b.hi || b.lo <= 0) throw B2NoProof{};
    if (a.lo == a.hi && a.lo % b.lo != 0) throw B2NoProof{};  // the kernel will raise: keep its checks
    auto fl = [](int64_t x, int64_t d) { return x >= 0 ? x / d : -((-x + d - 1) / d); };
    return b2i_t(B2I{fl(a.lo, b.lo), fl(a.hi, b.lo)});
}
static inline B2I b2i_pow2(B2I k) {  // monotonic: [2^lo, 2^hi]
    if (k.lo < 0 || k.hi > 61) throw B2NoProof{};
    return b2i_t(B2I{(int64_t)1 << k.lo, (int64_t)1 << k.hi});
}
static inline B2I b2i_join(B2I a, B2I b) { return B2I{a.lo < b.lo ? a.lo : b.lo, a.hi > b.hi ? a.hi : b.hi}; }
static inline int b2i_in(B2I ix, int64_t d) {  // every value of ix indexes [0, d)
    if (ix.lo < 0 || ix.hi >= d) throw B2NoProof{};
    return 0;
}
template <typename T> struct B2Host { T *p = nullptr; int64_t n = 0; int64_t rank = 0; int64_t dims[8] = {0}; uint8_t *init = nullptr; bool freed = false; bool owned = false; };
template <typename T> struct B2Dev { T *p = nullptr; int64_t n = 0; int64_t rank = 0; int64_t dims[8] = {0}; bool freed = false; };
// kernel-only device time of the last launch of each kernel (PAPER.md:1100-1102
// measures generated kernels this way: host copies excluded)
static float b2_kernel_ms[64];
static cudaEvent_t b2_ev0, b2_ev1;
extern "C" double b2g_kernel_ms(int k) { return (k >= 0 && k < 64) ? b2_kernel_ms[k] : -1.0; }
// which instantiation each kernel's last launch used (1 = bounds proved, checks elided)
static int b2_kernel_unchecked[64];
extern "C" int b2g_kernel_unchecked(int k) { return (k >= 0 && k < 64) ? b2_kernel_unchecked[k] : -1; }
static bool b2_prove_enabled() { const char *e = getenv("B2K_CODEGEN_PROVE"); return !(e && e[0] == '0'); }
// Host runtime services from libb200k.so (include/b2k.h): staged / pinned bulk
// copies, the caching device allocator, and the device this call runs on.
typedef struct { void *host; int64_t host_pitch; void *dev; int64_t dev_pitch; int64_t width; int64_t height; } b2_copy2d;
typedef int (*b2_step_fn)(void *, int, void *);
struct B2Ops {
    int (*h2d)(void *, const void *, size_t, int);
    int (*d2h)(void *, const void *, size_t, int);
    const char *(*last_error)(void);
    int (*alloc)(size_t, int, void **);
    int (*dfree)(void *, int);
    int64_t dev;
    int (*pipe)(int, const b2_copy2d *, const int64_t *, const b2_copy2d *, const int64_t *, b2_step_fn, void *, int);
    int64_t pipe_chunk;  // target bytes per pipeline step (0: pipelining off)
    int64_t coarsen;     // largest thread-coarsening factor for check-free launches (1: off)
    int64_t pack;        // most program blocks per CUDA block for check-free launches (1: off)
};
static const B2Ops *g_ops;
static std::vector<void *> *g_dev_allocs;
static std::vector<void *> *g_host_allocs;
template <typename T> static B2Dev<T> b2_dev_alloc(int64_t rank, std::initializer_list<int64_t> d) {
    B2Dev<T> a; a.rank = rank; a.n = 1; int i = 0;
    for (int64_t x : d) { a.dims[i++] = x; a.n *= x; }
    if (a.n < 0) a.n = 0;
    if (a.n > 0) {
        if (g_ops->alloc((size_t)a.n * sizeof(T), (int)g_ops->dev, (void **)&a.p))
            b2_throw(std::string("gmem_malloc: ") + g_ops->last_error());
        g_dev_allocs->push_back(a.p);
    }
    return a;
}
template <typename T> static B2Host<T> b2_host_alloc(int64_t rank, std::initializer_list<int64_t> d) {
    B2Host<T> a; a.rank = rank; a.n = 1; int i = 0;
    for (int64_t x : d) { a.dims[i++] = x; a.n *= x; }
    if (a.n < 0) a.n = 0;
    a.p = (T *)calloc((size_t)(a.n > 0 ? a.n : 1), sizeof(T));
    a.init = (uint8_t *)calloc((size_t)(a.n > 0 ? a.n : 1), 1);
    a.owned = true;
    g_host_allocs->push_back(a.p); g_host_allocs->push_back(a.init);
    return a;
}
template <typename T> static B2Host<T> b2_param(B2Arr *A) {
    B2Host<T> a; a.p = (T *)A->data; a.n = A->n; a.rank = A->rank;
    for (int i = 0; i < 8; ++i) a.dims[i] = A->dims[i];
    a.init = A->init; a.freed = A->freed != 0; return a;
}
// host element access with the interpreter's checks; the 1-D case (host loops over
// partials, A.5's `sum += p[i]`) takes an inlined fast path
static inline int64_t b2_off_h1(const int64_t *dims, int64_t rank, int64_t nidx, const int64_t *idx) {
    if (__builtin_expect(nidx == 1 && rank == 1 && idx[0] >= 0 && idx[0] < dims[0], 1)) return idx[0];
    return b2_off_h(dims, rank, nidx, idx);
}
template <typename T> static inline T b2_hread(B2Host<T> &a, int64_t nidx, const int64_t *idx) {
    if (a.freed) b2_throw("use after free");
    int64_t o = b2_off_h1(a.dims, a.rank, nidx, idx);
    if (a.init && !a.init[o]) b2_throw("read of uninitialized cell");
    return a.p[o];
}
template <typename T> static inline void b2_hwrite(B2Host<T> &a, int64_t nidx, const int64_t *idx, T v) {
    if (a.freed) b2_throw("use after free");
    int64_t o = b2_off_h1(a.dims, a.rank, nidx, idx);
    a.p[o] = v;
    if (a.init) a.init[o] = 1;
}
template <typename T, typename S> static void b2_h2d(B2Dev<T> &d, B2Host<S> &s, int64_t n) {
    static_assert(sizeof(T) == sizeof(S), "memcpy between different cell types");
    if (d.freed || s.freed) b2_throw("use after free");
    if (n <= 0) return;
    if (n > s.n || n > d.n) b2_throw("list index out of range");
    if (s.init) for (int64_t i = 0; i < n; ++i) if (!s.init[i]) b2_throw("memcpy of uninitialized data");
    if (g_ops->h2d(d.p, s.p, (size_t)n * sizeof(T), (int)g_ops->dev))
        b2_throw(std::string("memcpy_host_to_device: ") + g_ops->last_error());
}
template <typename T, typename S> static void b2_d2h(B2Host<T> &d, B2Dev<S> &s, int64_t n) {
    static_assert(sizeof(T) == sizeof(S), "memcpy between different cell types");
    if (d.freed || s.freed) b2_throw("use after free");
    if (n <= 0) return;
    if (n > s.n || n > d.n) b2_throw("list index out of range");
    if (g_ops->d2h(d.p, s.p, (size_t)n * sizeof(T), (int)g_ops->dev))
        b2_throw(std::string("memcpy_device_to_host: ") + g_ops->last_error());
    if (d.init) memset(d.init, 1, (size_t)n);
}
// ---- chunked copy -> kernel -> copy pipelines (b2_pipe_run, SURVEY 8f rank 2)
// A window `memcpy_host_to_device(d_i, h_i, n) ... kernel ... memcpy_device_to_host(h_o,
// d_o, n)` of full-array copies runs as C block-range chunks: the footprint proof of
// each chunk names the slab of every input it reads (copied just before it, never
// twice) and of every output it writes (copied right after it); cells no chunk
// writes are copied after the last one. Only proved (check-free) launches qualify.
static int b2_kernel_piped[64];
static int b2_kernel_coarsen[64];
static int b2_kernel_pack[64];
extern "C" int b2g_kernel_pack(int k) { return (k >= 0 && k < 64) ? b2_kernel_pack[k] : -1; }
static int b2_kernel_ix32[64];
extern "C" int b2g_kernel_ix32(int k) { return (k >= 0 && k < 64) ? b2_kernel_ix32[k] : -1; }
static bool b2_ix32_enabled() { const char *e = getenv("B2K_CODEGEN_IX32"); return !(e && e[0] == '0'); }
extern "C" int b2g_kernel_coarsen(int k) { return (k >= 0 && k < 64) ? b2_kernel_coarsen[k] : -1; }
// Thread coarsening / block packing of a check-free launch (tpb program threads and
// smem bytes of shared memory per program block): c program threads per CUDA thread,
// p program blocks per CUDA block of p * tpb / c threads. The base factor c (4 or 2)
// is the largest that keeps whole warps and a full SM's worth of CUDA threads (2048)
// resident: <= 32 blocks and their shared memory within 160 KB. Measured
// (profiles/r02h_codegen_coarsen.md): the 64x64-tile transpose (16.6 KB per block) at
// c = 4 could only keep 13 blocks = 1664 threads per SM and ran at 2.7 TB/s against
// 4.6 at c = 2. When that base configuration sits at the 32-blocks-per-SM cap (CUDA
// blocks of <= 64 threads: small program blocks such as A.5's), the cap, not the
// threads, limits the program blocks in flight; then two program blocks share one
// CUDA block at twice the factor (same block size, 2x the program blocks per SM: A.5
// 2.6 -> 3.0 TB/s, profiles/r02j_codegen_pack.md). 8-fold coarsening alone (A.4: 32
// program blocks per SM instead of 16) measured 4-7 % slower and is not used.
// Packing needs `packable` (no barrier under block-dependent control flow), an even
// block count and, like c = 8, 32-bit indices.
static void b2_pack_for(int64_t tpb, int64_t smem, int64_t grid, bool packable, bool ix32, int *co, int *pk) {
    *co = 1; *pk = 1;
    for (int c = 4; c > 1; c /= 2) {
        if (c > g_ops->coarsen || tpb % (32 * c) != 0) continue;
        const int64_t blocks = 2048 / (tpb / c);
        if (blocks <= 32 && blocks * smem <= 160 * 1024) { *co = c; break; }
    }
    const int64_t T = tpb / *co;
    if (*co > 1 && 2 * *co <= g_ops->coarsen && g_ops->pack >= 2 && packable && ix32 && grid % 2 == 0 &&
        2048 / T == 32 && 32 * 2 * smem <= 160 * 1024) {
        *co *= 2; *pk = 2;
    }
}
extern "C" int b2g_kernel_piped(int k) { return (k >= 0 && k < 64) ? b2_kernel_piped[k] : -1; }
static cudaEvent_t b2_pev[2][64];
static bool b2_pipe_on() { const char *e = getenv("B2K_CODEGEN_PIPE"); return !(e && e[0] == '0'); }
static bool b2_pipe_fn() { return g_ops->pipe && g_ops->pipe_chunk > 0; }
struct B2FP { int64_t lo[2][8][8], hi[2][8][8]; };  // [read, write][window slot][dim]
static inline void b2fp_init(B2FP &f) {
    for (int a = 0; a < 2; ++a) for (int b = 0; b < 8; ++b) for (int c = 0; c < 8; ++c) { f.lo[a][b][c] = INT64_MAX; f.hi[a][b][c] = INT64_MIN; }
}
static inline int b2fp_acc(B2FP &f, int rw, int slot, int k, B2I ix, int64_t d) {
    b2i_in(ix, d);
    for (int a = 0; a < 2; ++a) {
        if (!(rw == 2 || rw == a)) continue;
        if (ix.lo < f.lo[a][slot][k]) f.lo[a][slot][k] = ix.lo;
        if (ix.hi > f.hi[a][slot][k]) f.hi[a][slot][k] = ix.hi;
    }
    return 0;
}
struct B2PipeArr { char *host; char *dev; int64_t es; int64_t rank; int64_t dims[8]; int slot; bool in; };
template <typename T, typename S> static B2PipeArr b2_pipe_arr(B2Dev<T> &d, B2Host<S> &h, int slot, bool in) {
    B2PipeArr a; a.host = (char *)h.p; a.dev = (char *)d.p; a.es = sizeof(T); a.rank = d.rank > 0 ? d.rank : 1;
    for (int i = 0; i < 8; ++i) a.dims[i] = d.rank > 0 ? d.dims[i] : (i == 0 ? d.n : 1);
    a.slot = slot; a.in = in; return a;
}
// the copy qualifies: no error the sequential code could raise, the full arrays
template <typename T, typename S> static bool b2_pipe_ok(B2Dev<T> &d, B2Host<S> &h, int64_t n, bool in) {
    if (sizeof(T) != sizeof(S) || d.freed || h.freed || n <= 0 || n != d.n || n != h.n || !d.p || !h.p) return false;
    if (in && h.init) for (int64_t i = 0; i < n; ++i) if (!h.init[i]) return false;
    return true;
}
template <typename A, typename B> static bool b2_disjoint(B2Host<A> &a, B2Host<B> &b) {
    const char *a0 = (const char *)a.p, *a1 = a0 + a.n * sizeof(A), *b0 = (const char *)b.p, *b1 = b0 + b.n * sizeof(B);
    return a1 <= b0 || b1 <= a0;
}
// slab [x0, x1] of dimension p (all other dimensions full) as a 2-D copy region
static b2_copy2d b2_slab(const B2PipeArr &a, int p, int64_t x0, int64_t x1) {
    int64_t pre = 1, inner = 1;
    for (int i = 0; i < p; ++i) pre *= a.dims[i];
    for (int i = p + 1; i < a.rank; ++i) inner *= a.dims[i];
    const int64_t pitch = a.dims[p] * inner * a.es, off = x0 * inner * a.es;
    b2_copy2d c; c.host = a.host + off; c.dev = a.dev + off; c.host_pitch = c.dev_pitch = pitch;
    c.width = (x1 - x0 + 1) * inner * a.es; c.height = pre;
    if (pre == 1) c.host_pitch = c.dev_pitch = c.width;
    return c;
}
// a footprint box as one slab: the single dimension that is not full (or dim 0)
static bool b2_box_slab(const B2PipeArr &a, const int64_t *lo, const int64_t *hi, int &p, int64_t &x0, int64_t &x1) {
    if (lo[0] > hi[0]) return false;  // not accessed
    p = -1;
    for (int i = 0; i < a.rank; ++i) {
        if (lo[i] > 0 || hi[i] < a.dims[i] - 1) {
            if (p >= 0) { p = 0; x0 = 0; x1 = a.dims[0] - 1; return true; }  // several partial dims: whole array
            p = i; x0 = lo[i]; x1 = hi[i];
        }
    }
    if (p < 0) { p = 0; x0 = 0; x1 = a.dims[0] - 1; }
    return true;
}
struct B2Plan {
    int nchunk = 0;
    std::vector<int64_t> bnd;  // block bounds, nchunk + 1
    std::vector<b2_copy2d> h2d, d2h;
    std::vector<int64_t> h2d_off, d2h_off;
};
template <class FPF> static bool b2_plan(int64_t G, int64_t align, const std::vector<B2PipeArr> &arrs, FPF &fpf, B2Plan &pl) {
    int64_t bytes = 0;
    for (auto &a : arrs) { int64_t n = 1; for (int i = 0; i < a.rank; ++i) n *= a.dims[i]; bytes += n * a.es; }
    if (align < 1) align = 1;
    const int64_t units = (G + align - 1) / align;
    int64_t C = std::min<int64_t>(std::min<int64_t>(64, units), bytes / std::max<int64_t>(1, g_ops->pipe_chunk));
    if (C < 2) return false;
    pl.nchunk = (int)C;
    pl.bnd.resize(C + 1);
    for (int64_t c = 0; c <= C; ++c) pl.bnd[c] = std::min(G, (c * units / C) * align);
    std::vector<std::vector<b2_copy2d>> hc(C), dc(C);
    const size_t na = arrs.size();
    std::vector<int> pdim(na, -1);
    std::vector<int64_t> hi_done(na, -1);
    std::vector<bool> banded(na, true);
    std::vector<std::vector<std::pair<int64_t, int64_t>>> bands(na);
    for (int64_t c = 0; c < C; ++c) {
        B2FP fp; b2fp_init(fp);
        fpf(pl.bnd[c], pl.bnd[c + 1], fp);
        for (size_t k = 0; k < na; ++k) {
            const B2PipeArr &a = arrs[k];
            int p; int64_t x0, x1;
            if (a.in) {  // the slab this chunk reads, minus what earlier chunks already copied
                if (!b2_box_slab(a, fp.lo[0][a.slot], fp.hi[0][a.slot], p, x0, x1)) continue;
                if (pdim[k] < 0) pdim[k] = p;
                if (p != pdim[k]) { x0 = 0; x1 = a.dims[pdim[k]] - 1; }
                if (x1 > hi_done[k]) { hc[c].push_back(b2_slab(a, pdim[k], hi_done[k] + 1, x1)); hi_done[k] = x1; }
            } else if (banded[k]) {  // the slab this chunk writes, if disjoint from earlier ones
                if (!b2_box_slab(a, fp.lo[1][a.slot], fp.hi[1][a.slot], p, x0, x1)) continue;
                if (pdim[k] < 0) pdim[k] = p;
                if (p != pdim[k] || x0 <= hi_done[k]) { banded[k] = false; continue; }
                dc[c].push_back(b2_slab(a, p, x0, x1));
                bands[k].push_back({x0, x1});
                hi_done[k] = x1;
            }
        }
    }
    for (size_t k = 0; k < na; ++k) {  // the rest: after (inputs: before) the last chunk
        const B2PipeArr &a = arrs[k];
        const int p = pdim[k] < 0 ? 0 : pdim[k];
        if (a.in) {
            if (hi_done[k] < a.dims[p] - 1) hc[C - 1].push_back(b2_slab(a, p, hi_done[k] + 1, a.dims[p] - 1));
        } else if (!banded[k] || pdim[k] < 0) {
            dc[C - 1].push_back(b2_slab(a, 0, 0, a.dims[0] - 1));
        } else {
            int64_t nxt = 0;
            for (auto &b : bands[k]) { if (b.first > nxt) dc[C - 1].push_back(b2_slab(a, p, nxt, b.first - 1)); nxt = b.second + 1; }
            if (nxt <= a.dims[p] - 1) dc[C - 1].push_back(b2_slab(a, p, nxt, a.dims[p] - 1));
        }
    }
    pl.h2d_off.push_back(0); pl.d2h_off.push_back(0);
    for (int64_t c = 0; c < C; ++c) {
        for (auto &x : hc[c]) pl.h2d.push_back(x);
        for (auto &x : dc[c]) pl.d2h.push_back(x);
        pl.h2d_off.push_back((int64_t)pl.h2d.size()); pl.d2h_off.push_back((int64_t)pl.d2h.size());
    }
    return true;
}
template <class F> static int b2_tramp(void *ctx, int c, void *s) { return (*(F *)ctx)(c, (cudaStream_t)s); }
template <class F> static void b2_run_plan(B2Plan &pl, F &launch) {
    for (int c = 0; c < pl.nchunk && c < 64; ++c)
        if (!b2_pev[0][c]) { cudaEventCreate(&b2_pev[0][c]); cudaEventCreate(&b2_pev[1][c]); }
    if (g_ops->pipe(pl.nchunk, pl.h2d.data(), pl.h2d_off.data(), pl.d2h.data(), pl.d2h_off.data(), &b2_tramp<F>,
                    (void *)&launch, (int)g_ops->dev))
        b2_throw(std::string("pipelined copy / kernel: ") + g_ops->last_error());
}
static float b2_plan_ms(const B2Plan &pl) {  // kernel time: sum over the chunk launches
    float tot = 0;
    for (int c = 0; c < pl.nchunk && c < 64; ++c) {
        if (pl.bnd[c + 1] <= pl.bnd[c]) continue;
        float ms = 0; cudaEventElapsedTime(&ms, b2_pev[0][c], b2_pev[1][c]); tot += ms;
    }
    return tot;
}
static void b2_check_kernel(int *flags_dev, const char *name) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) b2_throw(std::string(name) + ": " + cudaGetErrorString(e));
    int f[5];
    cudaMemcpy(f, flags_dev, sizeof(f), cudaMemcpyDeviceToHost);
    if (f[0]) {
        int64_t a = (int64_t)(uint32_t)f[1] | ((int64_t)f[3] << 32), b = (int64_t)(uint32_t)f[2] | ((int64_t)f[4] << 32);
        if (f[0] == B2E_OOB) b2_throw("index " + std::to_string(a) + " out of bounds 0.." + std::to_string(b));
        if (f[0] == B2E_DIV) b2_throw("exact_div(" + std::to_string(a) + ", " + std::to_string(b) + ") is not exact");
        if (f[0] == B2E_WIDTH) b2_throw("thread for extent " + std::to_string(a) + " does not divide the context width " + std::to_string(b));
        b2_throw("device error");
    }
}
"""


# ----------------------------------------------------------------------------- generator


class _Gen:
    def __init__(self, fn):
        self.fn = fn
        self.syms: dict = {}
        self.kernels: list = []
        self.nk = 0
        self.tmp = 0
        self.params = []
        # binary64 code of ONE +, -, * of two binary32 values -> the same operation in
        # binary32 (see f32_op): what a float store of that code may emit instead
        self.f32ops: dict = {}
        for i, (pn, pt) in enumerate(fn.params):
            if pt.endswith("*"):
                s = Sym(pn, "param_arr", pt[:-1], index=i)
            else:
                s = Sym(pn, "param_int" if pt == "int" else "param_float", pt, index=i)
            self.syms[pn] = s
            self.params.append(s)

    def fresh(self, hint="t"):
        self.tmp += 1
        return f"_{hint}{self.tmp}"

    @contextlib.contextmanager
    def scope(self, kctx=None):
        """Block scoping of names (interp.py:248-249 pushes a frame per Seq): a
        declaration inside a block shadows the outer binding until the block ends."""
        syms = dict(self.syms)
        loc = set(kctx.local_syms) if kctx is not None else None
        try:
            yield
        finally:
            self.syms = syms
            if kctx is not None:
                kctx.local_syms = loc

    def sym(self, name):
        if name not in self.syms:
            raise UnsupportedProgram(f"unbound variable {name!r}")
        return self.syms[name]

    # ------------------------------------------------------------------ expressions
    def expr(self, e, dev=None):
        """-> (C code, type) with type in i (int64), f (binary32 value), d (double)."""
        c = _cls(e)
        if c == "IntLit":
            v = int(e.value)
            if dev is not None and -2**31 < v < 2**31:
                # kernel code: the index type of the instantiation (int32_t when the launch-time
                # proof bounds every integer expression of the kernel below 2^31, else int64_t);
                # array cell values stay int64_t and promote mixed expressions
                return f"((B2IX){v})", "i"
            return f"((int64_t){v}LL)", "i"
        if c == "FloatLit":
            return _f32_literal(e.value), "f"
        if c == "Var":
            s = self.sym(e.name)
            if s.is_array:
                raise UnsupportedProgram(f"array {e.name!r} used as a value")
            if s.kind == "param_float":
                return s.cname, "d"
            return s.cname, ("f" if s.ctype == "float" else "i")
        if c == "Access":
            return self.access_read(e.base, e.idxs, dev)
        if c == "BinOp":
            pair = self.cell_pair(e, dev)
            a, ta = self.expr(e.lhs, dev)
            b, tb = self.expr(e.rhs, dev)
            if pair is not None:
                a, b = pair(a, b)
            op = e.op
            if op in ("==", "!=", "<", "<=", ">", ">="):
                ity = "B2IX" if dev is not None else "int64_t"
                if ta == "i" and tb == "i":
                    return f"(({ity})({a} {op} {b}))", "i"
                return f"(({ity})((double)({a}) {op} (double)({b})))", "i"
            if ta == "i" and tb == "i":
                if op in ("+", "-", "*"):
                    return f"({a} {op} {b})", "i"
                if op == "/":
                    return f"b2_div({a}, {b})", "i"
                if op == "%":
                    return f"b2_mod({a}, {b})", "i"
            if op in ("+", "-", "*"):
                code = f"((double)({a}) {op} (double)({b}))"
                if ta == "f" and tb == "f":
                    self.f32_op(code, a, op, b, dev is not None)
                return code, "d"
            raise UnsupportedProgram(f"operator {op!r} on floating-point operands")
        if c == "Call":
            return self.call_expr(e, dev)
        raise UnsupportedProgram(f"cannot compile expression {c}")

    def call_expr(self, e, dev):
        if e.fn == "exact_div":
            a, ta = self.expr(e.args[0], dev)
            b, tb = self.expr(e.args[1], dev)
            if ta != "i" or tb != "i":
                raise UnsupportedProgram("exact_div on floating-point operands")
            if dev is None:
                return f"b2_exact_div_h({a}, {b})", "i"
            return f"b2_exact_div_d({a}, {b}, b2_err)", "i"
        if e.fn == "pow2":
            k, tk = self.expr(e.args[0], dev)
            return f"b2_pow2({k})", "i"
        if e.fn.startswith("DMINDEX"):
            k = len(e.args) // 2
            dims = [self.expr(a, dev)[0] for a in e.args[:k]]
            idxs = [self.expr(a, dev)[0] for a in e.args[k:]]
            out = "((B2IX)0)" if dev is not None else "((int64_t)0)"
            for d, ix in zip(dims, idxs):
                out = f"({out} * {d} + {ix})"
            return out, "i"
        raise UnsupportedProgram(f"cannot call {e.fn!r} in an expression")

    def int_expr(self, e, dev=None):
        code, t = self.expr(e, dev)
        if t != "i":
            raise UnsupportedProgram("integer expression expected")
        return code

    # ------------------------------------------------------------------ arrays
    def _indices(self, s, idxs, dev):
        idxs = list(idxs)
        if s.kind in ("smem_arr", "treg_arr"):
            # the interpreter prepends the block (thread) dimension; its index is
            # DMINDEX(...) of the current block, 0 in per-block storage
            if not idxs or _cls(idxs[0]) != "Call" or not idxs[0].fn.startswith("DMINDEX"):
                raise UnsupportedProgram(f"{s.name!r}: first index of a per-block array must be DMINDEX")
            idxs = idxs[1:]
        return [self.int_expr(i, dev) for i in idxs]

    def _dev_offset(self, s, codes):
        """Device offset with bounds checks; returns (ok_expr, off_expr, setup lines)."""
        dims = f"{s.cname}_dims"
        lines = []
        if len(codes) == s.rank + 1 and s.rank == 1:
            ix = self.fresh("ix")
            lines.append(f"const B2IX {ix} = {codes[0]} + {codes[1]};")
            return f"B2_CHK({ix}, {dims}[0])", ix, lines
        if len(codes) != s.rank:
            raise UnsupportedProgram(f"rank mismatch on {s.name!r}: {len(codes)} indices into {s.rank}-d array")
        ok, off = [], "((B2IX)0)"
        padded = s.kind == "smem_arr" and s.rank >= 2
        for k, cd in enumerate(codes):
            v = self.fresh("ix")
            lines.append(f"const B2IX {v} = {cd};")
            ok.append(f"B2_CHK({v}, {dims}[{k}])")
            # shared arrays: the last dimension is stored with a padded pitch
            stride = f"(B2IX){s.cname}_pitch" if (padded and k == s.rank - 1) else f"(B2IX){dims}[{k}]"
            off = f"({off} * {stride} + {v})"
        return "(" + " && ".join(ok or ["true"]) + ")", off, lines

    def access_read(self, base, idxs, dev):
        s = self.sym(base)
        if not s.is_array:
            raise UnsupportedProgram(f"{base!r} is not an array")
        t = "f" if s.ctype == "float" else "i"
        codes = self._indices(s, idxs, dev)
        if dev is None:
            if s.kind not in ("param_arr", "host_arr"):
                raise UnsupportedProgram(f"host code reads device/shared array {base!r}")
            arr = self.fresh("idx")
            self.pre.append(f"const int64_t {arr}[] = {{{', '.join(codes) or '0'}}};")
            return f"b2_hread({s.cname}, {len(codes)}, {arr})", t
        if s.kind not in ("dev_arr", "smem_arr", "treg_arr"):
            raise UnsupportedProgram(f"kernel reads host array {base!r}")
        dev.use(s)
        ok, off, lines = self._dev_offset(s, codes)
        self.pre.extend(lines)
        zero = "0.0f" if s.ctype == "float" else "0"
        return f"({ok} ? {s.cname}[{off}] : {zero})", t

    def cell_pair(self, e, dev):
        """Vector access (round 2): `d[i] op d[i + 1]` on a 1-D device array with i even
        for every value of its variables (a sum of even terms) reads both cells with one
        64-bit (float cells) / 128-bit (int64 cells) load in the check-free instantiation
        — the pair is aligned to its size (device allocations are 256-B aligned) and both
        cells are proved in bounds there.
        A.5's adjacent-pair load `d_a[b * 512 + 2 * t] + d_a[b * 512 + 2 * t + 1]` is
        the case. Returns a function rewriting the two scalar operand codes (evaluated
        only by the checked instantiation) or None."""
        if dev is None or e.op not in ("+", "-", "*") or _cls(e.lhs) != "Access" or _cls(e.rhs) != "Access":
            return None
        if e.lhs.base != e.rhs.base or len(e.lhs.idxs) != 1 or len(e.rhs.idxs) != 1:
            return None
        s = self.syms.get(e.lhs.base)
        if s is None or s.kind != "dev_arr" or s.rank != 1:
            return None
        i1, i2 = e.lhs.idxs[0], e.rhs.idxs[0]
        if _plus_one(i2, i1) and _even(i1):
            lo, first = i1, True
        elif _plus_one(i1, i2) and _even(i2):
            lo, first = i2, False
        else:
            return None
        (code,) = self._indices(s, [lo], dev)
        v = self.fresh("v2")
        # float cells: an 8-B float2; int cells (int64): a 16-B longlong2 (16-B aligned)
        vt, zero = ("float2", "make_float2(0.0f, 0.0f)") if s.ctype == "float" else \
            ("longlong2", "make_longlong2(0, 0)")
        self.pre.append(f"const {vt} {v} = B2CK ? {zero} : "
                        f"*reinterpret_cast<const {vt} *>({s.cname} + ({code}));")
        lo_c, hi_c = f"{v}.x", f"{v}.y"
        return lambda a, b: (f"(B2CK ? {a} : {lo_c if first else hi_c})", f"(B2CK ? {b} : {hi_c if first else lo_c})")

    def f32_op(self, code, a, op, b, device):
        """Record that the binary64 `code` is one +, -, * of the binary32 values a, b.
        The interpreter evaluates it in binary64 and rounds to binary32 at the store
        (interp.py:43-44, 83-84); with 53 >= 2 x 24 + 2 bits that double rounding is
        innocuous for a single +, -, * (the binary64 result rounded to binary32 is the
        correctly rounded binary32 result; products are even exact in binary64), so a
        float store of `code` may compute it directly in binary32: one FADD / FMUL
        instead of two F2F.F64, a DADD and an F2F back. __f*_rn never contract into
        FMAs; the host side is compiled with -ffp-contract=off."""
        if device:
            fn = {"+": "__fadd_rn", "-": "__fsub_rn", "*": "__fmul_rn"}[op]
            self.f32ops[code] = f"{fn}({a}, {b})"
        else:
            self.f32ops[code] = f"((float)({a}) {op} (float)({b}))"

    def plus_eq(self, s, old, val, t, device, icast):
        """`x += val` for the cell / scalar `old` of symbol s -> (code, type): int64 for
        int x and int val, else binary64 (interp.py:262-270), recorded as a binary32
        op when x is float and val a binary32 value."""
        if t == "i" and s.ctype == "int":
            return f"({icast}{old} + {val})", "i"
        code = f"((double){old} + (double)({val}))"
        if s.ctype == "float" and t == "f":
            self.f32_op(code, old, "+", val, device)
        return code, "d"

    def store_value(self, s, code, t):
        if s.ctype == "float":
            if t == "d" and code in self.f32ops:
                return self.f32ops[code]
            return f"(float)({code})" if t != "f" else code
        if t != "i":
            raise UnsupportedProgram("float value stored into an int cell")
        return code

    # ------------------------------------------------------------------ host statements
    def host_seq(self, seq, out, ind):
        stmts = _stmts(seq)
        i = 0
        while i < len(stmts):
            w = self._window(stmts, i)
            if w is None:
                self.host_stmt(stmts[i], out, ind)
                i += 1
                continue
            decls, h2d, k, d2h, end = w
            for d in decls:  # the window's gmem_mallocs first (no data effect)
                self.host_stmt(d, out, ind)
            self.pre = []
            self.kernel_scope(stmts[k], out, ind, window=(h2d, d2h))
            i = end

    @staticmethod
    def _is_copy(st, prefix):
        return (_cls(st) == "CallStmt" and st.fn.startswith(prefix) and len(st.args) >= 3
                and _cls(st.args[0]) == "Var" and _cls(st.args[1]) == "Var")

    def _window(self, stmts, i):
        """A pipelinable window starting at stmts[i]: full-array H2D copies (and
        gmem_mallocs), ONE kernel scope, then D2H copies, with every H2D'd device
        array only read by the kernel and every D2H'd one written by it (static
        read / write sets). -> (decls, h2d calls, kernel index, d2h calls, end) or None."""
        j, decls, h2d = i, [], []
        while j < len(stmts):
            st = stmts[j]
            if self._is_copy(st, "memcpy_host_to_device"):
                h2d.append(st)
            elif _cls(st) == "Decl" and st.alloc == "gmem_malloc":
                decls.append(st)
            else:
                break
            j += 1
        if j >= len(stmts) or not (_cls(stmts[j]) == "Seq" and _is_kernel_scope(stmts[j])):
            return None
        k = j
        j += 1
        d2h = []
        while j < len(stmts) and self._is_copy(stmts[j], "memcpy_device_to_host"):
            d2h.append(stmts[j])
            j += 1
        if not h2d and not d2h:
            return None
        reads, writes = _rw_sets(stmts[k])
        dev_in = [c.args[0].name for c in h2d]
        dev_out = [c.args[1].name for c in d2h]
        host_in = [c.args[1].name for c in h2d]
        host_out = [c.args[0].name for c in d2h]
        if (any(n not in reads or n in writes for n in dev_in) or any(n not in writes for n in dev_out)
                or len(set(dev_in)) != len(dev_in) or len(set(dev_out)) != len(dev_out)
                or set(dev_in) & set(dev_out) or set(host_in) & set(host_out) or len(set(host_out)) != len(host_out)
                or len(dev_in) + len(dev_out) > 8):
            return None
        if i == k:  # nothing before the kernel: start the window at the kernel
            pass
        return decls, h2d, k, d2h, j

    def host_stmt(self, st, out, ind):
        pad = "    " * ind
        self.pre = []
        c = _cls(st)
        lines = []
        if c == "Seq":
            if _is_kernel_scope(st):
                self.kernel_scope(st, out, ind)
                return
            out.append(pad + "{")
            with self.scope():
                self.host_seq(st, out, ind + 1)
            out.append(pad + "}")
            return
        if c == "Decl":
            lines = self.host_decl(st)
        elif c == "Assign":
            lines = self.host_assign(st)
        elif c == "For":
            start, stop = self.int_expr(st.range.start), self.int_expr(st.range.stop)
            if st.mode not in ("seq", "parallel"):
                raise UnsupportedProgram(f"{st.mode} for outside a kernel")
            v = "v_" + st.index
            e = self.fresh("stop")
            out.extend(pad + p for p in self.pre)
            out.append(pad + f"{{ const int64_t {e} = {stop};")
            out.append(pad + f"for (int64_t {v} = {start}; {v} < {e}; ++{v}) {{")
            with self.scope():
                self.syms[st.index] = Sym(st.index, "scalar", "int")
                self.syms[st.index].loop = True
                self.host_seq(st.body, out, ind + 1)
            out.append(pad + "} }")
            return
        elif c == "If":
            cond, _ = self.expr(st.cond)
            out.extend(pad + p for p in self.pre)
            out.append(pad + f"if ({cond}) {{")
            with self.scope():
                self.host_seq(st.then, out, ind + 1)
            if st.els is not None:
                out.append(pad + "} else {")
                with self.scope():
                    self.host_seq(st.els, out, ind + 1)
            out.append(pad + "}")
            return
        elif c == "Return":
            code, t = self.expr(st.value)
            if t == "i":
                lines = [f"*ret_i = {code}; *ret_kind = 1; return 0;"]
            else:
                lines = [f"*ret_f = (double)({code}); *ret_kind = 2; return 0;"]
        elif c == "CallStmt":
            lines = self.host_call(st)
        else:
            raise UnsupportedProgram(f"cannot compile statement {c}")
        out.extend(pad + p for p in self.pre + lines)

    def host_decl(self, d):
        if d.alloc is None:
            code, t = self.expr(d.init)
            s = Sym(d.name, "scalar", d.ctype)
            self.syms[d.name] = s
            if d.ctype == "float":
                return [f"float {s.cname} = {self.store_value(s, code, t)};"]
            if t != "i":
                raise UnsupportedProgram("int scalar initialised from a float")
            return [f"int64_t {s.cname} = {code};"]
        dims = [self.int_expr(x) for x in d.dims]
        if d.alloc in ("MALLOC", "gmem_malloc"):
            kind = "host_arr" if d.alloc == "MALLOC" else "dev_arr"
            s = Sym(d.name, kind, d.ctype, rank=len(dims))
            self.syms[d.name] = s
            fn = "b2_host_alloc" if kind == "host_arr" else "b2_dev_alloc"
            return [f"auto {s.cname} = {fn}<{s.elem}>({len(dims)}, {{{', '.join(dims)}}});"]
        raise UnsupportedProgram(f"{d.alloc} outside a kernel scope")

    def host_assign(self, a):
        s = self.sym(a.target.base)
        val, t = self.expr(a.value)
        if not s.is_array:
            if s.kind in ("param_int", "param_float"):
                raise UnsupportedProgram(f"assignment to parameter {s.name!r}")
            if s.loop:
                raise UnsupportedProgram(f"{s.name!r} is not assignable")
            if a.op == "+=":
                val, t = self.plus_eq(s, s.cname, val, t, False, "")
            return [f"{s.cname} = {self.store_value(s, val, t)};"]
        if s.kind not in ("param_arr", "host_arr"):
            raise UnsupportedProgram(f"host code writes device/shared array {s.name!r}")
        codes = self._indices(s, a.target.idxs, None)
        ix = self.fresh("idx")
        lines = [f"const int64_t {ix}[] = {{{', '.join(codes) or '0'}}};"]
        if a.op == "+=":
            old = f"b2_hread({s.cname}, {len(codes)}, {ix})"
            val, t = self.plus_eq(s, old, val, t, False, "(int64_t)")
        lines.append(f"b2_hwrite({s.cname}, {len(codes)}, {ix}, ({s.elem})({self.store_value(s, val, t)}));")
        return lines

    def host_call(self, cs):
        f = cs.fn
        if f in ("kernel_setup_end", "kernel_teardown_begin", "blocksync", "magic_barrier",
                 "kernel_teardown_sync"):
            return []
        if f in ("free", "gmem_free") or f.startswith("__smem_free"):
            if not cs.args or _cls(cs.args[0]) != "Var":
                raise UnsupportedProgram(f"{f} of a non-variable")
            s = self.sym(cs.args[0].name)
            return [f"{s.cname}.freed = true;"]
        if f.startswith("memcpy_host_to_device") or f.startswith("memcpy_device_to_host"):
            if len(cs.args) < 3 or _cls(cs.args[0]) != "Var" or _cls(cs.args[1]) != "Var":
                raise UnsupportedProgram(f"{f}: destination and source must be array names")
            d, s = self.sym(cs.args[0].name), self.sym(cs.args[1].name)
            n = " * ".join(f"({self.int_expr(x)})" for x in cs.args[2:])
            if f.startswith("memcpy_host_to_device"):
                if d.kind != "dev_arr" or s.kind not in ("param_arr", "host_arr"):
                    raise UnsupportedProgram(f"{f}: expects (device, host) arrays")
                return [f"b2_h2d({d.cname}, {s.cname}, {n});"]
            if s.kind != "dev_arr" or d.kind not in ("param_arr", "host_arr"):
                raise UnsupportedProgram(f"{f}: expects (host, device) arrays")
            return [f"b2_d2h({d.cname}, {s.cname}, {n});"]
        if f == "kernel_launch":
            raise UnsupportedProgram("kernel_launch must open a scoped block")
        raise UnsupportedProgram(f"call to {f!r} is not supported by the code generator")

    # ------------------------------------------------------------------ kernels
    def kernel_scope(self, seq, out, ind, window=None):
        """Emit one kernel scope: the __global__ function (once) and its host launch.
        With `window` = (h2d CallStmts, d2h CallStmts) the surrounding full-array
        copies are folded into a chunked copy -> kernel -> copy pipeline (SURVEY 8f
        rank 2, b2_pipe_run) whenever the launch is proved in bounds and the
        per-chunk footprints (the bounds proof run over block ranges) allow it;
        otherwise the copies and the launch run in program order as before."""
        pad = "    " * ind
        st = _stmts(seq)
        launch, body = st[0], st[1:]
        if not body or _cls(body[-1]) != "CallStmt" or body[-1].fn != "kernel_kill":
            raise UnsupportedProgram("kernel scope must end with kernel_kill()")
        body = body[:-1]
        self.pre = []
        bpg, tpb = self.int_expr(launch.args[0]), self.int_expr(launch.args[1])
        smem = []
        i = 0
        while i < len(body) and not (_cls(body[i]) == "CallStmt" and body[i].fn == "kernel_setup_end"):
            d = body[i]
            if _cls(d) != "Decl" or d.alloc not in ("__smem_malloc", "__treg_malloc"):
                raise UnsupportedProgram("only __smem_malloc / __treg_malloc may precede kernel_setup_end")
            smem.append(d)
            i += 1
        if i == len(body):
            raise UnsupportedProgram("kernel scope without kernel_setup_end()")
        i += 1
        j = len(body)
        for k in range(i, len(body)):
            if _cls(body[k]) == "CallStmt" and body[k].fn == "kernel_teardown_begin":
                j = k
                break
        kbody, teardown = body[i:j], body[j + 1:]
        for t in teardown:
            if not (_cls(t) == "CallStmt" and (t.fn.startswith("__smem_free") or t.fn == "kernel_teardown_sync")):
                raise UnsupportedProgram("only __smem_free may follow kernel_teardown_begin")
        name = f"b2g_kernel{self.nk}"
        self.nk += 1
        kctx = _KernelCtx(self, name)
        # shared / thread-register arrays: dims evaluated on the host
        host_lines = list(self.pre)
        self.pre = []
        smem_bytes = self.fresh("smem")
        host_lines.append(f"int64_t {smem_bytes} = 0;")
        for d in smem:
            dims = [self.int_expr(x) for x in d.dims]
            kind = "smem_arr" if d.alloc == "__smem_malloc" else "treg_arr"
            s = Sym(d.name, kind, d.ctype, rank=len(dims))
            self.syms[d.name] = s
            kctx.local_arrays.append((s, dims))
            host_lines.extend(self.pre)
            self.pre = []
            dv = f"{s.cname}_hdims"
            host_lines.append(f"const int64_t {dv}[8] = {{{', '.join(dims) or '0'}}};")
            if kind == "smem_arr":
                # The interpreter's shared arrays are plain row-major; on the device the
                # last dimension of a rank >= 2 array gets one cell of padding when it is
                # a multiple of 32 cells, so column accesses (the transpose's tile[x][y])
                # hit 32 different banks (the +1 of transposeNoBankConflicts,
                # PAPER.md:1104). Layout only: indices and bounds are unchanged.
                r = len(dims)
                last = f"{dv}[{r - 1}]" if r else "1"
                extra = f"(({last}) % 32 == 0 ? 1 : 0)" if r >= 2 else "0"
                host_lines.append(f"const int64_t {s.cname}_pitch = {last} + {extra};")
                host_lines.append(f"const int64_t {s.cname}_soff = {smem_bytes};")
                host_lines.append(f"{smem_bytes} += ((" + " * ".join([f"{dv}[{k}]" for k in range(r - 1)] +
                                                                     [f"{s.cname}_pitch"]) +
                                  f") * (int64_t)sizeof({s.elem}) + 15) / 16 * 16;")
        # kernel body
        dl = []
        kctx.assigned = _rw_sets(Seq_like(kbody))[1]
        kctx.block_node, kctx.block_depth = _block_level(kbody)
        kctx.emit_seq(kbody, dl, 1, "b2_w0", "b2_rel0")
        if kctx.block_node is None or kctx.block_hoist is None:
            kctx.coarsenable = False
        if any(s_.kind == "treg_arr" for s_, _ in kctx.local_arrays):
            kctx.coarsenable = False  # per-thread register arrays are not replicated
        self.kernels.append(kctx.render(dl))
        g, t = self.fresh("bpg"), self.fresh("tpb")
        proof = _Proof(self, kctx, f"({g} * {t})").run(kbody)
        args = kctx.host_args()
        info = dict(name=name, g=g, t=t, bpg=bpg, tpb=tpb, smem=smem_bytes, proof=proof, args=args, kctx=kctx)
        if window is None:
            out.extend(pad + ln for ln in host_lines)
            out.extend(pad + ln for ln in self._launch_block(info, [], []))
            return
        # ---- pipelined window
        h2d_calls, d2h_calls = window
        pairs = []  # (dev sym, host sym, n code, is_h2d, copy lines)
        for cs in h2d_calls + d2h_calls:
            self.pre = []
            lines = self.host_call(cs)
            a, b = self.sym(cs.args[0].name), self.sym(cs.args[1].name)
            n = " * ".join(f"({self.int_expr(x)})" for x in cs.args[2:])
            h2d = cs.fn.startswith("memcpy_host_to_device")
            dev_s, host_s = (a, b) if h2d else (b, a)
            pairs.append((dev_s, host_s, n, h2d, self.pre + lines))
        self.pre = []
        slots = {}
        for dev_s, _, _, _, _ in pairs:
            slots.setdefault(dev_s.name, len(slots))
        fp = _Proof(self, kctx, f"({g} * {t})", mode="footprint", slots=slots, tpb=t).run(kbody)
        info.update(fp=fp, slots=slots, pairs=pairs)
        h2d_lines = [ln for p_ in pairs if p_[3] for ln in p_[4]]
        d2h_lines = [ln for p_ in pairs if not p_[3] for ln in p_[4]]
        ok = " && ".join(
            [f"b2_pipe_ok({p_[0].cname}, {p_[1].cname}, {p_[2]}, {'true' if p_[3] else 'false'})" for p_ in pairs] +
            [f"b2_disjoint({a[1].cname}, {b[1].cname})" for a in pairs if a[3] for b in pairs if not b[3]])
        pw = self.fresh("pw")
        out.append(pad + f"{{ const bool {pw} = b2_pipe_on() && {ok};")
        out.append(pad + f"  if ({pw}) {{")
        out.extend(pad + "    " + ln for ln in host_lines)
        out.extend(pad + "    " + ln for ln in self._launch_block(info, h2d_lines, d2h_lines, piped=True))
        out.append(pad + "  } else {")
        out.extend(pad + "    " + ln for ln in h2d_lines)
        out.extend(pad + "    " + ln for ln in host_lines)
        out.extend(pad + "    " + ln for ln in self._launch_block(info, [], []))
        out.extend(pad + "    " + ln for ln in d2h_lines)
        out.append(pad + "  }")
        out.append(pad + "}")

    def _launch_block(self, info, h2d_lines, d2h_lines, piped=False):
        """Host code of one launch (lines, unindented). piped: try the chunked
        pipeline first (needs the bounds proof); the copies in h2d_lines /
        d2h_lines run around a plain launch when it does not apply."""
        name, g, t, smem_bytes, kctx = info["name"], info["g"], info["t"], info["smem"], info["kctx"]
        nk = int(name[len("b2g_kernel"):])
        args = ", ".join(info["args"])
        L = []
        L.append(f"{{ const int64_t {g} = {info['bpg']}, {t} = {info['tpb']};")
        L.append(f"  if ({g} < 0 || {g} > 2147483647LL || {t} < 0 || {t} > 1024 || {g} * {t} >= (1LL << 32)) "
                 f"b2_throw(\"kernel_launch(\" + std::to_string({g}) + \", \" + std::to_string({t}) + \") exceeds the B200 launch limits\");")
        L.append(f"  if ({g} > 0 && {t} > 0) {{")
        pv = self.fresh("proved")
        L.append(f"    bool {pv} = false;")
        for hp in kctx.hoist.values():
            L.append(f"    int64_t {name}{hp}_n = 0, {name}{hp}_s0 = 0; uint32_t {name}{hp}_w2 = 1; int {name}{hp}_sh = -1;")
        ix32 = self.fresh("ix32")
        info["ix32"] = ix32
        L.append(f"    bool {ix32} = false;")
        L.append("    if (b2_prove_enabled()) {")
        L.append("      try {")
        L.append("        b2i_maxabs = 0;")
        L.append("        [&]() {")
        L.extend("          " + ln for ln in info["proof"])
        L.append("        }();")
        L.append(f"        {pv} = true;")
        # 32-bit index arithmetic: every interval the proof saw, and every device array
        # the kernel addresses (flat offsets), below 2^31
        sizes = " && ".join(f"{s_.cname}.n < 2147483647LL" for s_ in kctx.arrays.values()) or "true"
        L.append(f"        {ix32} = b2_ix32_enabled() && b2i_maxabs < 2147483647LL && {sizes};")
        L.append("      } catch (B2NoProof &) {}")
        L.append("    }")
        if nk < 64:  # per-kernel evidence for the first 64 kernels of a program
            L.append(f"    b2_kernel_unchecked[{nk}] = {pv} ? 1 : 0;")
            L.append(f"    b2_kernel_piped[{nk}] = 0;")
            L.append(f"    b2_kernel_ix32[{nk}] = {ix32} ? 1 : 0;")
        L.append(f"    if ({smem_bytes} > 48 * 1024) {{")
        for inst in _INSTANCES:
            L.append(f"      cudaFuncSetAttribute({name}<{inst}>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int){smem_bytes});")
        L.append("    }")
        # thread coarsening (check-free launches of statically eligible kernels whose
        # outermost thread-for walks exactly the program blocks: its width == tpb)
        co, pk = self.fresh("co"), self.fresh("pk")
        info["co"], info["pk"] = co, pk
        blk = kctx.block_hoist
        L.append(f"    int {co} = 1, {pk} = 1;")
        if kctx.coarsenable and blk:
            L.append(f"    if ({pv} && (int64_t){name}{blk}_w2 == {t}) b2_pack_for({t}, {smem_bytes}, {g}, "
                     f"{'true' if kctx.packable else 'false'}, {ix32}, &{co}, &{pk});")
        if nk < 64:
            L.append(f"    b2_kernel_coarsen[{nk}] = {co};")
            L.append(f"    b2_kernel_pack[{nk}] = {pk};")
        done = self.fresh("piped")
        L.append(f"    bool {done} = false;")
        if piped:
            L.extend("    " + ln for ln in self._pipe_lines(info, pv, done, nk))
        L.append(f"    if (!{done}) {{")
        L.extend("      " + ln for ln in h2d_lines)
        L.append("      cudaMemset(b2_err_dev, 0, 5 * sizeof(int));")
        L.append("      cudaEventRecord(b2_ev0, 0);")
        L.extend("      " + ln for ln in _launch_switch(name, pv, ix32, co, pk, f"(unsigned){g}", t, smem_bytes, "0",
                                                   f"{args}, 0u, (uint32_t){g}"))
        L.append("      cudaEventRecord(b2_ev1, 0);")
        L.append(f"      b2_check_kernel(b2_err_dev, \"{name}\");")
        if nk < 64:
            L.append(f"      {{ float ms = 0; cudaEventElapsedTime(&ms, b2_ev0, b2_ev1); b2_kernel_ms[{nk}] = ms; }}")
        L.extend("      " + ln for ln in d2h_lines)
        L.append("    }")
        L.append("  } else {")
        L.extend("    " + ln for ln in h2d_lines + d2h_lines)
        L.append("  }")
        L.append("}")
        return L

    def _pipe_lines(self, info, pv, done, nk):
        """The chunked pipeline (host code): chunk the launch into block ranges
        aligned to the outermost thread-for level, evaluate each chunk's footprint
        on the window's device arrays with the footprint proof, turn footprints into
        2-D copy regions (b2_plan) and hand them to libb200k's b2_pipe_run."""
        name, g, t, smem_bytes, kctx = info["name"], info["g"], info["t"], info["smem"], info["kctx"]
        args = ", ".join(info["args"])
        slots, pairs = info["slots"], info["pairs"]
        arrs = []
        for dev_s, host_s, n, h2d, _ in pairs:
            arrs.append(f"b2_pipe_arr({dev_s.cname}, {host_s.cname}, {slots[dev_s.name]}, {'true' if h2d else 'false'})")
        root = kctx.root_hoist
        al = f"(((int64_t){name}{root}_w2 % {t}) == 0 ? (int64_t){name}{root}_w2 / {t} : 1)" if root else "1"
        L = [f"if ({pv} && b2_pipe_fn()) {{",
             "  try {",
             f"    const std::vector<B2PipeArr> _pa = {{{', '.join(arrs)}}};",
             f"    auto _fpf = [&](int64_t _B0, int64_t _B1, B2FP &_fp) {{"]
        L.extend("      " + ln for ln in info["fp"])
        L.extend([
            "    };",
            "    B2Plan _pl;",
            f"    if (b2_plan({g}, {al}, _pa, _fpf, _pl)) {{",
            f"      auto _lf = [&](int _c, cudaStream_t _s) -> int {{",
            "        const int64_t _b0 = _pl.bnd[_c], _b1 = _pl.bnd[_c + 1];",
            "        if (_b1 <= _b0) return 0;",
            "        if (_c < 64) cudaEventRecord(b2_pev[0][_c], _s);",
            *("        " + ln for ln in _launch_switch(name, "true", info["ix32"], info["co"], info["pk"], "(unsigned)(_b1 - _b0)", t,
                                                  smem_bytes, "_s", f"{args}, (uint32_t)_b0, (uint32_t){g}")),
            "        if (_c < 64) cudaEventRecord(b2_pev[1][_c], _s);",
            "        return cudaGetLastError() == cudaSuccess ? 0 : 1;",
            "      };",
            "      b2_run_plan(_pl, _lf);",
        ])
        if nk < 64:
            L.append(f"      b2_kernel_ms[{nk}] = b2_plan_ms(_pl); b2_kernel_piped[{nk}] = (int)_pl.nchunk;")
        L.extend([
            f"      {done} = true;",
            "    }",
            "  } catch (B2NoProof &) {}",
            "}",
        ])
        return L

    # ------------------------------------------------------------------ translation unit
    def render(self) -> str:
        body = []
        self.host_seq(self.fn.body, body, 2)
        decl = []
        for s in self.params:
            if s.kind == "param_arr":
                decl.append(f"    auto {s.cname} = b2_param<{s.elem}>(&arrs[{s.index}]);")
            elif s.kind == "param_int":
                decl.append(f"    const int64_t {s.cname} = ints[{s.index}];")
            else:
                decl.append(f"    const double {s.cname} = flts[{s.index}];")
        src = [PRELUDE]
        src.extend(self.kernels)
        src.append('extern "C" int b2g_main(B2Arr *arrs, const int64_t *ints, const double *flts, '
                   'int64_t *ret_i, double *ret_f, int *ret_kind, char *err, int errlen, const B2Ops *ops) {')
        src.append("    g_ops = ops;")
        src.append("    if (cudaSetDevice((int)ops->dev) != cudaSuccess) { snprintf(err, errlen, \"bad device\"); return 1; }")
        src.append("    std::vector<void *> dev_allocs, host_allocs;")
        src.append("    g_dev_allocs = &dev_allocs; g_host_allocs = &host_allocs;")
        src.append("    int *b2_err_dev = nullptr;")
        src.append("    struct Cleanup { std::vector<void *> &d, &h; int **e; ~Cleanup() {")
        src.append("        cudaDeviceSynchronize();")
        src.append("        for (void *p : d) g_ops->dfree(p, (int)g_ops->dev); for (void *p : h) free(p);")
        src.append("        if (*e) g_ops->dfree(*e, (int)g_ops->dev); } }")
        src.append("        cleanup{dev_allocs, host_allocs, &b2_err_dev};")
        src.append("    *ret_kind = 0;")
        src.append("    try {")
        src.append("        if (g_ops->alloc(8 * sizeof(int), (int)g_ops->dev, (void **)&b2_err_dev)) b2_throw(g_ops->last_error());")
        src.append("        if (!b2_ev0) { cudaEventCreate(&b2_ev0); cudaEventCreate(&b2_ev1); }")
        src.extend(decl)
        src.extend(body)
        src.append("        return 0;")
        src.append("    } catch (B2Err &e) {")
        src.append("        snprintf(err, errlen, \"%s\", e.msg.c_str());")
        src.append("        return 1;")
        src.append("    }")
        src.append("}")
        return "\n".join(src) + "\n"


class _KernelCtx:
    """Per-kernel state: captured host scalars, device arrays, local arrays."""

    def __init__(self, gen: _Gen, name: str):
        self.g = gen
        self.name = name
        self.arrays: dict = {}      # name -> Sym (dev arrays used)
        self.scalars: dict = {}     # name -> Sym (host scalars captured)
        self.local_arrays: list = []
        self.local_syms: set = set()
        # launch-uniform thread-for levels: their extent / width / shift are computed
        # on the host by the bounds proof and passed in (used by the B2CK = false
        # instantiation only); id(For node) -> parameter prefix
        self.hoist: dict = {}
        self.uniform_const: dict = {}  # id(For) of launch-uniform literal-extent levels
        self.uniform_w = {"b2_w0"}
        self.root_hoist = None  # first hoisted thread-for level directly under the launch width
        # thread coarsening: the "block level" is the innermost thread-for of the chain
        # of pass-through grid levels that open the kernel (A.4: by -> bx; A.5: b); its
        # iterations are the program blocks when its width equals tpb (checked at launch)
        self.block_node = None  # that For node (set by kernel_scope via find_block_level)
        self.block_depth = 0    # its thread-for depth
        self.block_w2 = None    # its per-iteration width variable
        self.block_hoist = None  # its hoisted-parameter prefix (must be hoisted)
        self.coarsenable = True  # statically safe to coarsen (see _emit_for / _emit_simple)
        self.packable = True     # every barrier under launch-uniform control flow only
        self.nonuniform_cf = 0   # depth of enclosing ifs / fors whose condition / bounds vary
        self.tf_depth = 0       # thread-for nesting depth during emission
        self.assigned: set = set()  # scalar names assigned anywhere in the kernel body
        self.tail_ifs: dict = {}    # id(If) -> stop flag of its coarsening loop

    def use(self, s):
        if s.kind == "dev_arr":
            self.arrays[s.name] = s

    def capture(self, name):
        s = self.g.sym(name)
        if not s.is_array and name not in self.local_syms:
            self.scalars[name] = s

    def host_args(self):
        args = []
        for s in self.arrays.values():
            args.append(f"{s.cname}.p")
            args.append(f"{s.cname}.dims[0], {s.cname}.dims[1], {s.cname}.dims[2], {s.cname}.dims[3]")
            args.append(f"{s.cname}.freed")
        for s, dims in self.local_arrays:
            for k in range(4):
                args.append(f"{s.cname}_hdims[{k}]")
            if s.kind == "smem_arr":
                args.append(f"{s.cname}_soff")
                args.append(f"{s.cname}_pitch")
        for s in self.scalars.values():
            args.append(s.cname)
        for hp in self.hoist.values():
            args.append(f"{self.name}{hp}_n, {self.name}{hp}_s0, {self.name}{hp}_w2, {self.name}{hp}_sh")
        args.append("b2_err_dev")
        return args

    def render(self, body_lines):
        params = []
        pro = []
        for s in self.arrays.values():
            params.append(f"{s.elem} *__restrict__ {s.cname}")
            params.append(", ".join(f"int64_t {s.cname}_d{k}" for k in range(4)))
            params.append(f"bool {s.cname}_freed")
            pro.append(f"    const int64_t {s.cname}_dims[4] = {{{s.cname}_d0, {s.cname}_d1, {s.cname}_d2, {s.cname}_d3}};")
            pro.append(f"    if ({s.cname}_freed) {{ b2_flag(b2_err, B2E_OOB, 0, 0); return; }}")
        treg = []
        for s, dims in self.local_arrays:
            params.append(", ".join(f"int64_t {s.cname}_d{k}" for k in range(4)))
            pro.append(f"    const int64_t {s.cname}_dims[4] = {{{s.cname}_d0, {s.cname}_d1, {s.cname}_d2, {s.cname}_d3}};")
            if s.kind == "smem_arr":
                params.append(f"int64_t {s.cname}_soff")
                params.append(f"int64_t {s.cname}_pitch")
                pro.append(f"    {s.elem} *{s.cname} = ({s.elem} *)(b2_smem + {s.cname}_soff);")
            else:
                treg.append(s)
        for s in self.scalars.values():
            ty = "double" if s.kind == "param_float" else ("float" if s.ctype == "float" else "int64_t")
            if ty == "int64_t":  # host ints enter kernel arithmetic in the index type
                params.append(f"const int64_t {s.cname}_p")
                pro.append(f"    const B2IX {s.cname} = (B2IX){s.cname}_p;")
            else:
                params.append(f"const {ty} {s.cname}")
        for hp in self.hoist.values():
            params.append(f"const int64_t {hp}_n, const int64_t {hp}_s0, const uint32_t {hp}_w2, const int {hp}_sh")
        params.append("int *b2_err")
        # block offset / total grid of a chunked launch (b2_pipe_run): a chunk covers
        # blocks [b2_boff, b2_boff + gridDim.x) of a b2_gtot-block launch
        params.append("const uint32_t b2_boff, const uint32_t b2_gtot")
        for s in treg:
            n = " * ".join(f"{s.cname}_d{k}" for k in range(s.rank)) or "1"
            pro.append(f"    {s.elem} {s.cname}[B2_TREG_MAX]; if (({n}) > B2_TREG_MAX) {{ b2_flag(b2_err, B2E_OOB, {n}, B2_TREG_MAX); return; }}")
        # B2CO > 1 (thread coarsening, check-free launches only): a CUDA block of tpb / B2CO
        # threads runs one program block of tpb threads; thread c plays program threads
        # c, c + b2_pbw, ... (b2_pbw = blockDim.x / B2PK) in every block-level thread-for
        # (see _emit_for)
        # B2PK > 1 (block packing): the CUDA block runs B2PK consecutive program blocks side
        # by side, b2_pbw CUDA threads each, every one with its own slice of the dynamic
        # shared memory; their barriers coincide (packing requires every barrier to sit in
        # launch-uniform control flow, see _emit_simple)
        out = [f"template <bool B2CK, int B2CO, int B2PK, typename B2IX> __global__ void {self.name}({', '.join(params)}) {{",
               "    extern __shared__ __align__(16) unsigned char b2_smem0[];",
               "    const uint32_t b2_pbw = blockDim.x / B2PK;",
               "    const uint32_t b2_sub = B2PK == 1 ? 0u : threadIdx.x / b2_pbw;",
               "    unsigned char *b2_smem = b2_smem0;",
               "    if (B2PK > 1) { uint32_t b2_dsm; asm(\"mov.u32 %0, %%dynamic_smem_size;\" : \"=r\"(b2_dsm)); "
               "b2_smem += b2_sub * (b2_dsm / B2PK); }",
               "    const uint32_t b2_w0 = b2_gtot * (b2_pbw * B2CO);",
               "    const uint32_t b2_rel0 = (blockIdx.x * B2PK + b2_sub + b2_boff) * (b2_pbw * B2CO) + (threadIdx.x - b2_sub * b2_pbw);"]
        if treg:
            out.insert(0, "#define B2_TREG_MAX 64")
        out.extend(pro)
        out.extend(body_lines)
        out.append("}")
        return "\n".join(out) + "\n"

    def _index_expr(self, e) -> bool:
        """Integer expression of literals, loop indices, host ints and index-kind
        locals only (no array reads): its intervals are what the bounds proof
        evaluates, so it may run in the 32-bit index type when they fit."""
        c = _cls(e)
        if c == "IntLit":
            return True
        if c == "Var":
            sym = self.g.syms.get(e.name)
            if sym is None or sym.is_array or sym.ctype == "float" or sym.kind == "param_float":
                return False
            if sym.loop or e.name not in self.local_syms:
                return True
            return getattr(sym, "ix", False)
        if c == "BinOp":
            return e.op in ("+", "-", "*", "/", "%") and self._index_expr(e.lhs) and self._index_expr(e.rhs)
        if c == "Call" and (e.fn in ("exact_div", "pow2") or e.fn.startswith("DMINDEX")):
            return all(self._index_expr(a) for a in e.args)
        return False

    def _uniform(self, e) -> bool:
        """Launch-uniform integer expression: constants and captured host ints only."""
        c = _cls(e)
        if c == "IntLit":
            return True
        if c == "Var":
            sym = self.g.syms.get(e.name)
            return (e.name not in self.local_syms and sym is not None and not sym.is_array
                    and sym.kind != "param_float" and sym.ctype != "float")
        if c == "BinOp":
            return e.op in ("+", "-", "*", "/", "%") and self._uniform(e.lhs) and self._uniform(e.rhs)
        if c == "Call" and (e.fn in ("exact_div", "pow2") or e.fn.startswith("DMINDEX")):
            return all(self._uniform(a) for a in e.args)
        return False

    # ------------------------------------------------------------------ device statements
    def emit_seq(self, stmts, out, ind, w, rel):
        for st in stmts:
            if _is_ghost(st):
                continue
            self.emit(st, out, ind, w, rel)

    def _scan_captures(self, node):
        """Record host scalars referenced by an expression."""
        c = _cls(node)
        if c == "Var":
            s = self.g.syms.get(node.name)
            if s is not None and not s.is_array:
                self.capture(node.name)
        elif c == "BinOp":
            self._scan_captures(node.lhs)
            self._scan_captures(node.rhs)
        elif c == "Call":
            for a in node.args:
                self._scan_captures(a)
        elif c in ("Access", "Ptr"):
            for a in node.idxs:
                self._scan_captures(a)

    def dexpr(self, e):
        self._scan_captures(e)
        return self.g.expr(e, self)

    def emit(self, st, out, ind, w, rel):
        g = self.g
        pad = "    " * ind
        g.pre = []
        c = _cls(st)
        if c == "Seq":
            out.append(pad + "{")
            with g.scope(self):
                self.emit_seq(st.stmts, out, ind + 1, w, rel)
            out.append(pad + "}")
            return
        if c == "For":
            with g.scope(self):
                if st.mode in ("thread", "magic_thread") and self.block_w2 is not None and w == self.block_w2:
                    # a block-level thread-for: under thread coarsening (B2CO > 1) each CUDA
                    # thread plays B2CO program threads, b2_pbw apart (coalescing kept)
                    rk = g.fresh("relk")
                    tail = self._tail_if(st)
                    if tail is not None:
                        # `thread for t { if (t < e) {...} }` with e the same for every program
                        # thread of the block: t grows with b2_k, so once a played thread fails
                        # the test every later one does too — stop there (the tree levels of
                        # A.5 skip most of their idle iterations)
                        stop = g.fresh("stop")
                        self.tail_ifs[id(tail)] = stop
                        out.append(pad + f"bool {stop} = false;")
                        out.append(pad + "#pragma unroll")
                        out.append(pad + f"for (int b2_k = 0; b2_k < B2CO && !{stop}; ++b2_k) {{")
                    else:
                        out.append(pad + "#pragma unroll")
                        out.append(pad + "for (int b2_k = 0; b2_k < B2CO; ++b2_k) {")
                    out.append(pad + f"    const uint32_t {rk} = {rel} + (uint32_t)b2_k * b2_pbw;")
                    self._emit_for(st, out, ind + 1, w, rk)
                    out.append(pad + "}")
                else:
                    self._emit_for(st, out, ind, w, rel)
            return
        if c == "If":
            cond, _ = self.dexpr(st.cond)
            out.extend(pad + p for p in g.pre)
            out.append(pad + f"if ({cond}) {{")
            nu = not self._uniform(st.cond)
            self.nonuniform_cf += nu
            with g.scope(self):
                self.emit_seq(st.then.stmts, out, ind + 1, w, rel)
            if st.els is not None:
                out.append(pad + "} else {")
                with g.scope(self):
                    self.emit_seq(st.els.stmts, out, ind + 1, w, rel)
            elif id(st) in self.tail_ifs:
                out.append(pad + f"}} else {{ {self.tail_ifs[id(st)]} = true;")
            self.nonuniform_cf -= nu
            out.append(pad + "}")
            return
        self._emit_simple(st, out, ind, w, rel)

    def _tail_if(self, st):
        """The If of `thread for t { if (t < e) {...} }` (or `<=`, no else) when e
        cannot change from one program thread of the block to the next (it reads
        no thread-level names and no arrays); else None."""
        body = [x for x in st.body.stmts if not _is_ghost(x)]
        if len(body) != 1 or _cls(body[0]) != "If" or body[0].els is not None:
            return None
        cond = body[0].cond
        if _cls(cond) != "BinOp" or cond.op not in ("<", "<=") or _cls(cond.lhs) != "Var" \
                or cond.lhs.name != st.index:
            return None

        def uniform(e):
            c = _cls(e)
            if c == "IntLit":
                return True
            if c == "Var":
                sym = self.g.syms.get(e.name)
                if sym is None or sym.is_array or e.name == st.index:
                    return False
                if e.name not in self.local_syms:
                    return True  # host scalar
                return getattr(sym, "depth", 99) <= self.block_depth
            if c == "BinOp":
                return uniform(e.lhs) and uniform(e.rhs)
            if c == "Call" and e.fn in ("pow2", "exact_div"):
                return all(uniform(a) for a in e.args)
            return False
        return body[0] if uniform(cond.rhs) else None

    def _emit_for(self, st, out, ind, w, rel):
        g = self.g
        pad = "    " * ind
        s0, _ = self.dexpr(st.range.start)
        s1, _ = self.dexpr(st.range.stop)
        pre = g.pre
        g.syms[st.index] = Sym(st.index, "scalar", "int")
        g.syms[st.index].loop = True
        g.syms[st.index].depth = self.tf_depth + (1 if st.mode in ("thread", "magic_thread") else 0)
        self.local_syms.add(st.index)
        v = "v_" + st.index
        out.extend(pad + p for p in pre)
        if st.mode in ("thread", "magic_thread"):
            n, w2, r2 = g.fresh("n"), g.fresh("w"), g.fresh("rel")
            # widths / positions are uint32 (launch guard: grid < 2^32 threads);
            # power-of-two widths (the usual tile shapes) split with shift / mask
            sh = g.fresh("sh")
            hp = None
            if w in self.uniform_w and not pre and self._uniform(st.range.start) and self._uniform(st.range.stop):
                self.uniform_w.add(w2)
                hp = f"_hp{len(self.hoist)}"
                self.hoist[id(st)] = hp
                if w == "b2_w0" and self.root_hoist is None:
                    self.root_hoist = hp
                if st is self.block_node:
                    self.block_hoist = hp
                if _is_const(st.range.start) and _is_const(st.range.stop):
                    # literal extent: nvcc folds n and the start; the host supplies
                    # the width split (loop-invariant, check-free) for proved launches
                    self.uniform_const[id(st)] = True
            if hp is None or id(st) in self.uniform_const:
                out.append(pad + f"{{ const int64_t {n} = ({s1}) - ({s0});")
                out.append(pad + f"  if ({n} > 0) {{")
                if hp is None:
                    out.append(pad + f"  if ({n} > (int64_t){w} || {w} % (uint32_t){n} != 0) "
                                     f"{{ b2_flag(b2_err, B2E_WIDTH, {n}, {w}); return; }}")
                    out.append(pad + f"  const uint32_t {w2} = {w} / (uint32_t){n};")
                    out.append(pad + f"  const int {sh} = ({w2} & ({w2} - 1u)) == 0u ? __ffs({w2}) - 1 : -1;")
                else:
                    out.append(pad + f"  if (B2CK && ({n} > (int64_t){w} || {w} % (uint32_t){n} != 0)) "
                                     f"{{ b2_flag(b2_err, B2E_WIDTH, {n}, {w}); return; }}")
                    out.append(pad + f"  const uint32_t {w2} = B2CK ? {w} / (uint32_t){n} : {hp}_w2;")
                    out.append(pad + f"  const int {sh} = B2CK ? (({w2} & ({w2} - 1u)) == 0u ? __ffs({w2}) - 1 : -1) : {hp}_sh;")
                out.append(pad + f"  const B2IX {v} = ({s0}) + (B2IX)({sh} >= 0 ? {rel} >> {sh} : {rel} / {w2});")
            else:  # proved launches take the host's values: no checks, no divisions
                out.append(pad + f"{{ const int64_t {n} = B2CK ? (({s1}) - ({s0})) : {hp}_n;")
                out.append(pad + f"  if ({n} > 0) {{")
                out.append(pad + f"  if (B2CK && ({n} > (int64_t){w} || {w} % (uint32_t){n} != 0)) "
                                 f"{{ b2_flag(b2_err, B2E_WIDTH, {n}, {w}); return; }}")
                out.append(pad + f"  const uint32_t {w2} = B2CK ? {w} / (uint32_t){n} : {hp}_w2;")
                out.append(pad + f"  const int {sh} = B2CK ? (({w2} & ({w2} - 1u)) == 0u ? __ffs({w2}) - 1 : -1) : {hp}_sh;")
                out.append(pad + f"  const B2IX {v} = (B2CK ? (B2IX)({s0}) : (B2IX){hp}_s0) + (B2IX)({sh} >= 0 ? {rel} >> {sh} : {rel} / {w2});")
            out.append(pad + f"  const uint32_t {r2} = {sh} >= 0 ? ({rel} & ({w2} - 1u)) : {rel} % {w2};")
            if st is self.block_node:
                self.block_w2 = w2
            self.tf_depth += 1
            self.emit_seq(st.body.stmts, out, ind + 1, w2, r2)
            self.tf_depth -= 1
            out.append(pad + "  } }")
            return
        e = g.fresh("stop")
        out.append(pad + f"{{ const B2IX {e} = {s1};")
        out.append(pad + f"for (B2IX {v} = {s0}; {v} < {e}; ++{v}) {{")
        nu = not (self._uniform(st.range.start) and self._uniform(st.range.stop))
        self.nonuniform_cf += nu
        self.emit_seq(st.body.stmts, out, ind + 1, w, rel)
        self.nonuniform_cf -= nu
        out.append(pad + "} }")

    def _emit_simple(self, st, out, ind, w, rel):
        g = self.g
        pad = "    " * ind
        c = _cls(st)
        if c == "CallStmt":
            if st.fn in ("blocksync", "kernel_teardown_sync"):
                if self.tf_depth != self.block_depth:  # a barrier off the block level: no coarsening
                    self.coarsenable = False
                if self.nonuniform_cf:  # packed program blocks could disagree on reaching it
                    self.packable = False
                out.append(pad + "__syncthreads();")
                return
            raise UnsupportedProgram(f"call to {st.fn!r} inside a kernel")
        if c == "Decl":
            if st.alloc is not None:
                raise UnsupportedProgram(f"{st.alloc} inside a kernel body")
            code, t = self.dexpr(st.init)
            ix = st.ctype == "int" and st.name not in self.assigned and self._index_expr(st.init)
            s = Sym(st.name, "scalar", st.ctype)
            s.ix = ix
            g.syms[st.name] = s
            self.local_syms.add(st.name)
            s.depth = self.tf_depth
            out.extend(pad + p for p in g.pre)
            if st.ctype == "float":
                out.append(pad + f"float {s.cname} = {g.store_value(s, code, t)};")
            else:
                # index-kind locals (never reassigned, built from literals, loop indices,
                # host ints and other such locals) take the instantiation's index type
                out.append(pad + f"{'B2IX' if s.ix else 'int64_t'} {s.cname} = {code};")
            return
        if c == "Assign":
            s = g.sym(st.target.base)
            val, t = self.dexpr(st.value)
            if not s.is_array:
                if s.loop:
                    raise UnsupportedProgram(f"{s.name!r} is not assignable")
                if st.target.base not in self.local_syms:
                    raise UnsupportedProgram(f"kernel assigns host scalar {s.name!r}")
                if self.tf_depth > self.block_depth and getattr(s, "depth", 0) <= self.block_depth:
                    self.coarsenable = False  # program threads write a block-level local
                if st.op == "+=":
                    val, t = g.plus_eq(s, s.cname, val, t, True, "")
                out.extend(pad + p for p in g.pre)
                out.append(pad + f"{s.cname} = {g.store_value(s, val, t)};")
                return
            if s.kind not in ("dev_arr", "smem_arr", "treg_arr"):
                raise UnsupportedProgram(f"kernel writes host array {s.name!r}")
            self.use(s)
            for ix in st.target.idxs:
                self._scan_captures(ix)
            codes = g._indices(s, st.target.idxs, self)
            ok, off, lines = g._dev_offset(s, codes)
            cell = f"{s.cname}[{off}]"
            if st.op == "+=":
                val, t = g.plus_eq(s, cell, val, t, True, "(int64_t)")
            # a memory write in a context wider than one thread runs once (interp semantics)
            guard = f"{rel} == 0 && " if w != "1" else ""
            body = g.pre + lines + [f"if ({guard}{ok}) {cell} = ({s.elem})({g.store_value(s, val, t)});"]
            out.append(pad + "{")
            out.extend(pad + "    " + b for b in body)
            out.append(pad + "}")
            return
        raise UnsupportedProgram(f"cannot compile statement {c} inside a kernel")


class _Proof:
    """Host code proving, for one concrete launch, that every array access of a
    kernel is in bounds (then the unchecked instantiation runs). Mirrors the
    kernel's statements with interval arithmetic (b2i_* in PRELUDE): a thread-for /
    for variable ranges over [start.lo, stop.hi - 1], both branches of an `if` are
    covered, captured host scalars are points. Throws B2NoProof (checked kernel)
    on anything it cannot bound: values read from arrays, locals reassigned in the
    kernel, inexact exact_div, non-constant divisors.

    mode="footprint" emits the same walk as the body of a lambda over a block range
    [_B0, _B1) that also records, per device array of a pipelined window (`slots`),
    the union of the index intervals it reads / writes (b2fp_acc): the outermost
    launch-uniform thread-for level is narrowed to the iterations those blocks run
    (v = s0 + rel / w2, rel in [_B0 * tpb, _B1 * tpb)); inner levels keep their full
    ranges, so the footprint over-approximates what the chunk touches."""

    def __init__(self, gen: "_Gen", kctx: "_KernelCtx", width: str, mode: str = "prove",
                 slots: dict = None, tpb: str = None):
        self.g = gen
        self.k = kctx
        self.locals: dict = {}     # kernel-local int name -> C++ interval variable, or None (unknown)
        self.n = 0
        self.width = [width]       # launch-uniform context widths of the enclosing hoisted levels
        self.mode = mode
        self.slots = slots or {}
        self.tpb = tpb

    def fresh(self):
        self.n += 1
        return f"_pi{self.n}"

    def run(self, kbody):
        self.reassigned, self.declared = set(), set()
        self._scan(kbody)
        out = []
        self.seq(kbody, out)
        return out

    def _scan(self, stmts):
        for st in stmts:
            c = _cls(st)
            if c == "Assign" and not self.g.syms.get(st.target.base, Sym("", "scalar", "int")).is_array:
                self.reassigned.add(st.target.base)
            if c == "Decl":  # declared twice (sibling scopes): do not trust either interval
                if st.name in self.declared:
                    self.reassigned.add(st.name)
                self.declared.add(st.name)
            for attr in ("body", "then", "els"):
                sub = getattr(st, attr, None)
                if sub is not None:
                    self._scan(_stmts(sub))
            if c == "Seq":
                self._scan(st.stmts)

    # expressions -> (C++ expression of type B2I, kind) with kind i (int interval),
    # v (a value we cannot bound: array cell / float); both still evaluate every
    # nested access check
    def expr(self, e):
        c = _cls(e)
        if c == "IntLit":
            return f"b2i_c({int(e.value)}LL)", "i"
        if c == "FloatLit":
            return "b2i_c(0)", "v"
        if c == "Var":
            if e.name in self.locals:
                iv = self.locals[e.name]
                if iv == "F":
                    return "b2i_c(0)", "v"
                return (iv, "i") if iv else ("b2i_unknown()", "i")
            sc = self.k.scalars.get(e.name)
            if sc is not None and sc.kind != "param_float" and sc.ctype != "float":
                return f"b2i_c((int64_t){sc.cname})", "i"
            return "b2i_c(0)", "v"
        if c == "Access":
            chk = self.access(e.base, e.idxs, rw=0)
            return f"({chk}, b2i_c(0))", "v"
        if c == "BinOp":
            a, ka = self.expr(e.lhs)
            b, kb = self.expr(e.rhs)
            if ka != "i" or kb != "i":
                return f"((void){a}, (void){b}, b2i_c(0))", "v"
            op = e.op
            if op in ("==", "!=", "<", "<=", ">", ">="):
                return f"((void){a}, (void){b}, B2I{{0, 1}})", "i"
            fn = {"+": "b2i_add", "-": "b2i_sub", "*": "b2i_mul", "/": "b2i_div", "%": "b2i_mod"}.get(op)
            if fn is None:
                return "b2i_unknown()", "i"
            return f"{fn}({a}, {b})", "i"
        if c == "Call":
            if e.fn == "exact_div":
                a, ka = self.expr(e.args[0])
                b, kb = self.expr(e.args[1])
                if ka != "i" or kb != "i":
                    return "b2i_unknown()", "i"
                return f"b2i_exact_div({a}, {b})", "i"
            if e.fn == "pow2":
                a, ka = self.expr(e.args[0])
                return (f"b2i_pow2({a})", "i") if ka == "i" else ("b2i_unknown()", "i")
            if e.fn.startswith("DMINDEX"):
                k = len(e.args) // 2
                out = "b2i_c(0)"
                for d, ix in zip(e.args[:k], e.args[k:]):
                    dc, kd = self.expr(d)
                    ic, ki = self.expr(ix)
                    if kd != "i" or ki != "i":
                        return "b2i_unknown()", "i"
                    out = f"b2i_add(b2i_mul({out}, {dc}), {ic})"
                return out, "i"
        return "b2i_unknown()", "i"

    def index(self, e):
        code, kind = self.expr(e)
        return code if kind == "i" else f"((void){code}, b2i_unknown())"

    def access(self, base, idxs, rw=0):
        """C++ expression (int) checking every index of one access (rw: 0 read,
        1 write, 2 both; footprint mode records the window arrays' intervals)."""
        sym = self.g.syms[base]
        idxs = list(idxs)
        if sym.kind in ("smem_arr", "treg_arr"):
            idxs = idxs[1:]  # the DMINDEX block index: 0 in per-block storage
            dims = f"{sym.cname}_hdims"
        else:
            dims = f"{sym.cname}.dims"
        slot = self.slots.get(base) if (self.mode == "footprint" and sym.kind == "dev_arr") else None

        def chk(code, k):
            if slot is None:
                return f"b2i_in({code}, {dims}[{k}])"
            return f"b2fp_acc(_fp, {rw}, {slot}, {k}, {code}, {dims}[{k}])"
        if len(idxs) == sym.rank + 1 and sym.rank == 1:
            return chk(f"b2i_add({self.index(idxs[0])}, {self.index(idxs[1])})", 0)
        if len(idxs) != sym.rank:
            return "(b2i_unknown(), 0)"
        return "(" + ", ".join(chk(self.index(ix), k) for k, ix in enumerate(idxs)) + ")" if idxs else "0"

    def refine(self, cond):
        """(local name, narrowed interval expression) for `v OP e` / `e OP v` with v an
        int local of known interval and e an int expression; else None."""
        if _cls(cond) != "BinOp" or cond.op not in ("<", "<=", ">", ">=", "=="):
            return None
        flip = {"<": ">", "<=": ">=", ">": "<", ">=": "<=", "==": "=="}
        for var, other, op in ((cond.lhs, cond.rhs, cond.op), (cond.rhs, cond.lhs, flip[cond.op])):
            if _cls(var) == "Var" and self.locals.get(var.name) not in (None, "F") and var.name in self.locals:
                e, kind = self.expr(other)
                if kind != "i":
                    return None
                iv = self.locals[var.name]
                lo, hi = f"{iv}.lo", f"{iv}.hi"
                if op == "<":
                    hi = f"std::min({iv}.hi, ({e}).hi - 1)"
                elif op == "<=":
                    hi = f"std::min({iv}.hi, ({e}).hi)"
                elif op == ">":
                    lo = f"std::max({iv}.lo, ({e}).lo + 1)"
                elif op == ">=":
                    lo = f"std::max({iv}.lo, ({e}).lo)"
                else:
                    lo, hi = f"std::max({iv}.lo, ({e}).lo)", f"std::min({iv}.hi, ({e}).hi)"
                return var.name, f"B2I{{{lo}, {hi}}}"
        return None

    # statements
    def block(self, stmts, out):
        """A nested block: its declarations end with it (interp.py:248-249 pushes a
        frame per Seq), so a shadowing Decl must not leak its interval outward."""
        saved = dict(self.locals)
        self.seq(stmts, out)
        self.locals = saved

    def seq(self, stmts, out):
        for st in stmts:
            if not _is_ghost(st):
                self.stmt(st, out)

    def stmt(self, st, out):
        c = _cls(st)
        if c == "Seq":
            out.append("{")
            self.block(st.stmts, out)
            out.append("}")
        elif c == "For":
            if st.index in self.reassigned:  # the emitter refuses this too ('k' is not assignable)
                out.append("throw B2NoProof{};")
                return
            a, b = self.index(st.range.start), self.index(st.range.stop)
            s0, s1, v = self.fresh(), self.fresh(), self.fresh()
            out.append(f"{{ const B2I {s0} = {a}, {s1} = {b};")
            hp = self.k.hoist.get(id(st))
            pushed = False
            if hp is not None:  # launch-uniform level: the values the check-free kernel uses
                q = f"{self.k.name}{hp}"
                out.append(f"  if ({s0}.lo != {s0}.hi || {s1}.lo != {s1}.hi) throw B2NoProof{{}};")
                out.append(f"  {q}_n = {s1}.lo - {s0}.lo; {q}_s0 = {s0}.lo;")
                out.append(f"  if ({q}_n > 0) {{ const int64_t _w = {self.width[-1]};")
                out.append(f"    if ({q}_n > _w || _w % {q}_n != 0) throw B2NoProof{{}};")
                out.append(f"    {q}_w2 = (uint32_t)(_w / {q}_n);")
                out.append(f"    {q}_sh = ({q}_w2 & ({q}_w2 - 1u)) == 0u ? __builtin_ctz({q}_w2) : -1; }}")
                self.width.append(f"(int64_t){q}_w2")
                pushed = True
            if pushed and self.mode == "footprint" and len(self.width) == 2:
                # outermost launch-uniform level: only the iterations of blocks [_B0, _B1)
                q = f"{self.k.name}{hp}"
                out.append(f"  const int64_t {v}_a = {s0}.lo + (_B0 * {self.tpb}) / (int64_t){q}_w2;")
                out.append(f"  const int64_t {v}_b = {s0}.lo + (_B1 * {self.tpb} - 1) / (int64_t){q}_w2;")
                out.append(f"  if ({s1}.hi > {s0}.lo && _B1 > _B0) {{ const B2I {v} = B2I{{std::max({s0}.lo, {v}_a), "
                           f"std::min({s1}.hi - 1, {v}_b)}};")
                out.append(f"  if ({v}.lo <= {v}.hi) {{")
            else:
                out.append(f"  if ({s1}.hi > {s0}.lo) {{ const B2I {v} = B2I{{{s0}.lo, {s1}.hi - 1}};")
                out.append("  {")
            saved = dict(self.locals)
            self.locals[st.index] = v
            self.seq(st.body.stmts, out)
            if pushed:
                self.width.pop()
            self.locals = saved
            out.append("} } }")
        elif c == "If":
            out.append(f"(void){self.expr(st.cond)[0]};")
            ref = self.refine(st.cond)
            if ref is None:
                self.block(st.then.stmts, out)
            else:  # `v < e` etc. on an int local: the then-branch sees v narrowed
                name, code = ref
                v, saved = self.fresh(), dict(self.locals)
                out.append(f"{{ const B2I {v} = {code};")
                out.append(f"  if ({v}.lo <= {v}.hi) {{")
                self.locals[name] = v
                self.seq(st.then.stmts, out)
                self.locals = saved
                out.append("} }")
            if st.els is not None:
                self.block(st.els.stmts, out)
        elif c == "Decl":
            code, kind = self.expr(st.init)
            if st.ctype == "int" and kind == "i" and st.name not in self.reassigned:
                v = self.fresh()
                out.append(f"const B2I {v} = {code};")
                self.locals[st.name] = v
            else:
                out.append(f"(void){code};")
                self.locals[st.name] = "F" if st.ctype == "float" else None
        elif c == "Assign":
            out.append(f"(void){self.expr(st.value)[0]};")
            sym = self.g.syms.get(st.target.base)
            if sym is not None and sym.is_array:
                out.append(f"(void){self.access(st.target.base, st.target.idxs, rw=2 if st.op == '+=' else 1)};")
        # CallStmt (blocksync): no access


# ----------------------------------------------------------------------------- compile + run

_NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--fmad=false",
               "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math", "-shared", "-cudart", "static",
               "-lineinfo", "-diag-suppress", "177,550"]
_lock = threading.Lock()
_loaded: dict = {}


def generate(fn) -> str:
    """CUDA C++ translation unit for a GPU-form entry function."""
    if not has_kernel(fn):
        raise UnsupportedProgram(
            f"function {fn.name!r} has no kernel_launch scope: not a GPU program "
            "(no CPU fallback)")
    return _Gen(fn).render()


class Compiled:
    def __init__(self, fn, path, source):
        self.fn = fn
        self.path = path
        self.source = source
        self.lib = ctypes.CDLL(path)
        self.lib.b2g_main.restype = ctypes.c_int
        self.lib.b2g_main.argtypes = [ctypes.c_void_p] * 9
        self.lib.b2g_kernel_ms.restype = ctypes.c_double
        self.lib.b2g_kernel_ms.argtypes = [ctypes.c_int]
        self.lib.b2g_kernel_unchecked.restype = ctypes.c_int
        self.lib.b2g_kernel_unchecked.argtypes = [ctypes.c_int]
        self.lib.b2g_kernel_piped.restype = ctypes.c_int
        self.lib.b2g_kernel_piped.argtypes = [ctypes.c_int]
        self.lib.b2g_kernel_coarsen.restype = ctypes.c_int
        self.lib.b2g_kernel_coarsen.argtypes = [ctypes.c_int]
        self.lib.b2g_kernel_pack.restype = ctypes.c_int
        self.lib.b2g_kernel_pack.argtypes = [ctypes.c_int]
        self.lib.b2g_kernel_ix32.restype = ctypes.c_int
        self.lib.b2g_kernel_ix32.argtypes = [ctypes.c_int]
        self.n_kernels = source.count("__global__ void b2g_kernel")
        # the generated host code keeps per-call state (ops table, allocation lists,
        # timing events) in statics of its .so: one call at a time per program
        self.lock = threading.Lock()

    def kernel_ms(self) -> list:
        """Device time (CUDA events) of each kernel's last launch, in ms."""
        return [self.lib.b2g_kernel_ms(k) for k in range(min(self.n_kernels, 64))]

    def kernel_piped(self) -> list:
        """Per kernel: number of chunks its last launch was pipelined into with the
        surrounding copies (b2_pipe_run), 0 if it ran as one launch between them."""
        return [self.lib.b2g_kernel_piped(k) for k in range(min(self.n_kernels, 64))]

    def kernel_coarsen(self) -> list:
        """Per kernel: program threads per CUDA thread in its last launch (1, 2, 4; 8 packed)."""
        return [self.lib.b2g_kernel_coarsen(k) for k in range(min(self.n_kernels, 64))]

    def kernel_pack(self) -> list:
        """Per kernel: program blocks per CUDA block in its last launch (1, 2)."""
        return [self.lib.b2g_kernel_pack(k) for k in range(min(self.n_kernels, 64))]

    def kernel_ix32(self) -> list:
        """Per kernel: True if its last launch used 32-bit index arithmetic."""
        return [self.lib.b2g_kernel_ix32(k) == 1 for k in range(min(self.n_kernels, 64))]

    def kernel_unchecked(self) -> list:
        """Per kernel: True if its last launch ran the check-free instantiation (all
        accesses proved in bounds on the host for that launch)."""
        return [self.lib.b2g_kernel_unchecked(k) == 1 for k in range(min(self.n_kernels, 64))]


class B2Ops(ctypes.Structure):
    """Host runtime services handed to generated code (libb200k.so copy engine)."""
    _fields_ = [("h2d", ctypes.c_void_p), ("d2h", ctypes.c_void_p), ("last_error", ctypes.c_void_p),
                ("alloc", ctypes.c_void_p), ("dfree", ctypes.c_void_p), ("dev", ctypes.c_int64),
                ("pipe", ctypes.c_void_p), ("pipe_chunk", ctypes.c_int64), ("coarsen", ctypes.c_int64),
                ("pack", ctypes.c_int64)]


def _ops(dev: int) -> B2Ops:
    from ._lib import lib
    L = lib()
    addr = lambda f: ctypes.cast(f, ctypes.c_void_p).value  # noqa: E731
    # bytes per pipeline step (tune key codegen.pipe_kb; 0 = no copy / kernel pipelining)
    chunk = int(L.b2_tune_get(b"codegen.pipe_kb")) * 1024
    # thread coarsening of check-free generated kernels (tune key codegen.coarsen; 1 = off)
    coarsen = max(1, int(L.b2_tune_get(b"codegen.coarsen")))
    # program blocks per CUDA block for small program blocks (tune key codegen.pack; 1 = off)
    pack = max(1, int(L.b2_tune_get(b"codegen.pack")))
    return B2Ops(addr(L.b2_copy_h2d), addr(L.b2_copy_d2h), addr(L.b2_last_error),
                 addr(L.b2_device_alloc), addr(L.b2_device_free), dev, addr(L.b2_pipe_run), max(chunk, 0),
                 coarsen, pack)


class B2Arr(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("n", ctypes.c_int64), ("rank", ctypes.c_int64),
                ("dims", ctypes.c_int64 * MAX_RANK), ("init", ctypes.c_void_p),
                ("freed", ctypes.c_int64)]


def _nvcc():
    from ._build import nvcc
    return nvcc()


def compile_fn(fn) -> Compiled:
    src = generate(fn)
    key = hashlib.sha256(src.encode() + " ".join(_NVCC_FLAGS).encode()).hexdigest()[:20]
    with _lock:
        if key in _loaded:
            return _loaded[key]
        os.makedirs(GEN_DIR, exist_ok=True)
        so = os.path.join(GEN_DIR, f"b2g_{key}.so")
        cu = os.path.join(GEN_DIR, f"b2g_{key}.cu")
        if not os.path.exists(so):
            with open(cu, "w") as f:
                f.write(src)
            r = subprocess.run([_nvcc(), *_NVCC_FLAGS, "-o", so + ".tmp", cu], capture_output=True, text=True)
            if r.returncode != 0:
                raise UnsupportedProgram("generated CUDA failed to compile:\n" + r.stderr[-4000:])
            os.replace(so + ".tmp", so)
        c = Compiled(fn, so, src)
        _loaded[key] = c
        return c


def run_compiled(c: Compiled, env: dict, arrays: dict):
    """Execute with the interpreter's marshalled environment; writes results back
    into the Arrays. Returns ("ret", v) or None like Interp.run."""
    fn = c.fn
    n = len(fn.params)
    arrs = (B2Arr * max(n, 1))()
    ints = (ctypes.c_int64 * max(n, 1))()
    flts = (ctypes.c_double * max(n, 1))()
    keep = []
    writeback = []
    for i, (pn, pt) in enumerate(fn.params):
        v = env[pn]
        if pt.endswith("*"):
            a = arrays[pn]
            buf, init, wb = _host_buffer(a, pt[:-1])
            keep.extend([buf, init])
            arrs[i].data = buf.ctypes.data
            arrs[i].n = buf.size
            arrs[i].rank = len(a.dims)
            if len(a.dims) > MAX_RANK:
                raise UnsupportedProgram("arrays of rank > 8")
            for k, d in enumerate(a.dims):
                arrs[i].dims[k] = int(d)
            arrs[i].init = init.ctypes.data if init is not None else None
            arrs[i].freed = 1 if a.freed else 0
            if wb is not None:
                writeback.append((a, buf, init, wb))
        elif pt == "int":
            ints[i] = int(v)
        else:
            flts[i] = float(v)
    ri = ctypes.c_int64(0)
    rf = ctypes.c_double(0.0)
    rk = ctypes.c_int(0)
    err = ctypes.create_string_buffer(1024)
    from .ops import _host_device
    ops = _ops(_host_device())
    with c.lock:
        rc = c.lib.b2g_main(ctypes.addressof(arrs), ctypes.addressof(ints), ctypes.addressof(flts),
                            ctypes.byref(ri), ctypes.byref(rf), ctypes.byref(rk), err, 1024, ctypes.byref(ops))
    for a, buf, init, wb in writeback:
        wb(buf, init)
    if rc != 0:
        raise InterpError(err.value.decode(errors="replace"))
    if rk.value == 1:
        return ("ret", int(ri.value))
    if rk.value == 2:
        return ("ret", float(rf.value))
    return None


def _host_buffer(a, ctype):
    """(numpy buffer, init mask or None, writeback fn or None) for an Array."""
    dt = np.float32 if a.ctype == "float" else np.int64
    data = a.data
    if isinstance(data, np.ndarray):
        flat = data.reshape(-1)
        if flat.dtype == dt and flat.flags.c_contiguous:
            return flat, None, None
        buf = flat.astype(dt)

        def wb(b, m, flat=flat):
            flat[...] = b.astype(flat.dtype)
        return buf, None, wb
    nones = [i for i, x in enumerate(data) if x is None]
    if nones:
        vals = [0 if x is None else x for x in data]
        init = np.ones(len(data), dtype=np.uint8)
        init[nones] = 0
    else:
        vals, init = data, None
    if dt == np.float32:
        buf = np.array(vals, dtype=np.float64).astype(np.float32)
    else:
        try:
            buf = np.array(vals, dtype=np.int64)
        except OverflowError:
            raise InterpError("int cell value outside the int64 range of compiled programs") from None

    def wb(b, m, data=data):
        vals = b.tolist()
        if m is None:
            data[:] = vals
        else:
            for i in np.flatnonzero(m).tolist():
                data[i] = vals[i]
    return buf, init, wb
