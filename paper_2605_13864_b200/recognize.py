"""Program recogniser: maps a `Program` entry function onto one of the B200
kernels, or refuses it.

The reference executes any Program by walking it (minigpu/interp.py:248-309).
This package executes only the OptiGPU hot-path programs — the transpose and
the reduction in their naive and GPU-derived forms (
PAPER.md:155-172, 395-433, 586-618, 1041-1068, 1120-1131) — and refuses every
other program loudly (there is no CPU fallback).

Recognition is alpha-equivalence against canonical templates (and against the
members of the A.4 / A.5 derivation families, programs.transpose_gpu_family /
reduce_tree_family, instantiated with parameters read off the program's own
literals): after removing
ghost calls (ast.py:473-494 `strip_ghosts`), the entry body must match a
template node for node, with every binder (parameter, local, loop index)
renamed consistently (a bijection) and every literal, operator, loop mode,
allocator and intrinsic identical. Parameter ORDER is free: parameters are
bound by the role they play in the body. Works on Programs from this package's
parser and from the reference's (matching is by node class name and fields).
"""
from __future__ import annotations

import functools
from dataclasses import dataclass, field

from .errors import UnsupportedProgram
from .lang import parse_program

# ----------------------------------------------------------------------------- templates
from .programs import (REDUCE_NAIVE as _R_NAIVE, REDUCE_NAIVE_ADD_L as _R_NAIVE_L,
                       REDUCE_NAIVE_ADD_R as _R_NAIVE_R, REDUCE_TREE as _R_TREE,
                       TRANSPOSE_GPU as _T_GPU, TRANSPOSE_NAIVE_XY as _T_NAIVE_XY,
                       TRANSPOSE_NAIVE_YX as _T_NAIVE_YX, reduce_tree_family, source,
                       transpose_gpu_family)


@dataclass
class Template:
    name: str
    kind: str      # "transpose" | "reduce"
    form: str      # "naive" | "gpu" | "tree512" | "tree"
    cell: str      # "float" | "int"
    fn: object     # parsed FnDef
    roles: dict = field(default_factory=dict)  # role -> template param name
    consts: dict = field(default_factory=dict)  # family parameters (T, R / B)


def _mk(name, kind, form, cell, text, roles, zero=None):
    fn = parse_program(source(text, cell, zero), f"<template {name}>").fns[0]
    return Template(name, kind, form, cell, fn, roles)


_TR = {"in": "in", "out": "out", "W": "W", "H": "H"}
_RR = {"arr": "arr", "N": "N"}
TEMPLATES = [
    _mk("transpose_naive_xy_float", "transpose", "naive", "float", _T_NAIVE_XY, _TR),
    _mk("transpose_naive_yx_float", "transpose", "naive", "float", _T_NAIVE_YX, _TR),
    _mk("transpose_naive_xy_int", "transpose", "naive", "int", _T_NAIVE_XY, _TR),
    _mk("transpose_naive_yx_int", "transpose", "naive", "int", _T_NAIVE_YX, _TR),
    _mk("transpose_gpu_float", "transpose", "gpu", "float", _T_GPU, _TR),
    _mk("reduce_naive_float", "reduce", "naive", "float", _R_NAIVE, _RR, zero="0."),
    _mk("reduce_naive_float_i0", "reduce", "naive", "float", _R_NAIVE, _RR, zero="0"),
    _mk("reduce_naive_int", "reduce", "naive", "int", _R_NAIVE, _RR, zero="0"),
    *[_mk(f"reduce_naive_{cell}_{side}{z}", "reduce", "naive", cell, text, _RR, zero=zero)
      for side, text in (("addl", _R_NAIVE_L), ("addr", _R_NAIVE_R))
      for cell, zero, z in (("float", "0.", ""), ("float", "0", "_i0"), ("int", "0", ""))],
    _mk("reduce_tree512_float", "reduce", "tree512", "float", _R_TREE, _RR),
]


# ----------------------------------------------------------------------------- matching

class NoMatch(Exception):
    pass


def _cls(x) -> str:
    return type(x).__name__


def strip_ghosts(stmts):
    return [s for s in stmts if not (_cls(s) == "CallStmt" and getattr(s, "ghost", False))]


class _Unifier:
    """Bijective renaming between template names and program names."""

    def __init__(self, params_t, params_p):
        self.t2p: dict = {}
        self.p2t: dict = {}
        self.params_t = dict(params_t)  # name -> ctype
        self.params_p = dict(params_p)

    def bind(self, tn: str, pn: str):
        if tn in self.t2p or pn in self.p2t:
            if self.t2p.get(tn) != pn or self.p2t.get(pn) != tn:
                raise NoMatch(f"name {pn!r} does not play the role of {tn!r}")
            return
        # parameters map to parameters of the same type; locals to locals
        if (tn in self.params_t) != (pn in self.params_p):
            raise NoMatch(f"{pn!r} vs {tn!r}: parameter/local mismatch")
        if tn in self.params_t and self.params_t[tn] != self.params_p[pn]:
            raise NoMatch(f"parameter {pn!r} has type {self.params_p[pn]}, "
                          f"expected {self.params_t[tn]}")
        self.t2p[tn] = pn
        self.p2t[pn] = tn

    # -- expressions
    def expr(self, t, p):
        ct, cp = _cls(t), _cls(p)
        if ct != cp:
            raise NoMatch(f"expression {cp} where {ct} expected")
        if ct == "IntLit":
            if t.value != p.value:
                raise NoMatch(f"literal {p.value} where {t.value} expected")
        elif ct == "FloatLit":
            if float(t.value) != float(p.value):
                raise NoMatch(f"literal {p.value} where {t.value} expected")
        elif ct == "Var":
            self.bind(t.name, p.name)
        elif ct == "BinOp":
            if t.op != p.op:
                raise NoMatch(f"operator {p.op} where {t.op} expected")
            self.expr(t.lhs, p.lhs)
            self.expr(t.rhs, p.rhs)
        elif ct == "Call":
            if t.fn != p.fn:
                raise NoMatch(f"call {p.fn} where {t.fn} expected")
            self.exprs(t.args, p.args)
        elif ct in ("Access", "Ptr"):
            self.bind(t.base, p.base)
            self.exprs(t.idxs, p.idxs)
        else:
            raise NoMatch(f"unsupported expression {ct}")

    def exprs(self, ts, ps):
        if len(ts) != len(ps):
            raise NoMatch("arity mismatch")
        for a, b in zip(ts, ps):
            self.expr(a, b)

    # -- statements
    def seq(self, t, p):
        ts, ps = strip_ghosts(t.stmts), strip_ghosts(p.stmts)
        if len(ts) != len(ps):
            raise NoMatch(f"block of {len(ps)} statements where {len(ts)} expected")
        for a, b in zip(ts, ps):
            self.stmt(a, b)

    def stmt(self, t, p):
        ct, cp = _cls(t), _cls(p)
        if ct != cp:
            raise NoMatch(f"statement {cp} where {ct} expected")
        if ct == "Seq":
            self.seq(t, p)
        elif ct == "For":
            if t.mode != p.mode:
                raise NoMatch(f"loop mode {p.mode} where {t.mode} expected")
            self.bind(t.index, p.index)
            self.expr(t.range.start, p.range.start)
            self.expr(t.range.stop, p.range.stop)
            self.seq(t.body, p.body)
        elif ct == "Assign":
            if t.op != p.op:
                raise NoMatch(f"assignment {p.op} where {t.op} expected")
            self.bind(t.target.base, p.target.base)
            self.exprs(t.target.idxs, p.target.idxs)
            self.expr(t.value, p.value)
        elif ct == "Decl":
            if (t.ctype, t.alloc) != (p.ctype, p.alloc):
                raise NoMatch(f"declaration {p.ctype}/{p.alloc} where {t.ctype}/{t.alloc} expected")
            self.bind(t.name, p.name)
            if (t.init is None) != (p.init is None):
                raise NoMatch("initialiser mismatch")
            if t.init is not None:
                self.expr(t.init, p.init)
            self.exprs(tuple(t.dims), tuple(p.dims))
        elif ct == "CallStmt":
            if t.fn != p.fn or bool(t.ghost) != bool(p.ghost):
                raise NoMatch(f"call {p.fn} where {t.fn} expected")
            self.exprs(t.args, p.args)
        elif ct == "If":
            self.expr(t.cond, p.cond)
            self.seq(t.then, p.then)
            if (t.els is None) != (p.els is None):
                raise NoMatch("else-branch mismatch")
            if t.els is not None:
                self.seq(t.els, p.els)
        elif ct == "Return":
            self.expr(t.value, p.value)
        else:
            raise NoMatch(f"unsupported statement {ct}")


@dataclass
class Plan:
    """What to run: a template plus the program's parameter names for its roles."""
    template: Template
    params: dict  # role -> program parameter name
    fn_name: str

    @property
    def kind(self):
        return self.template.kind

    @property
    def form(self):
        return self.template.form

    @property
    def cell(self):
        return self.template.cell

    @property
    def consts(self):
        return self.template.consts


def match(fn, tmpl: Template) -> Plan:
    tf = tmpl.fn
    if fn.body is None:
        raise NoMatch(f"function {fn.name!r} has no body (admitted)")
    if getattr(fn, "ret", "void") != tf.ret:
        raise NoMatch(f"return type {fn.ret} where {tf.ret} expected")
    if len(fn.params) != len(tf.params):
        raise NoMatch(f"{len(fn.params)} parameters where {len(tf.params)} expected")
    u = _Unifier(tf.params, fn.params)
    u.seq(tf.body, fn.body)
    missing = [n for n, _ in tf.params if n not in u.t2p]
    if missing:
        raise NoMatch(f"parameters {missing} unused")
    return Plan(tmpl, {role: u.t2p[tn] for role, tn in tmpl.roles.items()}, fn.name)


@functools.lru_cache(maxsize=256)
def _family_template(kind: str, a: int, b, cell: str) -> Template:
    if kind == "transpose":
        fn = parse_program(transpose_gpu_family(a, b), f"<template transpose_gpu_T{a}_R{b}>").fns[0]
        return Template(f"transpose_gpu_T{a}_R{b}", "transpose", "gpu", "float", fn, _TR, {"T": a, "R": b})
    fn = parse_program(reduce_tree_family(a, cell), f"<template reduce_tree_B{a}_{cell}>").fns[0]
    return Template(f"reduce_tree_B{a}_{cell}", "reduce", "tree", cell, fn, _RR, {"B": a})


def _int_literals(node, out):
    c = _cls(node)
    if c == "IntLit":
        out.add(node.value)
        return
    for f in ("lhs", "rhs", "value", "init", "cond", "then", "els", "body", "range", "start", "stop",
              "target"):
        v = getattr(node, f, None)
        if v is not None and not isinstance(v, (str, int, float)):
            _int_literals(v, out)
    for f in ("args", "idxs", "stmts", "dims"):
        for v in getattr(node, f, ()) or ():
            if not isinstance(v, (str, int, float)):
                _int_literals(v, out)


def family_candidates(fn):
    """Family members worth trying for this function: parameters drawn from its
    own integer literals (a tile side T with R | T, R * T <= 1024; a block B = 2t
    with t a power of two <= 1024)."""
    if fn.body is None:
        return []
    lits = set()
    _int_literals(fn.body, lits)
    out = []
    ret = getattr(fn, "ret", "void")
    if ret == "void" and len(fn.params) == 4:
        for T in sorted(lits):
            for R in sorted(lits):
                if 0 < R <= T and T % R == 0 and R * T <= 1024 and (T, R) != (32, 16):
                    out.append(("transpose", T, R, "float"))
    if ret in ("float", "int") and len(fn.params) == 2:
        for B in sorted(lits):
            t = B // 2
            if B >= 2 and B % 2 == 0 and t & (t - 1) == 0 and t <= 1024 and (B, ret) != (512, "float"):
                out.append(("reduce", B, None, ret))
    return out


def recognize(program, entry: str) -> Plan:
    fn = program.fn(entry)
    reasons = []
    for t in TEMPLATES:
        try:
            return match(fn, t)
        except NoMatch as e:
            reasons.append(f"{t.name}: {e}")
    for kind, a, b, cell in family_candidates(fn):
        t = _family_template(kind, a, b, cell)
        try:
            return match(fn, t)
        except NoMatch as e:
            reasons.append(f"{t.name}: {e}")
    raise UnsupportedProgram(
        f"function {entry!r} is not one of the programs this B200 backend executes "
        f"(transpose / reduce, naive or GPU-derived forms); no CPU fallback. "
        f"Closest mismatches: " + "; ".join(reasons[:3]))
