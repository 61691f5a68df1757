"""Canonical structural dump of a Program (reference or ours): executable
structure only, ghosts kept as names, annotation payloads dropped. Used to pin
our parser (paper_2605_13864_b200/lang.py) to the reference parser's output."""


def _e(x):
    c = type(x).__name__
    if c == "IntLit":
        return ["Int", x.value]
    if c == "FloatLit":
        return ["Float", float(x.value)]
    if c == "Var":
        return ["Var", x.name]
    if c == "BinOp":
        return ["Bin", x.op, _e(x.lhs), _e(x.rhs)]
    if c == "Call":
        return ["Call", x.fn, [_e(a) for a in x.args]]
    if c in ("Access", "Ptr"):
        return [c, x.base, [_e(a) for a in x.idxs]]
    if c == "Lam":
        return ["Lam", list(x.params), _e(x.body)]
    return [c]


def _s(s):
    c = type(s).__name__
    if c == "Seq":
        return ["Seq", [_s(t) for t in s.stmts]]
    if c == "For":
        return ["For", s.index, s.mode, _e(s.range.start), _e(s.range.stop), _s(s.body)]
    if c == "Assign":
        return ["Assign", s.target.base, [_e(i) for i in s.target.idxs], s.op, _e(s.value)]
    if c == "Decl":
        return ["Decl", s.name, s.ctype, s.alloc, _e(s.init) if s.init is not None else None,
                [_e(d) for d in s.dims]]
    if c == "CallStmt":
        return ["CallStmt", s.fn, bool(s.ghost), [_e(a) for a in s.args]]
    if c == "If":
        return ["If", _e(s.cond), _s(s.then), _s(s.els) if s.els is not None else None]
    if c == "Return":
        return ["Return", _e(s.value)]
    return [c]


def dump_program(p):
    return [{"name": f.name, "ret": f.ret, "params": [list(x) for x in f.params],
             "admitted": bool(f.admitted), "body": _s(f.body) if f.body is not None else None}
            for f in p.fns]
