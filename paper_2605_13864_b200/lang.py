"""The OptiGPU program language: AST node types and a parser for the program
grammar, so callers can build the `Program` objects that `run_program` takes
without the reference package installed.

Node classes and field names mirror the reference's (minigpu/ast.py:21-427), so
Programs from either parser are interchangeable: the recogniser
(`recognize.py`) dispatches on class *names* and fields only. Contract and
ghost annotations are kept as their raw strings: they carry proofs, not
behaviour (the reference interpreter ignores them too, interp.py:3, :331).

Grammar accepted (minigpu/parser.py:578-893, restated):
  program  := { __pure("..."); | __axiom(name, "..."); | fndef }
  fndef    := type name ( [type name {, type name}] ) { {clause} {stmt} }
  type     := float | int | void  [*]
  clause   := __requires|__ensures|__consumes|__produces|__preserves|__writes|__reads ("...");
              | __admitted(); | __ghost_fn();
  stmt     := { [__block_attr("...");]* {stmt} }
            | [parallel|thread|magic thread] for (int i = e; i < e; i++) { {loop-clause} {stmt} }
            | if (e) { stmts } [else { stmts }]   | return e;
            | __ghost(name [, "..."]);           | type name = e;
            | type* [const] name = ALLOCk<elem>(e, ...);
            | name(e, ...);                       | name{[e]} (= | +=) e;
  expr     := add [(==|!=|<|<=|>|>=) add | "|" add]; add := mul {(+|-) mul};
  mul      := unary {(*|/|%) unary}  ("/" is exact_div); unary := [-] atom
  atom     := int | float | (e) | &name{[e]} | fun x.. -> e | name(args) | name{[e]} | name
"""
from __future__ import annotations

import itertools
import re
from dataclasses import dataclass, field

# ----------------------------------------------------------------------------- expressions


@dataclass(frozen=True)
class Expr:
    pass


@dataclass(frozen=True)
class IntLit(Expr):
    value: int


@dataclass(frozen=True)
class FloatLit(Expr):
    value: float


@dataclass(frozen=True)
class Var(Expr):
    name: str


@dataclass(frozen=True)
class BinOp(Expr):
    op: str
    lhs: Expr
    rhs: Expr


@dataclass(frozen=True)
class Call(Expr):
    fn: str
    args: tuple = ()


@dataclass(frozen=True)
class Lam(Expr):
    params: tuple
    body: Expr


@dataclass(frozen=True)
class Ptr(Expr):
    base: str
    idxs: tuple = ()


@dataclass(frozen=True)
class Access(Expr):
    base: str
    idxs: tuple = ()


UNINIT = Var("__uninit__")


@dataclass(frozen=True)
class Range:
    start: Expr
    stop: Expr


@dataclass(frozen=True)
class Loc:
    base: str
    idxs: tuple = ()


# ----------------------------------------------------------------------------- statements

_nid = itertools.count(1)


@dataclass
class Stmt:
    nid: int = field(default_factory=lambda: next(_nid), init=False, compare=False)
    loc_info: tuple | None = field(default=None, init=False, compare=False)


@dataclass
class Decl(Stmt):
    name: str = ""
    ctype: str = "float"
    init: Expr | None = None
    alloc: str | None = None
    dims: tuple = ()


@dataclass
class Assign(Stmt):
    target: Loc = None
    op: str = "="
    value: Expr = None


@dataclass
class CallStmt(Stmt):
    fn: str = ""
    args: tuple = ()
    ghost: bool = False
    ghost_args: tuple = ()  # raw annotation string(s)


@dataclass
class Seq(Stmt):
    stmts: list = field(default_factory=list)
    scope: bool = False
    attrs: set = field(default_factory=set)


@dataclass
class For(Stmt):
    index: str = "i"
    range: Range = None
    mode: str = "seq"  # seq | parallel | thread | magic_thread
    contract: dict = None  # clause -> [raw strings]
    body: Seq = None


@dataclass
class If(Stmt):
    cond: Expr = None
    then: Seq = None
    els: Seq | None = None


@dataclass
class Return(Stmt):
    value: Expr = None


@dataclass
class FnDef:
    name: str
    params: list  # [(name, ctype)], ctype in {int, float, int*, float*}
    annots: dict  # clause -> [raw strings]
    body: Seq | None
    admitted: bool = False
    ghost: bool = False
    ret: str = "void"


@dataclass
class Program:
    pures: list = field(default_factory=list)   # raw "__pure" strings
    axioms: list = field(default_factory=list)  # (name, raw string)
    fns: list = field(default_factory=list)
    source: str = "<mem>"

    def fn(self, name: str) -> FnDef:
        for f in self.fns:
            if f.name == name:
                return f
        raise KeyError(name)

    def entry(self) -> FnDef:
        for f in reversed(self.fns):
            if not f.admitted and not f.ghost and f.body is not None:
                return f
        raise ValueError("program has no entry function")


# ----------------------------------------------------------------------------- tokens


class ParseError(Exception):
    def __init__(self, msg: str, line: int = 0, col: int = 0, filename: str = "<mem>"):
        super().__init__(f"{filename}:{line}:{col}: {msg}")
        self.msg, self.line, self.col, self.filename = msg, line, col, filename


_TOKENS = [
    ("skip", r"[ \t\r\n]+|//[^\n]*"),
    ("string", r'"(?:[^"\\]|\\.)*"'),
    ("float", r"\d+\.\d+f?|\d+\.(?!\.)f?"),
    ("int", r"\d+"),
    ("ident", r"[A-Za-z_]\w*"),
    ("op", r"\.\.\+|\.\.|\+\+|\+=|->|~>|:=|==|!=|<=|>=|[-+*/%<>=(){}\[\],;:.&|\\]"),
]
_TOKEN_RE = re.compile("|".join(f"(?P<{k}>{v})" for k, v in _TOKENS))


@dataclass
class Tok:
    kind: str
    val: str
    line: int
    col: int


def tokenize(text: str, filename: str = "<mem>") -> list[Tok]:
    out, pos, line, lstart = [], 0, 1, 0
    while pos < len(text):
        m = _TOKEN_RE.match(text, pos)
        if m is None:
            raise ParseError(f"unexpected character {text[pos]!r}", line, pos - lstart + 1, filename)
        kind, val = m.lastgroup, m.group()
        if kind != "skip":
            out.append(Tok(kind, val, line, pos - lstart + 1))
        nl = val.count("\n")
        if nl:
            line += nl
            lstart = pos + val.rfind("\n") + 1
        pos = m.end()
    out.append(Tok("eof", "", line, pos - lstart + 1))
    return out


# ----------------------------------------------------------------------------- parser

FN_CLAUSES = ("requires", "ensures", "consumes", "produces", "preserves", "writes", "reads")
LOOP_CLAUSES = ("spreserves", "sreads", "xconsumes", "xproduces", "xwrites", "xreads",
                "xrequires", "xensures")
ALLOCATORS = re.compile(r"(MALLOC|gmem_malloc|__smem_malloc|__treg_malloc)(\d)")
_CMP = ("==", "!=", "<=", ">=", "<", ">")


class _Parser:
    def __init__(self, text: str, filename: str):
        self.toks = tokenize(text, filename)
        self.i = 0
        self.filename = filename

    # -- token helpers
    def peek(self, k: int = 0) -> Tok:
        return self.toks[min(self.i + k, len(self.toks) - 1)]

    def take(self) -> Tok:
        t = self.peek()
        self.i += 1
        return t

    def is_(self, val: str, k: int = 0) -> bool:
        t = self.peek(k)
        return t.kind != "string" and t.val == val

    def eat(self, val: str) -> bool:
        if self.is_(val):
            self.i += 1
            return True
        return False

    def need(self, val: str) -> Tok:
        if not self.is_(val):
            self.err(f"expected {val!r}, found {self.peek().val!r}")
        return self.take()

    def need_kind(self, kind: str) -> Tok:
        if self.peek().kind != kind:
            self.err(f"expected {kind}, found {self.peek().val!r}")
        return self.take()

    def err(self, msg: str):
        t = self.peek()
        raise ParseError(msg, t.line, t.col, self.filename)

    def string(self) -> str:
        return self.need_kind("string").val[1:-1].replace('\\"', '"')

    # -- top level
    def program(self) -> Program:
        p = Program(source=self.filename)
        while self.peek().kind != "eof":
            if self.is_("__pure"):
                self.take(); self.need("("); s = self.string(); self.need(")"); self.need(";")
                p.pures.append(s)
            elif self.is_("__axiom"):
                self.take(); self.need("(")
                name = self.need_kind("ident").val
                self.need(","); s = self.string(); self.need(")"); self.need(";")
                p.axioms.append((name, s))
            else:
                p.fns.append(self.fndef())
        names = [f.name for f in p.fns] + [a[0] for a in p.axioms] + \
            [s.partition(":")[0].strip() for s in p.pures]
        dup = sorted({n for n in names if names.count(n) > 1})
        if dup:
            raise ParseError(f"duplicate top-level names: {dup}", 1, 1, self.filename)
        return p

    def ctype(self) -> str:
        t = self.take()
        if t.val not in ("float", "int", "void") or t.kind == "string":
            raise ParseError(f"expected a type, found {t.val!r}", t.line, t.col, self.filename)
        return t.val + ("*" if self.eat("*") else "")

    def fndef(self) -> FnDef:
        ret = self.ctype()
        name = self.need_kind("ident").val
        self.need("(")
        params = []
        if not self.is_(")"):
            while True:
                pt = self.ctype()
                params.append((self.need_kind("ident").val, pt))
                if not self.eat(","):
                    break
        self.need(")")
        self.need("{")
        annots: dict = {c: [] for c in FN_CLAUSES}
        admitted = ghost = False
        while True:
            v = self.peek().val
            if v in ("__admitted", "__ghost_fn") and self.peek().kind == "ident":
                self.take(); self.need("("); self.need(")"); self.need(";")
                admitted |= v == "__admitted"
                ghost |= v == "__ghost_fn"
            elif v.startswith("__") and v[2:] in FN_CLAUSES and self.peek().kind == "ident":
                self.take(); self.need("("); annots[v[2:]].append(self.string())
                self.need(")"); self.need(";")
            else:
                break
        body = self.block_rest()
        return FnDef(name, params, annots, None if admitted else body, admitted, ghost, ret)

    def block_rest(self) -> Seq:
        seq = Seq(scope=True)
        while not self.is_("}"):
            if self.peek().kind == "eof":
                self.err("unexpected end of input, missing '}'")
            seq.stmts.append(self.stmt())
        self.need("}")
        return seq

    # -- statements
    def stmt(self) -> Stmt:
        t = self.peek()
        s = self._stmt()
        s.loc_info = (t.line, t.col)
        return s

    def _loop_ahead(self) -> bool:
        v = self.peek().val
        if v == "for":
            return self.is_("(", 1)
        if v in ("parallel", "thread"):
            return self.is_("for", 1)
        if v == "magic":
            return self.is_("thread", 1) and self.is_("for", 2)
        return False

    def _stmt(self) -> Stmt:
        t = self.peek()
        if t.kind == "string":
            self.err("unexpected string at statement start")
        v = t.val
        if v == "{":
            self.take()
            seq = Seq(scope=True)
            while self.is_("__block_attr"):
                self.take(); self.need("("); seq.attrs.add(self.string()); self.need(")"); self.need(";")
            while not self.is_("}"):
                if self.peek().kind == "eof":
                    self.err("unexpected end of input, missing '}'")
                seq.stmts.append(self.stmt())
            self.need("}")
            return seq
        if self._loop_ahead():
            return self.loop()
        if v == "if":
            self.take(); self.need("(")
            cond = self.expr()
            self.need(")"); self.need("{")
            then = self.block_rest()
            els = None
            if self.eat("else"):
                self.need("{")
                els = self.block_rest()
            return If(cond=cond, then=then, els=els)
        if v == "return":
            self.take()
            e = self.expr()
            self.need(";")
            return Return(value=e)
        if v == "__ghost":
            self.take(); self.need("(")
            name = self.need_kind("ident").val
            gargs = ()
            if self.eat(","):
                gargs = (self.string(),)
            self.need(")"); self.need(";")
            return CallStmt(fn=name, ghost=True, ghost_args=gargs)
        if v in ("float", "int") and (self.is_("*", 1) or (
                self.peek(1).kind == "ident" and self.peek(1).val not in
                ("for", "parallel", "thread", "magic"))):
            return self.decl()
        if t.kind == "ident":
            if self.is_("(", 1):
                name = self.take().val
                args = self.args()
                self.need(";")
                return CallStmt(fn=name, args=args)
            base = self.take().val
            idxs = self.indices()
            op = self.take()
            if op.val not in ("=", "+=") or op.kind == "string":
                # reported at the token after the offending one, as parser.py:150-152 does
                nt = self.peek()
                raise ParseError(f"expected assignment, found {op.val!r}", nt.line, nt.col,
                                 self.filename)
            val = self.expr()
            self.need(";")
            return Assign(target=Loc(base, idxs), op=op.val, value=val)
        self.err(f"unexpected token {v!r} at statement start")

    def loop(self) -> For:
        mode = "seq"
        if self.eat("parallel"):
            mode = "parallel"
        elif self.eat("thread"):
            mode = "thread"
        elif self.eat("magic"):
            self.need("thread")
            mode = "magic_thread"
        self.need("for"); self.need("("); self.need("int")
        idx = self.need_kind("ident").val
        self.need("=")
        start = self.expr()
        self.need(";")
        if self.need_kind("ident").val != idx:
            self.err(f"loop condition must test index {idx!r}")
        self.need("<")
        stop = self.expr()
        self.need(";")
        if self.need_kind("ident").val != idx:
            self.err(f"loop increment must update index {idx!r}")
        self.need("++"); self.need(")"); self.need("{")
        contract: dict = {c: [] for c in LOOP_CLAUSES}
        while self.peek().kind == "ident" and self.peek().val.startswith("__") and \
                self.peek().val[2:] in LOOP_CLAUSES:
            c = self.take().val[2:]
            self.need("("); contract[c].append(self.string()); self.need(")"); self.need(";")
        body = self.block_rest()
        for s in body.stmts:
            if type(s).__name__ == "For" and s.index == idx:
                raise ParseError(f"loop index {idx!r} shadowed by nested loop", 0, 0, self.filename)
        return For(index=idx, range=Range(start, stop), mode=mode, contract=contract, body=body)

    def decl(self) -> Decl:
        ctype = self.take().val
        if self.eat("*"):
            self.eat("const")
            name = self.need_kind("ident").val
            self.need("=")
            at = self.need_kind("ident")
            m = ALLOCATORS.fullmatch(at.val)
            if not m:
                nt = self.peek()  # position of the next token (parser.py:150-152)
                raise ParseError(f"expected an allocator, found {at.val!r}", nt.line, nt.col,
                                 self.filename)
            self.need("<")
            elem = self.take().val
            self.need(">")
            dims = self.args()
            self.need(";")
            if len(dims) != int(m.group(2)):
                self.err(f"{at.val} takes {m.group(2)} dimensions, got {len(dims)}")
            return Decl(name=name, ctype=elem, alloc=m.group(1), dims=dims)
        name = self.need_kind("ident").val
        self.need("=")
        init = self.expr()
        self.need(";")
        return Decl(name=name, ctype=ctype, init=init)

    # -- expressions
    def args(self) -> tuple:
        self.need("(")
        out = []
        if not self.is_(")"):
            out.append(self.expr())
            while self.eat(","):
                out.append(self.expr())
        self.need(")")
        return tuple(out)

    def indices(self) -> tuple:
        idxs = []
        while self.eat("["):
            idxs.append(self.expr())
            self.need("]")
        return tuple(idxs)

    def expr(self) -> Expr:
        lhs = self.add()
        t = self.peek()
        if t.kind == "op" and t.val in _CMP:
            self.take()
            return BinOp(t.val, lhs, self.add())
        if self.is_("|"):
            self.take()
            return Call("divides", (lhs, self.add()))
        return lhs

    def add(self) -> Expr:
        e = self.mul()
        while self.peek().kind == "op" and self.peek().val in ("+", "-"):
            op = self.take().val
            e = BinOp(op, e, self.mul())
        return e

    def mul(self) -> Expr:
        e = self.unary()
        while self.peek().kind == "op" and self.peek().val in ("*", "/", "%"):
            op = self.take().val
            rhs = self.unary()
            e = Call("exact_div", (e, rhs)) if op == "/" else BinOp(op, e, rhs)
        return e

    def unary(self) -> Expr:
        if self.eat("-"):
            return BinOp("-", IntLit(0), self.unary())
        return self.atom()

    def atom(self) -> Expr:
        t = self.peek()
        if t.kind == "int":
            self.take()
            return IntLit(int(t.val))
        if t.kind == "float":
            self.take()
            return FloatLit(float(t.val.rstrip("f")))
        if self.eat("("):
            e = self.expr()
            self.need(")")
            return e
        if self.eat("&"):
            base = self.need_kind("ident").val
            return Ptr(base, self.indices())
        if t.kind == "ident" and t.val == "fun":
            self.take()
            params = [self.need_kind("ident").val]
            while self.peek().kind == "ident" and not self.is_("->"):
                params.append(self.take().val)
            self.need("->")
            return Lam(tuple(params), self.expr())
        if t.kind == "ident":
            self.take()
            if t.val == "UninitCell":
                return UNINIT
            if self.is_("("):
                return Call(t.val, self.args())
            if self.is_("["):
                return Access(t.val, self.indices())
            return Var(t.val)
        self.err(f"unexpected token {t.val!r} in expression")


def parse_program(text: str, filename: str = "<mem>") -> Program:
    """Parse an OptiGPU program (mirrors minigpu.parser.parse_program, parser.py:893)."""
    return _Parser(text, filename).program()
