"""Our program parser vs the reference parser (structural dumps generated from
minigpu.parser.parse_program by tests/golden/gen_golden.py)."""
import json
import os
import sys

import pytest

from conftest import GOLDEN, program_text

sys.path.insert(0, GOLDEN)
from tests_ast_dump import dump_program  # noqa: E402

from paper_2605_13864_b200 import ParseError, parse_program  # noqa: E402


def test_parser_matches_reference_asts():
    with open(os.path.join(GOLDEN, "ref_asts.json")) as f:
        ref = json.load(f)
    assert len(ref) >= 7
    for name, want in ref.items():
        got = json.loads(json.dumps(dump_program(parse_program(program_text(name), name))))
        assert got == want, name


def test_division_is_exact_div_and_unary_minus():
    p = parse_program("int f(int a) { return -a / 4 % 3; }")
    e = p.fn("f").body.stmts[0].value
    assert type(e).__name__ == "BinOp" and e.op == "%"
    assert e.lhs.fn == "exact_div"
    assert e.lhs.args[0].op == "-" and e.lhs.args[0].lhs.value == 0


def test_loop_modes_and_annotations_kept_raw():
    src = """void k(float* a, int n) {
        __reads("a ~> Matrix1(n, A)");
        parallel for (int i = 0; i < n; i++) { __xwrites("&a[i] ~> 0."); a[i] = 0.; }
        thread for (int j = 0; j < n; j++) { a[j] += 1.5f; }
        magic thread for (int q = 0; q < n; q++) { __ghost(foo, "x := 1"); }
    }"""
    fn = parse_program(src).fn("k")
    modes = [s.mode for s in fn.body.stmts]
    assert modes == ["parallel", "thread", "magic_thread"]
    assert fn.annots["reads"] == ["a ~> Matrix1(n, A)"]
    assert fn.body.stmts[0].contract["xwrites"] == ["&a[i] ~> 0."]
    assert fn.body.stmts[2].body.stmts[0].ghost


@pytest.mark.parametrize("bad", [
    "void f( { }",
    "void f() { for (int i = 0; j < 3; i++) { } }",
    "void f() { x = ; }",
    "void f() { float* a = notalloc1<float>(3); }",
    "void f() { float* a = MALLOC2<float>(3); }",
    "void f() { }  void f() { }",
    "void f() { for (int i = 0; i < 2; i++) { for (int i = 0; i < 2; i++) { } } }",
])
def test_parse_errors(bad):
    with pytest.raises(ParseError):
        parse_program(bad)


def test_parse_error_messages_match_reference():
    """Same exception type and message (file:line:col: text) as the reference's
    parser on malformed programs (tests/golden/ref_parse_errors.json)."""
    with open(os.path.join(GOLDEN, "ref_parse_errors.json")) as f:
        cases = json.load(f)
    assert len(cases) >= 35
    for c in cases:
        try:
            parse_program(c["src"])
            got = None
        except Exception as e:  # noqa: BLE001
            got = (type(e).__name__, str(e))
        want = None if c["error"] is None else (c["type"], c["error"])
        assert got == want, c["src"]
