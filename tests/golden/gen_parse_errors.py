"""Reference parse-error messages (minigpu.parser.parse_program, parser.py:893)
for malformed programs -> tests/golden/ref_parse_errors.json. Build container only:

    python tests/golden/gen_parse_errors.py
"""
import json
import os
import sys

sys.path.insert(0, os.environ.get("MINIGPU_REF", "/root/reference/pkg/src"))
from minigpu.parser import parse_program  # noqa: E402  (reference)

HERE = os.path.dirname(os.path.abspath(__file__))
BAD = [
    "void f( { }",
    "void f() { for (int i = 0; j < 3; i++) { } }",
    "void f() { x = ; }",
    "void f() { float* a = notalloc1<float>(3); }",
    "void f() { float* a = MALLOC2<float>(3); }",
    "void f() { }  void f() { }",
    "void f() { for (int i = 0; i < 2; i++) { for (int i = 0; i < 2; i++) { } } }",
    "void f() { return }",
    "void f() { int x = 3 }",
    "float f(float* a) { a[0] = 1.0 }",
    "void f() { if (x) { } else }",
    "void f() { for (int i = 0; i < 3; i--) { } }",
    "void f() { for (i = 0; i < 3; i++) { } }",
    "void f() { thread (int i = 0; i < 3; i++) { } }",
    "void f() { magic for (int i = 0; i < 3; i++) { } }",
    "double f() { }",
    "void f(int) { }",
    "void f(int a,) { }",
    "void f() { a[1 = 2; }",
    "void f() { a = b +; }",
    "void f() { a = (b; }",
    "void f() { a = @; }",
    "void f() { __ghost(); }",
    "__pure(3);",
    "__axiom(\"x\");",
    "void f() { float* const a = gmem_malloc1<float>(); }",
    "void f() { x += ; }",
    "void f() { x = 1; } extra",
    "void f() { for (int i = 0; i < 3; i++) }",
    "void f() { { }",
    "void f() {",
    "void f() { y = fun x -> ; }",
    "void f() { a[0][ = 1; }",
    "int f() { return 1.5.5; }",
    "void f() { int 3x = 1; }",
    "void f() { a ! b; }",
    "void f() {\n  int x = 1;\n  y = x *;\n}",
]


def main():
    out = []
    for src in BAD:
        try:
            parse_program(src)
            out.append({"src": src, "error": None})
        except Exception as e:  # noqa: BLE001
            out.append({"src": src, "type": type(e).__name__, "error": str(e)})
    with open(os.path.join(HERE, "ref_parse_errors.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(len(out), "cases")


if __name__ == "__main__":
    main()
