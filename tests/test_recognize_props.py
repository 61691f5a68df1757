"""Property tests of the recogniser (hypothesis): any consistent renaming of a
hot-path program's identifiers, in any parameter order, is recognised with the
right role mapping; changing a single literal is refused (the program would
compute something else)."""
import re

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2605_13864_b200 import parse_program, programs, recognize
from paper_2605_13864_b200.recognize import UnsupportedProgram

KEYWORDS = {"void", "float", "int", "for", "thread", "if", "return", "const"}
INTRINSICS = {"gmem_malloc1", "gmem_malloc2", "__smem_malloc1", "__smem_malloc2", "MALLOC1",
              "memcpy_host_to_device1", "memcpy_host_to_device2", "memcpy_device_to_host1",
              "memcpy_device_to_host2", "kernel_launch", "kernel_setup_end", "kernel_teardown_begin",
              "kernel_kill", "blocksync", "__smem_free1", "__smem_free2", "free", "gmem_free",
              "DMINDEX1", "DMINDEX2", "pow2", "transpose", "reduce"}
SOURCES = {
    "transpose_naive": programs.TRANSPOSE_NAIVE,
    "transpose_gpu": programs.TRANSPOSE_GPU,
    "reduce_naive_f32": programs.REDUCE_NAIVE_F32,
    "reduce_naive_int": programs.REDUCE_NAIVE_INT,
    "reduce_tree": programs.REDUCE_TREE_F32,
}
IDENT = re.compile(r"\b[A-Za-z_]\w*\b")


def idents(src):
    return sorted({m for m in IDENT.findall(src) if m not in KEYWORDS and m not in INTRINSICS})


def rename(src, mapping):
    return IDENT.sub(lambda m: mapping.get(m.group(0), m.group(0)), src)


def permute_params(src, order):
    m = re.search(r"\(([^()]*)\)\s*\{", src)
    params = [p.strip() for p in m.group(1).split(",")]
    new = ", ".join(params[i] for i in order)
    return src[:m.start(1)] + new + src[m.end(1):]


names = st.from_regex(r"[a-z][a-z0-9_]{0,6}", fullmatch=True).filter(
    lambda s: s not in KEYWORDS and s not in INTRINSICS)


@pytest.mark.parametrize("key", sorted(SOURCES))
@settings(max_examples=25, deadline=None)
@given(data=st.data())
def test_renaming_and_param_order_are_recognised(key, data):
    src = SOURCES[key]
    ids = idents(src)
    fresh = data.draw(st.lists(names, min_size=len(ids), max_size=len(ids), unique=True))
    mapping = dict(zip(ids, fresh))
    p = parse_program(src)
    roles = recognize(p, p.entry().name).params
    nparams = len(p.entry().params)
    order = data.draw(st.permutations(list(range(nparams))))
    src2 = permute_params(rename(src, mapping), order)
    p2 = parse_program(src2)
    plan = recognize(p2, p2.entry().name)
    assert plan.params == {role: mapping[name] for role, name in roles.items()}


LITERAL = re.compile(r"(?<![\w.])(\d+)(?![\w.])")


@pytest.mark.parametrize("key", ["transpose_gpu", "reduce_tree"])
@settings(max_examples=30, deadline=None)
@given(data=st.data())
def test_changing_one_literal_is_refused(key, data):
    src = SOURCES[key]
    lits = list(LITERAL.finditer(src))
    m = data.draw(st.sampled_from(lits))
    old = int(m.group(1))
    new = data.draw(st.integers(0, 4096).filter(lambda v: v != old))
    src2 = src[:m.start(1)] + str(new) + src[m.end(1):]
    try:
        p = parse_program(src2)
    except Exception:
        return  # e.g. MALLOC1 -> MALLOC2 arity change: not even a program
    with pytest.raises(UnsupportedProgram):
        recognize(p, p.entry().name)
