"""The maintainer-side ctypes stub printed in INTEGRATION.md §2 actually works:
extract it, point it at the in-tree libb200k.so and call its three functions."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle

pytestmark = pytest.mark.gpu


def _stub_source():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as f:
        text = f.read()
    m = re.search(r"```python\n# minigpu/_b200\.py.*?\n(.*?)```", text, re.S)
    assert m, "stub not found in INTEGRATION.md"
    lib = os.path.join(ROOT, "paper_2605_13864_b200", "libb200k.so")
    return m.group(1).replace('ctypes.CDLL("libb200k.so")', f"ctypes.CDLL({lib!r})")


def test_integration_stub_runs():
    ns = {}
    exec(compile(_stub_source(), "INTEGRATION.md:_b200.py", "exec"), ns)
    rng = np.random.default_rng(0)
    a = rng.standard_normal((300, 517)).astype(np.float32)
    assert np.array_equal(ns["transpose"](a), a.T)
    x = rng.integers(-2**31, 2**31, 100_003, dtype=np.int64).astype(np.int32)
    assert ns["reduce_int"](x) == oracle.reduce_i32(x)
    xf = rng.uniform(-1, 1, 512 * 33).astype(np.float32)
    want, _ = oracle.reduce_f32_tree512(xf)
    assert np.float32(ns["reduce_tree512"](xf)).view(np.uint32) == np.float32(want).view(np.uint32)
