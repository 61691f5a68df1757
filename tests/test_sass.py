"""Static SASS properties of the built library (no GPU needed: cuobjdump of the
in-tree libb200k.so): the default kernels keep their 128-bit loads, 256-bit
evict-first stores and swizzled 128-bit shared-memory traffic, and nothing spills."""
import re
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2605_13864_b200", "libb200k.so")
pytestmark = pytest.mark.skipif(not (os.path.exists(LIB) and shutil.which("cuobjdump")),
                                reason="needs the built library and cuobjdump")


@pytest.fixture(scope="module")
def table():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import sass_evidence
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "--dump-resource-usage", LIB], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for ln in sass.splitlines():
        if "Function : " in ln:
            cur = ln.split("Function : ")[1].strip()
            funcs[cur] = []
        elif cur:
            funcs[cur].append(ln)
    dem = dict(zip(funcs, sass_evidence.demangle(list(funcs))))
    return funcs, dem, res


def _body(table, prefix):
    funcs, dem, _ = table
    hits = [k for k, d in dem.items() if prefix in d]
    assert hits, prefix
    return "\n".join(funcs[hits[0]])


def test_bench_transpose_vector_memory_ops(table):
    for k in ("transpose_vec_kernel<4, 64, 32, 512>", "transpose_vec_kernel<8, 128, 32, 512>"):
        b = _body(table, k)
        assert "LDG.E.NA.128" in b and ".EFL2.256" in b, k
        assert "STS.128" in b and "LDS.128" in b, k


def test_cpa_transpose_async_copies(table):
    """The default large-matrix transpose (transpose_cpa.cu): tiles land in shared
    memory by cp.async (LDGSTS, no register staging), one barrier per tile, scalar
    conflict-free gathers, 256-bit evict-first stores; every cell width."""
    for k in ("transpose_cpa_kernel<4, 256, 16, 256, 2, 1>", "transpose_cpa_kernel<8, 256, 16, 256, 2, 1>",
              "transpose_cpa_kernel<2, 128, 16, 512, 4, 1>"):
        b = _body(table, k)
        assert "LDGSTS.E.BYPASS.128" in b and "LDGDEPBAR" in b and "DEPBAR.LE" in b, k
        assert "BAR.SYNC" in b and "LDS" in b and not re.search(r"\bSTS\b", b) and "LDG.E" not in b, k
        assert ".EFL2.256" in b or k.startswith("transpose_cpa_kernel<2"), k


def test_reduce_vector_loads_and_shuffles(table):
    b = _body(table, "reduce_kernel<int, 512, 4, 1>")
    assert "LDG.E.NA.128" in b and "SHFL.DOWN" in b and "BAR.SYNC" in b


def test_no_register_spills(table):
    _, _, res = table
    assert "LOCAL:" in res
    spills = [ln for ln in res.splitlines() if "LOCAL:" in ln and "LOCAL:0 " not in ln]
    assert not spills, spills[:3]


def test_tma_variant_and_tree_kernel(table):
    """The TMA-staged transpose variant really issues bulk tensor copies with
    mbarrier synchronisation on sm_100a, and the A.5 tree kernel evaluates its
    lane levels with warp shuffles."""
    b = _body(table, "transpose_tmar_kernel<256, 2, 2>")
    assert "UTMALDG" in b and "SYNCS" in b
    assert "SHFL" in _body(table, "tree_kernel<512, 256>")


def test_staged_odd_pitch_kernel_uses_cp_async(table):
    """The 2-byte odd-pitch path fetches 16-B chunks with cp.async (LDGSTS) into its
    shared-memory ring and waits on commit groups (DEPBAR), one barrier per tile."""
    for k in ("transpose_staged_kernel<unsigned short, 64, 128, 256, 4, 0>",    # 2-byte, >= 2^22 cells
              "transpose_staged_kernel<unsigned int, 128, 64, 256, 2, 0>",      # any width, > 256 MB
              "transpose_staged_kernel<unsigned long, 128, 32, 256, 2, 0>"):
        b = _body(table, k)
        assert "LDGSTS.E.BYPASS.128" in b and "DEPBAR" in b and "BAR.SYNC" in b, k


def test_fp32_sum_accumulates_in_binary64(table):
    """fp32 cells are widened (F2F.F64.F32) and added in binary64 (DADD)."""
    b = _body(table, "reduce_kernel<float, 512, 4, 1>")
    assert "F2F.F64.F32" in b and "DADD" in b
