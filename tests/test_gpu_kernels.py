"""GPU parity of the sm_100a kernels against the CPU oracle and the reference's
golden vectors (bit-exact transposes and integer sums; fp32 sums within the
north-star tolerance; the A.5 tree order bit-exact)."""
import numpy as np
import pytest

from oracle import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b2():
    import paper_2605_13864_b200 as b2
    return b2


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_golden_transposes_device(b2, golden):
    for c in golden:
        if c["kind"] != "transpose":
            continue
        a = c["inp"]
        if a.dtype == np.uint64:
            a = a.view(np.int64)
        out = b2.transpose(_dev(a)).cpu().numpy()
        assert out.tobytes() == c["out"].astype(a.dtype).tobytes(), c["id"]


def test_golden_reductions_device(b2, golden):
    for c in golden:
        if c["kind"] != "reduce":
            continue
        x = c["inp"]
        if "result_int" in c:
            got = int(b2.reduce_sum(_dev(x)).item())
            assert got == int(c["result_int"]), c["id"]
        elif "tree" in c["program"]:
            got = b2.reduce_tree512(_dev(x))
            assert np.float32(got).view(np.uint32) == np.uint32(c["result_f32_bits"]), c["id"]
        else:
            got = float(b2.reduce_sum(_dev(x)).item())
            exact, absum = oracle.sum_f64(x)
            assert abs(got - exact) <= oracle.f32_tolerance(x.size, exact, absum), c["id"]


SHAPES = [(1, 1), (1, 2**20), (2**20, 1), (33, 65), (1023, 1025), (64, 64), (128, 256),
          (4097, 8191), (4096, 4096), (100, 36), (8, 1000)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32, torch.float64])
def test_transpose_sweep(b2, shape, dt):
    g = torch.Generator(device="cuda").manual_seed(hash(shape) % 1000)
    a = torch.randn(shape, device="cuda", dtype=torch.float32, generator=g).to(dt)
    out = b2.transpose(a)
    torch.cuda.synchronize()
    ref = oracle.transpose(a.view(torch.int16 if dt == torch.bfloat16 else
                                  (torch.int32 if dt == torch.float32 else torch.int64)).cpu().numpy())
    got = out.view(torch.int16 if dt == torch.bfloat16 else
                   (torch.int32 if dt == torch.float32 else torch.int64)).cpu().numpy()
    assert np.array_equal(got, ref)


LOAD_SHAPES = [(64, 64), (256, 64), (300, 520), (4100, 4104), (1024, 2048), (8192, 1032), (520, 4096), (72, 9000)]


@pytest.mark.parametrize("setting", [(0, 0), (1, 0)] + [(2, v) for v in range(10)])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32, torch.float64])
def test_transpose_load_paths(b2, setting, dt):
    """Aligned interiors through every load path: the register-staged LDG tiles
    (transpose.cpa = 0), the default auto dispatch, and every cp.async geometry forced
    (transpose.cpa = 2): ragged tiles, pitched views whose neighbours must stay untouched;
    bit-exact against torch's transpose."""
    from paper_2605_13864_b200 import _lib
    cpa, variant = setting
    iv = {torch.bfloat16: torch.int16, torch.float32: torch.int32, torch.float64: torch.int64}[dt]
    _lib.tune("transpose.cpa", cpa)
    _lib.tune("transpose.cpa_variant", variant)
    try:
        for (r, c) in LOAD_SHAPES:
            g = torch.Generator(device="cuda").manual_seed(r * 31 + c)
            a = torch.randn((r, c), device="cuda", generator=g).to(dt)
            assert torch.equal(b2.transpose(a).view(iv), a.t().contiguous().view(iv)), (r, c)
            base = torch.randn((r, c + 32), device="cuda", generator=g).to(dt)
            view = base[:, 16:16 + c]  # pitch c + 32, 16-B aligned start for every width
            outb = torch.full((c, (r + 64 + 7) // 8 * 8), -7.0, device="cuda").to(dt)  # 16-B pitch
            b2.transpose(view, outb[:, 32:32 + r])
            assert torch.equal(outb[:, 32:32 + r].view(iv), view.t().contiguous().view(iv)), (r, c)
            assert bool((outb[:, :32] == -7).all()) and bool((outb[:, 32 + r:] == -7).all())
    finally:
        _lib.tune("transpose.cpa", 1)
        _lib.tune("transpose.cpa_variant", 0)


def test_transpose_pitched(b2):
    base = torch.arange(300 * 520, device="cuda", dtype=torch.float32).reshape(300, 520)
    view = base[:, 8:508]  # pitch 520, 16-B aligned start
    out = torch.full((520, 320), -1.0, device="cuda")
    b2.transpose(view, out[:500, :300])
    torch.cuda.synchronize()
    assert torch.equal(out[:500, :300], view.t())
    assert bool((out[:, 300:] == -1).all()) and bool((out[500:] == -1).all())
    odd = base[:, 3:400]  # misaligned start -> scalar path
    assert torch.equal(b2.transpose(odd), odd.t())


def test_degenerate_shapes_pitched(b2):
    row = torch.arange(100, device="cuda", dtype=torch.float32).reshape(1, 100)
    big = torch.zeros(100, 7, device="cuda")
    b2.transpose(row, big[:, 2:3])
    col = torch.arange(50, device="cuda", dtype=torch.float64).reshape(50, 1)
    wide = torch.zeros(5, 50, device="cuda", dtype=torch.float64)
    b2.transpose(torch.zeros(50, 9, device="cuda", dtype=torch.float64)[:, 4:5].copy_(col), wide[3:4])
    torch.cuda.synchronize()
    assert torch.equal(big[:, 2], row[0]) and float(big[:, [0, 1, 3]].abs().sum()) == 0
    assert torch.equal(wide[3], col[:, 0]) and float(wide[[0, 1, 2, 4]].abs().sum()) == 0


@pytest.mark.parametrize("n", [0, 1, 3, 17, 1000, 2**20 + 3, 2**24])
def test_reduce_int32_exact(b2, n):
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randint(-2**31, 2**31, (n,), device="cuda", dtype=torch.int64, generator=g).to(torch.int32)
    got = int(b2.reduce_sum(x).item())
    assert got == oracle.reduce_i32(x.cpu().numpy())


def test_reduce_int32_misaligned_views(b2):
    x = torch.randint(-2**31, 2**31, (100003,), device="cuda", dtype=torch.int64).to(torch.int32)
    for off in range(1, 4):
        v = x[off:]
        assert int(b2.reduce_sum(v).item()) == oracle.reduce_i32(v.cpu().numpy())


@pytest.mark.parametrize("n", [1, 7, 4096, 2**20, 2**24])
@pytest.mark.parametrize("lo", [0.0, -1.0])
def test_reduce_f32_tolerance(b2, n, lo):
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.rand((n,), device="cuda", generator=g) * (1 - lo) + lo
    got = float(b2.reduce_sum(x).item())
    xh = x.cpu().numpy()
    exact, absum = oracle.sum_f64(xh)
    assert abs(got - exact) <= oracle.f32_tolerance(n, exact, absum)
    # deterministic run to run
    assert float(b2.reduce_sum(x).item()) == got


@pytest.mark.parametrize("n", [512, 4096, 2**20, 2**24])
def test_tree512_bit_exact(b2, n):
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.rand((n,), device="cuda", generator=g) * 2 - 1
    want, parts = oracle.reduce_f32_tree512(x.cpu().numpy())
    got_parts = b2.reduce_tree512_partials(x).cpu().numpy()
    assert np.array_equal(got_parts.view(np.uint32), parts.view(np.uint32))
    assert np.float32(b2.reduce_tree512(x)).view(np.uint32) == np.float32(want).view(np.uint32)


def test_tree512_rejects_inexact(b2):
    with pytest.raises(b2.B2Error):
        b2.reduce_tree512(torch.ones(513, device="cuda"))


def test_reduce_f64(b2):
    x = torch.randn(1 << 20, device="cuda", dtype=torch.float64)
    got = float(b2.reduce_sum(x).item())
    assert abs(got - float(x.sum().item())) <= 1e-9 * float(x.abs().sum().item())


def test_host_paths(b2):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((3000, 2050)).astype(np.float32)
    assert np.array_equal(b2.transpose(a), a.T)
    xi = rng.integers(-2**31, 2**31, 5_000_001, dtype=np.int64).astype(np.int32)
    assert b2.reduce_sum(xi) == oracle.reduce_i32(xi)
    xf = rng.uniform(-1, 1, 1_000_003).astype(np.float32)
    exact, absum = oracle.sum_f64(xf)
    assert abs(b2.reduce_sum(xf) - exact) <= oracle.f32_tolerance(xf.size, exact, absum)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_paths_staging(b2, pinned):
    # pageable buffers go through the pinned staging ring + host copy pool; pinned
    # ones straight to the DMA engines; pitched sub-views of both directions
    from paper_2605_13864_b200 import _lib
    _lib.tune("host.chunk_mb", 1)  # many chunks: exercise ring reuse
    try:
        rng = np.random.default_rng(4)
        big_in = rng.standard_normal((700, 530)).astype(np.float32)
        big_out = np.full((520, 720), -3.0, dtype=np.float32)
        if pinned:
            t_in = torch.from_numpy(big_in).pin_memory()
            t_out = torch.from_numpy(big_out).pin_memory()
            big_in, big_out = t_in.numpy(), t_out.numpy()
        b2.transpose(big_in[:690, 4:524], big_out[:, 8:698])
        assert np.array_equal(big_out[:, 8:698], big_in[:690, 4:524].T)
        assert (big_out[:, :8] == -3).all() and (big_out[:, 698:] == -3).all()
        x = rng.uniform(-1, 1, 3 * 262144 + 512).astype(np.float32)
        want, _ = oracle.reduce_f32_tree512(x)
        assert np.float32(b2.reduce_tree512(x)).view(np.uint32) == np.float32(want).view(np.uint32)
        xi = rng.integers(-2**31, 2**31, 2_000_003, dtype=np.int64).astype(np.int32)
        assert b2.reduce_sum(xi) == oracle.reduce_i32(xi)
    finally:
        _lib.tune("host.chunk_mb", 64)


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.uint16])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("chunk_mb", [1, 3])
def test_host_transpose_2d_chunks(b2, dt, pinned, chunk_mb):
    """b2_transpose_host moves cr x cc blocks (>= 4 KB rows on both DMA sides):
    ragged last blocks, pitched sub-views, pinned and staged buffers."""
    from paper_2605_13864_b200 import _lib
    _lib.tune("host.chunk_mb", chunk_mb)
    try:
        rng = np.random.default_rng(7)
        big_in = rng.integers(0, 2**16, (1300, 3100)).astype(dt)
        big_out = np.zeros((3090, 1310), dtype=dt)
        if pinned:
            big_in = torch.from_numpy(big_in).pin_memory().numpy()
            big_out = torch.from_numpy(big_out).pin_memory().numpy()
        src = big_in[3:1298, 5:3085]
        dst = big_out[:3080, 7:1302]
        b2.transpose(src, dst)
        assert np.array_equal(dst, src.T)
        assert (big_out[:, :7] == 0).all() and (big_out[:, 1302:] == 0).all() and (big_out[3080:] == 0).all()
    finally:
        _lib.tune("host.chunk_mb", 64)


class _CAI:
    """Minimal foreign CUDA array (as CuPy / Numba expose it)."""

    def __init__(self, t):
        self._t = t
        self.__cuda_array_interface__ = {
            "shape": tuple(t.shape), "typestr": {torch.float32: "<f4", torch.int32: "<i4"}[t.dtype],
            "data": (t.data_ptr(), False), "version": 3,
            "strides": tuple(s * t.element_size() for s in t.stride())}


def test_cuda_array_interface_inputs(b2):
    a = torch.randn(300, 200, device="cuda")
    out = torch.empty(200, 300, device="cuda")
    b2.transpose(_CAI(a), _CAI(out))
    x = torch.randint(-2**31, 2**31, (10001,), device="cuda", dtype=torch.int64).to(torch.int32)
    s = b2.reduce_sum(_CAI(x))
    torch.cuda.synchronize()
    assert torch.equal(out, a.t())
    assert int(s.item()) == int(x.to(torch.int64).sum().item())


def test_launch_counter(b2):
    n0 = b2.launch_count()
    b2.reduce_sum(torch.ones(100, device="cuda"))
    torch.cuda.synchronize()
    assert b2.launch_count() == n0 + 1


_PATHS = {"staged": {"transpose.any": 0, "transpose.staged": 2},
          "scalar": {"transpose.any": 0, "transpose.staged": 0},
          "any": {"transpose.any": 1, "transpose.staged": 0}}


def _with_path(path, fn):
    from paper_2605_13864_b200 import _lib
    for k, v in _PATHS[path].items():
        _lib.tune(k, v)
    try:
        return fn()
    finally:
        _lib.tune("transpose.any", 0)
        _lib.tune("transpose.staged", 1)


@pytest.mark.parametrize("path", ["staged", "scalar", "any"])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("rows,cols,oin,oout", [(63, 65, 1, 3), (130, 257, 3, 0), (1, 77, 1, 1), (77, 2, 0, 1),
                                                (129, 129, 5, 7), (2000, 3, 1, 0), (3, 2000, 0, 2),
                                                (1025, 1023, 7, 5)])
def test_unaligned_views(b2, path, dt, rows, cols, oin, oout):
    # misaligned bases and odd pitches: the cp.async-staged kernel (default), the
    # padded scalar tile and the funnel-shift kernel; neighbours of the output view
    # must stay untouched
    iv = {torch.bfloat16: torch.int16, torch.float32: torch.int32, torch.float64: torch.int64}[dt]
    src = torch.randn(rows, cols + oin + 3, device="cuda").to(dt)
    view = src[:, oin:oin + cols]
    dst = torch.full((cols, rows + oout + 5), 7.0, device="cuda").to(dt)
    oview = dst[:, oout:oout + rows]
    _with_path(path, lambda: b2.transpose(view, oview))
    torch.cuda.synchronize()
    assert torch.equal(oview.view(iv), view.t().contiguous().view(iv))
    rest = torch.cat([dst[:, :oout].reshape(-1), dst[:, oout + rows:].reshape(-1)])
    assert bool((rest == 7.0).all())


@pytest.mark.parametrize("stages,ctas", [(4, 0), (3, 3), (2, 1)])
@pytest.mark.parametrize("dt", [torch.int16, torch.int32, torch.int64])
@pytest.mark.parametrize("rows,cols", [(4097, 8191), (16385, 16383), (777, 100003), (100003, 65), (64, 129)])
def test_staged_odd_pitch_full(b2, stages, ctas, dt, rows, cols):
    """The cp.async-staged kernel on the C5 odd shapes (every pitch odd, so every
    row starts at a different 16-B phase), all ring depths / residencies, whole
    result against the CPU oracle."""
    from paper_2605_13864_b200 import _lib
    if dt == torch.int64 and rows * cols > 1 << 28:
        pytest.skip("covered by the 2-/4-byte cases")
    info = torch.iinfo(dt)
    a = torch.randint(info.min, info.max, (rows, cols), device="cuda", dtype=dt)
    _lib.tune("transpose.staged_stages", stages)
    _lib.tune("transpose.staged_ctas", ctas)
    _lib.tune("transpose.staged", 2)
    _lib.tune("transpose.staged_geom", 6)  # the 64-row ring at every size
    try:
        t = b2.transpose(a)
    finally:
        _lib.tune("transpose.staged_stages", 4)
        _lib.tune("transpose.staged_ctas", 0)
        _lib.tune("transpose.staged", 1)
        _lib.tune("transpose.staged_geom", 0)
    assert np.array_equal(t.cpu().numpy(), oracle.transpose(a.cpu().numpy()))



@pytest.mark.parametrize("geom", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("dt", [torch.int16, torch.int32, torch.int64])
@pytest.mark.parametrize("rows,cols,oin,oout", [(4097, 8191, 0, 0), (777, 10003, 3, 1), (300, 65, 1, 2),
                                                (64, 129, 0, 5), (5000, 31, 7, 0)])
def test_staged_geometries(b2, geom, dt, rows, cols, oin, oout):
    """Every tile geometry of the staged kernel (64 / 128 / 256 tile rows, ring depth,
    residency, L2 hint) on odd pitches and misaligned views: whole result against the
    CPU oracle, neighbours of the output view untouched."""
    from paper_2605_13864_b200 import _lib
    info = torch.iinfo(dt)
    src = torch.randint(info.min, info.max, (rows, cols + oin + 3), device="cuda", dtype=dt)
    view = src[:, oin:oin + cols]
    dst = torch.full((cols, rows + oout + 5), 7, device="cuda", dtype=dt)
    oview = dst[:, oout:oout + rows]
    _lib.tune("transpose.staged_geom", geom)
    _lib.tune("transpose.staged", 2)
    try:
        b2.transpose(view, oview)
    finally:
        _lib.tune("transpose.staged_geom", 0)
        _lib.tune("transpose.staged", 1)
    assert np.array_equal(oview.contiguous().cpu().numpy(), oracle.transpose(view.contiguous().cpu().numpy()))
    rest = torch.cat([dst[:, :oout].reshape(-1), dst[:, oout + rows:].reshape(-1)])
    assert bool((rest == 7).all())


@pytest.mark.parametrize("shape", [(64, 64), (1000, 1000), (333, 516), (4096, 4096), (100, 36), (65, 4100)])
def test_tma_transpose_path(b2, shape):
    from paper_2605_13864_b200 import _lib
    _lib.tune("transpose.tma", 1)
    try:
        a = torch.randn(shape, device="cuda")
        out = b2.transpose(a)
        base = torch.zeros(shape[0], shape[1] + 12, device="cuda")
        view = base[:, 4:4 + shape[1]]  # 16-B aligned start, pitched
        view.copy_(a)
        out2 = torch.full((shape[1], shape[0] + 4), -1.0, device="cuda")
        b2.transpose(view, out2[:, :shape[0]])
        torch.cuda.synchronize()
        assert torch.equal(out, a.t())
        assert torch.equal(out2[:, :shape[0]], a.t()) and bool((out2[:, shape[0]:] == -1).all())
    finally:
        _lib.tune("transpose.tma", 0)


@pytest.mark.parametrize("variant", list(range(10)))
def test_reduce_variants_heads_and_tails(b2, variant):
    """Every reduce instantiation (incl. the 256-bit-load ones, LDG.E.256, whose
    head aligns to 32 B) over misaligned starts and ragged lengths."""
    from paper_2605_13864_b200 import _lib
    _lib.tune("reduce.variant", variant)
    try:
        rng = np.random.default_rng(variant)
        x = rng.integers(-2**31, 2**31, 200_017, dtype=np.int64).astype(np.int32)
        xf = rng.uniform(-1, 1, 200_017).astype(np.float32)
        t, tf = torch.from_numpy(x).cuda(), torch.from_numpy(xf).cuda()
        for off in range(8):
            for n in (0, 1, 7, 8, 9, 15, 16, 17, 31, 33, 1000, 65_537, 200_000):
                assert int(b2.reduce_sum(t[off:off + n]).item()) == int(x[off:off + n].astype(np.int64).sum())
            seg = xf[off:off + 123_457]
            exact, absum = oracle.sum_f64(seg)
            got = float(b2.reduce_sum(tf[off:off + 123_457]).item())
            assert abs(got - exact) <= oracle.f32_tolerance(seg.size, exact, absum)
    finally:
        _lib.tune("reduce.variant", 0)


@pytest.mark.parametrize("stages", [2, 3, 4, 6, 7, 8])
def test_tma_register_transpose_path(b2, stages):
    """transpose.tma = 2: TMA-loaded input stages, lane-rotated conflict-free LDS,
    register transpose, direct 128-bit stores; ragged tiles clipped by TMA."""
    from paper_2605_13864_b200 import _lib
    _lib.tune("transpose.tma", 2)
    _lib.tune("transpose.tma_stages", stages)
    try:
        for R, C in [(512, 256), (1000, 772), (4100, 132), (132, 4100), (2048, 3072)]:
            a = torch.rand((R, C), device="cuda")
            assert torch.equal(b2.transpose(a), a.t()), (R, C)
        a = torch.rand((1001, 771), device="cuda")  # not multiples of 4: falls back to the LDG path
        assert torch.equal(b2.transpose(a), a.t())
    finally:
        _lib.tune("transpose.tma", 0)
        _lib.tune("transpose.tma_stages", 2)
