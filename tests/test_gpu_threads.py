"""Concurrent host threads on one device (ctypes releases the GIL, so the calls
really overlap): the host-buffer pipelines run on one of the device's two pipeline
lanes each (a third concurrent call waits for lane 0),
device calls on per-thread streams with per-thread reduce workspaces run
concurrently, and run_program is re-entrant. Every result is checked against the
CPU oracle; none may be torn or mixed up between threads."""
import threading

import numpy as np
import pytest

from conftest import program_text
from oracle import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NT = 6
_oracle_mu = threading.Lock()  # the oracle's C thread pool is not re-entrant


def _t(a):
    with _oracle_mu:
        return oracle.transpose(a).view(np.uint32).tobytes()


def _s(x):
    with _oracle_mu:
        return oracle.reduce_i32(x)


def _run_threads(work):
    errs = []

    def wrap(k):
        try:
            work(k)
        except BaseException as e:  # noqa: BLE001 - reported below
            errs.append((k, repr(e)))

    ts = [threading.Thread(target=wrap, args=(k,)) for k in range(NT)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


def test_host_pipelines_from_threads():
    import paper_2605_13864_b200 as b2

    def work(k):
        rng = np.random.default_rng(100 + k)
        for it in range(4):
            r, c = 700 + 97 * k + it, 1500 - 61 * k
            a = rng.integers(0, 2**32, (r, c), dtype=np.uint32).view(np.float32)
            out = b2.transpose(a)
            assert out.view(np.uint32).tobytes() == _t(a), (k, it)
            x = rng.integers(-2**31, 2**31, 300_000 + 4099 * k, dtype=np.int32)
            assert b2.reduce_sum(x) == _s(x), (k, it)

    _run_threads(work)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_pipelines_on_lanes(pinned):
    """Many-chunk host pipelines (1 MiB stages) of every kind at once — transposes,
    int / fp32 sums, A.5 tree sums — so two lanes stream concurrently and further
    calls queue for lane 0; pageable sources go through each lane's own pinned ring."""
    import paper_2605_13864_b200 as b2
    from paper_2605_13864_b200 import _lib

    def buf(a):
        if not pinned:
            return a
        t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    def work(k):
        rng = np.random.default_rng(500 + k)
        for it in range(3):
            if k % 3 == 0:
                a = buf(rng.integers(0, 2**32, (1300 + k, 900 + 7 * it), dtype=np.uint32).view(np.float32))
                out = b2.transpose(a)
                assert out.view(np.uint32).tobytes() == _t(a), (k, it)
            elif k % 3 == 1:
                x = buf(rng.integers(-2**31, 2**31, 1_500_000 + 1031 * k, dtype=np.int32))
                assert b2.reduce_sum(x) == _s(x), (k, it)
            else:
                x = buf(rng.uniform(-1, 1, 512 * (3000 + k)).astype(np.float32))
                with _oracle_mu:
                    want, _ = oracle.reduce_f32_tree512(x)
                got = b2.reduce_tree512(x)
                assert np.float32(got).view(np.uint32) == np.float32(want).view(np.uint32), (k, it)

    prev = _lib.tuning("host.chunk_mb")
    _lib.tune("host.chunk_mb", 1)
    try:
        _run_threads(work)
    finally:
        _lib.tune("host.chunk_mb", prev)


def test_device_calls_on_per_thread_streams():
    import paper_2605_13864_b200 as b2
    from paper_2605_13864_b200 import _lib

    def work(k):
        g = torch.Generator(device="cuda").manual_seed(k)
        s = torch.cuda.Stream()
        n = (1 << 22) + 333 * k
        with torch.cuda.stream(s):
            ws = torch.zeros(b2.reduce_ws_bytes(n, _lib.I32), dtype=torch.uint8, device="cuda")
            a = torch.randint(-2**31, 2**31 - 1, (1024 + k, 2048 - k), device="cuda", dtype=torch.int32,
                              generator=g).view(torch.float32)
            x = torch.randint(-2**31, 2**31 - 1, (n,), device="cuda", dtype=torch.int32, generator=g)
            for _ in range(5):
                o = b2.transpose(a, stream=s)
                r = b2.reduce_sum(x, ws=ws, stream=s)
        s.synchronize()
        ah, xh = a.cpu().numpy(), x.cpu().numpy()
        assert o.cpu().numpy().view(np.uint32).tobytes() == _t(ah), k
        assert int(r.item()) == _s(xh), k

    _run_threads(work)


def test_run_program_reentrant():
    import paper_2605_13864_b200 as b2
    tprog = b2.parse_program(program_text("transpose_naive.optc"))
    rprog = b2.parse_program(program_text("reduce_naive_int.optc"))

    def work(k):
        rng = np.random.default_rng(7 * k)
        H, W = 33 + k, 65 - k
        a = rng.standard_normal((H, W)).astype(np.float32)
        _, outs = b2.run_program(tprog, "transpose", {"in": b2.Array([H, W], a.reshape(-1).tolist(), "float"),
                                                      "out": b2.Array.alloc([W, H], "float"), "W": W, "H": H})
        assert outs["out"] == a.T.reshape(-1).tolist(), k
        x = rng.integers(-2**31, 2**31, 5000 + k, dtype=np.int64).tolist()
        ret, _ = b2.run_program(rprog, "reduce", {"arr": x, "N": len(x)})
        assert ret == sum(x), k

    _run_threads(work)


def test_generated_program_from_threads():
    """generated programs keep per-call state in statics of their .so;
    concurrent calls of the SAME compiled program must neither free each other's
    allocations nor mix up results."""
    import paper_2605_13864_b200 as b2
    prog = b2.parse_program(program_text("transpose_gpu.optc"))

    def work(k):
        rng = np.random.default_rng(50 + k)
        H, W = 32 * (2 + k), 32 * (5 - k % 3)
        for it in range(3):
            a = rng.standard_normal((H, W)).astype(np.float32)
            _, outs = b2.run_program(prog, "transpose", {"in": b2.Array([H, W], a.reshape(-1).tolist(), "float"),
                                                         "out": b2.Array.alloc([W, H], "float"), "W": W, "H": H},
                                     backend="codegen")
            assert outs["out"] == a.T.reshape(-1).tolist(), (k, it)

    _run_threads(work)
