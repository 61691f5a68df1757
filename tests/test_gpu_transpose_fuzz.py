"""Randomised transposes through every dispatch path (GPU): cell width, shape, base
offset, row pitch of both sides and the path knob are drawn per case; each result is
compared bit for bit with torch's transpose, and the cells around the output view
(pitch padding, leading offset) must be left untouched. Paths: the default dispatch,
the LDG tiles (every tile variant), the cp.async tiles (every forced geometry), the
cp.async-staged odd-pitch kernel (every geometry), the padded scalar tile, the
funnel-shift kernel and the TMA variants (4-byte cells)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DTYPES = [(torch.int16, 2), (torch.int32, 4), (torch.int64, 8)]


def _paths(esize):
    p = [{}]
    p += [{"transpose.cpa": 0, "transpose.variant": v} for v in range(11)]
    p += [{"transpose.cpa": 2, "transpose.cpa_variant": v} for v in range(12)]
    p += [{"transpose.staged": 2, "transpose.staged_geom": g} for g in range(7)]
    p += [{"transpose.staged": 0}, {"transpose.any": 1, "transpose.staged": 0}]
    if esize == 4:
        p += [{"transpose.tma": 1}, {"transpose.tma": 2}]
    return p


RESET = {"transpose.cpa": 1, "transpose.cpa_variant": 0, "transpose.variant": 0, "transpose.staged": 1,
         "transpose.staged_geom": 0, "transpose.any": 0, "transpose.tma": 0}


@pytest.mark.parametrize("seed", range(20))
def test_random_transposes_every_path(seed):
    import paper_2605_13864_b200 as b2
    from paper_2605_13864_b200 import _lib
    rng = np.random.default_rng(1000 + seed)
    for case in range(60):
        dt, esize = DTYPES[rng.integers(len(DTYPES))]
        paths = _paths(esize)
        knobs = paths[rng.integers(len(paths))]
        rows = int(rng.choice([1, 2, 3, 31, 64, 65, 127, 256, 300, 517, 1024, 1500]))
        cols = int(rng.choice([1, 2, 5, 32, 63, 64, 129, 256, 333, 640, 1030, 2048]))
        oin, oout = int(rng.integers(0, 9)), int(rng.integers(0, 9))
        pin, pout = int(rng.integers(0, 11)), int(rng.integers(0, 11))
        info = torch.iinfo(dt)
        src = torch.randint(info.min, info.max, (rows * (cols + pin) + oin + 8,), device="cuda", dtype=dt)
        view = src[oin:oin + rows * (cols + pin)].view(rows, cols + pin)[:, :cols]
        dst = torch.full((cols * (rows + pout) + oout + 8,), 7, device="cuda", dtype=dt)
        oview = dst[oout:oout + cols * (rows + pout)].view(cols, rows + pout)[:, :rows]
        for k, v in knobs.items():
            _lib.tune(k, v)
        try:
            b2.transpose(view, oview)
        finally:
            for k, v in RESET.items():
                _lib.tune(k, v)
        torch.cuda.synchronize()
        tag = (seed, case, str(dt), rows, cols, oin, oout, pin, pout, knobs)
        assert torch.equal(oview, view.t()), tag
        mask = torch.ones_like(dst, dtype=torch.bool)
        mask[oout:oout + cols * (rows + pout)].view(cols, rows + pout)[:, :rows] = False
        assert bool((dst[mask] == 7).all()), tag
