"""K1 parity on the GPU: fused_kernel (the reference's kernels.cpp:27-145
contract) against the CPU oracle, bit-exact, for every kernel family the
engine dispatches. The oracle is the checker only."""
import numpy as np
import pytest

import paper_2309_08864_b200 as so2dr

pytestmark = pytest.mark.gpu


def _spec_and_oracle(kind, r, dtype, dim=2, seed=0):
    """(engine spec, oracle kind, oracle weights)"""
    import pyoracle as o

    if kind == "box":
        w = o.box_weights(r, dim, dtype)
        return so2dr.StencilSpec.box(r, w, dim), o.BOX, w
    if kind == "boxrand":
        rng = np.random.default_rng(seed)
        w = rng.uniform(-0.3, 0.5, (2 * r + 1) ** dim).astype(dtype).astype(np.float64)
        return so2dr.StencilSpec.box(r, w, dim), o.BOX, w
    if kind == "star":  # a box with zero off-axis weights (reference API) -> star kernel
        w = o.star_weights(r, dim, dtype)
        return so2dr.StencilSpec.box(r, w, dim), o.BOX, w
    if kind == "gradient":
        return so2dr.StencilSpec.gradient(), o.GRADIENT, np.zeros(9)
    raise ValueError(kind)


def _bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _check_region(engine, oracle, kind, r, steps, region, dtype=np.float32, sz=70, tile=16, seed=3):
    spec, okind, w = _spec_and_oracle(kind, r, dtype, seed=seed)
    g = oracle.init_grid(sz, r, seed, 2, dtype)
    p = g.shape[0]
    b0, b1 = g.copy(), g.copy()
    interior = (r, p - r, r, p - r)
    engine.fused_kernel(spec, b0, b1, 0, 0, steps, tile, region, interior, region)
    want = oracle.run(g, okind, r, w, steps)
    y0, y1, x0, x1 = region
    got = b1[y0:y1, x0:x1]
    exp = want[y0:y1, x0:x1]
    bad = np.argwhere(_bits(got) != _bits(exp))
    assert bad.size == 0, f"{kind} r={r} s={steps} {dtype.__name__}: {len(bad)} diffs, first {bad[:3] + [y0, x0]}"
    # write buffer untouched outside the region; read buffer untouched
    mask = np.ones_like(b1, dtype=bool)
    mask[y0:y1, x0:x1] = False
    assert (_bits(b1)[mask] == _bits(g)[mask]).all()
    assert (_bits(b0) == _bits(g)).all()


CASES_F32 = [("box", 1), ("box", 2), ("box", 3), ("box", 4), ("star", 1), ("star", 2), ("star", 3),
             ("star", 4), ("gradient", 1), ("boxrand", 1), ("boxrand", 2)]


@pytest.mark.parametrize("kind,r", CASES_F32)
def test_fused_full_width_all_steps(engine, oracle, kind, r):
    for steps in range(1, 10):
        p = 70 + 2 * r
        _check_region(engine, oracle, kind, r, steps, (r, p - r, 0, p))


@pytest.mark.parametrize("kind,r", CASES_F32)
def test_fused_subregions(engine, oracle, kind, r):
    rng = np.random.default_rng(100 + r)
    p = 70 + 2 * r
    for _ in range(6):
        steps = int(rng.integers(1, 9))
        y0 = int(rng.integers(0, p - 2))
        y1 = int(rng.integers(y0 + 1, p + 1))
        x0 = int(rng.integers(0, p - 2))
        x1 = int(rng.integers(x0 + 1, p + 1))
        _check_region(engine, oracle, kind, r, steps, (y0, y1, x0, x1), seed=int(rng.integers(1 << 30)))


@pytest.mark.parametrize("kind,r", [("box", 1), ("box", 2), ("star", 2), ("gradient", 1), ("box", 3)])
def test_fused_f64(engine, oracle, kind, r):
    for steps in (1, 2, 3, 5, 8):
        p = 50 + 2 * r
        _check_region(engine, oracle, kind, r, steps, (r, p - r, 0, p), dtype=np.float64, sz=50)


def test_fused_wide_grid_multi_cta(engine, oracle):
    # several column strips and y segments per launch
    for kind, r, steps in [("box", 1, 8), ("star", 1, 4), ("gradient", 1, 5), ("box", 2, 6)]:
        sz = 2100
        p = sz + 2 * r
        _check_region(engine, oracle, kind, r, steps, (r, p - r, 0, p), sz=sz, seed=11)


def test_fused_stats_match_reference(engine, oracle):
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    import ctypes

    R = oracle.ref()
    g = oracle.init_grid(62, 1, 9)
    for region, s, tile in [((20, 36, 20, 36), 2, 8), ((10, 26, 8, 40), 1, 64), ((1, 63, 0, 64), 3, 16),
                            ((5, 60, 3, 61), 4, 32)]:
        b0, b1 = g.copy(), g.copy()
        st = engine.fused_kernel(so2dr.StencilSpec.box(1), b0, b1, 0, 0, s, tile, region, (1, 63, 1, 63), region)
        r0, r1 = g.copy(), g.copy()
        stats = (ctypes.c_uint64 * 4)()
        reg = (ctypes.c_int * 4)(*region)
        inter = (ctypes.c_int * 4)(1, 63, 1, 63)
        err = ctypes.create_string_buffer(256)
        rc = R.ref_fused_kernel(0, 1, None, r0.ctypes.data, r1.ctypes.data, 0, 64, 64, 0, s, tile, reg, inter, reg,
                                stats, None, err, 256)
        assert rc == 0, err.value
        assert [st["scratch_load"], st["scratch_store"], st["updates"], st["redundant"]] == list(stats)
        assert (_bits(b1) == _bits(r1)).all()


def test_growing_zero_corner_box_keeps_box_chain(engine, oracle):
    """a box spec with zero off-axis weights whose weights can grow the
    field (all-ones star: sum|w| = 5) must NOT take the star shortcut -- once the
    field overflows to inf, the reference chain's fma(0, inf, acc) is NaN. 64
    steps of 5x growth overflow fp32; the engine must match the oracle's box chain
    (non-NaN cells bit-exact, NaN exactly where the oracle has NaN)."""
    w = np.zeros(9)
    w[[1, 3, 4, 5, 7]] = 1.0
    spec = so2dr.StencilSpec.box(1, w)
    g = oracle.init_grid(64, 1, 5, 2, np.float32)
    want = oracle.run(g, oracle.BOX, 1, w, 64)
    got = g.copy()
    engine.run("incore", got, spec, so2dr.RunConfig(sz=64, r=1, d=1, s_tb=8, k_on=4, n_strm=1, n=64),
               so2dr.KernelPlan(4, 32))
    assert np.isnan(want).any()  # overflowed to inf, then 0*inf = NaN spread
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert (_bits(got)[ok] == _bits(want)[ok]).all()
