"""3D (z-streamed) and fp64 paths of the device engine against the restated
CPU oracle. There is no reference implementation for either;
the oracle is pinned to the reference through its 2D / known-answer cases
(tests/test_host.py), and here the 3D engine is additionally checked against
the 2D reference semantics on the degenerate case (dz != 0 weights zero)."""
import numpy as np
import pytest

import paper_2309_08864_b200 as so2dr

pytestmark = pytest.mark.gpu


def _bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _spec3(kind, r, dtype):
    import pyoracle as o

    if kind == "box":
        w = o.box_weights(r, 3, dtype)
    elif kind == "star":
        w = o.star_weights(r, 3, dtype)
    else:  # random box weights, canonical (dz, dy, dx) order matters
        w = np.random.default_rng(r).uniform(-0.2, 0.4, (2 * r + 1) ** 3).astype(dtype).astype(np.float64)
    return so2dr.StencilSpec(so2dr.BOX, r, 3, w), o.BOX, w


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("kind,r", [("star", 1), ("box", 1), ("rand", 1), ("star", 2), ("box", 2)])
@pytest.mark.parametrize("mode", ["incore", "so2dr"])
def test_3d_modes_match_oracle(engine, oracle, dtype, kind, r, mode):
    sz = 40
    spec, okind, w = _spec3(kind, r, dtype)
    g = oracle.init_grid(sz, r, 11, 3, dtype)
    got = g.copy()
    for k_on in (1, 2, 3, 4):
        cfg = so2dr.RunConfig(sz=sz, r=r, d=2, s_tb=4, k_on=k_on, n_strm=2, n=6)
        if 2 * r * cfg.s_tb > sz // cfg.d:
            cfg.s_tb = sz // cfg.d // (2 * r)
            cfg.k_on = min(k_on, cfg.s_tb)
        got = g.copy()
        rep = engine.run(mode, got, spec, cfg, so2dr.KernelPlan(cfg.k_on, 32, 1 << 30))
        want = oracle.run(g, okind, r, w, cfg.n)
        diff = np.argwhere(_bits(got) != _bits(want))
        assert diff.size == 0, f"{mode} {kind}{r} {dtype.__name__} k_on={cfg.k_on}: {len(diff)} diffs, first {diff[:3]}"
        exp = so2dr.expected_ledger(mode, cfg, so2dr.KernelPlan(cfg.k_on, 32), dim=3, dtype=dtype)
        for key in ("htod", "dtoh", "ondevice", "kernel_invocations", "rounds"):
            assert rep.ledger[key] == exp[key], key


def test_3d_degenerate_equals_2d_reference_per_plane(engine, oracle):
    """box3d1r with every dz != 0 weight zero: each z-plane evolves exactly as the
    2D reference (box2d1r) on that plane -- ties the 3D path to the reference."""
    r, sz, n = 1, 48, 5
    w2 = oracle.box_weights(1)
    w3 = np.zeros(27)
    w3[9:18] = w2
    g3 = oracle.init_grid(sz, r, 3, 3)
    got = g3.copy()
    cfg = so2dr.RunConfig(sz=sz, r=r, d=4, s_tb=4, k_on=4, n=n)
    engine.run("so2dr", got, so2dr.StencilSpec(so2dr.BOX, 1, 3, w3), cfg, so2dr.KernelPlan(4, 32))
    for z in range(r, r + sz):
        plane = oracle.run(g3[z].copy(), oracle.BOX, r, w2, n)
        assert (_bits(got[z]) == _bits(plane)).all(), z


def test_3d_larger_multi_tile(engine, oracle):
    sz, r = 150, 1
    spec, okind, w = _spec3("star", 1, np.float32)
    g = oracle.init_grid(sz, r, 5, 3)
    got = g.copy()
    cfg = so2dr.RunConfig(sz=sz, r=r, d=3, s_tb=8, k_on=4, n=8)
    engine.run("so2dr", got, spec, cfg, so2dr.KernelPlan(4, 32))
    want = oracle.run(g, okind, r, w, 8)
    assert (_bits(got) == _bits(want)).all()


@pytest.mark.parametrize("kind,r", [("box", 1), ("star", 2), ("gradient", 1), ("box", 2)])
def test_2d_f64_engine(engine, oracle, kind, r):
    """fp64 (config 5 family: star2d2r / j2d9pt) through the out-of-core engine."""
    if kind == "gradient":
        spec, okind, w = so2dr.StencilSpec.gradient(), oracle.GRADIENT, np.zeros(9)
    elif kind == "star":
        w = oracle.star_weights(r, 2, np.float64, 1.0 / 9.0)
        spec, okind = so2dr.StencilSpec(so2dr.BOX, r, 2, w), oracle.BOX
    else:
        w = oracle.box_weights(r, 2, np.float64)
        spec, okind = so2dr.StencilSpec(so2dr.BOX, r, 2, w), oracle.BOX
    g = oracle.init_grid(256, r, 9, 2, np.float64)
    got = g.copy()
    cfg = so2dr.RunConfig(sz=256, r=r, d=4, s_tb=8, k_on=4, n=20)
    engine.run("so2dr", got, spec, cfg, so2dr.KernelPlan(4, 32))
    want = oracle.run(g, okind, r, w, 20)
    assert (_bits(got) == _bits(want)).all()
    # the stated fp64 tolerance (<= 1e-12 relative) holds trivially: bit-exact
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)) <= 1e-12


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
@pytest.mark.parametrize("kind,r", [("star", 1), ("box", 1), ("rand", 1), ("star", 2), ("box", 2)])
def test_3d_inner_tiles_every_depth(engine, oracle, dtype, kind, r):
    """Grids wide enough for inner tiles (the check-free streaming body) next to
    edge tiles, every fused depth the 3D K1 supports, out-of-core chunks with
    region sharing (so2dr) and in-core."""
    sz = 136 if r == 1 else 104
    spec, okind, w = _spec3(kind, r, dtype)
    g = oracle.init_grid(sz, r, 21 + r, 3, dtype)
    kmax = so2dr.k1_max_steps(3, dtype, so2dr.BOX if kind != "star" else so2dr.STAR, r)
    for k_on in range(1, kmax + 1):
        n = 2 * k_on
        for mode, d in (("incore", 1), ("so2dr", 2)):
            cfg = so2dr.RunConfig(sz=sz, r=r, d=d, s_tb=n, k_on=k_on, n_strm=2, n=n)
            got = g.copy()
            engine.run(mode, got, spec, cfg, so2dr.KernelPlan(k_on, 32, 1 << 30))
            want = oracle.run(g, okind, r, w, n)
            diff = np.argwhere(_bits(got) != _bits(want))
            assert diff.size == 0, f"{mode} {kind}{r} {np.dtype(dtype).name} k_on={k_on}: {len(diff)} diffs, first {diff[:3]}"
