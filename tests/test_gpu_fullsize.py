"""Parity at BASELINE.json's FULL sizes (out-of-core, ~2x the 16 GiB device budget).

The CPU oracle cannot evolve a 34 GB grid, so these tests use the light-cone
property of the stencil (pyoracle.window_expected, pinned against the
whole-grid oracle in test_host.py): the state of any window after n steps is
a function of the window's r*n neighbourhood only, so the oracle evolves a
small cut-out and the GPU result must match it BIT FOR BIT. Windows are taken
at the grid corners and edges (ring pass-through), across every chunk fence
(region sharing + recomputed trapezoid halo) and at seeded random points.
Plus size-independent invariants: ring cells untouched, ledger equals the
closed-form expected ledger, bytes moved over PCIe = one grid each way.
"""
import numpy as np
import pytest

import paper_2309_08864_b200 as so2dr

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

BUDGET = 16 << 30


def _windows(p, fences, h, w, rng, n_random, dim, max_windows):
    """(lo, hi) boxes of edge w: the two far corners, windows straddling chunk
    fences (the fence itself and fence +- h, the edges of the shared region),
    then seeded random ones; at most max_windows, spread over the categories."""
    def at(y):
        y = min(max(0, y), p - w)
        rest = tuple(int(rng.integers(0, p - w)) for _ in range(dim - 1))
        lo = (y,) + rest
        return lo, tuple(a + w for a in lo)

    corners = [((0,) * dim, (w,) * dim), ((p - w,) * dim, (p,) * dim)]
    inner = list(fences[1:-1])
    fence_boxes = []
    for j, f in enumerate(inner):
        fence_boxes.append(at(f + (-h, 0, h)[j % 3] - w // 2))
    rand = [at(int(rng.integers(0, p - w))) for _ in range(n_random)]
    budget = max(0, max_windows - len(corners) - len(rand))
    if len(fence_boxes) > budget:
        idx = np.linspace(0, len(fence_boxes) - 1, budget).round().astype(int) if budget else []
        fence_boxes = [fence_boxes[i] for i in idx]
    return corners + fence_boxes + rand


def _check_fullsize(engine_budget, oracle, dim, dtype, kind, r, sz, d, s_tb, k_on, n, w, n_random, max_windows,
                    scratch=1 << 40, every_fence=False):
    o = oracle
    eng = engine_budget
    if kind == "box":
        spec = so2dr.StencilSpec.box(r, dim=dim) if dim == 3 else so2dr.StencilSpec.box(r)
        wts, kc = o.box_weights(r, dim), o.BOX
    else:
        spec = so2dr.StencilSpec.star(r, dim=dim, dtype=dtype)
        wts, kc = o.star_weights(r, dim, dtype), o.STAR
    p = sz + 2 * r
    host = eng.host_array((p,) * dim, dtype)
    eng.init_grid(sz, r, 42, dim, dtype, out=host)
    ring_before = [np.array(host[(slice(0, r),)]), np.array(host[(slice(p - r, p),)])]
    cfg = so2dr.RunConfig(sz=sz, r=r, d=d, s_tb=s_tb, k_on=k_on, n_strm=3, n=n)
    rep = eng.run("so2dr", host, spec, cfg, so2dr.KernelPlan(k_on, 32, scratch), diag=False)
    # size-independent invariants
    exp = so2dr.expected_ledger("so2dr", cfg, so2dr.KernelPlan(k_on, 32, scratch), dim=dim, dtype=dtype)
    for k in ("htod", "dtoh", "ondevice", "kernel_invocations", "rounds"):
        assert rep.ledger[k] == exp[k], k
    assert np.array_equal(host[(slice(0, r),)], ring_before[0])
    assert np.array_equal(host[(slice(p - r, p),)], ring_before[1])
    assert rep.timing["device_bytes"] <= BUDGET
    grid_bytes = p ** dim * np.dtype(dtype).itemsize
    assert rep.timing["device_bytes"] < grid_bytes / 1.9  # genuinely out of core
    # light-cone windows, bit-exact
    fences, _ = so2dr.plan_chunks(cfg)
    rng = np.random.default_rng(7)
    boxes = _windows(p, list(fences), r * s_tb, w, rng, n_random, dim, max_windows)
    if every_fence:  # every inner fence at -h, 0 and +h (the shared region's edges)
        h = r * s_tb
        for f in list(fences)[1:-1]:
            for off in (-h, 0, h):
                y = min(max(0, f + off - w // 2), p - w)
                for x in (0, int(rng.integers(0, p - w)), p - w):
                    lo = (y, x) + tuple(int(rng.integers(0, p - w)) for _ in range(dim - 2))
                    boxes.append((lo, tuple(a + w for a in lo)))
    for lo, hi in boxes:
        want = o.window_expected(lambda a, b: o.init_block(a, b, 42, dtype), sz, r, n, lo, hi, kc, wts, dim)
        got = host[tuple(slice(a, b) for a, b in zip(lo, hi))]
        if not np.array_equal(np.ascontiguousarray(got).view(np.uint8), want.view(np.uint8)):
            bad = np.argwhere(got != want)[0]
            raise AssertionError(f"window {lo}-{hi}: first diff at {tuple(bad)}: got {got[tuple(bad)]!r} "
                                 f"want {want[tuple(bad)]!r}")
    del host, got
    import gc

    gc.collect()
    return rep


@pytest.fixture(scope="module")
def eng16():
    e = so2dr.Engine(0, BUDGET)
    yield e
    e.close()


def test_config2_box2d1r_fullsize_out_of_core(eng16, oracle):
    """BASELINE configs[1] = the bench workload: box2d1r fp32, sz=92160 (33.98 GB,
    1.98x the 16 GiB budget), 64 steps, d=16, S_TB=64, k_on=8."""
    rep = _check_fullsize(eng16, oracle, 2, np.float32, "box", 1, 92160, 16, 64, 8, 64, 48, 6, 64)
    assert rep.timing["h2d_bytes"] == (92162 ** 2) * 4


def test_config3_star3d1r_fullsize_out_of_core(eng16, oracle):
    """BASELINE configs[2]: star3d1r fp32, sz=2048 (34.5 GB), d=16, S_TB=8 (8 rounds), k_on=8, n=64."""
    _check_fullsize(eng16, oracle, 3, np.float32, "star", 1, 2048, 16, 8, 8, 64, 6, 2, 8)


def test_config4_box3d1r_fullsize_slab(eng16, oracle):
    """BASELINE configs[3] per-GPU slab shape: box3d1r fp32, sz=2048, d=32 (d=16 needs 17.8 GB of ping-pong buffers), S_TB=16, k_on=4, n=32."""
    _check_fullsize(eng16, oracle, 3, np.float32, "box", 1, 2048, 32, 16, 4, 32, 6, 2, 8)


def test_config5_star2d2r_f64_fullsize(eng16, oracle):
    """BASELINE configs[4] per-GPU shape: star2d2r (j2d9pt-shaped) fp64, sz=65536 (34.4 GB), S_TB=64, k_on=4."""
    _check_fullsize(eng16, oracle, 2, np.float64, "star", 2, 65536, 16, 64, 4, 64, 32, 6, 64)


def test_bench_workload_exact_geometry(eng16, oracle):
    """The EXACT workload bench.py times (its constants are imported, so the test
    follows the bench): box2d1r fp32, sz=92160 (33.98 GB host grid, 1.98x the
    16 GiB budget), n=64, d=64, S_TB=64, k_on=4, N_strm=3, KernelPlan(k_on, 32,
    64 MiB) -- i.e. ~1500-row K1 launches. Windows: both grid corners, every one
    of the 63 inner fences at fence-h, fence and fence+h (h = r*S_TB, the shared
    region's edges) at the left edge (ring columns), a random column and the right
    edge, plus random windows; all bit-exact against the oracle's light cone."""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert (bench.SZ1, bench.D_PER_RANK, bench.S_TB, bench.K_ON, bench.NSTEPS, bench.NSTRM, bench.R) == \
        (92160, 64, 64, 4, 64, 3, 1)
    assert bench.BUDGET == BUDGET
    rep = _check_fullsize(eng16, oracle, 2, np.float32, "box", bench.R, bench.SZ1, bench.D_PER_RANK, bench.S_TB,
                          bench.K_ON, bench.NSTEPS, 40, 8, 10, scratch=64 << 20, every_fence=True)
    assert rep.timing["h2d_bytes"] == (92162 ** 2) * 4
    assert rep.timing["kernel_launches"] == bench.D_PER_RANK * bench.S_TB // bench.K_ON
