"""K1 2D streaming path (k1_2d_stream.cuh) against the CPU oracle, bit-exact.

The small grids of test_gpu_kernels.py put almost every work item next to the
ring (EDGE variant). These grids are wide and tall enough that most items are
inner items (no pass-through cell: branch-free fill/drain, packed FFMA2 row
pairs), and the storage windows reproduce the engine's chunk geometry: a
buffer holding rows [base, base+rows) of the grid, a region shrunk by r*steps
from the storage edges (the trapezoid of a chunk inside the grid) or touching
the grid's ring rows (first / last chunk). The oracle is the checker only."""
import numpy as np
import pytest

import paper_2309_08864_b200 as so2dr

pytestmark = pytest.mark.gpu


def _weights(kind, r, dtype, rng):
    import pyoracle as o

    if kind == "box":
        return o.box_weights(r, 2, dtype)
    if kind == "star":
        return o.star_weights(r, 2, dtype)
    w = rng.uniform(-0.3, 0.5, (2 * r + 1) ** 2).astype(dtype).astype(np.float64)
    if kind == "starrand":
        w = w.reshape(2 * r + 1, 2 * r + 1)
        m = np.zeros_like(w)
        m[r, :] = 1
        m[:, r] = 1
        w = (w * m).ravel()
    return w


def _bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _run(engine, oracle, kind, r, steps, dtype, sz, base, rows, region, seed):
    import pyoracle as o

    rng = np.random.default_rng(seed)
    w = _weights(kind, r, dtype, rng)
    spec = so2dr.StencilSpec.box(r, w)
    g = oracle.init_grid(sz, r, seed, 2, dtype)
    p = g.shape[0]
    b0 = np.ascontiguousarray(g[base:base + rows])
    b1 = b0.copy()
    interior = (r, p - r, r, p - r)
    engine.fused_kernel(spec, b0, b1, base, 0, steps, 32, region, interior, region)
    want = oracle.run(g, o.BOX, r, w, steps)
    y0, y1, x0, x1 = region
    got = b1[y0 - base:y1 - base, x0:x1]
    exp = want[y0:y1, x0:x1]
    bad = np.argwhere(_bits(got) != _bits(exp))
    assert bad.size == 0, (f"{kind} r={r} s={steps} {np.dtype(dtype).name} sz={sz} base={base} rows={rows} "
                           f"region={region}: {len(bad)} diffs, first {bad[:3] + [y0, x0]}")
    mask = np.ones_like(b1, dtype=bool)
    mask[y0 - base:y1 - base, x0:x1] = False
    assert (_bits(b1)[mask] == _bits(b0)[mask]).all(), "cells outside the region were written"


MAXS = {np.float32: {1: 8, 2: 4, 3: 4, 4: 4}, np.float64: {1: 8, 2: 4, 3: 2, 4: 1}}


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
@pytest.mark.parametrize("kind", ["box", "star", "boxrand", "starrand"])
@pytest.mark.parametrize("r", [1, 2, 3, 4])
def test_stream_whole_grid_every_depth(engine, oracle, kind, r, dtype):
    sz = 600
    p = sz + 2 * r
    for steps in range(1, MAXS[dtype][r] + 1):
        _run(engine, oracle, kind, r, steps, dtype, sz, 0, p, (r, p - r, 0, p), seed=7 * steps + r)


@pytest.mark.parametrize("kind,r,dtype", [("box", 1, np.float32), ("star", 1, np.float32), ("boxrand", 2, np.float32),
                                          ("box", 3, np.float32), ("starrand", 4, np.float32),
                                          ("box", 1, np.float64), ("boxrand", 2, np.float64)])
def test_stream_chunk_windows(engine, oracle, kind, r, dtype):
    """Chunk-shaped storage windows: inner chunks (region = storage shrunk by
    r*steps), first / last chunks (storage holds the ring rows) and random
    column sub-ranges."""
    rng = np.random.default_rng(1000 + r)
    sz = 700
    p = sz + 2 * r
    for _ in range(8):
        steps = int(rng.integers(1, MAXS[dtype][r] + 1))
        h = r * steps
        rows = int(rng.integers(2 * h + 40, 400))
        where = int(rng.integers(0, 3))
        if where == 0:  # first chunk: storage starts at the top ring row
            base = 0
            y0, y1 = 0, rows - h
        elif where == 1:  # last chunk
            base = p - rows
            y0, y1 = base + h, p
        else:
            base = int(rng.integers(1, p - rows))
            y0, y1 = base + h, base + rows - h
        x0 = int(rng.integers(0, p // 3)) if rng.random() < 0.5 else 0
        x1 = int(rng.integers(2 * p // 3, p + 1)) if rng.random() < 0.5 else p
        _run(engine, oracle, kind, r, steps, dtype, sz, base, rows, (y0, y1, x0, x1), seed=int(rng.integers(1 << 30)))


def test_stream_bench_like_geometry(engine, oracle):
    """A scaled-down copy of the bench chunk: ~1500-row storage windows with the
    bench's k_on=4 on a wide grid, both inner and edge chunks."""
    sz = 2046
    p = sz + 2
    for base, rows, region in [(0, 300, (0, 296, 0, p)), (500, 400, (504, 896, 0, p)), (p - 300, 300, (p - 296, p, 0, p))]:
        _run(engine, oracle, "box", 1, 4, np.float32, sz, base, rows, region, seed=base + 1)
