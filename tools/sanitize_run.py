"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every K1 code path once -- 2D fp32/fp64 box/star at S = 1, 2 (CTA bulk-copy ring),
4, 8 (per-warp lane ring), the edge path, 3D star/box (interior and edge tiles) -- plus
an out-of-core so2dr run through the scheduler, each result checked bit-for-bit
against the CPU oracle (the oracle is only the checker here).
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402
import pyoracle as o  # noqa: E402


def bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def k1_2d(eng, kind, r, steps, dtype, sz=300):
    w = (o.box_weights if kind == "box" else o.star_weights)(r, 2, dtype)
    spec = so2dr.StencilSpec.box(r, w)
    g = o.init_grid(sz, r, 11 + steps, 2, dtype)
    p = g.shape[0]
    b0 = np.ascontiguousarray(g)
    b1 = b0.copy()
    region = (r, p - r, 0, p)
    eng.fused_kernel(spec, b0, b1, 0, 0, steps, 32, region, (r, p - r, r, p - r), region)
    want = o.run(g, o.BOX, r, w, steps)
    assert (bits(b1[r:p - r]) == bits(want[r:p - r])).all(), (kind, r, steps, dtype)


def incore_3d(eng, kind, steps, sz=96):
    w = o.box_weights(1, 3) if kind == "box" else o.star_weights(1, 3)
    spec = so2dr.StencilSpec.box(1, w, dim=3)
    grid = eng.init_grid(sz, 1, 5, 3)
    want = o.run(o.init_grid(sz, 1, 5, 3), o.BOX, 1, w, steps)
    cfg = so2dr.RunConfig(sz=sz, r=1, d=1, s_tb=steps, k_on=steps, n_strm=1, n=steps)
    eng.run("incore", grid, spec, cfg, so2dr.KernelPlan(steps, 32, 1 << 30), diag=False)
    assert (bits(grid) == bits(want)).all(), (kind, steps)


def so2dr_2d(eng):
    w = o.box_weights(1, 2)
    spec = so2dr.StencilSpec.box(1, w)
    cfg = so2dr.RunConfig(sz=512, r=1, d=4, s_tb=8, k_on=4, n_strm=3, n=16)
    grid = eng.init_grid(512, 1, 42)
    want = o.run(o.init_grid(512, 1, 42), o.BOX, 1, w, 16)
    eng.run("so2dr", grid, spec, cfg, so2dr.KernelPlan(4, 32))
    assert (bits(grid) == bits(want)).all()


def main():
    eng = so2dr.Engine(0)
    n = 0
    for dtype in (np.float32, np.float64):
        for kind in ("box", "star"):
            for steps in (1, 2, 4, 8):
                k1_2d(eng, kind, 1, steps, dtype)
                n += 1
    k1_2d(eng, "box", 2, 4, np.float32)
    n += 1
    for kind in ("star", "box"):
        for steps in (1, 2, 4):
            incore_3d(eng, kind, steps)
            n += 1
    so2dr_2d(eng)
    n += 1
    eng.close()
    print(f"sanitize workload ok: {n} runs bit-exact")


if __name__ == "__main__":
    main()
