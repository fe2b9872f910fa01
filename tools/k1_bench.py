"""K1 microbenchmark: in-core runs on an HBM-resident grid; prints per-launch
kernel GCell/s and algorithmic GB/s for a few (stencil, k_on) shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402

sz = int(os.environ.get("SZ", "16384"))
eng = so2dr.Engine(0)
out = []
for name, spec, r in [("box2d1r", so2dr.StencilSpec.box(1), 1), ("star2d1r", so2dr.StencilSpec.star(1), 1),
                      ("gradient2d", so2dr.StencilSpec.gradient(), 1), ("box2d2r", so2dr.StencilSpec.box(2), 2)]:
    g = torch.empty((sz + 2 * r, sz + 2 * r), dtype=torch.float32, device="cuda")
    eng.init_grid(sz, r, 42, out=g)
    for k in (1, 2, 4, 6, 8):
        if r == 2 and k > 6:
            continue
        n = 4 * k
        cfg = so2dr.RunConfig(sz=sz, r=r, d=1, s_tb=n, k_on=k, n_strm=1, n=n)
        eng.run("incore", g, spec, cfg, so2dr.KernelPlan(k, 32, 1 << 30), diag=False)  # warm
        rep = eng.run("incore", g, spec, cfg, so2dr.KernelPlan(k, 32, 1 << 30), diag=False)
        t = rep.timing
        upd = sz * sz * k
        ms = t["kernel_ms"] / t["kernel_launches"]
        row = {"stencil": name, "k_on": k, "ms_per_launch": ms, "GCell_s": upd / ms / 1e6,
               "alg_GBps": t["kernel_alg_bytes"] / t["kernel_launches"] / ms / 1e6}
        out.append(row)
        print(json.dumps(row), flush=True)
    del g
