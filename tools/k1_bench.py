"""K1 microbenchmark: in-core runs on an HBM-resident grid; prints per-launch
kernel GCell/s, algorithmic GB/s and the FMA-pipe rate for (stencil, k_on) shapes.
  SZ=32768 STENCILS=box2d1r,star2d1r KS=1,2,4,8 python tools/k1_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402

sz = int(os.environ.get("SZ", "32768"))
names = os.environ.get("STENCILS", "box2d1r,star2d1r,gradient2d,box2d2r").split(",")
ks = [int(x) for x in os.environ.get("KS", "1,2,4,6,8").split(",")]
eng = so2dr.Engine(0)
SPECS = {"box3d1r": (so2dr.StencilSpec.box(1, dim=3), 1, 27), "star3d1r": (so2dr.StencilSpec.star(1, dim=3), 1, 7),
         "box2d1r": (so2dr.StencilSpec.box(1), 1, 9), "star2d1r": (so2dr.StencilSpec.star(1), 1, 5),
         "gradient2d": (so2dr.StencilSpec.gradient(), 1, 9), "box2d2r": (so2dr.StencilSpec.box(2), 2, 25),
         "star2d2r": (so2dr.StencilSpec.star(2), 2, 9)}
FMA_PEAK = 148 * 128 * 1.965e9  # fp32 FMA/s at boost (4 SMSP x 32 lanes per SM)
for name in names:
    spec, r, taps = SPECS[name]
    dim = 3 if "3d" in name else 2
    szd = int(os.environ.get("SZ3", "768")) if dim == 3 else sz
    g = torch.empty((szd + 2 * r,) * dim, dtype=torch.float32, device="cuda")
    eng.init_grid(szd, r, 42, dim, out=g)
    for k in ks:
        n = 4 * k
        cfg = so2dr.RunConfig(sz=szd, r=r, d=1, s_tb=n, k_on=k, n_strm=1, n=n)
        try:
            eng.run("incore", g, spec, cfg, so2dr.KernelPlan(k, 32, 1 << 30), diag=False)  # warm
            rep = eng.run("incore", g, spec, cfg, so2dr.KernelPlan(k, 32, 1 << 30), diag=False)
        except so2dr.Error as e:
            print(json.dumps({"stencil": name, "k_on": k, "error": str(e)[:120]}), flush=True)
            continue
        t = rep.timing
        upd = szd ** dim * k
        ms = t["kernel_ms"] / t["kernel_launches"]
        row = {"stencil": name, "k_on": k, "sz": szd, "ms_per_launch": round(ms, 4), "GCell_s": round(upd / ms / 1e6, 1),
               "alg_GBps": round(t["kernel_alg_bytes"] / t["kernel_launches"] / ms / 1e6, 1),
               "fma_frac": round(upd * taps / (ms / 1e3) / FMA_PEAK, 3)}
        print(json.dumps(row), flush=True)
    del g
