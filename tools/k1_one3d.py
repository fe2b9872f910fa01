"""One in-core 3D K1 launch sequence (for ncu): python tools/k1_one3d.py <k_on> [sz] [box|star]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402

k = int(sys.argv[1])
sz = int(sys.argv[2]) if len(sys.argv) > 2 else 768
name = sys.argv[3] if len(sys.argv) > 3 else "star"
spec = so2dr.StencilSpec.star(1, dim=3) if name == "star" else so2dr.StencilSpec.box(1, dim=3)
eng = so2dr.Engine(0)
g = torch.empty((sz + 2,) * 3, dtype=torch.float32, device="cuda")
eng.init_grid(sz, 1, 42, 3, out=g)
cfg = so2dr.RunConfig(sz=sz, r=1, d=1, s_tb=2 * k, k_on=k, n_strm=1, n=2 * k)
rep = eng.run("incore", g, spec, cfg, so2dr.KernelPlan(k, 32, 1 << 30), diag=False)
print(rep.timing["kernel_ms"] / rep.timing["kernel_launches"], "ms/launch")
