"""Per-stage timeline of one out-of-core so2dr run (profiling mode): H2D / share /
kernel / D2H start and duration per chunk, and the effective transfer GB/s.
    python tools/pipe_profile.py [sz] [d] [k_on] [n_strm]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402

sz = int(sys.argv[1]) if len(sys.argv) > 1 else 92160
d = int(sys.argv[2]) if len(sys.argv) > 2 else 16
k_on = int(sys.argv[3]) if len(sys.argv) > 3 else 8
ns = int(sys.argv[4]) if len(sys.argv) > 4 else 3
eng = so2dr.Engine(0, 16 << 30)
if os.environ.get("HOST_ALLOC") == "torch":  # torch's pinned allocator instead of so2dr_host_alloc
    import torch

    host = torch.empty((sz + 2, sz + 2), dtype=torch.float32, pin_memory=True)
    eng.init_grid(sz, 1, 42, out=host)
else:
    host = eng.host_array((sz + 2, sz + 2), np.float32)
if not os.environ.get("HOST_ALLOC"):
    eng.init_grid(sz, 1, 42, out=host)
cfg = so2dr.RunConfig(sz=sz, r=1, d=d, s_tb=64, k_on=k_on, n_strm=ns, n=64)
spec = so2dr.StencilSpec.box(1)
eng.run("so2dr", host, spec, cfg, diag=False)  # warm
eng.set_profiling(True)
rep = eng.run("so2dr", host, spec, cfg)
t = rep.timing
print(json.dumps({"device_ms": t["device_ms"], "kernel_ms": t["kernel_ms"], "launches": t["kernel_launches"],
                  "GCell_s": sz * sz * 64 / t["device_ms"] / 1e6}))
for row in rep.diagnostics:
    gbs = row["bytes"] / row["ms"] / 1e6 if row["ms"] > 0 else 0
    print(f"r{row['round']} c{row['chunk']:2d} {row['stage']:11s} t0={row['t0_ms']:8.2f} ms={row['ms']:7.2f} "
          f"GB/s={gbs:7.1f}")
