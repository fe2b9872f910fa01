"""Sweep (d, N_strm, k_on) of the config-2 out-of-core run (pinned host grid, 16 GiB budget)."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402

sz = 92160
eng = so2dr.Engine(0, 16 << 30)
host = eng.host_array((sz + 2, sz + 2), np.float32)
eng.init_grid(sz, 1, 42, out=host)
spec = so2dr.StencilSpec.box(1)
for d, ns, k in itertools.product((16, 32, 48, 64), (3, 4, 6), (4, 8)):
    cfg = so2dr.RunConfig(sz=sz, r=1, d=d, s_tb=64, k_on=k, n_strm=ns, n=64)
    try:
        eng.run("so2dr", host, spec, cfg, diag=False)
        best = min(eng.run("so2dr", host, spec, cfg, diag=False).timing["device_ms"] for _ in range(2))
        print(json.dumps({"d": d, "n_strm": ns, "k_on": k, "ms": best, "GCell_s": sz * sz * 64 / best / 1e6}), flush=True)
    except so2dr.Error as e:
        print(json.dumps({"d": d, "n_strm": ns, "k_on": k, "error": str(e)[:100]}), flush=True)
