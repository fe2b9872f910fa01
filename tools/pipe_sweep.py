"""Sweep (d, N_strm, k_on) of the config-2 out-of-core run (pinned host grid, 16 GiB budget).
  DS=16,32,64 NS=3 KS=4,8 python tools/pipe_sweep.py"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402

sz = 92160
DS = [int(x) for x in os.environ.get("DS", "16,32,48,64").split(",")]
NS = [int(x) for x in os.environ.get("NS", "3,4").split(",")]
KS = [int(x) for x in os.environ.get("KS", "4,8").split(",")]
eng = so2dr.Engine(0, 16 << 30)
host = eng.host_array((sz + 2, sz + 2), np.float32)
eng.init_grid(sz, 1, 42, out=host)
spec = so2dr.StencilSpec.box(1)
for d, ns, k in itertools.product(DS, NS, KS):
    cfg = so2dr.RunConfig(sz=sz, r=1, d=d, s_tb=64, k_on=k, n_strm=ns, n=64)
    try:
        eng.run("so2dr", host, spec, cfg, diag=False)
        reps = [eng.run("so2dr", host, spec, cfg, diag=False).timing for _ in range(2)]
        best = min(reps, key=lambda t: t["device_ms"])
        print(json.dumps({"d": d, "n_strm": ns, "k_on": k, "ms": round(best["device_ms"], 1),
                          "GCell_s": round(sz * sz * 64 / best["device_ms"] / 1e6, 1),
                          "kernel_ms": round(best["kernel_ms"], 1),
                          "kernel_GCell_s": round(sz * sz * 64 / best["kernel_ms"] / 1e6, 1)}), flush=True)
    except so2dr.Error as e:
        print(json.dumps({"d": d, "n_strm": ns, "k_on": k, "error": str(e)[:100]}), flush=True)
