"""Copy-engine utilisation of one config-2 run: union of H2D / D2H / kernel busy time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402


def union(iv):
    iv = sorted(iv)
    tot, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    if cur:
        tot += cur[1] - cur[0]
    return tot


sz = 92160
eng = so2dr.Engine(0, 16 << 30)
host = eng.host_array((sz + 2, sz + 2), np.float32)
eng.init_grid(sz, 1, 42, out=host)
spec = so2dr.StencilSpec.box(1)
for d, ns in ((16, 3), (64, 3), (64, 4), (96, 3)):
    cfg = so2dr.RunConfig(sz=sz, r=1, d=d, s_tb=64, k_on=8, n_strm=ns, n=64)
    eng.set_profiling(False)
    eng.run("so2dr", host, spec, cfg, diag=False)
    eng.set_profiling(True)
    rep = eng.run("so2dr", host, spec, cfg)
    T = rep.timing["device_ms"]
    st = {}
    for r in rep.diagnostics:
        st.setdefault(r["stage"], []).append((r["t0_ms"], r["t0_ms"] + r["ms"]))
    h = sum(b for r in rep.diagnostics if r["stage"] == "htod" for b in [r["bytes"]])
    print(f"d={d} ns={ns} total={T:.1f} ms  GCell/s={sz*sz*64/T/1e6:.1f}  "
          + "  ".join(f"{k}: busy={union(v):.1f}ms sum={sum(b-a for a,b in v):.1f}ms" for k, v in st.items()),
          flush=True)
    first_k = min(a for a, b in st["kernel"])
    last_h = max(b for a, b in st["htod"])
    last_k = max(b for a, b in st["kernel"])
    print(f"   first kernel at {first_k:.1f} ms, last H2D end {last_h:.1f}, last kernel end {last_k:.1f}", flush=True)
