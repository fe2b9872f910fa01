"""Every fp32 K1 variant must stay bit-exact with the oracle: the default
scalar-FFMA pipeline, the packed FFMA2 kernel (SO2DR_K1_IMPL=pk), the hybrid
FFMA2/FFMA kernel (SO2DR_K1_IMPL=hyb) and the
paired-strip kernel (SO2DR_K1_IMPL=p2, S = 3..4). Run in a subprocess: the
variant is chosen once per process."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/oracle")
import numpy as np
import paper_2309_08864_b200 as so2dr
import pyoracle as o
eng = so2dr.Engine(0)
for kind, w, spec in (("box", o.box_weights(1), so2dr.StencilSpec.box(1)),
                      ("star", o.star_weights(1), so2dr.StencilSpec.star(1))):
    for sz, d, s_tb, k, n in ((300, 3, 8, 4, 12), (517, 1, 6, 3, 9), (1000, 4, 16, 4, 20)):
        if sz % d:
            continue
        g = eng.init_grid(sz, 1, 7)
        want = o.run(o.init_grid(sz, 1, 7), o.BOX if kind == "box" else o.STAR, 1, w, n)
        cfg = so2dr.RunConfig(sz=sz, r=1, d=d, s_tb=s_tb, k_on=k, n_strm=3, n=n)
        eng.run("so2dr" if d > 1 else "incore", g, spec, cfg, so2dr.KernelPlan(k, 32))
        assert (g.view(np.uint32) == want.view(np.uint32)).all(), (kind, sz, d, k, n)
print("ok")
"""


@pytest.mark.parametrize("impl", ["p2", "pk", "hyb", "default"])
def test_k1_variant_bit_exact(impl):
    env = dict(os.environ)
    env.pop("SO2DR_K1_IMPL", None)
    if impl != "default":
        env["SO2DR_K1_IMPL"] = impl
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
