"""K1 results must not depend on how a launch is cut into work items: the
same so2dr runs with 1, 3 and 16 items per resident warp (SO2DR_K1_IPW: long
segments vs many short ones, i.e. different mixes of inner / edge items and of
pipeline fills) stay bit-exact with the oracle. Run in a subprocess: the knob
is read once per process."""
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
    for sz, d, s_tb, k, n in ((300, 3, 8, 4, 12), (517, 1, 6, 3, 9), (1000, 4, 16, 4, 20), (1536, 4, 16, 8, 16)):
        if sz % d:
            continue
        g = eng.init_grid(sz, 1, 7)
        want = o.run(o.init_grid(sz, 1, 7), o.BOX if kind == "box" else o.STAR, 1, w, n)
        cfg = so2dr.RunConfig(sz=sz, r=1, d=d, s_tb=s_tb, k_on=k, n_strm=3, n=n)
        eng.run("so2dr" if d > 1 else "incore", g, spec, cfg, so2dr.KernelPlan(k, 32))
        assert (g.view(np.uint32) == want.view(np.uint32)).all(), (kind, sz, d, k, n)
print("ok")
"""


@pytest.mark.parametrize("ipw", ["1", "3", "16", "default"])
def test_k1_segmentation_bit_exact(ipw):
    env = dict(os.environ)
    env.pop("SO2DR_K1_IPW", None)
    if ipw != "default":
        env["SO2DR_K1_IPW"] = ipw
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
