"""Measure the BASELINE.json configs that are not the bench headline, on one B200,
end to end through the C ABI (pinned host grid, all H2D/D2H inside the timing).

  cfg1  star2d1r fp32 4096^2, d=4, n=8, S_TB=4, k_on=4 (the CPU-reference preset)
  cfg3  star3d1r fp32 sz=2048 (34.5 GB, ~2x a 16 GiB budget), d=16, S_TB=8, n=64, k_on 1/2/4/8
  cfg4  box3d1r fp32 per-GPU slab of the 8-GPU config: sz=2048, d=32, S_TB=16, k_on=4, n=32
  cfg5  star2d2r (j2d9pt-shaped) fp64 sz=65536 (34.4 GB), d=16, S_TB=64, k_on=4, n=64
  cfg5h the same stencil on the largest fp64 grid this host's RAM holds pinned:
        sz=131072 (137.4 GB; 196 GB host), d=64, S_TB=64, k_on=4, n=64
The PCIe roof is measured in the same process (bench.pcie_probe: duplex
per-direction rate, 2 GiB each way) and SM clocks are sampled during every run
(bench.ClockSampler). Prints one JSON line per run: GCell/s, device ms, the
measured R_pcie bound and the fraction, the B200 planner's prediction, clocks."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (pcie_probe, ClockSampler)
import paper_2309_08864_b200 as so2dr  # noqa: E402

eng = so2dr.Engine(0, 16 << 30)
which = sys.argv[1:] or ["cfg1", "cfg3", "cfg5", "cfg4", "cfg5h"]
PC = bench.pcie_probe(torch, torch.device("cuda", 0))
BW_DIR = PC["duplex_GBps_per_dir"]  # measured in this process
print(json.dumps({"pcie_measured": PC}), flush=True)
try:
    PROFILE = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                "b200.json")).read()
except OSError:
    PROFILE = None


def run(name, dim, dtype, spec, sz, d, s_tb, k_ons, n, reps=2):
    r = spec.radius
    p = sz + 2 * r
    t0 = time.perf_counter()
    host = eng.host_array((p,) * dim, dtype)
    eng.init_grid(sz, r, 42, dim, dtype, out=host)
    t_init = time.perf_counter() - t0
    b = np.dtype(dtype).itemsize
    for k in k_ons:
        cfg = so2dr.RunConfig(sz=sz, r=r, d=d, s_tb=s_tb, k_on=k, n_strm=3, n=n)
        eng.run("so2dr", host, spec, cfg, so2dr.KernelPlan(k, 32, 1 << 40), diag=False)
        best = None
        with bench.ClockSampler(0, 200) as clk:
            for _ in range(reps):
                rep = eng.run("so2dr", host, spec, cfg, so2dr.KernelPlan(k, 32, 1 << 40), diag=False)
                if best is None or rep.timing["device_ms"] < best.timing["device_ms"]:
                    best = rep
        t = best.timing
        upd = float(sz) ** dim * n
        g = upd / t["device_ms"] / 1e6
        r_pcie = BW_DIR * 1e9 * s_tb / b / 1e9
        try:
            pred = so2dr.predict_b200(sz, n, d, s_tb, k, r, spec.kind if spec.kind != so2dr.GRADIENT else so2dr.BOX,
                                      dim, dtype, budget_bytes=16 << 30, profile=PROFILE)
            pred = {"t_total_s": pred["t_total_s"], "gcell_per_s": pred["gcell_per_s"]}
        except so2dr.Error as e:
            pred = {"error": str(e)[:100]}
        print(json.dumps({"config": name, "dim": dim, "dtype": np.dtype(dtype).name, "sz": sz, "d": d,
                          "s_tb": s_tb, "k_on": k, "n": n, "grid_GB": p ** dim * b / 1e9,
                          "device_ms": t["device_ms"], "GCell_s": g, "kernel_ms": t["kernel_ms"],
                          "kernel_GCell_s": upd / t["kernel_ms"] / 1e6 if t["kernel_ms"] else None,
                          "R_pcie_GCell_s": r_pcie, "frac_R_pcie": g / r_pcie, "BW_dir_GBps": BW_DIR,
                          "kernel_launches": t["kernel_launches"], "planner": pred, "clocks": clk.summary(),
                          "init_s": t_init}), flush=True)
    del host


if "cfg1" in which:
    import pyoracle as o

    run("cfg1 star2d1r", 2, np.float32, so2dr.StencilSpec.box(1, o.star_weights(1)), 4096, 4, 4, [4], 8, reps=5)
if "cfg3" in which:  # the temporal-block depth sweep 1..8 (3D K1 fuses <= 4 steps per launch)
    run("cfg3 star3d1r", 3, np.float32, so2dr.StencilSpec.star(1, dim=3), 2048, 16, 8, [1, 2, 3, 4, 5, 6, 7, 8], 64,
        reps=1)
if "cfg5" in which:
    run("cfg5 star2d2r fp64", 2, np.float64, so2dr.StencilSpec.star(2, w=1.0 / 9.0, dtype=np.float64), 65536, 16,
        64, [4], 64, reps=2)
if "cfg5h" in which:
    run("cfg5h star2d2r fp64 host-RAM-sized", 2, np.float64, so2dr.StencilSpec.star(2, w=1.0 / 9.0, dtype=np.float64),
        131072, 64, 64, [4], 64, reps=1)
if "cfg4" in which:
    run("cfg4 box3d1r (per-GPU slab)", 3, np.float32, so2dr.StencilSpec.box(1, dim=3), 2048, 32, 16, [4], 32,
        reps=1)
