"""B200 run planner (include/so2dr/b200.hpp): host-only checks of
the model that replaces the reference's predict_bottleneck / feasible_configs
terms (proj/src/planner.cpp:14-89), the committed measured profile
(profiles/b200.json) and its agreement with the measured bench run."""
import json
import os

import numpy as np
import pytest

import paper_2309_08864_b200 as so2dr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILE = open(os.path.join(ROOT, "profiles", "b200.json")).read()
BENCH = dict(sz=92160, n=64, budget_bytes=16 << 30, profile=PROFILE)


def test_plan_best_is_the_fastest_feasible_candidate():
    best, cands = so2dr.plan_b200(all_candidates=True, **BENCH)
    feas = [c for c in cands if c["feasible"]]
    assert best["feasible"] and feas
    assert best["t_total_s"] <= min(c["t_total_s"] for c in feas) + 1e-12
    assert 92160 % best["d"] == 0 and 64 % best["s_tb"] == 0 and 1 <= best["k_on"] <= best["s_tb"]


def test_kernel_term_is_k_on_aware():
    """The reference prices S_TB one-step sweeps regardless of k_on; here fusing
    k_on steps per launch divides the HBM traffic (2b/k_on per update)."""
    t = {k: so2dr.predict_b200(d=64, s_tb=64, k_on=k, **BENCH)["t_kernel_s"] for k in (1, 2, 4)}
    assert t[1] > 1.5 * t[2] > 1.5 * 1.2 * t[4]


def test_memory_term_is_the_engine_footprint():
    """2 buffers per stream + share slots: the planner's footprint is the
    engine's (so2dr_device_bytes), and a budget below it is infeasible."""
    cfg = so2dr.RunConfig(sz=92160, r=1, d=64, s_tb=64, k_on=4, n_strm=3, n=64)
    need = so2dr.device_bytes(cfg)
    e = so2dr.predict_b200(d=64, s_tb=64, k_on=4, **BENCH)
    assert e["device_bytes"] == need
    small = dict(BENCH, budget_bytes=need - 1)
    assert not so2dr.predict_b200(d=64, s_tb=64, k_on=4, **small)["feasible"]
    assert so2dr.predict_b200(d=64, s_tb=64, k_on=4, **dict(BENCH, budget_bytes=need))["feasible"]
    # chunk smaller than the shared rows: infeasible (2 r S_TB <= sz/d)
    assert not so2dr.predict_b200(d=1024, s_tb=64, k_on=4, **BENCH)["feasible"]


def test_prediction_matches_the_measured_bench_run():
    """The bench configuration (d=64, S_TB=64, k_on=4) measured 733 ms per run
    end to end (profiles/r02_head/bench_line.json); the model is within 5%."""
    line = json.load(open(os.path.join(ROOT, "profiles", "r02_head", "bench_line.json")))
    measured = line["ms_per_step"] / 1e3
    pred = so2dr.predict_b200(d=64, s_tb=64, k_on=4, **BENCH)["t_total_s"]
    assert abs(pred - measured) / measured < 0.05, (pred, measured)


def test_profile_json_is_read_by_both_planners():
    """profiles/b200.json keeps the reference's flat keys, so the mirror's
    load_hardware_profile (proj/src/planner.cpp:115-143) reads it as well."""
    j = json.loads(PROFILE)
    for k in ("name", "c_dmem_bytes", "bw_dmem_bytes_per_s", "bw_intc_bytes_per_s", "b_elem"):
        assert k in j
    assert so2dr.plan_b200(**BENCH)["feasible"]
    assert so2dr.plan_b200(sz=92160, n=64, budget_bytes=16 << 30)["feasible"]  # built-in copy
    with pytest.raises(so2dr.Error):
        so2dr.plan_b200(sz=92160, n=64, profile='{"bw_dmem_bytes_per_s": -1}')


@pytest.mark.parametrize("dim,kind,r,dtype,sz,n", [(2, so2dr.STAR, 1, np.float32, 4096, 8),
                                                   (3, so2dr.STAR, 1, np.float32, 3264, 8),
                                                   (3, so2dr.BOX, 1, np.float32, 3264, 8),
                                                   (2, so2dr.STAR, 2, np.float64, 65536, 16)])
def test_plan_for_the_baseline_configs(dim, kind, r, dtype, sz, n):
    best = so2dr.plan_b200(sz, n, r, kind, dim, dtype, budget_bytes=16 << 30, profile=PROFILE)
    assert best["feasible"] and best["gcell_per_s"] > 0
    assert best["device_bytes"] <= 16 << 30
