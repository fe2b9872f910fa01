"""Spec files / presets end to end on the GPU: every desk preset (and the
BASELINE config-1 preset) parsed -> run_engine on the B200 -> the FNV-1a
checksum the reference's own code produced for the same spec
(tests/golden/golden.json, made by tests/golden/make_golden.py from the
compiled reference). The report/ledger writers are checked on the real run."""
import json
import os

import numpy as np
import pytest

import paper_2309_08864_b200 as so2dr

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def _golden(stencil, sz, n):
    for c in GOLD["checksums"]:
        if c["stencil"] == stencil and c["sz"] == sz and c["n"] == n:
            return c
    raise KeyError((stencil, sz, n))


@pytest.mark.parametrize("name", ["box2d1r-desk", "box2d2r-desk", "box2d3r-desk", "box2d4r-desk",
                                  "gradient2d-desk", "star2d1r-cfg1"])
def test_preset_runs_to_the_reference_checksum(engine, name):
    spec = so2dr.preset(name)
    gold = _golden(spec.stencil_name, spec.config.sz, spec.config.n)
    grid = engine.init_grid(spec.config.sz, spec.config.r, spec.seed)
    assert so2dr.grid_checksum(grid) == gold["in_fnv"]
    grid, rep = engine.run_spec(spec, grid=grid)
    assert so2dr.grid_checksum(grid) == gold["out_fnv"], name
    exp = so2dr.expected_ledger(spec.mode, spec.config, spec.kernel)
    for k in ("htod", "dtoh", "ondevice", "kernel_invocations", "rounds"):
        assert rep.ledger[k] == exp[k], k
    # run outputs in the reference's formats, from the real run
    j = json.loads(so2dr.report_to_json(rep, spec.stencil_name, so2dr.grid_checksum(grid)))
    assert j["checksum"] == "0x%016x" % gold["out_fnv"]
    assert j["rounds"] == rep.ledger["rounds"] == -(-spec.config.n // spec.config.s_tb)
    assert j["measured"]["kernel_launches"] > 0
    csv = so2dr.ledger_to_csv(rep.ledger)
    assert f"htod_bytes,{rep.ledger['htod']}\n" in csv
    diag = so2dr.diagnostics_to_csv(rep.diagnostics)
    assert diag.count("\n") == len(rep.diagnostics) + 1 and ",kernel," in diag


@pytest.mark.parametrize("mode", ["so2dr", "resreu", "incore"])
def test_spec_mode_override_gives_the_same_grid(engine, mode):
    """The CLI's --mode override (so2dr_main.cpp:147-148): every mode of the
    same spec lands on the same reference checksum."""
    spec = so2dr.parse_spec_json(so2dr.preset_json("box2d1r-desk").replace('"so2dr"', f'"{mode}"'))
    grid, _ = engine.run_spec(spec)
    assert so2dr.grid_checksum(grid) == _golden("box2d1r", 512, 64)["out_fnv"]
