"""Spec files, presets and run outputs (host-only, no device): the reference's
front-end formats -- proj/src/specfile.cpp:39-93 (parse_spec_json), the CLI
preset table proj/tools/so2dr_main.cpp:28-68 and proj/src/report.cpp:21-88.
The error behaviour follows the reference: syntax errors carry "line L, column
C", semantic errors name the field, an unknown kind/mode/preset is
InvalidSpecError."""
import glob
import json
import os

import numpy as np
import pytest

import paper_2309_08864_b200 as so2dr

REF_PRESETS = "/root/reference/proj/presets"
REFERENCE_NAMES = ["box2d1r-desk", "box2d2r-desk", "box2d3r-desk", "box2d4r-desk", "gradient2d-desk",
                   "box2d1r-paper", "box2d2r-paper", "box2d3r-paper", "box2d4r-paper", "gradient2d-paper"]


def test_preset_table_has_the_reference_presets_and_the_baseline_configs():
    names = so2dr.preset_names()
    assert names[:10] == REFERENCE_NAMES
    assert {"star2d1r-cfg1", "box2d1r-b200", "star3d1r-b200", "box3d1r-b200", "star2d2r-f64-b200"} <= set(names)
    with pytest.raises(so2dr.InvalidSpecError, match='unknown preset "nope"'):
        so2dr.preset_json("nope")


@pytest.mark.parametrize("name", REFERENCE_NAMES)
def test_reference_presets_parse(name):
    s = so2dr.preset(name)
    desk = name.endswith("-desk")
    kind, r = ("gradient", 1) if name.startswith("gradient") else ("box", int(name[5]))
    assert s.stencil_name == (f"box2d{r}r" if kind == "box" else "gradient2d")
    assert s.seed == (42 if desk else 7)
    assert s.mode == "so2dr"
    c = s.config
    assert (c.sz, c.r, c.d, c.k_on, c.n_strm, c.n, c.n_a) == ((512, r, 4, 4, 3, 64, 2) if desk else
                                                              (38400, r, 4, 4, 3, 640, 2))
    assert c.s_tb == (16 if desk else {1: 160, 2: 160, 3: 80, 4: 40}[r])
    assert s.kernel.k_on == c.k_on and s.kernel.tile == 32
    if kind == "box":  # the reference's box default fp32(1/(2r+1)^2)
        n = (2 * r + 1) ** 2
        assert np.all(s.stencil.weights == float(np.float32(1.0) / np.float32(n)))
    # every preset passes plan_chunks (paper presets are host-RAM-sized: plan only)
    fences, chunks = so2dr.plan_chunks(c)
    assert len(fences) == c.d + 1


@pytest.mark.skipif(not os.path.isdir(REF_PRESETS), reason="reference tree absent")
def test_shipped_reference_preset_files_match_the_table():
    """proj/presets/*.json (the files a reference user keeps) parse to exactly
    the built-in presets of the same name."""
    files = sorted(glob.glob(os.path.join(REF_PRESETS, "*.json")))
    assert len(files) == 10
    for f in files:
        name = os.path.basename(f)[:-5]
        a, b = so2dr.parse_spec_file(f), so2dr.preset(name)
        assert a.config == b.config and a.seed == b.seed and a.mode == b.mode, name
        assert a.stencil_name == b.stencil_name and np.array_equal(a.stencil.weights, b.stencil.weights)


def test_baseline_presets():
    c1 = so2dr.preset("star2d1r-cfg1")
    assert c1.stencil.kind == so2dr.STAR and c1.stencil_name == "star2d1r"
    w = c1.stencil.weights.reshape(3, 3)
    assert w[1, 1] == w[0, 1] == float(np.float32(0.2)) and w[0, 0] == 0.0
    assert (c1.config.sz, c1.config.d, c1.config.s_tb, c1.config.n) == (4096, 4, 4, 8)
    b = so2dr.preset("box2d1r-b200")
    assert (b.config.sz, b.config.d, b.config.s_tb, b.config.k_on, b.config.n) == (92160, 64, 64, 4, 64)
    s3 = so2dr.preset("star3d1r-b200")
    assert s3.stencil.dim == 3 and s3.stencil_name == "star3d1r"
    assert np.count_nonzero(s3.stencil.weights) == 7
    assert s3.stencil.weights[13] == float(np.float32(1.0) / np.float32(7.0))
    f64 = so2dr.preset("star2d2r-f64-b200")
    assert f64.dtype == np.float64 and f64.stencil_name == "star2d2r"
    assert f64.stencil.weights[12] == 1.0 / 9.0  # fp64 weights are not rounded to fp32


def _spec(**over):
    base = {"stencil": {"kind": "box", "radius": 1}, "grid": {"sz": 64, "seed": 3}, "mode": "so2dr",
            "config": {"d": 4, "s_tb": 8, "k_on": 4, "n_strm": 3, "n": 16}}
    for k, v in over.items():
        if v is None:
            base.pop(k)
        else:
            base[k] = v
    return json.dumps(base, indent=2)


def test_spec_defaults_and_optional_fields():
    s = so2dr.parse_spec_json(_spec(kernel={"tile": 16, "scratch_budget": 1 << 20}, hardware="hw.json",
                                    output={"grid_dump": "final.so2d"}))
    assert s.config.n_a == 2 and s.config.r == 1
    assert (s.kernel.k_on, s.kernel.tile, s.kernel.scratch_budget) == (4, 16, 1 << 20)
    assert s.hardware_path == "hw.json" and s.grid_dump_path == "final.so2d"
    s2 = so2dr.parse_spec_json(_spec())
    assert s2.hardware_path is None and s2.grid_dump_path is None and s2.kernel.tile == 32


def test_spec_syntax_error_reports_line_and_column():
    with pytest.raises(so2dr.IoError, match=r"bad\.json: JSON parse error at line 3, column 1"):
        so2dr.parse_spec_json('{\n  "stencil": {\n', "bad.json")
    with pytest.raises(so2dr.IoError, match=r"line 1, column 13"):
        so2dr.parse_spec_json('{"stencil": }', "x")


@pytest.mark.parametrize("over,msg", [
    ({"config": None}, "missing field config"),
    ({"config": {"d": 4, "s_tb": 8, "k_on": 4, "n": 16}}, "missing field config.n_strm"),
    ({"grid": {"sz": "64", "seed": 3}}, "field grid.sz has the wrong type"),
    ({"stencil": {"kind": "gradient", "radius": 2}}, 'stencil.radius 2 invalid for kind "gradient"'),
    ({"config": {"d": 5, "s_tb": 8, "k_on": 4, "n_strm": 3, "n": 16}}, "sz \\(64\\) must be divisible by d \\(5\\)"),
    ({"stencil": {"kind": "box", "radius": 1, "dim": 4}}, "stencil.dim 4 invalid"),
    ({"grid": {"sz": 64, "seed": 3, "dtype": "f16"}}, 'grid.dtype "f16" invalid'),
])
def test_spec_semantic_errors_name_the_field(over, msg):
    with pytest.raises(so2dr.IoError, match=msg):
        so2dr.parse_spec_json(_spec(**over), "s.json")


def test_spec_unknown_kind_and_mode_are_invalid_spec():
    with pytest.raises(so2dr.InvalidSpecError, match="unknown stencil kind"):
        so2dr.parse_spec_json(_spec(stencil={"kind": "hex", "radius": 1}))
    with pytest.raises(so2dr.InvalidSpecError):
        so2dr.parse_spec_json(_spec(mode="fastest"))
    with pytest.raises(so2dr.InvalidSpecError):
        so2dr.parse_spec_json(_spec(stencil={"kind": "box", "radius": 5}))


def test_spec_extensions_dim3_f64_weights():
    s = so2dr.parse_spec_json(_spec(stencil={"kind": "box", "radius": 1, "dim": 3},
                                    grid={"sz": 64, "seed": 1, "dtype": "f64"}))
    assert s.stencil.dim == 3 and s.dtype == np.float64 and s.stencil_name == "box3d1r"
    assert np.all(s.stencil.weights == 1.0 / 27.0)
    w = list(range(1, 10))
    s = so2dr.parse_spec_json(_spec(stencil={"kind": "box", "radius": 1, "weights": w}))
    assert np.array_equal(s.stencil.weights, np.array(w, dtype=np.float64))
    s = so2dr.parse_spec_json(_spec(stencil={"kind": "star", "radius": 2, "weights": [1, 2, 3, 4, 5, 6, 7, 8, 9]},
                                    grid={"sz": 64, "seed": 1, "dtype": "f64"}))
    e = s.stencil.weights.reshape(5, 5)
    assert list(e[:, 2]) == [1, 2, 5, 8, 9] and list(e[2, :]) == [3, 4, 5, 6, 7] and e[0, 0] == 0
    with pytest.raises(so2dr.IoError, match="stencil.weights needs 9"):
        so2dr.parse_spec_json(_spec(stencil={"kind": "box", "radius": 1, "weights": [1, 2]}))


def test_spec_file_round_trip(tmp_path):
    p = tmp_path / "spec.json"
    p.write_text(so2dr.preset_json("gradient2d-desk"))
    s = so2dr.parse_spec_file(str(p))
    assert s.stencil_name == "gradient2d" and s.config.sz == 512
    with pytest.raises(so2dr.IoError, match="cannot open spec file"):
        so2dr.parse_spec_file(str(tmp_path / "missing.json"))


def _fake_report(mode="so2dr"):
    cfg = so2dr.RunConfig(sz=64, r=1, d=4, s_tb=8, k_on=4, n_strm=3, n=16)
    led = {f: i + 1 for i, f in enumerate(so2dr.LEDGER_FIELDS)}
    tim = {f: 0 for f, _ in so2dr.TIMING_FIELDS}
    tim.update(wall_seconds=1.5, device_ms=2.0, kernel_launches=8, arena_peak=100, arena_capacity=200)
    return so2dr.RunReport(mode, cfg, led, tim, [])


def test_report_json_v1_keys_and_order():
    """proj/src/report.cpp:21-64: schema_version, mode, stencil, config, kernel,
    rounds, checksum, ledger, modeled_times, arena, transfer_time_excluded
    [, wall_seconds] -- in that order; deterministic output omits the clock."""
    txt = so2dr.report_to_json(_fake_report(), "box2d1r", 0xDEADBEEF)
    j = json.loads(txt)
    assert list(j)[:11] == ["schema_version", "mode", "stencil", "config", "kernel", "rounds", "checksum",
                            "ledger", "modeled_times", "arena", "transfer_time_excluded"]
    assert j["schema_version"] == 1 and j["checksum"] == "0x00000000deadbeef" and j["rounds"] == 9
    assert list(j["config"]) == ["sz", "r", "d", "s_tb", "k_on", "n_strm", "n", "n_a"]
    assert list(j["ledger"]) == ["htod_bytes", "dtoh_bytes", "ondevice_bytes", "scratch_load_bytes",
                                 "scratch_store_bytes", "element_updates", "redundant_updates",
                                 "kernel_invocations", "rounds"]
    assert j["arena"] == {"peak_bytes": 100, "capacity_bytes": 200}
    assert j["wall_seconds"] == 1.5 and j["measured"]["kernel_launches"] == 8
    assert txt.startswith('{\n  "schema_version": 1,\n  "mode": "so2dr",')
    det = so2dr.report_to_json(_fake_report(), "box2d1r", 7, deterministic=True)
    assert "wall_seconds" not in det and "measured" not in det
    assert det == so2dr.report_to_json(_fake_report(), "box2d1r", 7, deterministic=True)
    assert json.loads(so2dr.report_to_json(_fake_report("incore"), "x", 0))["transfer_time_excluded"] is True


def test_ledger_and_diagnostics_csv():
    led = {f: i for i, f in enumerate(so2dr.LEDGER_FIELDS)}
    assert so2dr.ledger_to_csv(led) == ("counter,value\nhtod_bytes,0\ndtoh_bytes,1\nondevice_bytes,2\n"
                                        "scratch_load_bytes,3\nscratch_store_bytes,4\nelement_updates,5\n"
                                        "redundant_updates,6\nkernel_invocations,7\nrounds,8\n")
    rows = [{"round": 0, "chunk": 1, "stage": "kernel", "bytes": 10, "updates": 20}]
    assert so2dr.diagnostics_to_csv(rows) == "round,chunk,stage,bytes,updates\n0,1,kernel,10,20\n"
    assert so2dr.diagnostics_to_csv([]) == "round,chunk,stage,bytes,updates\n"
