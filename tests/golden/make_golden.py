"""Generate tests/golden/golden.json from the REFERENCE itself.

Runs only in the build container, where /root/reference exists: it loads
oracle/_ref/libso2dr_ref.so (the unmodified reference sources compiled by
oracle/Makefile) and records its outputs. The GPU box never needs
/root/reference: the tests read the committed JSON.

    python tests/golden/make_golden.py
"""
import base64
import ctypes
import json
import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as o  # noqa: E402


def pack(a: np.ndarray) -> str:
    return base64.b64encode(zlib.compress(np.ascontiguousarray(a).tobytes(), 9)).decode()


def ref_grid(sz, r, seed):
    g = np.empty((sz + 2 * r, sz + 2 * r), np.float32)
    o.ref().ref_init_grid(sz, r, seed, g.ctypes.data)
    return g


def ref_run(kind, r, w, g, steps):
    out = np.empty_like(g)
    err = ctypes.create_string_buffer(256)
    wf = None if w is None else np.asarray(w, np.float32)
    rc = o.ref().ref_run_reference(kind, r, None if wf is None else wf.ctypes.data, g.shape[0] - 2 * r, r,
                                   g.ctypes.data, steps, out.ctypes.data, err, 256)
    assert rc == 0, err.value
    return out


def ref_engine(mode, kind, r, w, cfg, kp, g, budget=64 << 20):
    out = np.empty_like(g)
    led = (ctypes.c_uint64 * 9)()
    peak = ctypes.c_uint64()
    wall = ctypes.c_double()
    err = ctypes.create_string_buffer(512)
    wf = None if w is None else np.asarray(w, np.float32)
    rc = o.ref().ref_run_engine(mode, kind, r, None if wf is None else wf.ctypes.data, (ctypes.c_int * 8)(*cfg),
                                (ctypes.c_int * 2)(*kp), budget, 10737418240, 760e9, 15.75e9, 0, 0,
                                g.ctypes.data, out.ctypes.data, led, ctypes.byref(peak), ctypes.byref(wall), err, 512)
    assert rc == 0, err.value
    return out, list(led), peak.value


def main():
    R = o.ref()
    gold = {"source": "oracle/_ref/libso2dr_ref.so built from /root/reference/proj/src (unmodified)"}
    gold["cell_value"] = [[42, 0, 0, float.hex(float(o.lib().orc_cell_value(42, 0, 0)))],
                          [42, 1, 2, float.hex(float(o.lib().orc_cell_value(42, 1, 2)))],
                          [0, 0, 0, float.hex(float(o.lib().orc_cell_value(0, 0, 0)))]]
    star1 = o.star_weights(1).astype(np.float32)
    stencils = {"box2d1r": (0, 1, None), "box2d2r": (0, 2, None), "box2d3r": (0, 3, None),
                "box2d4r": (0, 4, None), "gradient2d": (1, 1, None), "star2d1r": (0, 1, star1)}

    # small full grids after n steps (run_reference), bit-exact fixtures
    small = []
    for name, (kind, r, w) in stencils.items():
        for sz, seed, n in [(24, 123, 3), (33, 7, 5)]:
            g = ref_grid(sz, r, seed)
            out = ref_run(kind, r, w, g, n)
            small.append({"stencil": name, "sz": sz, "r": r, "seed": seed, "n": n,
                          "in_fnv": o.fnv1a(g), "out_fnv": o.fnv1a(out), "out": pack(out)})
    gold["small_grids"] = small

    # checksums at desk / config-1 scale
    sums = []
    for name, (kind, r, w) in stencils.items():
        g = ref_grid(512, r, 42)
        sums.append({"stencil": name, "sz": 512, "r": r, "seed": 42, "n": 64, "in_fnv": o.fnv1a(g),
                     "out_fnv": o.fnv1a(ref_run(kind, r, w, g, 64))})
    for name in ("star2d1r", "box2d1r", "gradient2d"):
        kind, r, w = stencils[name]
        g = ref_grid(4096, r, 42)
        out = ref_run(kind, r, w, g, 8)
        sums.append({"stencil": name, "sz": 4096, "r": r, "seed": 42, "n": 8, "in_fnv": o.fnv1a(g),
                     "out_fnv": o.fnv1a(out), "cell_1_1": float.hex(float(out[1, 1])),
                     "cell_2048_2048": float.hex(float(out[2048, 2048]))})
    gold["checksums"] = sums

    # engine ledgers (reference run_engine) for a spread of configs and modes
    eng = []
    cfgs = [  # sz r d s_tb k_on n_strm n n_a ; kp k_on tile ; stencil
        ((64, 1, 4, 4, 2, 3, 8, 2), (2, 16), "box2d1r"),
        ((64, 1, 4, 4, 4, 3, 10, 2), (4, 16), "box2d1r"),
        ((64, 1, 4, 4, 4, 3, 8, 2), (4, 128), "box2d1r"),
        ((64, 2, 4, 4, 4, 3, 8, 2), (4, 256), "box2d2r"),
        ((64, 2, 4, 4, 2, 2, 8, 2), (2, 16), "box2d2r"),
        ((64, 1, 4, 4, 1, 3, 10, 2), (1, 32), "gradient2d"),
        ((96, 3, 2, 4, 3, 1, 11, 2), (3, 8), "box2d3r"),
        ((96, 4, 2, 3, 2, 2, 7, 2), (2, 32), "box2d4r"),
        ((512, 1, 4, 16, 4, 3, 64, 2), (4, 32), "box2d1r"),
        ((512, 1, 4, 4, 4, 3, 8, 2), (4, 32), "star2d1r"),
    ]
    for cfg, kp, name in cfgs:
        kind, r, w = stencils[name]
        g = ref_grid(cfg[0], r, 1000 + cfg[0] + r)
        for mode in (0, 1, 2):
            out, led, peak = ref_engine(mode, kind, r, w, cfg, kp, g)
            eng.append({"mode": ["so2dr", "resreu", "incore"][mode], "cfg": list(cfg), "kp": list(kp),
                        "stencil": name, "seed": 1000 + cfg[0] + r, "ledger": led, "arena_peak": peak,
                        "out_fnv": o.fnv1a(out)})
    gold["engine"] = eng

    # fused_kernel stats (kernels.cpp accounting), incl. proj/tests/test_engine.cpp:34-65 cases
    fk = []
    g = ref_grid(62, 1, 9)
    for region, s, tile in [((20, 36, 20, 36), 2, 8), ((10, 26, 8, 40), 1, 64), ((1, 63, 0, 64), 3, 16),
                            ((5, 60, 3, 61), 4, 32), ((1, 63, 0, 64), 8, 1024), ((0, 64, 0, 64), 2, 7),
                            ((30, 31, 0, 64), 5, 3)]:
        b0, b1 = g.copy(), g.copy()
        st = (ctypes.c_uint64 * 4)()
        err = ctypes.create_string_buffer(256)
        rc = R.ref_fused_kernel(0, 1, None, b0.ctypes.data, b1.ctypes.data, 0, 64, 64, 0, s, tile,
                                (ctypes.c_int * 4)(*region), (ctypes.c_int * 4)(1, 63, 1, 63),
                                (ctypes.c_int * 4)(*region), st, None, err, 256)
        assert rc == 0
        fk.append({"region": list(region), "steps": s, "tile": tile, "r": 1, "interior": [1, 63, 1, 63],
                   "rows": [0, 64], "cols": 64, "stats": list(st)})
    gold["fused_stats"] = fk

    # closed forms and the modeled arena formula
    ex = []
    for cfg, kp, _ in cfgs + [((4096, 1, 4, 4, 4, 3, 8, 2), (4, 32), "")]:
        for mode in (0, 1, 2):
            out6 = (ctypes.c_uint64 * 6)()
            exact = ctypes.c_int()
            R.ref_expected_ledger(mode, (ctypes.c_int * 8)(*cfg), (ctypes.c_int * 2)(*kp), out6, ctypes.byref(exact))
            ex.append({"mode": ["so2dr", "resreu", "incore"][mode], "cfg": list(cfg), "kp": list(kp),
                       "expected": list(out6), "exact": bool(exact.value)})
        ex[-1]["arena_bytes"] = R.ref_arena_bytes((ctypes.c_int * 8)(*cfg), (ctypes.c_int * 2)(*kp))
    gold["expected_ledger"] = ex

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(gold, f, indent=0)
    print("wrote", os.path.join(HERE, "golden.json"), os.path.getsize(os.path.join(HERE, "golden.json")), "bytes")


if __name__ == "__main__":
    main()
