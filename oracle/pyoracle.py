"""ctypes wrappers over the CPU oracle (liboracle.so) and the compiled reference
(_ref/libso2dr_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / reference legs of bench.py, always as the checker or the CPU
baseline -- never on the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "liboracle.so")
_REF_V3 = os.path.join(HERE, "_ref", "libso2dr_ref.so")
_REF_NATIVE = os.path.join(HERE, "_ref", "libso2dr_ref_native.so")
_NATIVE_FLAGS = os.path.join(HERE, "_ref", "native_flags.txt")


def _host_isa() -> set:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("flags"):
                return {f.replace("_", "") for f in line.split(":", 1)[1].split()}
    except OSError:
        pass
    return set()


def ref_build_info() -> dict:
    """Which reference build runs here: the -march=native build of the build host
    (oracle/Makefile) when this CPU has every ISA extension it enabled, else the
    portable -march=x86-64-v3 build."""
    info = {"path": _REF_V3, "march": "x86-64-v3", "missing_isa": []}
    try:
        lines = [l.split() for l in open(_NATIVE_FLAGS) if l.strip()]
    except OSError:
        return info
    march = next((l[1] for l in lines if l[0] == "march" and len(l) > 1), "native")
    need = {l[0].replace("_", "") for l in lines if l[0] != "march"}
    have = _host_isa()
    have |= {"bmi"} if "bmi1" in have else set()
    missing = sorted(need - have)
    if os.path.exists(_REF_NATIVE) and not missing:
        return {"path": _REF_NATIVE, "march": march, "missing_isa": []}
    info["missing_isa"] = missing
    info["native_march"] = march
    return info


_REF = ref_build_info()["path"]

BOX, GRADIENT, STAR = 0, 1, 2

_oracle = None
_ref = None


class _Stencil(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("dim", ctypes.c_int), ("radius", ctypes.c_int),
                ("w", ctypes.POINTER(ctypes.c_double))]


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    targets = ["all"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(_LIB):
            build()
        L = ctypes.CDLL(_LIB)
        vp, i, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64
        L.orc_cell_value.restype = ctypes.c_float
        L.orc_cell_value.argtypes = [u64, i, i]
        L.orc_cell_value3.restype = ctypes.c_float
        L.orc_cell_value3.argtypes = [u64, i, i, i]
        for t in ("f32", "f64"):
            getattr(L, f"orc_init_{t}").argtypes = [vp, i, i, i, u64]
            getattr(L, f"orc_step_{t}").argtypes = [vp, vp, i, i, ctypes.POINTER(_Stencil)]
            getattr(L, f"orc_run_{t}").argtypes = [vp, vp, i, i, ctypes.POINTER(_Stencil), i]
            getattr(L, f"orc_init_block_{t}").argtypes = [vp, i, i, i, i, i, i, i, u64]
            getattr(L, f"orc_run_block_{t}").argtypes = [vp, vp, i, i, i, i, ctypes.POINTER(_Stencil), i, vp, vp]
        L.orc_fnv1a.restype = u64
        L.orc_fnv1a.argtypes = [vp, ctypes.c_size_t]
        _oracle = L
    return _oracle


def have_ref() -> bool:
    return os.path.exists(_REF)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF):
            raise FileNotFoundError(_REF + " (built from /root/reference by oracle/Makefile)")
        L = ctypes.CDLL(_REF)
        vp, i, u64, cp = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_char_p
        L.ref_init_grid.argtypes = [i, i, u64, vp]
        L.ref_checksum.restype = u64
        L.ref_checksum.argtypes = [i, i, vp]
        L.ref_run_reference.argtypes = [i, i, vp, i, i, vp, i, vp, cp, i]
        L.ref_run_engine.argtypes = [i, i, i, vp, vp, vp, u64, u64, ctypes.c_double,
                                     ctypes.c_double, i, i, vp, vp, vp, vp, vp, cp, i]
        L.ref_fused_kernel.argtypes = [i, i, vp, vp, vp, i, i, i, i, i, i, vp, vp, vp, vp, vp, cp, i]
        L.ref_expected_ledger.argtypes = [i, vp, vp, vp, vp]
        L.ref_arena_bytes.restype = u64
        L.ref_arena_bytes.argtypes = [vp, vp]
        _ref = L
    return _ref


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def padded_shape(dim: int, sz: int, r: int):
    p = sz + 2 * r
    return (p, p, p) if dim == 3 else (p, p)


def init_grid(sz: int, r: int, seed: int, dim: int = 2, dtype=np.float32) -> np.ndarray:
    g = np.empty(padded_shape(dim, sz, r), dtype=dtype)
    fn = lib().orc_init_f32 if dtype == np.float32 else lib().orc_init_f64
    fn(_ptr(g), dim, sz, r, seed)
    return g


def _stencil(kind: int, dim: int, radius: int, weights) -> tuple:
    e = 2 * radius + 1
    n = e ** dim
    if weights is None:
        weights = np.zeros(n)
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).reshape(-1))
    assert w.size == n, (w.size, n)
    st = _Stencil(kind, dim, radius, w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return st, w


def run(grid: np.ndarray, kind: int, radius: int, weights, steps: int) -> np.ndarray:
    """The serial ping-pong oracle (proj/src/stencil.cpp:162-174) for dim 2/3, f32/f64."""
    dim = grid.ndim
    sz = grid.shape[0] - 2 * radius
    st, keep = _stencil(kind, dim, radius, weights)
    g = np.ascontiguousarray(grid)
    out = np.empty_like(g)
    fn = lib().orc_run_f32 if g.dtype == np.float32 else lib().orc_run_f64
    fn(_ptr(g), _ptr(out), sz, radius, ctypes.byref(st), steps)
    del keep
    return out


def init_block(lo, hi, seed: int, dtype=np.float32) -> np.ndarray:
    """init_grid values of the padded-grid box [lo, hi) (2 or 3 per-dim bounds)."""
    dim = len(lo)
    shape = tuple(b - a for a, b in zip(lo, hi))
    g = np.empty(shape, dtype=dtype)
    z0, y0, x0 = (0,) + tuple(lo) if dim == 2 else tuple(lo)
    nz, ny, nx = (1,) + shape if dim == 2 else shape
    fn = lib().orc_init_block_f32 if dtype == np.float32 else lib().orc_init_block_f64
    fn(_ptr(g), dim, z0, y0, x0, nz, ny, nx, seed)
    return g


def run_block(block: np.ndarray, kind: int, radius: int, weights, steps: int, window=None) -> np.ndarray:
    """run() on a rectangular padded block whose outer `radius` cells are held.
    window=(lo, hi) (block coordinates): only that window's dependency cone is
    evolved; only the window of the result is meaningful."""
    dim = block.ndim
    st, keep = _stencil(kind, dim, radius, weights)
    g = np.ascontiguousarray(block)
    out = np.empty_like(g)
    nz, ny, nx = (1,) + g.shape if dim == 2 else g.shape
    fn = lib().orc_run_block_f32 if g.dtype == np.float32 else lib().orc_run_block_f64
    wl = wh = None
    if window is not None:
        lo, hi = window
        if dim == 2:
            lo, hi = (0,) + tuple(lo), (1,) + tuple(hi)
        wl = (ctypes.c_int * 3)(*lo)
        wh = (ctypes.c_int * 3)(*hi)
    fn(_ptr(g), _ptr(out), nz, ny, nx, radius, ctypes.byref(st), steps,
       ctypes.cast(wl, ctypes.c_void_p) if wl else None, ctypes.cast(wh, ctypes.c_void_p) if wh else None)
    del keep
    return out


def window_expected(init_window, sz: int, radius: int, steps: int, lo, hi, kind: int, weights, dim: int = 2):
    """Light-cone check of a full-size run: the exact state after `steps` of the
    padded-grid window [lo, hi) (per-dim tuples), computed from a cut-out with a
    margin of radius*(steps+1) (clipped at the grid edge, where the real ring is
    held). `init_window(lo, hi)` returns the initial padded-grid values of a box."""
    p = sz + 2 * radius
    m = radius * (steps + 1)
    clo = tuple(max(0, a - m) for a in lo)
    chi = tuple(min(p, b + m) for b in hi)
    cut = init_window(clo, chi)
    wlo = tuple(a - c for a, c in zip(lo, clo))
    whi = tuple(b - c for b, c in zip(hi, clo))
    out = run_block(cut, kind, radius, weights, steps, (wlo, whi))
    return np.ascontiguousarray(out[tuple(slice(a, b) for a, b in zip(wlo, whi))])


def step(grid: np.ndarray, kind: int, radius: int, weights) -> np.ndarray:
    return run(grid, kind, radius, weights, 1)


def fnv1a(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a)
    return int(lib().orc_fnv1a(_ptr(a), a.nbytes))


def box_weights(radius: int, dim: int = 2, dtype=np.float32) -> np.ndarray:
    """proj/src/stencil.cpp:27-33 default weights fp(1/(2r+1)^dim), as float64 carrier."""
    n = (2 * radius + 1) ** dim
    w = dtype(1.0) / dtype(n)
    return np.full(n, float(w))


def star_weights(radius: int, dim: int = 2, dtype=np.float32, w=None) -> np.ndarray:
    """Star stencil as a box weight vector with zero off-axis entries."""
    e = 2 * radius + 1
    val = float(dtype(1.0) / dtype(2 * dim * radius + 1)) if w is None else float(dtype(w))
    out = np.zeros((e,) * dim)
    for idx in np.ndindex(*out.shape):
        if sum(1 for c in idx if c != radius) <= 1:
            out[idx] = val
    return out.reshape(-1)
