"""B200-native SO2DR out-of-core stencil engine (arXiv 2309.08864).

Python binding of the C ABI in include/so2dr_cuda.h (libso2dr_b200.so, built
in-tree by `make`). The names mirror the reference's C++ API
(proj/include/so2dr/*.hpp): StencilSpec, RunConfig, KernelPlan,
HardwareModel, EngineHooks, run_engine, fused_kernel, apply_step,
run_reference, init_grid, expected_ledger, plan_chunks, and the same error
types. Every compute call executes on the GPU; there is no CPU fallback --
without the built library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes
import json
import dataclasses
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SO2DR_LIB: load an experiment build instead (tools/build_variant.sh)
LIB_PATH = os.environ.get("SO2DR_LIB") or os.path.join(HERE, "libso2dr_b200.so")

# ---------------------------------------------------------------- errors --
# proj/include/so2dr/errors.hpp:11-63


class Error(RuntimeError):
    pass


class InvalidSpecError(Error):
    pass


class InfeasibleError(Error):
    def __init__(self, msg: str, constraint: str = ""):
        super().__init__(msg)
        self.constraint = constraint


class OutOfDeviceMemoryError(Error):
    def __init__(self, msg: str, allocation_id: str = ""):
        super().__init__(msg)
        self.allocation_id = allocation_id


class ContractError(Error):
    pass


class IoError(Error):
    pass


class DeviceError(Error):
    pass


# ------------------------------------------------------------- C structs --

class _Stencil(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("dim", ctypes.c_int32), ("radius", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("weights", ctypes.POINTER(ctypes.c_double))]


class _Cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("sz", "r", "d", "s_tb", "k_on", "n_strm", "n", "n_a")]


class _KPlan(ctypes.Structure):
    _fields_ = [("k_on", ctypes.c_int32), ("tile", ctypes.c_int32), ("scratch_budget", ctypes.c_uint64)]


class _HW(ctypes.Structure):
    _fields_ = [("c_dmem", ctypes.c_uint64), ("bw_dmem", ctypes.c_double), ("bw_intc", ctypes.c_double),
                ("b_elem", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class _Hooks(ctypes.Structure):
    _fields_ = [("corrupt_share", ctypes.c_int32), ("boundary", ctypes.c_int32)]


LEDGER_FIELDS = ("htod", "dtoh", "ondevice", "scratch_load", "scratch_store", "element_updates",
                 "redundant_updates", "kernel_invocations", "rounds")


class _Ledger(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in LEDGER_FIELDS]


TIMING_FIELDS = [("wall_seconds", ctypes.c_double), ("device_ms", ctypes.c_double),
                 ("kernel_ms", ctypes.c_double), ("kernel_max_ms", ctypes.c_double),
                 ("kernel_launches", ctypes.c_uint64), ("kernel_alg_bytes", ctypes.c_uint64),
                 ("cell_updates", ctypes.c_uint64), ("h2d_bytes", ctypes.c_uint64),
                 ("d2h_bytes", ctypes.c_uint64), ("d2d_bytes", ctypes.c_uint64),
                 ("peer_bytes", ctypes.c_uint64), ("arena_peak", ctypes.c_uint64),
                 ("arena_capacity", ctypes.c_uint64), ("device_bytes", ctypes.c_uint64)]


class _Timing(ctypes.Structure):
    _fields_ = TIMING_FIELDS


class _Spec(ctypes.Structure):
    _fields_ = [("stencil", _Stencil), ("weights_buf", ctypes.c_double * 125), ("config", _Cfg),
                ("kernel", _KPlan), ("seed", ctypes.c_uint64), ("mode", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("stencil_name", ctypes.c_char * 32), ("hardware_path", ctypes.c_char * 512),
                ("grid_dump_path", ctypes.c_char * 512)]


class _Diag(ctypes.Structure):
    _fields_ = [("round", ctypes.c_int32), ("chunk", ctypes.c_int32), ("stage", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("bytes", ctypes.c_uint64), ("updates", ctypes.c_uint64),
                ("ms", ctypes.c_double), ("t0_ms", ctypes.c_double)]


PEER_BLOB_BYTES = 512
STAGES = ("htod", "share_read", "share_write", "kernel", "dtoh")

_lib = None

EXPORTS = (
    "so2dr_abi_version", "so2dr_device_count", "so2dr_ctx_create", "so2dr_ctx_destroy",
    "so2dr_ctx_set_profiling", "so2dr_last_error", "so2dr_last_constraint",
    "so2dr_last_allocation_id", "so2dr_host_register", "so2dr_host_unregister", "so2dr_run",
    "so2dr_host_alloc", "so2dr_host_free",
    "so2dr_slab_rows", "so2dr_slab_prepare", "so2dr_slab_connect", "so2dr_slab_run",
    "so2dr_fused_kernel", "so2dr_apply_step", "so2dr_run_reference", "so2dr_init_grid",
    "so2dr_init_rows", "so2dr_grid_checksum", "so2dr_arena_bytes", "so2dr_device_bytes", "so2dr_k1_max_steps",
    "so2dr_plan_b200", "so2dr_predict_b200", "so2dr_device_numa_node", "so2dr_pci_numa_node", "so2dr_slab_info",
    "so2dr_plan_chunks", "so2dr_expected_ledger", "so2dr_kernel_stats",
    "so2dr_spec_parse", "so2dr_spec_parse_file", "so2dr_preset_count", "so2dr_preset_name",
    "so2dr_preset_json", "so2dr_report_json", "so2dr_ledger_csv", "so2dr_diagnostics_csv",
)


def lib():
    """Load libso2dr_b200.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build()) first")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
    P = ctypes.POINTER
    L.so2dr_abi_version.restype = i32
    L.so2dr_device_count.restype = i32
    L.so2dr_ctx_create.argtypes = [i32, u64, P(vp)]
    L.so2dr_ctx_destroy.argtypes = [vp]
    L.so2dr_ctx_destroy.restype = None
    L.so2dr_ctx_set_profiling.argtypes = [vp, i32]
    for f in ("so2dr_last_error", "so2dr_last_constraint", "so2dr_last_allocation_id"):
        getattr(L, f).argtypes = [vp]
        getattr(L, f).restype = ctypes.c_char_p
    L.so2dr_host_register.argtypes = [vp, vp, sz]
    L.so2dr_host_alloc.argtypes = [vp, sz, P(vp)]
    L.so2dr_host_free.argtypes = [vp, vp]
    L.so2dr_host_unregister.argtypes = [vp, vp]
    L.so2dr_run.argtypes = [vp, i32, P(_Stencil), P(_Cfg), P(_KPlan), P(_HW), P(_Hooks), i32, vp,
                            P(_Ledger), P(_Timing), P(_Diag), sz, P(sz)]
    L.so2dr_slab_rows.argtypes = [P(_Cfg), i32, i32, i32, P(i64), P(i64)]
    L.so2dr_slab_prepare.argtypes = [vp, P(_Stencil), P(_Cfg), i32, i32, i32, ctypes.c_char_p]
    L.so2dr_slab_connect.argtypes = [vp, ctypes.c_char_p, ctypes.c_char_p]
    L.so2dr_slab_run.argtypes = [vp, P(_Stencil), P(_Cfg), P(_KPlan), i32, vp, P(_Ledger), P(_Timing)]
    L.so2dr_fused_kernel.argtypes = [vp, P(_Stencil), i32, vp, vp, i32, i32, i32, i32, i32, i32,
                                     P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32), P(u64)]
    L.so2dr_apply_step.argtypes = [vp, P(_Stencil), i32, i32, i32, vp, vp, i32, i32]
    L.so2dr_run_reference.argtypes = [vp, P(_Stencil), i32, i32, i32, vp, vp, i32]
    L.so2dr_init_grid.argtypes = [vp, i32, i32, i32, i32, u64, vp]
    L.so2dr_init_rows.argtypes = [vp, i32, i32, i32, i32, u64, i64, i64, vp]
    L.so2dr_grid_checksum.argtypes = [vp, sz]
    L.so2dr_grid_checksum.restype = u64
    L.so2dr_arena_bytes.argtypes = [P(_Cfg), P(_KPlan), P(u64)]
    L.so2dr_device_bytes.argtypes = [P(_Cfg), i32, i32, P(u64)]
    L.so2dr_plan_chunks.argtypes = [P(_Cfg), P(ctypes.c_int32), P(ctypes.c_int32)]
    L.so2dr_kernel_stats.argtypes = [i32, i32, i32, P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32),
                                     i32, i32, i64, P(u64)]
    L.so2dr_expected_ledger.argtypes = [i32, P(_Cfg), P(_KPlan), i32, i32, P(u64), P(ctypes.c_int32)]
    cp = ctypes.c_char_p
    L.so2dr_spec_parse.argtypes = [cp, cp, P(_Spec)]
    L.so2dr_spec_parse_file.argtypes = [cp, P(_Spec)]
    L.so2dr_preset_count.restype = i32
    L.so2dr_preset_name.argtypes = [i32]
    L.so2dr_preset_name.restype = cp
    L.so2dr_preset_json.argtypes = [cp, cp, sz, P(sz)]
    L.so2dr_report_json.argtypes = [P(_ReportIn), cp, sz, P(sz)]
    L.so2dr_ledger_csv.argtypes = [P(_Ledger), cp, sz, P(sz)]
    L.so2dr_diagnostics_csv.argtypes = [P(_Diag), sz, cp, sz, P(sz)]
    _lib = L
    return L


class _ReportIn(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("deterministic", ctypes.c_int32), ("stencil_name", ctypes.c_char_p),
                ("config", _Cfg), ("kernel", _KPlan), ("checksum", ctypes.c_uint64), ("ledger", _Ledger),
                ("hw", ctypes.POINTER(_HW)), ("measured", ctypes.POINTER(_Timing))]


def _raise(status: int, ctx=None):
    L = lib()
    h = ctx if ctx is not None else None
    msg = (L.so2dr_last_error(h) or b"").decode()
    if status == 1:
        raise InvalidSpecError(msg)
    if status == 2:
        raise InfeasibleError(msg, (L.so2dr_last_constraint(h) or b"").decode())
    if status == 3:
        raise OutOfDeviceMemoryError(msg, (L.so2dr_last_allocation_id(h) or b"").decode())
    if status == 4:
        raise ContractError(msg)
    if status == 5:
        raise IoError(msg)
    if status == 6:
        raise DeviceError(msg)
    if status == 7:
        raise IndexError(msg)
    raise Error(f"status {status}: {msg}")


def _check(status: int, ctx=None):
    if status != 0:
        _raise(status, ctx)


# ------------------------------------------------------------ API types --
# proj/include/so2dr/stencil.hpp:14-45, layout.hpp:13-51, engine.hpp:22-65

BOX, GRADIENT, STAR = 0, 1, 2
MODES = {"so2dr": 0, "resreu": 1, "incore": 2}


@dataclasses.dataclass
class StencilSpec:
    kind: int
    radius: int
    dim: int = 2
    weights: Optional[np.ndarray] = None  # (2r+1)^dim canonical-order weights (float64 carrier)

    @staticmethod
    def box(radius: int, weights: Optional[Sequence[float]] = None, dim: int = 2,
            dtype=np.float32) -> "StencilSpec":
        n = (2 * radius + 1) ** dim
        if weights is None:
            weights = np.full(n, float(dtype(1.0) / dtype(n)))
        w = np.asarray(weights, dtype=np.float64).reshape(-1)
        if w.size != n:
            raise InvalidSpecError(f"box radius {radius} needs {n} weights, got {w.size}")
        return StencilSpec(BOX, radius, dim, w)

    @staticmethod
    def star(radius: int, w: Optional[float] = None, dim: int = 2, dtype=np.float32) -> "StencilSpec":
        e = 2 * radius + 1
        val = float(dtype(1.0) / dtype(2 * dim * radius + 1)) if w is None else float(dtype(w))
        arr = np.zeros((e,) * dim)
        for idx in np.ndindex(*arr.shape):
            if sum(1 for c in idx if c != radius) <= 1:
                arr[idx] = val
        return StencilSpec(STAR, radius, dim, arr.reshape(-1))

    @staticmethod
    def gradient() -> "StencilSpec":
        return StencilSpec(GRADIENT, 1, 2, np.zeros(9))

    def name(self) -> str:
        if self.kind == GRADIENT:
            return "gradient2d"
        return f"{'star' if self.kind == STAR else 'box'}{self.dim}d{self.radius}r"

    def _c(self):
        w = self.weights if self.weights is not None else np.zeros((2 * self.radius + 1) ** self.dim)
        w = np.ascontiguousarray(w, dtype=np.float64)
        return _Stencil(self.kind, self.dim, self.radius, 0, w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), w


@dataclasses.dataclass
class RunConfig:
    sz: int = 0
    r: int = 1
    d: int = 1
    s_tb: int = 1
    k_on: int = 1
    n_strm: int = 3
    n: int = 0
    n_a: int = 2

    def padded(self) -> int:
        return self.sz + 2 * self.r

    def _c(self):
        return _Cfg(self.sz, self.r, self.d, self.s_tb, self.k_on, self.n_strm, self.n, self.n_a)


@dataclasses.dataclass
class KernelPlan:
    k_on: int = 4
    tile: int = 32
    scratch_budget: int = 192 * 1024

    def _c(self):
        return _KPlan(self.k_on, self.tile, self.scratch_budget)


@dataclasses.dataclass
class HardwareModel:
    name: str = "b200"
    c_dmem: int = 183359 << 20
    bw_dmem: float = 6448.4e9
    bw_intc: float = 50.0e9
    b_elem: int = 4

    def _c(self):
        return _HW(self.c_dmem, self.bw_dmem, self.bw_intc, self.b_elem, 0)


def default_hardware() -> HardwareModel:  # proj/src/layout.cpp:12-20
    return HardwareModel("rtx3080-desktop", 10737418240, 760.0e9, 15.75e9, 4)


def desk_hardware() -> HardwareModel:  # proj/src/layout.cpp:22-30
    return HardwareModel("desk-sim", 2147483648, 40.0e9, 16.0e9, 4)


@dataclasses.dataclass
class EngineHooks:
    corrupt_share: bool = False
    boundary: int = 0


@dataclasses.dataclass
class RunReport:
    mode: str
    config: RunConfig
    ledger: dict
    timing: dict
    diagnostics: list
    checksum: Optional[int] = None


def _ptr(a) -> int:
    """Address of a numpy array or torch tensor (host or CUDA)."""
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ContractError("grid must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ContractError("grid must be contiguous")
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise ContractError(f"unsupported grid object {type(a)}")


def _dtype_code(a) -> int:
    dt = getattr(a, "dtype", None)
    s = str(dt)
    if s in ("float32", "torch.float32"):
        return 0
    if s in ("float64", "torch.float64"):
        return 1
    raise InvalidSpecError(f"grid dtype must be float32 or float64, got {dt}")


def _numel(a) -> int:
    return int(a.size) if isinstance(a, np.ndarray) else int(a.numel())


def _shape(a) -> tuple:
    return tuple(int(x) for x in a.shape)


def _contig(a) -> bool:
    return a.flags["C_CONTIGUOUS"] if isinstance(a, np.ndarray) else bool(a.is_contiguous())


def _check_buf(name: str, a, cells: int, dtype_code: Optional[int] = None):
    """The C ABI takes raw pointers: refuse a buffer whose size, dtype or layout
    does not match what the call will read/write (an out-of-bounds DMA otherwise)."""
    if not _contig(a):
        raise ContractError(f"{name}: buffer must be C-contiguous")
    if _numel(a) != cells:
        raise ContractError(f"{name}: buffer has {_numel(a)} cells, the call needs {cells}")
    if dtype_code is not None and _dtype_code(a) != dtype_code:
        raise ContractError(f"{name}: dtype differs from the other buffer")


class Engine:
    """One so2dr_ctx: a device, its streams, its HBM pool (capped by budget)."""

    def __init__(self, device: int = 0, budget_bytes: int = 0):
        L = lib()
        h = ctypes.c_void_p()
        _check(L.so2dr_ctx_create(device, budget_bytes, ctypes.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            lib().so2dr_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, st):
        if st != 0:
            _raise(st, self._h)

    def set_profiling(self, on: bool):
        self._ck(lib().so2dr_ctx_set_profiling(self._h, 1 if on else 0))

    def host_array(self, shape, dtype=np.float32) -> np.ndarray:
        """numpy array over pinned memory from so2dr_host_alloc (cudaHostAlloc); freed
        when the array is garbage-collected."""
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = ctypes.c_void_p()
        self._ck(lib().so2dr_host_alloc(self._h, nbytes, ctypes.byref(p)))
        buf = (ctypes.c_char * nbytes).from_address(p.value)
        arr = np.frombuffer(buf, dtype=dtype).reshape(shape)
        h, L = self._h, lib()
        import weakref

        weakref.finalize(buf, L.so2dr_host_free, h, p.value)
        return arr

    def host_register(self, arr):
        self._ck(lib().so2dr_host_register(self._h, _ptr(arr), arr.nbytes if isinstance(arr, np.ndarray)
                                           else arr.numel() * arr.element_size()))

    def host_unregister(self, arr):
        self._ck(lib().so2dr_host_unregister(self._h, _ptr(arr)))

    # -- run_engine (in place) -------------------------------------------
    def run(self, mode: str, grid, spec: StencilSpec, config: RunConfig,
            kernel: Optional[KernelPlan] = None, hw: Optional[HardwareModel] = None,
            hooks: Optional[EngineHooks] = None, diag: bool = True) -> RunReport:
        st, keep = spec._c()
        cfg = config._c()
        kp = (kernel or KernelPlan(k_on=config.k_on))._c()
        hwc = (hw or HardwareModel())._c()
        hk = _Hooks(1 if hooks and hooks.corrupt_share else 0, hooks.boundary if hooks else 0)
        led, tim = _Ledger(), _Timing()
        cap = 0
        rows = None
        n = ctypes.c_size_t(0)
        if diag:
            cap = 64 + 8 * max(1, config.d) * max(1, (config.n + max(config.s_tb, 1) - 1) // max(config.s_tb, 1))
            rows = (_Diag * cap)()
        _check_buf("engine: grid", grid, (config.sz + 2 * config.r) ** spec.dim)
        self._ck(lib().so2dr_run(self._h, MODES[mode], ctypes.byref(st), ctypes.byref(cfg),
                                 ctypes.byref(kp), ctypes.byref(hwc), ctypes.byref(hk),
                                 _dtype_code(grid), _ptr(grid), ctypes.byref(led), ctypes.byref(tim),
                                 rows, cap, ctypes.byref(n)))
        del keep
        dl = []
        if diag:
            for i in range(min(n.value, cap)):
                d = rows[i]
                dl.append({"round": d.round, "chunk": d.chunk, "stage": STAGES[d.stage],
                           "bytes": d.bytes, "updates": d.updates, "ms": d.ms, "t0_ms": d.t0_ms})
        return RunReport(mode, config, {f: getattr(led, f) for f in LEDGER_FIELDS},
                         {f: getattr(tim, f) for f, _ in TIMING_FIELDS}, dl)

    def run_spec(self, spec: "RunSpecFile", grid=None, hw: Optional[HardwareModel] = None, diag: bool = True):
        """The CLI's `run` (proj/tools/so2dr_main.cpp:146-162) for a parsed spec
        file / preset: init_grid(sz, r, seed) (unless `grid` is given), then
        run_engine in place. Returns (grid, RunReport)."""
        if grid is None:
            grid = self.init_grid(spec.config.sz, spec.config.r, spec.seed, spec.stencil.dim, spec.dtype)
        rep = self.run(spec.mode, grid, spec.stencil, spec.config, spec.kernel, hw, diag=diag)
        return grid, rep

    # -- secondary entry points -------------------------------------------
    def fused_kernel(self, spec: StencilSpec, buf0: np.ndarray, buf1: np.ndarray, base_row: int,
                     read: int, steps: int, tile: int, region, interior, owned) -> dict:
        st, keep = spec._c()
        rows, cols = buf0.shape
        _check_buf("fused_kernel: buf0", buf0, rows * cols)
        if _shape(buf1) != _shape(buf0):
            raise ContractError(f"fused_kernel: buf1 shape {_shape(buf1)} != buf0 shape {_shape(buf0)}")
        _check_buf("fused_kernel: buf1", buf1, rows * cols, _dtype_code(buf0))
        R = (ctypes.c_int32 * 4)(*region)
        I = (ctypes.c_int32 * 4)(*interior)
        O = (ctypes.c_int32 * 4)(*owned)
        out = (ctypes.c_uint64 * 4)()
        self._ck(lib().so2dr_fused_kernel(self._h, ctypes.byref(st), _dtype_code(buf0), _ptr(buf0),
                                          _ptr(buf1), base_row, rows, cols, read, steps, tile, R, I, O, out))
        del keep
        return {"scratch_load": out[0], "scratch_store": out[1], "updates": out[2], "redundant": out[3]}

    def apply_step(self, spec: StencilSpec, grid_in, grid_out, row_lo: int, row_hi: int):
        st, keep = spec._c()
        sz = grid_in.shape[0] - 2 * spec.radius
        _check_buf("apply_step: grid_in", grid_in, (sz + 2 * spec.radius) ** spec.dim)
        if _shape(grid_out) != _shape(grid_in):
            raise ContractError(f"apply_step: grid_out shape {_shape(grid_out)} != grid_in shape {_shape(grid_in)}")
        _check_buf("apply_step: grid_out", grid_out, _numel(grid_in), _dtype_code(grid_in))
        self._ck(lib().so2dr_apply_step(self._h, ctypes.byref(st), _dtype_code(grid_in), sz, spec.radius,
                                        _ptr(grid_in), _ptr(grid_out), row_lo, row_hi))
        del keep

    def run_reference(self, spec: StencilSpec, grid, steps: int):
        st, keep = spec._c()
        out = np.empty_like(grid)
        sz = grid.shape[0] - 2 * spec.radius
        _check_buf("run_reference: grid", grid, (sz + 2 * spec.radius) ** spec.dim)
        self._ck(lib().so2dr_run_reference(self._h, ctypes.byref(st), _dtype_code(grid), sz, spec.radius,
                                           _ptr(grid), _ptr(out), steps))
        del keep
        return out

    def init_grid(self, sz: int, r: int, seed: int, dim: int = 2, dtype=np.float32, out=None):
        if out is None:
            out = np.empty((sz + 2 * r,) * dim, dtype=dtype)
        self._ck(lib().so2dr_init_grid(self._h, _dtype_code(out), dim, sz, r, seed, _ptr(out)))
        return out

    def init_rows(self, sz: int, r: int, seed: int, lo: int, hi: int, out, dim: int = 2):
        self._ck(lib().so2dr_init_rows(self._h, _dtype_code(out), dim, sz, r, seed, lo, hi, _ptr(out)))
        return out

    # -- multi-rank slabs ---------------------------------------------------
    def slab_prepare(self, spec: StencilSpec, config: RunConfig, dtype, rank: int, world: int) -> bytes:
        st, keep = spec._c()
        cfg = config._c()
        blob = ctypes.create_string_buffer(PEER_BLOB_BYTES)
        code = 0 if np.dtype(dtype) == np.float32 else 1
        self._ck(lib().so2dr_slab_prepare(self._h, ctypes.byref(st), ctypes.byref(cfg), code, rank, world, blob))
        self._slab_rank = (rank, world)
        del keep
        return blob.raw

    def slab_connect(self, lower: Optional[bytes], upper: Optional[bytes]):
        self._ck(lib().so2dr_slab_connect(self._h, lower, upper))

    SLAB_TRANSPORTS = {0: "none", 1: "same-process", 2: "ipc-same-gpu", 3: "ipc-peer (p2p checked)",
                       4: "ipc-peer (not visible here)"}

    def slab_info(self) -> dict:
        """Rank, world and the halo transport of each slab edge after slab_connect."""
        out = (ctypes.c_int32 * 4)()
        self._ck(lib().so2dr_slab_info(self._h, out))
        return {"rank": out[0], "world": out[1], "lower": self.SLAB_TRANSPORTS[out[2]],
                "upper": self.SLAB_TRANSPORTS[out[3]]}

    def slab_run(self, spec: StencilSpec, config: RunConfig, slab, kernel: Optional[KernelPlan] = None):
        st, keep = spec._c()
        cfg = config._c()
        kp = (kernel or KernelPlan(k_on=config.k_on))._c()
        led, tim = _Ledger(), _Timing()
        rank, world = getattr(self, "_slab_rank", (0, 1))
        lo, hi = slab_rows(config, rank, world, dim=spec.dim)
        _check_buf("slab_run: slab", slab, (hi - lo) * (config.sz + 2 * config.r) ** (spec.dim - 1))
        self._ck(lib().so2dr_slab_run(self._h, ctypes.byref(st), ctypes.byref(cfg), ctypes.byref(kp),
                                      _dtype_code(slab), _ptr(slab), ctypes.byref(led), ctypes.byref(tim)))
        del keep
        return ({f: getattr(led, f) for f in LEDGER_FIELDS}, {f: getattr(tim, f) for f, _ in TIMING_FIELDS})


# -------------------------------------------------- host-only helpers --

def device_count() -> int:
    return int(lib().so2dr_device_count())


def grid_checksum(a) -> int:
    """FNV-1a 64 of the raw bytes (proj/src/stencil.cpp:176-186)."""
    a = np.ascontiguousarray(a)
    return int(lib().so2dr_grid_checksum(a.ctypes.data, a.nbytes))


def plan_chunks(config: RunConfig):
    """proj/src/layout.cpp:47-78 -> (fence, [dict(core, working, transfer, shared_in, shared_out)])."""
    fence = (ctypes.c_int32 * (config.d + 1))()
    ch = (ctypes.c_int32 * (10 * config.d))()
    _check(lib().so2dr_plan_chunks(ctypes.byref(config._c()), fence, ch))
    names = ("core", "working", "transfer", "shared_in", "shared_out")
    chunks = [{names[k]: (ch[10 * i + 2 * k], ch[10 * i + 2 * k + 1]) for k in range(5)} for i in range(config.d)]
    return list(fence), chunks


def slab_rows(config: RunConfig, rank: int, world: int, dim: int = 2):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().so2dr_slab_rows(ctypes.byref(config._c()), dim, rank, world, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def expected_ledger(mode: str, config: RunConfig, kernel: Optional[KernelPlan] = None, dim: int = 2,
                    dtype=np.float32) -> dict:
    out = (ctypes.c_uint64 * 6)()
    ex = ctypes.c_int32()
    kp = (kernel or KernelPlan(k_on=config.k_on))._c()
    code = 0 if np.dtype(dtype) == np.float32 else 1
    _check(lib().so2dr_expected_ledger(MODES[mode], ctypes.byref(config._c()), ctypes.byref(kp), dim, code,
                                       out, ctypes.byref(ex)))
    keys = ("htod", "dtoh", "ondevice", "kernel_invocations", "rounds", "redundant_updates")
    d = dict(zip(keys, list(out)))
    d["redundancy_exact"] = bool(ex.value)
    return d


def kernel_stats(radius: int, steps: int, tile: int, region, interior, owned, sy0: int, sy1: int,
                 cols: int) -> dict:
    """The reference's fused_kernel accounting (kernels.cpp:48-138), closed form, host only."""
    out = (ctypes.c_uint64 * 4)()
    a = lambda v: (ctypes.c_int32 * 4)(*v)  # noqa: E731
    _check(lib().so2dr_kernel_stats(radius, steps, tile, a(region), a(interior), a(owned), sy0, sy1, cols, out))
    return {"scratch_load": out[0], "scratch_store": out[1], "updates": out[2], "redundant": out[3]}


def arena_bytes(config: RunConfig, kernel: KernelPlan) -> int:
    out = ctypes.c_uint64()
    _check(lib().so2dr_arena_bytes(ctypes.byref(config._c()), ctypes.byref(kernel._c()), ctypes.byref(out)))
    return out.value


class _PlanEntry(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("s_tb", ctypes.c_int32), ("k_on", ctypes.c_int32),
                ("n_strm", ctypes.c_int32), ("feasible", ctypes.c_int32), ("launches", ctypes.c_int64),
                ("device_bytes", ctypes.c_uint64), ("t_pcie_s", ctypes.c_double), ("t_kernel_s", ctypes.c_double),
                ("t_fill_s", ctypes.c_double), ("t_total_s", ctypes.c_double), ("gcell_per_s", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _plan_args(profile, dim, dtype, kind, radius):
    prof = None if profile is None else (profile if isinstance(profile, str) else json.dumps(profile)).encode()
    code = 0 if np.dtype(dtype) == np.float32 else 1
    return prof, dim, code, 1 if kind == STAR else 0, radius


def plan_b200(sz: int, n: int, radius: int = 1, kind: int = BOX, dim: int = 2, dtype=np.float32,
              budget_bytes: int = 0, n_strm: int = 3, profile=None, all_candidates: bool = False):
    """B200 planner (include/so2dr/b200.hpp): the fastest feasible (d, S_TB, k_on)
    for an so2dr run, priced from profiles/b200.json (profile=None: built-in copy;
    a JSON string or dict overrides)."""
    prof, dim, code, star, radius = _plan_args(profile, dim, dtype, kind, radius)
    best = _PlanEntry()
    count = ctypes.c_int32()
    _check(lib().so2dr_plan_b200(prof, dim, code, star, radius, sz, n, ctypes.c_uint64(budget_bytes), n_strm,
                                 ctypes.byref(best), None, 0, ctypes.byref(count)))
    if not all_candidates:
        return best.as_dict()
    arr = (_PlanEntry * count.value)()
    _check(lib().so2dr_plan_b200(prof, dim, code, star, radius, sz, n, ctypes.c_uint64(budget_bytes), n_strm,
                                 ctypes.byref(best), arr, count.value, ctypes.byref(count)))
    return best.as_dict(), [e.as_dict() for e in arr]


def predict_b200(sz: int, n: int, d: int, s_tb: int, k_on: int, radius: int = 1, kind: int = BOX, dim: int = 2,
                 dtype=np.float32, budget_bytes: int = 0, n_strm: int = 3, profile=None) -> dict:
    """The B200 planner's prediction for one configuration."""
    prof, dim, code, star, radius = _plan_args(profile, dim, dtype, kind, radius)
    out = _PlanEntry()
    _check(lib().so2dr_predict_b200(prof, dim, code, star, radius, sz, n, ctypes.c_uint64(budget_bytes), d, s_tb,
                                    k_on, n_strm, ctypes.byref(out)))
    return out.as_dict()


def device_numa_node(device: int = 0) -> int:
    """NUMA node of a GPU (sysfs), -1 if unknown."""
    return int(lib().so2dr_device_numa_node(device))


def pci_numa_node(pci_bus_id: str, sysfs_root: str = "") -> int:
    """The sysfs lookup behind device_numa_node (host logic, no GPU needed)."""
    return int(lib().so2dr_pci_numa_node(sysfs_root.encode(), pci_bus_id.encode()))


def k1_max_steps(dim: int, dtype, kind: int, radius: int) -> int:
    """Largest step count one K1 launch fuses (longer calls are split); 0 = unsupported."""
    code = 0 if np.dtype(dtype) == np.float32 else 1
    return int(lib().so2dr_k1_max_steps(dim, code, kind, radius))


def device_bytes(config: RunConfig, dim: int = 2, dtype=np.float32) -> int:
    out = ctypes.c_uint64()
    code = 0 if np.dtype(dtype) == np.float32 else 1
    _check(lib().so2dr_device_bytes(ctypes.byref(config._c()), dim, code, ctypes.byref(out)))
    return out.value


_default_engine: Optional[Engine] = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine(0)
    return _default_engine


def run_engine(mode: str, grid, spec: StencilSpec, config: RunConfig, kernel: Optional[KernelPlan] = None,
               hw: Optional[HardwareModel] = None, hooks: Optional[EngineHooks] = None):
    """proj/include/so2dr/engine.hpp:79-81: returns (result grid, report); input untouched."""
    out = np.array(grid, copy=True)
    rep = default_engine().run(mode, out, spec, config, kernel, hw, hooks)
    rep.checksum = grid_checksum(out)
    return out, rep


# ------------------------------------ spec files, presets, run outputs --
# proj/include/so2dr/specfile.hpp:14-28, proj/tools/so2dr_main.cpp:28-68,
# proj/include/so2dr/report.hpp:11-24 (through the C ABI: one implementation)

@dataclasses.dataclass
class RunSpecFile:
    """A parsed spec file / preset (RunSpecFile, specfile.hpp:14-23, plus the
    dim/dtype/weights extensions)."""
    stencil: StencilSpec
    seed: int
    mode: str
    config: RunConfig
    kernel: KernelPlan
    dtype: type
    stencil_name: str
    hardware_path: Optional[str] = None
    grid_dump_path: Optional[str] = None


def _from_c_spec(c: "_Spec") -> RunSpecFile:
    st = c.stencil
    n = (2 * st.radius + 1) ** st.dim
    w = np.array(c.weights_buf[:n], dtype=np.float64)
    cfg = RunConfig(**{f: getattr(c.config, f) for f in ("sz", "r", "d", "s_tb", "k_on", "n_strm", "n", "n_a")})
    mode = {v: k for k, v in MODES.items()}[c.mode]
    return RunSpecFile(StencilSpec(st.kind, st.radius, st.dim, w), int(c.seed), mode, cfg,
                       KernelPlan(c.kernel.k_on, c.kernel.tile, c.kernel.scratch_budget),
                       np.float64 if c.dtype == 1 else np.float32, c.stencil_name.decode(),
                       c.hardware_path.decode() or None, c.grid_dump_path.decode() or None)


def parse_spec_json(text: str, origin: str = "spec") -> RunSpecFile:
    c = _Spec()
    _check(lib().so2dr_spec_parse(text.encode(), origin.encode(), ctypes.byref(c)))
    return _from_c_spec(c)


def parse_spec_file(path: str) -> RunSpecFile:
    c = _Spec()
    _check(lib().so2dr_spec_parse_file(str(path).encode(), ctypes.byref(c)))
    return _from_c_spec(c)


def preset_names() -> list:
    L = lib()
    return [L.so2dr_preset_name(i).decode() for i in range(L.so2dr_preset_count())]


def _text(fn, *args) -> str:
    n = ctypes.c_size_t(0)
    _check(fn(*args, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, n.value + 1, ctypes.byref(n)))
    return buf.value.decode()


def preset_json(name: str) -> str:
    return _text(lib().so2dr_preset_json, name.encode())


def preset(name: str) -> RunSpecFile:
    """--preset NAME: the preset's JSON through parse_spec_json (origin "preset NAME")."""
    return parse_spec_json(preset_json(name), "preset " + name)


def report_to_json(report: "RunReport", stencil_name: str, checksum: int, deterministic: bool = False,
                   hw: Optional[HardwareModel] = None, kernel: Optional[KernelPlan] = None) -> str:
    """report.json v1 (proj/src/report.cpp:21-64) of an Engine.run report."""
    led = _Ledger(*[report.ledger[f] for f in LEDGER_FIELDS])
    tim = _Timing(*[report.timing[f] for f, _ in TIMING_FIELDS])
    hwc = (hw or HardwareModel())._c()
    ri = _ReportIn(MODES[report.mode], 1 if deterministic else 0, stencil_name.encode(), report.config._c(),
                   (kernel or KernelPlan(k_on=report.config.k_on))._c(), checksum, led, ctypes.pointer(hwc),
                   ctypes.pointer(tim))
    return _text(lib().so2dr_report_json, ctypes.byref(ri))


def ledger_to_csv(ledger: dict) -> str:
    led = _Ledger(*[ledger[f] for f in LEDGER_FIELDS])
    return _text(lib().so2dr_ledger_csv, ctypes.byref(led))


def diagnostics_to_csv(rows: list) -> str:
    arr = (_Diag * max(1, len(rows)))()
    for i, r in enumerate(rows):
        arr[i].round, arr[i].chunk, arr[i].stage = r["round"], r["chunk"], STAGES.index(r["stage"])
        arr[i].bytes, arr[i].updates = r["bytes"], r["updates"]
    return _text(lib().so2dr_diagnostics_csv, arr, len(rows))
