#!/usr/bin/env python
"""SO2DR B200 benchmark -- BASELINE.json metric:
"GCell-updates/s end-to-end (incl. H2D/D2H) at 1/2/4/8 B200; % of roofline".

Workload (BASELINE configs[1]): box2d1r fp32 out-of-core, grid ~2x the device
budget on one B200, 64 timesteps: sz=92160 (92162^2 fp32 = 33.98 GB host grid),
16 GiB real HBM budget, d=64 chunks, S_TB=64 (one round), k_on=4, N_strm=3.
A "step" is one full so2dr run (64 timesteps over the whole grid).

  value, e2e : the BASELINE metric -- C-ABI so2dr_run on the pinned HOST grid,
          all PCIe traffic inside the timed region (CUDA events, first H2D ->
          last D2H); `value` == `e2e.value`
  hbm_resident : the same run with the grid already resident in HBM (the
          transfers become D2D copies) -- explains the kernel side, not the metric

Multi-GPU (torchrun): the d chunks are slab-partitioned over ranks (weak scaling:
each rank streams a ~34 GB slab of a sz~92160*sqrt(N) grid); inter-slab halos
move GPU-to-GPU over CUDA IPC peer memory. --impl reference times the
reference CPU solver (oracle/_ref, built from /root/reference) on a bounded
sample of the same workload.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
os.environ.setdefault("OMP_PROC_BIND", "spread")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

METRIC = "GCell-updates/s end-to-end (incl. H2D/D2H) at 1/2/4/8 B200; % of roofline"
UNIT = "GCell/s"
# d=64 chunks (not SURVEY's worked-example 16): 4x shorter pipeline fill/drain
# (first H2D + first chunk's kernels, last D2H) -- 780 vs 832 ms per run on
# this box (profiles/r01_pcie); k_on=4: K1 then binds on HBM (2b/k_on = 2 B per
# update => 3.3 TCell/s HBM roof < 3.5 TCell/s FMA roof), and e2e is unchanged
# vs k_on=8 (the kernel is hidden behind PCIe either way).
SZ1, D_PER_RANK, S_TB, K_ON, NSTEPS, NSTRM, R = 92160, 64, 64, 4, 64, 3, 1
FMA_PEAK = 36.88e12  # measured FFMA2 peak on this pool's B200 (profiles/r01_pcie/fma_peak.jsonl)
TAPS = 9  # box2d1r
BUDGET = 16 << 30


def host_numa_nodes() -> int:
    n = 0
    while os.path.isdir(f"/sys/devices/system/node/node{n}"):
        n += 1
    return n


def host_copy_gbps(torch, mib: int = 2048) -> float:
    """Host DRAM copy bandwidth (read + write bytes), best of 3: numpy copies of
    one slice per host thread (they release the GIL), so all cores stream."""
    from concurrent.futures import ThreadPoolExecutor

    n = os.cpu_count() or 1
    a = np.ones(mib << 18, dtype=np.float32)
    b = np.empty_like(a)
    step = (a.size + n - 1) // n
    bounds = [(i, min(i + step, a.size)) for i in range(0, a.size, step)]
    best = 0.0
    with ThreadPoolExecutor(n) as ex:
        for _ in range(3):
            t0 = time.perf_counter()
            list(ex.map(lambda r: np.copyto(b[r[0]:r[1]], a[r[0]:r[1]]), bounds))
            dt = time.perf_counter() - t0
            best = max(best, 2 * a.nbytes / dt / 1e9)
    return best


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def geometry(world: int, d_per_rank: int = D_PER_RANK):
    d = d_per_rank * world
    sz = SZ1 if world == 1 else int(round(SZ1 * math.sqrt(world) / d)) * d
    return sz, d


def workload_desc(world, sz, d, k_on=K_ON):
    gb = (sz + 2 * R) ** 2 * 4 / 1e9
    return (f"box2d1r fp32 out-of-core, sz={sz} ({gb:.2f} GB grid, {gb / world / (BUDGET / 1e9):.2f}x the "
            f"{BUDGET >> 30} GiB per-GPU HBM budget), n={NSTEPS} timesteps, d={d}, S_TB={S_TB}, k_on={k_on}, "
            f"N_strm={NSTRM}, slab-partitioned over {world} GPU(s)")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int, period_ms: int = 200):
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def pcie_probe(torch, dev, eng=None):
    """Pinned-host PCIe GB/s on this box, timed with CUDA events on the copy
    streams: H2D alone, D2H alone, and both at once (2 GiB each way, as 8 copies
    of 256 MiB per direction, best of 3). In duplex the host side caps the
    COMBINED rate (~94 GB/s here, tools/pcie_probe.py), so duplex_GBps_per_dir =
    combined / 2 is what a balanced pipeline can use. The host buffers come from
    the engine's own allocator (so2dr_host_alloc, as the bench grid) when torch
    sees them as pinned, else from torch's pinned allocator (the line says which)."""
    n = 2 << 30
    pieces = 8
    src = "torch pin_memory"
    h = h2 = None
    if eng is not None:
        try:
            ha = torch.from_numpy(eng.host_array((n,), np.uint8))
            hb = torch.from_numpy(eng.host_array((n,), np.uint8))
            if ha.is_pinned() and hb.is_pinned():
                h, h2, src = ha, hb, "so2dr_host_alloc"
        except Exception:  # noqa: BLE001 - fall back to torch's pinned memory
            h = h2 = None
    if h is None:
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    out = {}
    step = n // pieces
    for name in ("h2d", "d2h", "duplex"):
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_event(e0)
            s2.wait_event(e0)
            for i in range(pieces):
                sl = slice(i * step, (i + 1) * step)
                if name in ("h2d", "duplex"):
                    with torch.cuda.stream(s1):
                        d[sl].copy_(h[sl], non_blocking=True)
                if name in ("d2h", "duplex"):
                    with torch.cuda.stream(s2):
                        h2[sl].copy_(d2[sl], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize(dev)
            moved = n * (2 if name == "duplex" else 1)
            best = max(best, moved / e0.elapsed_time(e1) / 1e6)
        out[name + ("_combined_GBps" if name == "duplex" else "_GBps")] = round(best, 2)
    out["duplex_GBps_per_dir"] = round(out["duplex_combined_GBps"] / 2, 2)
    out["host_buffers"] = src
    del h, h2, d, d2
    return out


def _ref_engine_sample(sz):
    """One reference run_engine(so2dr) call (oracle/_ref: the unmodified reference
    sources, -O3 -ffp-contract=off -fopenmp) on a box2d1r grid of side sz with the
    bench's d, S_TB, k_on, n. Returns (GCell/s from RunReport.wall_seconds, s)."""
    import ctypes

    import pyoracle as o

    R_ = o.ref()
    d = D_PER_RANK
    g = np.empty((sz + 2 * R, sz + 2 * R), np.float32)
    R_.ref_init_grid(sz, R, 42, g.ctypes.data)
    out = np.empty_like(g)
    led = (ctypes.c_uint64 * 9)()
    peak, wall = ctypes.c_uint64(), ctypes.c_double()
    err = ctypes.create_string_buffer(256)
    t0 = time.perf_counter()
    rc = R_.ref_run_engine(0, 0, R, None, (ctypes.c_int * 8)(sz, R, d, S_TB, K_ON, NSTRM, NSTEPS, 2),
                           (ctypes.c_int * 2)(K_ON, 32), 64 << 20, 1 << 40, 760e9, 15.75e9, 0, 0,
                           g.ctypes.data, out.ctypes.data, led, ctypes.byref(peak), ctypes.byref(wall), err, 256)
    t = time.perf_counter() - t0
    if rc != 0:
        raise RuntimeError(err.value.decode())
    sec = wall.value if wall.value > 0 else t
    return sz * sz * NSTEPS / sec / 1e9, sec


def _ref_serial_sample():
    """The reference's serial oracle run_reference (stencil.cpp:162-174, one core):
    box2d1r sz=8192, 16 steps (1.07 G updates)."""
    import ctypes

    import pyoracle as o

    R_ = o.ref()
    sz, n = 8192, 16
    g = np.empty((sz + 2 * R, sz + 2 * R), np.float32)
    R_.ref_init_grid(sz, R, 42, g.ctypes.data)
    out = np.empty_like(g)
    err = ctypes.create_string_buffer(256)
    t0 = time.perf_counter()
    rc = R_.ref_run_reference(0, R, None, sz, R, g.ctypes.data, n, out.ctypes.data, err, 256)
    sec = time.perf_counter() - t0
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return {"value": sz * sz * n / sec / 1e9, "unit": UNIT, "cores": 1,
            "sample": f"reference run_reference (serial ping-pong oracle) box2d1r sz={sz} n={n} in {sec:.2f} s"}


def _ref_desc():
    import pyoracle as o

    bi = o.ref_build_info()
    s = f"-O3 -march={bi['march']} -ffp-contract=off -fopenmp"
    if bi.get("missing_isa"):
        s += f" (the -march={bi.get('native_march')} build needs {','.join(bi['missing_isa'][:4])}... absent here)"
    return s


def cpu_baseline_sample():
    """The reference's own CPU solver on a bounded sample of the workload: same
    stencil, d, S_TB, k_on, n; sz reduced 3x (1/9 of the cells, ~10 s on 16
    host threads)."""
    import pyoracle as o

    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    if o.have_ref():
        sz = SZ1 // 3
        v, sec = _ref_engine_sample(sz)
        return {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"reference run_engine(so2dr) box2d1r sz={sz} d={D_PER_RANK} S_TB={S_TB} k_on={K_ON} "
                          f"n={NSTEPS} ({(sz + 2 * R) ** 2 * 4 / 1e9:.2f} GB grid, {sz * sz * NSTEPS / 1e9:.1f} G "
                          f"updates) in {sec:.2f} s; RunReport.wall_seconds, OMP_NUM_THREADS={cores}, "
                          f"3 std::thread workers; built {_ref_desc()}",
                "seconds": sec}
    # fallback: the C restatement (serial)
    g = o.init_grid(SZ1 // 12, R, 42)
    t0 = time.perf_counter()
    o.run(g, o.BOX, R, o.box_weights(R), 4)
    sec = time.perf_counter() - t0
    s4 = SZ1 // 12
    return {"value": s4 * s4 * 4 / sec / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle port (serial C) box2d1r sz={s4} n=4 in {sec:.2f} s", "seconds": sec}


def run_reference_arm(args):
    """--impl reference: the reference's own CPU solver (run_engine(so2dr), all
    host cores) on the bench's config. The full 34 GB grid would take ~5 min per
    step, so each timed step is a bounded sample of the same workload: steps
    alternate sz/3 (3.8 GB) and sz/2 (8.5 GB) grids with the same d, S_TB, k_on, n,
    so the line shows GCell/s does not depend on the grid size (value = median
    over all timed steps; per-size medians in cpu_baseline.by_size). Warm-up steps
    run a sz/6 grid. The serial run_reference oracle is timed once beside it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # torchrun exports OMP_NUM_THREADS=1 to every rank; the reference CPU solver on
    # rank 0 gets all host cores (set before libgomp is loaded with oracle/_ref)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    import pyoracle as o

    cores = int(os.environ["OMP_NUM_THREADS"])
    if not o.have_ref():
        cb = cpu_baseline_sample()
        samples = [(0, cb["value"], cb["seconds"])]
        by_size = {}
        sample_desc = cb["sample"]
        kind = "port"
    else:
        for _ in range(args.warmup):
            _ref_engine_sample(SZ1 // 6)
        samples = []
        for i in range(args.steps):
            sz = SZ1 // 3 if i % 2 == 0 else SZ1 // 2
            v, sec = _ref_engine_sample(sz)
            samples.append((sz, v, sec))
        by_size = {}
        for sz in sorted({s[0] for s in samples}):
            vs = [s[1] for s in samples if s[0] == sz]
            by_size[f"sz={sz}"] = {"GCell_s_median": statistics.median(vs), "samples": len(vs),
                                   "grid_GB": (sz + 2 * R) ** 2 * 4 / 1e9}
        sample_desc = (f"reference run_engine(so2dr) box2d1r, same d={D_PER_RANK} S_TB={S_TB} k_on={K_ON} "
                       f"n={NSTEPS}; timed steps alternate sz={SZ1 // 3} and sz={SZ1 // 2} (the 34 GB sz={SZ1} "
                       f"grid would take ~5 min per step); RunReport.wall_seconds, OMP_NUM_THREADS={cores}, "
                       f"3 std::thread workers; built {_ref_desc()}")
        kind = "reference"
    v = statistics.median([s[1] for s in samples])
    try:
        serial = _ref_serial_sample() if o.have_ref() else None
    except Exception as e:  # never fail the line on the serial column
        serial = {"value": None, "sample": f"failed: {e}"}
    cb = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample_desc, "by_size": by_size,
          "serial_run_reference": serial}
    sz, d = geometry(1)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(s[2] for s in samples),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (splitmix64 init_grid, seed 42)",
            "config": {"workload": workload_desc(1, sz, d) + "; reference CPU solver timed on bounded samples "
                       "(sz/3 and sz/2, same d/S_TB/k_on/n)"},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--k-on", type=int, default=K_ON)
    ap.add_argument("--d", type=int, default=D_PER_RANK, help="chunks per rank")
    ap.add_argument("--plan", action="store_true",
                    help="take d and k_on from the B200 planner (include/so2dr/b200.hpp) instead of --d/--k-on")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hbm-leg", "--no-value-leg", dest="no_hbm_leg", action="store_true")
    ap.add_argument("--pcie-probe-before", action="store_true",
                    help="measure the PCIe roof before the timed e2e leg (default: right after it; the torch "
                         "probe's pinned buffers cost the e2e leg ~1.5%% when taken before)")
    ap.add_argument("--clock-ms", type=int, default=200, help="nvidia-smi sampling period during the timed e2e leg")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2309_08864_b200 as so2dr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl" if os.environ.get("SO2DR_SHARE_DEVICE") != "1" else "gloo")
    ndev = torch.cuda.device_count()
    dev_index = 0 if os.environ.get("SO2DR_SHARE_DEVICE") == "1" else local % max(ndev, 1)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)

    k_on = args.k_on
    sz, d = geometry(world, args.d)
    # B200 planner (profiles/b200.json): its choice for this workload and its
    # prediction for the configuration actually run
    try:
        prof = open(os.path.join(ROOT, "profiles", "b200.json")).read()
    except OSError:
        prof = None
    pick = so2dr.plan_b200(sz, NSTEPS, R, so2dr.BOX, budget_bytes=BUDGET, n_strm=NSTRM, profile=prof)
    if args.plan:
        k_on = pick["k_on"]
        sz, d = geometry(world, pick["d"])
    pred = so2dr.predict_b200(sz, NSTEPS, d // world, S_TB, k_on, R, so2dr.BOX, budget_bytes=BUDGET,
                              n_strm=NSTRM, profile=prof) if world == 1 else None
    cfg = so2dr.RunConfig(sz=sz, r=R, d=d, s_tb=S_TB, k_on=k_on, n_strm=NSTRM, n=NSTEPS)
    spec = so2dr.StencilSpec.box(R)
    kp = so2dr.KernelPlan(k_on, 32, 64 << 20)
    eng = so2dr.Engine(dev_index, BUDGET)
    lo, hi = so2dr.slab_rows(cfg, rank, world)
    p = sz + 2 * R
    shape = (hi - lo, p)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def connect():
        if world == 1:
            return
        blob = eng.slab_prepare(spec, cfg, np.float32, rank, world)
        blobs = [None] * world
        dist.all_gather_object(blobs, blob)
        eng.slab_connect(blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank < world - 1 else None)

    def run_once(grid):
        if world == 1:
            rep = eng.run("so2dr", grid, spec, cfg, kp, diag=False)
            return rep.timing, rep.ledger
        led, tim = eng.slab_run(spec, cfg, grid, kp)
        return tim, led

    def leg(grid, steps, warmup):
        for _ in range(warmup):
            run_once(grid)
        barrier()
        times, kms, kmax, launches, algb, h2d, d2h = [], 0.0, 0.0, 0, 0, 0, 0
        t0 = time.perf_counter()
        for _ in range(steps):
            tim, led = run_once(grid)
            times.append(tim["device_ms"])
            kms += tim["kernel_ms"]
            kmax = max(kmax, tim["kernel_max_ms"])
            launches += tim["kernel_launches"]
            algb += tim["kernel_alg_bytes"]
            h2d += tim["h2d_bytes"]
            d2h += tim["d2h_bytes"]
        barrier()
        wall = time.perf_counter() - t0
        dev_ms = allmax(sum(times))
        return {"device_ms_total": dev_ms, "wall_s": allmax(wall), "kernel_ms": kms, "kernel_max_ms": kmax,
                "launches": launches, "alg_bytes": algb, "h2d": h2d, "d2h": d2h, "per_step_ms": times,
                "rank_ms": sum(times)}

    total_updates = sz * sz * NSTEPS  # per step, whole job

    # ---- value leg: grid resident in HBM ---------------------------------
    value_res = None
    if not args.no_hbm_leg:
        gdev = torch.empty(shape, dtype=torch.float32, device=dev)
        eng.init_rows(sz, R, 42, lo, hi, gdev)
        connect()
        value_res = leg(gdev, args.steps, args.warmup)
        del gdev
        torch.cuda.empty_cache()

    # ---- e2e leg: pinned host grid through the C ABI ------------------------
    # pinned host grid from so2dr_host_alloc (cudaHostAlloc): 4 KiB-page
    # registered malloc memory only sustains ~43 GB/s per direction in duplex
    t0 = time.perf_counter()
    host = eng.host_array(shape, np.float32)
    t_reg = time.perf_counter() - t0
    eng.init_rows(sz, R, 42, lo, hi, host)
    connect()
    pc = pcie_probe(torch, dev, eng) if rank == 0 and args.pcie_probe_before else {}
    with ClockSampler(dev_index, args.clock_ms) as clk:
        e2e_res = leg(host, args.steps, args.warmup)
    clocks = clk.summary()
    if rank == 0 and not args.pcie_probe_before:
        pc = pcie_probe(torch, dev, eng)
    # multi-GPU evidence: every rank's own e2e time, its GPU's NUMA node and the
    # halo transport of its slab edges (all ranks take part in the gather)
    mine = {"rank": rank, "device_ms": e2e_res["rank_ms"], "numa_node": so2dr.device_numa_node(dev_index),
            "transport": eng.slab_info() if world > 1 else None}
    ranks = [mine]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    peak_src = ("MEASURED_PEAKS.json hbm_gbs (of measured copy)" if "hbm_gbs" in pk else
                "of fallback: 6650 GB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)")
    e2e_v = total_updates * args.steps / (e2e_res["device_ms_total"] / 1e3) / 1e9
    val_v = (total_updates * args.steps / (value_res["device_ms_total"] / 1e3) / 1e9) if value_res else None
    # K1 roofline: algorithmic bytes (input rows read once + output rows written once per launch)
    kr = e2e_res
    k_gbs = kr["alg_bytes"] / (kr["kernel_ms"] / 1e3) / 1e9 if kr["kernel_ms"] > 0 else 0.0
    per_launch = kr["alg_bytes"] / max(kr["launches"], 1)
    traffic, traffic_src = None, None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "k1_traffic.json")))
        if prof.get("k_on") == k_on and prof.get("d") == d:
            # ncu DRAM bytes per launch over a steady-state window, scaled to this run's
            # average launch by the window's measured traffic/algorithmic ratio
            traffic = per_launch * prof["dram_over_alg"]
            traffic_src = prof.get("source")
    except Exception:
        pass
    k_fma = total_updates * args.steps * TAPS / (kr["kernel_ms"] / 1e3) if kr["kernel_ms"] > 0 else 0.0
    bw_dir = pc.get("duplex_GBps_per_dir", 50.0)
    r_pcie = world * bw_dir * 1e9 * S_TB / 4 / 1e9
    r_hbm = world * hbm * 1e9 / (2 * 4 / k_on + 2 * 4 / S_TB) / 1e9
    r_bind = min(r_pcie, r_hbm)
    r_host = host_copy_gbps(torch)
    cb = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline_sample()
            cb.pop("seconds", None)
        except Exception as e:  # never fail the GPU line on the baseline
            cb = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference", "sample": f"failed: {e}"}
    line = {
        "metric": METRIC, "value": e2e_v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": e2e_res["device_ms_total"] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (splitmix64 init_grid, seed 42; grid generated on device)",
        "config": {"workload": workload_desc(world, sz, d, k_on), "sz": sz, "d": d, "s_tb": S_TB, "k_on": k_on,
                   "n": NSTEPS, "n_strm": NSTRM, "budget_bytes_per_gpu": BUDGET,
                   "grid_bytes": (sz + 2 * R) ** 2 * 4,
                   "l2": "no flush needed: every step streams the whole grid (>= 34 GB >> 126 MB L2)",
                   "value": "e2e: pinned host grid through the C ABI, H2D/D2H inside the timed region",
                   "timing": "CUDA events on the engine streams, first H2D enqueue -> last D2H completion, "
                             "summed over steps, max over ranks"},
        "hbm_resident": ({"value": val_v, "unit": UNIT,
                          "ms_per_step": value_res["device_ms_total"] / args.steps,
                          "note": "same so2dr run with the grid resident in HBM (transfers become D2D); "
                                  "not the BASELINE metric"} if value_res else None),
        "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": e2e_res["h2d"] // args.steps,
                "d2h_bytes_per_step": e2e_res["d2h"] // args.steps,
                "wall_s_per_step": e2e_res["wall_s"] / args.steps,
                "rank0_device_ms_per_step": [round(t, 2) for t in e2e_res["per_step_ms"]]},
        "roofline": {"bound": "hbm", "kernel": "K1 k1_stencil2d<float,1,%d,box>" % k_on, "achieved": k_gbs,
                     "peak": hbm, "unit": "GB/s", "frac": k_gbs / hbm, "traffic": traffic,
                     "alg_bytes_per_launch": per_launch,
                     "avg_launch_ms": kr["kernel_ms"] / max(kr["launches"], 1),
                     "kernel_share_of_step": kr["kernel_ms"] / max(e2e_res["device_ms_total"], 1e-9),
                     "peak_source": peak_src, "traffic_source": traffic_src,
                     "timing": "CUDA events bracketing every K1 launch on its own (compute) stream",
                     "fma": {"achieved_TFMAps": k_fma / 1e12, "peak_TFMAps": FMA_PEAK / 1e12,
                             "frac": k_fma / FMA_PEAK,
                             "note": "useful (non-redundant) FMAs: sz^2 * n * 9 per step; peak = measured FFMA2 "
                                     "rate (profiles/r01_pcie/fma_peak.jsonl)"}},
        "binding_roofline": {"R_pcie": r_pcie, "R_hbm": r_hbm, "R_bind": r_bind, "unit": UNIT,
                             "frac_e2e": e2e_v / r_bind, "frac_hbm_resident_vs_R_hbm": (val_v / r_hbm) if val_v else None,
                             "pcie_measured": pc,
                             "pcie_achieved_GBps_per_dir": {
                                 "h2d": e2e_res["h2d"] / (e2e_res["device_ms_total"] / 1e3) / 1e9,
                                 "d2h": e2e_res["d2h"] / (e2e_res["device_ms_total"] / 1e3) / 1e9,
                                 "note": "ledger bytes / e2e device time (includes pipeline fill and drain)"},
                             "formula": "R_pcie = G*BW_pcie_dir(duplex)*S_TB/b ; R_hbm = G*BW_hbm/(2b/k_on + 2b/S_TB)"},
        "planner": {"choice": {k: pick[k] for k in ("d", "s_tb", "k_on", "n_strm", "t_total_s", "gcell_per_s")},
                    "predicted_for_this_config": ({k: pred[k] for k in ("t_total_s", "t_pcie_s", "t_kernel_s",
                                                                          "t_fill_s", "gcell_per_s")}
                                                  if pred else None),
                    "source": "so2dr_plan_b200 over (d | sz, S_TB | n, k_on <= 8), profiles/b200.json",
                    "used": bool(args.plan)},
        "multi_gpu": {
            "per_rank": [{"rank": q["rank"], "e2e_GCell_s": total_updates / world * args.steps /
                          (q["device_ms"] / 1e3) / 1e9, "numa_node": q["numa_node"], "transport": q["transport"]}
                         for q in ranks],
            "host_numa_nodes": host_numa_nodes(),
            "R_host_copy_GBps": r_host,
            "R_host_note": "host DRAM copy bandwidth (read+write bytes, torch CPU copy, all threads); N ranks "
                           "stream 2 x BW_pcie_dir each, so host DRAM binds before PCIe once "
                           "N * 2 * BW_pcie_dir > R_host (SURVEY 7 hard part 7)",
            "halo_path": "CUDA IPC peer memory + stream memory operations (so2dr_slab_*), no NCCL on the data path"},
        "cpu_baseline": cb,
        "clocks": clocks,
        "gpu_launches": e2e_res["launches"],
        "host_register_s": t_reg,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
