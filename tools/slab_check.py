"""Multi-rank slab run, checked against the CPU oracle.

Launched as N processes (torchrun or tests/test_gpu_multirank.py); every rank
owns d/N chunks of the grid, exchanges its edge bands GPU-to-GPU through CUDA
IPC (so2dr_slab_*), and rank 0 reassembles the grid and compares it
bit-for-bit with the oracle. SO2DR_SHARE_DEVICE=1 puts every rank on cuda:0
(the multi-rank protocol on a single B200)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = 0 if os.environ.get("SO2DR_SHARE_DEVICE") == "1" else int(os.environ.get("LOCAL_RANK", rank))
    kind = os.environ.get("SLAB_KIND", "box")
    dim = int(os.environ.get("SLAB_DIM", "2"))
    dtype = np.float64 if os.environ.get("SLAB_DTYPE") == "f64" else np.float32
    sz = int(os.environ.get("SLAB_SZ", "256" if dim == 2 else "48"))
    r = 1
    cfg = so2dr.RunConfig(sz=sz, r=r, d=4 * world, s_tb=int(os.environ.get("SLAB_STB", "4")),
                          k_on=int(os.environ.get("SLAB_KON", "4")), n_strm=3, n=int(os.environ.get("SLAB_N", "10")))
    import pyoracle as o

    if kind == "star":
        w = o.star_weights(r, dim, dtype)
    else:
        w = o.box_weights(r, dim, dtype)
    spec = so2dr.StencilSpec(so2dr.BOX, r, dim, w)
    eng = so2dr.Engine(dev)
    lo, hi = so2dr.slab_rows(cfg, rank, world, dim)
    full = o.init_grid(sz, r, 42, dim, dtype)
    slab = full[lo:hi].copy()  # a view would let the engine advance `full` itself
    blob = eng.slab_prepare(spec, cfg, dtype, rank, world)
    blobs = [None] * world
    dist.all_gather_object(blobs, blob)
    eng.slab_connect(blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank < world - 1 else None)
    reps = int(os.environ.get("SLAB_REPS", "2"))
    want = full
    for _ in range(reps):  # repeated runs reuse the connection (epochs continue)
        led, tim = eng.slab_run(spec, cfg, slab)
        want = o.run(want, o.BOX, r, w, cfg.n) if rank == 0 else None
    parts = [None] * world
    dist.all_gather_object(parts, (lo, hi, slab.tobytes(), led))
    if rank == 0:
        got = np.empty_like(full)
        htod = 0
        for plo, phi, b, pled in parts:
            got[plo:phi] = np.frombuffer(b, dtype=dtype).reshape((phi - plo,) + full.shape[1:])
            htod += pled["htod"]
        bits = np.uint32 if dtype == np.float32 else np.uint64
        bad = np.argwhere(got.view(bits) != want.view(bits))
        unit = int(np.prod(full.shape[1:])) * full.itemsize
        rounds = (cfg.n + cfg.s_tb - 1) // cfg.s_tb
        ok_htod = htod == (sz + 2 * r) * unit * rounds  # no halo byte crossed PCIe twice
        print(f"SLAB world={world} dim={dim} {np.dtype(dtype).name} diffs={len(bad)} htod_ok={ok_htod}", flush=True)
        if len(bad) or not ok_htod:
            rows = np.unique(bad[:, 0])
            print("first diffs", bad[:5], "rows with diffs", rows[:20], "...", rows[-5:], "n rows", len(rows),
                  "slabs", [(a, b) for a, b, _, _ in parts], flush=True)
            sys.exit(1)
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
