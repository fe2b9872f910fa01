"""Multi-rank slab partitioning.

CPU (gloo, world 2 and 4): the slab geometry the engine uses (so2dr_slab_rows:
rank g owns rows [fence[g*d/G], fence[(g+1)*d/G]) plus the ring rows at the
global edges) and the per-round halo protocol (each rank ships its r*S_TB-row
edge bands to its neighbours, receives theirs, advances its slab S_TB steps
with trapezoid recompute) reproduce the single-domain oracle bit-for-bit.
Bands travel over torch.distributed (gloo) here; on GPUs the engine pushes
them over CUDA IPC peer memory (tests/test_gpu_multirank.py runs that path)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfgt, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch

    import paper_2309_08864_b200 as so2dr
    import pyoracle as o

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sz, r, d, s_tb, n = cfgt
    cfg = so2dr.RunConfig(sz=sz, r=r, d=d, s_tb=s_tb, k_on=s_tb, n=n)
    fence, _ = so2dr.plan_chunks(cfg)
    lo, hi = so2dr.slab_rows(cfg, rank, world)
    p = sz + 2 * r
    w = o.box_weights(r)
    full0 = o.init_grid(sz, r, 7)
    mine = full0[lo:hi].copy()
    dl = d // world
    rounds = (n + s_tb - 1) // s_tb
    for t in range(rounds):
        k = s_tb if (t < rounds - 1 or n % s_tb == 0) else n % s_tb
        h = r * s_tb
        # edge bands of this round (own rows only; exactly what so2dr_slab_run stages)
        ext = np.zeros((p, p), np.float32)
        ext[lo:hi] = mine
        reqs = []
        if rank > 0:
            band = torch.from_numpy(mine[fence[rank * dl] - lo: fence[rank * dl] - lo + h].copy())
            reqs.append(dist.isend(band, rank - 1))
            recv_lo = torch.empty((h, p))
            reqs.append(dist.irecv(recv_lo, rank - 1))
        if rank < world - 1:
            c = fence[(rank + 1) * dl]
            band = torch.from_numpy(mine[c - h - lo: c - lo].copy())
            reqs.append(dist.isend(band, rank + 1))
            recv_hi = torch.empty((h, p))
            reqs.append(dist.irecv(recv_hi, rank + 1))
        for rq in reqs:
            rq.wait()
        if rank > 0:
            c = fence[rank * dl]
            ext[c - h:c] = recv_lo.numpy()
        if rank < world - 1:
            c = fence[(rank + 1) * dl]
            ext[c:c + h] = recv_hi.numpy()
        # advance k steps; rows farther than r*k from the received halo edge are exact
        adv = o.run(ext, o.BOX, r, w, k)
        mine = adv[lo:hi].copy()
        # ring rows never change
        if rank == 0:
            mine[:r] = full0[:r]
        if rank == world - 1:
            mine[-r:] = full0[p - r:]
    parts = [None] * world
    dist.all_gather_object(parts, (lo, hi, mine))
    if rank == 0:
        got = np.empty_like(full0)
        for a, b, m in parts:
            got[a:b] = m
        want = o.run(full0, o.BOX, r, w, n)
        q.put(int((got.view(np.uint32) != want.view(np.uint32)).sum()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cfgt", [(2, (64, 1, 4, 4, 10)), (4, (96, 1, 8, 5, 12)), (2, (64, 2, 4, 2, 7))])
def test_slab_protocol_matches_single_domain(world, cfgt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, cfgt, q)) for rk in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    assert q.get(timeout=5) == 0


def test_slab_rows_partition_the_grid():
    sys.path.insert(0, ROOT)
    import paper_2309_08864_b200 as so2dr

    for world in (1, 2, 4, 8):
        cfg = so2dr.RunConfig(sz=1024, r=1, d=16, s_tb=8, k_on=4, n=16)
        cur = 0
        for g in range(world):
            lo, hi = so2dr.slab_rows(cfg, g, world)
            assert lo == cur
            cur = hi
        assert cur == 1026
    with pytest.raises(so2dr.InvalidSpecError):
        so2dr.slab_rows(so2dr.RunConfig(sz=1024, r=1, d=6, s_tb=8, k_on=4, n=16), 0, 4)
