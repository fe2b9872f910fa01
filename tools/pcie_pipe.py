"""Copy-only model of the so2dr pipeline (no kernels, no engine): 16 chunks of
2.12 GB through 3 device buffers, H2D(i) waits for D2H(i-3), D2H(i) waits for
H2D(i). Prints per-copy start/duration/GB/s on one common clock, for a few
issue patterns, to find one that keeps BOTH directions near the duplex cap.

  base      : one cudaMemcpyAsync per chunk and direction
  split<P>  : each chunk copy issued as P pieces
  lead<L>   : H2D(i) additionally waits for D2H(i-L) to START (L >= 1)
"""
import json
import sys

import torch

GB = 1 << 30
dev = torch.device("cuda", 0)
CH = 2_120_000_000 // 4096 * 4096
NCH = 16
host = torch.empty(CH * (NCH + 1) + 4096, dtype=torch.uint8, pin_memory=True)
bufs_raw = [torch.empty(CH + 8192, dtype=torch.uint8, device=dev) for _ in range(3)]
s_h, s_d = torch.cuda.Stream(), torch.cuda.Stream()


s_c = torch.cuda.Stream()
slots = [torch.empty(47_000_000, dtype=torch.uint8, device=dev) for _ in range(3)]


def run(pieces=1, lead=0, inplace=False, d2d=False, hoff=0, doff=0, head=0, tailcut=0):
    bufs = [b[doff:doff + CH] for b in bufs_raw]
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    s_h.wait_event(t0)
    s_d.wait_event(t0)
    ev = {}
    d2h_done, d2h_start = [None] * NCH, [None] * NCH
    for i in range(NCH):
        b = bufs[i % 3]
        with torch.cuda.stream(s_h):
            if i >= 3:
                s_h.wait_event(d2h_done[i - 3])
            if lead and i - lead >= 0 and d2h_start[i - lead] is not None:
                s_h.wait_event(d2h_start[i - lead])
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            pb = CH // pieces
            L = CH - tailcut
            if head:
                b[:head].copy_(host[hoff + i * CH:hoff + i * CH + head], non_blocking=True)
                b[head:L].copy_(host[hoff + i * CH + head:hoff + i * CH + L], non_blocking=True)
            else:
                for p in range(pieces):
                    hi = L if p == pieces - 1 else (p + 1) * pb
                    b[p * pb:hi].copy_(host[hoff + i * CH + p * pb:hoff + i * CH + hi], non_blocking=True)
            z.record()
            ev[("h", i)] = (a, z)
        if d2d:  # region sharing on a compute stream between H2D and D2H (engine: s_cmp)
            with torch.cuda.stream(s_c):
                s_c.wait_event(z)
                slots[i % 3].copy_(b[:47_000_000], non_blocking=True)
                b[CH - 47_000_000:].copy_(slots[(i + 2) % 3], non_blocking=True)
                z = torch.cuda.Event()
                z.record()
        dst0 = hoff + (i * CH if inplace else (i + 1) * CH)
        with torch.cuda.stream(s_d):
            s_d.wait_event(z)
            a2, z2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a2.record()
            d2h_start[i] = a2
            if head:
                host[dst0:dst0 + head].copy_(b[:head], non_blocking=True)
                host[dst0 + head:dst0 + L].copy_(b[head:L], non_blocking=True)
            else:
                for p in range(pieces):
                    hi = L if p == pieces - 1 else (p + 1) * pb
                    host[dst0 + p * pb:dst0 + hi].copy_(b[p * pb:hi], non_blocking=True)
            z2.record()
            d2h_done[i] = z2
            ev[("d", i)] = (a2, z2)
    torch.cuda.synchronize()
    total = max(t0.elapsed_time(z) for (a, z) in ev.values())
    rows = []
    for (k, i), (a, z) in sorted(ev.items(), key=lambda kv: (kv[0][1], kv[0][0])):
        ms = a.elapsed_time(z)
        rows.append((k, i, round(t0.elapsed_time(a), 1), round(ms, 1), round(CH / ms / 1e6, 1)))
    return total, rows


CASES = [("h0_d0", {}), ("h8_d8", {"hoff": 8, "doff": 8}), ("h8_d8_head120", {"hoff": 8, "doff": 8, "head": 120}),
         ("h0_tail_unaligned", {"tailcut": 1000}), ("h8_d8_head120_tail", {"hoff": 8, "doff": 8, "head": 120, "tailcut": 1000}),
         ("h0_head128", {"head": 128})]
run()
for trial in range(2):
    for name, kw in CASES:
        total, rows = run(**kw)
        mid = [r for r in rows if 4 <= r[1] < 12]
        h = sum(r[4] for r in mid if r[0] == "h") / 8
        d = sum(r[4] for r in mid if r[0] == "d") / 8
        print(json.dumps({"trial": trial, "pattern": name, "total_ms": round(total, 1),
                          "steady_h2d_GBps": round(h, 1), "steady_d2h_GBps": round(d, 1)}), flush=True)
