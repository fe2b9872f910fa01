"""Duplex copy split vs the host-address distance between the concurrently
read (H2D) and written (D2H) regions. Pipeline of NCH chunks (3 device buffers):
H2D(i) reads host[A + i*CH], D2H(i) writes host[A + delta + i*CH]; in steady
state D2H(i) overlaps H2D(i+1), i.e. the cursors are delta - CH apart."""
import json
import sys

import torch

GB = 1 << 30
dev = torch.device("cuda", 0)
CH = 2_120_000_000 // 4096 * 4096
NCH = 8
MAXD = 10 * GB
host = torch.empty(NCH * CH + MAXD + 4096, dtype=torch.uint8, pin_memory=True)
bufs = [torch.empty(CH, dtype=torch.uint8, device=dev) for _ in range(3)]
s_h, s_d = torch.cuda.Stream(), torch.cuda.Stream()


def run(delta):
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    s_h.wait_event(t0)
    s_d.wait_event(t0)
    done = [None] * NCH
    ev = {}
    for i in range(NCH):
        b = bufs[i % 3]
        with torch.cuda.stream(s_h):
            if i >= 3:
                s_h.wait_event(done[i - 3])
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            b.copy_(host[i * CH:(i + 1) * CH], non_blocking=True)
            z.record()
            ev[("h", i)] = (a, z)
        with torch.cuda.stream(s_d):
            s_d.wait_event(z)
            a2, z2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a2.record()
            host[delta + i * CH:delta + (i + 1) * CH].copy_(b, non_blocking=True)
            z2.record()
            done[i] = z2
            ev[("d", i)] = (a2, z2)
    torch.cuda.synchronize()
    mid = [(k, CH / a.elapsed_time(z) / 1e6) for (k, i), (a, z) in ev.items() if 2 <= i < 6]
    h = sum(r for k, r in mid if k == "h") / 4
    d = sum(r for k, r in mid if k == "d") / 4
    return max(t0.elapsed_time(z) for (a, z) in ev.values()), h, d


run(0)
for delta_mb in (0, 1024, 2048 - 512, 2048 - 128, 2048 - 64, 2048 - 32, 2048 - 16, 2048 - 4, 2048, 2048 + 4, 2048 + 64,
                 3072, 4096 - 64, 4096, 4096 + 64, 2022 + 2022, 6144, 8192 - 64, 8192):
    delta = delta_mb << 20
    t, h, d = run(delta)
    print(json.dumps({"delta_MiB": delta_mb, "cursor_gap_MiB": delta_mb - CH / 2**20, "total_ms": round(t, 1),
                      "h2d_GBps": round(h, 1), "d2h_GBps": round(d, 1)}), flush=True)
