"""Copy-only model of the so2dr pipeline with the ENGINE's exact geometry
(bench grid: 92162 fp32 rows of 368648 bytes, d=16, h=64): H2D(i) moves rows
[c_i + h, c_{i+1} + h), D2H(i) rows [c_i, c_{i+1}), in place, with the unaligned
head split off. Compares torch's copies (dynamic cudart) with the engine."""
import json

import torch

P = 92162
RB = P * 4
D, H = 16, 64
fence = [1 + i * 5760 for i in range(D + 1)]
dev = torch.device("cuda", 0)
host = torch.empty(P * RB, dtype=torch.uint8, pin_memory=True)
work = 6000
bufs = [torch.empty(work * RB + 4096, dtype=torch.uint8, device=dev) for _ in range(3)]
s_h, s_d = torch.cuda.Stream(), torch.cuda.Stream()


def rows_h2d(i):
    lo = 0 if i == 0 else fence[i] + H
    hi = P if i == D - 1 else fence[i + 1] + H
    return lo, hi


def copy(dst, src, nbytes, head_split, host_addr, tail_split=False, align=128):
    head = (align - host_addr % align) % align if head_split else 0
    tail = (host_addr + nbytes) % align if tail_split else 0
    if head:
        dst[:head].copy_(src[:head], non_blocking=True)
    dst[head:nbytes - tail].copy_(src[head:nbytes - tail], non_blocking=True)
    if tail:
        dst[nbytes - tail:nbytes].copy_(src[nbytes - tail:nbytes], non_blocking=True)


def run(head_split=True, congruent=True, tail_h=False, tail_d=False, align=128):
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    s_h.wait_event(t0)
    s_d.wait_event(t0)
    done = [None] * D
    ev = {}
    for i in range(D):
        b = bufs[i % 3]
        wlo = 0 if i == 0 else fence[i] - H
        lo, hi = rows_h2d(i)
        hb = host[lo * RB:hi * RB]
        shift = ((host.data_ptr() + wlo * RB) - b.data_ptr()) % 256 if congruent else 0
        dv = b[shift:]
        with torch.cuda.stream(s_h):
            if i >= 3:
                s_h.wait_event(done[i - 3])
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            copy(dv[(lo - wlo) * RB:], hb, (hi - lo) * RB, head_split, hb.data_ptr(), tail_h, align)
            z.record()
            ev[("h", i)] = (a, z, (hi - lo) * RB)
        with torch.cuda.stream(s_d):
            s_d.wait_event(z)
            a2, z2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a2.record()
            clo, chi = fence[i], fence[i + 1]
            hd = host[clo * RB:chi * RB]
            copy(hd, dv[(clo - wlo) * RB:], (chi - clo) * RB, head_split, hd.data_ptr(), tail_d, align)
            z2.record()
            done[i] = z2
            ev[("d", i)] = (a2, z2, (chi - clo) * RB)
    torch.cuda.synchronize()
    total = max(t0.elapsed_time(z) for (a, z, n) in ev.values())
    mid = [(k, n / a.elapsed_time(z) / 1e6) for (k, i), (a, z, n) in ev.items() if 4 <= i < 12]
    h = sum(r for k, r in mid if k == "h") / 8
    d = sum(r for k, r in mid if k == "d") / 8
    return total, h, d


run()
for trial in range(2):
    for name, kw in (("align128", {}), ("align512", {"align": 512}), ("align4096", {"align": 4096}),
                     ("align4096_tails", {"align": 4096, "tail_h": True, "tail_d": True}),
                     ("align65536", {"align": 65536})):
        t, h, d = run(**kw)
        print(json.dumps({"trial": trial, "pattern": name, "total_ms": round(t, 1), "steady_h2d_GBps": round(h, 1),
                          "steady_d2h_GBps": round(d, 1)}), flush=True)
