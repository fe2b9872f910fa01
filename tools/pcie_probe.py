"""PCIe duplex behaviour on this box: per-direction GB/s (CUDA events on each
copy stream) for pinned copies, looking for the copy pattern that keeps both
directions busy at the highest combined rate.

  A: 2 GiB single copies, alone / duplex (started together)
  B: duplex with D2H started 10 ms after H2D (the pipeline's situation)
  C: slices of one 34 GB pinned buffer (the bench grid), duplex
  D: duplex in pieces of P MB interleaved on one stream per direction
  E: duplex with 2 streams per direction
"""
import json
import time

import torch

dev = torch.device("cuda", 0)
GB = 1 << 30
N = 2 * GB
h1 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(N, dtype=torch.uint8, device=dev)
d2 = torch.empty(N, dtype=torch.uint8, device=dev)
S = [torch.cuda.Stream() for _ in range(4)]


def timed(fn_h, fn_d, delay_d_ms=0.0):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(S[0]):
        e[0].record()
        fn_h()
        e[1].record()
    with torch.cuda.stream(S[1]):
        if delay_d_ms:
            torch.cuda._sleep(int(delay_d_ms * 1.9e6))
        e[2].record()
        fn_d()
        e[3].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])


def rep(name, nbytes_h, nbytes_d, t):
    print(json.dumps({"case": name, "h2d_GBps": round(nbytes_h / t[0] / 1e6, 1),
                      "d2h_GBps": round(nbytes_d / t[1] / 1e6, 1),
                      "combined_GBps": round((nbytes_h + nbytes_d) / max(t) / 1e6, 1)}), flush=True)


for _ in range(2):
    t = timed(lambda: d1.copy_(h1, non_blocking=True), lambda: h2.copy_(d2, non_blocking=True))
rep("A duplex 2GiB", N, N, t)
t = timed(lambda: d1.copy_(h1, non_blocking=True), lambda: h2.copy_(d2, non_blocking=True), delay_d_ms=10)
rep("B duplex, D2H 10 ms late", N, N, t)
t = timed(lambda: d1.copy_(h1, non_blocking=True), lambda: None)
print(json.dumps({"case": "A h2d alone", "GBps": round(N / t[0] / 1e6, 1)}))

# C: one 34 GB pinned buffer, H2D from the front, D2H into the back
big = torch.empty(34 * GB, dtype=torch.uint8, pin_memory=True)
for off_h, off_d in ((0, 17 * GB), (4 * GB, 2 * GB)):
    t = timed(lambda: d1.copy_(big[off_h:off_h + N], non_blocking=True),
              lambda: big[off_d:off_d + N].copy_(d2, non_blocking=True))
    rep(f"C 34GB buffer h@{off_h >> 30}G d@{off_d >> 30}G", N, N, t)

# D: pieces interleaved
for P in (16, 64, 256):
    pb = P << 20
    n = N // pb

    def fh():
        for i in range(n):
            d1[i * pb:(i + 1) * pb].copy_(h1[i * pb:(i + 1) * pb], non_blocking=True)

    def fd():
        for i in range(n):
            h2[i * pb:(i + 1) * pb].copy_(d2[i * pb:(i + 1) * pb], non_blocking=True)

    t = timed(fh, fd)
    rep(f"D pieces {P} MB", N, N, t)

# E: 2 streams per direction
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
half = N // 2
for k, s in enumerate(S):
    s.wait_event(ev[0])
    with torch.cuda.stream(s):
        if k < 2:
            d1[k * half:(k + 1) * half].copy_(h1[k * half:(k + 1) * half], non_blocking=True)
        else:
            h2[(k - 2) * half:(k - 1) * half].copy_(d2[(k - 2) * half:(k - 1) * half], non_blocking=True)
for s in S:
    torch.cuda.current_stream().wait_stream(s)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1])
print(json.dumps({"case": "E 2 streams/dir", "combined_GBps": round(2 * N / ms / 1e6, 1)}), flush=True)

# F: D2H-first pacing: D2H ahead by one piece, H2D paced by events
for P in (64, 256):
    pb = P << 20
    n = N // pb
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S[0].wait_event(e0)
    S[1].wait_event(e0)
    done_d = []
    for i in range(n):
        with torch.cuda.stream(S[1]):
            h2[i * pb:(i + 1) * pb].copy_(d2[i * pb:(i + 1) * pb], non_blocking=True)
            ed = torch.cuda.Event()
            ed.record()
            done_d.append(ed)
        with torch.cuda.stream(S[0]):
            if i >= 1:
                S[0].wait_event(done_d[i - 1])
            d1[i * pb:(i + 1) * pb].copy_(h1[i * pb:(i + 1) * pb], non_blocking=True)
    torch.cuda.current_stream().wait_stream(S[0])
    torch.cuda.current_stream().wait_stream(S[1])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"case": f"F paced pieces {P} MB (H2D i waits D2H i-1)",
                      "combined_GBps": round(2 * N / ms / 1e6, 1)}), flush=True)
