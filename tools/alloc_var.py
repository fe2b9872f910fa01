"""Is the e2e run time a property of the host allocation? Allocate the bench
grid several times (so2dr_host_alloc, and malloc+THP+cudaHostRegister), run the
bench's so2dr config 3x on each, print per-allocation times."""
import ctypes
import json
import mmap
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2309_08864_b200 as so2dr  # noqa: E402

for f in ("/sys/kernel/mm/transparent_hugepage/enabled", "/sys/kernel/mm/transparent_hugepage/defrag",
          "/proc/sys/vm/nr_hugepages"):
    try:
        print(f, open(f).read().strip(), flush=True)
    except Exception as e:
        print(f, e)
try:
    print(open("/proc/cmdline").read().strip()[:300])
except Exception:
    pass
sz = 92160
p = sz + 2
eng = so2dr.Engine(0, 16 << 30)
spec = so2dr.StencilSpec.box(1)
cfg = so2dr.RunConfig(sz=sz, r=1, d=64, s_tb=64, k_on=4, n_strm=3, n=64)
for trial in range(3):
    host = eng.host_array((p, p), np.float32)
    eng.init_grid(sz, 1, 42, out=host)
    ts = [eng.run("so2dr", host, spec, cfg, diag=False).timing["device_ms"] for _ in range(3)]
    print(json.dumps({"alloc": f"cudaHostAlloc#{trial}", "addr_mod_2M": host.ctypes.data % (2 << 20),
                      "ms": [round(t, 1) for t in ts]}), flush=True)
    del host
# THP-backed anonymous memory, registered
nbytes = p * p * 4
libc = ctypes.CDLL("libc.so.6")
for trial in range(2):
    mm = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(mm))
    aligned = (base + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc.madvise(ctypes.c_void_p(aligned), ctypes.c_size_t(nbytes), 14)  # MADV_HUGEPAGE
    arr = np.frombuffer(mm, dtype=np.uint8, count=nbytes, offset=aligned - base).view(np.float32).reshape(p, p)
    arr[:] = 0  # fault in
    eng.host_register(arr)
    eng.init_grid(sz, 1, 42, out=arr)
    ts = [eng.run("so2dr", arr, spec, cfg, diag=False).timing["device_ms"] for _ in range(3)]
    try:
        thp = [l for l in open("/proc/self/smaps_rollup") if "AnonHugePages" in l]
    except Exception:
        thp = []
    print(json.dumps({"alloc": f"mmap+THP+register#{trial}", "ms": [round(t, 1) for t in ts], "thp": thp}), flush=True)
    eng.host_unregister(arr)
    del arr
    mm.close()
