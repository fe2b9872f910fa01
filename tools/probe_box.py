"""One-off probe of the GPU box: host CPU/RAM, PCIe pinned H2D/D2H/duplex GB/s."""
import json, os, subprocess, time
import torch

out = {}
out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
out["free"] = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout
out["smi"] = subprocess.run(["nvidia-smi", "-q", "-d", "CLOCK,PCI"], capture_output=True, text=True).stdout[-3000:]
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
out["numa"] = subprocess.run(["numactl", "-H"], capture_output=True, text=True).stdout if os.path.exists("/usr/bin/numactl") else "n/a"
dev = torch.device("cuda:0")
res = {}
for gb in [1, 4]:
    n = gb << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    for name in ["h2d", "d2h", "duplex"]:
        best = 0
        for it in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if name in ("h2d", "duplex"):
                with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
            if name in ("d2h", "duplex"):
                with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            bw = (n * (2 if name == "duplex" else 1)) / dt / 1e9
            best = max(best, bw)
        res[f"{name}_{gb}GiB_GBps"] = best
    del h, h2, d, d2
out["pcie"] = res
t0 = time.perf_counter(); a = torch.empty(8 << 30, dtype=torch.uint8); a.fill_(1); t1 = time.perf_counter()
b = torch.empty_like(a); t2 = time.perf_counter(); b.copy_(a); t3 = time.perf_counter()
out["host_fill_GBps"] = 8 * 1.074 / (t1 - t0)
out["host_copy_GBps_1thread_torch"] = 2 * 8 * 1.074 / (t3 - t2)
t0 = time.perf_counter(); torch.cuda.cudart().cudaHostRegister(a.data_ptr(), a.numel(), 0); t1 = time.perf_counter()
out["hostregister_8GiB_s"] = t1 - t0
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
print(json.dumps(out["pcie"]), out["host_fill_GBps"], out["hostregister_8GiB_s"])
