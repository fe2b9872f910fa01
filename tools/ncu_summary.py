"""Summarise ncu evidence (run here, on the CPU box, over files gpurun brought back).

  python tools/ncu_summary.py launches <launches.csv> <out.json>
      per-kernel launch count, total/avg device time and share of all launches
  python tools/ncu_summary.py full <report.ncu-rep> <out.json> [alg_bytes_per_launch]
      headline metrics of a --set full capture (duration, DRAM traffic, SM
      activity spread, FMA pipe, occupancy, top stall reasons)
"""
import csv
import io
import json
import re
import subprocess
import sys


def launches(path, out):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        full = r["Kernel Name"]
        key = full if len(full) < 160 else full[:160]
        ns = float(r["Metric Value"].replace(",", ""))
        e = per.setdefault(key, {"kernel": key, "short": name, "launches": 0, "total_ns": 0.0})
        e["launches"] += 1
        e["total_ns"] += ns
    tot = sum(e["total_ns"] for e in per.values()) or 1.0
    res = sorted(per.values(), key=lambda e: -e["total_ns"])
    for e in res:
        e["avg_ms"] = e["total_ns"] / e["launches"] / 1e6
        e["share"] = e["total_ns"] / tot
    json.dump({"source": path, "note": "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, "
               "serialised launches; compare shares, not absolutes", "kernels": res}, open(out, "w"), indent=1)
    for e in res:
        print(f"{e['launches']:5d} {e['avg_ms']:9.3f} ms  share {e['share']:.3f}  {e['short']}")


KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__cycles_active.avg": "sm_active_avg",
    "sm__cycles_active.max": "sm_active_max",
    "sm__cycles_active.min": "sm_active_min",
    "sm__cycles_elapsed.max": "sm_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_inst_pct_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_elapsed",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
              "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}


def full(path, out, alg=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        m = {"kernel": v[hdr.index("Kernel Name")][:200]}
        stalls = []
        for k, u, x in zip(hdr, units, v):
            try:
                f = float(x.replace(",", ""))
            except ValueError:
                continue
            if k in KEYS:
                m[KEYS[k]] = f * UNIT_SCALE.get(u, 1)
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                stalls.append((f, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(s for s, _ in stalls) or 1.0
        m["stalls_share"] = {k: round(s / tot, 3) for s, k in sorted(stalls, reverse=True)[:8]}
        if "dram_read" in m:
            m["dram_bytes"] = m["dram_read"] + m.get("dram_write", 0)
        if "duration_ns" in m and "dram_bytes" in m:
            m["dram_GBps"] = m["dram_bytes"] / m["duration_ns"]
        if alg:
            m["alg_bytes"] = float(alg)
            m["traffic_over_alg"] = m["dram_bytes"] / float(alg)
        if "sm_active_avg" in m and "sm_elapsed" in m:
            m["sm_active_avg_frac"] = m["sm_active_avg"] / m["sm_elapsed"]
        res.append(m)
    json.dump({"source": path, "captures": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
