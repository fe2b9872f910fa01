"""Per-launch DRAM traffic of the bench's K1 launches from an ncu metrics CSV
(gpu_round.sh ncu step: dram__bytes_read.sum + dram__bytes_write.sum over the
16 launches of chunk 5 of one bench step), against the bench's algorithmic
bytes per launch; writes the profiles/k1_traffic.json bench.py reads.
  python tools/k1_traffic.py <k1_traffic.csv> <bench_line.json> <out.json> <source-label>"""
import csv
import io
import json
import sys

text = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))
per = {}
for r in rows:
    if r["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        per[r["ID"]] = per.get(r["ID"], 0.0) + v * scale
line = json.load(open(sys.argv[2]))
alg = line["roofline"]["alg_bytes_per_launch"]
dram = sum(per.values()) / len(per)
out = {"d": line["config"]["d"], "k_on": line["config"]["k_on"], "launches_captured": len(per),
       "dram_bytes_per_launch": dram, "alg_bytes_per_launch_run_avg": alg, "dram_over_alg": dram / alg,
       "source": sys.argv[4]}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out))
