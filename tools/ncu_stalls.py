"""Per-opcode stall attribution from an ncu --page source --csv --print-source sass
dump: python tools/ncu_stalls.py <source.csv> [addr_lo addr_hi]  (hex offsets
relative to the kernel start select a loop)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
body = rows[2:]
base = int(body[0][ix["Address"]], 16)
lo = int(sys.argv[2], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 62
per = collections.defaultdict(collections.Counter)
ex = collections.Counter()
tot = collections.Counter()
for r in body:
    off = int(r[ix["Address"]], 16) - base
    if not lo <= off <= hi:
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[ix["Source"]].strip()).split()[0].split(".")[0]
    ex[op] += int(r[ix["Instructions Executed"]] or 0)
    for h in reasons:
        v = int(r[ix[h]] or 0)
        per[op][h[6:]] += v
        tot[h[6:]] += v
T = sum(tot.values())
print("total samples", T, "by reason:", ", ".join(f"{k} {v / T:.3f}" for k, v in tot.most_common(8)))
E = sum(ex.values())
for op, c in sorted(per.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    s = sum(c.values())
    print(f"{op:10s} samples {s / T:.3f} exec {ex[op] / E:.3f}  " + ", ".join(f"{k} {v / T:.3f}" for k, v in c.most_common(4)))
