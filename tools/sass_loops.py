"""List the loops (backward branches) of one SASS function dump with their
instruction mix: python tools/sass_loops.py <function.sass>"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA (?:`\(\.L_x_\d+\) )?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt <= a and tgt in addr_idx:
            loops.append((addr_idx[tgt], i))
for s, e in loops:
    c = collections.Counter()
    for _, t in ins[s:e + 1]:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
        c[op] += 1
    tot = sum(c.values())
    print(f"loop {ins[s][0]:#x}-{ins[e][0]:#x}: {tot} instr, FFMA2 {c['FFMA2']}, FFMA {c['FFMA']}; top: "
          + ", ".join(f"{k}:{v}" for k, v in c.most_common(12)))
