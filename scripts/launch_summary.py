"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if len(r) > 10 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        m = re.search(r"tc_gemm<\(?i?n?t?\)?(\d+), tbeam_dev::(\w+)", name)
        short = f"tc_gemm<{m.group(1)},{m.group(2)}>" if m else name.split("(")[0].replace("void ", "")
        agg[short].append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:45s} n={len(v):5d} total={sum(v)/1e3:9.1f}us avg={sum(v)/len(v)/1e3:7.2f}us share={sum(v)/tot*100:5.1f}%")
