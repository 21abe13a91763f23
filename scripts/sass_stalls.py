"""Top SASS instructions by warp-stall samples from
`ncu -i X.ncu-rep --page source --csv --print-source sass` (all kernels in
the report; one section per kernel)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
secs = []
for r in rows:
    if r and r[0] == "Kernel Name":
        secs.append([r[1], None, []])
    elif r and r[0] == "Address":
        secs[-1][1] = r
    elif secs and secs[-1][1] is not None and len(r) == len(secs[-1][1]):
        secs[-1][2].append(r)
for name, hdr, data in secs:
    i = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[i] or 0) for r in data) or 1
    print(f"== {name[:100]}  samples={tot:.0f}")
    order = sorted(range(len(data)), key=lambda k: -float(data[k][i] or 0))[:n]
    for k in order:
        r = data[k]
        print(f"  {float(r[i]) / tot * 100:5.1f}%  [{k:5d}] {r[1].strip()[:90]}")
