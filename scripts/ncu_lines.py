"""Top source lines by warp-stall samples from `ncu --page source --csv
--print-source cuda,sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur = None
hdr = None
data = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        try:
            v = float(r[4] or 0)
        except ValueError:
            continue
        data.append((v, cur, r[0], r[1].strip()[:110]))
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for v, f, l, s in sorted(data, reverse=True)[:n]:
    print(f"{v / tot * 100:5.1f}% {f}:{l} {s}")
