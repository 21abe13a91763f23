"""DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, from
`ncu --set full` reports) of the per-round kernels, merged into
profiles/kernel_traffic.json under a workload key -- bench.py reads it for
the `traffic` field of each roofline entry.

  python scripts/ncu_traffic.py KEY REPORT.ncu-rep [REPORT ...]   (KEY e.g. bench/bf16)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "kernel_traffic.json")
M = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]


def family(name: str) -> str:
    if "JointEpi" in name:
        return "joint"
    if "GatesEpi" in name:
        return "lstm_gates"
    if "ProjEpi" in name:
        return "lstm_proj"
    if "select_kernel" in name:
        return "select"
    return name.split("(")[0]


def main():
    key, reps = sys.argv[1], sys.argv[2:]
    acc = collections.defaultdict(list)
    for rep in reps:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            if len(r) != len(hdr):
                continue
            d = dict(zip(hdr, r))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = 0.0
            for m in M[:2]:
                u = units[hdr.index(m)]
                b += float(d[m].replace(",", "")) * mult.get(u, 1)
            acc[family(d["Kernel Name"])].append(b)
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data[key] = {k: sum(v) / len(v) for k, v in acc.items()}
    data[key + "/launches_captured"] = {k: len(v) for k, v in acc.items()}
    json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(data[key], indent=1))


if __name__ == "__main__":
    main()
