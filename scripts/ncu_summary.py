"""Per-kernel summary of an `ncu --set full` report (averages over the
captured launches of each kernel): duration, DRAM bytes, tensor-pipe and SM
throughput, grid, registers, smem, executed instructions.  Cold-cache,
serialised replay: compare shares, not absolutes.

  python scripts/ncu_summary.py REPORT.ncu-rep [title]
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__registers_per_thread",
           "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
agg = collections.OrderedDict()
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("tbeam_dev::", "")
    agg.setdefault(name, []).append(d)
print(f"== {title}")
for name, ds in agg.items():
    print(f"  {name}  (launches captured: {len(ds)})")
    for m in METRICS:
        if m not in hdr:
            continue
        vals = []
        for d in ds:
            try:
                vals.append(float(d[m].replace(",", "")))
            except ValueError:
                pass
        if vals:
            u = units[hdr.index(m)]
            print(f"     {m:70s} {sum(vals) / len(vals):16.3f} {u}")
