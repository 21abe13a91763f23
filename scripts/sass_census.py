"""SASS instruction census of the in-tree library (cuobjdump -sass, sm_100a):
static per-kernel counts of the instructions that prove the tensor-core path
(UTCHMMA = tcgen05.mma, UTMALDG = TMA load, LDTM = tcgen05.ld) and the
CUDA-core arithmetic (FFMA, DFMA, DADD).  CPU only.

  python scripts/sass_census.py [lib.so] > profiles/r02/sass_summary.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2506_00185_b200", "libtbeam_b200.so")
OPS = ["UTCHMMA", "UTMALDG", "LDTM", "FFMA", "DFMA", "DADD"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
counts = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(1)
        for o in OPS:
            if op == o:
                counts[cur][o] += 1

names = {}
if counts:
    dem = subprocess.run(["cu++filt"], input="\n".join(counts), capture_output=True, text=True)
    if dem.returncode == 0:
        names = dict(zip(counts, dem.stdout.splitlines()))
print(f"SASS instruction census of {os.path.relpath(LIB, ROOT)} (cuobjdump -sass, sm_100a):")
print("tcgen05 MMA = UTCHMMA, TMA loads = UTMALDG, TMEM loads = LDTM; per kernel (static counts)")
tot = collections.Counter()
for fn, c in counts.items():
    if not c:
        continue
    tot.update(c)
    print()
    print(names.get(fn, fn))
    print("    " + "  ".join(f"{o}={c[o]}" for o in OPS if c[o]))
print()
print("total: " + "  ".join(f"{o}={tot[o]}" for o in OPS))
