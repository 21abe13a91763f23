"""First round where the GPU and the oracle disagree on one stream: both
record the stream's slot state after every round (tbeam_debug_round_trace in
host-loop mode, oracle_round_trace), this prints the first differing round
with context.  Measurement aid, not a test.

  python scripts/round_diff.py --config c5 --stream 205 [--len 40] [--beam 16] [--algo aes] [--tol 1e-2]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.cpu import Oracle  # noqa: E402
from paper_2506_00185_b200 import _abi  # noqa: E402
from paper_2506_00185_b200.decoder import B200Decoder  # noqa: E402
from paper_2506_00185_b200.model import synthetic_vocabulary  # noqa: E402
from paper_2506_00185_b200.workloads import workload  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c5")
p.add_argument("--stream", type=int, default=205)
p.add_argument("--len", type=int, default=None)
p.add_argument("--beam", type=int, default=None)
p.add_argument("--algo", default=None, choices=[None, "alsd", "aes", "greedy"])
p.add_argument("--tol", type=float, default=1e-4)
p.add_argument("--prefix", type=int, default=1)
a = p.parse_args()

w = workload(a.config)
T = w.T
L = a.len or T
algo = {"alsd": _abi.ALGO_ALSD, "aes": _abi.ALGO_AES, "greedy": _abi.ALGO_GREEDY, None: w.runs[0][1]}[a.algo]
K = a.beam or w.runs[0][2]
cfg = w.config(K, return_nbest=4)
cfg.aes_prefix_search = bool(a.prefix)
enc = w.frames([a.stream])
orc = Oracle()
orc.lib.oracle_round_trace.restype = C.c_int64
orc.lib.oracle_round_trace.argtypes = [C.c_int32, C.c_void_p, C.c_int64]
olm = orc.lm(w.arpa, synthetic_vocabulary(w.model.spec.vocab_size)) if w.arpa else None
orc.lib.oracle_round_trace(0, None, 0)
want = orc.decode(w.model, cfg, algo, enc, [L], lm=olm)
n = orc.lib.oracle_round_trace(-1, None, 0)
obuf = np.zeros(n)
orc.lib.oracle_round_trace(-1, obuf.ctypes.data, n)

dec = B200Decoder(w.model)
if w.arpa:
    dec.set_lm(w.arpa)
lib = dec.lib
lib.tbeam_debug_round_trace.restype = C.c_int64
lib.tbeam_debug_round_trace.argtypes = [C.c_int32, C.c_void_p, C.c_int64]
dec.set_graph_mode(0)
lib.tbeam_debug_round_trace(0, None, 0)
got = dec.decode(algo, enc, [L], cfg)
n = lib.tbeam_debug_round_trace(-1, None, 0)
gbuf = np.zeros(n)
lib.tbeam_debug_round_trace(-1, gbuf.ctypes.data, n)

rec = 5 + 6 * K
o = obuf.reshape(-1, rec)
g = gbuf.reshape(-1, rec)
g = g[: int(np.argmax(g[:, 2] > 0)) + 1] if (g[:, 2] > 0).any() else g
print(f"oracle rounds {len(o)}, gpu rounds {len(g)}; final gpu {[round(e.score, 4) for e in got.streams[0].nbest]} "
      f"oracle {[round(e.score, 4) for e in want.streams[0].nbest]}")


def slots(r):
    s = r[5:].reshape(K, 6)
    return [(round(x[0], 5) if np.isfinite(x[0]) else None, int(x[1]), int(x[2]), int(x[3]),
             f"{int(x[4]):08x}{int(x[5]):08x}"[-6:]) for x in s]


def same(x, y):
    for (sa, fa, la, ta, ha), (sb, fb, lb, tb, hb) in zip(x, y):
        if (sa is None) != (sb is None):
            return False
        if sa is not None and (abs(sa - sb) > a.tol or fa != fb or la != lb or ta != tb or ha != hb):
            return False
    return True


for i in range(min(len(o), len(g))):
    if not same(slots(o[i]), slots(g[i])):
        print(f"first difference at round {i}")
        for j in range(max(0, i - 2), min(i + 2, len(o), len(g))):
            print(f"-- round {j}: oracle t={int(o[j][0])} r={int(o[j][1])} (K-th kept {o[j][3]:.6f}, best rejected "
                  f"{o[j][4]:.6f}) | gpu next t={int(g[j][0])} r={int(g[j][1])}")
            for k, (x, y) in enumerate(zip(slots(o[j]), slots(g[j]))):
                print(f"   slot {k:2d}  oracle {x}   gpu {y}")
        break
else:
    print("no difference in the common rounds")
