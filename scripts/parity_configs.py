"""Measure GPU-vs-oracle agreement at every BASELINE config's full shape
(no asserts; tests/test_gpu_configs.py is the gate).  Per config and
algorithm: max |dscore| over the sampled streams' n-best, token mismatches
(stream, entry, the oracle's margin there), counter mismatches.

  python scripts/parity_configs.py [--only c3,c5] [--sample 16] > parity.jsonl
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.cpu import Oracle  # noqa: E402
from paper_2506_00185_b200 import _abi  # noqa: E402
from paper_2506_00185_b200.decoder import B200Decoder  # noqa: E402
from paper_2506_00185_b200.model import synthetic_vocabulary  # noqa: E402
from paper_2506_00185_b200.workloads import workload  # noqa: E402


def compare(got, want):
    out = {"max_abs_dscore": 0.0, "mismatch": [], "counter_mismatch": 0, "frames_mismatch": 0}
    for s, (x, y) in enumerate(zip(got.streams, want.streams)):
        for ex, ey in zip(x.nbest, y.nbest):
            out["max_abs_dscore"] = max(out["max_abs_dscore"], abs(ex.score - ey.score))
        mism = next((i for i, (ex, ey) in enumerate(zip(x.nbest, y.nbest)) if ex.tokens != ey.tokens), None)
        if len(x.nbest) != len(y.nbest):
            out["mismatch"].append((s, -1, None))
        elif mism is None:
            out["counter_mismatch"] += int(x.counters != y.counters)
            out["frames_mismatch"] += int(any(ex.frames != ey.frames or ex.durations != ey.durations
                                              for ex, ey in zip(x.nbest, y.nbest)))
        else:
            sc = [e.score for e in y.nbest]
            margin = sc[mism] - sc[mism + 1] if mism + 1 < len(sc) else None
            out["mismatch"].append((s, mism, margin))
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--only", default="c1,c2,c3,c4,c5,bench")
    p.add_argument("--sample", type=int, default=16)
    a = p.parse_args()
    orc = Oracle()
    for name in a.only.split(","):
        t0 = time.time()
        w = workload(name)
        idx = sorted(set(np.linspace(0, w.B - 1, min(a.sample, w.B)).round().astype(int).tolist()))
        enc = w.frames()
        dec = B200Decoder(w.model)
        olm = None
        if w.arpa is not None:
            dec.set_lm(w.arpa)
            olm = orc.lm(w.arpa, synthetic_vocabulary(w.model.spec.vocab_size))
        setup = time.time() - t0
        for algo_name, algo, K in list(w.runs) + [("greedy", _abi.ALGO_GREEDY, w.runs[0][2])]:
            cfg = w.config(K, return_nbest=4)
            t1 = time.time()
            got = dec.decode(algo, enc, [w.T] * w.B, cfg)
            t2 = time.time()
            got.streams = [got.streams[i] for i in idx]
            want = orc.decode(w.model, cfg, algo, enc[idx], [w.T] * len(idx), lm=olm)
            t3 = time.time()
            r = compare(got, want)
            r.update(config=name, algo=algo_name, beam=K, B=w.B, T=w.T, streams=len(idx),
                     tokens=float(np.mean([len(s.nbest[0].tokens) for s in want.streams])),
                     gpu_s=round(t2 - t1, 2), oracle_s=round(t3 - t2, 2), setup_s=round(setup, 1))
            print(json.dumps(r), flush=True)
        dec.close()


if __name__ == "__main__":
    main()
