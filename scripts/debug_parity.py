"""Localise a GPU-vs-oracle divergence on a BASELINE config: decode chosen
streams inside batches of different compositions / feature toggles and report
which variants agree with the oracle.  Measurement aid, not a test.

  python scripts/debug_parity.py --config c5 --streams 205,614 [--pad 0,160,1024]
         [--frames 1500] [--algo aes] [--beam 16] [--lam 0.5] [--max-len 256]
"""
import argparse
import json
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
p.add_argument("--streams", default="205,614")
p.add_argument("--pad", default="0", help="comma list: batch = streams + the first N others")
p.add_argument("--frames", type=int, default=None)
p.add_argument("--algo", default=None, choices=[None, "alsd", "aes", "greedy"])
p.add_argument("--beam", type=int, default=None)
p.add_argument("--lam", type=float, default=None)
p.add_argument("--max-len", type=int, default=256)
p.add_argument("--nbest", type=int, default=4)
p.add_argument("--quirk", type=int, default=0)
p.add_argument("--prefix", type=int, default=1)
p.add_argument("--blank", default=None, choices=[None, "omit", "scored"])
p.add_argument("--prune", default=None, choices=[None, "early", "late"])
p.add_argument("--merge", default="logadd", choices=["logadd", "max"])
p.add_argument("--len", type=int, default=None, help="decode only the first LEN frames")
a = p.parse_args()

w = workload(a.config)
T = a.frames or w.T
algo = {"alsd": _abi.ALGO_ALSD, "aes": _abi.ALGO_AES, "greedy": _abi.ALGO_GREEDY,
        None: w.runs[0][1]}[a.algo]
K = a.beam or w.runs[0][2]
fusion = w.fusion
if a.lam is not None or a.blank or a.prune:
    fusion = _abi.FusionConfig(lam=fusion.lam if a.lam is None else a.lam,
                               blank_mode={"omit": _abi.BLANK_OMIT, "scored": _abi.BLANK_SCORED,
                                           None: fusion.blank_mode}[a.blank],
                               pruning={"early": _abi.PRUNE_EARLY, "late": _abi.PRUNE_LATE,
                                        None: fusion.pruning}[a.prune],
                               eos_enabled=fusion.eos_enabled)
cfg = _abi.DecodeConfig(beam=K, fusion=fusion, max_len=a.max_len, return_nbest=a.nbest)
cfg.aes_slot_donated_quirk = bool(a.quirk)
cfg.aes_prefix_search = bool(a.prefix)
cfg.merge_mode = _abi.MERGE_MAX if a.merge == "max" else _abi.MERGE_LOGSUMEXP
L = a.len or T
chosen = [int(x) for x in a.streams.split(",")]
orc = Oracle()
olm = orc.lm(w.arpa, synthetic_vocabulary(w.model.spec.vocab_size)) if (w.arpa and fusion.lam > 0) else None
want = orc.decode(w.model, cfg, algo, w.frames(chosen, T), [L] * len(chosen), lm=olm)
dec = B200Decoder(w.model)
if w.arpa:
    dec.set_lm(w.arpa)
for pad in [int(x) for x in a.pad.split(",")]:
    others = [i for i in range(w.B) if i not in chosen][:pad]
    batch = chosen + others
    got = dec.decode(algo, w.frames(batch, T), [L] * len(batch), cfg)
    for j, s in enumerate(chosen):
        g, o = got.streams[j], want.streams[j]
        same = [e.tokens for e in g.nbest] == [e.tokens for e in o.nbest]
        d = max(abs(x.score - y.score) for x, y in zip(g.nbest, o.nbest))
        first = None
        if not same:
            for x, y in zip(g.nbest[0].tokens, o.nbest[0].tokens):
                pass
            gt, ot = g.nbest[0].tokens, o.nbest[0].tokens
            first = next((i for i in range(min(len(gt), len(ot))) if gt[i] != ot[i]), min(len(gt), len(ot)))
        print(json.dumps({"config": a.config, "T": T, "K": K, "algo": a.algo, "lam": fusion.lam, "pad": pad,
                          "batch": len(batch), "stream": s, "tokens_equal": same, "max_dscore": d,
                          "counters_equal": g.counters == o.counters, "gpu_ctr": g.counters, "orc_ctr": o.counters,
                          "first_token_diff": first,
                          "first_diff_frame": (g.nbest[0].frames[first] if first is not None and first < len(g.nbest[0].frames) else None),
                          "gpu_scores": [round(e.score, 4) for e in g.nbest],
                          "orc_scores": [round(e.score, 4) for e in o.nbest],
                          "gpu_len": [len(e.tokens) for e in g.nbest], "orc_len": [len(e.tokens) for e in o.nbest],
                          "gpu_head": [(t, f) for t, f in zip(g.nbest[0].tokens[:6], g.nbest[0].frames[:6])],
                          "orc_head": [(t, f) for t, f in zip(o.nbest[0].tokens[:6], o.nbest[0].frames[:6])]}),
              flush=True)
