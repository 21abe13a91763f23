"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
compiled in place (oracle/_ref/libtbeam_ref.so).  Run in the build container
(the reference tree is not on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed):
  kats.json        update_hash / logadd / log1mexp / prune_topk known answers
  lm_queries.json  NGramLm score_vocab / score_token / score_eos / state
                   on lm_v40_o3.arpa (make_random_consistent_arpa seed 5, V=40, order 3)
  decodes.json     alsd_pp / reference_beam(kAes) / aes_pp / greedy_batched
                   results on seeded synthetic instances (weights from
                   paper_2506_00185_b200.model, seeds recorded), scalar kernels
"""
import hashlib
import json
import os
import sys

os.environ["TBEAM_KERNELS"] = "scalar"
os.environ["TBEAM_THREADS"] = "1"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle.cpu import REF_AES_PP, REF_ALSD_PP, REF_BEAM_AES, REF_GREEDY, RefLib  # noqa: E402
from paper_2506_00185_b200 import _abi  # noqa: E402
from tests.helpers import instance  # noqa: E402

M61 = (1 << 61) - 1

# (name, seed, kind, V, B, T, cfg kwargs, lm)
DECODE_CASES = [
    ("stateless_v12_k4", 1, _abi.PRED_STATELESS, 12, 3, 12, dict(beam=4, max_len=24, return_nbest=3), None),
    ("stateless_v6_k8_n1", 2, _abi.PRED_STATELESS, 6, 3, 10, dict(beam=8, max_len=16, return_nbest=4), None),
    ("lstm_v9_k3", 3, _abi.PRED_LSTM, 9, 3, 9, dict(beam=3, max_len=20, return_nbest=2), None),
    ("stateless_v40_lm_late_scored", 4, _abi.PRED_STATELESS, 40, 2, 10,
     dict(beam=4, max_len=30, return_nbest=2,
          fusion=dict(lam=0.6, blank_mode=_abi.BLANK_SCORED, pruning=_abi.PRUNE_LATE, eos_enabled=True)),
     "lm_v40_o3.arpa"),
    ("stateless_v40_lm_early_omit", 5, _abi.PRED_STATELESS, 40, 2, 10,
     dict(beam=4, max_len=30, return_nbest=2,
          fusion=dict(lam=0.4, blank_mode=_abi.BLANK_OMIT, pruning=_abi.PRUNE_EARLY, eos_enabled=False)),
     "lm_v40_o3.arpa"),
]

REF_ENTRY = {"alsd_pp": REF_ALSD_PP, "reference_beam_aes": REF_BEAM_AES, "aes_pp": REF_AES_PP,
             "greedy_batched": REF_GREEDY}


def make_cfg(kw):
    kw = dict(kw)
    fus = kw.pop("fusion", None)
    cfg = _abi.DecodeConfig(**kw)
    if fus:
        cfg.fusion = _abi.FusionConfig(lam=fus["lam"], blank_mode=fus["blank_mode"],
                                       pruning=fus["pruning"], eos_enabled=fus["eos_enabled"])
    return cfg


def weights_digest(model) -> str:
    h = hashlib.sha256()
    for k in sorted(model.weights):
        h.update(k.encode())
        h.update(model.weights[k].tobytes())
    return h.hexdigest()[:16]


def main():
    ref = RefLib()
    rng = np.random.default_rng(2024)
    # ---- KATs ---------------------------------------------------------------
    kats = {"update_hash": [], "logadd": [], "log1mexp": [], "prune_topk": []}
    for h, tok, base, mod in [(0, 5, 1_000_003, M61), (6, 7, 1_000_003, M61), (0, 0, 1_000_003, M61),
                              (M61 - 1, 1023, 1_000_003, M61), (12345, 3, 7, 1), (99, 4, 7, 97)]:
        kats["update_hash"].append([h, tok, base, mod, ref.update_hash(h, tok, base, mod)])
    for _ in range(200):
        h = int(rng.integers(0, M61))
        tok = int(rng.integers(0, 8193))
        kats["update_hash"].append([h, tok, 1_000_003, M61, ref.update_hash(h, tok)])
    for a, b in [(-1.0, -2.0), (-np.inf, -3.0), (-3.0, -np.inf), (0.0, 0.0), (-700.0, -1.0)]:
        kats["logadd"].append([a, b, ref.logadd(a, b)])
    for x in [-1e-12, -0.1, -0.69, -0.7, -5.0, -50.0, 0.0]:
        kats["log1mexp"].append([x, ref.log1mexp(x)])
    cases = [[3.0, 1.0, 2.0, -np.inf], [-np.inf, 1.0, -np.inf, -np.inf], [1.0, 1.0, 1.0, 0.5],
             [2.0, 2.0, 5.0, 2.0, 5.0, 2.0]]
    for _ in range(40):
        n = int(rng.integers(4, 40))
        v = np.round(rng.standard_normal(n), 1)  # ties on purpose
        v[rng.random(n) < 0.2] = -np.inf
        cases.append(v.tolist())
    for c in cases:
        for k in sorted({1, 2, min(4, len(c)), len(c)}):
            idx, sc = ref.prune_topk(c, k)
            kats["prune_topk"].append([c, k, idx.tolist(), sc.tolist()])
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats, f)

    # ---- LM queries -----------------------------------------------------------
    arpa = open(os.path.join(HERE, "lm_v40_o3.arpa")).read()
    lm = ref.lm(arpa, 40)
    hists = [[], [0], [3], [3, 7], [5, 5, 5], [39, 0, 1], [12, 30, 12, 30]]
    hists += [rng.integers(0, 40, size=int(rng.integers(1, 6))).tolist() for _ in range(12)]
    lmq = {"arpa": "lm_v40_o3.arpa", "vocab": 40, "order": ref.lib.ref_lm_order(lm.ptr),
           "nodes": int(ref.lib.ref_lm_num_nodes(lm.ptr)), "queries": []}
    for hst in hists:
        row = ref.lm_score_vocab(lm, hst, 40)
        lmq["queries"].append({
            "hist": hst, "state": ref.lm_state(lm, hst), "vocab_row": row.tolist(),
            "tokens": {str(t): ref.lm_score_token(lm, hst, t) for t in (0, 7, 19, 39)},
            "eos": ref.lm_score_eos(lm, hst)})
    with open(os.path.join(HERE, "lm_queries.json"), "w") as f:
        json.dump(lmq, f)

    # ---- decodes --------------------------------------------------------------------
    out = []
    for name, seed, kind, V, B, T, kw, lmfile in DECODE_CASES:
        model, enc, lens = instance(seed, kind=kind, V=V, B=B, T=T)
        cfg = make_cfg(kw)
        rlm = ref.lm(open(os.path.join(HERE, lmfile)).read(), V) if lmfile else None
        case = {"name": name, "seed": seed, "kind": kind, "V": V, "B": B, "T": T, "lengths": lens,
                "cfg": kw, "lm": lmfile, "weights_sha": weights_digest(model), "results": {}}
        for entry, which in REF_ENTRY.items():
            c = make_cfg(kw)
            if entry == "aes_pp":
                c.aes_slot_donated_quirk = True
            r = ref.decode(which, model, c, enc, lens, lm=rlm)
            case["results"][entry] = [
                {"nbest": [{"tokens": e.tokens, "score": e.score} for e in s.nbest],
                 "counters": s.counters} for s in r.streams]
        out.append(case)
    with open(os.path.join(HERE, "decodes.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
