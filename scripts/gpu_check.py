"""Quick GPU-vs-oracle parity sweep with diagnostics (run on the B200 box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2506_00185_b200 import _abi
from paper_2506_00185_b200.decoder import B200Decoder
from paper_2506_00185_b200.model import (SyntheticTransducer, TransducerSpec,
                                         synthetic_encoder_frames, synthetic_vocabulary)
from oracle.cpu import Oracle, RefLib


def compare(name, a, b, tol=1e-4):
    bad = 0
    worst = 0.0
    for s in range(len(a.streams)):
        ea, eb = a.streams[s].nbest, b.streams[s].nbest
        if [e.tokens for e in ea] != [e.tokens for e in eb]:
            bad += 1
            if bad <= 2:
                print(f"  [{name}] stream {s} tokens differ:\n    gpu {[e.tokens[:20] for e in ea][:2]} {[e.score for e in ea][:2]}\n    orc {[e.tokens[:20] for e in eb][:2]} {[e.score for e in eb][:2]}")
            continue
        for x, y in zip(ea, eb):
            worst = max(worst, abs(x.score - y.score))
            if x.frames is not None and y.frames is not None and x.frames != y.frames:
                bad += 1
                print(f"  [{name}] stream {s} frames differ {x.frames[:10]} {y.frames[:10]}")
                break
    print(f"{name}: streams={len(a.streams)} token-mismatch={bad} worst|dscore|={worst:.2e} "
          f"ctr_gpu={a.streams[0].counters} ctr_orc={b.streams[0].counters}")
    return bad == 0 and worst < tol


def main():
    o = Oracle()
    ok = True
    cases = []
    for kind in (_abi.PRED_STATELESS, _abi.PRED_LSTM):
        for durs in ((), (0, 1, 2, 3, 4)):
            for prec in (_abi.PREC_FP32, _abi.PREC_BF16):
                cases.append((kind, durs, prec))
    for kind, durs, prec in cases:
        spec = TransducerSpec(vocab_size=40, enc_dim=32, joint_dim=64, pred_kind=kind,
                              context_order=2, lstm_hidden=64, emb_dim=16, durations=durs,
                              precision=prec, seed=7, blank_bias=3.0)
        m = SyntheticTransducer(spec)
        enc = synthetic_encoder_frames(11, 5, 30, 32)
        lens = [30, 25, 17, 9, 1]
        dec = B200Decoder(m)
        for algo in (_abi.ALGO_GREEDY, _abi.ALGO_ALSD, _abi.ALGO_AES):
            cfg = _abi.DecodeConfig(beam=4, max_len=40, return_nbest=2)
            t0 = time.time()
            g = dec.decode(algo, enc, lens, cfg)
            t1 = time.time()
            r = o.decode(m, cfg, algo, enc, lens)
            tol = 1e-4 if prec == _abi.PREC_FP32 else 2e-3
            ok &= compare(f"kind={kind} tdt={bool(durs)} prec={prec} algo={algo} ({(t1-t0)*1e3:.1f}ms)", g, r, tol)
    # LM fusion
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libtbeam_ref.so")):
        ref = RefLib()
        arpa = ref.random_arpa(5, 40, 3)
    else:
        arpa = open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "lm_v40_o3.arpa")).read()
    spec = TransducerSpec(vocab_size=40, enc_dim=32, joint_dim=64, seed=9, blank_bias=3.0)
    m = SyntheticTransducer(spec)
    enc = synthetic_encoder_frames(3, 4, 25, 32)
    lens = [25, 20, 13, 6]
    dec = B200Decoder(m)
    dec.set_lm(arpa)
    olm = o.lm(arpa, synthetic_vocabulary(40))
    for bm in (_abi.BLANK_OMIT, _abi.BLANK_SCORED):
        for pm in (_abi.PRUNE_EARLY, _abi.PRUNE_LATE):
            for algo in (_abi.ALGO_GREEDY, _abi.ALGO_ALSD, _abi.ALGO_AES):
                cfg = _abi.DecodeConfig(beam=4, max_len=40, return_nbest=2,
                                        fusion=_abi.FusionConfig(lam=0.6, blank_mode=bm, pruning=pm,
                                                                 eos_enabled=True))
                g = dec.decode(algo, enc, lens, cfg)
                r = o.decode(m, cfg, algo, enc, lens, lm=olm)
                ok &= compare(f"LM blank={bm} prune={pm} algo={algo}", g, r, 1e-4)
    print("ALL OK" if ok else "SOME FAILED")


if __name__ == "__main__":
    main()
