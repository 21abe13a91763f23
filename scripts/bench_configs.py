"""RTFx of every BASELINE.json configuration on one B200 (device-resident
inputs, CUDA events on the launch stream, 1 warm-up + mean of 3 as the
paper's protocol), with the same-kernel greedy time beside each
beam search.  One JSON line per config; the headline bench is bench.py.

  C1 RNN-T ALSD++ K=4, stateless n=2, V=128, D=J=256, B=1, T=200 (fp32; runs on the CPU reference)
  C2 RNN-T AES++ K=4, LSTM H=640, J=640, V=1024, B=32, T=500, fp32
  C3 TDT ALSD++ and AES++ K=8, durations {0..4}, V=1024, B=128, T=1000, bf16 (LSTM pred-net)
  C4 AES++ K=8 + synthetic 4-gram LM (~1M n-grams), V=1024, scored blank, late pruning, lambda=0.5, B=128, T=500, bf16
  C5 TDT AES++ K=16, V=8192, J=640, B=1024, T=1500, LM on, bf16 (one GPU; the bench scales it over GPUs)

  python scripts/bench_configs.py [--only c1,c3] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_00185_b200 import _abi  # noqa: E402
from paper_2506_00185_b200.decoder import B200Decoder  # noqa: E402
from paper_2506_00185_b200.workloads import CONFIGS, workload  # noqa: E402


def timed(dec, algo, cfg, enc, lens, B, T, stream, reps):
    dec.prepare(algo, cfg, B, T)
    dec.decode_device(enc.data_ptr(), lens.data_ptr(), stream.cuda_stream)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        dec.decode_device(enc.data_ptr(), lens.data_ptr(), stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    r = dec.fetch(B, 1, cfg.max_len, stream.cuda_stream)
    stats = dec.launch_stats()
    toks = float(np.mean([len(s.nbest[0].tokens) for s in r.streams])) / T
    return ms, stats["rounds"], toks


def run(name, reps):
    t0 = time.time()
    w = workload(name)
    spec = w.model.spec
    B, T = w.B, w.T
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    dec = B200Decoder(w.model)
    lm_info = None
    if w.arpa is not None:
        dec.set_lm(w.arpa)
        lm_info = dec.lm_info()
    enc = torch.from_numpy(w.frames()).cuda()
    lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
    setup_s = time.time() - t0
    audio = w.audio_seconds()
    out = []
    for algo_name, algo, K in w.runs:
        cfg = w.config(K)
        ms, rounds, toks = timed(dec, algo, cfg, enc, lens, B, T, stream, reps)
        gms, grounds, gtoks = timed(dec, _abi.ALGO_GREEDY, cfg, enc, lens, B, T, stream, reps)
        out.append({"config": name, "algo": algo_name, "beam": K, "B": B, "T": T,
                    "precision": "bf16" if spec.precision == _abi.PREC_BF16 else "fp32",
                    "tdt": bool(spec.durations), "lm": lm_info,
                    "fusion": None if lm_info is None else CONFIGS[name]["fusion"],
                    "ms_per_decode": ms, "rtfx": audio / (ms * 1e-3), "rounds": rounds,
                    "tokens_per_frame": toks,
                    "greedy_ms": gms, "greedy_rtfx": audio / (gms * 1e-3), "greedy_rounds": grounds,
                    "greedy_tokens_per_frame": gtoks,
                    "beam_greedy_time_ratio": ms / gms, "setup_s": setup_s})
    dec.close()
    return out


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("--only", default="c1,c2,c3,c4,c5")
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    for name in a.only.split(","):
        for line in run(name, a.reps):
            print(json.dumps(line), flush=True)
