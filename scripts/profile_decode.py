"""One decode of the bench workload for profilers (ncu launch lists / full
captures).  Not a benchmark: numbers printed under a profiler are not valid.

  python scripts/profile_decode.py [--frames 60] [--algo alsd|aes|greedy] [--precision bf16]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_00185_b200 import _abi  # noqa: E402
from paper_2506_00185_b200.decoder import B200Decoder  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--frames", type=int, default=60)
p.add_argument("--batch", type=int, default=128)
p.add_argument("--algo", default="alsd", choices=["alsd", "aes", "greedy"])
p.add_argument("--precision", default="bf16")
p.add_argument("--graph", type=int, default=1)
p.add_argument("--reps", type=int, default=2)
p.add_argument("--config", default=None, help="a scripts/bench_configs.py config (c1..c5) instead of the bench")
a = p.parse_args()

algo = {"alsd": _abi.ALGO_ALSD, "aes": _abi.ALGO_AES, "greedy": _abi.ALGO_GREEDY}[a.algo]
from paper_2506_00185_b200.workloads import workload  # noqa: E402
w = workload(a.config or "bench", precision=_abi.PREC_BF16 if a.precision == "bf16" else _abi.PREC_FP32)
model = w.model
beam = w.runs[0][2]
if a.config:
    a.batch = w.B
    a.frames = min(a.frames, w.T)
fusion = w.fusion
dec = B200Decoder(model)
if w.arpa is not None:
    dec.set_lm(w.arpa)
enc = torch.from_numpy(w.frames(range(a.batch), T=a.frames)).cuda()
lens = torch.full((a.batch,), a.frames, dtype=torch.int32, device="cuda")
dec.set_graph_mode(a.graph)
cfg = _abi.DecodeConfig(beam=beam, fusion=fusion)
dec.prepare(algo, cfg, a.batch, a.frames)
s = torch.cuda.Stream()
for _ in range(a.reps):
    dec.decode_device(enc.data_ptr(), lens.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
r = dec.fetch(a.batch, 1, cfg.max_len, s.cuda_stream)
print("rounds", dec.launch_stats(), "tok/frame",
      np.mean([len(x.nbest[0].tokens) for x in r.streams]) / a.frames)
