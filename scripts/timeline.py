"""Device-wide launch timeline of one decode (CUDA-graph mode) of the bench
workload: per kernel the busy span (first dependency release -> last CTA exit),
the release skew and the handoff gap to the next kernel, averaged over rounds.
globaltimer stamps (tc_common.cuh tl_record); measurement aid, not a bench.

  python scripts/timeline.py [--algo alsd|aes|greedy] [--frames 100] [--precision bf16]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_00185_b200 import _abi  # noqa: E402
from paper_2506_00185_b200.decoder import B200Decoder  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--algo", default="alsd", choices=["alsd", "aes", "greedy"])
p.add_argument("--frames", type=int, default=100)
p.add_argument("--batch", type=int, default=128)
p.add_argument("--beam", type=int, default=4)
p.add_argument("--precision", default="bf16")
p.add_argument("--config", default=None, help="a workloads.py config (c1..c5) instead of the bench")
a = p.parse_args()
algo = {"alsd": _abi.ALGO_ALSD, "aes": _abi.ALGO_AES, "greedy": _abi.ALGO_GREEDY}[a.algo]
from paper_2506_00185_b200.workloads import workload  # noqa: E402
w = workload(a.config or "bench", precision=_abi.PREC_BF16 if a.precision == "bf16" else _abi.PREC_FP32)
model = w.model
if a.config:
    a.batch = w.B
    a.frames = min(a.frames, w.T)
    a.beam = w.runs[0][2] if a.algo != "greedy" else 1
fusion = w.fusion
dec = B200Decoder(model)
if w.arpa is not None:
    dec.set_lm(w.arpa)
enc = torch.from_numpy(w.frames(range(a.batch), T=a.frames)).cuda()
lens = torch.full((a.batch,), a.frames, dtype=torch.int32, device="cuda")
lib = dec.lib
lib.tbeam_debug_timeline.argtypes = [C.c_int32, C.POINTER(C.c_uint64)]
cfg = _abi.DecodeConfig(beam=a.beam, fusion=fusion)
buf = (C.c_uint64 * (4096 * 16))()
lib.tbeam_debug_timeline(1, buf)  # baked into the plan captured by prepare
dec.prepare(algo, cfg, a.batch, a.frames)
s = torch.cuda.Stream()
dec.decode_device(enc.data_ptr(), lens.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
lib.tbeam_debug_timeline(1, buf)  # reset after the warm-up
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
dec.decode_device(enc.data_ptr(), lens.data_ptr(), s.cuda_stream)
e1.record(s)
torch.cuda.synchronize()
lib.tbeam_debug_timeline(0, buf)
tl = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 4, 4).astype(np.float64)
names = ["joint", "gates", "proj", "select"]
order = [0, 3, 1, 2]  # launch order within a round
valid = tl[:, :, 3] > 0
rounds = int(valid[:, 0].sum())
print(f"decode {e0.elapsed_time(e1):.3f} ms, rounds with a joint launch: {rounds}, "
      f"{e0.elapsed_time(e1) * 1e3 / max(rounds, 1):.2f} us/round")
res = {}
for k in range(4):
    v = valid[:, k]
    if not v.any():
        continue
    span = (tl[v, k, 3] - tl[v, k, 1]) / 1e3
    skew = (tl[v, k, 2] - tl[v, k, 1]) / 1e3
    early = (tl[v, k, 1] - tl[v, k, 0]) / 1e3
    res[k] = (span.mean(), skew.mean(), early.mean(), np.median(span))
seq = [k for k in order if k in res]
gaps = {}
for i, k in enumerate(seq):
    nk = seq[(i + 1) % len(seq)]
    r = np.arange(4096)
    if nk == seq[0]:
        r2 = r + 1
    else:
        r2 = r
    ok = valid[:-1, k] & valid[np.minimum(r2, 4095)[:-1], nk]
    g = (tl[np.minimum(r2, 4095)[:-1][ok], nk, 1] - tl[:-1][ok, k, 3]) / 1e3
    gaps[k] = g.mean() if len(g) else float("nan")
tot = 0.0
for k in seq:
    sp, sk, ea, med = res[k]
    tot += sp + gaps[k]
    print(f"{names[k]:7s} busy {sp:7.2f} us (median {med:6.2f})  release skew {sk:5.2f}  "
          f"entry->release {ea:6.2f}  handoff->next {gaps[k]:6.2f} us")
print(f"sum busy+handoff per round: {tot:.2f} us")
# proj(r) -> joint(r+1) handoff split by round parity (r odd = across a
# CUDA-graph WHILE-body iteration)
for par in (0, 1):
    rr = np.arange(par, 4095, 2)
    ok = valid[rr, 2] & valid[rr + 1, 0]
    if ok.any():
        g = (tl[rr[ok] + 1, 0, 1] - tl[rr[ok], 2, 3]) / 1e3
        print(f"proj->joint handoff, round parity {par}: {g.mean():6.2f} us over {ok.sum()} rounds")
