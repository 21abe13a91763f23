"""Would two independent half-batch decodes overlap on one GPU?  Times one
B-stream decode against P decodes of B/P streams launched on P CUDA streams
at once (separate decoder contexts, same model).  Measurement aid.

  python scripts/concurrency_probe.py [--parts 2] [--algo alsd|greedy] [--reps 5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_00185_b200 import _abi  # noqa: E402
from paper_2506_00185_b200.decoder import B200Decoder  # noqa: E402
from paper_2506_00185_b200.workloads import workload  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--parts", type=int, default=2)
p.add_argument("--algo", default="alsd")
p.add_argument("--reps", type=int, default=5)
p.add_argument("--config", default="bench")
a = p.parse_args()
algo = {"alsd": _abi.ALGO_ALSD, "aes": _abi.ALGO_AES, "greedy": _abi.ALGO_GREEDY}[a.algo]
w = workload(a.config)
B, T = w.B, w.T
K = w.runs[0][2]
cfg = w.config(K)
enc = torch.from_numpy(w.frames()).cuda()
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


one = B200Decoder(w.model)
s0 = torch.cuda.Stream()
one.prepare(algo, cfg, B, T)


def run_one():
    ev = torch.cuda.Event()
    ev.record()
    s0.wait_event(ev)
    one.decode_device(enc.data_ptr(), lens.data_ptr(), s0.cuda_stream)
    ev2 = torch.cuda.Event()
    ev2.record(s0)
    torch.cuda.current_stream().wait_event(ev2)


print(f"{a.config} {a.algo} K={K}: one decode of B={B}: {timed(run_one, a.reps):.3f} ms")
P = a.parts
Bp = B // P
decs = [B200Decoder(w.model) for _ in range(P)]
ss = [torch.cuda.Stream() for _ in range(P)]
for d in decs:
    d.prepare(algo, cfg, Bp, T)


def run_parts():
    ev = torch.cuda.Event()
    ev.record()
    for i, (d, s) in enumerate(zip(decs, ss)):
        s.wait_event(ev)
        d.decode_device(enc[i * Bp:].data_ptr(), lens[i * Bp:].data_ptr(), s.cuda_stream)
    for s in ss:
        e = torch.cuda.Event()
        e.record(s)
        torch.cuda.current_stream().wait_event(e)


def run_parts_serial():
    for i, d in enumerate(decs):
        d.decode_device(enc[i * Bp:].data_ptr(), lens[i * Bp:].data_ptr(), s0.cuda_stream)
    e = torch.cuda.Event()
    e.record(s0)
    torch.cuda.current_stream().wait_event(e)


print(f"  {P} x B={Bp} concurrent on {P} streams: {timed(run_parts, a.reps):.3f} ms")
print(f"  {P} x B={Bp} one after another:        {timed(run_parts_serial, a.reps):.3f} ms")
