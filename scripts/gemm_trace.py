"""Phase breakdown of the tensor-core GEMM launches (CTA (0,0) clock64 trace)
for one host-driven decode of the bench workload; one GEMM family at a time
via --only (joint|gates|proj)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_00185_b200 import _abi  # noqa: E402
from paper_2506_00185_b200.decoder import B200Decoder  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 100
config = sys.argv[2] if len(sys.argv) > 2 else None  # a workloads.py config
from paper_2506_00185_b200.workloads import workload  # noqa: E402
w = workload(config or "bench")
model = w.model
B, beam, algo = w.B, w.runs[0][2], w.runs[0][1]
frames = min(frames, w.T)
fusion = w.fusion
enc = torch.from_numpy(w.frames(range(B), T=frames)).cuda()
lens = torch.full((B,), frames, dtype=torch.int32, device="cuda")
dec = B200Decoder(model)
if w.arpa is not None:
    dec.set_lm(w.arpa)
lib = dec.lib
lib.tbeam_debug_gemm_trace.argtypes = [C.c_int32, C.POINTER(C.c_int64)]
cfg = _abi.DecodeConfig(beam=beam, fusion=fusion)
out = (C.c_int64 * (40 + 1024 * 32))()
lib.tbeam_debug_gemm_trace(1, out)  # baked into the plan captured by prepare
dec.prepare(algo, cfg, B, frames)
s = torch.cuda.Stream()
dec.decode_device(enc.data_ptr(), lens.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
lib.tbeam_debug_gemm_trace(1, out)  # reset after the warm-up
dec.decode_device(enc.data_ptr(), lens.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
lib.tbeam_debug_gemm_trace(0, out)
import numpy as np  # noqa: E402
sel16 = np.frombuffer(out, dtype=np.int64)[40:].reshape(1024, 32).astype(np.float64)
sel = sel16[:, :8]
live = sel[:, 0] > 0
avg = sel[live] / sel[live, 0:1]
tot = avg[:, 7] + avg[:, 6]
worst = int(np.argmax(tot))
names = ["combine", "prefix", "cand/merge/rank", "expand", "state"]
print("select per-CTA avg cycles (mean over CTAs | slowest CTA %d):" % np.flatnonzero(live)[worst])
for k, nm in enumerate(names):
    print(f"  {nm:16s} {avg[:, k + 1].mean():8.0f} | {avg[worst, k + 1]:8.0f}")
print(f"  {'pred-stage':16s} {(avg[:, 7] - avg[:, 1:6].sum(1)).mean():8.0f} | {avg[worst, 7] - avg[worst, 1:6].sum():8.0f}")
print(f"  {'stream total':16s} {avg[:, 7].mean():8.0f} | {avg[worst, 7]:8.0f}   max {avg[:, 7].max():.0f}")
print(f"  {'tail':16s} {avg[:, 6].mean():8.0f} | {avg[worst, 6]:8.0f}")
sub = sel16[live][:, 8:] / sel[live, 0:1]
print("  combine sub-phases (slot 0, mean): stage-loads %.0f  max+sum+lse %.0f  dur %.0f  merge %.0f  fuse %.0f  combine-total %.0f"
      % tuple(sub.mean(0)[:6]))
if sub.mean(0)[11:15].sum() > 0:
    print("  prefix split: edges %.0f  sort %.0f  donor values %.0f  serial application %.0f  (edges per CTA-round %.1f)"
          % (tuple(sub.mean(0)[11:15]) + (sub.mean(0)[15],)))
print("  phase-3 split: recombination %.0f  rank %.0f (rest of cand/merge/rank: the prefix-to-recombination gap)"
      % tuple(sub.mean(0)[6:8]))
print("  expand split: select+trie %.0f  pool %.0f  state machine %.0f  (+ 'expand' above = atomics issue)"
      % tuple(sub.mean(0)[8:11]))
n0 = max(out[0], 1)
print(f"joint epilogue sub-phases: loads+LM+sync={out[33]/n0:.0f} chunks={out[34]/n0:.0f}"
      + (f" chunks-again(warm)={out[35]/n0:.0f}" if out[35] else ""))
if out[36]:  # fp32 tensor-core joint (tc_gemm_s3): CTA (0,0,0)'s wrapper phases
    nl = max(out[39], 1)
    print(f"s3 joint wrapper: tmem+fp64={out[36]/n0:.0f} partial+ticket={out[37]/n0:.0f} "
          f"reduce={out[38]/nl:.0f} (last in {out[39]}/{out[0]} launches)")
for k, name in enumerate(("joint", "gates", "proj")):
    o = out[8 * k: 8 * k + 8]
    n = max(o[0], 1)
    print(f"{name:8s} CTA(0,0) launches={o[0]:5d} avg cycles: prologue={o[1]/n:7.0f} dep_wait={o[2]/n:7.0f} "
          f"mainloop={o[3]/n:7.0f} [first stage {o[5]/n:6.0f}, last stage {o[6]/n:6.0f}] epilogue={o[4]/n:7.0f}")
