"""Phase breakdown of the tensor-core GEMM launches (CTA (0,0) clock64 trace)
for one host-driven decode of the bench workload; one GEMM family at a time
via --only (joint|gates|proj)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_00185_b200 import _abi  # noqa: E402
from paper_2506_00185_b200.decoder import B200Decoder  # noqa: E402
from paper_2506_00185_b200.model import synthetic_encoder_frames  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 100
model = bench.make_model("bf16")
enc = torch.from_numpy(synthetic_encoder_frames(1000, 128, frames, 640)).cuda()
lens = torch.full((128,), frames, dtype=torch.int32, device="cuda")
dec = B200Decoder(model)
lib = dec.lib
lib.tbeam_debug_gemm_trace.argtypes = [C.c_int32, C.POINTER(C.c_int64)]
cfg = _abi.DecodeConfig(beam=4)
dec.prepare(_abi.ALGO_ALSD, cfg, 128, frames)
s = torch.cuda.Stream()
dec.decode_device(enc.data_ptr(), lens.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
out = (C.c_int64 * 48)()
lib.tbeam_debug_gemm_trace(1, out)
dec.decode_device(enc.data_ptr(), lens.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
lib.tbeam_debug_gemm_trace(0, out)
o = out[40:48]
n = max(o[0], 1)
print(f"select   CTA 0 launches={o[0]:5d} avg cycles: combine={o[1]/n:7.0f} prefix={o[2]/n:7.0f} "
      f"cand/merge/rank={o[3]/n:7.0f} expand={o[4]/n:7.0f} state={o[5]/n:7.0f} total={o[7]/n:7.0f}")
n0 = max(out[0], 1)
print(f"joint epilogue sub-phases: loads+LM+sync={out[33]/n0:.0f} chunks={out[34]/n0:.0f}")
for k, name in enumerate(("joint", "gates", "proj")):
    o = out[8 * k: 8 * k + 8]
    n = max(o[0], 1)
    print(f"{name:8s} CTA(0,0) launches={o[0]:5d} avg cycles: prologue={o[1]/n:7.0f} dep_wait={o[2]/n:7.0f} "
          f"mainloop={o[3]/n:7.0f} [first stage {o[5]/n:6.0f}, last stage {o[6]/n:6.0f}] epilogue={o[4]/n:7.0f}")
