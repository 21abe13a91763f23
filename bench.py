#!/usr/bin/env python
"""Benchmark: RTFx of batched ALSD++ beam search (beam 4, B=128 per GPU) on
the B200 kernels, with AES++ and same-kernel greedy beside it.

Workload (BASELINE.json metric "RTFx ... ALSD++/AES++ beam=4 B=128; beam/greedy
time ratio", on config 2's model shape): RNN-T, LSTM prediction network H=640,
joint 640, V=1024, encoder width D=640, T=500 frames per utterance, 80 ms
frames (RTFx = audio seconds / wall seconds), synthetic N(0,1) encoder frames,
seeded random-init weights.  A step = one full decode of the batch (encoder
projection + the whole per-frame search loop + n-best backtrace), which is one
CUDA-graph launch.

  value   device-resident (inputs already in HBM), CUDA events on the launch
          stream, max over ranks; inputs (164 MB/GPU) exceed the 126 MB L2.
  e2e     same metric through the public C-ABI call with pinned HOST buffers:
          H2D of the step's encoder frames + D2H of the n-best every step.
  roofline  the joint kernel (dominant family), FLOPs of the scored rows per
          launch / its event-timed average launch duration (instrumented run).
  cpu_baseline  the unmodified reference decoder (oracle/_ref) on the host
          cores, bounded sample of the same workload.

Multi-GPU: one process per GPU (torchrun), utterance-sharded (weak scaling,
128 utterances per GPU), no collective in the data path; the MAX of the
per-rank step times is taken with one NCCL all-reduce outside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

FRAME_SEC = 0.08
WORKLOAD = dict(vocab=1024, enc_dim=640, joint_dim=640, lstm_hidden=640, emb_dim=640,
                frames=500, batch=128, beam=4, logit_scale=4.0, blank_bias=None, seed=1, peaky=True)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--precision", default=os.environ.get("TBEAM_BENCH_PREC", "bf16"),
                   choices=["fp32", "bf16"])
    p.add_argument("--batch", type=int, default=WORKLOAD["batch"])
    p.add_argument("--frames", type=int, default=WORKLOAD["frames"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def make_model(precision: str):
    from paper_2506_00185_b200 import _abi
    from paper_2506_00185_b200.model import SyntheticTransducer, TransducerSpec
    w = WORKLOAD
    spec = TransducerSpec(vocab_size=w["vocab"], enc_dim=w["enc_dim"], joint_dim=w["joint_dim"],
                          pred_kind=_abi.PRED_LSTM, lstm_hidden=w["lstm_hidden"], emb_dim=w["emb_dim"],
                          precision=_abi.PREC_BF16 if precision == "bf16" else _abi.PREC_FP32,
                          logit_scale=w["logit_scale"], blank_bias=w["blank_bias"], seed=w["seed"],
                          peaky=w["peaky"])
    return SyntheticTransducer(spec)


def workload_config(args, n_gpus):
    w = WORKLOAD
    return {"workload": "RNN-T ALSD++ beam 4 (AES++ and same-kernel greedy beside), LSTM pred-net "
                        f"H={w['lstm_hidden']}, joint {w['joint_dim']}, V={w['vocab']}, D={w['enc_dim']}, "
                        f"B={args.batch}/GPU, T={args.frames} frames x 80 ms, no LM",
            "global_batch": args.batch * n_gpus, "frames": args.frames, "beam": w["beam"],
            "parallelism": f"utterance-sharded dp{n_gpus}", "l2": "inputs larger than L2 (164 MB/GPU)",
            "model_seed": w["seed"], "logit_scale": w["logit_scale"],
            "model": "peaky synthetic transducer (latent-alignment encoder frames, token-suppressing "
                     "prediction network; model.py)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference_rtfx(model, enc, frames, count, threads, which=None):
    """The reference's own CPU decoder (oracle/_ref; else the oracle port) on
    `count` utterances with `threads` workers; returns (rtfx, wall, kind)."""
    from paper_2506_00185_b200 import _abi
    from oracle.cpu import REF_ALSD_PP, REF_SO, Oracle, RefLib
    os.environ.setdefault("TBEAM_THREADS", "1")
    cfg = _abi.DecodeConfig(beam=WORKLOAD["beam"])
    lens = [frames] * count
    if os.path.exists(REF_SO):
        ref = RefLib()
        wall = ref.decode_pool(REF_ALSD_PP if which is None else which, model, cfg, enc[:count], lens,
                               count, threads)
        kind = "reference"
    else:
        from concurrent.futures import ThreadPoolExecutor
        o = Oracle()
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda b: o.decode(model, cfg, _abi.ALGO_ALSD, enc[b:b + 1], [frames]), range(count)))
        wall = time.perf_counter() - t0
        kind = "port"
    return count * frames * FRAME_SEC / wall, wall, kind


def run_reference_arm(args):
    """--impl reference: the reference CPU path on all host threads, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    model = make_model("fp32")
    cores = cpu_cores()
    frames = args.frames
    count = max(1, min(cores, 64))
    enc = model.encoder_frames(1000, count, frames)
    for _ in range(args.warmup):
        cpu_reference_rtfx(model, enc, min(frames, 50), min(count, cores), cores)
    walls = []
    kind = "reference"
    for _ in range(args.steps):
        rtfx, wall, kind = cpu_reference_rtfx(model, enc, frames, count, cores)
        walls.append(wall)
    wall = statistics.mean(walls)
    value = count * frames * FRAME_SEC / wall
    cfg = workload_config(args, args.gpus)
    print(json.dumps({
        "impl": "reference", "metric": "RTFx (audio-sec decoded / sec), ALSD++ beam 4",
        "value": value, "unit": "audio-sec/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "audio-sec/s", "cores": cores, "kind": kind,
                         "sample": f"{count} utterances x {frames} frames per step, B=1 sessions on a "
                                   f"{cores}-thread pool, AVX2 kernels"},
        "e2e": {"value": value, "unit": "audio-sec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch
    from paper_2506_00185_b200 import _abi
    from paper_2506_00185_b200.decoder import B200Decoder
    from paper_2506_00185_b200.model import synthetic_encoder_frames

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    B, T = args.batch, args.frames
    model = make_model(args.precision)
    enc_np = model.encoder_frames(1000 + rank, B, T)
    lens_np = np.full(B, T, np.int32)
    enc = torch.from_numpy(enc_np).to(dev)
    lens = torch.from_numpy(lens_np).to(dev)
    dec = B200Decoder(model, device=local)
    # a dedicated stream: the library launches on it and the CUDA events are
    # recorded on it (torch's legacy default stream would be a different one)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    assert sptr != 0
    cfg = _abi.DecodeConfig(beam=WORKLOAD["beam"])

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def timed(algo, steps, warmup):
        dec.prepare(algo, cfg, B, T)
        for _ in range(warmup):
            dec.decode_device(enc.data_ptr(), lens.data_ptr(), sptr)
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            dec.decode_device(enc.data_ptr(), lens.data_ptr(), sptr)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    audio = world * B * T * FRAME_SEC
    with ClockSampler(local) as clk:
        ms_alsd = timed(_abi.ALGO_ALSD, args.steps, args.warmup)
    res = dec.fetch(B, 1, cfg.max_len, sptr)
    launches = dec.launch_stats()
    tok_rate = float(np.mean([len(s.nbest[0].tokens) for s in res.streams])) / T
    rounds_alsd = launches["rounds"]
    ms_aes = timed(_abi.ALGO_AES, max(2, args.steps // 2), 2)
    dec.fetch(B, 1, cfg.max_len, sptr)
    rounds_aes = dec.launch_stats()["rounds"]
    ms_greedy = timed(_abi.ALGO_GREEDY, max(2, args.steps // 2), 2)
    g_res = dec.fetch(B, 1, cfg.max_len, sptr)
    rounds_greedy = dec.launch_stats()["rounds"]
    g_tok_rate = float(np.mean([len(s.nbest[0].tokens) for s in g_res.streams])) / T

    # ---- e2e through the public API with pinned host buffers --------------------
    enc_host = torch.from_numpy(enc_np).pin_memory()
    from paper_2506_00185_b200._abi import ResultBuffers
    import ctypes as C
    rb = ResultBuffers(B, 1, cfg.max_len)
    ccfg = cfg.to_c(_abi.ALGO_ALSD)
    lens_c = np.ascontiguousarray(lens_np)

    def e2e_once():
        rc = dec.lib.tbeam_decode(dec.ctx, C.byref(ccfg), C.c_void_p(enc_host.data_ptr()), 0,
                                  lens_c.ctypes.data_as(C.POINTER(C.c_int32)), B, T, C.byref(rb.c),
                                  C.c_void_p(sptr))
        assert rc == 0, dec.lib.tbeam_last_error()
    for _ in range(2):
        e2e_once()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_once()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = B * T * WORKLOAD["enc_dim"] * 4 + B * 4
    d2h = B * (4 + 4 + 8 + 3 * 4 * cfg.max_len + 5 * 8)

    # ---- instrumented run: per-kernel-family device time ------------------------------
    dec.prepare(_abi.ALGO_ALSD, cfg, B, T)
    prof = dec.profile_device(enc.data_ptr(), lens.data_ptr(), sptr)
    J, V, ND = WORKLOAD["joint_dim"], WORKLOAD["vocab"], 0
    n_joint = max(1, prof["launches"]["joint"])
    joint_ms = prof["ms"]["joint"] / n_joint
    flops_per_launch = prof["scored_rows"] / n_joint * 2.0 * J * (V + 1 + ND)
    total_prof = sum(prof["ms"].values())
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("bf16_tflops_sustained", 1405.3)
    achieved = flops_per_launch / (joint_ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "joint_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.precision)
        except Exception:
            traffic = None

    # ---- CPU baseline (rank 0, N=1) -----------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = cpu_cores()
        # bounded sample: ~4 utterances per host thread x 250 frames (10-30 s of
        # CPU work on a 16-core host)
        count = max(1, min(4 * cores, 128))
        cframes = min(T, 250)
        cmodel = make_model("fp32")
        cenc = cmodel.encoder_frames(1000, count, cframes)
        rtfx, wall, kind = cpu_reference_rtfx(cmodel, cenc, cframes, count, cores)
        cpu = {"value": rtfx, "unit": "audio-sec/s", "cores": cores, "kind": kind,
               "sample": f"ALSD++ beam 4, {count} utterances x {cframes} frames (same model), B=1 sessions "
                         f"on a {cores}-thread pool, AVX2 kernels, wall {wall:.1f}s"}

    value = audio / (ms_alsd * 1e-3)
    out = {
        "metric": "RTFx (audio-sec decoded / sec), ALSD++ beam 4, B=128 per GPU",
        "value": value, "unit": "audio-sec/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_alsd, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16" if args.precision == "bf16" else "fp32",
        "data": "synthetic: peaky synthetic transducer (seeded structured random weights, latent-alignment encoder frames; model.py)",
        "config": workload_config(args, world),
        "aes_pp": {"value": audio / (ms_aes * 1e-3), "ms_per_step": ms_aes, "rounds": rounds_aes},
        "greedy": {"value": audio / (ms_greedy * 1e-3), "ms_per_step": ms_greedy, "rounds": rounds_greedy,
                   "tokens_per_frame": g_tok_rate},
        "beam_greedy_time_ratio": {"alsd_pp": ms_alsd / ms_greedy, "aes_pp": ms_aes / ms_greedy},
        "search_stats": {"alsd_rounds": rounds_alsd, "alsd_tokens_per_frame": tok_rate,
                         "alsd_scored_rows": prof["scored_rows"]},
        "e2e": {"value": audio / e2e_s, "unit": "audio-sec/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "roofline": {"bound": "tensor", "kernel": "joint", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                     "flops_per_launch": flops_per_launch, "avg_launch_ms": joint_ms,
                     "share_of_step": prof["ms"]["joint"] / total_prof if total_prof else None},
        "kernel_profile_ms_per_decode": {k: round(v, 4) for k, v in prof["ms"].items()},
        "kernel_launches_per_decode": prof["launches"],
        "gpu_launches": int(launches["launches"]) * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(out))
    dec.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
