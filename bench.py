#!/usr/bin/env python
"""Benchmark: RTFx of batched ALSD++ / AES++ beam search (beam 4, B=128 per
GPU) on the B200 kernels, with same-kernel greedy beside it -- the BASELINE.json
metric "RTFx (audio-sec decoded/sec) ALSD++/AES++ beam=4 B=128; beam/greedy
time ratio".

Workload (paper_2506_00185_b200/workloads.py "bench", config 2's model shape
at the metric's B=128): RNN-T, LSTM prediction network H=640, joint 640,
V=1024, encoder width D=640, T=500 frames per utterance, 80 ms frames (RTFx =
audio seconds / wall seconds), the peaky synthetic transducer (seeded
structured random-init weights, latent-alignment encoder frames), bf16 GEMM
operands / fp32 accumulation on tcgen05, fp64 hypothesis scores.  A step = one
full decode of the batch (encoder projection + the whole per-frame search
loop + n-best backtrace), one CUDA-graph launch.

  value   ALSD++ RTFx, device-resident inputs, CUDA events on the launch stream,
          max over ranks; inputs (164 MB/GPU) exceed the 126 MB L2.
  e2e     same metric through the public C-ABI serving calls (tbeam_stage_inputs
          + tbeam_decode_staged) with pinned HOST buffers: every step's H2D of
          its encoder frames + D2H of its n-best, the next step's copy
          overlapping the current decode.
  roofline  the dominant kernel (select: HBM-class work, SURVEY §8(d) bytes per
          launch / event-timed average launch); `roofline_kernels` lists every
          per-round kernel (joint / gates / proj on the tensor pipe).
  cpu_baseline  the unmodified reference decoder (oracle/_ref) on the host
          cores, bounded sample of the same workload.

Multi-GPU: one process per GPU.  `--gpus N` without a torchrun environment
re-launches itself under torch.distributed.run with N ranks.  Default
workload: utterance-sharded weak scaling, 128 utterances per GPU, no
collective in the data path; `--workload c5` is BASELINE config 5's strong
scaling (1024 utterances x 1500 frames, TDT AES++ beam 16, V=8192, LM on,
split over the ranks, results gathered on rank 0 after the timed region).
Step times are reduced with MAX over ranks (NCCL all-reduce, outside the
timed region; TBEAM_DIST_BACKEND=gloo for ranks sharing a GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload bench|c5]
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

FRAME_SEC = 0.08
# BASELINE.json "metric", verbatim, on both arms
METRIC = "RTFx (audio-sec decoded/sec) ALSD++/AES++ beam=4 B=128; beam/greedy time ratio"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="bench", choices=["bench", "c5"])
    p.add_argument("--precision", default=os.environ.get("TBEAM_BENCH_PREC", "bf16"),
                   choices=["fp32", "bf16"])
    p.add_argument("--batch", type=int, default=None, help="utterances per GPU (bench workload)")
    p.add_argument("--frames", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def relaunch_distributed(n: int) -> int:
    """--gpus N outside torchrun: run this script under torch.distributed.run
    with N ranks on this node (rendezvous on 127.0.0.1)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def the_workload(args, precision=None):
    from paper_2506_00185_b200 import _abi
    from paper_2506_00185_b200.workloads import workload
    prec = {"bf16": _abi.PREC_BF16, "fp32": _abi.PREC_FP32}[precision or args.precision]
    w = workload(args.workload, precision=prec)
    if args.frames:
        w.T = args.frames
    return w


def per_rank_batch(args, w, world):
    if args.workload == "bench":
        return args.batch or w.B
    return w.B  # c5: the global batch, split over the ranks


def workload_config(args, w, world):
    B = per_rank_batch(args, w, world)
    if args.workload == "bench":
        return {"workload": "RNN-T ALSD++ beam 4 (AES++ and same-kernel greedy beside), LSTM pred-net "
                            f"H=640, joint 640, V=1024, D=640, B={B}/GPU, T={w.T} frames x 80 ms, no LM",
                "global_batch": B * world, "frames": w.T, "beam": 4,
                "parallelism": f"utterance-sharded dp{world}", "l2": "inputs larger than L2 (164 MB/GPU)",
                "model_seed": 1, "logit_scale": 4.0,
                "model": "peaky synthetic transducer (latent-alignment encoder frames, token-suppressing "
                         "prediction network; workloads.py / model.py)"}
    return {"workload": "BASELINE config 5: TDT AES++ beam 16, durations {0..4}, LSTM pred-net H=640, joint 640, "
                        f"V=8192, D=640, {B} utterances x T={w.T} frames split over {world} GPU(s), consistent "
                        "4-gram LM (~1M n-grams) late pruning + scored blank, lambda 0.5",
            "global_batch": B, "frames": w.T, "beam": 16, "parallelism": f"utterance-sharded dp{world}",
            "l2": "inputs larger than L2", "model_seed": 1, "logit_scale": 4.0,
            "model": "peaky synthetic transducer (workloads.py / model.py)"}


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


def cpu_reference_rtfx(model, enc, frames, count, threads, beam=4):
    """The reference's own CPU decoder (oracle/_ref alsd_pp; else the oracle
    port) on `count` utterances with `threads` workers; returns (rtfx, wall, kind)."""
    from paper_2506_00185_b200 import _abi
    from oracle.cpu import REF_ALSD_PP, REF_SO, Oracle, RefLib
    os.environ.setdefault("TBEAM_THREADS", "1")
    cfg = _abi.DecodeConfig(beam=beam)
    lens = [frames] * count
    if os.path.exists(REF_SO):
        wall = RefLib().decode_pool(REF_ALSD_PP, model, cfg, enc[:count], lens, count, threads)
        kind = "reference"
    else:
        os.environ["ORACLE_THREADS"] = str(threads)
        t0 = time.perf_counter()
        Oracle().decode(model, cfg, _abi.ALGO_ALSD, enc[:count], lens)
        wall = time.perf_counter() - t0
        kind = "port"
    return count * frames * FRAME_SEC / wall, wall, kind


def run_reference_arm(args):
    """--impl reference: the reference CPU path on all host threads, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    w = the_workload(args, precision="fp32")
    cores = cpu_cores()
    frames = w.T
    count = max(1, min(cores, 64))
    enc = w.frames(range(count))
    for _ in range(args.warmup):
        cpu_reference_rtfx(w.model, enc[:, :min(frames, 50)].copy(), min(frames, 50), count, cores)
    walls = []
    kind = "reference"
    for _ in range(args.steps):
        _, wall, kind = cpu_reference_rtfx(w.model, enc, frames, count, cores)
        walls.append(wall)
    wall = statistics.mean(walls)
    value = count * frames * FRAME_SEC / wall
    print(json.dumps({
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "audio-sec/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.workload == "bench" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, w, world),
        "cpu_baseline": {"value": value, "unit": "audio-sec/s", "cores": cores, "kind": kind,
                         "sample": f"ALSD++ beam 4, {count} utterances x {frames} frames per step (same model, "
                                   f"fp64), B=1 sessions on a {cores}-thread pool, AVX2 kernels"},
        "e2e": {"value": value, "unit": "audio-sec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def load_json(path):
    try:
        return json.load(open(path))
    except Exception:
        return {}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch
    from paper_2506_00185_b200 import _abi
    from paper_2506_00185_b200.decoder import B200Decoder
    from paper_2506_00185_b200.sharding import gather_results, shard_bounds

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev_index = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    backend = os.environ.get("TBEAM_DIST_BACKEND", "nccl")
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    red_dev = dev if (world > 1 and backend == "nccl") else torch.device("cpu")

    def reduce_max(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=red_dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    w = the_workload(args)
    T = w.T
    if args.workload == "bench":
        B = per_rank_batch(args, w, world)
        streams = list(range(rank * B, (rank + 1) * B))  # rank r's shard of the global batch
        algo_main, K = _abi.ALGO_ALSD, 4
    else:
        s0, s1 = shard_bounds(w.B, world, rank)
        streams = list(range(s0, s1))
        B = len(streams)
        algo_main, K = _abi.ALGO_AES, 16
    enc_np = w.frames(streams)
    lens_np = np.full(B, T, np.int32)
    enc = torch.from_numpy(enc_np).to(dev)
    lens = torch.from_numpy(lens_np).to(dev)
    dec = B200Decoder(w.model, device=dev_index)
    if w.arpa is not None:
        dec.set_lm(w.arpa)
    # a dedicated stream: the library launches on it and the CUDA events are
    # recorded on it (torch's legacy default stream would be a different one)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    assert sptr != 0
    cfg = w.config(K)

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
        return reduce_max(e0.elapsed_time(e1) / steps)

    audio = w.audio_seconds(B * world if args.workload == "bench" else w.B)
    with ClockSampler(dev_index) as clk:
        ms_main = timed(algo_main, args.steps, args.warmup)
    res = dec.fetch(B, cfg.return_nbest, cfg.max_len, sptr)
    launches = dec.launch_stats()
    tok_rate = float(np.mean([len(s.nbest[0].tokens) for s in res.streams])) / T
    rounds_main = launches["rounds"]
    gathered = None
    if args.workload != "bench":
        # the final result gather (outside the timed region): rank 0 holds all
        # utterances' n-best in global order
        local_nbest = [[(e.tokens, e.score) for e in s.nbest] for s in res.streams]
        if world > 1:
            gathered = len(gather_results(local_nbest, np.asarray(streams), w.B))
        else:
            gathered = len(local_nbest)
    extra = {}
    if args.workload == "bench":
        ms_aes = timed(_abi.ALGO_AES, max(2, args.steps // 2), 2)
        dec.fetch(B, 1, cfg.max_len, sptr)
        extra["aes_pp"] = {"value": audio / (ms_aes * 1e-3), "ms_per_step": ms_aes,
                           "rounds": dec.launch_stats()["rounds"]}
    ms_greedy = timed(_abi.ALGO_GREEDY, max(2, args.steps // 2), 2)
    g_res = dec.fetch(B, 1, cfg.max_len, sptr)
    rounds_greedy = dec.launch_stats()["rounds"]
    g_tok_rate = float(np.mean([len(s.nbest[0].tokens) for s in g_res.streams])) / T
    ratio = {("alsd_pp" if algo_main == _abi.ALGO_ALSD else "aes_pp"): ms_main / ms_greedy}
    if "aes_pp" in extra:
        ratio["aes_pp"] = extra["aes_pp"]["ms_per_step"] / ms_greedy

    # ---- e2e through the public API with pinned host buffers --------------------
    # The serving path of the C-ABI: tbeam_stage_inputs copies a batch's frames
    # from pinned host memory into the next device input slot on a copy
    # stream, tbeam_decode_staged decodes it and reads the n-best back -- so
    # step i+1's H2D overlaps step i's decode.  Every step's H2D (frames +
    # lengths) and D2H (n-best) is inside the timed region.
    enc_host = torch.from_numpy(enc_np).pin_memory()
    enc_host_np = enc_host.numpy()
    lens_c = np.ascontiguousarray(lens_np)
    e2e_steps = args.steps if args.workload == "bench" else max(1, min(args.steps, 2))

    def e2e_run(steps):
        dec.stage_inputs(enc_host_np, lens_c)
        for i in range(steps):
            if i + 1 < steps:
                dec.stage_inputs(enc_host_np, lens_c)
            dec.decode_staged(algo_main, cfg, sptr, raw=True)  # n-best arrays read back, no Python objects
    e2e_run(2)
    barrier()
    t0 = time.perf_counter()
    e2e_run(e2e_steps)
    e2e_s = reduce_max((time.perf_counter() - t0) / e2e_steps)
    h2d = B * T * w.model.spec.enc_dim * 4 + B * 4
    d2h = B * cfg.return_nbest * (4 + 8 + 3 * 4 * cfg.max_len) + B * (4 + 5 * 8)

    # ---- instrumented run: per-kernel-family device time, roofline -------------------
    dec.prepare(algo_main, cfg, B, T)
    prof = dec.profile_device(enc.data_ptr(), lens.data_ptr(), sptr)
    spec = w.model.spec
    J, V, ND, H = spec.joint_dim, spec.vocab_size, len(spec.durations), spec.lstm_hidden
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    tc_peak = peaks.get("bf16_tflops_sustained", 1405.3)
    hbm_peak = peaks.get("hbm_gbs", 6553.0)
    traffic = load_json(os.path.join(ROOT, "profiles", "kernel_traffic.json")).get(
        f"{args.workload}/{args.precision}", {})
    rows = prof["scored_rows"]
    n = prof["launches"]
    total_prof = sum(prof["ms"].values())

    def avg_ms(f):
        return prof["ms"][f] / max(1, n[f])

    n_round = max(1, n["select"])
    # token rows (LSTM step): the hypotheses that emitted this round (tokens per
    # frame x frames x utterances over the decode)
    token_rows = tok_rate * T * B
    kernels = {}
    jf = rows / max(1, n["joint"]) * 2.0 * J * (V + 1 + ND)
    kernels["joint"] = {"bound": "tensor", "unit": "TFLOP/s", "work_per_launch": jf,
                        "avg_launch_ms": avg_ms("joint"), "peak": tc_peak, "family": "joint"}
    if spec.pred_kind == _abi.PRED_LSTM and n["lstm_gates"]:
        kernels["lstm_gates"] = {"bound": "tensor", "unit": "TFLOP/s", "family": "lstm_gates",
                                 "work_per_launch": token_rows / n["lstm_gates"] * 2.0 * 4 * H * H,
                                 "avg_launch_ms": avg_ms("lstm_gates"), "peak": tc_peak}
        kernels["lstm_proj"] = {"bound": "tensor", "unit": "TFLOP/s", "family": "lstm_proj",
                                "work_per_launch": token_rows / n["lstm_proj"] * 2.0 * H * J,
                                "avg_launch_ms": avg_ms("lstm_proj"), "peak": tc_peak}
    # select: SURVEY §8(d) bytes -- fused candidates K x (4 B index + 8 B score)
    # per scored row + ~32 B per hypothesis per round (token, parent, length,
    # last, hash, score) of the store
    sb = rows / n_round * K * 12.0 + B * K * 32.0
    kernels["select"] = {"bound": "hbm", "unit": "GB/s", "work_per_launch": sb, "family": "select",
                         "avg_launch_ms": avg_ms("select"), "peak": hbm_peak}
    for name, k in kernels.items():
        scale = 1e12 if k["unit"] == "TFLOP/s" else 1e9
        k["achieved"] = k["work_per_launch"] / (k["avg_launch_ms"] * 1e-3) / scale
        k["frac"] = k["achieved"] / k["peak"]
        tr = traffic.get(name)
        k["traffic"] = tr
        if tr:  # measured DRAM bytes per launch (ncu) over the event-timed launch
            k["traffic_gbs"] = tr / (k["avg_launch_ms"] * 1e-3) / 1e9
        k["share_of_instrumented_decode"] = prof["ms"][k.pop("family")] / total_prof if total_prof else None
    dom = max(kernels, key=lambda k: kernels[k]["avg_launch_ms"])
    d = kernels[dom]
    roofline = {"bound": d["bound"], "kernel": dom, "achieved": d["achieved"], "peak": d["peak"], "unit": d["unit"],
                "frac": d["frac"], "traffic": d["traffic"],
                "work_per_launch": d["work_per_launch"], "avg_launch_ms": d["avg_launch_ms"],
                "peak_source": "MEASURED_PEAKS.json " + ("hbm_gbs" if d["bound"] == "hbm" else "bf16_tflops_sustained"),
                "share_of_instrumented_decode": d["share_of_instrumented_decode"]}

    # ---- CPU baseline (rank 0, N=1) -----------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "bench":
        cores = cpu_cores()
        # bounded sample: ~4 utterances per host thread x 250 frames (10-30 s of
        # CPU work on a 16-core host)
        count = max(1, min(4 * cores, 128))
        cframes = min(T, 250)
        cw = the_workload(args, precision="fp32")
        cenc = cw.frames(range(count), T=cframes)
        rtfx, wall, kind = cpu_reference_rtfx(cw.model, cenc, cframes, count, cores)
        cpu = {"value": rtfx, "unit": "audio-sec/s", "cores": cores, "kind": kind,
               "sample": f"ALSD++ beam 4, {count} utterances x {cframes} frames (same model, fp64), B=1 "
                         f"sessions on a {cores}-thread pool, AVX2 kernels, wall {wall:.1f}s"}

    out = {
        "metric": METRIC,
        "value": audio / (ms_main * 1e-3), "unit": "audio-sec/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_main, "higher_is_better": True,
        "scaling": "weak" if args.workload == "bench" else "strong",
        "vs_baseline": None,
        "dtype": "bf16" if args.precision == "bf16" else "fp32",
        "data": "synthetic: peaky synthetic transducer (seeded structured random weights, latent-alignment "
                "encoder frames; workloads.py / model.py)",
        "config": workload_config(args, w, world),
        **extra,
        "greedy": {"value": audio / (ms_greedy * 1e-3), "ms_per_step": ms_greedy, "rounds": rounds_greedy,
                   "tokens_per_frame": g_tok_rate},
        "beam_greedy_time_ratio": ratio,
        "search_stats": {"rounds": rounds_main, "tokens_per_frame": tok_rate, "scored_rows": rows},
        "e2e": {"value": audio / e2e_s, "unit": "audio-sec/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "roofline": roofline,
        "roofline_kernels": kernels,
        "kernel_profile_ms_per_decode": {k: round(v, 4) for k, v in prof["ms"].items()},
        "kernel_launches_per_decode": prof["launches"],
        "gpu_launches": int(launches["launches"]) * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if gathered is not None:
        out["gathered_streams"] = gathered
    if rank == 0:
        print(json.dumps(out))
    dec.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
