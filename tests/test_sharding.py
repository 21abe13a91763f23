"""Multi-process (gloo, world size 2, CPU) coverage of the utterance-sharded
multi-GPU path: the shard/gather logic bench.py and users run under torchrun,
and that decoding shards independently reproduces the full-batch decode
(the batch-invariance property the sharding relies on; checked with the CPU
oracle as the per-rank decoder)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_00185_b200 import _abi
from paper_2506_00185_b200.sharding import gather_results, shard_bounds, shard_indices


def test_shard_bounds_cover_everything():
    for total in (1, 7, 128, 1024):
        for world in (1, 2, 4, 8):
            spans = [shard_bounds(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_shard_indices_balanced_partition():
    rng = np.random.default_rng(0)
    lens = rng.integers(100, 1500, size=1000)
    parts = [shard_indices(lens, 8, r) for r in range(8)]
    allidx = np.sort(np.concatenate(parts))
    assert np.array_equal(allidx, np.arange(1000))
    frames = [lens[p].sum() for p in parts]
    assert max(frames) / min(frames) < 1.01


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.cpu import Oracle
        from tests.helpers import instance
        model, enc, lens = instance(7, V=16, B=6, T=10)
        idx = shard_indices(lens, world, rank)
        cfg = _abi.DecodeConfig(beam=3, max_len=20, return_nbest=2)
        res = Oracle().decode(model, cfg, _abi.ALGO_ALSD, enc[idx], [lens[i] for i in idx])
        local = [[(e.tokens, e.score) for e in s.nbest] for s in res.streams]
        full = gather_results(local, idx, len(lens))
        if rank == 0:
            out_q.put(full)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_and_gather_equals_full_batch(oracle):
    from tests.helpers import instance
    model, enc, lens = instance(7, V=16, B=6, T=10)
    cfg = _abi.DecodeConfig(beam=3, max_len=20, return_nbest=2)
    ref = oracle.decode(model, cfg, _abi.ALGO_ALSD, enc, lens)
    want = [[(e.tokens, e.score) for e in s.nbest] for s in ref.streams]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == want


def _gpu_worker(rank, world, port, out_q):
    """One rank of the utterance-sharded GPU path: its own B200 decoder context
    (both ranks share cuda:0 on a one-GPU box; gloo carries the gather)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_00185_b200.decoder import B200Decoder
        from tests.helpers import instance
        model, enc, lens = instance(11, kind=_abi.PRED_LSTM, V=24, D=16, J=32, H=32, E=8, B=7, T=16,
                                    durations=(0, 1, 2), precision=_abi.PREC_BF16)
        idx = shard_indices(lens, world, rank)
        cfg = _abi.DecodeConfig(beam=4, max_len=30, return_nbest=2)
        dec = B200Decoder(model, device=0)
        res = dec.decode(_abi.ALGO_AES, enc[idx], [lens[i] for i in idx], cfg)
        local = [[(e.tokens, e.score, e.frames, e.durations) for e in s.nbest] for s in res.streams]
        full = gather_results(local, idx, len(lens))
        dec.close()
        if rank == 0:
            out_q.put(full)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gpu_shard_and_gather_equals_full_batch():
    """The multi-GPU path end to end on the GPU library: two ranks decode
    disjoint length-balanced shards with their own contexts and gather on rank
    0; the result equals one full-batch GPU decode bitwise (batch invariance)."""
    from paper_2506_00185_b200.decoder import B200Decoder
    from tests.helpers import instance
    model, enc, lens = instance(11, kind=_abi.PRED_LSTM, V=24, D=16, J=32, H=32, E=8, B=7, T=16,
                                durations=(0, 1, 2), precision=_abi.PREC_BF16)
    cfg = _abi.DecodeConfig(beam=4, max_len=30, return_nbest=2)
    dec = B200Decoder(model)
    ref = dec.decode(_abi.ALGO_AES, enc, lens, cfg)
    dec.close()
    want = [[(e.tokens, e.score, e.frames, e.durations) for e in s.nbest] for s in ref.streams]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == want
