"""Shared builders for the parity tests: seeded synthetic transducers,
encoder frames, configs, and result comparison."""
from __future__ import annotations

import numpy as np

from paper_2506_00185_b200 import _abi
from paper_2506_00185_b200.model import (SyntheticTransducer, TransducerSpec,
                                         synthetic_encoder_frames)


def instance(seed: int, kind: int = _abi.PRED_STATELESS, V: int = 12, D: int = 8, J: int = 16,
             B: int = 3, T: int = 12, n: int = 2, H: int = 12, E: int = 8, durations=(),
             precision: int = _abi.PREC_FP32, blank_bias=None, logit_scale: float = 3.0,
             ragged: bool = True):
    rng = np.random.default_rng(seed + 1000)
    bb = blank_bias if blank_bias is not None else float(np.log(V) + rng.uniform(-1.0, 2.5))
    spec = TransducerSpec(vocab_size=V, enc_dim=D, joint_dim=J, pred_kind=kind, context_order=n,
                          lstm_hidden=H, emb_dim=E, durations=tuple(durations),
                          precision=precision, seed=seed, blank_bias=bb, logit_scale=logit_scale)
    model = SyntheticTransducer(spec)
    enc = synthetic_encoder_frames(seed + 7, B, T, D)
    if ragged:
        lens = [T] + [int(x) for x in rng.integers(1, T + 1, size=B - 1)]
    else:
        lens = [T] * B
    return model, enc, lens


def same_tokens(a, b) -> bool:
    return all([e.tokens for e in x.nbest] == [e.tokens for e in y.nbest]
               for x, y in zip(a.streams, b.streams))


def max_score_diff(a, b) -> float:
    worst = 0.0
    for x, y in zip(a.streams, b.streams):
        for ex, ey in zip(x.nbest, y.nbest):
            if ex.score == ey.score:
                continue
            worst = max(worst, abs(ex.score - ey.score))
    return worst


def describe(a, b) -> str:
    out = []
    for s, (x, y) in enumerate(zip(a.streams, b.streams)):
        tx = [(e.tokens, round(e.score, 6)) for e in x.nbest]
        ty = [(e.tokens, round(e.score, 6)) for e in y.nbest]
        if tx != ty:
            out.append(f"stream {s}:\n  a={tx}\n  b={ty}")
    return "\n".join(out[:3])


def margin_ok(result, min_margin: float) -> bool:
    """True when every stream's n-best scores are separated by > min_margin
    (the parity contract: tokens must match where the margin exceeds the fp
    tolerance)."""
    for s in result.streams:
        sc = [e.score for e in s.nbest]
        for i in range(len(sc) - 1):
            if abs(sc[i] - sc[i + 1]) <= min_margin:
                return False
    return True
