"""Synthetic transducer definition: shapes, seeded random-init weights and
encoder frames.

There are no trained checkpoints offline, so -- like the reference's seeded
``ToyModel`` (proj/src/model.cpp:305-367) -- weights are drawn from a seeded
generator.  A plain random joint is near-uniform over V+1 outcomes and makes
greedy emit >1 token per frame (SURVEY §7 "synthetic-workload degeneracy"),
so the blank logit gets a bias and the output projection a scale, tuned so
greedy emits roughly 0.3-0.4 tokens per frame.

The math the weights feed is documented in include/tbeam_b200.h.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _abi


@dataclass
class TransducerSpec:
    vocab_size: int = 128
    enc_dim: int = 256
    joint_dim: int = 256
    pred_kind: int = _abi.PRED_STATELESS
    context_order: int = 2
    lstm_hidden: int = 640
    emb_dim: int = 256
    durations: Sequence[int] = ()
    precision: int = _abi.PREC_FP32
    blank_bias: Optional[float] = None   # default: ln(V) + 2.5
    logit_scale: float = 3.0
    seed: int = 1
    # "peaky" synthetic transducer (see SyntheticTransducer): encoder frames
    # carry a latent alignment, the prediction network suppresses the token it
    # just emitted and lifts blank -- beam and greedy then emit at similar,
    # realistic rates (a plain random joint makes beam search prefer blank).
    peaky: bool = False
    event_rate: float = 0.35     # fraction of frames that carry a token
    peak_gain: float = 5.0       # gamma: encoder evidence for the frame's token
    suppress: float = 6.0        # alpha: pred-net push away from the last token
    blank_lift: float = 1.0      # beta: pred-net push towards blank
    runner_up: float = 0.6       # relative gain of a frame's competing token

    @property
    def is_tdt(self) -> bool:
        return len(self.durations) > 0

    def dims(self) -> _abi.CModelDims:
        d = _abi.CModelDims()
        d.vocab_size = self.vocab_size
        d.enc_dim = self.enc_dim
        d.joint_dim = self.joint_dim
        d.pred_kind = self.pred_kind
        d.context_order = self.context_order
        d.lstm_hidden = self.lstm_hidden if self.pred_kind == _abi.PRED_LSTM else 0
        d.emb_dim = self.emb_dim if self.pred_kind == _abi.PRED_LSTM else 0
        d.num_durations = len(self.durations)
        for i, v in enumerate(self.durations):
            d.durations[i] = int(v)
        d.precision = self.precision
        return d


class SyntheticTransducer:
    """Seeded random-init weights (fp32, row-major) for a TransducerSpec."""

    def __init__(self, spec: TransducerSpec):
        self.spec = spec
        s = spec
        rng = np.random.default_rng(s.seed)
        V, D, J = s.vocab_size, s.enc_dim, s.joint_dim
        R = V + 1

        def normal(shape, std):
            return (rng.standard_normal(shape) * std).astype(np.float32)

        w: Dict[str, np.ndarray] = {}
        w["w_enc"] = normal((J, D), 1.0 / math.sqrt(D))
        w["b_enc"] = normal((J,), 0.1)
        w["b_pred"] = normal((J,), 0.1)
        if s.peaky:
            self._peaky_weights(w, rng, normal)
            self.weights = {k: np.ascontiguousarray(v) for k, v in w.items()}
            self._c_weights = None
            self._enc_map = None
            return
        if s.pred_kind == _abi.PRED_LSTM:
            H, E = s.lstm_hidden, s.emb_dim
            w["emb"] = normal((R, E), 1.0)
            w["w_ih"] = normal((4 * H, E), 1.0 / math.sqrt(E))
            w["w_hh"] = normal((4 * H, H), 1.0 / math.sqrt(H))
            b = normal((4 * H,), 0.1)
            b[H:2 * H] += 1.0  # forget-gate bias
            w["b_lstm"] = b
            w["w_pred"] = normal((J, H), 1.5 / math.sqrt(H))
        else:
            w["pred_table"] = normal((R, J), 0.8)
        w["w_out"] = normal((R, J), s.logit_scale / math.sqrt(J))
        bias = normal((R,), 0.1)
        bb = s.blank_bias if s.blank_bias is not None else math.log(V) + 2.5
        bias[V] += np.float32(bb)
        w["b_out"] = bias
        if s.is_tdt:
            ND = len(s.durations)
            w["w_dur"] = normal((ND, J), 1.0 / math.sqrt(J))
            bd = normal((ND,), 0.1)
            # mild preference for short hops, no preference for 0
            for i, dv in enumerate(s.durations):
                bd[i] += np.float32(0.5 if dv in (1, 2) else 0.0)
            w["b_dur"] = bd
        self.weights = {k: np.ascontiguousarray(v) for k, v in w.items()}
        self._c_weights = None

    def _peaky_weights(self, w, rng, normal):
        """Structured seeded weights (same model math, include/tbeam_b200.h):
        u_k = W_out[k] / |W_out[k]|; after emitting token v the prediction
        output is d_v = clip(-alpha u_v + beta u_blank) -- the LSTM is built
        memoryless (i, o gates open, f shut, W_ih = identity on the g gate,
        W_pred = identity, emb[v] = atanh(atanh(d_v))) so h = d_v; the
        stateless table row is d_v.  Encoder frames are then drawn by
        encoder_frames() through W_enc^-1 so enc_proj points at u_k on event
        frames."""
        s = self.spec
        V, D, J = s.vocab_size, s.enc_dim, s.joint_dim
        R = V + 1
        if D != J or (s.pred_kind == _abi.PRED_LSTM and not (s.lstm_hidden == J and s.emb_dim == J)):
            raise ValueError("peaky synthetic model needs enc_dim == joint_dim (== lstm_hidden == emb_dim)")
        w_out = normal((R, J), s.logit_scale / math.sqrt(J))
        u = w_out.astype(np.float64) / np.linalg.norm(w_out.astype(np.float64), axis=1, keepdims=True)
        d = np.clip(-s.suppress * u + s.blank_lift * u[V][None, :], -0.7, 0.7)
        d[V] = np.clip(s.blank_lift * u[V], -0.7, 0.7)  # BOS: no token to suppress
        w["b_pred"] = np.zeros(J, np.float32)
        if s.pred_kind == _abi.PRED_LSTM:
            H = s.lstm_hidden
            w["emb"] = np.arctanh(np.arctanh(d)).astype(np.float32)
            w_ih = np.zeros((4 * H, H), np.float32)
            w_ih[2 * H:3 * H] = np.eye(H, dtype=np.float32)
            w["w_ih"] = w_ih
            w["w_hh"] = normal((4 * H, H), 0.02 / math.sqrt(H))
            b = np.zeros(4 * H, np.float32)
            b[0:H] = 8.0          # input gate open
            b[H:2 * H] = -8.0     # forget gate shut: memoryless
            b[3 * H:4 * H] = 8.0  # output gate open
            w["b_lstm"] = b
            w["w_pred"] = np.eye(J, dtype=np.float32)
        else:
            w["pred_table"] = d.astype(np.float32)
        w["w_out"] = w_out
        bias = normal((R,), 0.1)
        bb = s.blank_bias if s.blank_bias is not None else 0.5 * s.logit_scale * s.peak_gain
        bias[V] += np.float32(bb)
        w["b_out"] = bias
        if s.is_tdt:
            ND = len(s.durations)
            w["w_dur"] = normal((ND, J), 1.0 / math.sqrt(J))
            bd = normal((ND,), 0.1)
            # the synthetic frames carry no silence structure: hops of one
            # frame dominate (a skipped event frame loses its token)
            for i, dv in enumerate(s.durations):
                bd[i] += np.float32(6.0 if dv == 1 else 2.0 if dv == 2 else 0.0)
            w["b_dur"] = bd
        self._u = u

    def encoder_frames(self, seed: int, batch: int, frames: int,
                       successors: Optional[np.ndarray] = None) -> np.ndarray:
        """Encoder frames for this model, fp32 [batch, frames, enc_dim].  Plain
        models: N(0, 1).  Peaky models: a latent alignment -- each frame is a
        token event with probability event_rate (token uniform over V, with a
        30% chance of a runner-up token at 0.9 x the gain, so the search has
        real alternatives) -- mapped through W_enc^-1 so that enc_proj ~
        gain * u_token + noise."""
        s = self.spec
        if not s.peaky:
            return synthetic_encoder_frames(seed, batch, frames, s.enc_dim)
        return self.encoder_frames_for(seed, range(batch), frames, successors)

    def encoder_frames_for(self, seed: int, streams: Sequence[int], frames: int,
                           successors: Optional[np.ndarray] = None) -> np.ndarray:
        """Peaky encoder frames of the given stream indices: stream b draws
        from its own generator (seed, b), so any subset of a batch can be
        regenerated alone (the parity tests check sampled streams of the
        full-size BASELINE batches against the CPU oracle)."""
        s = self.spec
        V, J = s.vocab_size, s.joint_dim
        u = self._u
        if self._enc_map is None:
            w_enc = self.weights["w_enc"].astype(np.float64)
            self._enc_map = (np.linalg.inv(w_enc).T, self.weights["b_enc"].astype(np.float64))
        inv_t, b_enc = self._enc_map
        if successors is not None:
            nsucc = (successors >= 0).sum(axis=1)
        streams = list(streams)
        out = np.empty((len(streams), frames, J), np.float32)
        for i, b in enumerate(streams):
            rng = np.random.default_rng([seed, b])
            y = rng.standard_normal((frames, J)) * (0.3 / math.sqrt(J))
            ev = rng.random(frames) < s.event_rate
            k1 = rng.integers(0, V, frames)
            if successors is not None:
                # the spoken token stream follows the LM's bigrams (successors[v]
                # = continuations of v, -1 padded) so shallow fusion has text to
                # agree with -- a random LM otherwise only penalises every token
                pick = rng.integers(0, 1 << 30, frames)
                prev = -1
                for t in np.flatnonzero(ev):
                    if prev >= 0 and nsucc[prev] > 0:
                        k1[t] = successors[prev, pick[t] % nsucc[prev]]
                    prev = k1[t]
            k2 = rng.integers(0, V, frames)
            two = rng.random(frames) < 0.3
            y += np.where(ev[:, None], s.peak_gain * u[k1], 0.0)
            y += np.where((ev & two)[:, None], s.runner_up * s.peak_gain * u[k2], 0.0)
            out[i] = ((y - b_enc) @ inv_t).astype(np.float32)
        return out

    def c_weights(self) -> _abi.CModelWeights:
        if self._c_weights is None:
            cw = _abi.CModelWeights()
            for name, _ in _abi.CModelWeights._fields_:
                arr = self.weights.get(name)
                setattr(cw, name, arr.ctypes.data_as(C.POINTER(C.c_float)) if arr is not None
                        else C.POINTER(C.c_float)())
            self._c_weights = cw
        return self._c_weights

    def dims(self) -> _abi.CModelDims:
        return self.spec.dims()


def synthetic_encoder_frames(seed: int, batch: int, frames: int, enc_dim: int) -> np.ndarray:
    """enc[b, t, :] ~ N(0, 1), fp32 (BASELINE.md §3 inputs)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((batch, frames, enc_dim)).astype(np.float32)


def synthetic_vocabulary(size: int) -> List[str]:
    """Restates ``Vocabulary::synthetic`` (proj/src/model.cpp:55-75): short
    letter strings, a word-start marker on every third token."""
    out = []
    for i in range(size):
        body = []
        v = i
        while True:
            body.append(chr(ord("a") + v % 26))
            v //= 26
            if v == 0:
                break
        body = "".join(body)
        out.append("▁" + body if i % 3 == 0 else body + str(i % 10))
    return out
