"""The BASELINE.json configurations as concrete synthetic workloads (model
spec, batch, frames, LM, fusion settings, the algorithms each is quoted on),
shared by bench.py, scripts/bench_configs.py and the config-shape parity
tests (tests/test_gpu_configs.py).

  bench RNN-T ALSD++ K=4 (AES++, greedy beside), LSTM H=640, J=640, V=1024, D=640, B=128, T=500, bf16
        -- the BASELINE metric's workload ("ALSD++/AES++ beam=4 B=128", config 2's model)
  c1    RNN-T ALSD++ K=4, stateless n=2, V=128, D=J=256, B=1, T=200, fp32
  c2    RNN-T AES++ K=4, LSTM H=640, J=640, V=1024, B=32, T=500, fp32
  c3    TDT ALSD++ and AES++ K=8, durations {0..4}, V=1024, B=128, T=1000, bf16 (LSTM pred-net)
  c4    AES++ K=8 + consistent 4-gram LM (~1M n-grams), V=1024, scored blank, late pruning,
        lambda=0.5, B=128, T=500, bf16
  c5    TDT AES++ K=16, V=8192, J=640, B=1024, T=1500, LM on, bf16 (utterance-sharded over GPUs)

Every model is the peaky synthetic transducer (model.py) with seed 1; the
encoder frames of stream b are drawn from generator (7, b) (bench: (1000, b)),
so any stream subset can be regenerated alone.  Unstated dimensions (D for
C2-C5, T for C4) follow SURVEY.md §8(d): D = J = 640, T = 500.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .model import SyntheticTransducer, TransducerSpec

FRAME_SEC = 0.08
LSTM = _abi.PRED_LSTM
BF16, FP32 = _abi.PREC_BF16, _abi.PREC_FP32
_M640 = dict(vocab_size=1024, enc_dim=640, joint_dim=640, pred_kind=LSTM, lstm_hidden=640, emb_dim=640,
             logit_scale=4.0, peaky=True)
_LATE_SCORED = dict(lam=0.5, blank_mode=_abi.BLANK_SCORED, pruning=_abi.PRUNE_LATE)

CONFIGS: Dict[str, dict] = {
    "bench": dict(spec=dict(_M640, precision=BF16), B=128, T=500, enc_seed=1000,
                  runs=[("alsd_pp", _abi.ALGO_ALSD, 4), ("aes_pp", _abi.ALGO_AES, 4)]),
    "c1": dict(spec=dict(vocab_size=128, enc_dim=256, joint_dim=256, pred_kind=_abi.PRED_STATELESS,
                         context_order=2, precision=FP32, logit_scale=4.0, peaky=True),
               B=1, T=200, runs=[("alsd_pp", _abi.ALGO_ALSD, 4)]),
    "c2": dict(spec=dict(_M640, precision=FP32), B=32, T=500, runs=[("aes_pp", _abi.ALGO_AES, 4)]),
    "c3": dict(spec=dict(_M640, precision=BF16, durations=(0, 1, 2, 3, 4)), B=128, T=1000,
               runs=[("alsd_pp", _abi.ALGO_ALSD, 8), ("aes_pp", _abi.ALGO_AES, 8)]),
    "c4": dict(spec=dict(_M640, precision=BF16), B=128, T=500, lm=(1024, 4, 1_000_000),
               fusion=_LATE_SCORED, runs=[("aes_pp", _abi.ALGO_AES, 8)]),
    "c5": dict(spec=dict(_M640, vocab_size=8192, precision=BF16, durations=(0, 1, 2, 3, 4)),
               B=1024, T=1500, lm=(8192, 4, 1_000_000), fusion=_LATE_SCORED,
               runs=[("aes_pp", _abi.ALGO_AES, 16)]),
}


@dataclass
class Workload:
    name: str
    model: SyntheticTransducer
    B: int
    T: int
    enc_seed: int
    runs: List[Tuple[str, int, int]]
    arpa: Optional[str] = None
    successors: Optional[np.ndarray] = None
    fusion: _abi.FusionConfig = field(default_factory=_abi.FusionConfig)

    def frames(self, streams: Optional[Sequence[int]] = None, T: Optional[int] = None) -> np.ndarray:
        """Encoder frames [len(streams), T, D] fp32 (all B streams by default)."""
        streams = range(self.B) if streams is None else streams
        return self.model.encoder_frames_for(self.enc_seed, streams, T or self.T, self.successors)

    def config(self, beam: int, **kw) -> _abi.DecodeConfig:
        return _abi.DecodeConfig(beam=beam, fusion=self.fusion, max_len=256, **kw)

    def audio_seconds(self, batch: Optional[int] = None) -> float:
        return (batch or self.B) * self.T * FRAME_SEC


@lru_cache(maxsize=None)
def _model(name: str, precision: Optional[int]) -> SyntheticTransducer:
    spec = dict(CONFIGS[name]["spec"])
    if precision is not None:
        spec["precision"] = precision
    return SyntheticTransducer(TransducerSpec(seed=1, **spec))


@lru_cache(maxsize=None)
def _lm(vocab: int, order: int, ngrams: int):
    from .lmgen import arpa_successors, make_consistent_arpa
    arpa = make_consistent_arpa(vocab, order, ngrams)
    return arpa, arpa_successors(arpa, vocab)


def workload(name: str, precision: Optional[int] = None) -> Workload:
    c = CONFIGS[name]
    w = Workload(name=name, model=_model(name, precision), B=c["B"], T=c["T"],
                 enc_seed=c.get("enc_seed", 7), runs=list(c["runs"]))
    if "lm" in c:
        w.arpa, w.successors = _lm(*c["lm"])
        w.fusion = _abi.FusionConfig(**c["fusion"])
    return w
