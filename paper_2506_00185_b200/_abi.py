"""ctypes mirror of include/tbeam_b200.h (the C-ABI boundary).

Plain data only: struct layouts, enum values, defaults and result buffers.
The structs mirror the reference's configuration types field for field:
``DecodeConfig`` (proj/include/tbeam/decoder.hpp:23-42), ``FusionConfig``
(fusion.hpp:19-24) and ``HashParams`` (hyp_store.hpp:15-18).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

TBEAM_OK = 0
TBEAM_INVALID_ARGUMENT = 1
TBEAM_CAPACITY = 2
TBEAM_PARSE = 3
TBEAM_VALIDATION = 4
TBEAM_CUDA = 5
TBEAM_UNSUPPORTED = 6

ALGO_GREEDY, ALGO_ALSD, ALGO_AES = 0, 1, 2
BLANK_OMIT, BLANK_SCORED = 0, 1
PRUNE_EARLY, PRUNE_LATE = 0, 1
MERGE_LOGSUMEXP, MERGE_MAX = 0, 1
PRED_STATELESS, PRED_LSTM = 0, 1
PREC_FP32, PREC_BF16 = 0, 1
MAX_DURATIONS = 8
NUM_COUNTERS = 5
COUNTER_NAMES = ("frames", "scoring_rounds", "scored_slots", "lm_token_queries",
                 "lm_vocab_queries")
MERSENNE61 = (1 << 61) - 1


class CDecodeConfig(C.Structure):
    _fields_ = [
        ("algo", C.c_int32),
        ("beam", C.c_int32),
        ("max_symbols_per_frame", C.c_int32),
        ("aes_expansions_per_frame", C.c_int32),
        ("max_len", C.c_int32),
        ("return_nbest", C.c_int32),
        ("aes_prefix_search", C.c_int32),
        ("lm_weight", C.c_double),
        ("blank_mode", C.c_int32),
        ("prune_mode", C.c_int32),
        ("eos_enabled", C.c_int32),
        ("merge_mode", C.c_int32),
        ("hash_base", C.c_uint64),
        ("hash_modulus", C.c_uint64),
        ("aes_slot_donated_quirk", C.c_int32),
        ("reserved", C.c_int32 * 7),
    ]


class CModelDims(C.Structure):
    _fields_ = [
        ("vocab_size", C.c_int32),
        ("enc_dim", C.c_int32),
        ("joint_dim", C.c_int32),
        ("pred_kind", C.c_int32),
        ("context_order", C.c_int32),
        ("lstm_hidden", C.c_int32),
        ("emb_dim", C.c_int32),
        ("num_durations", C.c_int32),
        ("durations", C.c_int32 * MAX_DURATIONS),
        ("precision", C.c_int32),
        ("reserved", C.c_int32 * 3),
    ]


_FP = C.POINTER(C.c_float)


class CModelWeights(C.Structure):
    _fields_ = [(n, _FP) for n in (
        "w_enc", "b_enc", "pred_table", "b_pred", "emb", "w_ih", "w_hh", "b_lstm",
        "w_pred", "w_out", "b_out", "w_dur", "b_dur")]


class CResults(C.Structure):
    _fields_ = [
        ("batch", C.c_int32),
        ("nbest", C.c_int32),
        ("max_len", C.c_int32),
        ("nbest_count", C.POINTER(C.c_int32)),
        ("lengths", C.POINTER(C.c_int32)),
        ("scores", C.POINTER(C.c_double)),
        ("tokens", C.POINTER(C.c_int32)),
        ("frames", C.POINTER(C.c_int32)),
        ("durations", C.POINTER(C.c_int32)),
        ("counters", C.POINTER(C.c_uint64)),
    ]


# ---------------------------------------------------------------------------
# Python-side mirrors of the reference config types
# ---------------------------------------------------------------------------

@dataclass
class FusionConfig:
    """tbeam::FusionConfig (fusion.hpp:19-24)."""
    lam: float = 0.0
    blank_mode: int = BLANK_OMIT
    pruning: int = PRUNE_LATE
    eos_enabled: bool = False


@dataclass
class HashParams:
    """tbeam::HashParams (hyp_store.hpp:15-18)."""
    base: int = 1_000_003
    modulus: int = MERSENNE61


@dataclass
class DecodeConfig:
    """tbeam::DecodeConfig (decoder.hpp:23-42) plus the B200 additions."""
    beam: int = 4
    max_symbols_per_frame: int = 10
    aes_expansions_per_frame: int = 2
    max_len: int = 256
    return_nbest: int = 1
    aes_prefix_search: bool = True
    fusion: FusionConfig = field(default_factory=FusionConfig)
    hash_params: HashParams = field(default_factory=HashParams)
    merge_mode: int = MERGE_LOGSUMEXP
    aes_slot_donated_quirk: bool = False

    def to_c(self, algo: int) -> CDecodeConfig:
        c = CDecodeConfig()
        c.algo = algo
        c.beam = self.beam
        c.max_symbols_per_frame = self.max_symbols_per_frame
        c.aes_expansions_per_frame = self.aes_expansions_per_frame
        c.max_len = self.max_len
        c.return_nbest = self.return_nbest
        c.aes_prefix_search = int(bool(self.aes_prefix_search))
        c.lm_weight = float(self.fusion.lam)
        c.blank_mode = int(self.fusion.blank_mode)
        c.prune_mode = int(self.fusion.pruning)
        c.eos_enabled = int(bool(self.fusion.eos_enabled))
        c.merge_mode = int(self.merge_mode)
        c.hash_base = int(self.hash_params.base)
        c.hash_modulus = int(self.hash_params.modulus)
        c.aes_slot_donated_quirk = int(bool(self.aes_slot_donated_quirk))
        return c


@dataclass
class NBestEntry:
    """tbeam::NBestEntry (decoder.hpp:52-55) + alignment / TDT durations."""
    tokens: List[int]
    score: float
    frames: Optional[List[int]] = None
    durations: Optional[List[int]] = None


@dataclass
class StreamResult:
    nbest: List[NBestEntry]
    counters: dict


@dataclass
class DecodeResult:
    streams: List[StreamResult]
    wall_seconds: float = 0.0

    def total_frames(self) -> int:
        return sum(s.counters.get("frames", 0) for s in self.streams)


class ResultBuffers:
    """Caller-owned host arrays behind a ``tbeam_results`` struct."""

    def __init__(self, batch: int, nbest: int, max_len: int):
        self.batch, self.nbest, self.max_len = batch, nbest, max_len
        self.nbest_count = np.zeros(batch, np.int32)
        self.lengths = np.zeros((batch, nbest), np.int32)
        self.scores = np.full((batch, nbest), -np.inf, np.float64)
        self.tokens = np.zeros((batch, nbest, max_len), np.int32)
        self.frames = np.zeros((batch, nbest, max_len), np.int32)
        self.durations = np.zeros((batch, nbest, max_len), np.int32)
        self.counters = np.zeros((batch, NUM_COUNTERS), np.uint64)
        self.c = CResults()
        self.c.batch, self.c.nbest, self.c.max_len = batch, nbest, max_len
        self.c.nbest_count = self.nbest_count.ctypes.data_as(C.POINTER(C.c_int32))
        self.c.lengths = self.lengths.ctypes.data_as(C.POINTER(C.c_int32))
        self.c.scores = self.scores.ctypes.data_as(C.POINTER(C.c_double))
        self.c.tokens = self.tokens.ctypes.data_as(C.POINTER(C.c_int32))
        self.c.frames = self.frames.ctypes.data_as(C.POINTER(C.c_int32))
        self.c.durations = self.durations.ctypes.data_as(C.POINTER(C.c_int32))
        self.c.counters = self.counters.ctypes.data_as(C.POINTER(C.c_uint64))

    def to_result(self, with_alignment: bool = True) -> DecodeResult:
        streams = []
        for b in range(self.batch):
            nb = []
            for r in range(int(self.nbest_count[b])):
                L = int(self.lengths[b, r])
                nb.append(NBestEntry(
                    tokens=self.tokens[b, r, :L].tolist(),
                    score=float(self.scores[b, r]),
                    frames=self.frames[b, r, :L].tolist() if with_alignment else None,
                    durations=self.durations[b, r, :L].tolist() if with_alignment else None))
            ctr = {n: int(self.counters[b, i]) for i, n in enumerate(COUNTER_NAMES)}
            streams.append(StreamResult(nbest=nb, counters=ctr))
        return DecodeResult(streams=streams)
