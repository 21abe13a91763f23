"""Host-side mirror of the reference decoder API over the C-ABI library.

Reference interface (proj/include/tbeam/decoder.hpp:75-91)::

    DecodeResult greedy_batched(std::span<const StreamInput>, const DecodeConfig&);
    DecodeResult alsd_pp       (std::span<const StreamInput>, const DecodeConfig&);
    DecodeResult aes_pp        (std::span<const StreamInput>, const DecodeConfig&);

Here a ``StreamInput`` carries the stream's encoder frames instead of a
virtual ``EmissionModel`` (the model weights live on the device inside a
:class:`B200Decoder`), and the same three entry points run the B200 kernels.
Errors follow the reference's taxonomy: ``ValueError`` for
``std::invalid_argument`` (decoder.cpp:16-38), :class:`ParseError` for
``tbeam::ParseError``, :class:`CapacityError`, :class:`ValidationError`.

There is no CPU fallback: constructing a decoder without the built
``libtbeam_b200.so`` or without an sm_100 GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import DecodeConfig, DecodeResult, FusionConfig, HashParams  # noqa: F401
from .model import SyntheticTransducer, synthetic_vocabulary

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TBEAM_LIB", os.path.join(_HERE, "libtbeam_b200.so"))  # env: measurement variants

_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)


class ParseError(ValueError):
    """tbeam::ParseError (types.hpp:29-44)."""


class ValidationError(ValueError):
    """tbeam::ValidationError (types.hpp:46-49)."""


class CapacityError(RuntimeError):
    """tbeam::CapacityError (types.hpp:51-54)."""


class CudaError(RuntimeError):
    pass


class UnsupportedError(RuntimeError):
    pass


_lib = None


def symbols() -> List[str]:
    """Every entry point include/tbeam_b200.h declares."""
    return ["tbeam_decode_config_init", "tbeam_create", "tbeam_destroy", "tbeam_set_model",
            "tbeam_set_lm_arpa", "tbeam_lm_parse_check", "tbeam_lm_export", "tbeam_clear_lm",
            "tbeam_lm_info", "tbeam_decode",
            "tbeam_prepare", "tbeam_decode_device", "tbeam_fetch_results", "tbeam_launch_stats",
            "tbeam_stage_inputs", "tbeam_decode_staged",
            "tbeam_set_graph_mode", "tbeam_last_error", "tbeam_abi_version",
            "tbeam_profile_decode"]


def load_library(path: str = LIB_PATH):
    """Load libtbeam_b200.so (no fallback: raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(
            f"{path} is missing; build it with `python -m paper_2506_00185_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    lib.tbeam_last_error.restype = C.c_char_p
    lib.tbeam_abi_version.restype = C.c_int32
    lib.tbeam_decode_config_init.argtypes = [C.POINTER(_abi.CDecodeConfig)]
    lib.tbeam_create.argtypes = [C.c_int, C.POINTER(_P)]
    lib.tbeam_destroy.argtypes = [_P]
    lib.tbeam_set_model.argtypes = [_P, C.POINTER(_abi.CModelDims), C.POINTER(_abi.CModelWeights)]
    lib.tbeam_set_lm_arpa.argtypes = [_P, C.c_char_p, C.c_size_t, C.POINTER(C.c_char_p),
                                      C.c_int32, C.c_int32]
    lib.tbeam_lm_parse_check.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_char_p), C.c_int32,
                                         C.c_int32, C.POINTER(C.c_int64)]
    lib.tbeam_lm_export.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_char_p), C.c_int32, C.c_int32,
                                    C.POINTER(C.c_int64)] + [C.c_void_p] * 9
    lib.tbeam_clear_lm.argtypes = [_P]
    lib.tbeam_lm_info.argtypes = [_P, C.POINTER(C.c_int64)]
    lib.tbeam_decode.argtypes = [_P, C.POINTER(_abi.CDecodeConfig), C.c_void_p, C.c_int32,
                                 _I32P, C.c_int32, C.c_int32, C.POINTER(_abi.CResults), C.c_void_p]
    lib.tbeam_prepare.argtypes = [_P, C.POINTER(_abi.CDecodeConfig), C.c_int32, C.c_int32]
    lib.tbeam_decode_device.argtypes = [_P, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.tbeam_fetch_results.argtypes = [_P, C.POINTER(_abi.CResults), C.c_void_p]
    lib.tbeam_stage_inputs.argtypes = [_P, C.c_void_p, _I32P, C.c_int32, C.c_int32]
    lib.tbeam_decode_staged.argtypes = [_P, C.POINTER(_abi.CDecodeConfig), C.POINTER(_abi.CResults), C.c_void_p]
    lib.tbeam_launch_stats.restype = C.c_int32
    lib.tbeam_launch_stats.argtypes = [_P, C.POINTER(C.c_int64), C.c_int32]
    lib.tbeam_set_graph_mode.argtypes = [_P, C.c_int32]
    lib.tbeam_profile_decode.restype = C.c_int32
    lib.tbeam_profile_decode.argtypes = [_P, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int64)]
    for name in ("tbeam_create", "tbeam_destroy", "tbeam_set_model", "tbeam_set_lm_arpa",
                 "tbeam_lm_parse_check", "tbeam_lm_export",
                 "tbeam_clear_lm", "tbeam_lm_info", "tbeam_decode", "tbeam_prepare",
                 "tbeam_decode_device", "tbeam_fetch_results", "tbeam_set_graph_mode",
                 "tbeam_stage_inputs", "tbeam_decode_staged"):
        getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def _raise(status: int) -> None:
    if status == _abi.TBEAM_OK:
        return
    msg = _lib.tbeam_last_error().decode(errors="replace")
    cls = {
        _abi.TBEAM_INVALID_ARGUMENT: ValueError,
        _abi.TBEAM_CAPACITY: CapacityError,
        _abi.TBEAM_PARSE: ParseError,
        _abi.TBEAM_VALIDATION: ValidationError,
        _abi.TBEAM_CUDA: CudaError,
        _abi.TBEAM_UNSUPPORTED: UnsupportedError,
    }.get(status, RuntimeError)
    err = cls(msg)
    err.status = status
    raise err


@dataclass
class StreamInput:
    """tbeam::StreamInput (decoder.hpp:18-21): one stream's encoder frames
    ([T, D] fp32) and how many of them to consume."""
    enc: np.ndarray
    num_frames: int


def pack_streams(streams: Sequence[StreamInput]):
    if len(streams) == 0:
        raise ValueError("decode: no streams")
    D = streams[0].enc.shape[1]
    for s in streams:
        # decoder.cpp:22-24: "decode: bad stream input"
        if s.enc.ndim != 2 or s.enc.shape[1] != D:
            raise ValueError("decode: bad stream input (encoder frames must be [T, D], one D)")
        if s.num_frames < 1 or s.num_frames > s.enc.shape[0]:
            raise ValueError("decode: bad stream input (num_frames outside [1, frames supplied])")
    T = max(s.enc.shape[0] for s in streams)
    enc = np.zeros((len(streams), T, D), np.float32)
    for b, s in enumerate(streams):
        enc[b, :s.enc.shape[0]] = s.enc
    return enc, np.array([s.num_frames for s in streams], np.int32)


class B200Decoder:
    """One decoder context on one CUDA device: weights (+ optional LM) live on
    the device; decode calls run the sm_100a kernels as one CUDA graph."""

    def __init__(self, model: SyntheticTransducer, device: int = 0):
        lib = load_library()
        self.lib = lib
        self.model = model
        self._ctx = _P()
        _raise(lib.tbeam_create(device, C.byref(self._ctx)))
        dims, w = model.dims(), model.c_weights()
        _raise(lib.tbeam_set_model(self._ctx, C.byref(dims), C.byref(w)))
        self._lm_vocab = None

    def close(self) -> None:
        if self._ctx:
            self.lib.tbeam_destroy(self._ctx)
            self._ctx = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ctx(self):
        return self._ctx

    def set_graph_mode(self, mode: int) -> None:
        _raise(self.lib.tbeam_set_graph_mode(self._ctx, mode))

    def set_lm(self, arpa_text: str, vocab: Optional[Sequence[str]] = None,
               strict: bool = False) -> None:
        """NGramLm::parse_arpa_text against the ASR token table, uploaded."""
        vocab = list(vocab) if vocab is not None else synthetic_vocabulary(
            self.model.spec.vocab_size)
        arr = (C.c_char_p * len(vocab))(*[v.encode() for v in vocab])
        data = arpa_text.encode()
        _raise(self.lib.tbeam_set_lm_arpa(self._ctx, data, len(data), arr, len(vocab),
                                          int(strict)))

    def clear_lm(self) -> None:
        _raise(self.lib.tbeam_clear_lm(self._ctx))

    def lm_info(self):
        out = (C.c_int64 * 4)()
        _raise(self.lib.tbeam_lm_info(self._ctx, out))
        return {"order": out[0], "nodes": out[1], "edges": out[2], "oov_mapped": out[3]}

    def decode(self, algo: int, enc: np.ndarray, lengths: Sequence[int],
               cfg: Optional[DecodeConfig] = None) -> DecodeResult:
        cfg = cfg or DecodeConfig()
        enc = np.ascontiguousarray(enc, dtype=np.float32)
        if enc.ndim != 3:
            raise ValueError("decode: enc must be [B, T, D]")
        B, T = enc.shape[0], enc.shape[1]
        if enc.shape[2] != self.model.spec.enc_dim:
            # the C-ABI reads batch * max_frames * enc_dim floats from enc
            raise ValueError(f"decode: encoder frames have width {enc.shape[2]}, "
                             f"the model's enc_dim is {self.model.spec.enc_dim}")
        lens = np.ascontiguousarray(np.asarray(lengths, np.int32))
        if lens.shape[0] != B:
            raise ValueError("decode: lengths must have one entry per stream")
        nbest = 1 if algo == _abi.ALGO_GREEDY else cfg.return_nbest
        res = _abi.ResultBuffers(B, nbest, cfg.max_len)
        ccfg = cfg.to_c(algo)
        _raise(self.lib.tbeam_decode(self._ctx, C.byref(ccfg), enc.ctypes.data_as(C.c_void_p), 0,
                                     lens.ctypes.data_as(_I32P), B, T, C.byref(res.c), None))
        return res.to_result()

    # -- pipelined host-buffer path (serving) -----------------------------------
    def stage_inputs(self, enc: np.ndarray, lengths: Sequence[int]) -> None:
        """tbeam_stage_inputs: async H2D of a batch into the next input slot
        (pinned host memory overlaps it with a running decode).  `enc` and
        the lengths array must stay alive until decode_staged of the batch."""
        if enc.ndim != 3 or enc.dtype != np.float32 or not enc.flags["C_CONTIGUOUS"]:
            raise ValueError("stage_inputs: enc must be a C-contiguous float32 [B, T, D] array")
        if enc.shape[2] != self.model.spec.enc_dim:
            raise ValueError(f"decode: encoder frames have width {enc.shape[2]}, "
                             f"the model's enc_dim is {self.model.spec.enc_dim}")
        lens = np.ascontiguousarray(np.asarray(lengths, np.int32))
        if lens.shape[0] != enc.shape[0]:
            raise ValueError("decode: lengths must have one entry per stream")
        self._staged = getattr(self, "_staged", [])
        self._staged.append((enc, lens))
        _raise(self.lib.tbeam_stage_inputs(self._ctx, enc.ctypes.data_as(C.c_void_p),
                                           lens.ctypes.data_as(_I32P), enc.shape[0], enc.shape[1]))

    def decode_staged(self, algo: int, cfg: Optional[DecodeConfig] = None, stream: int = 0,
                      raw: bool = False):
        """tbeam_decode_staged: decode the oldest staged batch, fetch results
        (raw=True: the filled result arrays, _abi.ResultBuffers, without the
        per-entry Python objects)."""
        cfg = cfg or DecodeConfig()
        enc, _ = self._staged[0]
        nbest = 1 if algo == _abi.ALGO_GREEDY else cfg.return_nbest
        res = _abi.ResultBuffers(enc.shape[0], nbest, cfg.max_len)
        ccfg = cfg.to_c(algo)
        try:
            _raise(self.lib.tbeam_decode_staged(self._ctx, C.byref(ccfg), C.byref(res.c), C.c_void_p(stream)))
        finally:
            self._staged.pop(0)
        return res if raw else res.to_result()

    # -- device-resident path (benchmarks) -------------------------------------
    def prepare(self, algo: int, cfg: DecodeConfig, batch: int, max_frames: int) -> None:
        ccfg = cfg.to_c(algo)
        _raise(self.lib.tbeam_prepare(self._ctx, C.byref(ccfg), batch, max_frames))

    def decode_device(self, enc_ptr: int, lengths_ptr: int, stream: int = 0) -> None:
        _raise(self.lib.tbeam_decode_device(self._ctx, C.c_void_p(enc_ptr),
                                            C.c_void_p(lengths_ptr), C.c_void_p(stream)))

    def fetch(self, batch: int, nbest: int, max_len: int, stream: int = 0) -> DecodeResult:
        res = _abi.ResultBuffers(batch, nbest, max_len)
        _raise(self.lib.tbeam_fetch_results(self._ctx, C.byref(res.c), C.c_void_p(stream)))
        return res.to_result()

    FAMILIES = ("enc_proj", "init", "joint", "select", "lstm_gates", "lstm_proj", "finalize")

    def profile_device(self, enc_ptr: int, lengths_ptr: int, stream: int = 0) -> dict:
        """Instrumented (host-driven, event-bracketed) decode: per kernel family
        device ms and launch counts, plus scored rows and rounds."""
        ms = (C.c_double * 7)()
        n = (C.c_int64 * 7)()
        rows = (C.c_int64 * 2)()
        k = self.lib.tbeam_profile_decode(self._ctx, C.c_void_p(enc_ptr), C.c_void_p(lengths_ptr),
                                          C.c_void_p(stream), ms, n, rows)
        if k < 0:
            _raise(_abi.TBEAM_INVALID_ARGUMENT)
        return {"ms": {f: ms[i] for i, f in enumerate(self.FAMILIES)},
                "launches": {f: n[i] for i, f in enumerate(self.FAMILIES)},
                "scored_rows": rows[0], "rounds": rows[1]}

    def launch_stats(self):
        out = (C.c_int64 * 3)()
        n = self.lib.tbeam_launch_stats(self._ctx, out, 3)
        return {"launches": out[0], "rounds": out[1] if n > 1 else 0,
                "kernels_per_round": out[2] if n > 2 else 0}


def lm_export(arpa_text: str, vocab: Sequence[str], strict: bool = False) -> dict:
    """The frozen trie the device queries walk (tbeam_lm_export), as numpy
    arrays: for inspection and the CPU parser tests (no GPU needed)."""
    lib = load_library()
    arr = (C.c_char_p * len(vocab))(*[v.encode() for v in vocab])
    data = arpa_text.encode()
    out = (C.c_int64 * 4)()
    nul = [None] * 9
    _raise(lib.tbeam_lm_export(data, len(data), arr, len(vocab), int(strict), out, *nul))
    order, n, e, initial = (int(x) for x in out)
    a = {"prob": np.zeros(n, np.float64), "backoff": np.zeros(n, np.float64),
         "suffix": np.zeros(n, np.int32), "depth": np.zeros(n, np.int32),
         "cbeg": np.zeros(n, np.int32), "cend": np.zeros(n, np.int32),
         "etok": np.zeros(max(e, 1), np.int32), "enode": np.zeros(max(e, 1), np.int32),
         "remap": np.zeros(len(vocab), np.int32)}
    ptrs = [a[k].ctypes.data_as(C.c_void_p) for k in
            ("prob", "backoff", "suffix", "depth", "cbeg", "cend", "etok", "enode", "remap")]
    _raise(lib.tbeam_lm_export(data, len(data), arr, len(vocab), int(strict), out, *ptrs))
    a.update(order=order, nodes=n, edges=e, initial=initial, V=len(vocab))
    return a


def parse_arpa_check(arpa_text: str, vocab: Sequence[str], strict: bool = False) -> dict:
    """Host-only ARPA validation with the product parser (no GPU needed);
    raises ParseError like NGramLm::parse_arpa_text (ngram_lm.cpp:52-318)."""
    lib = load_library()
    arr = (C.c_char_p * len(vocab))(*[v.encode() for v in vocab])
    data = arpa_text.encode()
    out = (C.c_int64 * 4)()
    _raise(lib.tbeam_lm_parse_check(data, len(data), arr, len(vocab), int(strict), out))
    return {"order": out[0], "nodes": out[1], "edges": out[2], "oov_mapped": out[3]}


# ---- the reference's three entry points ---------------------------------------

def greedy_batched(decoder: B200Decoder, streams: Sequence[StreamInput],
                   cfg: Optional[DecodeConfig] = None) -> DecodeResult:
    """tbeam::greedy_batched (decoder.hpp:75-76, decoder.cpp:429-442)."""
    enc, lens = pack_streams(streams)
    return decoder.decode(_abi.ALGO_GREEDY, enc, lens, cfg)


def alsd_pp(decoder: B200Decoder, streams: Sequence[StreamInput],
            cfg: Optional[DecodeConfig] = None) -> DecodeResult:
    """tbeam::alsd_pp (decoder.hpp:79, decoder.cpp:444-448)."""
    enc, lens = pack_streams(streams)
    return decoder.decode(_abi.ALGO_ALSD, enc, lens, cfg)


def aes_pp(decoder: B200Decoder, streams: Sequence[StreamInput],
           cfg: Optional[DecodeConfig] = None) -> DecodeResult:
    """tbeam::aes_pp (decoder.hpp:83, decoder.cpp:450-454); canonical AES++
    semantics unless ``cfg.aes_slot_donated_quirk``."""
    enc, lens = pack_streams(streams)
    return decoder.decode(_abi.ALGO_AES, enc, lens, cfg)
