"""TEST INFRASTRUCTURE -- ctypes front end of the two CPU checkers.

* ``Oracle``  -> oracle/liboracle.so : my CPU restatement (tbeam_oracle.cpp).
* ``RefLib``  -> oracle/_ref/libtbeam_ref.so : the unmodified reference
  (/root/reference/proj/src) compiled in place + ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may use this module, and only as the checker or the
timed CPU baseline -- never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

from paper_2506_00185_b200 import _abi

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtbeam_ref.so")

# reference entry points (ref_shim.cpp)
REF_GREEDY, REF_ALSD_PP, REF_AES_PP, REF_BEAM_ALSD, REF_BEAM_AES = range(5)

_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_DP = C.POINTER(C.c_double)


def build(quiet: bool = True) -> None:
    """Build liboracle.so (always) and _ref (when /root/reference exists)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class _LmHandle:
    def __init__(self, lib, ptr, destroy):
        self.lib, self.ptr, self._destroy = lib, ptr, destroy

    def __del__(self):
        if self.ptr:
            self._destroy(self.ptr)
            self.ptr = None


class Oracle:
    """My CPU restatement (oracle/tbeam_oracle.cpp)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.oracle_last_error.restype = C.c_char_p
        lib.oracle_update_hash.restype = C.c_uint64
        lib.oracle_update_hash.argtypes = [C.c_uint64, C.c_int32, C.c_uint64, C.c_uint64]
        lib.oracle_logadd.restype = C.c_double
        lib.oracle_logadd.argtypes = [C.c_double, C.c_double]
        lib.oracle_log1mexp.restype = C.c_double
        lib.oracle_log1mexp.argtypes = [C.c_double]
        lib.oracle_lm_create.restype = _P
        lib.oracle_lm_create.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_int32]
        lib.oracle_lm_destroy.argtypes = [_P]
        lib.oracle_lm_order.argtypes = [_P]
        lib.oracle_lm_score_token.restype = C.c_double
        lib.oracle_lm_score_token.argtypes = [_P, _I32P, C.c_int32, C.c_int32]
        lib.oracle_lm_score_eos.restype = C.c_double
        lib.oracle_lm_score_eos.argtypes = [_P, _I32P, C.c_int32]
        lib.oracle_lm_score_vocab.argtypes = [_P, _I32P, C.c_int32, _DP]
        lib.oracle_joint_rows.argtypes = [
            C.POINTER(_abi.CModelDims), C.POINTER(_abi.CModelWeights), C.POINTER(C.c_float),
            _I32P, _I32P, C.c_int32, C.c_int32, _DP, _DP]
        lib.oracle_decode.argtypes = [
            C.POINTER(_abi.CModelDims), C.POINTER(_abi.CModelWeights), _P,
            C.POINTER(_abi.CDecodeConfig), C.POINTER(C.c_float), _I32P, C.c_int32, C.c_int32,
            C.POINTER(_abi.CResults)]
        self.lib = lib

    def err(self) -> str:
        return self.lib.oracle_last_error().decode()

    def update_hash(self, h: int, tok: int, base: int = 1_000_003,
                    mod: int = _abi.MERSENNE61) -> int:
        return int(self.lib.oracle_update_hash(h, tok, base, mod))

    def logadd(self, a: float, b: float) -> float:
        return float(self.lib.oracle_logadd(a, b))

    def log1mexp(self, x: float) -> float:
        return float(self.lib.oracle_log1mexp(x))

    def lm(self, arpa: str, vocab: Sequence[str]) -> _LmHandle:
        arr = (C.c_char_p * len(vocab))(*[v.encode() for v in vocab])
        p = self.lib.oracle_lm_create(arpa.encode(), arr, len(vocab))
        if not p:
            raise ValueError(self.err())
        return _LmHandle(self.lib, p, self.lib.oracle_lm_destroy)

    def lm_score_vocab(self, lm: _LmHandle, hist: Sequence[int], vocab: int) -> np.ndarray:
        h = _i32(hist)
        out = np.zeros(vocab, np.float64)
        self.lib.oracle_lm_score_vocab(lm.ptr, h.ctypes.data_as(_I32P), len(h),
                                       out.ctypes.data_as(_DP))
        return out

    def lm_score_token(self, lm: _LmHandle, hist: Sequence[int], tok: int) -> float:
        h = _i32(hist)
        return float(self.lib.oracle_lm_score_token(lm.ptr, h.ctypes.data_as(_I32P), len(h), tok))

    def lm_score_eos(self, lm: _LmHandle, hist: Sequence[int]) -> float:
        h = _i32(hist)
        return float(self.lib.oracle_lm_score_eos(lm.ptr, h.ctypes.data_as(_I32P), len(h)))

    def joint_rows(self, model, enc_frames: np.ndarray, histories: List[List[int]]):
        """Normalised (token, duration) log-prob rows for (frame, history) pairs."""
        spec = model.spec
        R = len(histories)
        mh = max(1, max((len(h) for h in histories), default=1))
        hist = np.full((R, mh), -1, np.int32)
        hl = np.zeros(R, np.int32)
        for i, h in enumerate(histories):
            hist[i, :len(h)] = h
            hl[i] = len(h)
        enc = np.ascontiguousarray(enc_frames, dtype=np.float32)
        tok = np.zeros((R, spec.vocab_size + 1), np.float64)
        dur = np.zeros((R, max(1, len(spec.durations))), np.float64)
        dims, w = model.dims(), model.c_weights()
        rc = self.lib.oracle_joint_rows(C.byref(dims), C.byref(w),
                                        enc.ctypes.data_as(C.POINTER(C.c_float)),
                                        hist.ctypes.data_as(_I32P), hl.ctypes.data_as(_I32P),
                                        mh, R, tok.ctypes.data_as(_DP), dur.ctypes.data_as(_DP))
        if rc != 0:
            raise ValueError(self.err())
        return tok, dur

    def decode(self, model, cfg: _abi.DecodeConfig, algo: int, enc: np.ndarray,
               lengths: Sequence[int], lm: Optional[_LmHandle] = None) -> _abi.DecodeResult:
        enc = np.ascontiguousarray(enc, dtype=np.float32)
        B, T = enc.shape[0], enc.shape[1]
        lens = _i32(lengths)
        nbest = 1 if algo == _abi.ALGO_GREEDY else cfg.return_nbest
        res = _abi.ResultBuffers(B, nbest, cfg.max_len)
        ccfg = cfg.to_c(algo)
        dims, w = model.dims(), model.c_weights()
        rc = self.lib.oracle_decode(C.byref(dims), C.byref(w), lm.ptr if lm else None,
                                    C.byref(ccfg), enc.ctypes.data_as(C.POINTER(C.c_float)),
                                    lens.ctypes.data_as(_I32P), B, T, C.byref(res.c))
        if rc != 0:
            raise _status_error(rc, self.err())
        return res.to_result()


class StatusError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def _status_error(rc: int, msg: str) -> Exception:
    if rc == _abi.TBEAM_INVALID_ARGUMENT:
        e = ValueError(msg)
        e.status = rc
        return e
    return StatusError(rc, msg)


class RefLib:
    """The unmodified reference compiled in place (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (build with `make -C oracle`)")
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_kernels_name.restype = C.c_char_p
        lib.ref_update_hash.restype = C.c_uint64
        lib.ref_update_hash.argtypes = [C.c_uint64, C.c_int32, C.c_uint64, C.c_uint64]
        lib.ref_logadd.restype = C.c_double
        lib.ref_logadd.argtypes = [C.c_double, C.c_double]
        lib.ref_log1mexp.restype = C.c_double
        lib.ref_log1mexp.argtypes = [C.c_double]
        lib.ref_prune_topk.argtypes = [_DP, C.c_int32, C.c_int32, _I32P, _DP]
        lib.ref_vocab_token.argtypes = [C.c_int32, C.c_int32, C.c_char_p, C.c_int32]
        lib.ref_random_arpa.restype = C.c_void_p
        lib.ref_random_arpa.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32]
        lib.ref_free.argtypes = [C.c_void_p]
        lib.ref_lm_create.restype = _P
        lib.ref_lm_create.argtypes = [C.c_char_p, C.c_int32, C.c_int32]
        lib.ref_lm_destroy.argtypes = [_P]
        lib.ref_lm_num_nodes.restype = C.c_int64
        lib.ref_lm_num_nodes.argtypes = [_P]
        lib.ref_lm_order.argtypes = [_P]
        lib.ref_lm_state.argtypes = [_P, _I32P, C.c_int32]
        lib.ref_lm_score_token.restype = C.c_double
        lib.ref_lm_score_token.argtypes = [_P, _I32P, C.c_int32, C.c_int32]
        lib.ref_lm_score_eos.restype = C.c_double
        lib.ref_lm_score_eos.argtypes = [_P, _I32P, C.c_int32]
        lib.ref_lm_score_vocab.argtypes = [_P, _I32P, C.c_int32, _DP]
        lib.ref_decode.argtypes = [
            C.c_int32, C.POINTER(_abi.CModelDims), C.POINTER(_abi.CModelWeights), _P,
            C.POINTER(_abi.CDecodeConfig), C.POINTER(C.c_float), _I32P, C.c_int32, C.c_int32,
            C.POINTER(_abi.CResults), _DP]
        lib.ref_decode_pool.restype = C.c_double
        lib.ref_decode_pool.argtypes = [
            C.c_int32, C.POINTER(_abi.CModelDims), C.POINTER(_abi.CModelWeights), _P,
            C.POINTER(_abi.CDecodeConfig), C.POINTER(C.c_float), _I32P, C.c_int32, C.c_int32,
            C.c_int32, C.POINTER(_abi.CResults)]
        self.lib = lib

    def err(self) -> str:
        return self.lib.ref_last_error().decode()

    def kernels_name(self) -> str:
        return self.lib.ref_kernels_name().decode()

    def update_hash(self, h, tok, base=1_000_003, mod=_abi.MERSENNE61) -> int:
        return int(self.lib.ref_update_hash(h, tok, base, mod))

    def logadd(self, a, b) -> float:
        return float(self.lib.ref_logadd(a, b))

    def log1mexp(self, x) -> float:
        return float(self.lib.ref_log1mexp(x))

    def prune_topk(self, scores: Sequence[float], k: int):
        s = np.ascontiguousarray(scores, dtype=np.float64)
        idx = np.zeros(k, np.int32)
        out = np.zeros(k, np.float64)
        rc = self.lib.ref_prune_topk(s.ctypes.data_as(_DP), len(s), k,
                                     idx.ctypes.data_as(_I32P), out.ctypes.data_as(_DP))
        if rc != 0:
            raise ValueError(self.err())
        return idx, out

    def vocab(self, size: int) -> List[str]:
        buf = C.create_string_buffer(64)
        out = []
        for i in range(size):
            self.lib.ref_vocab_token(size, i, buf, 64)
            out.append(buf.value.decode())
        return out

    def random_arpa(self, seed: int, vocab: int, order: int, with_eos: bool = True) -> str:
        p = self.lib.ref_random_arpa(seed, vocab, order, int(with_eos))
        s = C.string_at(p).decode()
        self.lib.ref_free(p)
        return s

    def lm(self, arpa: str, vocab: int, strict: bool = False) -> _LmHandle:
        p = self.lib.ref_lm_create(arpa.encode(), vocab, int(strict))
        if not p:
            raise ValueError(self.err())
        return _LmHandle(self.lib, p, self.lib.ref_lm_destroy)

    def lm_state(self, lm, hist) -> int:
        h = _i32(hist)
        return int(self.lib.ref_lm_state(lm.ptr, h.ctypes.data_as(_I32P), len(h)))

    def lm_score_vocab(self, lm, hist, vocab: int) -> np.ndarray:
        h = _i32(hist)
        out = np.zeros(vocab, np.float64)
        self.lib.ref_lm_score_vocab(lm.ptr, h.ctypes.data_as(_I32P), len(h),
                                    out.ctypes.data_as(_DP))
        return out

    def lm_score_token(self, lm, hist, tok) -> float:
        h = _i32(hist)
        return float(self.lib.ref_lm_score_token(lm.ptr, h.ctypes.data_as(_I32P), len(h), tok))

    def lm_score_eos(self, lm, hist) -> float:
        h = _i32(hist)
        return float(self.lib.ref_lm_score_eos(lm.ptr, h.ctypes.data_as(_I32P), len(h)))

    def decode(self, which: int, model, cfg: _abi.DecodeConfig, enc: np.ndarray,
               lengths: Sequence[int], lm: Optional[_LmHandle] = None) -> _abi.DecodeResult:
        enc = np.ascontiguousarray(enc, dtype=np.float32)
        B, T = enc.shape[0], enc.shape[1]
        lens = _i32(lengths)
        nbest = 1 if which == REF_GREEDY else cfg.return_nbest
        res = _abi.ResultBuffers(B, nbest, cfg.max_len)
        algo = {REF_GREEDY: _abi.ALGO_GREEDY, REF_ALSD_PP: _abi.ALGO_ALSD,
                REF_BEAM_ALSD: _abi.ALGO_ALSD}.get(which, _abi.ALGO_AES)
        ccfg = cfg.to_c(algo)
        dims, w = model.dims(), model.c_weights()
        wall = C.c_double(0.0)
        rc = self.lib.ref_decode(which, C.byref(dims), C.byref(w), lm.ptr if lm else None,
                                 C.byref(ccfg), enc.ctypes.data_as(C.POINTER(C.c_float)),
                                 lens.ctypes.data_as(_I32P), B, T, C.byref(res.c),
                                 C.byref(wall))
        if rc != 0:
            raise _status_error(rc, self.err())
        r = res.to_result(with_alignment=False)
        r.wall_seconds = wall.value
        return r

    def decode_pool(self, which: int, model, cfg: _abi.DecodeConfig, enc: np.ndarray,
                    lengths: Sequence[int], count: int, threads: int,
                    lm: Optional[_LmHandle] = None) -> float:
        """Wall seconds to decode utterances [0, count) on `threads` workers."""
        enc = np.ascontiguousarray(enc, dtype=np.float32)
        lens = _i32(lengths)
        algo = {REF_GREEDY: _abi.ALGO_GREEDY, REF_ALSD_PP: _abi.ALGO_ALSD,
                REF_BEAM_ALSD: _abi.ALGO_ALSD}.get(which, _abi.ALGO_AES)
        ccfg = cfg.to_c(algo)
        dims, w = model.dims(), model.c_weights()
        wall = self.lib.ref_decode_pool(which, C.byref(dims), C.byref(w),
                                        lm.ptr if lm else None, C.byref(ccfg),
                                        enc.ctypes.data_as(C.POINTER(C.c_float)),
                                        lens.ctypes.data_as(_I32P), count, enc.shape[1],
                                        threads, None)
        if wall < 0:
            raise RuntimeError(self.err())
        return wall
