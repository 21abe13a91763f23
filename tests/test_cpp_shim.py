"""The header-only C++ shim (include/tbeam_b200.hpp) that re-exposes the
reference's greedy_batched / alsd_pp / aes_pp: it compiles and links against
the sm_100a library (CPU), and on the GPU its results equal the CPU oracle."""
import ctypes as C
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2506_00185_b200 import _abi
from tests.conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp")
LIBDIR = os.path.join(ROOT, "paper_2506_00185_b200")


def build(tmp_path):
    exe = str(tmp_path / "shim_demo")
    subprocess.run(["g++", "-std=c++20", "-O1", SRC, "-I", os.path.join(ROOT, "include"), "-L", LIBDIR,
                    "-ltbeam_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


class _Model:
    """Adapter: weights from the C++ demo -> the oracle's model interface."""

    def __init__(self, w):
        self.weights = {k: np.ascontiguousarray(np.array(w[k], np.float32)) for k in
                        ("w_enc", "b_enc", "pred_table", "b_pred", "w_out", "b_out")}
        self.spec = type("S", (), {"vocab_size": 20, "durations": ()})()

    def dims(self):
        d = _abi.CModelDims()
        d.vocab_size, d.enc_dim, d.joint_dim, d.pred_kind, d.context_order = 20, 16, 32, 0, 2
        return d

    def c_weights(self):
        cw = _abi.CModelWeights()
        for name, _ in _abi.CModelWeights._fields_:
            a = self.weights.get(name)
            setattr(cw, name, a.ctypes.data_as(C.POINTER(C.c_float)) if a is not None else C.POINTER(C.c_float)())
        return cw


@pytest.mark.gpu
def test_shim_matches_oracle(tmp_path, oracle):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True, check=True).stdout
    d = json.loads(out)
    assert d["invalid_argument_raised"] is True
    m = _Model(d)
    enc = np.array(d["enc"], np.float32).reshape(3, 12, 16)
    cfg = _abi.DecodeConfig(return_nbest=2, max_len=20)
    for name, algo in (("greedy", _abi.ALGO_GREEDY), ("alsd", _abi.ALGO_ALSD), ("aes", _abi.ALGO_AES)):
        o = oracle.decode(m, cfg, algo, enc, d["lens"])
        for got, want in zip(d["results"][name], o.streams):
            assert [e["tokens"] for e in got] == [e.tokens for e in want.nbest]
            for a, b in zip(got, want.nbest):
                assert abs(a["score"] - b.score) < 1e-4
