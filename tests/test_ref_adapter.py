"""The reference-typed adapter (include/tbeam_b200_reference.hpp): the B200
decoder behind the reference's OWN DecodeFn signature, picked by name through
an algo_fn and run through decode_chunked the way the reference CLI does
(commands.cpp:138-173, :374-415).  oracle/_ref/ref_adapter_demo is built in the
build container against the unmodified reference (headers + objects) and the
B200 library; on the GPU every "<algo>-b200" result must equal the reference's
own "<algo>" on the same streams (fp32 model: tokens and counters exact,
scores within 1e-4)."""
import json
import os
import struct
import subprocess

import numpy as np
import pytest

from paper_2506_00185_b200 import _abi
from tests.conftest import ROOT
from tests.helpers import instance

DEMO = os.path.join(ROOT, "oracle", "_ref", "ref_adapter_demo")
G = os.path.join(ROOT, "tests", "golden")


def write_model(path, model, enc, lens):
    with open(path, "wb") as f:
        f.write(bytes(model.dims()))
        for name, _ in _abi.CModelWeights._fields_:
            a = model.weights.get(name)
            a = np.zeros(0, np.float32) if a is None else np.ascontiguousarray(a, np.float32).ravel()
            f.write(struct.pack("<q", a.size))
            f.write(a.tobytes())
        B, T, D = enc.shape
        f.write(struct.pack("<iii", B, T, D))
        f.write(np.ascontiguousarray(enc, np.float32).tobytes())
        f.write(np.asarray(lens, np.int32).tobytes())


def run(path, *args):
    out = subprocess.run([DEMO, path, *args], check=True, capture_output=True, text=True, timeout=600).stdout
    return [json.loads(line) for line in out.splitlines() if line.startswith("{")]


def test_demo_links_the_b200_library():
    """Built here next to the reference objects; it must resolve the in-tree
    libtbeam_b200.so (rpath $ORIGIN/../../paper_2506_00185_b200)."""
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/ref_adapter_demo not built (reference tree absent at build time)")
    out = subprocess.run(["ldd", DEMO], capture_output=True, text=True).stdout
    assert "paper_2506_00185_b200/libtbeam_b200.so" in out


def pairs(rows):
    by = {r["algo"]: r for r in rows}
    for name, r in by.items():
        if not name.endswith("-b200"):
            yield name, r, by[name + "-b200"]


CASES = [
    ("stateless", dict(kind=_abi.PRED_STATELESS, V=24, D=16, J=32, B=5, T=30), ["--beam", "4", "--nbest", "3"]),
    ("lstm", dict(kind=_abi.PRED_LSTM, V=20, D=16, J=32, H=24, E=8, B=4, T=24), ["--beam", "3", "--nbest", "2"]),
    ("lm_late_scored", dict(kind=_abi.PRED_STATELESS, V=40, D=16, J=32, B=4, T=16),
     ["--beam", "4", "--lm", os.path.join(G, "lm_v40_o3.arpa"), "--lambda", "0.5", "--blank", "scored",
      "--pruning", "late", "--eos"]),
    ("lm_early_chunked", dict(kind=_abi.PRED_STATELESS, V=40, D=16, J=32, B=5, T=16),
     ["--beam", "4", "--lm", os.path.join(G, "lm_v40_o3.arpa"), "--lambda", "0.3", "--blank", "omit",
      "--pruning", "early", "--batch", "2"]),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,inst,args", CASES, ids=[c[0] for c in CASES])
def test_adapter_equals_reference(tmp_path, name, inst, args):
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/ref_adapter_demo not built")
    model, enc, lens = instance(200 + len(name), **inst)
    path = str(tmp_path / "model.bin")
    write_model(path, model, enc, lens)
    rows = run(path, *args, "--algos", "greedy,alsd++,aes++,aes-ref")
    assert len(rows) == 8
    for algo, ref, b200 in pairs(rows):
        assert len(ref["streams"]) == len(b200["streams"]) == len(lens)
        for s, (x, y) in enumerate(zip(ref["streams"], b200["streams"])):
            assert [n["tokens"] for n in x["nbest"]] == [n["tokens"] for n in y["nbest"]], (algo, s)
            for a, b in zip(x["nbest"], y["nbest"]):
                assert abs(a["score"] - b["score"]) <= 1e-4, (algo, s, a["score"], b["score"])
            assert x["counters"] == y["counters"], (algo, s)


@pytest.mark.gpu
def test_adapter_bench_grid(tmp_path):
    """cmd_bench's grid (algo x batch x beam, warm-up + repeats, RTFx) over the
    reference's and the B200's DecodeFn."""
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/ref_adapter_demo not built")
    model, enc, lens = instance(300, V=32, D=16, J=32, B=8, T=40, ragged=False)
    path = str(tmp_path / "model.bin")
    write_model(path, model, enc, lens)
    rows = run(path, "--bench", "--algos", "alsd++,alsd++-b200,greedy-b200", "--batch-grid", "2,8",
               "--beam-grid", "2,4", "--repeats", "2")
    assert len(rows) == 3 * 2 * 2
    for r in rows:
        assert r["frames"] == 8 * 40 and r["rtfx"] > 0
