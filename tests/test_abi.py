"""CPU checks of the C-ABI boundary: the sm_100a library builds/loads, exports
every entry point include/tbeam_b200.h declares, its struct layouts match the
C header, defaults mirror the reference's DecodeConfig, the host-side ARPA
parser mirrors NGramLm::parse_arpa_text, and -- with no GPU -- it refuses to
run instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2506_00185_b200 import _abi
from paper_2506_00185_b200.decoder import (LIB_PATH, ParseError, load_library, parse_arpa_check,
                                           symbols)
from paper_2506_00185_b200.model import synthetic_vocabulary
from tests.conftest import ROOT, have_gpu

HEADER = os.path.join(ROOT, "include", "tbeam_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB_PATH):
        from paper_2506_00185_b200.build import build
        build()
    return load_library()


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tbeam_[a-z_]+)\s*\(", text)))


def test_exports_every_header_symbol(lib):
    declared = header_functions()
    assert set(declared) == set(symbols())
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tbeam_\w+)", out))
    for name in declared:
        assert name in exported, name
        assert hasattr(lib, name)


def test_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(f'#include "{HEADER}"\n#include <stdio.h>\n#include <stddef.h>\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(tbeam_decode_config),'
                   ' sizeof(tbeam_model_dims), sizeof(tbeam_model_weights), sizeof(tbeam_results),'
                   ' offsetof(tbeam_decode_config, hash_base), offsetof(tbeam_results, counters));}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(_abi.CDecodeConfig), C.sizeof(_abi.CModelDims), C.sizeof(_abi.CModelWeights),
            C.sizeof(_abi.CResults), _abi.CDecodeConfig.hash_base.offset,
            _abi.CResults.counters.offset]
    assert got == want


def test_config_defaults_mirror_reference(lib):
    """decoder.hpp:23-42, fusion.hpp:19-24, hyp_store.hpp:15-18."""
    c = _abi.CDecodeConfig()
    lib.tbeam_decode_config_init(C.byref(c))
    py = _abi.DecodeConfig().to_c(_abi.ALGO_ALSD)
    for name, _ in _abi.CDecodeConfig._fields_:
        if name == "reserved":
            continue
        assert getattr(c, name) == getattr(py, name), name
    assert (c.beam, c.max_symbols_per_frame, c.aes_expansions_per_frame, c.max_len) == (4, 10, 2, 256)
    assert c.hash_base == 1_000_003 and c.hash_modulus == (1 << 61) - 1


@pytest.mark.skipif(have_gpu(), reason="checks the no-GPU refusal path")
def test_no_cpu_fallback(lib):
    ctx = C.c_void_p()
    rc = lib.tbeam_create(0, C.byref(ctx))
    assert rc == _abi.TBEAM_UNSUPPORTED
    assert b"device" in lib.tbeam_last_error()


def test_arpa_parse_matches_reference_semantics(ref):
    """Product ARPA parser vs NGramLm::parse_arpa_text on the reference's own
    generator output: same order and node count."""
    for seed, V, order in [(1, 10, 2), (2, 40, 3), (3, 64, 4)]:
        arpa = ref.random_arpa(seed, V, order)
        info = parse_arpa_check(arpa, synthetic_vocabulary(V))
        rlm = ref.lm(arpa, V)
        assert info["order"] == ref.lib.ref_lm_order(rlm.ptr)
        assert info["nodes"] == ref.lib.ref_lm_num_nodes(rlm.ptr)
        assert info["edges"] == info["nodes"] - 1


BAD_ARPA = {
    "no data": "hello\n",
    "missing end": "\\data\\\nngram 1=1\n\n\\1-grams:\n-1.0\ta\n",
    "count mismatch": "\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0\t▁a\n\\end\\\n",
    "non contiguous": "\\data\\\nngram 2=1\n",
    "bad fields": "\\data\\\nngram 1=1\n\n\\1-grams:\n-1.0\n\\end\\\n",
    "bad prob": "\\data\\\nngram 1=1\n\n\\1-grams:\nabc\t▁a\n\\end\\\n",
}


@pytest.mark.parametrize("name", sorted(BAD_ARPA))
def test_arpa_parse_errors(lib, name, ref):
    """ngram_lm.cpp:112-226: the same inputs are ParseErrors for both."""
    vocab = synthetic_vocabulary(4)
    with pytest.raises(ParseError):
        parse_arpa_check(BAD_ARPA[name], vocab)
    with pytest.raises(ValueError):
        ref.lm(BAD_ARPA[name], 4)


def test_arpa_strict_oov(lib):
    text = "\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0\t▁a\n-1.0\tzzz\n\\end\\\n"
    vocab = synthetic_vocabulary(4)
    assert parse_arpa_check(text, vocab)["oov_mapped"] == 1
    with pytest.raises(ParseError):
        parse_arpa_check(text, vocab, strict=True)
