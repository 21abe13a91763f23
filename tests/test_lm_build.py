"""The product ARPA -> trie builder (csrc/lm_build.cpp) against the reference's
NGramLm (proj/src/ngram_lm.cpp:52-438), on the CPU.

The builder's frozen arrays (tbeam_lm_export) are walked here with the same
queries the device runs (csrc/device_fns.cuh: lm_score_token, lm_advance,
lm_vocab_value, lm_score_eos -- restated below in Python), and compared with
the reference's own queries on random histories: score_token / score_eos
exactly, score_vocab rows exactly.  Malformed inputs must be ParseErrors for
both parsers."""
import math

import numpy as np
import pytest

from paper_2506_00185_b200.decoder import ParseError, lm_export, parse_arpa_check
from paper_2506_00185_b200.model import synthetic_vocabulary

FLOOR = -1e9


class Walker:
    """device_fns.cuh's LM queries over the exported arrays."""

    def __init__(self, a):
        self.a = a
        self.V = a["V"]
        self.order = a["order"]
        root = {}
        for e in range(a["cbeg"][0], a["cend"][0]):
            root[int(a["etok"][e])] = int(a["enode"][e])
        self.root = root
        unk = self.child(0, self.V + 2)
        self.unk = a["prob"][unk] if unk >= 0 and not math.isnan(a["prob"][unk]) else -math.inf

    def child(self, node, tok):
        a = self.a
        lo, hi = int(a["cbeg"][node]), int(a["cend"][node])
        et = a["etok"]
        while lo < hi:
            mid = (lo + hi) >> 1
            if et[mid] < tok:
                lo = mid + 1
            else:
                hi = mid
        if lo < a["cend"][node] and et[lo] == tok:
            return int(a["enode"][lo])
        return -1

    def internal(self, state, tok):
        a = self.a
        acc, c = 0.0, state
        while True:
            n = self.child(c, tok)
            if n >= 0 and not math.isnan(a["prob"][n]):
                return max(acc + a["prob"][n], FLOOR)
            if c == 0:
                return None
            acc += a["backoff"][c]
            c = int(a["suffix"][c])

    def score_token(self, state, tok):
        it = int(self.a["remap"][tok])
        if it < 0:
            return FLOOR
        v = self.internal(state, it)
        return FLOOR if v is None else v

    def score_eos(self, state):
        v = self.internal(state, self.V + 1)
        return FLOOR if v is None else v

    def vocab_value(self, state, tok):
        a = self.a
        acc, c = 0.0, state
        while True:
            n = self.child(c, tok)
            if n >= 0 and not math.isnan(a["prob"][n]):
                return max(acc + a["prob"][n], FLOOR)
            if c == 0:
                break
            acc += a["backoff"][c]
            c = int(a["suffix"][c])
        return max(acc + self.unk, FLOOR) if math.isfinite(self.unk) else FLOOR

    def advance(self, state, tok):
        a = self.a
        it = int(a["remap"][tok])
        if it < 0:
            return 0
        c = state
        while True:
            n = self.child(c, it)
            if n >= 0:
                return int(a["suffix"][n]) if a["depth"][n] == self.order else n
            if c == 0:
                return 0
            c = int(a["suffix"][c])

    def state(self, hist):
        s = self.a["initial"]
        for t in hist:
            s = self.advance(s, t)
        return s


@pytest.mark.parametrize("seed,V,order", [(1, 10, 2), (2, 40, 3), (3, 64, 4), (7, 24, 5)])
def test_queries_match_reference(ref, seed, V, order):
    arpa = ref.random_arpa(seed, V, order)
    vocab = synthetic_vocabulary(V)
    a = lm_export(arpa, vocab)
    w = Walker(a)
    rlm = ref.lm(arpa, V)
    assert a["order"] == ref.lib.ref_lm_order(rlm.ptr)
    assert a["nodes"] == ref.lib.ref_lm_num_nodes(rlm.ptr)
    rng = np.random.default_rng(seed)
    for rep in range(60):
        hist = [int(x) for x in rng.integers(0, V, size=int(rng.integers(0, 2 * order + 1)))]
        s = w.state(hist)
        for tok in rng.integers(0, V, size=6):
            assert w.score_token(s, int(tok)) == ref.lm_score_token(rlm, hist, int(tok)), (hist, tok)
        assert w.score_eos(s) == ref.lm_score_eos(rlm, hist), hist
        if rep % 6 == 0:
            row = ref.lm_score_vocab(rlm, hist, V)
            mine = np.array([w.vocab_value(s, t) for t in range(V)])
            np.testing.assert_array_equal(mine, row)


def test_children_are_contiguous_sorted_ranges(ref):
    """Level-sorted layout: edge e is node e + 1, every child list sorted."""
    a = lm_export(ref.random_arpa(5, 32, 4), synthetic_vocabulary(32))
    assert (a["enode"][: a["edges"]] == np.arange(1, a["nodes"])).all()
    for x in range(a["nodes"]):
        b, e = a["cbeg"][x], a["cend"][x]
        assert b <= e
        toks = a["etok"][b:e]
        assert (np.diff(toks) > 0).all()
        assert (a["depth"][a["enode"][b:e]] == a["depth"][x] + 1).all()
    # suffix links point one or more levels up
    assert (a["depth"][a["suffix"][1:]] < a["depth"][1:]).all()


def test_repeated_ngram_last_wins_backoff_only_when_given(ref):
    """ngram_lm.cpp:208-214: a repeat overwrites the probability; the backoff
    only when the repeat lists one."""
    V = 4
    vocab = synthetic_vocabulary(V)
    a0, a1 = vocab[0], vocab[1]
    text = ("\\data\\\nngram 1=4\nngram 2=1\n\n\\1-grams:\n"
            f"-1.0\t{a0}\t-0.5\n-1.2\t{a1}\n-2.0\t{a0}\n-0.7\t</s>\n\n"
            f"\\2-grams:\n-0.3\t{a0} {a1}\n\\end\\\n")
    a = lm_export(text, vocab)
    w = Walker(a)
    rlm = ref.lm(text, V)
    n0 = w.child(0, 0)
    assert a["prob"][n0] == pytest.approx(-2.0 * math.log(10), abs=0)
    assert a["backoff"][n0] == pytest.approx(-0.5 * math.log(10), abs=0)
    for hist in ([], [0], [1], [0, 1], [1, 0]):
        s = w.state(hist)
        for t in range(V):
            assert w.score_token(s, t) == ref.lm_score_token(rlm, hist, t)


BAD = {
    "no data": "hello\n",
    "missing end": "\\data\\\nngram 1=1\n\n\\1-grams:\n-1.0\ta\n",
    "count mismatch": "\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0\t▁a\n\\end\\\n",
    "non contiguous": "\\data\\\nngram 2=1\n",
    "bad fields": "\\data\\\nngram 1=1\n\n\\1-grams:\n-1.0\n\\end\\\n",
    "bad prob": "\\data\\\nngram 1=1\n\n\\1-grams:\nabc\t▁a\n\\end\\\n",
    "bad backoff": "\\data\\\nngram 1=1\n\n\\1-grams:\n-1\t▁a\txyz\n\\end\\\n",
    "overflow prob": "\\data\\\nngram 1=1\n\n\\1-grams:\n-1e999\t▁a\n\\end\\\n",
    "bad count line": "\\data\\\nngram x=1\n\\end\\\n",
    "count line without =": "\\data\\\nngram 1 1\n\\end\\\n",
    "end before sections": "\\data\\\nngram 1=1\n\\end\\\n",
    "no orders": "\\data\\\n\\end\\\n",
    "entry before header": "\\data\\\nngram 1=1\n-1.0\t▁a\n\\end\\\n",
    "section out of order": "\\data\\\nngram 1=1\nngram 2=1\n\\2-grams:\n-1 ▁a ▁b\n\\end\\\n",
    "section beyond declared": "\\data\\\nngram 1=1\n\\1-grams:\n-1 ▁a\n\\2-grams:\n\\end\\\n",
    "bad section number": "\\data\\\nngram 1=1\n\\x-grams:\n\\end\\\n",
    "missing higher section": "\\data\\\nngram 1=1\nngram 2=1\n\\1-grams:\n-1 ▁a\n\\end\\\n",
}


@pytest.mark.parametrize("name", sorted(BAD))
def test_malformed_is_parse_error_for_both(ref, name):
    vocab = synthetic_vocabulary(4)
    with pytest.raises(ParseError) as e:
        parse_arpa_check(BAD[name], vocab)
    assert str(e.value).startswith("lm.arpa:")
    with pytest.raises(ValueError):
        ref.lm(BAD[name], 4)


GOOD = {
    "crlf and blanks": "junk\r\n\r\n\\data\\\r\nngram 1=2\r\n\r\n\\1-grams:\r\n-1.0\t▁a\r\n \t\r\n-1.0\t▁b\r\n\\end\\\r\n",
    "trailing text after numbers": "\\data\\\nngram 1=2xyz\n\\1-grams:\n-1.0abc ▁a -0.1q\n-2 ▁b\n\\end\\\n",
    "no final newline": "\\data\\\nngram 1=1\n\\1-grams:\n-1 ▁a\n\\end\\",
    "unk upper": "\\data\\\nngram 1=2\n\\1-grams:\n-1 ▁a\n-3 <UNK>\n\\end\\\n",
    "text after end ignored": "\\data\\\nngram 1=1\n\\1-grams:\n-1 ▁a\n\\end\\\ngarbage here\n",
}


@pytest.mark.parametrize("name", sorted(GOOD))
def test_accepted_inputs_agree(ref, name):
    V = 4
    vocab = synthetic_vocabulary(V)
    a = lm_export(GOOD[name], vocab)
    rlm = ref.lm(GOOD[name], V)
    assert a["nodes"] == ref.lib.ref_lm_num_nodes(rlm.ptr)
    w = Walker(a)
    for hist in ([], [0], [1, 2]):
        for t in range(V):
            assert w.score_token(w.state(hist), t) == ref.lm_score_token(rlm, hist, t)


def test_strict_oov_and_counting():
    vocab = synthetic_vocabulary(4)
    text = "\\data\\\nngram 1=2\nngram 2=1\n\n\\1-grams:\n-1.0\t▁a\n-1.0\tzzz\n\\2-grams:\n-1 zzz qqq\n\\end\\\n"
    assert parse_arpa_check(text, vocab)["oov_mapped"] == 3  # every OOV occurrence
    with pytest.raises(ParseError):
        parse_arpa_check(text, vocab, strict=True)


def test_scaled_generator_is_consistent(ref):
    """paper_2506_00185_b200/lmgen.py (the C4/C5 LM recipe, fixtures.cpp:155-248 scaled):
    every context's distribution over V + </s> sums to one under the
    reference's own backoff scorer, and the product parser agrees with it."""
    from paper_2506_00185_b200.lmgen import make_consistent_arpa
    V = 24
    text = make_consistent_arpa(V, 4, 4000, seed=3)
    rlm = ref.lm(text, V)
    a = lm_export(text, synthetic_vocabulary(V))
    assert a["order"] == 4 and a["nodes"] == ref.lib.ref_lm_num_nodes(rlm.ptr)
    assert a["nodes"] > 1500
    w = Walker(a)
    rng = np.random.default_rng(0)
    for _ in range(40):
        hist = [int(x) for x in rng.integers(0, V, size=int(rng.integers(0, 6)))]
        row = ref.lm_score_vocab(rlm, hist, V)
        total = np.exp(row).sum() + math.exp(ref.lm_score_eos(rlm, hist))
        assert abs(total - 1.0) < 1e-6, (hist, total)
        s = w.state(hist)
        np.testing.assert_array_equal([w.vocab_value(s, t) for t in range(V)], row)
