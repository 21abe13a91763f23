"""Output-path helpers (paper_2506_00185_b200/metrics.py) against the
reference's own known answers (proj/tests/test_metrics.cpp:72-160) and an
independent edit-distance recursion."""
import functools
import random

import pytest

from paper_2506_00185_b200.metrics import WerReport, detokenize, wer
from paper_2506_00185_b200.model import synthetic_vocabulary


def test_wer_known_answers():
    refs = [["a", "b", "c"]]
    r = wer(refs, [["a", "b", "c"]])
    assert r.wer() == 0.0 and r.substitutions == 0
    r = wer(refs, [["a", "x", "c"]])
    assert (r.substitutions, r.insertions, r.deletions) == (1, 0, 0)
    assert r.wer() == pytest.approx(1.0 / 3.0)
    r = wer(refs, [["a", "b", "c", "p", "q"]])  # appending k words costs k insertions
    assert (r.substitutions, r.insertions, r.deletions) == (0, 2, 0)
    with pytest.raises(ValueError):
        wer([[]], [[]])
    with pytest.raises(ValueError):
        wer([["a"]], [])


def _edit_distance(a, b):
    @functools.lru_cache(maxsize=None)
    def d(i, j):
        if i == 0:
            return j
        if j == 0:
            return i
        return min(d(i - 1, j - 1) + (a[i - 1] != b[j - 1]), d(i - 1, j) + 1, d(i, j - 1) + 1)
    return d(len(a), len(b))


def test_wer_total_matches_edit_distance():
    rng = random.Random(5)
    alphabet = ["w%d" % i for i in range(5)]
    refs, hyps, total, nref = [], [], 0, 0
    for _ in range(60):
        r = [rng.choice(alphabet) for _ in range(rng.randint(1, 9))]
        h = [rng.choice(alphabet) for _ in range(rng.randint(0, 9))]
        refs.append(r)
        hyps.append(h)
        total += _edit_distance(tuple(r), tuple(h))
        nref += len(r)
    rep = wer(refs, hyps)
    assert rep.substitutions + rep.insertions + rep.deletions == total
    assert rep.reference_words == nref
    # deterministic decomposition: deletion-only and insertion-only pairs
    assert wer([["a", "b"]], [[]]).deletions == 2
    assert wer([["a"]], [["a", "b", "c"]]).insertions == 2


def test_detokenize_word_marker():
    v = synthetic_vocabulary(6)
    assert v[0].startswith("▁") and not v[1].startswith("▁")
    w = detokenize(v, [0, 1, 2, 3, 4])
    assert w == [v[0][1:] + v[1] + v[2], v[3][1:] + v[4]]
    assert len(detokenize(v, [1])) == 1  # a dangling continuation still forms a word
    assert detokenize(v, []) == []
    assert isinstance(WerReport().substitutions, int)
