"""Output path after the decode: detokenisation of the
n-best token sequences and corpus WER, host-side like the reference's
(metrics.cpp:16-125).  The decode itself hands back token ids; these turn
them into words and score them.

* ``wer(refs, hyps)``: per-pair Levenshtein alignment with unit costs; the
  S/I/D decomposition is made deterministic by preferring, on equal cost, the
  diagonal (match / substitution), then deletion, then insertion (the tie
  order of metrics.cpp:36-49); counts are pooled over the corpus before
  dividing; an empty reference corpus raises (metrics.cpp:86-88).
* ``detokenize(vocab, tokens)``: pieces starting with the word marker U+2581
  open a new word (marker stripped), others continue the current one
  (metrics.cpp:95-111), then whitespace split (metrics.cpp:113-125).
"""
from __future__ import annotations

from dataclasses import dataclass
import re
from typing import List, Sequence

WORD_MARKER = "▁"


@dataclass
class WerReport:
    substitutions: int = 0
    insertions: int = 0
    deletions: int = 0
    reference_words: int = 0

    def wer(self) -> float:
        return (self.substitutions + self.insertions + self.deletions) / self.reference_words


def _align(ref: Sequence[str], hyp: Sequence[str], rep: WerReport) -> None:
    nr, nh = len(ref), len(hyp)
    # rolling DP rows of (cost, op) with op 0 = diag, 1 = del, 2 = ins; the
    # full back-pointer table is kept for the deterministic traceback
    back = [[0] * (nh + 1) for _ in range(nr + 1)]
    prev = list(range(nh + 1))
    for j in range(1, nh + 1):
        back[0][j] = 2
    for i in range(1, nr + 1):
        cur = [i] + [0] * nh
        back[i][0] = 1
        ri = ref[i - 1]
        for j in range(1, nh + 1):
            best = prev[j - 1] + (0 if ri == hyp[j - 1] else 1)
            op = 0
            if prev[j] + 1 < best:
                best, op = prev[j] + 1, 1
            if cur[j - 1] + 1 < best:
                best, op = cur[j - 1] + 1, 2
            cur[j] = best
            back[i][j] = op
        prev = cur
    i, j = nr, nh
    while i > 0 or j > 0:
        op = back[i][j]
        if op == 0:
            if ref[i - 1] != hyp[j - 1]:
                rep.substitutions += 1
            i -= 1
            j -= 1
        elif op == 1:
            rep.deletions += 1
            i -= 1
        else:
            rep.insertions += 1
            j -= 1
    rep.reference_words += nr


def wer(refs: Sequence[Sequence[str]], hyps: Sequence[Sequence[str]]) -> WerReport:
    if len(refs) != len(hyps):
        raise ValueError("wer: reference/hypothesis count mismatch")
    rep = WerReport()
    for r, h in zip(refs, hyps):
        _align(r, h, rep)
    if rep.reference_words == 0:
        raise ValueError("wer: empty reference corpus, WER undefined")
    return rep


def detokenize_text(vocab: Sequence[str], tokens: Sequence[int]) -> str:
    text = ""
    for t in tokens:
        # Vocabulary::token uses tokens_.at(id): an id outside the table throws
        if t < 0 or t >= len(vocab):
            raise IndexError(f"detokenize: token id {t} outside the vocabulary (size {len(vocab)})")
        piece = vocab[t]
        if piece.startswith(WORD_MARKER):
            if text:
                text += " "
            text += piece[len(WORD_MARKER):]
        else:
            text += piece
    return text


def detokenize(vocab: Sequence[str], tokens: Sequence[int]) -> List[str]:
    # istringstream >> splits on ASCII whitespace only (not Unicode spaces)
    return [w for w in re.split("[ \t\n\v\f\r]+", detokenize_text(vocab, tokens)) if w]
