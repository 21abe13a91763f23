"""Synthetic large ARPA n-gram LM for throughput runs (BASELINE configs 4/5:
"~1M n-grams, V=1024").  The reference's own generator
(make_random_consistent_arpa, fixtures.cpp:155-248) yields only ~8k n-grams
at V=1024, so this scales the same recipe -- every k-gram extends an
existing (k-1)-gram context, probabilities and backoffs are log10 values --
without renormalising each context (speed runs only; parity runs use the
reference's consistent generator).

  python scripts/make_arpa.py --vocab 1024 --order 4 --ngrams 1000000 > lm.arpa
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_00185_b200.model import synthetic_vocabulary  # noqa: E402


def make_arpa(vocab: int, order: int, ngrams: int, seed: int = 1) -> str:
    rng = np.random.default_rng(seed)
    words = synthetic_vocabulary(vocab) + ["</s>", "<s>"]
    V = vocab
    eos, bos = V, V + 1
    per_order = [V + 2]
    rest = max(ngrams - (V + 2), 0)
    # geometric split of the remaining n-grams over orders 2..N
    if order > 1:
        w = np.array([2.0 ** k for k in range(order - 1)])
        per_order += [int(x) for x in rest * w / w.sum()]
    levels = []
    # unigrams
    uni = np.arange(V + 2)
    lp = np.log10(rng.dirichlet(np.ones(V + 1)))
    u_lp = np.concatenate([lp, [-99.0]])  # <s> has no probability
    u_bo = np.log10(rng.uniform(0.2, 0.9, size=V + 2)) if order > 1 else None
    levels.append((uni[:, None], u_lp, u_bo))
    for k in range(2, order + 1):
        prev = levels[-1][0]
        # contexts: previous-order entries not ending in </s>
        ctx_ok = prev[:, -1] != eos
        ctxs = prev[ctx_ok]
        n = per_order[k - 1]
        pick = rng.integers(0, len(ctxs), size=n)
        cont = rng.integers(0, V + 1, size=n)  # tokens or </s>
        grams = np.concatenate([ctxs[pick], cont[:, None]], axis=1)
        grams = np.unique(grams, axis=0)
        g_lp = np.log10(rng.uniform(0.01, 0.6, size=len(grams)))
        g_bo = np.log10(rng.uniform(0.2, 0.9, size=len(grams))) if k < order else None
        levels.append((grams, g_lp, g_bo))
    out = ["\\data\\"]
    for k, (g, _, _) in enumerate(levels, 1):
        out.append(f"ngram {k}={len(g)}")
    out.append("")
    for k, (g, lp, bo) in enumerate(levels, 1):
        out.append(f"\\{k}-grams:")
        for i in range(len(g)):
            toks = " ".join(words[t] for t in g[i])
            if bo is not None and g[i, -1] != eos:
                out.append(f"{lp[i]:.6f}\t{toks}\t{bo[i]:.6f}")
            else:
                out.append(f"{lp[i]:.6f}\t{toks}")
        out.append("")
    out.append("\\end\\")
    return "\n".join(out) + "\n"


def arpa_successors(text: str, vocab: int, cap: int = 16) -> np.ndarray:
    """successors[v] = up to `cap` ASR ids w with a bigram "v w" in the ARPA
    (-1 padded): drives the synthetic encoder's token stream (model.py)."""
    words = synthetic_vocabulary(vocab)
    ids = {w: i for i, w in enumerate(words)}
    succ = np.full((vocab, cap), -1, np.int32)
    n = np.zeros(vocab, np.int32)
    sec = False
    for line in text.splitlines():
        if line.startswith("\\2-grams:"):
            sec = True
            continue
        if sec:
            if not line or line.startswith("\\"):
                break
            parts = line.split("\t")
            if len(parts) < 2:
                continue
            ws = parts[1].split(" ")
            a, b = ids.get(ws[0], -1), ids.get(ws[1], -1)
            if a >= 0 and b >= 0 and n[a] < cap:
                succ[a, n[a]] = b
                n[a] += 1
    return succ


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("--vocab", type=int, default=1024)
    p.add_argument("--order", type=int, default=4)
    p.add_argument("--ngrams", type=int, default=1_000_000)
    p.add_argument("--seed", type=int, default=1)
    a = p.parse_args()
    sys.stdout.write(make_arpa(a.vocab, a.order, a.ngrams, a.seed))
