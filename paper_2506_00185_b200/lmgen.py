"""Synthetic large, CONSISTENT-backoff ARPA n-gram LM (BASELINE configs 4/5:
"~1M n-grams, V=1024").

The reference's own generator (make_random_consistent_arpa,
proj/src/fixtures.cpp:155-248) yields only ~8k n-grams at V=1024.  This scales
the same recipe, vectorised over whole levels with numpy:

  * unigrams: a full random distribution over the V tokens and </s>; <s> has
    only a backoff (rendered -99);
  * level k >= 2: contexts are (k-1)-grams not ending in </s>; a kept context
    c picks a few continuation words w, whose raw weight is (0.5 + u) times
    the already-built model's fully backed-off P(w | suffix(c)); a mass
    m in [0.3, 0.8) is spread over them in proportion, and c's backoff is set
    to (1 - m) / (1 - sum_w P(w | suffix(c))) -- so every context's
    distribution over V + </s> sums to one (test_lm_build.py checks it on the
    reference's own scorer).

Contexts whose continuations already carry >= 0.999 of the lower-order mass
are skipped, like the reference's.  Keys are int64 codes in base V + 2 (order
<= 5 at V <= 8192 fits), looked up with searchsorted.

  python scripts/make_arpa.py --vocab 1024 --order 4 --ngrams 1000000 > lm.arpa
  (or python -m paper_2506_00185_b200.lmgen ...)
"""
import argparse
import sys

import numpy as np

from .model import synthetic_vocabulary


class _Level:
    """The k-grams of one order: sorted codes, linear prob and backoff."""

    def __init__(self, codes, prob, backoff, has_bo):
        o = np.argsort(codes, kind="stable")
        self.codes, self.prob, self.bo, self.has_bo = codes[o], prob[o], backoff[o], has_bo[o]

    def find(self, codes):
        i = np.searchsorted(self.codes, codes)
        i = np.minimum(i, len(self.codes) - 1)
        hit = self.codes[i] == codes if len(self.codes) else np.zeros(len(codes), bool)
        return i, hit


def make_consistent_arpa(vocab: int, order: int, ngrams: int, seed: int = 1) -> str:
    rng = np.random.default_rng(seed)
    V = vocab
    eos, bos = V, V + 1
    base = np.int64(V + 2)
    names = synthetic_vocabulary(vocab) + ["</s>", "<s>"]
    assert (V + 2) ** order < 2 ** 62, "codes overflow int64"

    def code(seqs):  # [n, L] -> int64
        c = np.zeros(len(seqs), np.int64)
        for j in range(seqs.shape[1]):
            c = c * base + seqs[:, j].astype(np.int64)
        return c

    levels = []
    # unigrams (+ <s>, backoff only)
    events = np.arange(V + 1)
    mass = 0.2 + rng.random(V + 1)
    uni_p = np.concatenate([mass / mass.sum(), [1.0]])
    uni_seq = np.arange(V + 2)[:, None]
    uni_hb = np.full(V + 2, order > 1)
    uni_hb[eos] = False
    levels.append(_Level(code(uni_seq), uni_p, np.ones(V + 2), uni_hb))
    seqs = [uni_seq[np.argsort(code(uni_seq))]]

    def score(ctx, w):
        """fully backed-off P(w | ctx) of the model built so far; ctx [n, L]"""
        n, L = ctx.shape
        out = np.zeros(n)
        mult = np.ones(n)
        todo = np.ones(n, bool)
        for l in range(L, -1, -1):  # longest context first
            sub = ctx[:, L - l:]
            key = code(np.concatenate([sub, w[:, None]], axis=1))
            i, hit = levels[l].find(key)
            take = todo & hit
            out[take] = mult[take] * levels[l].prob[i[take]]
            todo &= ~hit
            if l > 0:
                ci, chit = levels[l - 1].find(code(sub))
                mult = np.where(todo & chit, mult * levels[l - 1].bo[ci], mult)
        return out

    # continuation counts per level, scaled to the requested total
    rest = max(ngrams - (V + 2), 0)
    per = {2: 64, 3: 5, 4: 2, 5: 2, 6: 2}
    keep = {2: 1.0, 3: 1.0, 4: 0.75, 5: 0.5, 6: 0.5}
    est, n_ctx = 0, V
    for k in range(2, order + 1):
        est += n_ctx * keep[k] * per[k]
        n_ctx = int(n_ctx * keep[k] * per[k])
    scale = rest / est if est else 1.0
    for k in range(2, order + 1):
        prev = seqs[-1]
        ctxs = prev[prev[:, -1] != eos]
        kept = ctxs[(rng.random(len(ctxs)) < keep[k]) | (ctxs[:, 0] == bos)]
        m = max(1, int(round(per[k] * (scale if k == 2 else scale ** (1.0 / (order - 1))))))
        m = min(m, V + 1)
        # m distinct continuation events per context
        nc = len(kept)
        cont = np.argsort(rng.random((nc, V + 1)), axis=1)[:, :m] if m * 4 > V else \
            rng.integers(0, V + 1, size=(nc, m))
        ctx_rep = np.repeat(kept, m, axis=0)
        w = events[cont.reshape(-1)]
        # drop duplicate (ctx, w) pairs
        full = np.concatenate([ctx_rep, w[:, None]], axis=1)
        fcode = code(full)
        _, first = np.unique(fcode, return_index=True)
        sel = np.zeros(len(fcode), bool)
        sel[first] = True
        ctx_id = np.repeat(np.arange(nc), m)[sel]
        full, w, ctx_rep = full[sel], w[sel], ctx_rep[sel]
        lower = score(ctx_rep[:, 1:], w)
        raw = (0.5 + rng.random(len(w))) * lower
        lower_tot = np.bincount(ctx_id, lower, minlength=nc)
        raw_tot = np.bincount(ctx_id, raw, minlength=nc)
        ok_ctx = (lower_tot < 0.999) & (raw_tot > 0.0)
        ctx_mass = 0.3 + 0.5 * rng.random(nc)
        ok = ok_ctx[ctx_id]
        prob = ctx_mass[ctx_id] * raw / np.where(raw_tot[ctx_id] > 0, raw_tot[ctx_id], 1.0)
        # the contexts' backoffs (level k - 1)
        pl = levels[k - 2]
        ci, chit = pl.find(code(kept[ok_ctx]))
        assert chit.all()
        pl.bo[ci] = (1.0 - ctx_mass[ok_ctx]) / (1.0 - lower_tot[ok_ctx])
        pl.has_bo[ci] = True
        full, prob, w = full[ok], prob[ok], w[ok]
        hb = np.full(len(full), k < order) & (w != eos)
        lev = _Level(code(full), prob, np.ones(len(full)), hb)
        levels.append(lev)
        seqs.append(full[np.argsort(code(full), kind="stable")])

    out = ["\\data\\"]
    out += [f"ngram {k}={len(lv.codes)}" for k, lv in enumerate(levels, 1)]
    out.append("")
    for k, (lv, sq) in enumerate(zip(levels, seqs), 1):
        out.append(f"\\{k}-grams:")
        lp = np.log10(lv.prob)
        lb = np.log10(lv.bo)
        for i in range(len(sq)):
            toks = " ".join(names[t] for t in sq[i])
            p = "-99" if (k == 1 and sq[i, 0] == bos) else f"{lp[i]:.9g}"
            out.append(f"{p}\t{toks}\t{lb[i]:.9g}" if lv.has_bo[i] else f"{p}\t{toks}")
        out.append("")
    out.append("\\end\\")
    return "\n".join(out) + "\n"


# the name the bench / config scripts import
make_arpa = make_consistent_arpa


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
    sys.stdout.write(make_consistent_arpa(a.vocab, a.order, a.ngrams, a.seed))
