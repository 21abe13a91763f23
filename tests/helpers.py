"""Shared builders for the parity tests: seeded synthetic transducers,
encoder frames, configs, and result comparison."""
from __future__ import annotations

import numpy as np

from paper_2506_00185_b200 import _abi
from paper_2506_00185_b200.model import (SyntheticTransducer, TransducerSpec,
                                         synthetic_encoder_frames)


def instance(seed: int, kind: int = _abi.PRED_STATELESS, V: int = 12, D: int = 8, J: int = 16,
             B: int = 3, T: int = 12, n: int = 2, H: int = 12, E: int = 8, durations=(),
             precision: int = _abi.PREC_FP32, blank_bias=None, logit_scale: float = 3.0,
             ragged: bool = True):
    rng = np.random.default_rng(seed + 1000)
    bb = blank_bias if blank_bias is not None else float(np.log(V) + rng.uniform(-1.0, 2.5))
    spec = TransducerSpec(vocab_size=V, enc_dim=D, joint_dim=J, pred_kind=kind, context_order=n,
                          lstm_hidden=H, emb_dim=E, durations=tuple(durations),
                          precision=precision, seed=seed, blank_bias=bb, logit_scale=logit_scale)
    model = SyntheticTransducer(spec)
    enc = synthetic_encoder_frames(seed + 7, B, T, D)
    if ragged:
        lens = [T] + [int(x) for x in rng.integers(1, T + 1, size=B - 1)]
    else:
        lens = [T] * B
    return model, enc, lens


def same_tokens(a, b) -> bool:
    return all([e.tokens for e in x.nbest] == [e.tokens for e in y.nbest]
               for x, y in zip(a.streams, b.streams))


def max_score_diff(a, b) -> float:
    worst = 0.0
    for x, y in zip(a.streams, b.streams):
        for ex, ey in zip(x.nbest, y.nbest):
            if ex.score == ey.score:
                continue
            worst = max(worst, abs(ex.score - ey.score))
    return worst


def describe(a, b) -> str:
    out = []
    for s, (x, y) in enumerate(zip(a.streams, b.streams)):
        tx = [(e.tokens, round(e.score, 6)) for e in x.nbest]
        ty = [(e.tokens, round(e.score, 6)) for e in y.nbest]
        if tx != ty:
            out.append(f"stream {s}:\n  a={tx}\n  b={ty}")
    return "\n".join(out[:3])


def margin_ok(result, min_margin: float) -> bool:
    """True when every stream's n-best scores are separated by > min_margin
    (the parity contract: tokens must match where the margin exceeds the fp
    tolerance)."""
    for s in result.streams:
        sc = [e.score for e in s.nbest]
        for i in range(len(sc) - 1):
            if abs(sc[i] - sc[i + 1]) <= min_margin:
                return False
    return True


def check_parity(gpu, orc, tol: float, max_exempt: int = None, label: str = "",
                 counter_rtol: float = 0.0, verify=None, tol_at=None) -> dict:
    """The parity contract (BASELINE.json north star) between a GPU result and
    the oracle's, stream by stream:

    * n-best scores agree rank by rank within `tol`; where the token sequences
      agree, frames, durations and the per-stream counters agree too (counters
      exactly, or within `counter_rtol` relative for long bf16 decodes: a
      near-tie at the beam's K-th place can swap a hypothesis for another of
      equal score within the tolerance and change the work done later);
    * a stream that does not agree is exempt only at a near-tie the fp
      tolerance cannot order:
        - with `verify` (stream index -> first_divergence(...) result): the
          per-round traces must diverge at a round where the oracle's own
          prune margin (K-th kept - best rejected) is <= 2 tol (or 2
          tol_at(frame) -- the bound accumulated up to that frame);
        - without: the n-best scores still agree within tol and the first
          differing entry i is a near-tie of the oracle's ranking
          (score[i] - score[i+1] <= tol) or the last entry;
    * exemptions are counted and capped: trace-verified ones at
      max(1, streams // 4), the others at max(1, streams // 8) (or `max_exempt`).

    Returns {"streams", "exact", "exempt": [...], "max_abs_dscore"}."""
    n = len(orc.streams)
    assert len(gpu.streams) == n
    st = {"label": label, "streams": n, "exact": 0, "exempt": [], "max_abs_dscore": 0.0}
    for s, (x, y) in enumerate(zip(gpu.streams, orc.streams)):
        assert len(x.nbest) == len(y.nbest), (label, s, describe(gpu, orc))
        d = max((abs(ex.score - ey.score) for ex, ey in zip(x.nbest, y.nbest)), default=0.0)
        mism = next((i for i, (ex, ey) in enumerate(zip(x.nbest, y.nbest)) if ex.tokens != ey.tokens), None)
        why = None
        if d > tol:
            why = f"|dscore| {d:.3g} > {tol:.3g}"
        elif mism is not None:
            why = f"tokens differ at n-best entry {mism}"
        else:
            for ex, ey in zip(x.nbest, y.nbest):
                assert ex.frames == ey.frames, (label, s)
                assert ex.durations == ey.durations, (label, s)
            if counter_rtol == 0.0:
                assert x.counters == y.counters, (label, s, x.counters, y.counters)
            else:
                for k, v in y.counters.items():
                    assert abs(x.counters[k] - v) <= counter_rtol * max(v, 1), (label, s, k, x.counters, y.counters)
                st["counters_differ"] = st.get("counters_differ", 0) + int(x.counters != y.counters)
            st["max_abs_dscore"] = max(st["max_abs_dscore"], d)
            st["exact"] += 1
            continue
        if verify is not None:
            div = verify(s)
            assert div is not None, f"{label} stream {s}: {why}, yet the per-round traces never diverge"
            rnd, margin, frame = div
            bound = 2 * (tol_at(frame) if tol_at is not None else tol)
            assert margin <= bound, (f"{label} stream {s}: {why}; the searches diverge at round {rnd} (frame "
                                     f"{frame}) where the oracle's prune margin {margin:.3g} exceeds {bound:.3g}")
            st["exempt"].append({"stream": s, "why": why, "round": rnd, "frame": frame, "oracle_margin": margin,
                                 "bound": bound})
            continue
        assert d <= tol, f"{label} stream {s}: {why}\n" + describe(gpu, orc)
        sc = [e.score for e in y.nbest]
        if mism < len(sc) - 1:
            margin = sc[mism] - sc[mism + 1]
            assert margin <= tol, (f"{label} stream {s}: tokens differ at n-best entry {mism} where the "
                                   f"oracle's margin {margin:.3g} exceeds tol {tol:.3g}\n" + describe(gpu, orc))
        st["max_abs_dscore"] = max(st["max_abs_dscore"], d)
        st["exempt"].append({"stream": s, "why": why, "entry": mism})
    verified = verify is not None
    cap = max_exempt if max_exempt is not None else max(1, n // 4 if verified else n // 8)
    assert len(st["exempt"]) <= cap, f"{label}: {len(st['exempt'])} near-tie exemptions > cap {cap}: {st['exempt']}"
    return st


# ---- near-tie verification through per-round traces --------------------------

TRACE_HEAD = 5  # t, r, done, the oracle's K-th kept score, its best rejected score


def _trace(lib_fn, run):
    import ctypes as C
    lib_fn.restype = C.c_int64
    lib_fn.argtypes = [C.c_int32, C.c_void_p, C.c_int64]
    lib_fn(0, None, 0)
    try:
        result = run()
    finally:
        n = lib_fn(-1, None, 0)
    buf = np.zeros(max(n, 1))
    lib_fn(-1, buf.ctypes.data, n)
    return result, buf[:n]


def first_divergence(dec, oracle, model, cfg, algo, enc_row, length, olm=None):
    """Decode one stream on the GPU (host-loop graph mode, per-round slot
    trace) and in the oracle (the same trace plus the prune margin of every
    round); return (round, oracle_margin, frame) at the first round whose kept slot
    SETS differ (keys: hash, length, last token, frame), or None.

    Why this bounds a legitimate divergence: if the GPU keeps a candidate X the
    oracle rejected and drops a Y the oracle kept, with every candidate's GPU
    score within eps of the oracle's, then s_Y - s_X <= 2 eps, so the oracle's
    own margin between its K-th kept and its best rejected candidate at that
    round is <= 2 eps.  A larger margin there is a real search difference."""
    K = 1 if algo == _abi.ALGO_GREEDY else cfg.beam
    enc_row = np.ascontiguousarray(enc_row[None], np.float32)
    _, o = _trace(oracle.lib.oracle_round_trace,
                  lambda: oracle.decode(model, cfg, algo, enc_row, [length], lm=olm))
    dec.set_graph_mode(0)
    try:
        _, g = _trace(dec.lib.tbeam_debug_round_trace, lambda: dec.decode(algo, enc_row, [length], cfg))
    finally:
        dec.set_graph_mode(1)
    rec = TRACE_HEAD + 6 * K
    o, g = o.reshape(-1, rec), g.reshape(-1, rec)

    def keys(r):
        s = r[TRACE_HEAD:].reshape(K, 6)
        return {(int(x[4]), int(x[5]), int(x[2]), int(x[3]), int(x[1])) for x in s if np.isfinite(x[0])}

    for i in range(min(len(o), len(g))):
        if keys(o[i]) != keys(g[i]):
            return i, float(o[i][3] - o[i][4]), int(o[i][0])
    return None
