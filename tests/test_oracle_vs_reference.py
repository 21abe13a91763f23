"""Pin the CPU restatement (oracle/liboracle.so) against the UNMODIFIED
reference compiled in place (oracle/_ref), on the reference's own decoders:
alsd_pp / reference_beam(kAlsd) / reference_beam(kAes) / aes_pp /
greedy_batched (decoder.hpp:75-97).  Scalar kernels, one thread
(TBEAM_KERNELS=scalar, TBEAM_THREADS=1): the restatement must agree bit for
bit, counters included.

Replays the reference's differential campaigns:
  test_decoders.cpp:156-195  fast vs reference, {omit,scored} x {early,late} x eos
  test_decoders.cpp:77-96    beam-1 ALSD++ == AES++ == greedy
  test_decoders.cpp:383-412  degenerate hash modulus {7,1}
  test_decoders.cpp:197-216  batch invariance
"""
import os
import numpy as np
import pytest

from oracle.cpu import (REF_AES_PP, REF_ALSD_PP, REF_BEAM_AES, REF_BEAM_ALSD, REF_GREEDY)
from paper_2506_00185_b200 import _abi
from paper_2506_00185_b200.model import synthetic_vocabulary
from tests.helpers import describe, instance


def _eq(a, b):
    assert len(a.streams) == len(b.streams)
    for x, y in zip(a.streams, b.streams):
        assert [e.tokens for e in x.nbest] == [e.tokens for e in y.nbest], describe(a, b)
        for ex, ey in zip(x.nbest, y.nbest):
            assert ex.score == pytest.approx(ey.score, abs=1e-12, rel=0), describe(a, b)
        assert x.counters == y.counters


@pytest.mark.parametrize("kind", [_abi.PRED_STATELESS, _abi.PRED_LSTM])
@pytest.mark.parametrize("seed", range(8))
def test_alsd_greedy_aes_match_reference(oracle, ref, kind, seed):
    model, enc, lens = instance(seed, kind=kind, V=4 + seed % 9, B=3, T=6 + seed % 7)
    cfg = _abi.DecodeConfig(beam=1 + seed % 6, max_len=16 + seed, return_nbest=1 + seed % 3,
                            max_symbols_per_frame=2 + seed % 6,
                            aes_expansions_per_frame=seed % 4)
    _eq(oracle.decode(model, cfg, _abi.ALGO_ALSD, enc, lens), ref.decode(REF_ALSD_PP, model, cfg, enc, lens))
    _eq(oracle.decode(model, cfg, _abi.ALGO_ALSD, enc, lens), ref.decode(REF_BEAM_ALSD, model, cfg, enc, lens))
    _eq(oracle.decode(model, cfg, _abi.ALGO_GREEDY, enc, lens), ref.decode(REF_GREEDY, model, cfg, enc, lens))
    # canonical AES++ == reference_beam(kAes) (SURVEY §5 recommendation)
    _eq(oracle.decode(model, cfg, _abi.ALGO_AES, enc, lens), ref.decode(REF_BEAM_AES, model, cfg, enc, lens))
    # the shipped aes_pp, bit for bit, with its stale per-slot donated[] flag
    cfg.aes_slot_donated_quirk = True
    _eq(oracle.decode(model, cfg, _abi.ALGO_AES, enc, lens), ref.decode(REF_AES_PP, model, cfg, enc, lens))


@pytest.mark.parametrize("blank_mode", [_abi.BLANK_OMIT, _abi.BLANK_SCORED])
@pytest.mark.parametrize("pruning", [_abi.PRUNE_EARLY, _abi.PRUNE_LATE])
@pytest.mark.parametrize("eos", [False, True])
def test_lm_fusion_matches_reference(oracle, ref, blank_mode, pruning, eos):
    V = 10
    arpa = ref.random_arpa(31 + blank_mode * 4 + pruning * 2 + eos, V, 3)
    olm = oracle.lm(arpa, synthetic_vocabulary(V))
    rlm = ref.lm(arpa, V)
    for seed in range(4):
        model, enc, lens = instance(100 + seed, V=V, B=2, T=8)
        cfg = _abi.DecodeConfig(beam=3, max_len=20, return_nbest=2,
                                fusion=_abi.FusionConfig(lam=0.3 + 0.4 * seed, blank_mode=blank_mode,
                                                         pruning=pruning, eos_enabled=eos))
        for algo, which in ((_abi.ALGO_ALSD, REF_ALSD_PP), (_abi.ALGO_GREEDY, REF_GREEDY),
                            (_abi.ALGO_AES, REF_BEAM_AES)):
            _eq(oracle.decode(model, cfg, algo, enc, lens, lm=olm),
                ref.decode(which, model, cfg, enc, lens, lm=rlm))


def test_beam1_equals_greedy(oracle):
    """test_decoders.cpp:77-96: beam-1 ALSD++ == AES++ == greedy."""
    for seed in range(20):
        model, enc, lens = instance(200 + seed, V=2 + seed % 6, B=2, T=2 + seed % 7)
        cfg = _abi.DecodeConfig(beam=1, max_len=24)
        cfg.aes_expansions_per_frame = cfg.max_symbols_per_frame - 1
        g = oracle.decode(model, cfg, _abi.ALGO_GREEDY, enc, lens)
        a = oracle.decode(model, cfg, _abi.ALGO_ALSD, enc, lens)
        e = oracle.decode(model, cfg, _abi.ALGO_AES, enc, lens)
        for s in range(2):
            assert a.streams[s].nbest[0].tokens == g.streams[s].nbest[0].tokens
            assert e.streams[s].nbest[0].tokens == g.streams[s].nbest[0].tokens


def test_degenerate_hash_modulus(oracle, ref):
    """test_decoders.cpp:383-412: HashParams{7,1} -- every transcript hashes to
    0, so HypKey merges on (length, last) alone; the hash-keyed engines agree
    with each other and (somewhere) disagree with token-compare reference_beam."""
    diverged = 0
    for seed in range(12):
        model, enc, lens = instance(300 + seed, V=3, B=2, T=8, blank_bias=0.5)
        cfg = _abi.DecodeConfig(beam=6, max_len=20, return_nbest=3,
                                hash_params=_abi.HashParams(base=7, modulus=1))
        o = oracle.decode(model, cfg, _abi.ALGO_ALSD, enc, lens)
        _eq(o, ref.decode(REF_ALSD_PP, model, cfg, enc, lens))
        r = ref.decode(REF_BEAM_ALSD, model, cfg, enc, lens)
        if any([e.tokens for e in x.nbest] != [e.tokens for e in y.nbest]
               for x, y in zip(o.streams, r.streams)):
            diverged += 1
    assert diverged > 0


def test_batch_invariance(oracle):
    """test_decoders.cpp:197-216: batch-5 == each stream alone, exact."""
    model, enc, lens = instance(400, V=8, B=5, T=10)
    cfg = _abi.DecodeConfig(beam=4, max_len=20, return_nbest=2)
    for algo in (_abi.ALGO_ALSD, _abi.ALGO_AES):
        full = oracle.decode(model, cfg, algo, enc, lens)
        for b in range(5):
            one = oracle.decode(model, cfg, algo, enc[b:b + 1], lens[b:b + 1])
            assert [e.tokens for e in one.streams[0].nbest] == [e.tokens for e in full.streams[b].nbest]
            assert [e.score for e in one.streams[0].nbest] == [e.score for e in full.streams[b].nbest]


def test_invalid_arguments(oracle, ref):
    """validate_streams (decoder.cpp:16-38): the same configs are rejected."""
    model, enc, lens = instance(500, V=5, B=2, T=4)
    bad = [dict(beam=0), dict(max_symbols_per_frame=0), dict(max_len=0), dict(return_nbest=0),
           dict(aes_expansions_per_frame=-1)]
    for kw in bad:
        cfg = _abi.DecodeConfig(**kw)
        with pytest.raises(ValueError):
            oracle.decode(model, cfg, _abi.ALGO_ALSD, enc, lens)
        with pytest.raises(ValueError):
            ref.decode(REF_ALSD_PP, model, cfg, enc, lens)
    cfg = _abi.DecodeConfig(fusion=_abi.FusionConfig(lam=0.5))
    with pytest.raises(ValueError):  # LM weight set but no LM given
        oracle.decode(model, cfg, _abi.ALGO_ALSD, enc, lens)
    with pytest.raises(ValueError):
        ref.decode(REF_ALSD_PP, model, cfg, enc, lens)
    with pytest.raises(ValueError):  # frames out of range
        oracle.decode(model, _abi.DecodeConfig(), _abi.ALGO_ALSD, enc, [5, 1])


def test_peaky_model_oracle_matches_reference():
    """The structured bench model through the unmodified reference decoder
    (oracle/_ref) and the restatement: bit-identical search results."""
    import pytest as _pt
    from oracle.cpu import REF_SO, RefLib, Oracle, REF_ALSD_PP
    if not os.path.exists(REF_SO):
        _pt.skip("oracle/_ref not built")
    from paper_2506_00185_b200 import _abi
    from paper_2506_00185_b200.model import SyntheticTransducer, TransducerSpec
    spec = TransducerSpec(vocab_size=96, enc_dim=64, joint_dim=64, pred_kind=_abi.PRED_LSTM, lstm_hidden=64,
                          emb_dim=64, logit_scale=4.0, seed=3, peaky=True)
    model = SyntheticTransducer(spec)
    enc = model.encoder_frames(5, 3, 40)
    lens = [40, 33, 17]
    cfg = _abi.DecodeConfig(beam=4, max_len=48, return_nbest=2)
    got = Oracle().decode(model, cfg, _abi.ALGO_ALSD, enc, lens)
    ref = RefLib().decode(REF_ALSD_PP, model, cfg, enc, lens)
    for a, b in zip(got.streams, ref.streams):
        assert [e.tokens for e in a.nbest] == [e.tokens for e in b.nbest]
        for x, y in zip(a.nbest, b.nbest):
            assert abs(x.score - y.score) <= 1e-9
    assert sum(len(s.nbest[0].tokens) for s in got.streams) > 5
