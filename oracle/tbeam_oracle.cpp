// TEST INFRASTRUCTURE -- oracle only.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline leg may load liboracle.so, and only as the
// checker.  The product path (paper_2506_00185_b200/) never links it.
//
// CPU restatement of the reference's batched beam search, generalised to the
// B200 build's scope:
//   * BeamEngine::run_lane          decoder.cpp:106-356   (ALSD++ / AES++)
//   * greedy_lane                   decoder.cpp:360-425   (= the K=1 ALSD++ instance;
//                                                          beam-1 == greedy, test_decoders.cpp:77-96)
//   * selection_row / early term    decoder.cpp:40-71, fusion.cpp:11-43
//   * update_hash / logadd          hyp_store.cpp:13-44
//   * prune_topk total order        hyp_store.cpp:199-228 (score desc, index asc)
//   * AES++ prefix pass             decoder.cpp:186-229 (canonical per-hypothesis
//                                   donated flag, reference_decoder.cpp:232-234;
//                                   optional slot quirk of the shipped aes_pp)
//   * blank-column recombination    decoder.cpp:256-277
//   * EOS + ranking + n-best        decoder.cpp:329-355
// It keeps one object per hypothesis with its materialised transcript (like
// reference_decoder.cpp), but merges by HypKey (hash, length, last) exactly as
// the batched engine does, so the degenerate-modulus behaviour carries over.
//
// Extensions beyond the reference (its SPEC marks them out of scope; the
// semantics are frozen here first and the GPU follows this file):
//   * LSTM prediction network (state carried per hypothesis);
//   * alignments: the frame of every emitted token;
//   * TDT: candidates are (token, duration) pairs with log p = lp_tok + lp_dur;
//     every hypothesis carries the frame f it next emits at; a stream's
//     current frame is t = min f over live hypotheses; "active" = f == t,
//     "complete" (carried) = f > t.  Blank needs duration >= 1.  The last
//     round of a frame admits only candidates that leave the frame
//     (duration >= 1).  Recombination runs over the frame-leaving blank
//     candidates and the carries, keyed by (HypKey, destination frame);
//     destinations clamp to T_b (two blanks of one hypothesis that both land
//     on T_b merge as well).  RNN-T is the special case durations = {}:
//     token -> f = t, blank -> f = t + 1.
//   * merge_mode MAX (keep the larger score instead of log-sum-exp).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle_lm.hpp"
#include "synthetic_model.hpp"
#include "tbeam_b200.h"

namespace oracle {
namespace {

constexpr double kNegInf = -std::numeric_limits<double>::infinity();
constexpr std::uint64_t kMersenne61 = (std::uint64_t{1} << 61) - 1;

thread_local std::string g_err;

// hyp_store.cpp:13-37
std::uint64_t update_hash(std::uint64_t h, std::int32_t tok, std::uint64_t base,
                          std::uint64_t mod) {
    if (tok < 0) throw std::invalid_argument("update_hash: blank or invalid token");
    const unsigned __int128 x =
        static_cast<unsigned __int128>(h) * base + static_cast<std::uint64_t>(tok) + 1;
    if (mod == kMersenne61) {
        std::uint64_t r = static_cast<std::uint64_t>(x & kMersenne61) +
                          static_cast<std::uint64_t>(x >> 61);
        r = (r & kMersenne61) + (r >> 61);
        if (r >= kMersenne61) r -= kMersenne61;
        return r;
    }
    return static_cast<std::uint64_t>(x % mod);
}

// hyp_store.cpp:39-44
double logadd(double a, double b) {
    if (a == kNegInf) return b;
    if (b == kNegInf) return a;
    const double m = std::max(a, b);
    return m + std::log1p(std::exp(std::min(a, b) - m));
}

// fusion.cpp:11-22
double log1mexp(double x) {
    if (x > 0.0) throw std::invalid_argument("log1mexp: argument must be <= 0");
    if (x == 0.0) return kNegInf;
    if (x > -M_LN2) return std::log(-std::expm1(x));
    return std::log1p(-std::exp(x));
}

struct Hyp {
    bool alive = false;
    double score = kNegInf;
    int f = 0;  // frame of the next emission
    bool donated = false;
    std::vector<std::int32_t> tokens, tok_frames, tok_durs;
    std::uint64_t hash = 0;
    std::int32_t last = -1;
    OracleLm::Ctx lm_state;
    std::vector<std::int32_t> window;      // stateless
    std::shared_ptr<const LstmState> lstm;  // LSTM
};

struct Cand {
    double score;
    std::int64_t idx;
    int slot, k, di, dest;
    bool leaves;  // blank-class (blank or carry): participates in recombination
};

// prune_topk's total order (hyp_store.cpp:199-228): score desc, index asc
bool better(const Cand& x, const Cand& y) {
    if (x.score != y.score) return x.score > y.score;
    return x.idx < y.idx;
}
bool better_inv(const Cand& x, const Cand& y) { return better(y, x); }

struct StreamOut {
    std::vector<Hyp> nbest;
    std::uint64_t ctr[TBEAM_NUM_COUNTERS] = {0, 0, 0, 0, 0};
    std::vector<double>* trace = nullptr;  // debug: per-round slot state
};

int g_trace_stream = -1;
std::vector<double> g_trace_buf;

class Engine {
public:
    Engine(const SyntheticModel& m, const OracleLm* lm, const tbeam_decode_config& c)
        : M(m), LM(lm), cfg(c) {
        V = M.V;
        ND = M.ND;
        ndx = ND > 0 ? ND : 1;
        with_lm = LM != nullptr && cfg.lm_weight > 0.0;
        late = with_lm && cfg.prune_mode == TBEAM_PRUNE_LATE;
        early = with_lm && cfg.prune_mode == TBEAM_PRUNE_EARLY;
        aes = cfg.algo == TBEAM_ALGO_AES;
        beam = cfg.algo == TBEAM_ALGO_GREEDY ? 1 : cfg.beam;
        rounds = aes ? cfg.aes_expansions_per_frame + 1 : cfg.max_symbols_per_frame;
        di0 = -1;
        for (int d = 0; d < ND; ++d)
            if (M.dims.durations[d] == 0) di0 = d;
    }

    double merge(double a, double b) const {
        return cfg.merge_mode == TBEAM_MERGE_MAX ? std::max(a, b) : logadd(a, b);
    }

    // decoder.cpp:47-61 (selection_row) on one normalised ASR row
    void selection_row(const double* asr, const double* lm_row, double* out) const {
        for (int k = 0; k <= V; ++k) out[k] = asr[k];
        if (!with_lm) return;
        const double lam = cfg.lm_weight;
        if (late) {
            if (cfg.blank_mode == TBEAM_BLANK_OMIT) {
                for (int k = 0; k < V; ++k) out[k] = asr[k] + lam * lm_row[k];
                out[V] = asr[V];
            } else {
                const double l1m = log1mexp(asr[V]);
                for (int k = 0; k < V; ++k) out[k] = asr[k] + lam * (lm_row[k] + l1m);
                out[V] = (1.0 + lam) * asr[V];
            }
            return;
        }
        if (cfg.blank_mode == TBEAM_BLANK_SCORED) out[V] = (1.0 + lam) * asr[V];
    }

    // decoder.cpp:64-71
    double early_term(const Hyp& h, int tok, double asr_blank) const {
        double term = LM->score_token(h.lm_state, tok);
        if (cfg.blank_mode == TBEAM_BLANK_SCORED) term += log1mexp(asr_blank);
        return cfg.lm_weight * term;
    }

    void pred_of(const Hyp& h, double* out) const {
        if (M.lstm) {
            std::copy(h.lstm->pred.begin(), h.lstm->pred.end(), out);
        } else {
            M.stateless_pred(h.window.data(), out);
        }
    }

    void run(const float* enc /*[T, D]*/, int T, StreamOut& out) {
        const char* dbg = std::getenv("ORACLE_DEBUG_T");
        const int debug_t = dbg ? std::atoi(dbg) : -1;
        const int J = M.J;
        const int row = V + 1;
        std::vector<double> encp(static_cast<std::size_t>(T) * J);
        for (int t = 0; t < T; ++t) M.enc_proj(enc + static_cast<std::size_t>(t) * M.D, &encp[t * J]);

        std::vector<Hyp> hyps(beam);
        hyps[0].alive = true;
        hyps[0].score = 0.0;
        hyps[0].f = 0;
        if (with_lm) hyps[0].lm_state = LM->initial_state();
        if (M.lstm) hyps[0].lstm = std::make_shared<LstmState>(M.lstm_start());
        else hyps[0].window.assign(M.n, -1);
        for (int i = 1; i < beam; ++i) {
            hyps[i].alive = false;
            hyps[i].window.assign(M.n, -1);
        }

        std::vector<double> emis(static_cast<std::size_t>(beam) * row), fused(emis.size());
        std::vector<double> dur(static_cast<std::size_t>(beam) * ndx, 0.0);
        std::vector<double> lm_row(V);
        std::vector<double> preds(static_cast<std::size_t>(beam) * J), emis_act(emis.size()),
            dur_act(dur.size());
        std::vector<const double*> pred_ptr(beam);
        std::vector<int> act, lstm_dst, lstm_tok;
        std::vector<const LstmState*> lstm_src;
        std::vector<std::uint8_t> slot_donated(beam, 0);  // aes_pp quirk only
        const int token_rounds = rounds - 1;

        int t = 0;
        while (t < T) {
            std::fill(slot_donated.begin(), slot_donated.end(), 0);
            for (auto& h : hyps) h.donated = false;
            for (int r = 0; r < rounds; ++r) {
                bool any_active = false;
                for (const auto& h : hyps)
                    if (h.alive && h.f == t) any_active = true;
                if (!any_active) break;
                const bool last_round = r == token_rounds;

                // every active slot's row in one pass over the joint weights
                // (SyntheticModel::joint_many: bit-identical to per-row joint())
                act.clear();
                for (int i = 0; i < beam; ++i)
                    if (hyps[i].alive && hyps[i].f == t) act.push_back(i);
                for (std::size_t q = 0; q < act.size(); ++q) {
                    pred_of(hyps[act[q]], &preds[q * J]);
                    pred_ptr[q] = &preds[q * J];
                }
                M.joint_many(&encp[static_cast<std::size_t>(t) * J], pred_ptr.data(),
                             static_cast<int>(act.size()), emis_act.data(), row,
                             ND > 0 ? dur_act.data() : nullptr, ndx);
                for (std::size_t q = 0; q < act.size(); ++q) {
                    const std::size_t i = static_cast<std::size_t>(act[q]);
                    std::copy(&emis_act[q * row], &emis_act[q * row] + row, &emis[i * row]);
                    std::copy(&dur_act[q * ndx], &dur_act[q * ndx] + ndx, &dur[i * ndx]);
                }
                for (int i = 0; i < beam; ++i) {
                    const Hyp& h = hyps[i];
                    if (!h.alive || h.f != t) continue;
                    double* asr = &emis[static_cast<std::size_t>(i) * row];
                    ++out.ctr[2];
                    if (late) {
                        LM->score_vocab(h.lm_state, lm_row.data());
                        ++out.ctr[4];
                    }
                    selection_row(asr, lm_row.data(), &fused[static_cast<std::size_t>(i) * row]);
                }
                ++out.ctr[1];

                // AES++ maximum-length prefix combination (decoder.cpp:186-229)
                if (aes && cfg.aes_prefix_search && r == 0 && (ND == 0 || di0 >= 0)) {
                    struct Edge { int donor, receiver; };
                    std::vector<Edge> edges;
                    for (int a = 0; a < beam; ++a) {
                        if (!hyps[a].alive || hyps[a].f != t) continue;
                        for (int c = 0; c < beam; ++c) {
                            if (c == a || !hyps[c].alive || hyps[c].f != t) continue;
                            const int la = static_cast<int>(hyps[a].tokens.size());
                            const int lc = static_cast<int>(hyps[c].tokens.size());
                            if (lc != la + 1) continue;
                            const std::int32_t last = hyps[c].last;
                            const std::uint64_t ext =
                                update_hash(hyps[a].hash, last, cfg.hash_base, cfg.hash_modulus);
                            if (ext == hyps[c].hash && la + 1 == lc && last == hyps[c].last)
                                edges.push_back({a, c});
                        }
                    }
                    std::sort(edges.begin(), edges.end(), [&](const Edge& x, const Edge& y) {
                        const auto kx = std::make_tuple(hyps[x.receiver].tokens.size(), x.receiver, x.donor);
                        const auto ky = std::make_tuple(hyps[y.receiver].tokens.size(), y.receiver, y.donor);
                        return kx < ky;
                    });
                    for (const Edge& e : edges) {
                        const std::int32_t last = hyps[e.receiver].last;
                        double donation = hyps[e.donor].score +
                                          fused[static_cast<std::size_t>(e.donor) * row + last];
                        if (ND > 0) donation += dur[static_cast<std::size_t>(e.donor) * ndx + di0];
                        if (early) {
                            donation += early_term(hyps[e.donor], last,
                                                   emis[static_cast<std::size_t>(e.donor) * row + V]);
                            ++out.ctr[3];
                        }
                        if (debug_t == t)
                            std::fprintf(stderr, "ORC prefix t=%d edge %d->%d last=%d sc_a=%.9f sc_c=%.9f don=%.9f\n", t,
                                         e.donor, e.receiver, last, hyps[e.donor].score, hyps[e.receiver].score,
                                         donation - hyps[e.donor].score);
                        hyps[e.receiver].score = merge(hyps[e.receiver].score, donation);
                        hyps[e.donor].donated = true;
                        slot_donated[e.donor] = 1;
                    }
                }

                // candidates (decoder.cpp:231-254), slot-major; blank/carry last.
                // Token candidates never recombine, so only those that can still
                // reach the top `beam` are kept (a candidate not better than the
                // current beam-th best of a pruned set never can; the order is
                // total), which keeps V = 8192 rounds cheap.
                std::vector<Cand> cands, tokc;
                bool have_thr = false;
                Cand thr{};
                const auto push_tok = [&](const Cand& c) {
                    if (c.score == kNegInf || (have_thr && !better(c, thr))) return;
                    tokc.push_back(c);
                    if (tokc.size() >= static_cast<std::size_t>(8 * beam + 256)) {
                        std::nth_element(tokc.begin(), tokc.begin() + (beam - 1), tokc.end(), better);
                        tokc.resize(beam);
                        thr = *std::min_element(tokc.begin(), tokc.end(), better_inv);
                        have_thr = true;
                    }
                };
                for (int i = 0; i < beam; ++i) {
                    const Hyp& h = hyps[i];
                    if (!h.alive) continue;
                    const double base = h.score;
                    const std::int64_t slot_base = static_cast<std::int64_t>(i) * row * ndx;
                    if (h.f != t) {  // complete: carry
                        cands.push_back({base, slot_base + static_cast<std::int64_t>(V) * ndx,
                                         i, V, 0, h.f, true});
                        continue;
                    }
                    const bool donated = cfg.aes_slot_donated_quirk ? slot_donated[i] != 0
                                                                    : h.donated;
                    const bool allow_tokens = !donated &&
                                              static_cast<int>(h.tokens.size()) < cfg.max_len;
                    const double* fr = &fused[static_cast<std::size_t>(i) * row];
                    if (ND == 0) {
                        if (allow_tokens && !last_round)
                            for (int k = 0; k < V; ++k)
                                push_tok({fr[k] + base, slot_base + k, i, k, 0, t, false});
                        cands.push_back({base + fr[V], slot_base + V, i, V, 0, std::min(t + 1, T), true});
                    } else {
                        const double* dr = &dur[static_cast<std::size_t>(i) * ndx];
                        for (int k = 0; k <= V; ++k) {
                            if (k < V && !allow_tokens) continue;
                            for (int d = 0; d < ND; ++d) {
                                const int dv = M.dims.durations[d];
                                if (k == V && dv == 0) continue;   // blank must advance
                                if (last_round && dv == 0) continue;  // last round leaves the frame
                                const double s = base + (fr[k] + dr[d]);
                                const Cand c{s, slot_base + static_cast<std::int64_t>(k) * ndx + d, i, k, d,
                                             std::min(t + dv, T), k == V};
                                if (k == V) cands.push_back(c);
                                else push_tok(c);
                            }
                        }
                    }
                }

                // recombination over the frame-leaving blank column (decoder.cpp:256-277)
                // (only the blank-class entries take part; visiting them in
                // candidate order keeps the i < j pairing of the reference)
                std::vector<std::size_t> leave;
                for (std::size_t a = 0; a < cands.size(); ++a)
                    if (cands[a].leaves) leave.push_back(a);
                for (std::size_t ia = 0; ia < leave.size(); ++ia) {
                    Cand& ca = cands[leave[ia]];
                    if (ca.score == kNegInf) continue;
                    for (std::size_t ib = ia + 1; ib < leave.size(); ++ib) {
                        Cand& cb = cands[leave[ib]];
                        if (cb.score == kNegInf) continue;
                        const Hyp& ha = hyps[ca.slot];
                        const Hyp& hb = hyps[cb.slot];
                        if (ha.hash == hb.hash && ha.tokens.size() == hb.tokens.size() &&
                            ha.last == hb.last && ca.dest == cb.dest) {
                            ca.score = merge(ca.score, cb.score);
                            cb.score = kNegInf;
                        }
                    }
                }

                if (debug_t == t) {
                    for (const Cand& c : cands)
                        std::fprintf(stderr, "ORC blank t=%d r=%d slot %d d %d dest %d after %.9f\n", t, r, c.slot, c.di,
                                     c.dest, c.score);
                    for (const Cand& c : tokc)
                        std::fprintf(stderr, "ORC token t=%d r=%d slot %d k %d v %.9f\n", t, r, c.slot, c.k, c.score);
                }
                // prune_topk: (score desc, index asc), -inf never beats finite
                std::vector<Cand> fin;
                for (const Cand& c : cands)
                    if (c.score != kNegInf) fin.push_back(c);
                fin.insert(fin.end(), tokc.begin(), tokc.end());
                // the order is total (indices are unique), so the first `beam`
                // entries of a partial sort are exactly those of a full sort
                const std::size_t keep = std::min<std::size_t>(static_cast<std::size_t>(beam), fin.size());
                std::partial_sort(fin.begin(), fin.begin() + keep, fin.end(), better);

                std::vector<Hyp> next(beam);
                lstm_dst.clear();
                lstm_src.clear();
                lstm_tok.clear();
                for (int j = 0; j < beam; ++j) {
                    if (j >= static_cast<int>(fin.size())) {
                        next[j].alive = false;
                        next[j].score = kNegInf;
                        continue;
                    }
                    const Cand& c = fin[j];
                    const Hyp& p = hyps[c.slot];
                    Hyp h = p;
                    h.donated = false;
                    double s = c.score;
                    if (c.k == V) {  // blank (or carry)
                        h.f = c.dest;
                    } else {
                        if (early) {
                            s += early_term(p, c.k, emis[static_cast<std::size_t>(c.slot) * row + V]);
                            ++out.ctr[3];
                        }
                        h.tokens.push_back(c.k);
                        h.tok_frames.push_back(t);
                        h.tok_durs.push_back(ND > 0 ? M.dims.durations[c.di] : 0);
                        h.hash = update_hash(p.hash, c.k, cfg.hash_base, cfg.hash_modulus);
                        h.last = c.k;
                        h.f = c.dest;
                        if (M.lstm) {
                            lstm_dst.push_back(j);  // stepped below, all children at once
                            lstm_src.push_back(p.lstm.get());
                            lstm_tok.push_back(c.k);
                        } else if (M.n > 0) {
                            for (int q = 0; q + 1 < M.n; ++q) h.window[q] = h.window[q + 1];
                            h.window[M.n - 1] = c.k;
                        }
                        if (with_lm) h.lm_state = LM->advance(p.lm_state, c.k);
                    }
                    h.score = p.score + (s - p.score);  // decoder.cpp:319 + hyp_store.cpp:124
                    next[j] = std::move(h);
                }
                if (!lstm_dst.empty()) {
                    std::vector<LstmState> st = M.lstm_step_many(
                        lstm_src.data(), lstm_tok.data(), static_cast<int>(lstm_dst.size()));
                    for (std::size_t q = 0; q < lstm_dst.size(); ++q)
                        next[lstm_dst[q]].lstm = std::make_shared<LstmState>(std::move(st[q]));
                }
                hyps.swap(next);
                if (out.trace) {
                    // the prune's margin: the K-th kept score and the best rejected one
                    double kth = kNegInf, next_best = kNegInf;
                    if (static_cast<int>(fin.size()) >= beam) kth = fin[beam - 1].score;
                    for (std::size_t q = static_cast<std::size_t>(beam); q < fin.size(); ++q)
                        next_best = std::max(next_best, fin[q].score);
                    out.trace->push_back(t);
                    out.trace->push_back(r);
                    out.trace->push_back(0);
                    out.trace->push_back(kth);
                    out.trace->push_back(next_best);
                    for (const Hyp& h : hyps) {
                        out.trace->push_back(h.alive ? h.score : kNegInf);
                        out.trace->push_back(h.f);
                        out.trace->push_back(static_cast<double>(h.tokens.size()));
                        out.trace->push_back(h.last);
                        out.trace->push_back(static_cast<double>(h.hash >> 32));
                        out.trace->push_back(static_cast<double>(h.hash & 0xffffffffull));
                    }
                }
            }
            ++out.ctr[0];
            int nt = T;
            for (const auto& h : hyps)
                if (h.alive) nt = std::min(nt, h.f);
            if (nt <= t) nt = t + 1;  // defensive; unreachable by construction
            t = nt;
        }

        // final recombination (merge_duplicates_stream, hyp_store.cpp:169-191):
        // a no-op for RNN-T, whose blank column already merged every finisher;
        // TDT tokens that jump to T_b arrive unmerged
        for (int i = 0; i < beam; ++i) {
            if (!hyps[i].alive) continue;
            for (int j = i + 1; j < beam; ++j) {
                if (!hyps[j].alive) continue;
                if (hyps[i].hash == hyps[j].hash && hyps[i].tokens.size() == hyps[j].tokens.size() &&
                    hyps[i].last == hyps[j].last) {
                    hyps[i].score = merge(hyps[i].score, hyps[j].score);
                    hyps[j].alive = false;
                    hyps[j].score = kNegInf;
                }
            }
        }
        if (with_lm && cfg.eos_enabled) {
            for (auto& h : hyps)
                if (h.alive) {
                    h.score += cfg.lm_weight * LM->score_eos(h.lm_state);
                    ++out.ctr[3];
                }
        }
        std::vector<std::pair<double, int>> ranked;
        for (int i = 0; i < beam; ++i)
            if (hyps[i].alive) ranked.emplace_back(hyps[i].score, i);
        std::sort(ranked.begin(), ranked.end(), [](const auto& a, const auto& b) {
            if (a.first != b.first) return a.first > b.first;
            return a.second < b.second;
        });
        const int nb = cfg.algo == TBEAM_ALGO_GREEDY ? 1 : cfg.return_nbest;
        const int take = std::min<int>(nb, static_cast<int>(ranked.size()));
        for (int r = 0; r < take; ++r) {
            Hyp h = hyps[ranked[r].second];
            h.score = ranked[r].first;
            out.nbest.push_back(std::move(h));
        }
    }

    const SyntheticModel& M;
    const OracleLm* LM;
    tbeam_decode_config cfg;
    int V, ND, ndx, beam, rounds, di0;
    bool with_lm, late, early, aes;
};

int validate(const tbeam_decode_config& c, int batch, const int32_t* lengths, int max_frames,
             bool has_lm) {
    if (batch < 1) { g_err = "decode: no streams"; return TBEAM_INVALID_ARGUMENT; }
    for (int b = 0; b < batch; ++b)
        if (lengths[b] < 1 || lengths[b] > max_frames) {
            g_err = "decode: bad stream input";
            return TBEAM_INVALID_ARGUMENT;
        }
    if (c.beam < 1 || c.max_symbols_per_frame < 1 || c.aes_expansions_per_frame < 0 ||
        c.max_len < 1 || c.return_nbest < 1 || c.algo < 0 || c.algo > 2) {
        g_err = "decode: bad config";
        return TBEAM_INVALID_ARGUMENT;
    }
    if (c.lm_weight < 0.0) { g_err = "decode: negative LM weight"; return TBEAM_INVALID_ARGUMENT; }
    if (c.lm_weight > 0.0 && !has_lm) {
        g_err = "decode: LM weight set but no LM given";
        return TBEAM_INVALID_ARGUMENT;
    }
    return TBEAM_OK;
}

}  // namespace
}  // namespace oracle

using namespace oracle;

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

// debug aid: the per-round slot state of stream `stream` in later decodes
// (record = t, r, 0, the K-th kept candidate score, the best rejected one, then
// per slot: score, f, len, last, hash >> 32, hash & 0xffffffff); returns the count
// recorded so far; with out != null copies up to cap and clears.
int64_t oracle_round_trace(int32_t stream, double* out, int64_t cap) {
    const int64_t n = static_cast<int64_t>(g_trace_buf.size());
    if (out)
        for (int64_t i = 0; i < n && i < cap; ++i) out[i] = g_trace_buf[static_cast<std::size_t>(i)];
    if (out) g_trace_buf.clear();
    g_trace_stream = stream;
    return n;
}

uint64_t oracle_update_hash(uint64_t h, int32_t tok, uint64_t base, uint64_t mod) {
    return update_hash(h, tok, base, mod);
}
double oracle_logadd(double a, double b) { return logadd(a, b); }
double oracle_log1mexp(double x) { return log1mexp(x); }

void* oracle_lm_create(const char* text, const char* const* tokens, int32_t vocab) {
    try {
        std::vector<std::string> v(tokens, tokens + vocab);
        return new OracleLm(std::string(text), v);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void oracle_lm_destroy(void* lm) { delete static_cast<OracleLm*>(lm); }
int32_t oracle_lm_order(void* lm) { return static_cast<OracleLm*>(lm)->order(); }

// Queries on a context given as a token path from the initial state.
static OracleLm::Ctx walk(const OracleLm* lm, const int32_t* hist, int32_t n) {
    OracleLm::Ctx s = lm->initial_state();
    for (int i = 0; i < n; ++i) s = lm->advance(s, hist[i]);
    return s;
}
double oracle_lm_score_token(void* lm, const int32_t* hist, int32_t n, int32_t tok) {
    auto* p = static_cast<OracleLm*>(lm);
    return p->score_token(walk(p, hist, n), tok);
}
double oracle_lm_score_eos(void* lm, const int32_t* hist, int32_t n) {
    auto* p = static_cast<OracleLm*>(lm);
    return p->score_eos(walk(p, hist, n));
}
void oracle_lm_score_vocab(void* lm, const int32_t* hist, int32_t n, double* out) {
    auto* p = static_cast<OracleLm*>(lm);
    p->score_vocab(walk(p, hist, n), out);
}

// Emission rows of the synthetic model (for kernel-level parity tests).
int32_t oracle_joint_rows(const tbeam_model_dims* dims, const tbeam_model_weights* w,
                          const float* enc_frames /*[R, D]*/, const int32_t* histories,
                          const int32_t* hist_len, int32_t max_hist, int32_t rows,
                          double* tok_out /*[R, V+1]*/, double* dur_out /*[R, ND]*/) {
    try {
        SyntheticModel M(*dims, *w);
        std::vector<double> encp(M.J), pred(M.J);
        for (int r = 0; r < rows; ++r) {
            M.enc_proj(enc_frames + static_cast<std::size_t>(r) * M.D, encp.data());
            const int32_t* h = histories + static_cast<std::size_t>(r) * max_hist;
            if (M.lstm) {
                LstmState s = M.lstm_start();
                for (int i = 0; i < hist_len[r]; ++i) s = M.lstm_step(s, h[i]);
                pred = s.pred;
            } else {
                std::vector<int32_t> win(M.n, -1);
                for (int i = 0; i < hist_len[r]; ++i) {
                    for (int q = 0; q + 1 < M.n; ++q) win[q] = win[q + 1];
                    if (M.n > 0) win[M.n - 1] = h[i];
                }
                M.stateless_pred(win.data(), pred.data());
            }
            M.joint(encp.data(), pred.data(), tok_out + static_cast<std::size_t>(r) * (M.V + 1),
                    dur_out ? dur_out + static_cast<std::size_t>(r) * std::max(M.ND, 1) : nullptr);
        }
        return TBEAM_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TBEAM_INVALID_ARGUMENT;
    }
}

int32_t oracle_decode(const tbeam_model_dims* dims, const tbeam_model_weights* w, void* lm,
                      const tbeam_decode_config* cfg, const float* enc, const int32_t* lengths,
                      int32_t batch, int32_t max_frames, tbeam_results* res) {
    try {
        const int st = validate(*cfg, batch, lengths, max_frames, lm != nullptr);
        if (st != TBEAM_OK) return st;
        SyntheticModel M(*dims, *w);
        Engine eng(M, static_cast<const OracleLm*>(lm), *cfg);
        // Streams are independent (batch invariance, test_decoders.cpp:197-216):
        // decode them on a pool of ORACLE_THREADS workers (default: all cores).
        std::vector<StreamOut> outs(batch);
        if (g_trace_stream >= 0 && g_trace_stream < batch) outs[g_trace_stream].trace = &g_trace_buf;
        std::atomic<int> next{0};
        std::mutex mu;
        std::string first_err;
        const auto work = [&]() {
            for (int b = next++; b < batch; b = next++) {
                try {
                    eng.run(enc + static_cast<std::size_t>(b) * max_frames * M.D, lengths[b], outs[b]);
                } catch (const std::exception& e) {
                    std::lock_guard<std::mutex> g(mu);
                    if (first_err.empty()) first_err = e.what();
                }
            }
        };
        int nt = static_cast<int>(std::thread::hardware_concurrency());
        if (const char* env = std::getenv("ORACLE_THREADS")) nt = std::atoi(env);
        nt = std::max(1, std::min(nt, batch));
        std::vector<std::thread> pool;
        for (int i = 1; i < nt; ++i) pool.emplace_back(work);
        work();
        for (auto& th : pool) th.join();
        if (!first_err.empty()) throw std::invalid_argument(first_err);
        for (int b = 0; b < batch; ++b) {
            const StreamOut& so = outs[b];
            res->nbest_count[b] = static_cast<int32_t>(so.nbest.size());
            for (int r = 0; r < res->nbest; ++r) {
                const std::size_t e = static_cast<std::size_t>(b) * res->nbest + r;
                res->lengths[e] = 0;
                res->scores[e] = kNegInf;
                if (r >= static_cast<int>(so.nbest.size())) continue;
                const Hyp& h = so.nbest[r];
                const int L = std::min<int>(static_cast<int>(h.tokens.size()), res->max_len);
                res->lengths[e] = L;
                res->scores[e] = h.score;
                for (int i = 0; i < L; ++i) {
                    res->tokens[e * res->max_len + i] = h.tokens[i];
                    if (res->frames) res->frames[e * res->max_len + i] = h.tok_frames[i];
                    if (res->durations) res->durations[e * res->max_len + i] = h.tok_durs[i];
                }
            }
            if (res->counters)
                for (int i = 0; i < TBEAM_NUM_COUNTERS; ++i)
                    res->counters[static_cast<std::size_t>(b) * TBEAM_NUM_COUNTERS + i] = so.ctr[i];
        }
        return TBEAM_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TBEAM_INVALID_ARGUMENT;
    }
}

}  // extern "C"
