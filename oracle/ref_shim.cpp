// TEST INFRASTRUCTURE -- oracle only.  Linked against the UNMODIFIED reference
// sources compiled from /root/reference/proj/src (see oracle/Makefile) into
// oracle/_ref/libtbeam_ref.so.  Nothing here is product code.
//
// It supplies the reference's own extension point -- a tbeam::EmissionModel
// subclass (model.hpp:62-74) -- for the synthetic transducer of
// oracle/synthetic_model.hpp, and exposes the reference's decoders, LM, hash
// and top-k through a C ABI so Python tests can
//   * pin the CPU restatement (liboracle.so) against the reference itself,
//   * generate the golden fixtures under tests/golden/, and
//   * time the reference's CPU decoder for bench.py --impl reference.
//
// LSTM models use context_order = max_len: the reference's window then holds
// the whole transcript (advance_state shifts left, model.cpp:109-121), and the
// LSTM state of each transcript is cached (the reference has no LSTM).
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "synthetic_model.hpp"
#include "tbeam/decoder.hpp"
#include "tbeam/fixtures.hpp"
#include "tbeam/hyp_store.hpp"
#include "tbeam/kernels.hpp"
#include "tbeam/ngram_lm.hpp"
#include "tbeam_b200.h"

namespace {

thread_local std::string g_err;

class ShimModel : public tbeam::EmissionModel {
public:
    ShimModel(const oracle::SyntheticModel& m, const float* enc, int frames, int max_len)
        : M_(m), vocab_(tbeam::Vocabulary::synthetic(m.V)), frames_(frames) {
        order_ = M_.lstm ? max_len : M_.n;
        encp_.resize(static_cast<std::size_t>(frames) * M_.J);
        for (int t = 0; t < frames; ++t)
            M_.enc_proj(enc + static_cast<std::size_t>(t) * M_.D, &encp_[static_cast<std::size_t>(t) * M_.J]);
    }
    const tbeam::Vocabulary& vocab() const override { return vocab_; }
    int context_order() const override { return order_; }
    int num_frames() const override { return frames_; }
    void score_row(int frame, std::span<const tbeam::TokenId> window,
                   std::span<double> out) const override {
        std::vector<double> pred(M_.J);
        if (M_.lstm) {
            std::vector<std::int32_t> tx;
            for (const auto t : window)
                if (t != tbeam::kNoToken) tx.push_back(t);
            pred = state_of(tx)->pred;
        } else {
            M_.stateless_pred(window.data(), pred.data());
        }
        M_.joint(&encp_[static_cast<std::size_t>(frame) * M_.J], pred.data(), out.data(), nullptr);
    }

private:
    std::shared_ptr<const oracle::LstmState> state_of(const std::vector<std::int32_t>& tx) const {
        auto it = cache_.find(tx);
        if (it != cache_.end()) return it->second;
        std::shared_ptr<const oracle::LstmState> s;
        if (tx.empty()) {
            s = std::make_shared<oracle::LstmState>(M_.lstm_start());
        } else {
            std::vector<std::int32_t> prefix(tx.begin(), tx.end() - 1);
            s = std::make_shared<oracle::LstmState>(M_.lstm_step(*state_of(prefix), tx.back()));
        }
        cache_.emplace(tx, s);
        return s;
    }

    const oracle::SyntheticModel& M_;
    tbeam::Vocabulary vocab_;
    int frames_;
    int order_;
    std::vector<double> encp_;
    mutable std::map<std::vector<std::int32_t>, std::shared_ptr<const oracle::LstmState>> cache_;
};

// which reference entry point to call
enum { REF_GREEDY = 0, REF_ALSD_PP = 1, REF_AES_PP = 2, REF_BEAM_ALSD = 3, REF_BEAM_AES = 4 };

tbeam::DecodeConfig to_ref_cfg(const tbeam_decode_config& c, const tbeam::NGramLm* lm) {
    tbeam::DecodeConfig r;
    r.beam = c.beam;
    r.max_symbols_per_frame = c.max_symbols_per_frame;
    r.aes_expansions_per_frame = c.aes_expansions_per_frame;
    r.max_len = c.max_len;
    r.return_nbest = c.return_nbest;
    r.aes_prefix_search = c.aes_prefix_search != 0;
    r.lm = lm;
    r.fusion.lambda = c.lm_weight;
    r.fusion.blank_mode = c.blank_mode == TBEAM_BLANK_SCORED ? tbeam::BlankMode::kScored
                                                            : tbeam::BlankMode::kOmit;
    r.fusion.pruning = c.prune_mode == TBEAM_PRUNE_EARLY ? tbeam::PruneMode::kEarly
                                                        : tbeam::PruneMode::kLate;
    r.fusion.eos_enabled = c.eos_enabled != 0;
    r.hash_params.base = c.hash_base;
    r.hash_params.modulus = c.hash_modulus;
    return r;
}

tbeam::DecodeResult run_ref(int which, std::span<const tbeam::StreamInput> streams,
                            const tbeam::DecodeConfig& cfg) {
    switch (which) {
        case REF_GREEDY: return tbeam::greedy_batched(streams, cfg);
        case REF_ALSD_PP: return tbeam::alsd_pp(streams, cfg);
        case REF_AES_PP: return tbeam::aes_pp(streams, cfg);
        case REF_BEAM_ALSD: return tbeam::reference_beam(streams, cfg, tbeam::RefAlgo::kAlsd);
        default: return tbeam::reference_beam(streams, cfg, tbeam::RefAlgo::kAes);
    }
}

void store_result(const tbeam::StreamResult& s, int b, tbeam_results* res) {
    res->nbest_count[b] = static_cast<int32_t>(s.nbest.size());
    for (int r = 0; r < res->nbest; ++r) {
        const std::size_t e = static_cast<std::size_t>(b) * res->nbest + r;
        res->lengths[e] = 0;
        res->scores[e] = -std::numeric_limits<double>::infinity();
        if (r >= static_cast<int>(s.nbest.size())) continue;
        const auto& nb = s.nbest[r];
        const int L = std::min<int>(static_cast<int>(nb.tokens.size()), res->max_len);
        res->lengths[e] = L;
        res->scores[e] = nb.score;
        for (int i = 0; i < L; ++i) res->tokens[e * res->max_len + i] = nb.tokens[i];
    }
    if (res->counters) {
        uint64_t* c = res->counters + static_cast<std::size_t>(b) * TBEAM_NUM_COUNTERS;
        c[0] = s.counters.frames;
        c[1] = s.counters.scoring_rounds;
        c[2] = s.counters.scored_slots;
        c[3] = s.counters.lm_token_queries;
        c[4] = s.counters.lm_vocab_queries;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

const char* ref_kernels_name() { return tbeam::kernels::active().name.data(); }

uint64_t ref_update_hash(uint64_t h, int32_t tok, uint64_t base, uint64_t mod) {
    tbeam::HashParams p;
    p.base = base;
    p.modulus = mod;
    return tbeam::update_hash(h, tok, p);
}
double ref_logadd(double a, double b) { return tbeam::logadd(a, b); }
double ref_log1mexp(double x) { return tbeam::log1mexp(x); }

int32_t ref_prune_topk(const double* scores, int32_t n, int32_t k, int32_t* idx, double* out) {
    try {
        tbeam::prune_topk(std::span<const double>(scores, n), k, std::span<int32_t>(idx, k),
                          std::span<double>(out, k));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Synthetic vocabulary token string (Vocabulary::synthetic, model.cpp:55-75).
// Returns the byte length written (without NUL) or -1.
int32_t ref_vocab_token(int32_t vocab, int32_t id, char* buf, int32_t cap) {
    static thread_local std::unique_ptr<tbeam::Vocabulary> cache;
    if (!cache || cache->size() != vocab) cache = std::make_unique<tbeam::Vocabulary>(tbeam::Vocabulary::synthetic(vocab));
    const std::string& s = cache->token(id);
    if (static_cast<int32_t>(s.size()) + 1 > cap) return -1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int32_t>(s.size());
}

// make_random_consistent_arpa (fixtures.cpp:155-248); caller frees with ref_free.
char* ref_random_arpa(uint64_t seed, int32_t vocab, int32_t order, int32_t with_eos) {
    const std::string s = tbeam::make_random_consistent_arpa(
        seed, tbeam::Vocabulary::synthetic(vocab), order, with_eos != 0);
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}
void ref_free(void* p) { std::free(p); }

// ---- LM -----------------------------------------------------------------------
void* ref_lm_create(const char* text, int32_t vocab, int32_t strict) {
    try {
        return new tbeam::NGramLm(tbeam::NGramLm::parse_arpa_text(
            text, "lm.arpa", tbeam::Vocabulary::synthetic(vocab), strict != 0));
    } catch (const tbeam::ParseError& e) {
        g_err = e.what();
        return nullptr;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_lm_destroy(void* lm) { delete static_cast<tbeam::NGramLm*>(lm); }
int64_t ref_lm_num_nodes(void* lm) { return static_cast<int64_t>(static_cast<tbeam::NGramLm*>(lm)->num_nodes()); }
int32_t ref_lm_order(void* lm) { return static_cast<tbeam::NGramLm*>(lm)->order(); }
static tbeam::NGramLm::State ref_walk(const tbeam::NGramLm* lm, const int32_t* h, int32_t n) {
    auto s = lm->initial_state();
    for (int i = 0; i < n; ++i) s = lm->advance(s, h[i]);
    return s;
}
int32_t ref_lm_state(void* lm, const int32_t* h, int32_t n) {
    return ref_walk(static_cast<tbeam::NGramLm*>(lm), h, n);
}
double ref_lm_score_token(void* lm, const int32_t* h, int32_t n, int32_t tok) {
    auto* p = static_cast<tbeam::NGramLm*>(lm);
    return p->score_token(ref_walk(p, h, n), tok);
}
double ref_lm_score_eos(void* lm, const int32_t* h, int32_t n) {
    auto* p = static_cast<tbeam::NGramLm*>(lm);
    return p->score_eos(ref_walk(p, h, n));
}
void ref_lm_score_vocab(void* lm, const int32_t* h, int32_t n, double* out) {
    auto* p = static_cast<tbeam::NGramLm*>(lm);
    tbeam::NGramLm::Scratch scratch;
    p->score_vocab(ref_walk(p, h, n), std::span<double>(out, p->vocab_size()), scratch);
}

// ---- decoders -------------------------------------------------------------------
// which: 0 greedy_batched, 1 alsd_pp, 2 aes_pp, 3 reference_beam(kAlsd),
//        4 reference_beam(kAes).  One call = one batched session.
int32_t ref_decode(int32_t which, const tbeam_model_dims* dims, const tbeam_model_weights* w,
                   void* lm, const tbeam_decode_config* cfg, const float* enc,
                   const int32_t* lengths, int32_t batch, int32_t max_frames,
                   tbeam_results* res, double* wall_seconds) {
    try {
        if (dims->num_durations > 0) {
            g_err = "reference has no TDT decoder (SPEC.md:14)";
            return TBEAM_UNSUPPORTED;
        }
        oracle::SyntheticModel M(*dims, *w, tbeam::kernels::active().matvec,
                                 tbeam::kernels::active().log_softmax);
        std::vector<std::unique_ptr<ShimModel>> models;
        std::vector<tbeam::StreamInput> streams;
        for (int b = 0; b < batch; ++b) {
            models.push_back(std::make_unique<ShimModel>(
                M, enc + static_cast<std::size_t>(b) * max_frames * M.D, max_frames, cfg->max_len));
            streams.push_back({models.back().get(), lengths[b]});
        }
        const auto rc = to_ref_cfg(*cfg, static_cast<const tbeam::NGramLm*>(lm));
        const tbeam::DecodeResult r = run_ref(which, streams, rc);
        for (int b = 0; b < batch; ++b) store_result(r.streams[b], b, res);
        if (wall_seconds) *wall_seconds = r.wall_seconds;
        return TBEAM_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return TBEAM_INVALID_ARGUMENT;
    } catch (const tbeam::CapacityError& e) {
        g_err = e.what();
        return TBEAM_CAPACITY;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TBEAM_VALIDATION;
    }
}

// CPU baseline harness: an external pool of `threads`
// workers, each decoding B=1 sessions from a shared utterance queue (the
// reference's own multi-stream sessions race).  Decodes utterances
// [0, count) of the batch; returns wall seconds or -1.
double ref_decode_pool(int32_t which, const tbeam_model_dims* dims, const tbeam_model_weights* w,
                       void* lm, const tbeam_decode_config* cfg, const float* enc,
                       const int32_t* lengths, int32_t count, int32_t max_frames,
                       int32_t threads, tbeam_results* res) {
    try {
        oracle::SyntheticModel M(*dims, *w, tbeam::kernels::active().matvec,
                                 tbeam::kernels::active().log_softmax);
        const auto rc = to_ref_cfg(*cfg, static_cast<const tbeam::NGramLm*>(lm));
        std::atomic<int> next{0};
        std::mutex mu;
        std::string err;
        const auto t0 = std::chrono::steady_clock::now();
        auto worker = [&]() {
            try {
                for (int b = next.fetch_add(1); b < count; b = next.fetch_add(1)) {
                    ShimModel sm(M, enc + static_cast<std::size_t>(b) * max_frames * M.D,
                                 max_frames, cfg->max_len);
                    const tbeam::StreamInput s{&sm, lengths[b]};
                    const tbeam::DecodeResult r =
                        run_ref(which, std::span<const tbeam::StreamInput>(&s, 1), rc);
                    if (res) store_result(r.streams[0], b, res);
                }
            } catch (const std::exception& e) {
                std::lock_guard<std::mutex> g(mu);
                err = e.what();
            }
        };
        std::vector<std::thread> pool;
        for (int i = 1; i < threads; ++i) pool.emplace_back(worker);
        worker();
        for (auto& th : pool) th.join();
        const double wall =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (!err.empty()) {
            g_err = err;
            return -1.0;
        }
        return wall;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

}  // extern "C"
