// tbeam_b200.hpp -- header-only C++ shim over the C-ABI (tbeam_b200.h) that
// re-exposes the reference decoder API (proj/include/tbeam/decoder.hpp:18-91)
// for drop-in use from C++:
//
//   tbeam::greedy_batched(streams, cfg)  ->  tbeam_b200::greedy_batched(dec, streams, cfg)
//   tbeam::alsd_pp(streams, cfg)         ->  tbeam_b200::alsd_pp(dec, streams, cfg)
//   tbeam::aes_pp(streams, cfg)          ->  tbeam_b200::aes_pp(dec, streams, cfg)
//
// DecodeConfig / FusionConfig / HashParams / NBestEntry / StreamResult /
// DecodeResult keep the reference's field names and defaults; errors map back
// onto the reference's exception types (std::invalid_argument, ParseError,
// ValidationError, CapacityError -- types.hpp:29-52).  The one structural
// change: a StreamInput carries encoder frames (the model lives on the GPU in
// a Decoder) instead of an EmissionModel pointer; see INTEGRATION.md.
#pragma once

#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "tbeam_b200.h"

namespace tbeam_b200 {

using TokenId = std::int32_t;

class ParseError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ValidationError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class CapacityError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(tbeam_status s) {
    if (s == TBEAM_OK) return;
    const std::string msg = tbeam_last_error();
    switch (s) {
        case TBEAM_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case TBEAM_PARSE: throw ParseError(msg);
        case TBEAM_VALIDATION: throw ValidationError(msg);
        case TBEAM_CAPACITY: throw CapacityError(msg);
        default: throw CudaError(msg);
    }
}

enum class BlankMode { kOmit = TBEAM_BLANK_OMIT, kScored = TBEAM_BLANK_SCORED };
enum class PruneMode { kEarly = TBEAM_PRUNE_EARLY, kLate = TBEAM_PRUNE_LATE };

struct FusionConfig {  // fusion.hpp:19-24
    double lambda = 0.0;
    BlankMode blank_mode = BlankMode::kOmit;
    PruneMode pruning = PruneMode::kLate;
    bool eos_enabled = false;
};

struct HashParams {  // hyp_store.hpp:15-18
    std::uint64_t base = 1'000'003;
    std::uint64_t modulus = (std::uint64_t{1} << 61) - 1;
};

struct DecodeConfig {  // decoder.hpp:23-42 (+ B200 additions)
    int beam = 4;
    int max_symbols_per_frame = 10;
    int aes_expansions_per_frame = 2;
    int max_len = 256;
    int return_nbest = 1;
    bool aes_prefix_search = true;
    FusionConfig fusion;
    HashParams hash_params;
    int merge_mode = TBEAM_MERGE_LOGSUMEXP;
    bool aes_slot_donated_quirk = false;

    tbeam_decode_config to_c(int algo) const {
        tbeam_decode_config c;
        tbeam_decode_config_init(&c);
        c.algo = algo;
        c.beam = beam;
        c.max_symbols_per_frame = max_symbols_per_frame;
        c.aes_expansions_per_frame = aes_expansions_per_frame;
        c.max_len = max_len;
        c.return_nbest = return_nbest;
        c.aes_prefix_search = aes_prefix_search ? 1 : 0;
        c.lm_weight = fusion.lambda;
        c.blank_mode = static_cast<int32_t>(fusion.blank_mode);
        c.prune_mode = static_cast<int32_t>(fusion.pruning);
        c.eos_enabled = fusion.eos_enabled ? 1 : 0;
        c.merge_mode = merge_mode;
        c.hash_base = hash_params.base;
        c.hash_modulus = hash_params.modulus;
        c.aes_slot_donated_quirk = aes_slot_donated_quirk ? 1 : 0;
        return c;
    }
};

struct Counters {  // decoder.hpp:44-50
    std::uint64_t frames = 0, scoring_rounds = 0, scored_slots = 0, lm_token_queries = 0,
                  lm_vocab_queries = 0;
};

struct NBestEntry {  // decoder.hpp:52-55 + alignment / TDT durations
    std::vector<TokenId> tokens;
    double score = 0.0;
    std::vector<std::int32_t> frames;
    std::vector<std::int32_t> durations;
};

struct StreamResult {
    std::vector<NBestEntry> nbest;
    Counters counters;
};

struct DecodeResult {
    std::vector<StreamResult> streams;
    double wall_seconds = 0.0;
    std::uint64_t total_frames() const {
        std::uint64_t n = 0;
        for (const auto& s : streams) n += s.counters.frames;
        return n;
    }
};

// decoder.hpp:18-21 with encoder frames in place of the EmissionModel*:
// enc points at >= num_frames rows of enc_dim floats (host memory).
struct StreamInput {
    const float* enc = nullptr;
    int num_frames = 0;
};

// One GPU decoder context holding the model (and optional LM).
class Decoder {
public:
    explicit Decoder(int device = 0) { check(tbeam_create(device, &ctx_)); }
    ~Decoder() {
        if (ctx_) tbeam_destroy(ctx_);
    }
    Decoder(const Decoder&) = delete;
    Decoder& operator=(const Decoder&) = delete;

    void set_model(const tbeam_model_dims& dims, const tbeam_model_weights& w) {
        check(tbeam_set_model(ctx_, &dims, &w));
        dims_ = dims;
    }
    // NGramLm::parse_arpa_text against the ASR token table (ngram_lm.hpp:38-42)
    void set_lm(const std::string& arpa, const std::vector<std::string>& vocab, bool strict = false) {
        std::vector<const char*> p;
        p.reserve(vocab.size());
        for (const auto& s : vocab) p.push_back(s.c_str());
        check(tbeam_set_lm_arpa(ctx_, arpa.data(), arpa.size(), p.data(), static_cast<int32_t>(p.size()),
                                strict ? 1 : 0));
    }
    void clear_lm() { check(tbeam_clear_lm(ctx_)); }

    DecodeResult decode(int algo, std::span<const StreamInput> streams, const DecodeConfig& cfg) {
        if (streams.empty()) throw std::invalid_argument("decode: no streams");
        int T = 0;
        for (const auto& s : streams) {
            if (s.enc == nullptr) throw std::invalid_argument("decode: bad stream input");
            T = std::max(T, s.num_frames);
        }
        const int B = static_cast<int>(streams.size());
        const int D = dims_.enc_dim;
        std::vector<float> enc(static_cast<std::size_t>(B) * T * D, 0.f);
        std::vector<std::int32_t> lens(B);
        for (int b = 0; b < B; ++b) {
            lens[b] = streams[b].num_frames;
            if (lens[b] > 0)
                std::memcpy(enc.data() + static_cast<std::size_t>(b) * T * D, streams[b].enc,
                            sizeof(float) * lens[b] * D);
        }
        const int nb = algo == TBEAM_ALGO_GREEDY ? 1 : cfg.return_nbest;
        const int L = cfg.max_len;
        std::vector<std::int32_t> cnt(B), len(static_cast<std::size_t>(B) * nb), tok(static_cast<std::size_t>(B) * nb * L),
            fr(tok.size()), du(tok.size());
        std::vector<double> sc(static_cast<std::size_t>(B) * nb);
        std::vector<std::uint64_t> ctr(static_cast<std::size_t>(B) * TBEAM_NUM_COUNTERS);
        tbeam_results r{B, nb, L, cnt.data(), len.data(), sc.data(), tok.data(), fr.data(), du.data(), ctr.data()};
        const tbeam_decode_config c = cfg.to_c(algo);
        check(tbeam_decode(ctx_, &c, enc.data(), 0, lens.data(), B, T, &r, nullptr));
        DecodeResult out;
        out.streams.resize(B);
        for (int b = 0; b < B; ++b) {
            auto& s = out.streams[b];
            for (int q = 0; q < cnt[b]; ++q) {
                const std::size_t e = static_cast<std::size_t>(b) * nb + q;
                NBestEntry n;
                n.score = sc[e];
                n.tokens.assign(tok.begin() + e * L, tok.begin() + e * L + len[e]);
                n.frames.assign(fr.begin() + e * L, fr.begin() + e * L + len[e]);
                n.durations.assign(du.begin() + e * L, du.begin() + e * L + len[e]);
                s.nbest.push_back(std::move(n));
            }
            const std::uint64_t* cc = ctr.data() + static_cast<std::size_t>(b) * TBEAM_NUM_COUNTERS;
            s.counters = Counters{cc[0], cc[1], cc[2], cc[3], cc[4]};
        }
        return out;
    }

    // Pipelined serving (tbeam_stage_inputs / tbeam_decode_staged): stage
    // batch i+1 (async H2D into the next of two device slots) before decoding
    // batch i.  enc is [B, T, enc_dim] fp32 host memory (pinned for overlap)
    // and must stay unchanged until decode_staged of its batch returns.
    void stage(const float* enc, const std::vector<std::int32_t>& lengths, int max_frames) {
        check(tbeam_stage_inputs(ctx_, enc, lengths.data(), static_cast<int32_t>(lengths.size()), max_frames));
        staged_.push_back(static_cast<int>(lengths.size()));
    }
    DecodeResult decode_staged(int algo, const DecodeConfig& cfg) {
        if (staged_.empty()) throw std::invalid_argument("decode: nothing staged");
        const int B = staged_.front();
        staged_.erase(staged_.begin());
        const int nb = algo == TBEAM_ALGO_GREEDY ? 1 : cfg.return_nbest;
        Buffers buf(B, nb, cfg.max_len);
        tbeam_results r = buf.view();
        const tbeam_decode_config c = cfg.to_c(algo);
        check(tbeam_decode_staged(ctx_, &c, &r, nullptr));
        return buf.result();
    }

private:
    // caller-side result arrays of one decode (tbeam_results views them)
    struct Buffers {
        int B, nb, L;
        std::vector<std::int32_t> cnt, len, tok, fr, du;
        std::vector<double> sc;
        std::vector<std::uint64_t> ctr;
        Buffers(int b, int n, int l)
            : B(b), nb(n), L(l), cnt(b), len(static_cast<std::size_t>(b) * n), tok(static_cast<std::size_t>(b) * n * l),
              fr(tok.size()), du(tok.size()), sc(static_cast<std::size_t>(b) * n),
              ctr(static_cast<std::size_t>(b) * TBEAM_NUM_COUNTERS) {}
        tbeam_results view() {
            return tbeam_results{B, nb, L, cnt.data(), len.data(), sc.data(), tok.data(), fr.data(), du.data(),
                                 ctr.data()};
        }
        DecodeResult result() const {
            DecodeResult out;
            out.streams.resize(B);
            for (int b = 0; b < B; ++b) {
                auto& s = out.streams[b];
                for (int q = 0; q < cnt[b]; ++q) {
                    const std::size_t e = static_cast<std::size_t>(b) * nb + q;
                    NBestEntry n;
                    n.score = sc[e];
                    n.tokens.assign(tok.begin() + e * L, tok.begin() + e * L + len[e]);
                    n.frames.assign(fr.begin() + e * L, fr.begin() + e * L + len[e]);
                    n.durations.assign(du.begin() + e * L, du.begin() + e * L + len[e]);
                    s.nbest.push_back(std::move(n));
                }
                const std::uint64_t* cc = ctr.data() + static_cast<std::size_t>(b) * TBEAM_NUM_COUNTERS;
                s.counters = Counters{cc[0], cc[1], cc[2], cc[3], cc[4]};
            }
            return out;
        }
    };

    tbeam_ctx* ctx_ = nullptr;
    tbeam_model_dims dims_{};
    std::vector<int> staged_;
};

inline DecodeResult greedy_batched(Decoder& d, std::span<const StreamInput> s, const DecodeConfig& cfg) {
    return d.decode(TBEAM_ALGO_GREEDY, s, cfg);
}
inline DecodeResult alsd_pp(Decoder& d, std::span<const StreamInput> s, const DecodeConfig& cfg) {
    return d.decode(TBEAM_ALGO_ALSD, s, cfg);
}
inline DecodeResult aes_pp(Decoder& d, std::span<const StreamInput> s, const DecodeConfig& cfg) {
    return d.decode(TBEAM_ALGO_AES, s, cfg);
}

}  // namespace tbeam_b200
