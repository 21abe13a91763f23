// tbeam_b200_reference.hpp -- the B200 decoder behind the reference's OWN
// types and function signatures, for the reference's CLI / callers:
//
//   using DecodeFn = tbeam::DecodeResult (*)(std::span<const tbeam::StreamInput>,
//                                            const tbeam::DecodeConfig&);   // commands.cpp:136
//
//   tbeam_b200::reference::algo_fn("alsd++-b200")  -> a DecodeFn (likewise
//   "aes++-b200", "greedy-b200", and "aes-ref-b200" = canonical AES++, the
//   reference_beam(kAes) semantics) that the reference's decode_chunked
//   (commands.cpp:156-173) and cmd_bench grid (commands.cpp:374-415) call
//   unchanged.
//
// Include path: -I<repo>/include -I<reference>/proj/include; link
// -ltbeam_b200.  Header-only on top of tbeam_b200.hpp (the C-ABI shim).
//
// What a caller provides beyond the reference's inputs:
//   * bind(decoder): the GPU context holding the model weights
//     (Decoder::set_model) -- the device model replaces the virtual
//     EmissionModel::score_row calls;
//   * every StreamInput::model must also implement FrameSource (its encoder
//     frames, [num_frames, enc_dim] fp32) -- decode() checks with
//     dynamic_cast and throws std::invalid_argument otherwise;
//   * bind_lm(lm, arpa_text, vocab): the LM the config's `lm` pointer names is
//     uploaded from the same ARPA text (NGramLm::parse_arpa_text semantics,
//     ngram_lm.cpp:52-318); a config naming a different LM is rejected.
// Errors keep the reference's taxonomy: std::invalid_argument for the
// validate_streams checks (decoder.cpp:16-38), tbeam::ParseError /
// ValidationError / CapacityError for the matching statuses.
#pragma once

#include <algorithm>
#include <chrono>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "tbeam/decoder.hpp"
#include "tbeam/types.hpp"
#include "tbeam_b200.hpp"

namespace tbeam_b200::reference {

// The encoder side of a stream's model: what the GPU decoder consumes in
// place of score_row (model.hpp:62-74).
class FrameSource {
public:
    virtual ~FrameSource() = default;
    virtual const float* encoder_frames() const = 0;  // [num_frames(), encoder_dim()]
    virtual int encoder_dim() const = 0;
};

struct Binding {
    tbeam_b200::Decoder* decoder = nullptr;
    const tbeam::NGramLm* lm = nullptr;  // the reference LM object the uploaded one mirrors
};

inline Binding& binding() {
    static Binding b;
    return b;
}

inline void bind(tbeam_b200::Decoder* decoder) { binding().decoder = decoder; }

inline void bind_lm(const tbeam::NGramLm* lm, const std::string& arpa, const std::vector<std::string>& vocab,
                    bool strict = false) {
    Binding& b = binding();
    if (b.decoder == nullptr) throw std::invalid_argument("bind_lm: bind a decoder first");
    try {
        b.decoder->set_lm(arpa, vocab, strict);
    } catch (const tbeam_b200::ParseError& e) {
        throw tbeam::ParseError("lm.arpa", 0, e.what());
    } catch (const tbeam_b200::ValidationError& e) {
        throw tbeam::ValidationError(e.what());
    }
    b.lm = lm;
}

// tbeam::DecodeConfig (decoder.hpp:23-42) -> the B200 config, field for field
inline tbeam_b200::DecodeConfig convert(const tbeam::DecodeConfig& cfg, bool aes_pp_quirk) {
    tbeam_b200::DecodeConfig c;
    c.beam = cfg.beam;
    c.max_symbols_per_frame = cfg.max_symbols_per_frame;
    c.aes_expansions_per_frame = cfg.aes_expansions_per_frame;
    c.max_len = cfg.max_len;
    c.return_nbest = cfg.return_nbest;
    c.aes_prefix_search = cfg.aes_prefix_search;
    c.fusion.lambda = cfg.fusion.lambda;
    c.fusion.blank_mode = cfg.fusion.blank_mode == tbeam::BlankMode::kScored ? tbeam_b200::BlankMode::kScored
                                                                            : tbeam_b200::BlankMode::kOmit;
    c.fusion.pruning = cfg.fusion.pruning == tbeam::PruneMode::kEarly ? tbeam_b200::PruneMode::kEarly
                                                                     : tbeam_b200::PruneMode::kLate;
    c.fusion.eos_enabled = cfg.fusion.eos_enabled;
    c.hash_params.base = cfg.hash_params.base;
    c.hash_params.modulus = cfg.hash_params.modulus;
    c.aes_slot_donated_quirk = aes_pp_quirk;
    return c;
}

// One decode through the bound GPU context with the reference's types.
inline tbeam::DecodeResult decode(int algo, bool aes_pp_quirk, std::span<const tbeam::StreamInput> streams,
                                  const tbeam::DecodeConfig& cfg) {
    const auto t0 = std::chrono::steady_clock::now();
    Binding& bd = binding();
    if (bd.decoder == nullptr) throw std::invalid_argument("decode: no B200 decoder bound");
    if (streams.empty()) throw std::invalid_argument("decode: no streams");
    if (cfg.lm != nullptr && cfg.lm != bd.lm)
        throw std::invalid_argument("decode: the config's LM is not the one uploaded to the B200 decoder");
    std::vector<tbeam_b200::StreamInput> in;
    in.reserve(streams.size());
    for (const tbeam::StreamInput& s : streams) {
        // decoder.cpp:22-24
        if (s.model == nullptr || s.num_frames < 1 || s.num_frames > s.model->num_frames())
            throw std::invalid_argument("decode: bad stream input");
        const auto* fs = dynamic_cast<const FrameSource*>(s.model);
        if (fs == nullptr)
            throw std::invalid_argument("decode: the stream's model carries no encoder frames (FrameSource)");
        in.push_back({fs->encoder_frames(), s.num_frames});
    }
    const tbeam_b200::DecodeConfig c = convert(cfg, aes_pp_quirk);
    tbeam_b200::DecodeResult r;
    try {
        if (cfg.fusion.lambda > 0.0 && cfg.lm == nullptr)
            throw std::invalid_argument("decode: LM weight set but no LM given");
        r = bd.decoder->decode(algo, in, c);
    } catch (const tbeam_b200::ParseError& e) {
        throw tbeam::ParseError("lm.arpa", 0, e.what());
    } catch (const tbeam_b200::ValidationError& e) {
        throw tbeam::ValidationError(e.what());
    } catch (const tbeam_b200::CapacityError& e) {
        throw tbeam::CapacityError(e.what());
    }
    tbeam::DecodeResult out;
    out.streams.resize(r.streams.size());
    for (std::size_t b = 0; b < r.streams.size(); ++b) {
        for (auto& n : r.streams[b].nbest) out.streams[b].nbest.push_back({std::move(n.tokens), n.score});
        const auto& k = r.streams[b].counters;
        out.streams[b].counters = {k.frames, k.scoring_rounds, k.scored_slots, k.lm_token_queries,
                                   k.lm_vocab_queries};
    }
    out.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

// decoder.hpp:75-83, on the GPU
inline tbeam::DecodeResult greedy_batched(std::span<const tbeam::StreamInput> s, const tbeam::DecodeConfig& c) {
    return decode(TBEAM_ALGO_GREEDY, false, s, c);
}
inline tbeam::DecodeResult alsd_pp(std::span<const tbeam::StreamInput> s, const tbeam::DecodeConfig& c) {
    return decode(TBEAM_ALGO_ALSD, false, s, c);
}
// the shipped aes_pp, bit for bit (its stale per-slot donated flag)
inline tbeam::DecodeResult aes_pp(std::span<const tbeam::StreamInput> s, const tbeam::DecodeConfig& c) {
    return decode(TBEAM_ALGO_AES, true, s, c);
}
// canonical AES++ (reference_beam(kAes) semantics)
inline tbeam::DecodeResult aes_canonical(std::span<const tbeam::StreamInput> s, const tbeam::DecodeConfig& c) {
    return decode(TBEAM_ALGO_AES, false, s, c);
}

using DecodeFn = tbeam::DecodeResult (*)(std::span<const tbeam::StreamInput>, const tbeam::DecodeConfig&);

// commands.cpp:138-153's algo_fn, B200 entries: nullptr for any other name
// (the caller's own algo_fn handles those)
inline DecodeFn algo_fn(const std::string& algo) {
    if (algo == "greedy-b200") return &greedy_batched;
    if (algo == "alsd++-b200") return &alsd_pp;
    if (algo == "aes++-b200") return &aes_pp;
    if (algo == "aes-ref-b200") return &aes_canonical;
    return nullptr;
}

// commands.cpp:156-173: sessions of at most `batch` streams
inline tbeam::DecodeResult decode_chunked(DecodeFn fn, std::span<const tbeam::StreamInput> streams,
                                          const tbeam::DecodeConfig& cfg, int batch) {
    tbeam::DecodeResult all;
    const auto start = std::chrono::steady_clock::now();
    for (std::size_t off = 0; off < streams.size(); off += static_cast<std::size_t>(batch)) {
        const std::size_t n = std::min<std::size_t>(static_cast<std::size_t>(batch), streams.size() - off);
        tbeam::DecodeResult part = fn(streams.subspan(off, n), cfg);
        for (auto& s : part.streams) all.streams.push_back(std::move(s));
    }
    all.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    return all;
}

}  // namespace tbeam_b200::reference
