// TEST INFRASTRUCTURE -- the reference-typed adapter (include/tbeam_b200_reference.hpp)
// driven the way the reference's CLI drives its decoders: algo_fn by name ->
// decode_chunked (commands.cpp:138-173), and a cmd_bench-style grid
// (commands.cpp:374-415).  Built by oracle/Makefile against the UNMODIFIED
// reference (its headers and objects, oracle/_ref/obj) and the B200 library;
// tests/test_ref_adapter.py runs it on the GPU and checks that every
// "<algo>-b200" result equals the reference's own "<algo>" on the same streams.
//
//   ref_adapter_demo <model.bin> [--lm file.arpa --lambda L --blank omit|scored
//                    --pruning early|late --eos] [--beam K] [--nbest N] [--batch C]
//                    [--algos a,b,...] [--bench --batch-grid 1,8 --beam-grid 2,4 --repeats R]
//
// model.bin: tbeam_model_dims (raw), then per tbeam_model_weights field (in
// declaration order) an int64 count + that many floats, then int32 B, T, D,
// B*T*D floats of encoder frames and B int32 lengths.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "synthetic_model.hpp"
#include "tbeam/decoder.hpp"
#include "tbeam/model.hpp"
#include "tbeam/ngram_lm.hpp"
#include "tbeam_b200_reference.hpp"

namespace {

// A stream of the synthetic transducer, seen by BOTH decoders: the reference
// scores it through EmissionModel::score_row (model.hpp:62-74), the B200 path
// reads its encoder frames (FrameSource).  LSTM: the window is the whole
// transcript (context_order = max_len), states cached per transcript.
class Stream : public tbeam::EmissionModel, public tbeam_b200::reference::FrameSource {
public:
    Stream(const oracle::SyntheticModel& m, const float* enc, int frames, int max_len)
        : M_(m), vocab_(tbeam::Vocabulary::synthetic(m.V)), frames_(frames), enc_(enc) {
        order_ = M_.lstm ? max_len : M_.n;
        encp_.resize(static_cast<std::size_t>(frames) * M_.J);
        for (int t = 0; t < frames; ++t)
            M_.enc_proj(enc + static_cast<std::size_t>(t) * M_.D, &encp_[static_cast<std::size_t>(t) * M_.J]);
    }
    const tbeam::Vocabulary& vocab() const override { return vocab_; }
    int context_order() const override { return order_; }
    int num_frames() const override { return frames_; }
    void score_row(int frame, std::span<const tbeam::TokenId> window, std::span<double> out) const override {
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
    const float* encoder_frames() const override { return enc_; }
    int encoder_dim() const override { return M_.D; }

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
    int frames_, order_;
    const float* enc_;
    std::vector<double> encp_;
    mutable std::map<std::vector<std::int32_t>, std::shared_ptr<const oracle::LstmState>> cache_;
};

using RefFn = tbeam::DecodeResult (*)(std::span<const tbeam::StreamInput>, const tbeam::DecodeConfig&);

// the reference's own algo_fn (commands.cpp:138-153)
RefFn ref_algo_fn(const std::string& a) {
    if (a == "greedy") return &tbeam::greedy_batched;
    if (a == "alsd++") return &tbeam::alsd_pp;
    if (a == "aes++") return &tbeam::aes_pp;
    if (a == "aes-ref")
        return +[](std::span<const tbeam::StreamInput> s, const tbeam::DecodeConfig& c) {
            return tbeam::reference_beam(s, c, tbeam::RefAlgo::kAes);
        };
    return nullptr;
}

std::vector<std::string> split(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string x;
    while (std::getline(ss, x, ',')) out.push_back(x);
    return out;
}

void print_result(const char* algo, const tbeam::DecodeResult& r) {
    std::printf("{\"algo\": \"%s\", \"wall\": %.6f, \"streams\": [", algo, r.wall_seconds);
    for (std::size_t b = 0; b < r.streams.size(); ++b) {
        const auto& s = r.streams[b];
        std::printf("%s{\"nbest\": [", b ? ", " : "");
        for (std::size_t q = 0; q < s.nbest.size(); ++q) {
            std::printf("%s{\"score\": %.17g, \"tokens\": [", q ? ", " : "", s.nbest[q].score);
            for (std::size_t i = 0; i < s.nbest[q].tokens.size(); ++i)
                std::printf(i ? ",%d" : "%d", s.nbest[q].tokens[i]);
            std::printf("]}");
        }
        const auto& k = s.counters;
        std::printf("], \"counters\": [%llu, %llu, %llu, %llu, %llu]}", (unsigned long long)k.frames,
                    (unsigned long long)k.scoring_rounds, (unsigned long long)k.scored_slots,
                    (unsigned long long)k.lm_token_queries, (unsigned long long)k.lm_vocab_queries);
    }
    std::printf("]}\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_adapter_demo model.bin [options]\n");
        return 2;
    }
    std::map<std::string, std::string> opt;
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        if (k == "--eos" || k == "--bench") opt[k] = "1";
        else if (i + 1 < argc) opt[k] = argv[++i];
    }
    auto get = [&](const char* k, const char* d) { return opt.count(k) ? opt[k] : std::string(d); };

    std::ifstream in(argv[1], std::ios::binary);
    tbeam_model_dims dims{};
    in.read(reinterpret_cast<char*>(&dims), sizeof dims);
    constexpr int kFields = sizeof(tbeam_model_weights) / sizeof(const float*);
    std::vector<std::vector<float>> store(kFields);
    tbeam_model_weights w{};
    const float** slots = reinterpret_cast<const float**>(&w);
    for (int f = 0; f < kFields; ++f) {
        std::int64_t n = 0;
        in.read(reinterpret_cast<char*>(&n), 8);
        store[f].resize(static_cast<std::size_t>(n));
        in.read(reinterpret_cast<char*>(store[f].data()), 4 * n);
        slots[f] = n > 0 ? store[f].data() : nullptr;
    }
    std::int32_t B = 0, T = 0, D = 0;
    in.read(reinterpret_cast<char*>(&B), 4);
    in.read(reinterpret_cast<char*>(&T), 4);
    in.read(reinterpret_cast<char*>(&D), 4);
    std::vector<float> enc(static_cast<std::size_t>(B) * T * D);
    std::vector<std::int32_t> lens(B);
    in.read(reinterpret_cast<char*>(enc.data()), 4 * enc.size());
    in.read(reinterpret_cast<char*>(lens.data()), 4 * B);
    if (!in) {
        std::fprintf(stderr, "bad model.bin\n");
        return 2;
    }

    tbeam::DecodeConfig cfg;
    cfg.beam = std::atoi(get("--beam", "4").c_str());
    cfg.return_nbest = std::atoi(get("--nbest", "2").c_str());
    cfg.max_len = std::atoi(get("--max-len", "256").c_str());
    const oracle::SyntheticModel model(dims, w);
    std::vector<std::unique_ptr<Stream>> owners;
    std::vector<tbeam::StreamInput> streams;
    for (int b = 0; b < B; ++b) {
        owners.push_back(std::make_unique<Stream>(model, enc.data() + static_cast<std::size_t>(b) * T * D, lens[b],
                                                  cfg.max_len));
        streams.push_back({owners.back().get(), lens[b]});
    }

    tbeam_b200::Decoder dec(0);
    dec.set_model(dims, w);
    tbeam_b200::reference::bind(&dec);
    std::unique_ptr<tbeam::NGramLm> lm;
    if (opt.count("--lm")) {
        std::ifstream f(opt["--lm"]);
        std::stringstream ss;
        ss << f.rdbuf();
        const tbeam::Vocabulary vocab = tbeam::Vocabulary::synthetic(dims.vocab_size);
        lm = std::make_unique<tbeam::NGramLm>(tbeam::NGramLm::parse_arpa_text(ss.str(), "lm.arpa", vocab, false));
        std::vector<std::string> words;
        for (int i = 0; i < dims.vocab_size; ++i) words.push_back(vocab.token(i));
        tbeam_b200::reference::bind_lm(lm.get(), ss.str(), words);
        cfg.lm = lm.get();
        cfg.fusion.lambda = std::atof(get("--lambda", "0.5").c_str());
        cfg.fusion.blank_mode = get("--blank", "omit") == "scored" ? tbeam::BlankMode::kScored : tbeam::BlankMode::kOmit;
        cfg.fusion.pruning = get("--pruning", "late") == "early" ? tbeam::PruneMode::kEarly : tbeam::PruneMode::kLate;
        cfg.fusion.eos_enabled = opt.count("--eos") > 0;
    }
    const std::span<const tbeam::StreamInput> all(streams);
    const int batch = std::atoi(get("--batch", "1000000").c_str());

    if (!opt.count("--bench")) {
        for (const std::string& a : split(get("--algos", "greedy,alsd++,aes++,aes-ref"))) {
            RefFn rf = ref_algo_fn(a);
            auto bf = tbeam_b200::reference::algo_fn(a == "aes-ref" ? "aes-ref-b200" : a + "-b200");
            if (!rf || !bf) {
                std::fprintf(stderr, "unknown algo %s\n", a.c_str());
                return 2;
            }
            print_result(a.c_str(), tbeam_b200::reference::decode_chunked(rf, all, cfg, batch));
            const std::string name = a + "-b200";
            print_result(name.c_str(), tbeam_b200::reference::decode_chunked(bf, all, cfg, batch));
        }
        return 0;
    }
    // cmd_bench grid: algo x batch x beam, warm-up then mean of `repeats` runs,
    // RTFx = frames * seconds_per_frame / wall (metrics.cpp:128-158)
    const double spf = std::atof(get("--seconds-per-frame", "0.08").c_str());
    const int repeats = std::atoi(get("--repeats", "3").c_str());
    for (const std::string& a : split(get("--algos", "alsd++,alsd++-b200"))) {
        RefFn fn = a.find("-b200") != std::string::npos ? tbeam_b200::reference::algo_fn(a) : ref_algo_fn(a);
        if (!fn) {
            std::fprintf(stderr, "unknown algo %s\n", a.c_str());
            return 2;
        }
        for (const std::string& bs : split(get("--batch-grid", "8"))) {
            for (const std::string& ks : split(get("--beam-grid", "4"))) {
                tbeam::DecodeConfig c = cfg;
                c.beam = std::atoi(ks.c_str());
                const int bb = std::atoi(bs.c_str());
                tbeam_b200::reference::decode_chunked(fn, all, c, bb);  // warm-up
                double wall = 0.0;
                std::uint64_t frames = 0;
                for (int r = 0; r < repeats; ++r) {
                    const tbeam::DecodeResult res = tbeam_b200::reference::decode_chunked(fn, all, c, bb);
                    wall += res.wall_seconds;
                    frames = res.total_frames();
                }
                wall /= repeats;
                std::printf("{\"algo\": \"%s\", \"batch\": %d, \"beam\": %d, \"frames\": %llu, \"wall\": %.6f, "
                            "\"rtfx\": %.3f}\n",
                            a.c_str(), bb, c.beam, (unsigned long long)frames, wall,
                            static_cast<double>(frames) * spf / wall);
            }
        }
    }
    return 0;
}
