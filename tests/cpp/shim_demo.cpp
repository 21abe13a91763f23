// Drop-in demo of include/tbeam_b200.hpp: decode a few streams through the
// reference-shaped C++ API (greedy_batched / alsd_pp / aes_pp) and print the
// model, inputs and results as JSON so tests/test_cpp_shim.py can check them
// against the CPU oracle.
#include <cstdio>
#include <cstdint>
#include <vector>

#include "tbeam_b200.hpp"

namespace {
struct Rng {
    std::uint64_t s;
    double normal() {  // sum of 12 uniforms - 6
        double a = 0;
        for (int i = 0; i < 12; ++i) {
            s += 0x9e3779b97f4a7c15ull;
            std::uint64_t z = s;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            z ^= z >> 31;
            a += static_cast<double>(z >> 11) * 0x1.0p-53;
        }
        return a - 6.0;
    }
};
void dump(const char* name, const std::vector<float>& v, bool last = false) {
    std::printf("\"%s\": [", name);
    for (std::size_t i = 0; i < v.size(); ++i) std::printf(i ? ",%.9g" : "%.9g", v[i]);
    std::printf("]%s\n", last ? "" : ",");
}
}  // namespace

int main() {
    const int V = 20, D = 16, J = 32, B = 3, T = 12;
    Rng rng{42};
    auto fill = [&](std::size_t n, double sd) {
        std::vector<float> v(n);
        for (auto& x : v) x = static_cast<float>(rng.normal() * sd);
        return v;
    };
    std::vector<float> w_enc = fill(J * D, 0.25), b_enc = fill(J, 0.1), table = fill((V + 1) * J, 0.8),
                       b_pred = fill(J, 0.1), w_out = fill((V + 1) * J, 0.5), b_out = fill(V + 1, 0.1);
    b_out[V] += 3.0f;
    std::vector<float> enc = fill(static_cast<std::size_t>(B) * T * D, 1.0);
    tbeam_model_dims dims{};
    dims.vocab_size = V;
    dims.enc_dim = D;
    dims.joint_dim = J;
    dims.pred_kind = TBEAM_PRED_STATELESS;
    dims.context_order = 2;
    dims.precision = TBEAM_PREC_FP32;
    tbeam_model_weights w{};
    w.w_enc = w_enc.data();
    w.b_enc = b_enc.data();
    w.pred_table = table.data();
    w.b_pred = b_pred.data();
    w.w_out = w_out.data();
    w.b_out = b_out.data();

    std::printf("{\n");
    dump("w_enc", w_enc);
    dump("b_enc", b_enc);
    dump("pred_table", table);
    dump("b_pred", b_pred);
    dump("w_out", w_out);
    dump("b_out", b_out);
    dump("enc", enc);
    const int lens[B] = {12, 9, 5};
    std::printf("\"lens\": [12, 9, 5],\n\"results\": {\n");
    try {
        tbeam_b200::Decoder dec(0);
        dec.set_model(dims, w);
        std::vector<tbeam_b200::StreamInput> streams;
        for (int b = 0; b < B; ++b) streams.push_back({enc.data() + static_cast<std::size_t>(b) * T * D, lens[b]});
        tbeam_b200::DecodeConfig cfg;
        cfg.return_nbest = 2;
        cfg.max_len = 20;
        const char* names[3] = {"greedy", "alsd", "aes"};
        for (int a = 0; a < 3; ++a) {
            const tbeam_b200::DecodeResult r =
                a == 0 ? tbeam_b200::greedy_batched(dec, streams, cfg)
                       : a == 1 ? tbeam_b200::alsd_pp(dec, streams, cfg) : tbeam_b200::aes_pp(dec, streams, cfg);
            std::printf("\"%s\": [", names[a]);
            for (int b = 0; b < B; ++b) {
                std::printf(b ? ",[" : "[");
                for (std::size_t q = 0; q < r.streams[b].nbest.size(); ++q) {
                    const auto& n = r.streams[b].nbest[q];
                    std::printf(q ? ",{\"score\": %.17g, \"tokens\": [" : "{\"score\": %.17g, \"tokens\": [", n.score);
                    for (std::size_t i = 0; i < n.tokens.size(); ++i) std::printf(i ? ",%d" : "%d", n.tokens[i]);
                    std::printf("]}");
                }
                std::printf("]");
            }
            std::printf("]%s\n", a < 2 ? "," : "");
        }
        // the reference's error taxonomy survives the boundary
        tbeam_b200::DecodeConfig bad;
        bad.beam = 0;
        bool threw = false;
        try {
            tbeam_b200::alsd_pp(dec, streams, bad);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        std::printf("}, \"invalid_argument_raised\": %s\n}\n", threw ? "true" : "false");
    } catch (const std::exception& e) {
        std::printf("}, \"error\": \"%s\"\n}\n", e.what());
        return 2;
    }
    return 0;
}
