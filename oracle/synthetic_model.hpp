// TEST INFRASTRUCTURE -- oracle only.  Never linked into the product library.
//
// fp64 restatement of the synthetic transducer that the B200 decoder scores
// (joint + stateless or LSTM prediction network + optional TDT duration head;
// the math is documented in include/tbeam_b200.h).  It plays the role of the
// reference's seeded ToyModel (proj/src/model.cpp:305-367): a frame embedding
// (here the projected encoder frame) plus a prediction-network output, a tanh
// hidden layer and a log-softmax over V+1 outcomes with the blank last.
//
// Shared by
//   * oracle/tbeam_oracle.cpp  -- the CPU restatement of the search, and
//   * oracle/ref_shim.cpp      -- an EmissionModel subclass plugged into the
//                                  compiled reference (oracle/_ref), which pins
//                                  the restatement against the reference's own
//                                  alsd_pp / aes_pp / reference_beam / greedy.
//
// matvec / log_softmax are injectable so the shim can run the reference's own
// kernels (tbeam::kernels::active(), kernels.hpp:13-48).  The defaults below
// restate the reference's scalar kernels (scalar.cpp:41-73) operation for
// operation, so with TBEAM_KERNELS=scalar both sides round identically.
//
// bf16 mode: every GEMM operand the GPU feeds to the tensor cores is rounded
// to bf16 here as well (encoder frame + W_enc, LSTM h + W_hh, h' + W_pred,
// joint z + W_out / W_dur); accumulation stays fp64.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "tbeam_b200.h"

namespace oracle {

using MatvecFn = void (*)(const double* w, const double* x, const double* bias,
                          double* out, std::size_t m, std::size_t n);
using LogSoftmaxFn = void (*)(double* x, std::size_t n);

// scalar.cpp:63-73
inline void matvec_scalar(const double* w, const double* x, const double* bias,
                          double* out, std::size_t m, std::size_t n) {
    for (std::size_t r = 0; r < m; ++r) {
        const double* row = w + r * n;
        double acc = 0.0;
        for (std::size_t i = 0; i < n; ++i) acc += row[i] * x[i];
        out[r] = acc + bias[r];
    }
}

// scalar.cpp:41-61
inline void log_softmax_scalar(double* x, std::size_t n) {
    double m = -std::numeric_limits<double>::infinity();
    for (std::size_t i = 0; i < n; ++i) m = std::max(m, x[i]);
    double lz = m;
    if (std::isfinite(m)) {
        double sum = 0.0;
        for (std::size_t i = 0; i < n; ++i) sum += std::exp(x[i] - m);
        lz = m + std::log(sum);
    }
    for (std::size_t i = 0; i < n; ++i) x[i] -= lz;
}

// fp64 -> fp32 -> bf16 (round to nearest even), the rounding path the GPU
// takes (its values are fp32 before the operand conversion).
inline double round_bf16(double x) {
    float f = static_cast<float>(x);
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return x;  // inf / nan
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    std::memcpy(&f, &u, 4);
    return static_cast<double>(f);
}

struct LstmState {
    std::vector<double> h, c, pred;  // [H], [H], [J]
};

class SyntheticModel {
public:
    SyntheticModel(const tbeam_model_dims& d, const tbeam_model_weights& w,
                   MatvecFn mv = matvec_scalar, LogSoftmaxFn ls = log_softmax_scalar)
        : dims(d), matvec(mv), log_softmax(ls) {
        V = d.vocab_size;
        D = d.enc_dim;
        J = d.joint_dim;
        n = d.context_order;
        H = d.lstm_hidden;
        E = d.emb_dim;
        ND = d.num_durations;
        lstm = d.pred_kind == TBEAM_PRED_LSTM;
        bf16 = d.precision == TBEAM_PREC_BF16;
        if (V < 1 || D < 1 || J < 1 || ND < 0 || ND > TBEAM_MAX_DURATIONS ||
            (!lstm && n < 0) || (lstm && (H < 1 || E < 1)))
            throw std::invalid_argument("SyntheticModel: bad dims");
        const auto cp = [&](const float* src, std::size_t cnt, bool round) {
            if (src == nullptr) throw std::invalid_argument("SyntheticModel: missing weight");
            std::vector<double> v(cnt);
            for (std::size_t i = 0; i < cnt; ++i)
                v[i] = round ? round_bf16(src[i]) : static_cast<double>(src[i]);
            return v;
        };
        const std::size_t R = static_cast<std::size_t>(V) + 1;
        w_enc = cp(w.w_enc, static_cast<std::size_t>(J) * D, bf16);
        b_enc = cp(w.b_enc, J, false);
        b_pred = cp(w.b_pred, J, false);
        w_out = cp(w.w_out, R * J, bf16);
        b_out = cp(w.b_out, R, false);
        if (ND > 0) {
            w_dur = cp(w.w_dur, static_cast<std::size_t>(ND) * J, bf16);
            b_dur = cp(w.b_dur, ND, false);
        }
        if (lstm) {
            emb = cp(w.emb, R * E, false);
            w_ih = cp(w.w_ih, 4ull * H * E, false);
            b_l = cp(w.b_lstm, 4ull * H, false);
            w_hh = cp(w.w_hh, 4ull * H * H, bf16);
            w_pred = cp(w.w_pred, static_cast<std::size_t>(J) * H, bf16);
            // X[v] = W_ih . emb[v] + b : the input half of every LSTM step is a
            // table lookup (the GPU keeps the same table in fp32).  Rows are
            // filled on first use (thread-safe): at V = 8192 the full table
            // is 13 G multiply-adds, most of them for tokens never emitted.
            xtab.resize(R * 4 * H);
            xdone = std::make_unique<std::once_flag[]>(R);
        } else {
            table = cp(w.pred_table, R * J, false);
        }
    }

    // enc_proj = W_enc . frame + b_enc  (frame: D fp32 values)
    void enc_proj(const float* frame, double* out) const {
        std::vector<double> x(D);
        for (int i = 0; i < D; ++i) x[i] = bf16 ? round_bf16(frame[i]) : frame[i];
        matvec(w_enc.data(), x.data(), b_enc.data(), out, J, D);
    }

    // stateless: pred = b_pred + (1/n) sum table[w]   (BOS kNoToken -> row V)
    void stateless_pred(const std::int32_t* window, double* out) const {
        for (int j = 0; j < J; ++j) out[j] = 0.0;
        if (n > 0) {
            const double inv = 1.0 / n;
            for (int i = 0; i < n; ++i) {
                const int row = window[i] < 0 ? V : window[i];
                const double* tr = table.data() + static_cast<std::size_t>(row) * J;
                for (int j = 0; j < J; ++j) out[j] += inv * tr[j];
            }
        }
        for (int j = 0; j < J; ++j) out[j] = b_pred[j] + out[j];
    }

    LstmState lstm_start() const {
        LstmState s;
        s.h.assign(H, 0.0);
        s.c.assign(H, 0.0);
        return lstm_step(s, V);
    }

    LstmState lstm_step(const LstmState& s, int tok) const {
        std::vector<double> hin(H), gates(4ull * H);
        for (int i = 0; i < H; ++i) hin[i] = bf16 ? round_bf16(s.h[i]) : s.h[i];
        const double* x = xrow(tok);
        matvec(w_hh.data(), hin.data(), x, gates.data(), 4ull * H, H);
        LstmState o;
        o.h.resize(H);
        o.c.resize(H);
        for (int u = 0; u < H; ++u) {
            const double ig = sigmoid(gates[u]);
            const double fg = sigmoid(gates[H + u]);
            const double gg = std::tanh(gates[2 * H + u]);
            const double og = sigmoid(gates[3 * H + u]);
            o.c[u] = fg * s.c[u] + ig * gg;
            o.h[u] = og * std::tanh(o.c[u]);
        }
        std::vector<double> hq(H);
        for (int i = 0; i < H; ++i) hq[i] = bf16 ? round_bf16(o.h[i]) : o.h[i];
        o.pred.resize(J);
        matvec(w_pred.data(), hq.data(), b_pred.data(), o.pred.data(), J, H);
        return o;
    }

    // Normalised log-prob rows: tok_out[V+1] (blank last), dur_out[ND].
    void joint(const double* encp, const double* pred, double* tok_out,
               double* dur_out) const {
        std::vector<double> z(J);
        for (int j = 0; j < J; ++j) {
            const double v = std::tanh(encp[j] + pred[j]);
            z[j] = bf16 ? round_bf16(v) : v;
        }
        matvec(w_out.data(), z.data(), b_out.data(), tok_out, V + 1, J);
        log_softmax(tok_out, V + 1);
        if (ND > 0 && dur_out != nullptr) {
            matvec(w_dur.data(), z.data(), b_dur.data(), dur_out, ND, J);
            log_softmax(dur_out, ND);
        }
    }

    // joint() for `cnt` (pred) rows that share one projected frame, with one
    // pass over W_out / W_dur for all of them.  Per output element the
    // arithmetic is matvec_scalar's exactly (acc = 0; acc += w[i]*z[i] in
    // order i = 0..J-1; + bias), only interleaved across rows, so each row
    // is bit-identical to joint() with the default kernels.  This is what
    // lets the oracle check the large BASELINE shapes (V = 8192) in seconds
    // per stream instead of minutes.
    void joint_many(const double* encp, const double* const* preds, int cnt, double* tok_out,
                    std::size_t tok_stride, double* dur_out, std::size_t dur_stride) const {
        if (cnt < 1) return;
        if (matvec != matvec_scalar) {  // injected kernels: row by row
            for (int q = 0; q < cnt; ++q)
                joint(encp, preds[q], tok_out + static_cast<std::size_t>(q) * tok_stride,
                      dur_out ? dur_out + static_cast<std::size_t>(q) * dur_stride : nullptr);
            return;
        }
        std::vector<double> z(static_cast<std::size_t>(cnt) * J);
        std::vector<const double*> zp(cnt), bo(cnt, b_out.data()), bd(cnt, b_dur.data());
        for (int q = 0; q < cnt; ++q) {
            for (int j = 0; j < J; ++j) {
                const double v = std::tanh(encp[j] + preds[q][j]);
                z[static_cast<std::size_t>(q) * J + j] = bf16 ? round_bf16(v) : v;
            }
            zp[q] = &z[static_cast<std::size_t>(q) * J];
        }
        gemv_many(w_out.data(), V + 1, J, zp.data(), bo.data(), cnt, tok_out, tok_stride);
        for (int q = 0; q < cnt; ++q) log_softmax(tok_out + static_cast<std::size_t>(q) * tok_stride, V + 1);
        if (ND > 0 && dur_out != nullptr) {
            gemv_many(w_dur.data(), ND, J, zp.data(), bd.data(), cnt, dur_out, dur_stride);
            for (int q = 0; q < cnt; ++q) log_softmax(dur_out + static_cast<std::size_t>(q) * dur_stride, ND);
        }
    }

    // lstm_step() for `cnt` (state, token) pairs, the W_hh / W_pred passes
    // shared; bit-identical to lstm_step() per pair (gemv_many).
    std::vector<LstmState> lstm_step_many(const LstmState* const* s, const int* tok, int cnt) const {
        std::vector<LstmState> o(cnt);
        if (cnt < 1) return o;
        if (matvec != matvec_scalar) {
            for (int q = 0; q < cnt; ++q) o[q] = lstm_step(*s[q], tok[q]);
            return o;
        }
        std::vector<double> hin(static_cast<std::size_t>(cnt) * H), gates(static_cast<std::size_t>(cnt) * 4 * H);
        std::vector<const double*> hp(cnt), xb(cnt), bp(cnt, b_pred.data());
        for (int q = 0; q < cnt; ++q) {
            for (int i = 0; i < H; ++i) hin[static_cast<std::size_t>(q) * H + i] = bf16 ? round_bf16(s[q]->h[i]) : s[q]->h[i];
            hp[q] = &hin[static_cast<std::size_t>(q) * H];
            xb[q] = xrow(tok[q]);
        }
        gemv_many(w_hh.data(), 4 * H, H, hp.data(), xb.data(), cnt, gates.data(), 4ull * H);
        std::vector<double> hq(static_cast<std::size_t>(cnt) * H);
        for (int q = 0; q < cnt; ++q) {
            const double* g = &gates[static_cast<std::size_t>(q) * 4 * H];
            o[q].h.resize(H);
            o[q].c.resize(H);
            for (int u = 0; u < H; ++u) {
                const double ig = sigmoid(g[u]);
                const double fg = sigmoid(g[H + u]);
                const double gg = std::tanh(g[2 * H + u]);
                const double og = sigmoid(g[3 * H + u]);
                o[q].c[u] = fg * s[q]->c[u] + ig * gg;
                o[q].h[u] = og * std::tanh(o[q].c[u]);
                hq[static_cast<std::size_t>(q) * H + u] = bf16 ? round_bf16(o[q].h[u]) : o[q].h[u];
            }
            hp[q] = &hq[static_cast<std::size_t>(q) * H];
            o[q].pred.resize(J);
        }
        std::vector<double> pred(static_cast<std::size_t>(cnt) * J);
        gemv_many(w_pred.data(), J, H, hp.data(), bp.data(), cnt, pred.data(), J);
        for (int q = 0; q < cnt; ++q)
            std::copy(&pred[static_cast<std::size_t>(q) * J], &pred[static_cast<std::size_t>(q) * J] + J,
                      o[q].pred.begin());
        return o;
    }

    // out_q[r] = (sum_i w[r][i] * x_q[i]) + bias_q[r] for q < cnt: the
    // per-element operation sequence of matvec_scalar, interleaved over q
    // (eight independent accumulators) so each weight row is read once.
    static void gemv_many(const double* w, int rows, int n, const double* const* x,
                          const double* const* bias, int cnt, double* out, std::size_t stride) {
        constexpr int L = 8;
        const int nb = (cnt + L - 1) / L;
        std::vector<double> xt(static_cast<std::size_t>(n) * nb * L, 0.0);  // [n][nb*L]
        for (int q = 0; q < cnt; ++q)
            for (int i = 0; i < n; ++i) xt[static_cast<std::size_t>(i) * nb * L + q] = x[q][i];
        typedef double v4 __attribute__((vector_size(32)));
        constexpr int RB = 4;  // weight rows per pass (independent accumulator chains)
        for (int r0 = 0; r0 < rows; r0 += RB) {
            const int nr = std::min(RB, rows - r0);
            const double* wr[RB];
            for (int k = 0; k < RB; ++k) wr[k] = w + static_cast<std::size_t>(r0 + std::min(k, nr - 1)) * n;
            for (int g = 0; g < nb; ++g) {
                v4 a[RB][2];
                for (int k = 0; k < RB; ++k) a[k][0] = a[k][1] = v4{0.0, 0.0, 0.0, 0.0};
                const double* xc = xt.data() + g * L;
                for (int i = 0; i < n; ++i) {
                    v4 x0, x1;
                    std::memcpy(&x0, xc + static_cast<std::size_t>(i) * nb * L, sizeof x0);
                    std::memcpy(&x1, xc + static_cast<std::size_t>(i) * nb * L + 4, sizeof x1);
                    for (int k = 0; k < RB; ++k) {
                        const double wi = wr[k][i];
                        const v4 wv = {wi, wi, wi, wi};
                        a[k][0] += wv * x0;  // separate mul and add (-ffp-contract=off)
                        a[k][1] += wv * x1;
                    }
                }
                for (int k = 0; k < nr; ++k) {
                    double acc[L];
                    std::memcpy(acc, &a[k][0], sizeof(v4));
                    std::memcpy(acc + 4, &a[k][1], sizeof(v4));
                    const int r = r0 + k;
                    for (int l = 0; l < L && g * L + l < cnt; ++l)
                        out[static_cast<std::size_t>(g * L + l) * stride + r] = acc[l] + bias[g * L + l][r];
                }
            }
        }
    }

    static double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

    tbeam_model_dims dims;
    int V = 0, D = 0, J = 0, n = 0, H = 0, E = 0, ND = 0;
    bool lstm = false, bf16 = false;
    MatvecFn matvec;
    LogSoftmaxFn log_softmax;
    const double* xrow(int tok) const {
        double* x = xtab.data() + static_cast<std::size_t>(tok) * 4 * H;
        std::call_once(xdone[tok], [&] {
            matvec_scalar(w_ih.data(), emb.data() + static_cast<std::size_t>(tok) * E, b_l.data(), x,
                          4ull * H, E);
        });
        return x;
    }

    mutable std::vector<double> xtab;
    std::unique_ptr<std::once_flag[]> xdone;
    std::vector<double> emb, w_ih, b_l;
    std::vector<double> w_enc, b_enc, table, b_pred, w_hh, w_pred, w_out, b_out,
        w_dur, b_dur;
};

}  // namespace oracle
