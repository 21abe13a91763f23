// TEST INFRASTRUCTURE -- oracle only.  Never linked into the product library.
//
// Map-based restatement of the reference's ARPA n-gram LM
// (proj/src/ngram_lm.cpp).  Where the reference freezes a trie with CSR
// children and suffix links, this keeps every context as an explicit token
// sequence in an ordered map, so it is an independent second implementation
// of the same semantics:
//   parse          ngram_lm.cpp:52-226  (log10 -> ln, OOV -> <unk>, last entry wins)
//   token remap    ngram_lm.cpp:299-309
//   initial state  ngram_lm.cpp:311-316
//   score_internal ngram_lm.cpp:330-344   (backoff walk, floor -1e9)
//   score_token    ngram_lm.cpp:346-356
//   score_eos      ngram_lm.cpp:358-361
//   score_vocab    ngram_lm.cpp:363-416   (stamped chain walk + <unk> fill)
//   advance        ngram_lm.cpp:418-438   (longest suffix; full order -> suffix)
// A state is the context token sequence (internal ids), i.e. the trie node.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace oracle {

constexpr double kLogZeroFloor = -1e9;  // types.hpp:27

class OracleLm {
public:
    using Ctx = std::vector<std::int32_t>;

    OracleLm(const std::string& text, const std::vector<std::string>& vocab) {
        V_ = static_cast<int>(vocab.size());
        std::unordered_map<std::string, std::int32_t> index;
        for (int i = 0; i < V_; ++i) index.emplace(vocab[i], i);
        nodes_[Ctx{}] = Node{};  // root
        std::istringstream in(text);
        std::string line;
        bool in_data = false;
        int order = 0, declared = 0;
        while (std::getline(in, line)) {
            if (!line.empty() && line.back() == '\r') line.pop_back();
            if (line.find_first_not_of(" \t") == std::string::npos) continue;
            if (line == "\\data\\") { in_data = true; continue; }
            if (!in_data) continue;
            if (line == "\\end\\") break;
            if (line.rfind("ngram ", 0) == 0) { ++declared; continue; }
            if (line.front() == '\\' && line.find("-grams:") != std::string::npos) {
                order = std::stoi(line.substr(1, line.find("-grams:") - 1));
                continue;
            }
            std::istringstream f(line);
            std::vector<std::string> fields;
            std::string w;
            while (f >> w) fields.push_back(w);
            const double logp = std::stod(fields[0]) * M_LN10;
            const bool has_bo = static_cast<int>(fields.size()) == order + 2;
            Ctx key;
            for (int i = 0; i < order; ++i) {
                const std::string& word = fields[1 + i];
                std::int32_t id;
                if (word == "<s>") id = bos();
                else if (word == "</s>") id = eos();
                else if (word == "<unk>" || word == "<UNK>") id = unk();
                else {
                    auto it = index.find(word);
                    id = it == index.end() ? unk() : it->second;
                }
                key.push_back(id);
                if (!nodes_.count(key)) nodes_[key] = Node{};  // implicit prefix
            }
            Node& nd = nodes_[key];
            nd.prob = logp;
            if (has_bo) nd.backoff = std::stod(fields[order + 1]) * M_LN10;
        }
        order_ = declared;
        const Node* un = find({unk()});
        has_unk_ = un != nullptr && !std::isnan(un->prob);
        unk_prob_ = has_unk_ ? un->prob : -std::numeric_limits<double>::infinity();
        remap_.assign(V_, -1);
        for (int k = 0; k < V_; ++k) {
            const Node* c = find({k});
            if (c != nullptr && !std::isnan(c->prob)) remap_[k] = k;
            else if (has_unk_) remap_[k] = unk();
        }
        // child lists per context, so a vocabulary row visits only the
        // n-grams that exist (V = 8192 rows stay cheap)
        for (const auto& kv : nodes_)
            if (!kv.first.empty() && kv.first.back() < V_)
                children_[Ctx(kv.first.begin(), kv.first.end() - 1)].emplace_back(kv.first.back(), &kv.second);
        initial_ = Ctx{};
        if (find({bos()}) != nullptr)
            initial_ = order_ == 1 ? longest_proper_suffix({bos()}) : Ctx{bos()};
    }

    int order() const { return order_; }
    const Ctx& initial_state() const { return initial_; }

    double score_token(const Ctx& s, int tok) const {
        const std::int32_t it = remap_.at(tok);
        if (it < 0) return kLogZeroFloor;
        return score_internal(s, it);
    }
    double score_eos(const Ctx& s) const { return score_internal(s, eos()); }

    void score_vocab(const Ctx& s, double* out) const {
        std::vector<char> done(V_, 0);
        double acc = 0.0;
        const auto chain = suffix_chain(s);
        for (std::size_t li = 0; li < chain.size(); ++li) {
            const Ctx& c = chain[li];
            const auto ch = children_.find(c);
            if (ch != children_.end())
                for (const auto& [k, nd] : ch->second) {
                    if (done[k] || std::isnan(nd->prob)) continue;
                    out[k] = std::max(acc + nd->prob, kLogZeroFloor);
                    done[k] = 1;
                }
            if (c.empty()) break;
            acc += find(c)->backoff;
        }
        for (int k = 0; k < V_; ++k)
            if (!done[k])
                out[k] = std::isfinite(unk_prob_) ? std::max(acc + unk_prob_, kLogZeroFloor)
                                                  : kLogZeroFloor;
    }

    Ctx advance(const Ctx& s, int tok) const {
        const std::int32_t it = remap_.at(tok);
        if (it < 0) return Ctx{};
        for (const Ctx& c : suffix_chain(s)) {
            Ctx key = c;
            key.push_back(it);
            if (find(key) != nullptr)
                return static_cast<int>(key.size()) == order_ ? longest_proper_suffix(key)
                                                              : key;
        }
        return Ctx{};
    }

private:
    struct Node {
        double prob = std::numeric_limits<double>::quiet_NaN();
        double backoff = 0.0;
    };

    std::int32_t bos() const { return V_; }
    std::int32_t eos() const { return V_ + 1; }
    std::int32_t unk() const { return V_ + 2; }

    const Node* find(const Ctx& k) const {
        auto it = nodes_.find(k);
        return it == nodes_.end() ? nullptr : &it->second;
    }

    // every suffix of s present as a context, longest first, ending at root
    std::vector<Ctx> suffix_chain(const Ctx& s) const {
        std::vector<Ctx> out;
        for (std::size_t i = 0; i <= s.size(); ++i) {
            Ctx suf(s.begin() + i, s.end());
            if (find(suf) != nullptr) out.push_back(std::move(suf));
        }
        return out;
    }

    Ctx longest_proper_suffix(const Ctx& s) const {
        for (std::size_t i = 1; i <= s.size(); ++i) {
            Ctx suf(s.begin() + i, s.end());
            if (find(suf) != nullptr) return suf;
        }
        return Ctx{};
    }

    double score_internal(const Ctx& s, std::int32_t tok) const {
        double acc = 0.0;
        for (const Ctx& c : suffix_chain(s)) {
            Ctx key = c;
            key.push_back(tok);
            const Node* nd = find(key);
            if (nd != nullptr && !std::isnan(nd->prob))
                return std::max(acc + nd->prob, kLogZeroFloor);
            if (c.empty()) return kLogZeroFloor;
            acc += find(c)->backoff;
        }
        return kLogZeroFloor;
    }

    int V_ = 0;
    int order_ = 0;
    bool has_unk_ = false;
    double unk_prob_ = 0.0;
    std::vector<std::int32_t> remap_;
    Ctx initial_;
    std::map<Ctx, Node> nodes_;
    std::map<Ctx, std::vector<std::pair<std::int32_t, const Node*>>> children_;
};

}  // namespace oracle
