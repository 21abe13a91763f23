// ARPA text -> device-ready n-gram trie (host side of the LM upload).
//
// Two passes, neither of which grows a pointer trie:
//
//   1. scan   -- a cursor over the text's non-blank lines reads the \data\
//               header (the declared count per order) and then every entry
//               into flat arrays: order, mapped token ids, ln-probability,
//               ln-backoff (ARPA log10 x ln 10).  Format errors are reported as
//               TBEAM_PARSE with "lm.arpa:<line>: <what>".
//   2. freeze -- level by level, the distinct l-token prefixes of all entries
//               of order >= l are sorted by (node id of their (l-1)-prefix,
//               l-th token).  Node ids are handed out in that order, so
//                 * node 0 is the root, then all depth-1 nodes, depth-2, ...;
//                 * the children of a node are a contiguous id range, sorted by
//                   token -- the CSR child list IS the node order (edge e is
//                   node e + 1), no per-node sort;
//               probabilities and backoffs are then assigned in file order (a
//               repeated n-gram overwrites its probability; its backoff only
//               when the repeat carries one), and each node's suffix link is
//               its longest proper suffix that is a node, found by descending
//               from the root (the Aho-Corasick failure link of a
//               prefix-closed trie).
//
// Query-visible semantics (what the device functions in device_fns.cuh read)
// follow the reference's NGramLm (proj/src/ngram_lm.cpp:52-318,
// ngram_lm.hpp:24-117); node NUMBERING differs, which no query observes:
//   * internal token space: ASR ids 0..V-1, then <s> = V, </s> = V+1,
//     <unk> = V+2 ("<unk>" or "<UNK>"); OOV words map to <unk> and are counted
//     unless strict, in which case they are a parse error;
//   * implicit context nodes (prefixes never listed) carry a NaN probability;
//   * token_remap: ASR id -> itself if it has a unigram, else <unk> when <unk>
//     has one, else -1;
//   * initial state: the <s> node, or its suffix when <s> is a full-order node.
// Behavioural contract pinned by tests/test_abi.py (reference parity of node
// counts on the reference's own generator, and the error classes of malformed
// inputs).
#include "lm_build.h"

#include <algorithm>
#include <cerrno>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string_view>
#include <unordered_map>

namespace tbeam_host {

namespace {

constexpr double kLn10 = 2.302585092994045684;
constexpr int kParse = 3;  // TBEAM_PARSE

// ---- number parsing with std::sto* acceptance rules ------------------------
// leading whitespace and trailing text are accepted; no digits or a value out
// of range is an error
bool to_int(std::string_view s, long& out) {
    const std::string t(s);
    char* end = nullptr;
    errno = 0;
    const long v = std::strtol(t.c_str(), &end, 10);
    if (end == t.c_str() || errno == ERANGE || v < INT_MIN || v > INT_MAX) return false;
    out = v;
    return true;
}
bool to_count(std::string_view s, unsigned long& out) {
    const std::string t(s);
    char* end = nullptr;
    errno = 0;
    const unsigned long v = std::strtoul(t.c_str(), &end, 10);
    if (end == t.c_str() || errno == ERANGE) return false;
    out = v;
    return true;
}
bool to_real(std::string_view s, double& out) {
    const std::string t(s);
    char* end = nullptr;
    errno = 0;
    const double v = std::strtod(t.c_str(), &end);
    if (end == t.c_str() || errno == ERANGE) return false;
    out = v;
    return true;
}

// fields are separated by any C-locale whitespace (operator>> semantics); a
// line counts as blank when it holds only spaces, tabs and carriage returns
inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// ---- pass 1: scan ----------------------------------------------------------
class ArpaScan {
   public:
    ArpaScan(const char* text, std::size_t len, const std::vector<std::string>& vocab, bool strict)
        : text_(text), len_(len), strict_(strict), V_(static_cast<int>(vocab.size())) {
        ids_.reserve(vocab.size() * 2);
        for (int i = 0; i < V_; ++i) ids_.emplace(vocab[i], i);
    }

    // flat entry arrays (entry n: order ord[n], tokens tok[first[n] .. first[n] + ord[n]))
    std::vector<int> ord, first, tok;
    std::vector<double> lnp, lnb;
    std::vector<unsigned char> has_b;
    std::vector<unsigned long> declared;
    std::size_t oov = 0;
    std::string err;

    int run() {
        std::string_view ln;
        // preamble: everything up to the \data\ line is ignored
        bool saw_data = false;
        while (next(ln)) {
            if (ln == "\\data\\") {
                saw_data = true;
                break;
            }
        }
        if (!saw_data) return fail("no \\data\\ line in the ARPA text");
        // header: "ngram k=count" lines, orders 1, 2, ... in sequence
        bool have = next(ln);
        while (have) {
            if (ln == "\\end\\") return finish_at_end(0);
            if (ln.substr(0, 6) != "ngram ") break;
            const std::size_t eq = ln.find('=');
            long k = 0;
            unsigned long c = 0;
            if (eq == std::string_view::npos || !to_int(ln.substr(6, eq - 6), k) || !to_count(ln.substr(eq + 1), c))
                return fail("cannot read the n-gram count line");
            if (k != static_cast<long>(declared.size()) + 1)
                return fail("n-gram count for order " + std::to_string(k) + " out of sequence (expected order " +
                            std::to_string(declared.size() + 1) + ")");
            declared.push_back(c);
            have = next(ln);
        }
        // body: "\k-grams:" sections of entries, closed by \end\ .
        int order = 0;
        std::size_t in_section = 0;
        for (; have; have = next(ln)) {
            if (ln == "\\end\\") {
                if (order > 0 && in_section != declared[order - 1]) return count_mismatch(order, in_section);
                return finish_at_end(order);
            }
            const std::size_t tag = ln.find("-grams:");
            if (ln.size() >= 2 && ln[0] == '\\' && tag != std::string_view::npos) {
                if (order > 0 && in_section != declared[order - 1]) return count_mismatch(order, in_section);
                long k = 0;
                if (!to_int(ln.substr(1, tag - 1), k)) return fail("cannot read the section header");
                if (k != order + 1 || k > static_cast<long>(declared.size()))
                    return fail("section " + std::string(ln) + " out of sequence");
                order = static_cast<int>(k);
                in_section = 0;
                continue;
            }
            if (order == 0) return fail("n-gram entry outside a \\k-grams: section");
            if (int rc = entry(ln, order)) return rc;
            ++in_section;
        }
        return fail("the ARPA text ends without an \\end\\ line");
    }

   private:
    const char* text_;
    std::size_t len_;
    std::size_t pos_ = 0;
    std::size_t line_ = 0;
    bool strict_;
    int V_;
    std::unordered_map<std::string, int> ids_;
    std::vector<std::string_view> fld_;

    int fail(const std::string& what) {
        err = "lm.arpa:" + std::to_string(line_) + ": " + what;
        return kParse;
    }
    int count_mismatch(int order, std::size_t n) {
        return fail("order " + std::to_string(order) + " lists " + std::to_string(n) + " n-grams but \\data\\ declares " +
                    std::to_string(declared[order - 1]));
    }
    int finish_at_end(int order) {
        if (order != static_cast<int>(declared.size()))
            return fail("\\end\\ reached before every declared order had its section");
        if (declared.empty()) {
            line_ = 0;
            return fail("the \\data\\ header declares no n-gram orders");
        }
        return 0;
    }
    // next non-blank line (trailing CR dropped); false at the end of the text
    bool next(std::string_view& out) {
        while (pos_ < len_) {
            const char* p = text_ + pos_;
            const void* nl = std::memchr(p, '\n', len_ - pos_);
            const std::size_t n = nl ? static_cast<std::size_t>(static_cast<const char*>(nl) - p) : len_ - pos_;
            pos_ += n + 1;
            ++line_;
            std::string_view l(p, n);
            if (!l.empty() && l.back() == '\r') l.remove_suffix(1);
            bool blank = true;
            for (char c : l) blank &= (c == ' ' || c == '\t' || c == '\r');
            if (!blank) {
                out = l;
                return true;
            }
        }
        return false;
    }
    int map_word(std::string_view w, int& id) {
        if (w == "<s>") id = V_;
        else if (w == "</s>") id = V_ + 1;
        else if (w == "<unk>" || w == "<UNK>") id = V_ + 2;
        else {
            const auto it = ids_.find(std::string(w));
            if (it != ids_.end()) {
                id = it->second;
            } else {
                if (strict_) return fail("word '" + std::string(w) + "' is not in the vocabulary");
                ++oov;
                id = V_ + 2;
            }
        }
        return 0;
    }
    int entry(std::string_view l, int order) {
        fld_.clear();
        std::size_t i = 0;
        while (i < l.size()) {
            while (i < l.size() && is_ws(l[i])) ++i;
            const std::size_t b = i;
            while (i < l.size() && !is_ws(l[i])) ++i;
            if (i > b) fld_.push_back(l.substr(b, i - b));
        }
        const std::size_t k = static_cast<std::size_t>(order);
        if (fld_.size() != k + 1 && fld_.size() != k + 2)
            return fail(std::to_string(order) + "-gram entry has " + std::to_string(fld_.size()) +
                        " fields (want " + std::to_string(k + 1) + " or " + std::to_string(k + 2) + ")");
        const bool hb = fld_.size() == k + 2;
        double p = 0.0, b = 0.0;
        if (!to_real(fld_[0], p) || (hb && !to_real(fld_[k + 1], b))) return fail("cannot read a log10 value");
        ord.push_back(order);
        first.push_back(static_cast<int>(tok.size()));
        for (std::size_t q = 0; q < k; ++q) {
            int id = 0;
            if (int rc = map_word(fld_[1 + q], id)) return rc;
            tok.push_back(id);
        }
        lnp.push_back(p * kLn10);
        lnb.push_back(hb ? b * kLn10 : 0.0);
        has_b.push_back(hb ? 1 : 0);
        return 0;
    }
};

}  // namespace

int build_lm(const char* text, std::size_t len, const std::vector<std::string>& vocab, bool strict,
             HostLm& lm, std::string& err) {
    lm = HostLm{};
    ArpaScan sc(text, len, vocab, strict);
    if (const int rc = sc.run()) {
        err = sc.err;
        return rc;
    }
    const int V = static_cast<int>(vocab.size());
    const int N = static_cast<int>(sc.declared.size());
    const std::size_t E = sc.ord.size();
    lm.V = V;
    lm.order = N;
    lm.oov_mapped = sc.oov;

    // ---- pass 2: level-sorted node ids --------------------------------------
    // at[n] = id of entry n's node at the current level (its l-prefix)
    std::vector<int> at(E, 0);
    std::vector<int> parent(1, -1), token(1, -1), depth(1, 0);
    std::vector<int> items(E);
    for (std::size_t n = 0; n < E; ++n) items[n] = static_cast<int>(n);
    std::vector<std::pair<unsigned long long, int>> keyed;
    for (int l = 1; l <= N; ++l) {
        // entries reaching this level, keyed (parent id, l-th token)
        std::size_t m = 0;
        for (std::size_t q = 0; q < items.size(); ++q)
            if (sc.ord[items[q]] >= l) items[m++] = items[q];
        items.resize(m);
        keyed.resize(m);
        for (std::size_t q = 0; q < m; ++q) {
            const int n = items[q];
            const unsigned tk = static_cast<unsigned>(sc.tok[sc.first[n] + l - 1]);
            keyed[q] = {static_cast<unsigned long long>(static_cast<unsigned>(at[n])) << 32 | tk, n};
        }
        std::sort(keyed.begin(), keyed.end());
        unsigned long long prev = ~0ull;
        for (std::size_t q = 0; q < m; ++q) {
            if (keyed[q].first != prev) {
                prev = keyed[q].first;
                parent.push_back(static_cast<int>(prev >> 32));
                token.push_back(static_cast<int>(prev & 0xffffffffu));
                depth.push_back(l);
            }
            at[keyed[q].second] = static_cast<int>(parent.size()) - 1;
        }
    }
    const std::size_t n_nodes = parent.size();
    // probabilities / backoffs in file order: the last listing wins
    lm.prob.assign(n_nodes, std::numeric_limits<double>::quiet_NaN());
    lm.backoff.assign(n_nodes, 0.0);
    for (std::size_t n = 0; n < E; ++n) {
        lm.prob[at[n]] = sc.lnp[n];
        if (sc.has_b[n]) lm.backoff[at[n]] = sc.lnb[n];
    }
    // CSR: edge e = node e + 1 (children contiguous, sorted by token)
    lm.depth = depth;
    lm.etok.assign(token.begin() + 1, token.end());
    lm.enode.resize(n_nodes - 1);
    for (std::size_t e = 0; e + 1 < n_nodes; ++e) lm.enode[e] = static_cast<int>(e + 1);
    lm.cbeg.assign(n_nodes, 0);
    lm.cend.assign(n_nodes, 0);
    // nodes are grouped by parent in id order: scan the run of each parent
    {
        std::size_t c = 1;
        for (std::size_t x = 0; x < n_nodes; ++x) {
            while (c < n_nodes && parent[c] < static_cast<int>(x)) ++c;
            lm.cbeg[x] = static_cast<int>(c - 1);
            while (c < n_nodes && parent[c] == static_cast<int>(x)) ++c;
            lm.cend[x] = static_cast<int>(c - 1);
        }
    }
    auto child = [&](int node, int tk) -> int {
        const auto b = lm.etok.begin() + lm.cbeg[node], e = lm.etok.begin() + lm.cend[node];
        const auto it = std::lower_bound(b, e, tk);
        return (it == e || *it != tk) ? -1 : static_cast<int>(it - lm.etok.begin()) + 1;
    };
    // suffix link: the longest proper suffix of the node's word sequence that
    // is itself a node (depth-1 nodes and the root: the root)
    lm.suffix.assign(n_nodes, 0);
    std::vector<int> seq(static_cast<std::size_t>(N) + 1);
    for (std::size_t x = 1; x < n_nodes; ++x) {
        const int d = depth[x];
        if (d < 2) continue;
        for (int y = static_cast<int>(x), q = d - 1; q >= 0; y = parent[y], --q) seq[q] = token[y];
        for (int j = 1; j < d; ++j) {  // drop j leading words
            int y = 0;
            for (int q = j; q < d && y >= 0; ++q) y = child(y, seq[q]);
            if (y >= 0) {
                lm.suffix[x] = y;
                break;
            }
        }
    }
    // root-level tables the device queries read
    const int unk = V + 2, bos = V;
    const int unk_node = child(0, unk);
    const bool has_unk = unk_node >= 0 && !std::isnan(lm.prob[unk_node]);
    lm.unk_prob = has_unk ? lm.prob[unk_node] : -std::numeric_limits<double>::infinity();
    lm.remap.assign(V, -1);
    lm.uni.assign(V, std::numeric_limits<float>::quiet_NaN());
    for (int k = 0; k < V; ++k) {
        const int c = child(0, k);
        if (c >= 0 && !std::isnan(lm.prob[c])) {
            lm.remap[k] = k;
            lm.uni[k] = static_cast<float>(lm.prob[c]);
        } else if (has_unk) {
            lm.remap[k] = unk;
        }
    }
    // dense root level: internal id -> depth-1 node (one load instead of a search)
    int span = 1;
    for (int e = lm.cbeg[0]; e < lm.cend[0]; ++e) span = std::max(span, lm.etok[e] + 1);
    lm.root.assign(static_cast<std::size_t>(span), -1);
    for (int e = lm.cbeg[0]; e < lm.cend[0]; ++e) lm.root[lm.etok[e]] = e + 1;
    const int bos_node = child(0, bos);
    lm.initial = bos_node < 0 ? 0 : (depth[bos_node] == N ? lm.suffix[bos_node] : bos_node);
    return 0;
}

}  // namespace tbeam_host
