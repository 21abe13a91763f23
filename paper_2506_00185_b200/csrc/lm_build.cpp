// ARPA text -> frozen device-ready n-gram trie (host side of the LM upload).
//
// Follows the reference parser's semantics (NGramLm::parse_arpa_text,
// proj/src/ngram_lm.cpp:52-318) so device queries match it:
//   * sections \data\ / ngram k=n / \k-grams: / \end\, orders contiguous,
//     declared counts enforced, 1+k or 2+k fields per entry (ngram_lm.cpp:112-226);
//   * log10 -> ln on load; a repeated n-gram overwrites (last wins);
//   * internal token space: ASR ids 0..V-1, then <s>=V, </s>=V+1, <unk>=V+2;
//     OOV words -> <unk> unless strict (ngram_lm.cpp:77-90);
//   * every n-gram prefix is a node; implicit context nodes carry NaN prob;
//   * children CSR sorted by token; suffix link = longest proper suffix that
//     is a node (ngram_lm.cpp:228-297);
//   * token_remap: ASR id -> itself if it has a unigram, else <unk> if <unk>
//     has a unigram, else -1 (ngram_lm.cpp:299-309);
//   * initial state = <s> node (or its suffix at full order) (ngram_lm.cpp:311-316).
// Plus the dense unigram row the fused late-pruning epilogue reads.
#include "lm_build.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <sstream>
#include <unordered_map>

namespace tbeam_host {

namespace {

struct TmpNode {
    double prob = std::numeric_limits<double>::quiet_NaN();
    double backoff = 0.0;
    int parent = -1;
    int token = -1;
    int depth = 0;
};

bool blank_line(const std::string& s) { return s.find_first_not_of(" \t\r") == std::string::npos; }

std::vector<std::string> fields_of(const std::string& line) {
    std::vector<std::string> out;
    std::istringstream iss(line);
    std::string f;
    while (iss >> f) out.push_back(std::move(f));
    return out;
}

bool parse_double(const std::string& s, double& v) {
    char* end = nullptr;
    v = std::strtod(s.c_str(), &end);
    return end != s.c_str();  // std::stod semantics: trailing text ignored
}

}  // namespace

int build_lm(const char* text, std::size_t len, const std::vector<std::string>& vocab, bool strict,
             HostLm& lm, std::string& err) {
    const std::string src = "lm.arpa";
    auto fail = [&](std::size_t line, const std::string& what) {
        err = src + ":" + std::to_string(line) + ": " + what;
        return 3;  // TBEAM_PARSE
    };
    lm = HostLm{};
    const int V = static_cast<int>(vocab.size());
    lm.V = V;
    const long long space = static_cast<long long>(V) + 3;
    const int bos = V, eos = V + 1, unk = V + 2;
    std::unordered_map<std::string, int> index;
    index.reserve(vocab.size() * 2);
    for (int i = 0; i < V; ++i) index.emplace(vocab[i], i);

    std::vector<TmpNode> tmp(1);
    std::unordered_map<long long, int> child;
    auto ensure_child = [&](int parent, int token) {
        const long long key = static_cast<long long>(parent) * space + token;
        auto it = child.find(key);
        if (it != child.end()) return it->second;
        const int id = static_cast<int>(tmp.size());
        child.emplace(key, id);
        TmpNode nd;
        nd.parent = parent;
        nd.token = token;
        nd.depth = tmp[parent].depth + 1;
        tmp.push_back(nd);
        return id;
    };

    enum { kPre, kData, kGrams, kDone } section = kPre;
    std::vector<std::size_t> declared, seen;
    int cur = 0;
    std::size_t line_no = 0;
    std::string strict_err;
    auto map_word = [&](const std::string& w, int& out) {
        if (w == "<s>") out = bos;
        else if (w == "</s>") out = eos;
        else if (w == "<unk>" || w == "<UNK>") out = unk;
        else {
            auto it = index.find(w);
            if (it != index.end()) out = it->second;
            else {
                if (strict) return false;
                ++lm.oov_mapped;
                out = unk;
            }
        }
        return true;
    };
    auto section_complete = [&](std::size_t at) -> int {
        if (cur == 0) return 0;
        if (seen[cur - 1] != declared[cur - 1]) {
            std::ostringstream o;
            o << "\\" << cur << "-grams: section has " << seen[cur - 1] << " entries, header declared "
              << declared[cur - 1];
            return fail(at, o.str());
        }
        return 0;
    };

    std::size_t pos = 0;
    while (pos <= len) {
        std::size_t nl = pos;
        while (nl < len && text[nl] != '\n') ++nl;
        if (pos == len) break;
        std::string line(text + pos, nl - pos);
        pos = nl + 1;
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (blank_line(line)) continue;
        if (section == kPre) {
            if (line == "\\data\\") section = kData;
            continue;
        }
        if (line == "\\end\\") {
            if (int rc = section_complete(line_no)) return rc;
            if (cur != static_cast<int>(declared.size()))
                return fail(line_no, "missing n-gram sections before \\end\\");
            section = kDone;
            break;
        }
        if (section == kData) {
            if (line.rfind("ngram ", 0) == 0) {
                const auto eq = line.find('=');
                if (eq == std::string::npos) return fail(line_no, "malformed ngram count line");
                char* e1 = nullptr;
                char* e2 = nullptr;
                const std::string ks = line.substr(6, eq - 6), cs = line.substr(eq + 1);
                const long k = std::strtol(ks.c_str(), &e1, 10);
                const unsigned long cnt = std::strtoul(cs.c_str(), &e2, 10);
                if (e1 == ks.c_str() || e2 == cs.c_str()) return fail(line_no, "malformed ngram count line");
                if (k != static_cast<long>(declared.size()) + 1)
                    return fail(line_no, "ngram orders must be contiguous from 1");
                declared.push_back(cnt);
                continue;
            }
            section = kGrams;
            seen.assign(declared.size(), 0);
        }
        // section == kGrams
        if (line.size() >= 2 && line.front() == '\\' && line.find("-grams:") != std::string::npos) {
            if (int rc = section_complete(line_no)) return rc;
            const std::string ks = line.substr(1, line.find("-grams:") - 1);
            char* e1 = nullptr;
            const long k = std::strtol(ks.c_str(), &e1, 10);
            if (e1 == ks.c_str()) return fail(line_no, "malformed section header");
            if (k != cur + 1 || k > static_cast<long>(declared.size()))
                return fail(line_no, "unexpected section " + line + " (orders must be contiguous)");
            cur = static_cast<int>(k);
            continue;
        }
        if (cur == 0) return fail(line_no, "entry before any n-gram section header");
        const auto f = fields_of(line);
        const std::size_t k = static_cast<std::size_t>(cur);
        if (f.size() != k + 1 && f.size() != k + 2) {
            std::ostringstream o;
            o << "\\" << cur << "-grams: expected " << (k + 1) << " or " << (k + 2) << " fields, got "
              << f.size();
            return fail(line_no, o.str());
        }
        double logp = 0.0, bo = 0.0;
        const bool has_bo = f.size() == k + 2;
        if (!parse_double(f[0], logp) || (has_bo && !parse_double(f[k + 1], bo)))
            return fail(line_no, "malformed log probability");
        int ctx = 0;
        int id = 0;
        for (std::size_t i = 0; i + 1 < k; ++i) {
            if (!map_word(f[1 + i], id)) return fail(line_no, "token '" + f[1 + i] + "' not in vocabulary");
            ctx = ensure_child(ctx, id);
        }
        if (!map_word(f[k], id)) return fail(line_no, "token '" + f[k] + "' not in vocabulary");
        const int node = ensure_child(ctx, id);
        tmp[node].prob = logp * M_LN10;
        if (has_bo) tmp[node].backoff = bo * M_LN10;
        ++seen[cur - 1];
    }
    if (section != kDone)
        return fail(line_no, section == kPre ? "no \\data\\ section found" : "missing \\end\\ terminator");
    if (declared.empty()) return fail(0, "ARPA file declares no n-gram orders");
    lm.order = static_cast<int>(declared.size());

    // freeze: CSR children sorted by token
    const std::size_t n = tmp.size();
    lm.prob.resize(n);
    lm.backoff.resize(n);
    lm.depth.resize(n);
    lm.suffix.assign(n, 0);
    lm.cbeg.assign(n, 0);
    lm.cend.assign(n, 0);
    std::vector<int> cnt(n, 0);
    for (std::size_t i = 1; i < n; ++i) ++cnt[tmp[i].parent];
    int off = 0;
    for (std::size_t i = 0; i < n; ++i) {
        lm.cbeg[i] = off;
        lm.cend[i] = off;
        off += cnt[i];
    }
    lm.etok.resize(n > 0 ? n - 1 : 0);
    lm.enode.resize(lm.etok.size());
    for (std::size_t i = 1; i < n; ++i) {
        const int e = lm.cend[tmp[i].parent]++;
        lm.etok[e] = tmp[i].token;
        lm.enode[e] = static_cast<int>(i);
    }
    for (std::size_t i = 0; i < n; ++i) {
        std::vector<std::pair<int, int>> pr;
        for (int e = lm.cbeg[i]; e < lm.cend[i]; ++e) pr.emplace_back(lm.etok[e], lm.enode[e]);
        std::sort(pr.begin(), pr.end());
        for (std::size_t j = 0; j < pr.size(); ++j) {
            lm.etok[lm.cbeg[i] + j] = pr[j].first;
            lm.enode[lm.cbeg[i] + j] = pr[j].second;
        }
        lm.prob[i] = tmp[i].prob;
        lm.backoff[i] = tmp[i].backoff;
        lm.depth[i] = tmp[i].depth;
    }
    auto find_child = [&](int node, int tok) {
        const auto b = lm.etok.begin() + lm.cbeg[node], e = lm.etok.begin() + lm.cend[node];
        const auto it = std::lower_bound(b, e, tok);
        if (it == e || *it != tok) return -1;
        return lm.enode[it - lm.etok.begin()];
    };
    // suffix links in depth order (parents before children)
    std::vector<int> by_depth;
    by_depth.reserve(n);
    for (std::size_t i = 1; i < n; ++i) by_depth.push_back(static_cast<int>(i));
    std::stable_sort(by_depth.begin(), by_depth.end(),
                     [&](int a, int b) { return lm.depth[a] < lm.depth[b]; });
    for (const int node : by_depth) {
        if (lm.depth[node] == 1) {
            lm.suffix[node] = 0;
            continue;
        }
        int s = lm.suffix[tmp[node].parent];
        while (true) {
            const int c = find_child(s, tmp[node].token);
            if (c >= 0) {
                lm.suffix[node] = c;
                break;
            }
            if (s == 0) {
                lm.suffix[node] = 0;
                break;
            }
            s = lm.suffix[s];
        }
    }
    const int unk_node = find_child(0, unk);
    const bool has_unk = unk_node >= 0 && !std::isnan(lm.prob[unk_node]);
    lm.unk_prob = has_unk ? lm.prob[unk_node] : -std::numeric_limits<double>::infinity();
    lm.remap.assign(V, -1);
    lm.uni.assign(V, std::numeric_limits<float>::quiet_NaN());
    for (int k = 0; k < V; ++k) {
        const int c = find_child(0, k);
        if (c >= 0 && !std::isnan(lm.prob[c])) {
            lm.remap[k] = k;
            lm.uni[k] = static_cast<float>(lm.prob[c]);
        } else if (has_unk) {
            lm.remap[k] = unk;
        }
    }
    // dense root level (one load instead of a binary search over |V| children)
    int n_ids = 0;
    for (int e = lm.cbeg[0]; e < lm.cend[0]; ++e) n_ids = std::max(n_ids, lm.etok[e] + 1);
    lm.root.assign(static_cast<size_t>(std::max(n_ids, 1)), -1);
    for (int e = lm.cbeg[0]; e < lm.cend[0]; ++e) lm.root[lm.etok[e]] = lm.enode[e];
    lm.initial = 0;
    const int bos_node = find_child(0, bos);
    if (bos_node >= 0) lm.initial = lm.depth[bos_node] == lm.order ? lm.suffix[bos_node] : bos_node;
    return 0;
}

}  // namespace tbeam_host
