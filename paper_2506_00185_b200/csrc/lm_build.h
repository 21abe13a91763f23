#pragma once

#include <cstddef>
#include <string>
#include <vector>

namespace tbeam_host {

// Frozen ARPA trie, host copy of DevLm's arrays (see lm_build.cpp).
struct HostLm {
    int order = 0;
    int V = 0;
    int initial = 0;
    std::size_t oov_mapped = 0;
    double unk_prob = 0.0;
    std::vector<double> prob, backoff;
    std::vector<int> suffix, depth, cbeg, cend, etok, enode, remap;
    std::vector<float> uni;
    std::vector<int> root;  // dense root children: internal id -> node or -1
};

// 0 on success, 3 (TBEAM_PARSE) with `err` = "source:line: what" on failure.
int build_lm(const char* text, std::size_t len, const std::vector<std::string>& vocab, bool strict,
             HostLm& lm, std::string& err);

}  // namespace tbeam_host
