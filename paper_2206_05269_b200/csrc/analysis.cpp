// analysis.cpp -- top_k and distinctive_words over exported count tables
// (/root/reference/proj/src/analysis.cpp:58-132), host side of the C ABI.
//
// The counts come from the device tables; what is left is ordering at most V rows with
// the reference's exact comparators (count desc / score desc by exact double compare,
// then word asc), which is container work, not arithmetic of the path.  Scores use the
// reference's expression verbatim so the doubles are bit-identical.  wfcu_counter_distinctive
// (capi.cu) joins and pre-selects the candidates on the device and ranks them with the same function.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace wfcu {

namespace {
struct Key {
    const uint8_t* p;
    uint32_t len;
};
inline int key_cmp(const Key& a, const Key& b) {
    const uint32_t m = a.len < b.len ? a.len : b.len;
    const int r = m ? std::memcmp(a.p, b.p, m) : 0;
    if (r) return r;
    return (a.len > b.len) - (a.len < b.len);
}
std::vector<Key> keys_of(const uint8_t* bytes, const uint32_t* lens, uint64_t n) {
    std::vector<Key> k(n);
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; ++i) {
        k[i] = {bytes + off, lens[i]};
        off += lens[i];
    }
    return k;
}
}  // namespace

uint64_t analysis_top_k(const uint8_t* bytes, const uint32_t* lens, const uint64_t* counts, uint64_t n, uint64_t k,
                        uint64_t* out_idx, double* out_rel, uint64_t* total) {
    const std::vector<Key> keys = keys_of(bytes, lens, n);
    uint64_t tot = 0;
    std::vector<uint64_t> order(n);
    for (uint64_t i = 0; i < n; ++i) {
        tot += counts[i];
        order[i] = i;
    }
    const uint64_t keep = std::min(k, n);
    std::partial_sort(order.begin(), order.begin() + keep, order.end(), [&](uint64_t a, uint64_t b) {
        if (counts[a] != counts[b]) return counts[a] > counts[b];
        return key_cmp(keys[a], keys[b]) < 0;
    });
    for (uint64_t r = 0; r < keep; ++r) {
        out_idx[r] = order[r];
        out_rel[r] = double(counts[order[r]]) / double(tot);
    }
    *total = tot;
    return keep;
}

// One row of a distinctiveness ranking; `tag` is the caller's (which table / which candidate it is).
struct ScoredRow {
    const uint8_t* key;
    uint32_t len;
    uint64_t in_target, in_others, tag;
    double score;
};
// Scores the rows with the reference's expression (proj/src/analysis.cpp:104-110; `vocab` = size of the union
// vocabulary, which may be larger than rows.size() when the caller only passes the rows that can make the cut) and
// puts the best min(k, rows) in front: score descending by exact double compare, word ascending (:125-128).
// The ONE implementation of this order: the host-table call below and the device path (capi.cu) both end here.
uint64_t analysis_rank_rows(std::vector<ScoredRow>& rows, uint64_t vocab, uint64_t t_total, uint64_t o_total, uint64_t k) {
    const double t_den = double(t_total) + double(vocab);
    const double o_den = double(o_total) + double(vocab);
    for (auto& r : rows)
        r.score = std::log((double(r.in_target) + 1.0) / t_den) - std::log((double(r.in_others) + 1.0) / o_den);
    const uint64_t keep = std::min<uint64_t>(k, rows.size());
    std::partial_sort(rows.begin(), rows.begin() + keep, rows.end(), [](const ScoredRow& a, const ScoredRow& b) {
        if (a.score != b.score) return a.score > b.score;
        return key_cmp(Key{a.key, a.len}, Key{b.key, b.len}) < 0;
    });
    return keep;
}

uint64_t analysis_distinctive(const uint8_t* t_bytes, const uint32_t* t_lens, const uint64_t* t_counts, uint64_t nt,
                              const uint8_t* o_bytes, const uint32_t* o_lens, const uint64_t* o_counts, uint64_t no,
                              uint64_t k, int32_t* out_src, uint64_t* out_idx, double* out_score) {
    if (nt == 0 && no == 0) return 0;
    const std::vector<Key> tk = keys_of(t_bytes, t_lens, nt), ok = keys_of(o_bytes, o_lens, no);
    uint64_t t_total = 0, o_total = 0;
    for (uint64_t i = 0; i < nt; ++i) t_total += t_counts[i];
    for (uint64_t i = 0; i < no; ++i) o_total += o_counts[i];
    std::vector<ScoredRow> rows;
    rows.reserve(nt + no);
    uint64_t i = 0, j = 0;
    while (i < nt || j < no) {   // union of the two ordered tables; tag = 2 * index + (1 if the row is the others')
        const int c = j >= no ? -1 : i >= nt ? 1 : key_cmp(tk[i], ok[j]);
        if (c < 0) { rows.push_back({tk[i].p, tk[i].len, t_counts[i], 0, 2 * i, 0.0}); ++i; }
        else if (c > 0) { rows.push_back({ok[j].p, ok[j].len, 0, o_counts[j], 2 * j + 1, 0.0}); ++j; }
        else { rows.push_back({tk[i].p, tk[i].len, t_counts[i], o_counts[j], 2 * i, 0.0}); ++i; ++j; }
    }
    const uint64_t keep = analysis_rank_rows(rows, rows.size(), t_total, o_total, k);
    for (uint64_t r = 0; r < keep; ++r) {
        out_src[r] = int32_t(rows[r].tag & 1);
        out_idx[r] = rows[r].tag >> 1;
        out_score[r] = rows[r].score;
    }
    return keep;
}

}  // namespace wfcu
