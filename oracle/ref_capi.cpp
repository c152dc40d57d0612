// oracle/ref_capi.cpp -- extern "C" view of the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/wfc_oracle.c).  This file is ours; it is
// compiled by oracle/Makefile together with the reference's own translation
// units taken where they lie (/root/reference/proj/src/*.cpp, never copied into
// this repo) into oracle/_ref/libwfc_ref.so.  It exposes the reference's C++
// API (proj/include/wfc/*.hpp) with the same C shapes as wfc_oracle.c (prefix
// wfr_ instead of wfo_) so one Python harness can drive both, and so that
// bench.py --impl reference can time the real reference on the host cores.
#include <cstdint>
#include <cstring>
#include <random>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "wfc/analysis.hpp"
#include "wfc/engine.hpp"
#include "wfc/pipeline.hpp"
#include "wfc/reduce.hpp"
#include "wfc/shuffle.hpp"
#include "wfc/text.hpp"
#include "wfc/unicode.hpp"

#define WFR_API extern "C" __attribute__((visibility("default")))

namespace {

struct Decoded { uint32_t cp; uint32_t len; int32_t valid; };

std::string_view sv(const uint8_t* p, uint64_t n) {
    return std::string_view(reinterpret_cast<const char*>(p), std::size_t(n));
}

wfc::WordList unpack(const uint8_t* bytes, const uint32_t* lens, uint64_t ntok, bool sorted) {
    wfc::WordList wl;
    wl.words.reserve(ntok);
    uint64_t off = 0;
    for (uint64_t i = 0; i < ntok; ++i) {
        wl.words.emplace_back(reinterpret_cast<const char*>(bytes + off), lens[i]);
        off += lens[i];
    }
    wl.sorted = sorted;
    return wl;
}

wfc::CountMap unpack_counts(const uint8_t* bytes, const uint32_t* lens, const uint64_t* counts, uint64_t n) {
    wfc::CountMap m;
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; ++i) {
        m.emplace_hint(m.end(), std::string(reinterpret_cast<const char*>(bytes + off), lens[i]), counts[i]);
        off += lens[i];
    }
    return m;
}

std::vector<wfc::RawDocument> make_docs(const uint8_t* const* docs, const uint64_t* lens, uint64_t nd) {
    std::vector<wfc::RawDocument> v;
    v.reserve(nd);
    for (uint64_t d = 0; d < nd; ++d)
        v.push_back({"doc" + std::to_string(d), std::string(reinterpret_cast<const char*>(docs[d]), lens[d])});
    return v;
}

wfc::MapKind kind_of(int k) { return static_cast<wfc::MapKind>(k); }

}  // namespace

struct wfr_counts { wfc::CountMap map; };

WFR_API Decoded wfr_utf8_decode(const uint8_t* s, uint64_t n, uint64_t pos) {
    const wfc::DecodedChar d = wfc::utf8_decode(sv(s, n), pos);
    return {uint32_t(d.cp), d.length, d.valid ? 1 : 0};
}
WFR_API int wfr_is_space(uint32_t cp) { return wfc::is_unicode_space(cp); }
WFR_API int wfr_is_word_char(uint32_t cp) { return wfc::is_word_char(cp); }
WFR_API uint32_t wfr_simple_lower(uint32_t cp) { return uint32_t(wfc::simple_lower(cp)); }
WFR_API int wfr_utf8_valid(const uint8_t* s, uint64_t n) { return wfc::utf8_valid(sv(s, n)); }
WFR_API uint64_t wfr_utf8_sanitize(const uint8_t* s, uint64_t n, uint8_t* out) {
    const std::string r = wfc::utf8_sanitize(sv(s, n));
    std::memcpy(out, r.data(), r.size());
    return r.size();
}

WFR_API uint64_t wfr_normalize_word(const uint8_t* frag, uint64_t n, uint8_t* out) {
    const auto w = wfc::normalize_word(sv(frag, n));
    if (!w) return 0;
    std::memcpy(out, w->data(), w->size());
    return w->size();
}

WFR_API int wfr_tokenize(const uint8_t* text, uint64_t n, uint8_t* out_bytes, uint64_t bytes_cap,
                         uint32_t* out_lens, uint64_t lens_cap, uint64_t* n_tokens, uint64_t* n_bytes) {
    const wfc::WordList wl = wfc::tokenize({"doc", std::string(sv(text, n))});
    uint64_t nb = 0;
    for (const auto& w : wl.words) nb += w.size();
    *n_tokens = wl.words.size();
    *n_bytes = nb;
    if (wl.words.size() > lens_cap || nb > bytes_cap) return 1;
    uint64_t off = 0;
    for (std::size_t i = 0; i < wl.words.size(); ++i) {
        std::memcpy(out_bytes + off, wl.words[i].data(), wl.words[i].size());
        out_lens[i] = uint32_t(wl.words[i].size());
        off += wl.words[i].size();
    }
    return 0;
}

WFR_API wfr_counts* wfr_counts_new() { return new wfr_counts; }
WFR_API void wfr_counts_free(wfr_counts* c) { delete c; }

// serial_wordcount restricted to one document, accumulated by merge_counts.
WFR_API void wfr_counts_add_document(wfr_counts* c, const uint8_t* text, uint64_t n) {
    const std::vector<wfc::RawDocument> one{{"doc", std::string(sv(text, n))}};
    const std::vector<wfc::CountMap> both{std::move(c->map), wfc::serial_wordcount(one)};
    c->map = wfc::merge_counts(both);
}

WFR_API wfr_counts* wfr_serial_wordcount(const uint8_t* const* docs, const uint64_t* lens, uint64_t nd) {
    auto* c = new wfr_counts;
    c->map = wfc::serial_wordcount(make_docs(docs, lens, nd));
    return c;
}

// timings_ns: 7 values in StageTimings order (may be null).  Returns null and
// fills err (if given) on exception.
WFR_API wfr_counts* wfr_run_wordcount(const uint8_t* const* docs, const uint64_t* lens, uint64_t nd,
                                      uint64_t n_workers, uint64_t* timings_ns, char* err, uint64_t err_cap) {
    try {
        const wfc::RunResult r = wfc::run_wordcount(make_docs(docs, lens, nd), n_workers);
        if (timings_ns) {
            const auto& t = r.timings;
            const uint64_t v[7] = {t.map_ns, t.sort_ns, t.encode_ns, t.exchange_ns, t.reduce_ns, t.repair_ns, t.total_ns};
            std::memcpy(timings_ns, v, sizeof(v));
        }
        auto* c = new wfr_counts;
        c->map = r.counts;
        return c;
    } catch (const std::exception& e) {
        if (err && err_cap) { std::strncpy(err, e.what(), err_cap - 1); err[err_cap - 1] = 0; }
        return nullptr;
    }
}

WFR_API uint64_t wfr_counts_distinct(const wfr_counts* c) { return c->map.size(); }
WFR_API uint64_t wfr_counts_total(const wfr_counts* c) {
    uint64_t t = 0;
    for (const auto& [w, n] : c->map) t += n;
    return t;
}
WFR_API uint64_t wfr_counts_key_bytes(const wfr_counts* c) {
    uint64_t t = 0;
    for (const auto& [w, n] : c->map) t += w.size();
    return t;
}
WFR_API void wfr_counts_export(const wfr_counts* c, uint8_t* key_bytes, uint32_t* key_lens, uint64_t* counts) {
    uint64_t off = 0, i = 0;
    for (const auto& [w, n] : c->map) {
        std::memcpy(key_bytes + off, w.data(), w.size());
        off += w.size();
        key_lens[i] = uint32_t(w.size());
        counts[i] = n;
        ++i;
    }
}
WFR_API void wfr_counts_merge(wfr_counts* dst, const wfr_counts* src) {
    const std::vector<wfc::CountMap> both{std::move(dst->map), src->map};
    dst->map = wfc::merge_counts(both);
}

WFR_API void wfr_sort_words(const uint8_t* bytes, const uint32_t* lens, uint64_t ntok,
                            uint8_t* out_bytes, uint32_t* out_lens) {
    const wfc::WordList s = wfc::sort_words(unpack(bytes, lens, ntok, false));
    uint64_t off = 0;
    for (std::size_t i = 0; i < s.words.size(); ++i) {
        std::memcpy(out_bytes + off, s.words[i].data(), s.words[i].size());
        out_lens[i] = uint32_t(s.words[i].size());
        off += s.words[i].size();
    }
}

// Same contract as wfo_reduce_sorted.  The reference trusts the `sorted` flag;
// the flag is set here only when the list really is sorted so that the
// reference's own std::invalid_argument is what reports an unsorted input.
WFR_API uint64_t wfr_reduce_sorted(const uint8_t* bytes, const uint32_t* lens, uint64_t ntok,
                                   uint64_t* run_first, uint64_t* run_count) {
    wfc::WordList wl = unpack(bytes, lens, ntok, true);
    for (std::size_t i = 1; i < wl.words.size(); ++i)
        if (wl.words[i - 1] > wl.words[i]) wl.sorted = false;
    try {
        const wfc::CountMap m = wfc::reduce_sorted(wl);
        uint64_t r = 0, first = 0;
        for (const auto& [w, n] : m) {   // map order == sorted order
            run_first[r] = first;
            run_count[r] = n;
            first += n;
            ++r;
        }
        return r;
    } catch (const std::invalid_argument&) {
        return UINT64_MAX;
    }
}

WFR_API int wfr_plan_partition(uint64_t k, uint64_t worker_id, uint64_t n_workers, uint64_t* boundaries) {
    wfc::WordList wl;
    wl.words.assign(k, "w");
    wl.sorted = true;
    try {
        const wfc::ShardPlan p = wfc::plan_partition(wl, worker_id, n_workers);
        for (std::size_t i = 0; i < p.boundaries.size(); ++i) boundaries[i] = p.boundaries[i];
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

WFR_API double wfr_map_reduce_serial_f64(const double* v, uint64_t n, int kind) {
    return wfc::map_reduce_serial(std::span<const double>(v, n), kind_of(kind));
}
WFR_API double wfr_map_reduce_blocked_f64(const double* v, uint64_t n, int kind, uint64_t block,
                                          unsigned workers, int* err) {
    if (err) *err = 0;
    try {
        return wfc::map_reduce_blocked(std::span<const double>(v, n), kind_of(kind), {std::size_t(block), workers});
    } catch (const std::invalid_argument&) {
        if (err) *err = 1;
        return 0.0;
    }
}
WFR_API double wfr_alternating_harmonic(uint64_t n, uint64_t block, unsigned workers, int* err) {
    if (err) *err = 0;
    try {
        return wfc::alternating_harmonic(n, {std::size_t(block), workers});
    } catch (const std::invalid_argument&) {
        if (err) *err = 1;
        return 0.0;
    }
}

WFR_API uint64_t wfr_top_k(const uint8_t* key_bytes, const uint32_t* key_lens, const uint64_t* counts,
                           uint64_t n, uint64_t k, uint64_t* out_idx, double* out_rel, uint64_t* total) {
    const wfc::CountMap m = unpack_counts(key_bytes, key_lens, counts, n);
    const wfc::FrequencyTable t = wfc::top_k(m, "t", k);
    *total = t.total_words;
    for (std::size_t r = 0; r < t.rows.size(); ++r) {
        out_idx[r] = uint64_t(std::distance(m.begin(), m.find(t.rows[r].word)));
        out_rel[r] = t.rows[r].rel_freq;
    }
    return t.rows.size();
}

WFR_API uint64_t wfr_distinctive(const uint8_t* t_bytes, const uint32_t* t_lens, const uint64_t* t_counts, uint64_t nt,
                                 const uint8_t* o_bytes, const uint32_t* o_lens, const uint64_t* o_counts, uint64_t no,
                                 uint64_t k, int32_t* out_src, uint64_t* out_idx, double* out_score) {
    const wfc::CountMap t = unpack_counts(t_bytes, t_lens, t_counts, nt);
    const wfc::CountMap o = unpack_counts(o_bytes, o_lens, o_counts, no);
    const wfc::DistinctivenessReport rep = wfc::distinctive_words(t, o, "t", k);
    for (std::size_t r = 0; r < rep.rows.size(); ++r) {
        const auto it = t.find(rep.rows[r].word);
        if (it != t.end()) {
            out_src[r] = 0;
            out_idx[r] = uint64_t(std::distance(t.begin(), it));
        } else {
            out_src[r] = 1;
            out_idx[r] = uint64_t(std::distance(o.begin(), o.find(rep.rows[r].word)));
        }
        out_score[r] = rep.rows[r].score;
    }
    return rep.rows.size();
}

// The reference bench's input recipe, with the real std:: classes
// (proj/src/cli.cpp:120-125) -- checks wfcu_synth_uniform.
WFR_API void wfr_fill_uniform(uint64_t seed, double* out, uint64_t n) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(0.0, 1.0);
    for (uint64_t i = 0; i < n; ++i) out[i] = dist(rng);
}
