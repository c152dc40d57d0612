// tests/relink/api_bench.cpp -- TEST INFRASTRUCTURE: one caller, two libraries.
// Written against the reference's public headers only (wfc/pipeline.hpp, wfc/text.hpp, wfc/analysis.hpp,
// wfc/engine.hpp; proj/include/wfc/pipeline.hpp:44-57, text.hpp:12-31, analysis.hpp, engine.hpp).  paper_2206_05269_b200/
// build.py compiles it twice: against the drop-in's headers + libwfc_b200.so (lib/reftests/api_bench_b200) and, where
// /root/reference exists, against the reference's own headers + oracle/_ref/libwfc_ref.so (oracle/_ref/api_bench_ref).
// Both print one JSON line: seconds per call and a checksum of every result, so that the two runs can be compared
// value by value (tests/test_gpu_dropin.py) and timed side by side.
//
// usage: api_bench <documents of 1 MiB> <workers> <repetitions>
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "wfc/analysis.hpp"
#include "wfc/engine.hpp"
#include "wfc/pipeline.hpp"
#include "wfc/text.hpp"

namespace {
// deterministic corpus: words of 3..10 letters drawn with a skewed distribution from a 40 k vocabulary, some
// capitalised, punctuation attached, a few accented and long ones; documents of exactly `bytes` bytes
struct Rng {
    std::uint64_t s;
    std::uint32_t next() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (std::uint32_t)(s >> 33); }
};
std::string make_document(std::uint64_t seed, std::size_t bytes) {
    Rng r{seed * 0x9E3779B97F4A7C15ull + 1};
    std::string out;
    out.reserve(bytes + 32);
    while (out.size() < bytes) {
        std::uint32_t u = r.next();
        std::uint32_t rank = u % 40000u;
        if (u & 0x10000u) rank %= 2000u;          // half of the draws from the top 2000
        if (u & 0x20000u) rank %= 100u;           // a quarter from the top 100
        Rng w{rank + 77u};
        const std::uint32_t len = 3 + w.next() % 8;
        std::string word;
        for (std::uint32_t i = 0; i < len; ++i) word.push_back((char)('a' + w.next() % 26));
        if (rank % 97 == 0) word += "\xC3\xA9";    // an accented letter
        if (rank % 4001 == 0) word += "abcdefghijklmnop";   // longer than 16 bytes
        if ((u >> 20) % 11 == 0) word[0] = (char)(word[0] - 32);
        out += word;
        const std::uint32_t p = (u >> 24) % 16;
        if (p == 0) out += ".";
        else if (p == 1) out += ",";
        out += (p == 2) ? "\n" : " ";
    }
    out.resize(bytes);
    out.back() = '\n';
    return out;
}
std::uint64_t fnv(std::uint64_t h, const std::string& s) {
    for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
    return h;
}
std::uint64_t checksum(const wfc::CountMap& m) {
    std::uint64_t h = 1469598103934665603ull;
    for (const auto& [w, c] : m) h = fnv(h, w) * 31 + c;
    return h;
}
double seconds(std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
}
}  // namespace

int main(int argc, char** argv) {
    const std::size_t n_docs = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 16;
    const std::size_t workers = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 4;
    const int reps = argc > 3 ? std::atoi(argv[3]) : 3;
    std::vector<wfc::RawDocument> docs;
    for (std::size_t d = 0; d < n_docs; ++d) docs.push_back({"doc" + std::to_string(d), make_document(d, 1u << 20)});
    const double gb = (double)n_docs * (1u << 20) / 1e9;

    // warm-up (library initialisation, first allocations), then the timed calls
    wfc::RunResult run = wfc::run_wordcount(docs, workers);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) run = wfc::run_wordcount(docs, workers);
    const double t_run = seconds(t0) / reps;

    wfc::CountMap serial = wfc::serial_wordcount(docs);
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) serial = wfc::serial_wordcount(docs);
    const double t_serial = seconds(t0) / reps;

    wfc::WordList words = wfc::tokenize(docs[0]);
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) words = wfc::tokenize(docs[0]);
    const double t_tok = seconds(t0) / reps;
    std::uint64_t h_words = 1469598103934665603ull;
    for (const auto& w : words.words) h_words = fnv(h_words, w);

    const wfc::FrequencyTable top = wfc::top_k(run.counts, "bench", 25);
    std::uint64_t h_top = 1469598103934665603ull;
    for (const auto& row : top.rows) h_top = fnv(h_top, row.word) * 31 + row.count;

    std::vector<double> values(1u << 24);
    Rng r{42};
    for (double& v : values) v = (double)(r.next() >> 8) / (double)(1u << 24);
    const wfc::BlockConfig cfg{256, std::max(1u, std::thread::hardware_concurrency())};
    double folded = wfc::map_reduce_blocked(values, wfc::MapKind::square_root, cfg);
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) folded = wfc::map_reduce_blocked(values, wfc::MapKind::square_root, cfg);
    const double t_fold = seconds(t0) / reps;

    std::uint64_t pre = 0;
    for (const auto& shard : run.pre_repair_shards) pre = pre * 1315423911ull + checksum(shard);
    std::printf("{\"documents\": %zu, \"workers\": %zu, \"corpus_GB\": %.6f, "
                "\"run_wordcount_s\": %.6f, \"run_wordcount_GBps\": %.4f, \"serial_wordcount_s\": %.6f, \"serial_wordcount_GBps\": %.4f, "
                "\"tokenize_1MiB_s\": %.6f, \"map_reduce_blocked_2p24_s\": %.6f, "
                "\"counts\": %zu, \"counts_checksum\": \"%016llx\", \"serial_checksum\": \"%016llx\", \"pre_repair_checksum\": \"%016llx\", "
                "\"tokens_doc0\": %zu, \"tokens_checksum\": \"%016llx\", \"top25_checksum\": \"%016llx\", \"fold\": \"%.17g\", "
                "\"map_ns\": %llu, \"sort_ns\": %llu, \"exchange_ns\": %llu, \"reduce_ns\": %llu, \"total_ns\": %llu}\n",
                n_docs, workers, gb, t_run, gb / t_run, t_serial, gb / t_serial, t_tok, t_fold, run.counts.size(),
                (unsigned long long)checksum(run.counts), (unsigned long long)checksum(serial), (unsigned long long)pre,
                words.words.size(), (unsigned long long)h_words, (unsigned long long)h_top, folded,
                (unsigned long long)run.timings.map_ns, (unsigned long long)run.timings.sort_ns,
                (unsigned long long)run.timings.exchange_ns, (unsigned long long)run.timings.reduce_ns,
                (unsigned long long)run.timings.total_ns);
    return checksum(run.counts) == checksum(serial) ? 0 : 1;
}
