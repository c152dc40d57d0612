// dropin_tests.cpp -- the drop-in exercised the way the reference's own suites exercise
// the reference: same call sites, same expectations (each case cites the reference test
// it mirrors, paths relative to /root/reference/proj/tests/).  Needs a B200; run by
// tests/test_gpu_dropin.py.  No test framework dependency: a 20-line CHECK harness.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "wfc/analysis.hpp"
#include "wfc/engine.hpp"
#include "wfc/pipeline.hpp"
#include "wfc/reduce.hpp"
#include "wfc/shuffle.hpp"
#include "wfc/text.hpp"
#include "wfc/transport.hpp"
#include "wfc/unicode.hpp"
#include "wfc/wire.hpp"

using namespace wfc;

static int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_failed;                                                          \
            std::printf("FAILED %s:%d  %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, Type)                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        bool threw = false;                                                      \
        try { (void)(expr); } catch (const Type&) { threw = true; } catch (...) {} \
        if (!threw) { ++g_failed; std::printf("FAILED %s:%d  %s should throw %s\n", __FILE__, __LINE__, #expr, #Type); } \
    } while (0)

using Rng = std::mt19937_64;

static std::string vocab_word(std::size_t i) {          // support.hpp:18-22
    char buf[16];
    std::snprintf(buf, sizeof(buf), "w%04zu", i);
    return buf;
}
static std::vector<RawDocument> iid_corpus(Rng& rng, std::size_t docs, std::size_t words_per_doc, std::size_t vocab) {
    std::vector<RawDocument> corpus;               // support.hpp:42-51
    std::uniform_int_distribution<std::size_t> pick(0, vocab - 1);
    for (std::size_t d = 0; d < docs; ++d) {
        std::string text;
        for (std::size_t w = 0; w < words_per_doc; ++w) {
            if (!text.empty()) text += ' ';
            text += vocab_word(pick(rng));
        }
        corpus.push_back({"doc" + std::to_string(d), text});
    }
    return corpus;
}
// independent host oracle for the tests only: whitespace split of generator output
static CountMap naive_count(const std::vector<RawDocument>& corpus) {
    CountMap m;
    for (const auto& d : corpus) {
        std::size_t i = 0;
        while (i < d.text.size()) {
            while (i < d.text.size() && d.text[i] == ' ') ++i;
            std::size_t j = i;
            while (j < d.text.size() && d.text[j] != ' ') ++j;
            if (j > i) ++m[d.text.substr(i, j - i)];
            i = j;
        }
    }
    return m;
}
static std::vector<double> random_uniforms(std::size_t n, std::uint64_t seed) {   // engine_test.cpp:14-20
    Rng rng(seed);
    std::uniform_real_distribution<double> uniform(0.0, 1.0);
    std::vector<double> v(n);
    for (auto& x : v) x = uniform(rng);
    return v;
}

static const std::vector<RawDocument> kTwoDocs{{"doc1", "I want to test MapReduce"},
                                               {"doc2", "MapReduce is a cool algorithm to test."}};

static void text_cases() {
    // text_test.cpp:40-58
    CHECK(normalize_word("Dog") == "dog");
    CHECK(normalize_word("dog.") == "dog");
    CHECK(normalize_word("---") == std::nullopt);
    CHECK(normalize_word("don't") == "don't");
    CHECK(normalize_word("re-elect") == "re-elect");
    CHECK(normalize_word("\"quoted!\"") == "quoted");
    CHECK(normalize_word("2021") == "2021");
    CHECK(normalize_word("") == std::nullopt);
    CHECK(normalize_word("''") == std::nullopt);
    CHECK(normalize_word("\xE2\x80\x9Cword\xE2\x80\x9D") == "word");
    CHECK(normalize_word("caf\xC3\xA9") == "caf\xC3\xA9");
    CHECK(normalize_word("CAF\xC3\x89") == "caf\xC3\xA9");
    CHECK(normalize_word("word\xE2\x80\xA6") == "word");
    CHECK(normalize_word("\xE2\x80\x94") == std::nullopt);
    // text_test.cpp:60-72, batched: 5000 random printable-ASCII fragments vs tolower/isalnum trim
    {
        Rng rng(2024);
        std::uniform_int_distribution<int> len(1, 12), ch('!', '~');
        std::vector<std::string> frags;
        for (int i = 0; i < 5000; ++i) {
            std::string f;
            const int n = len(rng);
            for (int c = 0; c < n; ++c) f.push_back(char(ch(rng)));
            frags.push_back(f);
        }
        const auto got = normalize_words(frags);
        for (std::size_t i = 0; i < frags.size(); ++i) {
            std::string s = frags[i];
            for (auto& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
            std::size_t b = 0, e = s.size();
            while (b < e && !std::isalnum(static_cast<unsigned char>(s[b]))) ++b;
            while (e > b && !std::isalnum(static_cast<unsigned char>(s[e - 1]))) --e;
            const std::optional<std::string> want = b == e ? std::nullopt : std::optional<std::string>(s.substr(b, e - b));
            CHECK(got[i] == want);
        }
        // idempotence, text_test.cpp:74-92
        std::vector<std::string> once;
        for (const auto& g : got) if (g) once.push_back(*g);
        const auto twice = normalize_words(once);
        for (std::size_t i = 0; i < once.size(); ++i) CHECK(twice[i] == once[i]);
    }
    // text_test.cpp:94-118
    CHECK(tokenize({"d", "I want to test MapReduce"}).words == (std::vector<std::string>{"i", "want", "to", "test", "mapreduce"}));
    CHECK(tokenize({"d", "MapReduce is a cool algorithm to test."}).words ==
          (std::vector<std::string>{"mapreduce", "is", "a", "cool", "algorithm", "to", "test"}));
    CHECK(tokenize({"d", ""}).words.empty());
    CHECK(!tokenize({"d", "a b"}).sorted);
    CHECK(tokenize({"d", "Dog dog. DOG!"}).words == (std::vector<std::string>{"dog", "dog", "dog"}));
    CHECK(tokenize({"d", "a\xC2\xA0" "b\xE2\x80\x83" "c"}).words == (std::vector<std::string>{"a", "b", "c"}));
    CHECK(tokenize({"d", "one\ttwo\nthree"}).words == (std::vector<std::string>{"one", "two", "three"}));
    CHECK(tokenize({"d", "--- a !!! b ..."}).words == (std::vector<std::string>{"a", "b"}));
    // text_test.cpp:143-169
    CHECK(sort_words(WordList{{"i", "want", "to", "test", "mapreduce"}, false}).words ==
          (std::vector<std::string>{"i", "mapreduce", "test", "to", "want"}));
    CHECK(sort_words(WordList{}).words.empty());
    CHECK(sort_words(WordList{}).sorted);
    {
        Rng rng(4242);
        std::uniform_int_distribution<int> len(0, 200), word(0, 30);
        for (int i = 0; i < 20; ++i) {
            std::vector<std::string> words;
            const int n = len(rng);
            for (int w = 0; w < n; ++w) words.push_back("w" + std::to_string(word(rng)));
            const WordList sorted = sort_words(WordList{words, false});
            std::vector<std::string> want = words;
            std::stable_sort(want.begin(), want.end());
            CHECK(sorted.sorted);
            CHECK(sorted.words == want);
        }
    }
}

static void unicode_cases() {
    // text_test.cpp:171-187: invalid bytes are replaced, valid tokens stay countable
    const std::string bytes = std::string("good ") + char(0xFF) + " word";
    const std::string clean = utf8_sanitize(bytes);
    CHECK(clean == "good \xEF\xBF\xBD word");
    CHECK(utf8_valid(clean));
    // text_test.cpp:180-187
    CHECK(utf8_valid("plain ascii"));
    CHECK(utf8_valid("caf\xC3\xA9 \xE3\x81\x82"));
    CHECK(!utf8_valid(std::string("\xC0\xAF")));
    CHECK(!utf8_valid(std::string("\xED\xA0\x80")));
    CHECK(!utf8_valid(std::string("\xF5\x80\x80\x80")));
    CHECK(!utf8_valid(std::string("\x80")));
    CHECK((tokenize(RawDocument{"d", clean}).words == std::vector<std::string>{"good", "word"}));
    CHECK(utf8_sanitize("") == "");
    CHECK(utf8_sanitize("caf\xC3\xA9 \xE2\x80\x9Cq\xE2\x80\x9D") == "caf\xC3\xA9 \xE2\x80\x9Cq\xE2\x80\x9D");   // valid text is unchanged
    CHECK(utf8_sanitize("\xC0\xAF") == "\xEF\xBF\xBD\xEF\xBF\xBD");                 // overlong: one replacement per byte
    CHECK(utf8_sanitize("\xED\xA0\x80") == "\xEF\xBF\xBD\xEF\xBF\xBD\xEF\xBF\xBD");   // surrogate
    CHECK(utf8_sanitize("a\xE2\x82") == "a\xEF\xBF\xBD\xEF\xBF\xBD");                 // truncated at the end
    CHECK(utf8_sanitize(clean) == clean);                                               // idempotent
}

static void reduce_cases() {
    // reduce_test.cpp:28-58
    CHECK(reduce_sorted(WordList{{"a", "algorithm", "cool", "i", "is", "mapreduce"}, true}) ==
          (CountMap{{"a", 1}, {"algorithm", 1}, {"cool", 1}, {"i", 1}, {"is", 1}, {"mapreduce", 1}}));
    CHECK(reduce_sorted(WordList{{"mapreduce", "test", "test", "to", "to", "want"}, true}) ==
          (CountMap{{"mapreduce", 1}, {"test", 2}, {"to", 2}, {"want", 1}}));
    CHECK(reduce_sorted(WordList{{}, true}).empty());
    CHECK_THROWS_AS(reduce_sorted(WordList{{"b", "a"}, false}), std::invalid_argument);
    // reduce_test.cpp:60-135
    {
        ShardedCounts pre{{{"a", 1}, {"mapreduce", 1}}, {{"mapreduce", 1}, {"test", 2}}};
        const ShardedCounts post = boundary_repair(pre);
        CHECK(post[0] == (CountMap{{"a", 1}, {"mapreduce", 2}}));
        CHECK(post[1] == (CountMap{{"test", 2}}));
        CHECK(count_unreduced_words(pre) == 1);
        CHECK(count_unreduced_words(post) == 0);
        ShardedCounts three{{{"x", 1}}, {{"x", 2}}, {}, {{"x", 4}, {"y", 1}}};
        const ShardedCounts r3 = boundary_repair(three);
        CHECK(r3[0] == (CountMap{{"x", 7}}));
        CHECK(r3[1].empty());
        CHECK(r3[3] == (CountMap{{"y", 1}}));
    }
    // reduce_test.cpp:112-155
    {
        const std::vector<CountMap> maps{{{"a", 1}, {"b", 2}}, {{"b", 3}, {"c", 4}}, {}};
        CHECK(merge_counts(maps) == (CountMap{{"a", 1}, {"b", 5}, {"c", 4}}));
        const std::vector<CountMap> rev{maps[1], maps[0]};
        CHECK(merge_counts(rev) == merge_counts(maps));
        CHECK(merge_counts(std::vector<CountMap>{}).empty());
    }
}

static void pipeline_cases() {
    const CountMap expected{{"a", 1}, {"algorithm", 1}, {"cool", 1}, {"i", 1}, {"is", 1},
                            {"mapreduce", 2}, {"test", 2}, {"to", 2}, {"want", 1}};
    // pipeline_test.cpp:26-54, acceptance_test.cpp:155-162: the paper's worked example, pre-repair shards included
    {
        const RunResult r = run_wordcount(kTwoDocs, 2);
        CHECK(r.counts == expected);
        CHECK(r.counts == serial_wordcount(kTwoDocs));
        CHECK(merge_counts(r.shards) == r.counts);
        CHECK(r.n_workers == 2);
        CHECK(r.pre_repair_shards.size() == 2);
        CHECK(r.pre_repair_shards[0] == (CountMap{{"a", 1}, {"algorithm", 1}, {"cool", 1}, {"i", 1}, {"is", 1}, {"mapreduce", 1}}));
        CHECK(r.pre_repair_shards[1] == (CountMap{{"mapreduce", 1}, {"test", 2}, {"to", 2}, {"want", 1}}));
        CHECK(count_unreduced_words(r.pre_repair_shards) == 1);
        CHECK(count_unreduced_words(r.shards) == 0);
        CHECK(r.shards[0].at("mapreduce") == 2);
        // the hash-partitioned fast path: same counts, disjoint shards, nothing to repair
        const RunResult h = run_wordcount_hashed(kTwoDocs, 2);
        CHECK(h.counts == expected);
        CHECK(h.shards.size() == 2);
        CHECK(h.pre_repair_shards == h.shards);
        CHECK(count_unreduced_words(h.shards) == 0);
        CHECK(merge_counts(h.shards) == h.counts);
        CHECK(h.timings.map_ns > 0);
        CHECK(run_wordcount_hashed(kTwoDocs, 5).counts == expected);
        const auto& t = r.timings;
        CHECK(t.total_ns >= std::max({t.map_ns, t.sort_ns, t.encode_ns, t.exchange_ns, t.reduce_ns, t.repair_ns}));
        CHECK(run_wordcount(kTwoDocs, 1).counts == expected);
    }
    // pipeline_test.cpp:56-80
    {
        const std::vector<RawDocument> empty;
        const RunResult r = run_wordcount(empty, 4);
        CHECK(r.counts.empty());
        CHECK(r.shards.size() == 4);
        CHECK(r.timings.map_ns == 0 && r.timings.sort_ns == 0 && r.timings.encode_ns == 0);
        CHECK(r.timings.exchange_ns == 0 && r.timings.reduce_ns == 0 && r.timings.repair_ns == 0);
        CHECK_THROWS_AS(run_wordcount(kTwoDocs, 0), std::invalid_argument);
    }
    // pipeline_test.cpp:82-95
    {
        Rng rng(1001);
        for (int round = 0; round < 4; ++round) {
            const std::size_t docs = std::uniform_int_distribution<std::size_t>(1, 40)(rng);
            const std::size_t words = std::uniform_int_distribution<std::size_t>(1, 300)(rng);
            const auto corpus = iid_corpus(rng, docs, words, 60);
            const CountMap oracle = serial_wordcount(corpus);
            CHECK(oracle == naive_count(corpus));
            for (std::size_t n : {1, 2, 3, 5, 8}) {
                const RunResult r = run_wordcount(corpus, n);
                CHECK(r.counts == oracle);
                CHECK(merge_counts(r.shards) == r.counts);
                CHECK(count_unreduced_words(r.shards) == 0);
            }
        }
    }
    // pipeline_test.cpp:97-104, 129-141
    {
        Rng rng(77);
        const auto corpus = iid_corpus(rng, 100, 1000, 500);
        const CountMap oracle = serial_wordcount(corpus);
        CHECK(oracle == naive_count(corpus));
        for (std::size_t n : {2, 4, 8}) CHECK(run_wordcount(corpus, n).counts == oracle);
        Rng rng2(505);
        const auto small = iid_corpus(rng2, 3, 50, 10);
        const RunResult r = run_wordcount(small, 8);
        CHECK(r.counts == serial_wordcount(small));
        CHECK(r.pre_repair_shards.size() == 8);
        CHECK(serial_wordcount(std::vector<RawDocument>{}).empty());
        CHECK(serial_wordcount(std::vector<RawDocument>{{"d", "a a b"}}) == (CountMap{{"a", 2}, {"b", 1}}));
    }
}

static void range_partition_cases() {
    // shuffle_test.cpp:91-118
    auto cuts = [](std::size_t k, std::size_t j, std::size_t n) {
        WordList wl;
        wl.words.assign(k, "w");
        wl.sorted = true;
        return plan_partition(wl, j, n).boundaries;
    };
    CHECK(cuts(5, 0, 2) == (std::vector<std::size_t>{0, 2, 5}));
    CHECK(cuts(7, 1, 2) == (std::vector<std::size_t>{0, 4, 7}));
    CHECK(cuts(10, 1, 3) == (std::vector<std::size_t>{0, 4, 7, 10}));
    CHECK(cuts(9, 0, 1) == (std::vector<std::size_t>{0, 9}));
    CHECK_THROWS_AS(cuts(3, 3, 3), std::invalid_argument);
    CHECK_THROWS_AS(plan_partition(WordList{{"b", "a"}, false}, 0, 2), std::invalid_argument);
    // pipeline_test.cpp:26-48: the worked example, BEFORE and after repair
    const RunResult r = run_wordcount_range_partitioned(kTwoDocs, 2);
    CHECK(r.pre_repair_shards.size() == 2);
    CHECK(r.pre_repair_shards[0] == (CountMap{{"a", 1}, {"algorithm", 1}, {"cool", 1}, {"i", 1}, {"is", 1}, {"mapreduce", 1}}));
    CHECK(r.pre_repair_shards[1] == (CountMap{{"mapreduce", 1}, {"test", 2}, {"to", 2}, {"want", 1}}));
    CHECK(r.counts == serial_wordcount(kTwoDocs));
    CHECK(merge_counts(r.shards) == r.counts);
    CHECK(count_unreduced_words(r.pre_repair_shards) == 1);
    CHECK(count_unreduced_words(r.shards) == 0);
    // pipeline_test.cpp:82-95, 116-127 on the range-partitioned path
    Rng rng(404);
    for (int round = 0; round < 3; ++round) {
        const auto corpus = iid_corpus(rng, 12, 150, 40);
        const CountMap oracle = serial_wordcount(corpus);
        for (std::size_t n : {1, 2, 4, 8}) {
            const RunResult rr = run_wordcount_range_partitioned(corpus, n);
            CHECK(rr.counts == oracle);
            CHECK(rr.counts == run_wordcount(corpus, n).counts);
            CHECK(merge_counts(rr.shards) == rr.counts);
        }
    }
    CHECK(run_wordcount_range_partitioned(std::vector<RawDocument>{}, 3).shards.size() == 3);
}

static void engine_cases() {
    const std::vector<double> v{1.0, 4.0, 9.0};
    // engine_test.cpp:24-36
    CHECK(map_reduce_serial(v, MapKind::square_root) == 6.0);
    CHECK(map_reduce_serial({}, MapKind::square_root) == 0.0);
    CHECK(map_reduce_serial({}, MapKind::identity) == 0.0);
    CHECK(map_reduce_blocked(v, MapKind::square_root, {1, 1}) == 6.0);
    CHECK(map_reduce_blocked(v, MapKind::square_root, {1, 4}) == 6.0);
    CHECK(map_reduce_blocked({}, MapKind::identity, {16, 2}) == 0.0);
    // engine_test.cpp:38-45
    {
        const auto values = random_uniforms(1537, 9001);
        for (MapKind map : {MapKind::identity, MapKind::square_root}) {
            const double serial = map_reduce_serial(values, map);
            double host = 0.0;
            for (double x : values) host += (map == MapKind::identity ? x : std::sqrt(x));
            CHECK(serial == host);   // the left fold, bit for bit
            CHECK(map_reduce_blocked(values, map, {values.size(), 1}) == serial);
            CHECK(map_reduce_blocked(values, map, {values.size() + 100, 3}) == serial);
        }
    }
    // engine_test.cpp:47-79
    {
        double expected = 0.0;
        for (int i = 1; i <= 10; ++i) expected += (i % 2 == 1 ? 1.0 : -1.0) / i;
        const std::vector<double> ignored(10, 0.0);
        CHECK(map_reduce_serial(ignored, MapKind::alternating_harmonic_term) == expected);
        CHECK(alternating_harmonic(0) == 0.0);
        CHECK(alternating_harmonic(1) == 1.0);
        CHECK(alternating_harmonic(2) == 0.5);
        const std::vector<double> zeros(1000, 0.0);
        CHECK(alternating_harmonic(1000, {64, 2}) == map_reduce_blocked(zeros, MapKind::alternating_harmonic_term, {64, 2}));
        Rng rng(321);
        std::uniform_int_distribution<std::uint64_t> n_dist(1, 50000);
        for (int i = 0; i < 10; ++i) {
            const std::uint64_t n = n_dist(rng);
            CHECK(std::abs(alternating_harmonic(n) - 0.6931471805599453) <= 1.0 / double(n + 1));
        }
    }
    // engine_test.cpp:81-116
    {
        const auto values = random_uniforms(100000, 555);
        for (MapKind map : {MapKind::identity, MapKind::square_root, MapKind::alternating_harmonic_term}) {
            for (std::size_t block : {std::size_t(7), std::size_t(256), std::size_t(100000)}) {
                const double reference = map_reduce_blocked(values, map, {block, 1});
                for (unsigned workers : {2u, 8u}) CHECK(map_reduce_blocked(values, map, {block, workers}) == reference);
            }
            if (map != MapKind::alternating_harmonic_term) {
                const double serial = map_reduce_serial(values, map);
                CHECK(std::abs(map_reduce_blocked(values, map, {256, 4}) - serial) / std::max(1.0, std::abs(serial)) <= 1e-12);
                CHECK(std::abs(map_reduce_fast(values, map) - serial) / std::max(1.0, std::abs(serial)) <= 1e-12);
            }
        }
        const std::vector<double> neg{4.0, -1.0};
        CHECK(std::isnan(map_reduce_serial(neg, MapKind::square_root)));
        CHECK(std::isnan(map_reduce_blocked(neg, MapKind::square_root, {1, 2})));
        const std::vector<double> one{1.0};
        CHECK_THROWS_AS(map_reduce_blocked(one, MapKind::identity, {0, 1}), std::invalid_argument);
        CHECK_THROWS_AS(map_reduce_blocked(one, MapKind::identity, {4, 0}), std::invalid_argument);
        std::vector<float> f(values.begin(), values.end());
        double sq = 0.0;
        for (float x : f) sq += double(x) * double(x);
        CHECK(std::abs(map_reduce_fast(std::span<const float>(f), MapKind::square) - sq) / sq <= 1e-5);
    }
}

static void analysis_cases() {
    // analysis_test.cpp:91-145
    const CountMap m{{"the", 50}, {"a", 20}, {"union", 5}};
    const FrequencyTable table = top_k(m, "t", 2);
    CHECK(table.rows.size() == 2);
    CHECK(table.rows[0].word == "the" && table.rows[0].count == 50);
    CHECK(table.rows[1].word == "a" && table.rows[1].count == 20);
    CHECK(table.total_words == 75);
    CHECK(table.rows[0].rel_freq == 50.0 / 75.0);
    CHECK(top_k(CountMap{}, "e", 3).rows.empty());
    const FrequencyTable ties = top_k(CountMap{{"b", 2}, {"a", 2}, {"c", 1}}, "t", 3);
    CHECK(ties.rows[0].word == "a" && ties.rows[1].word == "b");
    const DistinctivenessReport rep = distinctive_words(CountMap{{"war", 2}, {"peace", 1}}, CountMap{{"peace", 2}, {"love", 1}}, "t", 1);
    CHECK(rep.rows.size() == 1 && rep.rows[0].word == "war");
    CHECK(std::abs(rep.rows[0].score - 1.0986122886681098) <= 1e-12);
    for (const auto& row : distinctive_words(CountMap{{"a", 3}, {"b", 1}}, CountMap{{"a", 3}, {"b", 1}}, "t", 10).rows) CHECK(row.score == 0.0);
    // application check (acceptance_test.cpp:297-330 shape): counts from the GPU pipeline feed top_k
    const RunResult r = run_wordcount(kTwoDocs, 2);
    const FrequencyTable top = top_k(r.counts, "two-docs", 3);
    CHECK(top.rows[0].word == "mapreduce" && top.rows[1].word == "test" && top.rows[2].word == "to");
    CHECK(top.total_words == 12);
}

static void report_cases() {
    // cli_test.cpp:45-63: the byte-exact table of `wfc wordcount --input two-docs --workers 2 --format tsv`
    // (counts_for_directory -> run_wordcount -> top_k(.., 25) -> write_frequency_tsv, cli.cpp:79-104)
    const RunResult r = run_wordcount(kTwoDocs, 2);
    std::ostringstream out;
    write_frequency_tsv(out, top_k(r.counts, "two-docs", 25));
    CHECK(out.str() ==
          "mapreduce\t2\t0.166666666667\n"
          "test\t2\t0.166666666667\n"
          "to\t2\t0.166666666667\n"
          "a\t1\t0.0833333333333\n"
          "algorithm\t1\t0.0833333333333\n"
          "cool\t1\t0.0833333333333\n"
          "i\t1\t0.0833333333333\n"
          "is\t1\t0.0833333333333\n"
          "want\t1\t0.0833333333333\n");
    CHECK(format_double(1.0986122886681098) == "1.09861228867");
    const FrequencyTable t = top_k(CountMap{{"war", 2}, {"peace", 1}}, "A", 1);
    const DistinctivenessReport d = distinctive_words(CountMap{{"war", 2}, {"peace", 1}}, CountMap{{"peace", 2}, {"love", 1}}, "A", 1);
    std::ostringstream cmp;
    write_compare_tsv(cmp, t, d);
    CHECK(cmp.str() == "A\ttop\twar\t2\t0.666666666667\nA\tdistinct\twar\t1.09861228867\n");
    std::ostringstream tim;
    write_timings_tsv(tim, r.timings);
    CHECK(tim.str().rfind("timing\tmap\t", 0) == 0);
    CHECK(tim.str().find("timing\ttotal\t") != std::string::npos);
}


// ---- the paper's own exchange: WCX1 frames, transports, shuffle ---------------------------------
static std::vector<std::string> batch(std::initializer_list<const char*> words) { return {words.begin(), words.end()}; }
template <typename Fn>
static bool wire_error_kind(Fn&& fn, WireError::Kind kind) {
    try {
        fn();
    } catch (const WireError& e) {
        return e.kind() == kind;
    } catch (...) {
    }
    return false;
}
template <typename Ex, typename Fn>
static bool throws_with(Fn&& fn, const char* needle) {
    try {
        fn();
    } catch (const Ex& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
    }
    return false;
}

static void wire_cases() {
    // wire_test.cpp:38-50 -- golden bytes
    CHECK((encode_message(batch({})) == WireMessage{0x57, 0x43, 0x58, 0x31, 0x00, 0x00, 0x00, 0x00}));
    CHECK((encode_message(batch({"a"})) == WireMessage{0x57, 0x43, 0x58, 0x31, 0x01, 0x00, 0x00, 0x00, 0x01, 0x00, 0x00, 0x00, 0x61}));
    CHECK((encode_message(batch({"to", "a"})) == WireMessage{0x57, 0x43, 0x58, 0x31, 0x02, 0x00, 0x00, 0x00, 0x02, 0x00, 0x00, 0x00,
                                                           0x01, 0x00, 0x00, 0x00, 0x74, 0x6F, 0x61}));
    // wire_test.cpp:52-70 -- round trips
    CHECK(decode_message(WireMessage{0x57, 0x43, 0x58, 0x31, 0x00, 0x00, 0x00, 0x00}).empty());
    for (const auto& words : {batch({"test", "to", "want"}), batch({"", "a", ""}), batch({"caf\xc3\xa9", "\xe6\xbc\xa2\xe5\xad\x97", "x"})})
        CHECK(decode_message(encode_message(words)) == words);
    Rng rng(9);
    for (int round = 0; round < 20; ++round) {
        std::vector<std::string> words(std::uniform_int_distribution<int>(0, 40)(rng));
        std::size_t payload = 0;
        for (auto& w : words) {
            const int len = std::uniform_int_distribution<int>(0, 12)(rng);
            for (int i = 0; i < len; ++i) utf8_append(w, std::uniform_int_distribution<int>(0, 3)(rng) ? U'a' + (rng() % 26) : char32_t(0xC0 + rng() % 0x2F00));
            payload += w.size();
        }
        const WireMessage frame = encode_message(words);
        CHECK(frame.size() == 8 + 4 * words.size() + payload);       // wire_test.cpp:120-131
        CHECK(decode_message(frame) == words);
    }
    // wire_test.cpp:72-118 -- every way a frame can be wrong
    {
        WireMessage frame = encode_message(batch({"a"}));
        frame[0] = 0x58;
        CHECK(wire_error_kind([&] { decode_message(frame); }, WireError::Kind::BadMagic));
        CHECK(throws_with<WireError>([&] { decode_message(frame); }, "magic"));
        CHECK_THROWS_AS(decode_message(WireMessage{0x57, 0x43}), WireError);
        const WireMessage two = encode_message(batch({"test", "to"}));
        for (std::size_t cut : {std::size_t(5), std::size_t(9), two.size() - 1}) {
            const WireMessage shorter(two.begin(), two.begin() + cut);
            CHECK(wire_error_kind([&] { decode_message(shorter); }, WireError::Kind::Truncated));
        }
        WireMessage longer = encode_message(batch({"a", "b"}));
        longer.push_back(0x00);
        CHECK(wire_error_kind([&] { decode_message(longer); }, WireError::Kind::TrailingBytes));
        const WireMessage not_utf8{0x57, 0x43, 0x58, 0x31, 0x01, 0x00, 0x00, 0x00, 0x01, 0x00, 0x00, 0x00, 0xFF};
        CHECK(wire_error_kind([&] { decode_message(not_utf8); }, WireError::Kind::BadEncoding));
    }
}

namespace {
class RecordingTransport final : public Transport {        // shuffle_test.cpp:37-60
public:
    explicit RecordingTransport(std::size_t n) : inner_(n) {}
    void send(std::size_t from, std::size_t to, WireMessage frame) override {
        {
            std::lock_guard<std::mutex> lock(mu_);
            frames.push_back(frame);
        }
        inner_.send(from, to, std::move(frame));
    }
    WireMessage recv(std::size_t at, std::size_t from) override { return inner_.recv(at, from); }
    std::vector<WireMessage> frames;

private:
    InProcessTransport inner_;
    std::mutex mu_;
};
class FailingTransport final : public Transport {          // shuffle_test.cpp:62-68
public:
    void send(std::size_t, std::size_t, WireMessage) override { throw TransportError("link down"); }
    WireMessage recv(std::size_t, std::size_t) override { throw TransportError("link down"); }
};
class CorruptingTransport final : public Transport {       // shuffle_test.cpp:70-86, pipeline_test.cpp:146-160
public:
    CorruptingTransport(std::size_t n, std::size_t victim) : inner_(n), victim_(victim) {}
    void send(std::size_t from, std::size_t to, WireMessage frame) override { inner_.send(from, to, std::move(frame)); }
    WireMessage recv(std::size_t at, std::size_t from) override {
        WireMessage frame = inner_.recv(at, from);
        if ((victim_ == ~std::size_t(0) || at == victim_) && !frame.empty()) frame[0] = 0x00;
        return frame;
    }

private:
    InProcessTransport inner_;
    std::size_t victim_;
};
}  // namespace

static WordList sorted_list(std::vector<std::string> words) { return sort_words(WordList{std::move(words), false}); }
static std::vector<WorkerShard> make_shards(std::vector<WordList> lists) {
    std::vector<WorkerShard> shards;
    for (std::size_t j = 0; j < lists.size(); ++j) shards.push_back({plan_partition(lists[j], j, lists.size()), lists[j]});
    return shards;
}

static void shuffle_cases() {
    // shuffle_test.cpp:154-162
    {
        const WordList doc1 = sorted_list({"i", "want", "to", "test", "mapreduce"});
        const EncodedShard shard = encode_outgoing(plan_partition(doc1, 0, 2), doc1);
        CHECK((shard.kept == std::vector<std::string>{"i", "mapreduce"}));
        CHECK(shard.outgoing.size() == 1 && shard.outgoing[0].first == 1);
        CHECK((decode_message(shard.outgoing[0].second) == std::vector<std::string>{"test", "to", "want"}));
        CHECK_THROWS_AS(encode_outgoing(plan_partition(doc1, 0, 2), WordList{{"b", "a"}, false}), std::invalid_argument);
    }
    // shuffle_test.cpp:164-182
    {
        const auto out = wfc::exchange(make_shards({sorted_list({"i", "want", "to", "test", "mapreduce"}),
                                               sorted_list({"mapreduce", "is", "a", "cool", "algorithm", "to", "test"})}));
        CHECK(out.size() == 2);
        CHECK((out[0].words == std::vector<std::string>{"a", "algorithm", "cool", "i", "is", "mapreduce"}));
        CHECK((out[1].words == std::vector<std::string>{"mapreduce", "test", "test", "to", "to", "want"}));
        CHECK(out[0].sorted && out[1].sorted);
        const auto one = wfc::exchange(make_shards({sorted_list({"b", "a", "c", "a"})}));
        CHECK((one.size() == 1 && one[0].words == std::vector<std::string>{"a", "a", "b", "c"}));
    }
    // shuffle_test.cpp:184-230 -- conservation, sortedness, determinism; :232-255 -- every frame is a valid message
    {
        Rng rng(31);
        for (std::size_t n : {2, 4, 8}) {
            std::vector<WordList> lists;
            std::map<std::string, int> before, after;
            for (std::size_t j = 0; j < n; ++j) {
                std::vector<std::string> words(std::uniform_int_distribution<std::size_t>(0, 400)(rng));
                for (auto& w : words) w = vocab_word(rng() % 50);
                for (const auto& w : words) ++before[w];
                lists.push_back(sorted_list(std::move(words)));
            }
            const auto shards = make_shards(lists);
            std::size_t sent = 0;
            for (const auto& sh : shards) sent += sh.plan.local_count - sh.plan.chunk_size(sh.plan.worker_id);
            RecordingTransport transport(n);
            const auto out = wfc::exchange(shards, transport);
            for (const auto& o : out) {
                CHECK(o.sorted && std::is_sorted(o.words.begin(), o.words.end()));
                for (const auto& w : o.words) ++after[w];
            }
            CHECK(before == after);
            CHECK(transport.frames.size() == n * (n - 1));
            std::size_t decoded = 0;
            for (const auto& f : transport.frames) decoded += decode_message(f).size();
            CHECK(decoded == sent);
            const auto again = wfc::exchange(shards);
            for (std::size_t j = 0; j < n; ++j) CHECK(again[j].words == out[j].words);
        }
    }
    // shuffle_test.cpp:257-279 -- failures name the pair / the worker; layout validation
    {
        const auto shards = make_shards({sorted_list({"a", "b"}), sorted_list({"c", "d"})});
        FailingTransport failing;
        CHECK(throws_with<ExchangeError>([&] { wfc::exchange(shards, failing); }, "worker 0 -> worker 1"));
        CorruptingTransport corrupting(2, 0);
        CHECK(throws_with<ExchangeError>([&] { wfc::exchange(shards, corrupting); }, "worker 0 got an invalid frame from worker 1"));
        const WordList list = sorted_list({"a"});
        std::vector<WorkerShard> bad;
        bad.push_back({plan_partition(list, 0, 3), list});
        CHECK_THROWS_AS(wfc::exchange(bad), std::invalid_argument);
        CHECK_THROWS_AS(wfc::exchange(std::vector<WorkerShard>{}), std::invalid_argument);
        CHECK_THROWS_AS(InProcessTransport(0), TransportError);
    }
    // pipeline_test.cpp:106-127, 162-175 -- the transport overload: same counts, the reference's pre-repair shards,
    // and a failure inside the exchange is attributed to its stage
    {
        InProcessTransport transport(2);
        const RunResult r = run_wordcount(kTwoDocs, 2, transport);
        CHECK(r.counts == serial_wordcount(kTwoDocs));
        CHECK(r.pre_repair_shards.size() == 2 && r.pre_repair_shards[0].count("mapreduce") && r.pre_repair_shards[1].count("mapreduce"));
        CHECK(count_unreduced_words(r.pre_repair_shards) == 1 && count_unreduced_words(r.shards) == 0);
        Rng rng(303);
        const auto corpus = iid_corpus(rng, 20, 200, 80);
        for (std::size_t n : {1, 3, 8}) {
            RecordingTransport rec(n);
            const RunResult rr = run_wordcount(corpus, n, rec);
            CHECK(rr.counts == serial_wordcount(corpus));
            CHECK(rec.frames.size() == n * (n - 1));
        }
        CorruptingTransport broken(2, ~std::size_t(0));
        bool attributed = false;
        try {
            run_wordcount(kTwoDocs, 2, broken);
        } catch (const PipelineError& e) {
            const std::string what = e.what();
            attributed = e.stage() == "exchange" && what.find("exchange stage") != std::string::npos &&
                         what.find("invalid frame") != std::string::npos;
        }
        CHECK(attributed);
    }
}

static void code_point_cases() {
    // text_test.cpp:171-187 and unicode.cpp's pinned classes, through the per-code-point accessors
    CHECK(utf8_decode("a", 0).valid && utf8_decode("a", 0).cp == U'a' && utf8_decode("a", 0).length == 1);
    const std::string e_acute = "\xc3\xa9", kanji = "\xe6\xbc\xa2", emoji = "\xf0\x9f\x98\x80";
    CHECK(utf8_decode(e_acute, 0).cp == 0xE9 && utf8_decode(e_acute, 0).length == 2);
    CHECK(utf8_decode(kanji, 0).cp == 0x6F22 && utf8_decode(kanji, 0).length == 3);
    CHECK(utf8_decode(emoji, 0).cp == 0x1F600 && utf8_decode(emoji, 0).length == 4);
    for (const std::string bad : {"\xff", "\xc0\x80", "\xe0\x80\x80", "\xed\xa0\x80", "\xf4\x90\x80\x80", "\xc3", "\xe6\xbc", "\x80"}) {
        const DecodedChar d = utf8_decode(bad, 0);
        CHECK(!d.valid && d.length == 1 && d.cp == kReplacementChar);
    }
    for (char32_t cp : {char32_t(0x24), char32_t(0xE9), char32_t(0x6F22), char32_t(0x1F600), char32_t(0x7FF), char32_t(0x800), char32_t(0xFFFF), char32_t(0x10FFFF)}) {
        std::string s;
        utf8_append(s, cp);
        const DecodedChar d = utf8_decode(s, 0);
        CHECK(d.valid && d.cp == cp && d.length == s.size());
        CHECK(utf8_valid(s));                                        // the device validator agrees
    }
    for (char32_t cp : {0x09, 0x0D, 0x20, 0x85, 0xA0, 0x1680, 0x2000, 0x200A, 0x2028, 0x2029, 0x202F, 0x205F, 0x3000}) CHECK(is_unicode_space(cp));
    for (char32_t cp : {0x08, 0x0E, 0x1F, 0x21, 0x84, 0x200B, 0x2060, 0x3001, 0xFEFF}) CHECK(!is_unicode_space(cp));
    for (char32_t cp : {U'0', U'9', U'a', U'Z', char32_t(0xAA), char32_t(0xB5), char32_t(0xBA), char32_t(0xC0), char32_t(0x80), char32_t(0x3B1), char32_t(0x6F22), char32_t(0x2070), char32_t(0x3040), char32_t(0xFF10), char32_t(0xFF21), char32_t(0xFF66), char32_t(0x1F600)})
        CHECK(is_word_char(cp));
    for (char32_t cp : {U'_', U'-', U'\'', U' ', char32_t(0x7F), char32_t(0x85), char32_t(0xA0), char32_t(0xA1), char32_t(0xBF), char32_t(0xD7), char32_t(0xF7), char32_t(0x2019), char32_t(0x206F), char32_t(0x3000), char32_t(0x303F), char32_t(0xFF01), char32_t(0xFF0F), char32_t(0xFF1A), char32_t(0xFF20), char32_t(0xFF3B), char32_t(0xFF40), char32_t(0xFF5B), char32_t(0xFF65), char32_t(0xFFFD), char32_t(0x1680)})
        CHECK(!is_word_char(cp));
    CHECK(simple_lower(U'A') == U'a' && simple_lower(U'Z') == U'z' && simple_lower(U'a') == U'a' && simple_lower(U'0') == U'0');
    CHECK(simple_lower(0xC0) == 0xE0 && simple_lower(0xDE) == 0xFE && simple_lower(0xD7) == 0xD7 && simple_lower(0xDF) == 0xDF);
    CHECK(simple_lower(0x391) == 0x391 && simple_lower(0x178) == 0x178);
    // the accessors and the device tokenizer agree: a word character survives normalize_word, anything else is trimmed
    for (char32_t cp : {char32_t(0xAA), char32_t(0xD7), char32_t(0x2019), char32_t(0x6F22), char32_t(0xFF0F), char32_t(0xFF10), char32_t(0x80), char32_t(0x3B1)}) {
        std::string s;
        utf8_append(s, cp);
        if (is_unicode_space(cp)) continue;
        const auto w = normalize_word(s);
        CHECK(w.has_value() == is_word_char(cp));
    }
}

int main() {
    try {
        text_cases();
        unicode_cases();
        reduce_cases();
        pipeline_cases();
        range_partition_cases();
        wire_cases();
        shuffle_cases();
        code_point_cases();
        engine_cases();
        analysis_cases();
        report_cases();
    } catch (const std::exception& e) {
        std::printf("FAILED with exception: %s\n", e.what());
        return 2;
    }
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
