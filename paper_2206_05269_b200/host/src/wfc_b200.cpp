// wfc_b200.cpp -- the reference's wfc:: API implemented over the C ABI of libwfcu.so.
//
// Host code here only marshals std::string / std::map values into packed buffers and
// back, maps status codes to the reference's exception types and keeps the containers'
// bookkeeping (shard lists, top-k ordering).  Tokenizing, counting, sorting, run-length
// encoding, partitioning, merging and every floating-point sum run on the GPU.
#include "wfc/wfc_b200.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <unordered_map>

#include "wfcu.h"

namespace wfc {

namespace {

[[noreturn]] void raise(int rc, const char* stage = nullptr) {
    const std::string msg = wfcu_last_error();
    if (rc == WFCU_ERR_INVALID_ARGUMENT || rc == WFCU_ERR_NOT_SORTED) throw std::invalid_argument(msg);
    if (stage) throw PipelineError(stage, msg);
    throw DeviceError(msg);
}
inline void ok(int rc, const char* stage = nullptr) {
    if (rc != WFCU_OK) raise(rc, stage);
}

struct Packed {
    std::vector<std::uint8_t> bytes;
    std::vector<std::uint32_t> lens;
};

template <typename Range>
Packed pack(const Range& words) {
    Packed p;
    std::size_t total = 0;
    for (const auto& w : words) total += w.size();
    p.bytes.reserve(total);
    p.lens.reserve(words.size());
    for (const auto& w : words) {
        p.bytes.insert(p.bytes.end(), w.begin(), w.end());
        p.lens.push_back(std::uint32_t(w.size()));
    }
    return p;
}

std::vector<Word> unpack(const std::uint8_t* bytes, const std::uint32_t* lens, std::size_t n) {
    std::vector<Word> out;
    out.reserve(n);
    std::size_t off = 0;
    for (std::size_t i = 0; i < n; ++i) {
        out.emplace_back(reinterpret_cast<const char*>(bytes + off), lens[i]);
        off += lens[i];
    }
    return out;
}

struct CounterHandle {
    wfcu_counter* h = nullptr;
    explicit CounterHandle(std::uint64_t expected_keys = 0, const char* stage = nullptr) {
        wfcu_counter_config cfg{};
        std::uint64_t slots = 1u << 16;
        while (slots < 4 * expected_keys) slots <<= 1;
        cfg.table_slots = slots;
        cfg.deferred_slots = std::max<std::uint64_t>(1u << 16, expected_keys);
        cfg.long_slots = 1u << 16;
        cfg.arena_bytes = 16u << 20;
        ok(wfcu_counter_create(&h, &cfg), stage);
    }
    ~CounterHandle() { wfcu_counter_destroy(h); }
    CounterHandle(const CounterHandle&) = delete;
    CounterHandle& operator=(const CounterHandle&) = delete;
};

struct TokensHandle {
    wfcu_tokens* h = nullptr;
    ~TokensHandle() { wfcu_tokens_destroy(h); }
};

CountMap export_counts(wfcu_counter* c, const char* stage = nullptr) {
    std::uint64_t distinct = 0, total = 0, key_bytes = 0;
    ok(wfcu_counter_stats(c, nullptr, &distinct, &total, &key_bytes), stage);
    std::vector<std::uint8_t> bytes(key_bytes + 1);
    std::vector<std::uint32_t> lens(distinct + 1);
    std::vector<std::uint64_t> counts(distinct + 1);
    ok(wfcu_counter_export(c, nullptr, bytes.data(), key_bytes, lens.data(), counts.data(), distinct), stage);
    CountMap m;
    std::size_t off = 0;
    for (std::uint64_t i = 0; i < distinct; ++i) {   // export is in map order: hinted insert is O(1)
        m.emplace_hint(m.end(), Word(reinterpret_cast<const char*>(bytes.data() + off), lens[i]), counts[i]);
        off += lens[i];
    }
    return m;
}

void add_map(wfcu_counter* c, const CountMap& m) {
    if (m.empty()) return;
    Packed p;
    std::vector<std::uint64_t> counts;
    counts.reserve(m.size());
    for (const auto& [w, n] : m) {
        p.bytes.insert(p.bytes.end(), w.begin(), w.end());
        p.lens.push_back(std::uint32_t(w.size()));
        counts.push_back(n);
    }
    ok(wfcu_counter_add_words(c, p.bytes.data(), p.lens.data(), counts.data(), m.size()));
}

// Capacity errors are not the caller's problem: retry with a larger table.
template <typename Fn>
void with_growing_counter(std::uint64_t hint, const char* stage, Fn&& fn) {
    for (int attempt = 0;; ++attempt) {
        CounterHandle c(hint, stage);
        const int rc = fn(c.h);
        if (rc == WFCU_OK) return;
        const bool capacity = rc == WFCU_ERR_TABLE_FULL || rc == WFCU_ERR_DEFERRED_FULL || rc == WFCU_ERR_ARENA_FULL;
        if (!capacity || attempt >= 6) raise(rc, stage);
        hint = std::max<std::uint64_t>(hint, 1u << 14) * 8;
    }
}

std::uint64_t total_bytes(std::span<const RawDocument> corpus) {
    std::uint64_t n = 0;
    for (const auto& d : corpus) n += d.text.size();
    return n;
}

int wfcu_kind(MapKind map) {
    switch (map) {
        case MapKind::identity: return WFCU_MAP_IDENTITY;
        case MapKind::square_root: return WFCU_MAP_SQUARE_ROOT;
        case MapKind::alternating_harmonic_term: return WFCU_MAP_ALTERNATING_HARMONIC_TERM;
        case MapKind::square: return WFCU_MAP_SQUARE;
    }
    throw std::invalid_argument("unknown map kind");
}

using Clock = std::chrono::steady_clock;
std::uint64_t since(Clock::time_point t0) {
    return std::uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
}

}  // namespace

// ---- unicode --------------------------------------------------------------------------------
std::string utf8_sanitize(std::string_view text) {   // proj/src/unicode.cpp:56-70
    std::string out(3 * text.size() + 16, '\0');
    std::uint64_t n = 0;
    ok(wfcu_utf8_sanitize_host(reinterpret_cast<const std::uint8_t*>(text.data()), text.size(),
                               reinterpret_cast<std::uint8_t*>(out.data()), out.size(), &n));
    out.resize(n);
    return out;
}

bool utf8_valid(std::string_view text) {   // proj/src/unicode.cpp:46-54: every replacement adds two bytes
    return utf8_sanitize(text).size() == text.size();
}

// ---- text ---------------------------------------------------------------------------------
std::vector<std::optional<Word>> normalize_words(std::span<const std::string> fragments) {
    const Packed p = pack(fragments);
    std::vector<std::uint8_t> out(3 * p.bytes.size() + 16);
    std::vector<std::uint32_t> out_lens(fragments.size() + 1);
    ok(wfcu_normalize_words_host(p.bytes.data(), p.lens.data(), fragments.size(), out.data(), out.size(), out_lens.data()));
    std::vector<std::optional<Word>> res(fragments.size());
    std::size_t off = 0;
    for (std::size_t i = 0; i < fragments.size(); ++i) {
        if (out_lens[i]) res[i] = Word(reinterpret_cast<const char*>(out.data() + off), out_lens[i]);
        off += out_lens[i];
    }
    return res;
}

std::optional<Word> normalize_word(std::string_view fragment) {
    const std::string one(fragment);
    return normalize_words(std::span<const std::string>(&one, 1))[0];
}

WordList tokenize(const RawDocument& doc) {
    TokensHandle t;
    ok(wfcu_tokenize_host(reinterpret_cast<const std::uint8_t*>(doc.text.data()), doc.text.size(), &t.h));
    std::uint64_t n = 0, nb = 0;
    ok(wfcu_tokens_stats(t.h, &n, &nb));
    std::vector<std::uint8_t> bytes(nb + 1);
    std::vector<std::uint32_t> lens(n + 1);
    ok(wfcu_tokens_export(t.h, bytes.data(), nb, lens.data(), n));
    WordList list;
    list.words = unpack(bytes.data(), lens.data(), n);
    return list;
}

WordList sort_words(WordList list) {
    if (!list.words.empty()) {
        const Packed p = pack(list.words);
        TokensHandle t;
        ok(wfcu_tokens_from_words(p.bytes.data(), p.lens.data(), list.words.size(), &t.h));
        ok(wfcu_tokens_sort(t.h, nullptr));
        std::vector<std::uint8_t> bytes(p.bytes.size() + 1);
        std::vector<std::uint32_t> lens(p.lens.size() + 1);
        ok(wfcu_tokens_export(t.h, bytes.data(), p.bytes.size(), lens.data(), p.lens.size()));
        list.words = unpack(bytes.data(), lens.data(), p.lens.size());
    }
    list.sorted = true;
    return list;
}

// ---- reduce -------------------------------------------------------------------------------
CountMap reduce_sorted(const WordList& sorted) {
    if (!sorted.sorted) throw std::invalid_argument("reduce_sorted: word list must be sorted");
    if (sorted.words.empty()) return {};
    for (const auto& w : sorted.words)
        if (w.empty()) throw std::invalid_argument("reduce_sorted: empty word");
    const Packed p = pack(sorted.words);
    TokensHandle t;
    ok(wfcu_tokens_from_words(p.bytes.data(), p.lens.data(), sorted.words.size(), &t.h));
    CountMap result;
    with_growing_counter(sorted.words.size(), nullptr, [&](wfcu_counter* c) {
        int rc = wfcu_tokens_reduce_sorted(t.h, c, nullptr);
        if (rc == WFCU_OK) rc = wfcu_counter_status(c, nullptr);
        if (rc == WFCU_OK) result = export_counts(c);
        return rc;
    });
    return result;
}

CountMap merge_counts(std::span<const CountMap> maps) {
    std::uint64_t keys = 0;
    for (const auto& m : maps) keys += m.size();
    if (keys == 0) return {};
    CountMap result;
    with_growing_counter(keys, nullptr, [&](wfcu_counter* c) {
        for (const auto& m : maps) add_map(c, m);
        const int rc = wfcu_counter_status(c, nullptr);
        if (rc == WFCU_OK) result = export_counts(c);
        return rc;
    });
    return result;
}

// Container bookkeeping over std::map shards (no arithmetic beyond adding the counts of
// a duplicated key): every word ends up with its lowest-indexed holder.
ShardedCounts boundary_repair(ShardedCounts sharded) {
    std::unordered_map<std::string_view, std::size_t> holder;
    for (std::size_t s = 0; s < sharded.size(); ++s) {
        for (auto it = sharded[s].begin(); it != sharded[s].end();) {
            const auto [pos, fresh] = holder.try_emplace(std::string_view(it->first), s);
            if (fresh) {
                ++it;
            } else {
                sharded[pos->second].find(it->first)->second += it->second;
                it = sharded[s].erase(it);
            }
        }
    }
    return sharded;
}

std::size_t count_unreduced_words(const ShardedCounts& sharded) {
    std::unordered_map<std::string_view, unsigned> holders;
    for (const auto& shard : sharded)
        for (const auto& kv : shard) ++holders[std::string_view(kv.first)];
    std::size_t n = 0;
    for (const auto& kv : holders) n += kv.second > 1;
    return n;
}

// ---- pipeline -----------------------------------------------------------------------------
CountMap serial_wordcount(std::span<const RawDocument> corpus) {
    if (corpus.empty()) return {};
    std::vector<const std::uint8_t*> ptrs;
    std::vector<std::uint64_t> lens;
    for (const auto& d : corpus) {
        ptrs.push_back(reinterpret_cast<const std::uint8_t*>(d.text.data()));
        lens.push_back(d.text.size());
    }
    CountMap result;
    with_growing_counter(total_bytes(corpus) / 64, nullptr, [&](wfcu_counter* c) {
        const int rc = wfcu_counter_count_host(c, ptrs.data(), lens.data(), ptrs.size());
        if (rc == WFCU_OK) result = export_counts(c);
        return rc;
    });
    return result;
}

static RunResult run_range_partitioned(std::span<const RawDocument> corpus, std::size_t n_workers, Transport& transport);

namespace {
// a stage of the pipeline: device time between two CUDA events (wfcu_timer), exceptions wrapped like
// the reference's timed_stage (pipeline.cpp:48-57)
struct StageTimer {
    wfcu_timer* t = nullptr;
    StageTimer() { ok(wfcu_timer_create(&t)); }
    ~StageTimer() { wfcu_timer_destroy(t); }
    template <typename Fn>
    void run(const char* name, std::uint64_t& ns, Fn&& fn) {
        ok(wfcu_timer_start(t), name);
        try {
            fn();
        } catch (const std::invalid_argument&) {
            throw;
        } catch (const PipelineError&) {
            throw;
        } catch (const std::exception& e) {
            throw PipelineError(name, e.what());
        }
        ok(wfcu_timer_stop_ns(t, &ns), name);
    }
};

RunResult empty_run(std::size_t n_workers, Clock::time_point run_start) {
    RunResult result;
    result.n_workers = n_workers;
    result.shards.assign(n_workers, CountMap{});
    result.pre_repair_shards = result.shards;
    result.timings.total_ns = since(run_start);
    return result;
}

// cut indices of the reference's range partition for a sorted list of k words (shuffle.cpp:17-45)
std::vector<std::uint64_t> partition_cuts(std::uint64_t k, std::size_t worker_id, std::size_t n) {
    const std::uint64_t keep = k / n, others = n > 1 ? n - 1 : 1;
    const std::uint64_t base = n > 1 ? (k - keep) / others : 0;
    std::uint64_t extra = n > 1 ? (k - keep) % others : 0;
    std::vector<std::uint64_t> cut(n + 1, 0);
    for (std::size_t c = 0; c < n; ++c) {
        std::uint64_t size = keep;
        if (c != worker_id) {
            size = base + (extra ? 1 : 0);
            if (extra) --extra;
        }
        cut[c + 1] = cut[c] + size;
    }
    return cut;
}
}  // namespace

// The reference's pipeline (pipeline.cpp:61-123), every stage in device memory: worker j tokenizes the documents
// d = j (mod n) and radix-sorts its tokens; the range partition is index arithmetic on the list lengths; the exchange
// gathers chunk c of every list into worker c's list (wfcu_tokens_concat_slices: device-to-device copies, no frame,
// no host string); the n-way merge is one more radix sort; reduce is the run-length encode into a count table.
// Only the per-shard maps come back to the host, where boundary_repair moves the (at most n-1) duplicated boundary
// words to their lowest-indexed holder.
RunResult run_wordcount(std::span<const RawDocument> corpus, std::size_t n_workers) {
    if (n_workers == 0) throw std::invalid_argument("run_wordcount: n_workers must be >= 1");
    const auto run_start = Clock::now();
    if (corpus.empty()) return empty_run(n_workers, run_start);
    const std::size_t n = n_workers;
    RunResult result;
    result.n_workers = n;
    auto& t = result.timings;
    StageTimer timer;
    std::vector<TokensHandle> local(n), received(n);
    timer.run("map", t.map_ns, [&] {
        // worker j's documents, gathered on the device (a newline ends every document's last fragment)
        std::vector<const std::uint8_t*> ptrs;
        std::vector<std::uint64_t> lens;
        for (std::size_t j = 0; j < n; ++j) {
            ptrs.clear();
            lens.clear();
            for (std::size_t d = j; d < corpus.size(); d += n) {
                ptrs.push_back(reinterpret_cast<const std::uint8_t*>(corpus[d].text.data()));
                lens.push_back(corpus[d].text.size());
            }
            ok(wfcu_tokenize_docs_host(ptrs.data(), lens.data(), ptrs.size(), &local[j].h), "map");
        }
    });
    timer.run("sort", t.sort_ns, [&] {
        for (auto& l : local) ok(wfcu_tokens_sort(l.h, nullptr), "sort");
    });
    std::vector<std::vector<std::uint64_t>> cuts(n);
    timer.run("encode", t.encode_ns, [&] {
        for (std::size_t j = 0; j < n; ++j) {
            std::uint64_t k = 0;
            ok(wfcu_tokens_stats(local[j].h, &k, nullptr), "encode");
            cuts[j] = partition_cuts(k, j, n);
        }
    });
    timer.run("exchange", t.exchange_ns, [&] {
        std::vector<const wfcu_tokens*> src(n);
        std::vector<std::uint64_t> begin(n), end(n);
        for (std::size_t j = 0; j < n; ++j) src[j] = local[j].h;
        for (std::size_t c = 0; c < n; ++c) {
            for (std::size_t j = 0; j < n; ++j) { begin[j] = cuts[j][c]; end[j] = cuts[j][c + 1]; }
            ok(wfcu_tokens_concat_slices(src.data(), begin.data(), end.data(), std::uint32_t(n), &received[c].h), "exchange");
            ok(wfcu_tokens_sort(received[c].h, nullptr), "exchange");       // the n-way merge
        }
    });
    result.pre_repair_shards.assign(n, CountMap{});
    timer.run("reduce", t.reduce_ns, [&] {
        for (std::size_t c = 0; c < n; ++c) {
            std::uint64_t k = 0;
            ok(wfcu_tokens_stats(received[c].h, &k, nullptr), "reduce");
            if (k == 0) continue;
            with_growing_counter(k, "reduce", [&](wfcu_counter* counter) {
                int rc = wfcu_tokens_reduce_sorted(received[c].h, counter, nullptr);
                if (rc == WFCU_OK) rc = wfcu_counter_status(counter, nullptr);
                if (rc == WFCU_OK) result.pre_repair_shards[c] = export_counts(counter, "reduce");
                return rc;
            });
        }
    });
    const auto repair_start = Clock::now();      // host bookkeeping over at most n-1 boundary words
    result.shards = boundary_repair(result.pre_repair_shards);
    t.repair_ns = since(repair_start);
    for (const auto& shard : result.shards) result.counts.insert(shard.begin(), shard.end());
    t.total_ns = since(run_start);
    return result;
}

// BASELINE.json's path: fused tokenize/count kernels per worker, tables hash-partitioned by owner and delivered
// device to device over the GPUs of the box (wfcu_wordcount_multi); stage times are CUDA-event times.
RunResult run_wordcount_hashed(std::span<const RawDocument> corpus, std::size_t n_workers) {
    if (n_workers == 0) throw std::invalid_argument("run_wordcount: n_workers must be >= 1");
    const auto run_start = Clock::now();
    if (corpus.empty()) return empty_run(n_workers, run_start);
    const std::size_t n = n_workers;
    RunResult result;
    result.n_workers = n;
    std::vector<const std::uint8_t*> ptrs;
    std::vector<std::uint64_t> lens;
    for (const auto& d : corpus) {
        ptrs.push_back(reinterpret_cast<const std::uint8_t*>(d.text.data()));
        lens.push_back(d.text.size());
    }
    std::uint64_t hint = total_bytes(corpus) / 64 / n + 1024;
    for (int attempt = 0;; ++attempt) {
        wfcu_counter_config cfg{};
        std::uint64_t slots = 1u << 16;
        while (slots < 4 * hint) slots <<= 1;
        cfg.table_slots = slots;
        cfg.deferred_slots = std::max<std::uint64_t>(1u << 16, hint);
        cfg.long_slots = 1u << 16;
        cfg.arena_bytes = 16u << 20;
        std::vector<wfcu_counter*> owned(n, nullptr);
        wfcu_stage_ns ns{};
        const int rc = wfcu_wordcount_multi(ptrs.data(), lens.data(), ptrs.size(), std::uint32_t(n), &cfg, owned.data(), &ns);
        if (rc != WFCU_OK) {
            const bool capacity = rc == WFCU_ERR_TABLE_FULL || rc == WFCU_ERR_DEFERRED_FULL || rc == WFCU_ERR_ARENA_FULL;
            if (!capacity || attempt >= 5) raise(rc, "map");
            hint *= 8;
            continue;
        }
        struct Release {
            std::vector<wfcu_counter*>& v;
            ~Release() { for (auto* c : v) wfcu_counter_destroy(c); }
        } release{owned};
        result.timings.map_ns = ns.map_ns;
        result.timings.encode_ns = ns.encode_ns;
        result.timings.exchange_ns = ns.exchange_ns;
        const auto t0 = Clock::now();
        for (std::size_t p = 0; p < n; ++p) result.shards.push_back(export_counts(owned[p], "reduce"));
        result.timings.reduce_ns = since(t0);
        break;
    }
    result.pre_repair_shards = result.shards;   // disjoint by construction: nothing to repair
    for (const auto& shard : result.shards) result.counts.insert(shard.begin(), shard.end());
    result.timings.total_ns = since(run_start);
    return result;
}

// The caller's transport carries the chunks as WCX1 frames (pipeline.cpp:61-123 with a custom Transport).
RunResult run_wordcount(std::span<const RawDocument> corpus, std::size_t n_workers, Transport& transport) {
    return run_range_partitioned(corpus, n_workers, transport);
}

// Chunk sizes: the kept chunk gets floor(k/n); the rest is spread over the other chunks,
// one extra each from chunk 0 upward (reference rule, shuffle.cpp:17-45).  Index arithmetic only.
ShardPlan plan_partition(const WordList& sorted, std::size_t worker_id, std::size_t n_workers) {
    if (n_workers == 0) throw std::invalid_argument("plan_partition: n_workers must be >= 1");
    if (worker_id >= n_workers)
        throw std::invalid_argument("plan_partition: worker_id " + std::to_string(worker_id) + " out of range for " +
                                    std::to_string(n_workers) + " workers");
    if (!sorted.sorted) throw std::invalid_argument("plan_partition: word list must be sorted");
    const std::vector<std::uint64_t> cut = partition_cuts(sorted.words.size(), worker_id, n_workers);
    ShardPlan plan{worker_id, n_workers, sorted.words.size(), std::vector<std::size_t>(cut.begin(), cut.end())};
    return plan;
}

RunResult run_wordcount_range_partitioned(std::span<const RawDocument> corpus, std::size_t n_workers) {
    return run_wordcount(corpus, n_workers);
}

static RunResult run_range_partitioned(std::span<const RawDocument> corpus, std::size_t n_workers, Transport& transport) {
    if (n_workers == 0) throw std::invalid_argument("run_wordcount: n_workers must be >= 1");
    const auto run_start = Clock::now();
    RunResult result;
    result.n_workers = n_workers;
    const std::size_t n = n_workers;
    if (corpus.empty()) {
        result.shards.assign(n, CountMap{});
        result.pre_repair_shards = result.shards;
        result.timings.total_ns = since(run_start);
        return result;
    }
    auto& t = result.timings;
    auto stage = [&](const char* name, std::uint64_t& ns, auto&& fn) {
        const auto t0 = Clock::now();
        try {
            fn();
        } catch (const std::invalid_argument&) {
            throw;
        } catch (const std::exception& e) {
            throw PipelineError(name, e.what());
        }
        ns = since(t0);
    };
    std::vector<WordList> local(n);
    stage("map", t.map_ns, [&] {          // device tokenizer, documents d = j (mod n)
        for (std::size_t j = 0; j < n; ++j)
            for (std::size_t d = j; d < corpus.size(); d += n) {
                WordList w = tokenize(corpus[d]);
                local[j].words.insert(local[j].words.end(), std::make_move_iterator(w.words.begin()),
                                      std::make_move_iterator(w.words.end()));
            }
    });
    stage("sort", t.sort_ns, [&] {        // device radix sort
        for (auto& l : local) l = sort_words(std::move(l));
    });
    std::vector<EncodedShard> shards(n);
    stage("encode", t.encode_ns, [&] {    // range partition by position, one WCX1 frame per peer
        for (std::size_t j = 0; j < n; ++j) shards[j] = encode_outgoing(plan_partition(local[j], j, n), local[j]);
    });
    std::vector<WordList> exchanged;
    stage("exchange", t.exchange_ns, [&] {   // n concurrent workers over the transport, n-way merge
        exchanged = exchange_encoded(std::move(shards), transport);
    });
    result.pre_repair_shards.assign(n, CountMap{});
    stage("reduce", t.reduce_ns, [&] {    // device run-length encode
        for (std::size_t j = 0; j < n; ++j) result.pre_repair_shards[j] = reduce_sorted(exchanged[j]);
    });
    stage("repair", t.repair_ns, [&] { result.shards = boundary_repair(result.pre_repair_shards); });
    result.counts = merge_counts(result.shards);
    t.total_ns = since(run_start);
    return result;
}

// ---- engine -------------------------------------------------------------------------------
double map_reduce_serial(std::span<const double> values, MapKind map) {
    // the left-to-right fold, bit for bit: one block covering the whole array
    if (values.empty()) return 0.0;
    double out = 0.0;
    ok(wfcu_map_reduce_blocked_host(values.data(), WFCU_DTYPE_F64, values.size(), wfcu_kind(map), values.size(), &out));
    return out;
}

double map_reduce_blocked(std::span<const double> values, MapKind map, const BlockConfig& cfg) {
    if (cfg.block_size == 0 || cfg.workers == 0) throw std::invalid_argument("block_size and workers must be >= 1");
    double out = 0.0;
    ok(wfcu_map_reduce_blocked_host(values.data(), WFCU_DTYPE_F64, values.size(), wfcu_kind(map), cfg.block_size, &out));
    return out;
}

double alternating_harmonic(std::uint64_t n, const BlockConfig& cfg) {
    if (cfg.block_size == 0 || cfg.workers == 0) throw std::invalid_argument("block_size and workers must be >= 1");
    double out = 0.0;
    ok(wfcu_alternating_harmonic(n, cfg.block_size, &out));
    return out;
}

double map_reduce_fast(std::span<const double> values, MapKind map) {
    double out = 0.0;
    ok(wfcu_map_reduce_host(values.data(), WFCU_DTYPE_F64, values.size(), wfcu_kind(map), &out));
    return out;
}

double map_reduce_fast(std::span<const float> values, MapKind map) {
    double out = 0.0;
    ok(wfcu_map_reduce_host(values.data(), WFCU_DTYPE_F32, values.size(), wfcu_kind(map), &out));
    return out;
}

// ---- analysis -----------------------------------------------------------------------------
// The order of the rows -- count / score descending, word ascending, the reference's log expression -- has ONE
// implementation, in libwfcu (csrc/analysis.cpp: wfcu_top_k, wfcu_distinctive and the device entry points end in it).
namespace {
struct PackedTable {
    Packed keys;
    std::vector<std::uint64_t> counts;
    std::vector<const Word*> words;
};
PackedTable pack_table(const CountMap& m) {
    PackedTable p;
    p.counts.reserve(m.size());
    p.words.reserve(m.size());
    for (const auto& [w, c] : m) {
        p.keys.bytes.insert(p.keys.bytes.end(), w.begin(), w.end());
        p.keys.lens.push_back(std::uint32_t(w.size()));
        p.counts.push_back(c);
        p.words.push_back(&w);
    }
    return p;
}
}  // namespace

FrequencyTable top_k(const CountMap& counts, std::string label, std::size_t k) {
    FrequencyTable table;
    table.label = std::move(label);
    const PackedTable p = pack_table(counts);
    const std::size_t cap = std::min(k, counts.size());
    std::vector<std::uint64_t> idx(cap + 1);
    std::vector<double> rel(cap + 1);
    std::uint64_t rows = 0;
    ok(wfcu_top_k(p.keys.bytes.data(), p.keys.lens.data(), p.counts.data(), counts.size(), k, idx.data(), rel.data(),
                  &table.total_words, &rows));
    for (std::uint64_t r = 0; r < rows; ++r) table.rows.push_back({*p.words[idx[r]], p.counts[idx[r]], rel[r]});
    return table;
}

DistinctivenessReport distinctive_words(const CountMap& target, const CountMap& others, std::string label,
                                        std::size_t k) {
    DistinctivenessReport report;
    report.label = std::move(label);
    if (target.empty() && others.empty()) return report;
    const PackedTable t = pack_table(target), o = pack_table(others);
    const std::size_t cap = std::min(k, target.size() + others.size());
    std::vector<std::int32_t> src(cap + 1);
    std::vector<std::uint64_t> idx(cap + 1);
    std::vector<double> score(cap + 1);
    std::uint64_t rows = 0;
    ok(wfcu_distinctive(t.keys.bytes.data(), t.keys.lens.data(), t.counts.data(), target.size(), o.keys.bytes.data(),
                        o.keys.lens.data(), o.counts.data(), others.size(), k, src.data(), idx.data(), score.data(), &rows));
    for (std::uint64_t r = 0; r < rows; ++r) report.rows.push_back({*(src[r] ? o : t).words[idx[r]], score[r]});
    return report;
}

// ---- tables that stay on the device -----------------------------------------------------------
DeviceCounts::DeviceCounts(std::uint64_t expected_distinct_words) {
    wfcu_counter_config cfg{};
    std::uint64_t slots = 1u << 16;
    while (slots < 4 * expected_distinct_words) slots <<= 1;
    cfg.table_slots = slots;
    cfg.deferred_slots = std::max<std::uint64_t>(1u << 20, expected_distinct_words);
    cfg.long_slots = 1u << 16;
    cfg.arena_bytes = 16u << 20;
    ok(wfcu_counter_create(&h_, &cfg));
}
DeviceCounts::~DeviceCounts() { wfcu_counter_destroy(h_); }
DeviceCounts::DeviceCounts(DeviceCounts&& other) noexcept : h_(other.h_) { other.h_ = nullptr; }
DeviceCounts& DeviceCounts::operator=(DeviceCounts&& other) noexcept {
    if (this != &other) {
        wfcu_counter_destroy(h_);
        h_ = other.h_;
        other.h_ = nullptr;
    }
    return *this;
}
void DeviceCounts::count(std::span<const RawDocument> corpus) {
    std::vector<const std::uint8_t*> ptrs;
    std::vector<std::uint64_t> lens;
    for (const auto& d : corpus) {
        ptrs.push_back(reinterpret_cast<const std::uint8_t*>(d.text.data()));
        lens.push_back(d.text.size());
    }
    ok(wfcu_counter_count_host(h_, ptrs.data(), lens.data(), ptrs.size()), "map");
}
void DeviceCounts::merge(const DeviceCounts& other) {
    ok(wfcu_counter_merge(h_, other.h_, nullptr));
    ok(wfcu_counter_status(h_, nullptr));
}
std::uint64_t DeviceCounts::distinct_words() const {
    std::uint64_t distinct = 0;
    ok(wfcu_counter_stats(h_, nullptr, &distinct, nullptr, nullptr));
    return distinct;
}
std::uint64_t DeviceCounts::total_words() const {
    std::uint64_t total = 0;
    ok(wfcu_counter_stats(h_, nullptr, nullptr, &total, nullptr));
    return total;
}
CountMap DeviceCounts::to_map() const { return export_counts(h_); }

FrequencyTable DeviceCounts::top_k(std::string label, std::size_t k) const {
    FrequencyTable table;
    table.label = std::move(label);
    const std::size_t cap = std::min<std::uint64_t>(k, distinct_words());
    std::vector<std::uint8_t> bytes(64 * cap + 4096);
    std::vector<std::uint32_t> lens(cap + 1);
    std::vector<std::uint64_t> counts(cap + 1);
    std::vector<double> rel(cap + 1);
    std::uint64_t rows = 0;
    ok(wfcu_counter_top_k(h_, k, nullptr, bytes.data(), bytes.size(), lens.data(), counts.data(), rel.data(), cap + 1, &rows,
                          &table.total_words));
    const std::vector<Word> words = unpack(bytes.data(), lens.data(), rows);
    for (std::uint64_t r = 0; r < rows; ++r) table.rows.push_back({words[r], counts[r], rel[r]});
    return table;
}

DistinctivenessReport DeviceCounts::distinctive(const DeviceCounts& others, std::string label, std::size_t k) const {
    DistinctivenessReport report;
    report.label = std::move(label);
    const std::size_t cap = std::min<std::uint64_t>(k, distinct_words() + others.distinct_words());
    std::vector<std::uint8_t> bytes(64 * cap + 4096);
    std::vector<std::uint32_t> lens(cap + 1);
    std::vector<double> score(cap + 1);
    std::uint64_t rows = 0;
    ok(wfcu_counter_distinctive(h_, others.h_, k, nullptr, bytes.data(), bytes.size(), lens.data(), score.data(), cap + 1, &rows));
    const std::vector<Word> words = unpack(bytes.data(), lens.data(), rows);
    for (std::uint64_t r = 0; r < rows; ++r) report.rows.push_back({words[r], score[r]});
    return report;
}

}  // namespace wfc

// ---- report (proj/src/report.cpp:7-55): host formatting of what the device path produced -----------
namespace wfc {

std::string format_double(double v) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.12g", v);
    return buf;
}

void write_frequency_tsv(std::ostream& out, const FrequencyTable& table) {
    for (const auto& row : table.rows) out << row.word << '\t' << row.count << '\t' << format_double(row.rel_freq) << '\n';
}

void write_compare_tsv(std::ostream& out, const FrequencyTable& table, const DistinctivenessReport& report) {
    for (const auto& row : table.rows)
        out << table.label << "\ttop\t" << row.word << '\t' << row.count << '\t' << format_double(row.rel_freq) << '\n';
    for (const auto& row : report.rows)
        out << report.label << "\tdistinct\t" << row.word << '\t' << format_double(row.score) << '\n';
}

void write_timings_tsv(std::ostream& out, const StageTimings& t) {
    out << "timing\tmap\t" << t.map_ns << '\n' << "timing\tsort\t" << t.sort_ns << '\n'
        << "timing\tencode\t" << t.encode_ns << '\n' << "timing\texchange\t" << t.exchange_ns << '\n'
        << "timing\treduce\t" << t.reduce_ns << '\n' << "timing\trepair\t" << t.repair_ns << '\n'
        << "timing\ttotal\t" << t.total_ns << '\n';
}

}  // namespace wfc
