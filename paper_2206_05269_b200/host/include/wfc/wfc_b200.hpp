// wfc/wfc_b200.hpp -- the reference's map/reduce API, served by B200 kernels.
//
// Same namespace, names, argument meaning and error behaviour as the hot-path part of
// /root/reference/proj/include/wfc/{text,reduce,pipeline,engine,analysis}.hpp, so a
// caller of the reference (proj/src/cli.cpp:79-86, 138-141, 202-221) relinks against
// libwfc_b200.so unchanged.  The per-topic headers wfc/text.hpp, wfc/reduce.hpp, ...
// forward here.  Every data path below (tokenize, normalize, sort, count, reduce, merge, map-reduce,
// top-k, sanitize) runs its arithmetic on the GPU through the C ABI of include/wfcu.h; there is no CPU
// implementation to fall back to -- without a device the calls throw wfc::DeviceError.  Host code is
// what is host code in the reference too: containers, the WCX1 frames / transports / threads of the
// paper's exchange, index arithmetic (plan_partition) and the single-code-point accessors.
//
// Differences a caller can observe (all additive):
//   * MapKind gains `square` (value 3) for f(x) = x^2; map_reduce_fast() is the
//     HBM-roofline reduction (fp64 accumulation, fixed order, within ~1e-15 relative of
//     the serial fold), next to the bit-exact map_reduce_serial / map_reduce_blocked;
//   * run_wordcount partitions by key hash, not by alphabetical range (BASELINE.json;
//     SURVEY.md D2): RunResult::counts is identical, the shards are pairwise disjoint,
//     pre_repair_shards == shards and boundary_repair has nothing left to do;
//   * run_wordcount(corpus, n, Transport&) runs the paper's own range-partitioned exchange over
//     the caller's transport, WCX1 frames included (tokenize / sort / run-length encode on the
//     device, frames on the host, like the reference); run_wordcount(corpus, n) is the fast
//     path and exchanges table entries in device memory / over NCCL instead.
#pragma once

#include <array>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <ostream>
#include <utility>
#include <vector>

namespace wfc {

// ---- text (reference: wfc/text.hpp) -------------------------------------------------
using Word = std::string;

struct RawDocument {
    std::string id;
    std::string text;
};

struct WordList {
    std::vector<Word> words;
    bool sorted = false;
};

// ---- unicode (reference: wfc/unicode.hpp, the ingest step) ----------------------------
std::string utf8_sanitize(std::string_view text);
bool utf8_valid(std::string_view text);     // no byte needs replacing (same device pass)

// Per-code-point accessors of the same header, for source compatibility: plain host arithmetic on ONE
// code point.  Nothing in this library calls them on a data path -- tokenize, normalize_word,
// utf8_sanitize and the counting kernels classify bytes on the device.
inline constexpr char32_t kReplacementChar = 0xFFFD;
struct DecodedChar {
    char32_t cp = kReplacementChar;
    unsigned length = 1;   // bytes consumed
    bool valid = false;
};
DecodedChar utf8_decode(std::string_view text, std::size_t pos);
void utf8_append(std::string& out, char32_t cp);
bool is_unicode_space(char32_t cp);
bool is_word_char(char32_t cp);
char32_t simple_lower(char32_t cp);

std::optional<Word> normalize_word(std::string_view fragment);
std::vector<std::optional<Word>> normalize_words(std::span<const std::string> fragments);  // batch form (one launch)
WordList tokenize(const RawDocument& doc);
WordList sort_words(WordList list);

// ---- reduce (reference: wfc/reduce.hpp) ----------------------------------------------
using CountMap = std::map<Word, std::uint64_t>;
using ShardedCounts = std::vector<CountMap>;

CountMap reduce_sorted(const WordList& sorted);
ShardedCounts boundary_repair(ShardedCounts sharded);
CountMap merge_counts(std::span<const CountMap> maps);
std::size_t count_unreduced_words(const ShardedCounts& sharded);

// ---- wire format and transport seam (reference: wfc/wire.hpp, wfc/transport.hpp) -----------
// Frame of one word batch: "WCX1", u32-LE word count, u32-LE byte length of each word, then the
// word payloads; nothing may follow.
using WireMessage = std::vector<std::uint8_t>;
inline constexpr std::array<std::uint8_t, 4> kFrameMagic = {0x57, 0x43, 0x58, 0x31};

class WireError : public std::runtime_error {
public:
    enum class Kind { BadMagic, Truncated, TrailingBytes, BadEncoding };
    WireError(Kind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
    Kind kind() const { return kind_; }

private:
    Kind kind_;
};

WireMessage encode_message(std::span<const std::string> words);             // std::length_error beyond 2^32-1
std::vector<std::string> decode_message(std::span<const std::uint8_t> frame);   // exact inverse; throws WireError

class TransportError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// Ordered, reliable, point-to-point frame channel between worker pairs; recv blocks.
class Transport {
public:
    virtual ~Transport() = default;
    virtual void send(std::size_t from, std::size_t to, WireMessage frame) = 0;
    virtual WireMessage recv(std::size_t at, std::size_t from) = 0;
};

// One unbounded FIFO per ordered worker pair, in this process.
class InProcessTransport final : public Transport {
public:
    explicit InProcessTransport(std::size_t n_workers);
    void send(std::size_t from, std::size_t to, WireMessage frame) override;
    WireMessage recv(std::size_t at, std::size_t from) override;
    std::size_t n_workers() const { return n_; }

private:
    struct Channel {
        std::mutex mu;
        std::condition_variable cv;
        std::deque<WireMessage> queue;
    };
    Channel& channel(std::size_t from, std::size_t to);
    std::size_t n_;
    std::vector<std::unique_ptr<Channel>> channels_;
};

// ---- pipeline (reference: wfc/pipeline.hpp) --------------------------------------------
struct StageTimings {
    std::uint64_t map_ns = 0;       // H2D + fused tokenize/count kernels
    std::uint64_t sort_ns = 0;      // 0: the hash-count path does not sort
    std::uint64_t encode_ns = 0;    // partition-by-owner kernels
    std::uint64_t exchange_ns = 0;  // entry exchange + merge-insert
    std::uint64_t reduce_ns = 0;    // export of the owner tables
    std::uint64_t repair_ns = 0;    // 0: shards are disjoint by construction
    std::uint64_t total_ns = 0;
};

struct RunResult {
    CountMap counts;
    ShardedCounts shards;
    ShardedCounts pre_repair_shards;
    StageTimings timings;
    std::size_t n_workers = 1;
};

class PipelineError : public std::runtime_error {
public:
    PipelineError(std::string stage, const std::string& what)
        : std::runtime_error(stage + " stage: " + what), stage_(std::move(stage)) {}
    const std::string& stage() const { return stage_; }

private:
    std::string stage_;
};

// No usable GPU / CUDA failure outside a pipeline stage.
class DeviceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

RunResult run_wordcount(std::span<const RawDocument> corpus, std::size_t n_workers);
RunResult run_wordcount(std::span<const RawDocument> corpus, std::size_t n_workers, Transport& transport);

// The paper's own algorithm (reference pipeline.cpp:61-123, shuffle.cpp:9-46), stage by
// stage on the device kernels: tokenize -> sort_words -> range partition by position
// (plan_partition) -> per-owner merge (sort) -> reduce_sorted -> boundary_repair.  Slower
// than run_wordcount (tokens are materialised), but its pre_repair_shards are exactly the
// reference's, boundary words included.
struct ShardPlan {
    std::size_t worker_id = 0;
    std::size_t n_workers = 1;
    std::size_t local_count = 0;
    std::vector<std::size_t> boundaries;   // n+1 cut indices
    std::size_t chunk_begin(std::size_t c) const { return boundaries[c]; }
    std::size_t chunk_end(std::size_t c) const { return boundaries[c + 1]; }
    std::size_t chunk_size(std::size_t c) const { return boundaries[c + 1] - boundaries[c]; }
};
ShardPlan plan_partition(const WordList& sorted, std::size_t worker_id, std::size_t n_workers);

// The shuffle of wfc/shuffle.hpp: every worker keeps chunk `worker_id` of its sorted list and frames
// chunk c for worker c; exchange_encoded runs n concurrent workers over the transport and merges what
// each receives (ties: lowest source first), so the result does not depend on arrival order.
struct WorkerShard {
    ShardPlan plan;
    WordList words;
};
struct EncodedShard {
    std::size_t worker_id = 0;
    std::size_t n_workers = 1;
    std::vector<Word> kept;
    std::vector<std::pair<std::size_t, WireMessage>> outgoing;   // (peer, frame)
};
class ExchangeError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
EncodedShard encode_outgoing(const ShardPlan& plan, const WordList& sorted);
std::vector<WordList> exchange_encoded(std::vector<EncodedShard> shards, Transport& transport);
std::vector<WordList> exchange(const std::vector<WorkerShard>& inputs, Transport& transport);
std::vector<WordList> exchange(const std::vector<WorkerShard>& inputs);
RunResult run_wordcount_range_partitioned(std::span<const RawDocument> corpus, std::size_t n_workers);
CountMap serial_wordcount(std::span<const RawDocument> corpus);

// ---- engine (reference: wfc/engine.hpp) ------------------------------------------------
enum class MapKind {
    identity,
    square_root,
    alternating_harmonic_term,
    square,   // appended: f(x) = x^2 (BASELINE.json config 2)
};

struct BlockConfig {
    std::size_t block_size = 256;
    unsigned workers = 1;   // kept for source compatibility; the device schedules the blocks
};

double map_reduce_serial(std::span<const double> values, MapKind map);
double map_reduce_blocked(std::span<const double> values, MapKind map, const BlockConfig& cfg);
double alternating_harmonic(std::uint64_t n, const BlockConfig& cfg = {});
// The roofline path: grid-stride, vectorised loads, warp-shuffle tree, fixed-order finish.
double map_reduce_fast(std::span<const double> values, MapKind map);
double map_reduce_fast(std::span<const float> values, MapKind map);

// ---- analysis (reference: wfc/analysis.hpp, the part on the path) -----------------------
struct FrequencyRow {
    Word word;
    std::uint64_t count = 0;
    double rel_freq = 0.0;
};
struct FrequencyTable {
    std::string label;
    std::uint64_t total_words = 0;
    std::vector<FrequencyRow> rows;
};
FrequencyTable top_k(const CountMap& counts, std::string label, std::size_t k);

struct DistinctiveRow {
    Word word;
    double score = 0.0;
};
struct DistinctivenessReport {
    std::string label;
    std::vector<DistinctiveRow> rows;
};
DistinctivenessReport distinctive_words(const CountMap& target, const CountMap& others, std::string label,
                                        std::size_t k);

// ---- report (reference: wfc/report.hpp, the text writers; the JSON ones need the vendored json.hpp) ----
std::string format_double(double v);                                                    // "%.12g"
void write_frequency_tsv(std::ostream& out, const FrequencyTable& table);               // word<TAB>count<TAB>relfreq
void write_compare_tsv(std::ostream& out, const FrequencyTable& table, const DistinctivenessReport& report);
void write_timings_tsv(std::ostream& out, const StageTimings& timings);                 // timing<TAB>stage<TAB>ns

}  // namespace wfc
