// wfc/wfc_b200.hpp -- the reference's map/reduce API, served by B200 kernels.
//
// Same namespace, names, argument meaning and error behaviour as the hot-path part of
// /root/reference/proj/include/wfc/{text,reduce,pipeline,engine,analysis}.hpp, so a
// caller of the reference (proj/src/cli.cpp:79-86, 138-141, 202-221) relinks against
// libwfc_b200.so unchanged.  The per-topic headers wfc/text.hpp, wfc/reduce.hpp, ...
// forward here.  The data paths (tokenize, normalize, sort, count, run-length encode, merge, partition,
// map-reduce, sanitize, the joins and selections behind DeviceCounts::top_k / distinctive) run on the GPU
// through the C ABI of include/wfcu.h; there is no CPU implementation to fall back to -- without a device
// the calls throw wfc::DeviceError.  Host code is what is left of host work: std:: containers and their
// bookkeeping (boundary_repair, count_unreduced_words), the final ordering of the few candidate rows of
// top_k / distinctive_words with the reference's comparators (one implementation, in libwfcu), WCX1 frames
// and transports for callers that bring their own Transport, file reading (ingest_directory), index
// arithmetic (plan_partition) and the single-code-point accessors.
//
// Differences a caller can observe (all additive):
//   * MapKind gains `square` (value 3) for f(x) = x^2; map_reduce_fast() is the
//     HBM-roofline reduction (fp64 accumulation, fixed order, within ~1e-15 relative of
//     the serial fold), next to the bit-exact map_reduce_serial / map_reduce_blocked;
//   * run_wordcount(corpus, n) is the reference's pipeline, range partition and boundary repair included
//     (pre_repair_shards are the reference's, proj/tests/pipeline_test.cpp:26-33): tokenize, sort, the
//     exchange of the chunks, the n-way merge and the run-length encode all stay in device memory;
//     run_wordcount(corpus, n, Transport&) sends the same chunks as WCX1 frames over the caller's transport;
//   * run_wordcount_hashed(corpus, n) is the fast path of BASELINE.json: fused tokenize/count kernels, worker j
//     on GPU j mod device_count, tables hash-partitioned by owner and delivered device to device.  Its
//     RunResult::counts is identical; the shards are disjoint by construction (pre_repair_shards == shards);
//   * DeviceCounts keeps a table on the device: per-speaker top-k / distinctive words (cli.cpp:176-230) without
//     exporting a million-word map.
#pragma once

#include <array>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <deque>
#include <filesystem>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <ostream>
#include <unordered_set>
#include <utility>
#include <vector>

struct wfcu_counter;   // include/wfcu.h

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
    std::size_t mailbox(std::size_t from, std::size_t to) const;   // throws TransportError off the grid
    std::size_t n_;
    std::mutex mu_;                                  // one lock and one wake-up for the whole grid:
    std::condition_variable arrived_;                // a frame is a pointer move, there is nothing to contend for
    std::vector<std::deque<WireMessage>> boxes_;     // [to * n + from]
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
// The fast path: fused tokenize/count, hash-partitioned device-to-device merge over the box's GPUs
// (wfcu_wordcount_multi).  StageTimings are CUDA-event times.
RunResult run_wordcount_hashed(std::span<const RawDocument> corpus, std::size_t n_workers);

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
RunResult run_wordcount_range_partitioned(std::span<const RawDocument> corpus, std::size_t n_workers);   // == run_wordcount(corpus, n)
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

// A count table that stays on the device (wfcu_counter): the compare command of the reference
// (proj/src/cli.cpp:176-230) -- count every corpus, pool the others, top-k and distinctive words per corpus --
// without a std::map in between.
class DeviceCounts {
public:
    explicit DeviceCounts(std::uint64_t expected_distinct_words = 0);
    ~DeviceCounts();
    DeviceCounts(DeviceCounts&& other) noexcept;
    DeviceCounts& operator=(DeviceCounts&& other) noexcept;
    DeviceCounts(const DeviceCounts&) = delete;
    DeviceCounts& operator=(const DeviceCounts&) = delete;

    void count(std::span<const RawDocument> corpus);          // += serial_wordcount(corpus)
    void merge(const DeviceCounts& other);                    // += other (merge_counts, reduce.cpp:83-89)
    std::uint64_t distinct_words() const;
    std::uint64_t total_words() const;
    CountMap to_map() const;
    FrequencyTable top_k(std::string label, std::size_t k) const;
    DistinctivenessReport distinctive(const DeviceCounts& others, std::string label, std::size_t k) const;
    wfcu_counter* handle() const { return h_; }

private:
    wfcu_counter* h_ = nullptr;
};

// ---- ingest (reference: wfc/analysis.hpp, the file side) ------------------------------------------------
struct Corpus {
    std::string label;
    std::vector<RawDocument> documents;
};
class IngestError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
// Every .txt / .text file of `dir` as one document, in file-name order, invalid UTF-8 replaced by U+FFFD
// (utf8_sanitize, on the device: the files of the directory are sanitised as one batch).
Corpus ingest_directory(const std::filesystem::path& dir, std::string label);
std::unordered_set<Word> load_stopwords(const std::filesystem::path& file);   // one tokenised word list
CountMap remove_stopwords(CountMap counts, const std::unordered_set<Word>& stopwords);

// ---- report (reference: wfc/report.hpp, the text writers; the JSON ones need the vendored json.hpp) ----
std::string format_double(double v);                                                    // "%.12g"
void write_frequency_tsv(std::ostream& out, const FrequencyTable& table);               // word<TAB>count<TAB>relfreq
void write_compare_tsv(std::ostream& out, const FrequencyTable& table, const DistinctivenessReport& report);
void write_timings_tsv(std::ostream& out, const StageTimings& timings);                 // timing<TAB>stage<TAB>ns

}  // namespace wfc
