// wfc_shuffle.cpp -- the host side of the paper's own exchange, behind the reference's names:
// WCX1 frames (reference: /root/reference/proj/include/wfc/wire.hpp, proj/src/wire.cpp:27-87), the
// transport seam (wfc/transport.hpp, proj/src/transport.cpp), encode_outgoing / exchange_encoded /
// exchange (wfc/shuffle.hpp, proj/src/shuffle.cpp:48-185) and the per-code-point accessors of
// wfc/unicode.hpp (proj/src/unicode.cpp:11-44, 72-121).
//
// Frames, queues and threads are host work in the reference too; what surrounds them in
// run_wordcount(corpus, n, Transport&) -- tokenize, sort, run-length encode -- runs on the device
// (wfc_b200.cpp).  The code-point accessors are single-value helpers for source compatibility;
// no data path of this library goes through them.
#include <algorithm>
#include <exception>
#include <iterator>
#include <thread>

#include "wfc/wfc_b200.hpp"

namespace wfc {

// ---- one code point -------------------------------------------------------------------
namespace {
// strict UTF-8: {first lead, last lead, continuation bytes, lowest / highest second byte}
struct LeadClass {
    unsigned char lo, hi, extra, second_lo, second_hi;
};
constexpr LeadClass kLeads[] = {
    {0xC2, 0xDF, 1, 0x80, 0xBF}, {0xE0, 0xE0, 2, 0xA0, 0xBF}, {0xE1, 0xEC, 2, 0x80, 0xBF}, {0xED, 0xED, 2, 0x80, 0x9F},
    {0xEE, 0xEF, 2, 0x80, 0xBF}, {0xF0, 0xF0, 3, 0x90, 0xBF}, {0xF1, 0xF3, 3, 0x80, 0xBF}, {0xF4, 0xF4, 3, 0x80, 0x8F},
};
struct Range {
    char32_t lo, hi;
};
// non-ASCII code points that are NOT word characters, apart from the whitespace set
constexpr Range kNotWord[] = {{0xA1, 0xA9},     {0xAB, 0xB4},     {0xB6, 0xB9},     {0xBB, 0xBF},     {0xD7, 0xD7},
                              {0xF7, 0xF7},     {0x2000, 0x206F}, {0x3000, 0x303F}, {0xFF01, 0xFF0F}, {0xFF1A, 0xFF20},
                              {0xFF3B, 0xFF40}, {0xFF5B, 0xFF65}, {0xFFFD, 0xFFFD}};
constexpr Range kSpace[] = {{0x09, 0x0D},     {0x20, 0x20},     {0x85, 0x85},     {0xA0, 0xA0},     {0x1680, 0x1680}, {0x2000, 0x200A},
                            {0x2028, 0x2029}, {0x202F, 0x202F}, {0x205F, 0x205F}, {0x3000, 0x3000}};
template <std::size_t N>
bool in_ranges(const Range (&ranges)[N], char32_t cp) {
    for (const Range& r : ranges)
        if (cp >= r.lo && cp <= r.hi) return true;
    return false;
}
}  // namespace

DecodedChar utf8_decode(std::string_view text, std::size_t pos) {
    DecodedChar bad;   // U+FFFD, one byte, invalid
    if (pos >= text.size()) return bad;
    const auto byte = [&](std::size_t i) { return static_cast<unsigned char>(text[i]); };
    const unsigned char b0 = byte(pos);
    if (b0 < 0x80) return DecodedChar{b0, 1, true};
    for (const LeadClass& lc : kLeads) {
        if (b0 < lc.lo || b0 > lc.hi) continue;
        if (pos + lc.extra >= text.size()) return bad;
        const unsigned char b1 = byte(pos + 1);
        if (b1 < lc.second_lo || b1 > lc.second_hi) return bad;
        char32_t cp = (char32_t(b0) & (0x3Fu >> lc.extra)) << 6 | (b1 & 0x3F);
        for (unsigned k = 2; k <= lc.extra; ++k) {
            const unsigned char b = byte(pos + k);
            if ((b & 0xC0) != 0x80) return bad;
            cp = cp << 6 | (b & 0x3F);
        }
        return DecodedChar{cp, lc.extra + 1u, true};
    }
    return bad;   // 80..C1, F5..FF
}

void utf8_append(std::string& out, char32_t cp) {
    const unsigned n = cp < 0x80 ? 1 : cp < 0x800 ? 2 : cp < 0x10000 ? 3 : 4;
    if (n == 1) {
        out.push_back(char(cp));
        return;
    }
    static constexpr unsigned char kMark[5] = {0, 0, 0xC0, 0xE0, 0xF0};
    out.push_back(char(kMark[n] | (cp >> (6 * (n - 1)))));
    for (unsigned k = n - 1; k-- > 0;) out.push_back(char(0x80 | ((cp >> (6 * k)) & 0x3F)));
}

bool is_unicode_space(char32_t cp) { return in_ranges(kSpace, cp); }

bool is_word_char(char32_t cp) {
    if (cp < 0x80) return (cp >= '0' && cp <= '9') || ((cp | 0x20) >= 'a' && (cp | 0x20) <= 'z');
    return !in_ranges(kNotWord, cp) && !in_ranges(kSpace, cp);
}

char32_t simple_lower(char32_t cp) {
    const bool ascii_upper = cp >= 'A' && cp <= 'Z';
    const bool latin1_upper = cp >= 0xC0 && cp <= 0xDE && cp != 0xD7;
    return ascii_upper || latin1_upper ? cp + 0x20 : cp;
}

// ---- WCX1 frames ------------------------------------------------------------------------
namespace {
void put_u32(WireMessage& out, std::uint64_t v) {
    for (int k = 0; k < 4; ++k) out.push_back(std::uint8_t(v >> (8 * k)));
}
std::uint64_t get_u32(std::span<const std::uint8_t> frame, std::size_t at) {
    return std::uint64_t(frame[at]) | std::uint64_t(frame[at + 1]) << 8 | std::uint64_t(frame[at + 2]) << 16 |
           std::uint64_t(frame[at + 3]) << 24;
}
bool strictly_utf8(std::string_view s) {
    for (std::size_t pos = 0; pos < s.size();) {
        const DecodedChar d = utf8_decode(s, pos);
        if (!d.valid) return false;
        pos += d.length;
    }
    return true;
}
}  // namespace

WireMessage encode_message(std::span<const std::string> words) {
    constexpr std::uint64_t kMax = 0xFFFFFFFFull;
    if (words.size() > kMax) throw std::length_error("word batch exceeds 2^32-1 words");
    std::uint64_t payload = 0;
    for (const std::string& w : words) {
        if (w.size() > kMax) throw std::length_error("word exceeds 2^32-1 bytes");
        payload += w.size();
    }
    WireMessage out;
    out.reserve(8 + 4 * words.size() + payload);
    out.insert(out.end(), kFrameMagic.begin(), kFrameMagic.end());
    put_u32(out, words.size());
    for (const std::string& w : words) put_u32(out, w.size());
    for (const std::string& w : words) out.insert(out.end(), w.begin(), w.end());
    return out;
}

std::vector<std::string> decode_message(std::span<const std::uint8_t> frame) {
    using Kind = WireError::Kind;
    if (frame.size() < 4 || !std::equal(kFrameMagic.begin(), kFrameMagic.end(), frame.begin()))
        throw WireError(Kind::BadMagic, "malformed frame: bad magic");
    if (frame.size() < 8) throw WireError(Kind::Truncated, "truncated frame: missing word count");
    const std::uint64_t count = get_u32(frame, 4);
    if ((frame.size() - 8) / 4 < count) throw WireError(Kind::Truncated, "truncated frame: missing word lengths");
    const std::size_t payload_at = 8 + 4 * std::size_t(count);
    std::uint64_t payload = 0;
    for (std::uint64_t i = 0; i < count; ++i) payload += get_u32(frame, 8 + 4 * std::size_t(i));
    if (frame.size() - payload_at < payload) throw WireError(Kind::Truncated, "truncated frame: payload short of declared lengths");
    if (frame.size() - payload_at > payload) throw WireError(Kind::TrailingBytes, "framing error: trailing bytes after payload");
    std::vector<std::string> words;
    words.reserve(std::size_t(count));
    std::size_t at = payload_at;
    for (std::uint64_t i = 0; i < count; ++i) {
        const std::size_t len = std::size_t(get_u32(frame, 8 + 4 * std::size_t(i)));
        std::string w(reinterpret_cast<const char*>(frame.data()) + at, len);
        if (!strictly_utf8(w)) throw WireError(Kind::BadEncoding, "encoding error: word payload is not UTF-8");
        words.push_back(std::move(w));
        at += len;
    }
    return words;
}

// ---- in-process transport -----------------------------------------------------------------
InProcessTransport::InProcessTransport(std::size_t n_workers) : n_(n_workers) {
    if (n_ == 0) throw TransportError("transport needs at least one worker");
    channels_.resize(n_ * n_);
    for (auto& c : channels_) c = std::make_unique<Channel>();
}

InProcessTransport::Channel& InProcessTransport::channel(std::size_t from, std::size_t to) {
    if (from >= n_ || to >= n_)
        throw TransportError("no channel between worker " + std::to_string(from) + " and worker " + std::to_string(to));
    return *channels_[from * n_ + to];
}

void InProcessTransport::send(std::size_t from, std::size_t to, WireMessage frame) {
    Channel& c = channel(from, to);
    {
        std::lock_guard<std::mutex> lock(c.mu);
        c.queue.push_back(std::move(frame));
    }
    c.cv.notify_one();
}

WireMessage InProcessTransport::recv(std::size_t at, std::size_t from) {
    Channel& c = channel(from, at);
    std::unique_lock<std::mutex> lock(c.mu);
    c.cv.wait(lock, [&] { return !c.queue.empty(); });
    WireMessage frame = std::move(c.queue.front());
    c.queue.pop_front();
    return frame;
}

// ---- shuffle --------------------------------------------------------------------------------
EncodedShard encode_outgoing(const ShardPlan& plan, const WordList& sorted) {
    if (!sorted.sorted) throw std::invalid_argument("encode_outgoing: word list must be sorted");
    if (plan.local_count != sorted.words.size()) throw std::invalid_argument("encode_outgoing: plan does not match word list");
    EncodedShard shard;
    shard.worker_id = plan.worker_id;
    shard.n_workers = plan.n_workers;
    const std::span<const Word> all(sorted.words);
    for (std::size_t c = 0; c < plan.n_workers; ++c) {
        const std::span<const Word> chunk = all.subspan(plan.chunk_begin(c), plan.chunk_size(c));
        if (c == plan.worker_id) shard.kept.assign(chunk.begin(), chunk.end());
        else shard.outgoing.emplace_back(c, encode_message(chunk));
    }
    return shard;
}

namespace {
std::string arrow(std::size_t from, std::size_t to) { return "worker " + std::to_string(from) + " -> worker " + std::to_string(to); }

// what worker j does: send its frames, receive one frame per peer, merge the n sorted chunks.
// std::merge takes from its first range on ties, so folding the sources in index order keeps
// "lowest source first".
WordList exchange_worker(EncodedShard& shard, Transport& transport) {
    const std::size_t j = shard.worker_id, n = shard.n_workers;
    for (auto& [peer, frame] : shard.outgoing) {
        try {
            transport.send(j, peer, std::move(frame));
        } catch (const std::exception& e) {
            throw ExchangeError("exchange send failed (" + arrow(j, peer) + "): " + e.what());
        }
    }
    std::vector<Word> merged;
    for (std::size_t src = 0; src < n; ++src) {
        std::vector<Word> chunk;
        if (src == j) {
            chunk = std::move(shard.kept);
        } else {
            WireMessage frame;
            try {
                frame = transport.recv(j, src);
            } catch (const std::exception& e) {
                throw ExchangeError("exchange receive failed (" + arrow(src, j) + "): " + e.what());
            }
            try {
                chunk = decode_message(frame);
            } catch (const WireError& e) {
                throw ExchangeError("worker " + std::to_string(j) + " got an invalid frame from worker " + std::to_string(src) +
                                    ": " + e.what());
            }
        }
        std::vector<Word> next;
        next.reserve(merged.size() + chunk.size());
        std::merge(std::make_move_iterator(merged.begin()), std::make_move_iterator(merged.end()),
                   std::make_move_iterator(chunk.begin()), std::make_move_iterator(chunk.end()), std::back_inserter(next));
        merged = std::move(next);
    }
    return WordList{std::move(merged), true};
}
}  // namespace

std::vector<WordList> exchange_encoded(std::vector<EncodedShard> shards, Transport& transport) {
    const std::size_t n = shards.size();
    if (n == 0) throw std::invalid_argument("exchange: need at least one worker");
    for (std::size_t j = 0; j < n; ++j)
        if (shards[j].worker_id != j || shards[j].n_workers != n)
            throw std::invalid_argument("exchange: shard " + std::to_string(j) + " does not agree on worker layout");
    std::vector<WordList> out(n);
    if (n == 1) {
        out[0] = WordList{std::move(shards[0].kept), true};
        return out;
    }
    std::vector<std::exception_ptr> failure(n);
    std::vector<std::thread> workers;
    workers.reserve(n);
    for (std::size_t j = 0; j < n; ++j)
        workers.emplace_back([&, j] {
            try {
                out[j] = exchange_worker(shards[j], transport);
            } catch (...) {
                failure[j] = std::current_exception();
            }
        });
    for (auto& w : workers) w.join();
    for (const auto& f : failure)
        if (f) std::rethrow_exception(f);
    return out;
}

std::vector<WordList> exchange(const std::vector<WorkerShard>& inputs, Transport& transport) {
    std::vector<EncodedShard> shards;
    shards.reserve(inputs.size());
    for (std::size_t j = 0; j < inputs.size(); ++j) {
        if (inputs[j].plan.worker_id != j || inputs[j].plan.n_workers != inputs.size())
            throw std::invalid_argument("exchange: plan " + std::to_string(j) + " does not agree on worker layout");
        shards.push_back(encode_outgoing(inputs[j].plan, inputs[j].words));
    }
    return exchange_encoded(std::move(shards), transport);
}

std::vector<WordList> exchange(const std::vector<WorkerShard>& inputs) {
    InProcessTransport transport(std::max<std::size_t>(inputs.size(), 1));
    return wfc::exchange(inputs, transport);
}

}  // namespace wfc
