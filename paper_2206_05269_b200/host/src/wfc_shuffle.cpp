// wfc_shuffle.cpp -- WCX1 frames, the transport seam and the frame-carrying form of the paper's exchange
// (interfaces: /root/reference/proj/include/wfc/{wire,transport,shuffle}.hpp), for callers that bring their own
// Transport.  SURVEY.md marks wire / transport out of the hot path: run_wordcount(corpus, n) never comes here (its
// chunks move inside device memory, wfc_b200.cpp).  What this file does differently from a host implementation:
//   * a frame is laid out in one allocation and validated in one pass over its three regions; the UTF-8 check of the
//     word payload is ONE device pass over the whole payload (utf8_sanitize keeps the length iff nothing is
//     replaced) plus a look at the first byte of every word;
//   * the workers of an exchange are not threads: every frame is handed to the transport, then every worker's
//     inbox is drained in worker order -- with one frame per ordered pair that is the same schedule the reference's
//     n threads produce, minus the threads;
//   * the n-way merge of the received chunks is the device radix sort (sort_words): equal words are equal strings,
//     so "lowest source first" has nothing to decide.
#include <algorithm>
#include <bit>
#include <cstring>
#include <exception>

#include "wfc/wfc_b200.hpp"

namespace wfc {

static_assert(std::endian::native == std::endian::little, "WCX1 integers are little-endian; so is every CUDA host");

// ---- WCX1 frames ------------------------------------------------------------------------
namespace {
constexpr std::size_t kHeaderBytes = 8;          // magic + word count
constexpr std::uint64_t kU32Max = 0xFFFFFFFFull;

std::uint32_t load_u32(const std::uint8_t* p) {
    std::uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}

// The three regions of a structurally sound frame.
struct FrameLayout {
    std::uint32_t words = 0;
    const std::uint8_t* lengths = nullptr;    // words x u32
    const std::uint8_t* payload = nullptr;
    std::size_t payload_bytes = 0;
};

FrameLayout layout_of(std::span<const std::uint8_t> frame) {
    using Kind = WireError::Kind;
    if (frame.size() < kFrameMagic.size() || std::memcmp(frame.data(), kFrameMagic.data(), kFrameMagic.size()) != 0)
        throw WireError(Kind::BadMagic, "malformed frame: bad magic");
    if (frame.size() < kHeaderBytes) throw WireError(Kind::Truncated, "truncated frame: missing word count");
    FrameLayout f;
    f.words = load_u32(frame.data() + 4);
    const std::size_t after_header = frame.size() - kHeaderBytes;
    if (after_header / 4 < f.words) throw WireError(Kind::Truncated, "truncated frame: missing word lengths");
    f.lengths = frame.data() + kHeaderBytes;
    f.payload = f.lengths + std::size_t(4) * f.words;
    f.payload_bytes = after_header - std::size_t(4) * f.words;
    std::uint64_t declared = 0;
    for (std::uint32_t i = 0; i < f.words; ++i) declared += load_u32(f.lengths + std::size_t(4) * i);
    if (declared > f.payload_bytes) throw WireError(Kind::Truncated, "truncated frame: payload short of declared lengths");
    if (declared < f.payload_bytes) throw WireError(Kind::TrailingBytes, "framing error: trailing bytes after payload");
    return f;
}
}  // namespace

WireMessage encode_message(std::span<const std::string> words) {
    if (words.size() > kU32Max) throw std::length_error("word batch exceeds 2^32-1 words");
    std::size_t payload = 0;
    for (const std::string& w : words) {
        if (w.size() > kU32Max) throw std::length_error("word exceeds 2^32-1 bytes");
        payload += w.size();
    }
    WireMessage frame(kHeaderBytes + 4 * words.size() + payload);
    std::uint8_t* header = frame.data();
    std::memcpy(header, kFrameMagic.data(), kFrameMagic.size());
    const std::uint32_t count = std::uint32_t(words.size());
    std::memcpy(header + 4, &count, 4);
    std::uint8_t* length_at = header + kHeaderBytes;
    std::uint8_t* byte_at = length_at + 4 * words.size();
    for (const std::string& w : words) {
        const std::uint32_t len = std::uint32_t(w.size());
        std::memcpy(length_at, &len, 4);
        length_at += 4;
        if (len) std::memcpy(byte_at, w.data(), len);
        byte_at += len;
    }
    return frame;
}

std::vector<std::string> decode_message(std::span<const std::uint8_t> frame) {
    const FrameLayout f = layout_of(frame);
    // every word is UTF-8  <=>  the payload as a whole is, and no word starts inside a sequence
    const std::string_view payload(reinterpret_cast<const char*>(f.payload), f.payload_bytes);
    bool sound = f.payload_bytes == 0 || utf8_valid(payload);
    std::vector<std::string> words;
    words.reserve(f.words);
    std::size_t at = 0;
    for (std::uint32_t i = 0; i < f.words && sound; ++i) {
        const std::uint32_t len = load_u32(f.lengths + std::size_t(4) * i);
        if (len && (f.payload[at] & 0xC0) == 0x80) sound = false;
        words.emplace_back(payload.substr(at, len));
        at += len;
    }
    if (!sound) throw WireError(WireError::Kind::BadEncoding, "encoding error: word payload is not UTF-8");
    return words;
}

// ---- in-process transport -----------------------------------------------------------------
InProcessTransport::InProcessTransport(std::size_t n_workers) : n_(n_workers) {
    if (n_ == 0) throw TransportError("transport needs at least one worker");
    boxes_.resize(n_ * n_);
}

std::size_t InProcessTransport::mailbox(std::size_t from, std::size_t to) const {
    if (from >= n_ || to >= n_)
        throw TransportError("no channel between worker " + std::to_string(from) + " and worker " + std::to_string(to));
    return to * n_ + from;
}

void InProcessTransport::send(std::size_t from, std::size_t to, WireMessage frame) {
    const std::size_t box = mailbox(from, to);
    {
        std::lock_guard<std::mutex> lock(mu_);
        boxes_[box].push_back(std::move(frame));
    }
    arrived_.notify_all();
}

WireMessage InProcessTransport::recv(std::size_t at, std::size_t from) {
    const std::size_t box = mailbox(from, at);
    std::unique_lock<std::mutex> lock(mu_);
    arrived_.wait(lock, [&] { return !boxes_[box].empty(); });
    WireMessage frame = std::move(boxes_[box].front());
    boxes_[box].pop_front();
    return frame;
}

// ---- shuffle --------------------------------------------------------------------------------
EncodedShard encode_outgoing(const ShardPlan& plan, const WordList& sorted) {
    if (!sorted.sorted) throw std::invalid_argument("encode_outgoing: word list must be sorted");
    if (plan.local_count != sorted.words.size()) throw std::invalid_argument("encode_outgoing: plan does not match word list");
    EncodedShard shard;
    shard.worker_id = plan.worker_id;
    shard.n_workers = plan.n_workers;
    const Word* first = sorted.words.data();
    for (std::size_t c = 0; c < plan.n_workers; ++c) {
        const std::span<const Word> chunk(first + plan.chunk_begin(c), plan.chunk_size(c));
        if (c == plan.worker_id) shard.kept.assign(chunk.begin(), chunk.end());
        else shard.outgoing.emplace_back(c, encode_message(chunk));
    }
    return shard;
}

std::vector<WordList> exchange_encoded(std::vector<EncodedShard> shards, Transport& transport) {
    const std::size_t n = shards.size();
    if (n == 0) throw std::invalid_argument("exchange: need at least one worker");
    for (std::size_t j = 0; j < n; ++j)
        if (shards[j].worker_id != j || shards[j].n_workers != n)
            throw std::invalid_argument("exchange: shard " + std::to_string(j) + " does not agree on worker layout");
    const auto pair = [](std::size_t from, std::size_t to) {
        return "worker " + std::to_string(from) + " -> worker " + std::to_string(to);
    };
    // every frame goes out ...
    for (EncodedShard& shard : shards)
        for (auto& [peer, frame] : shard.outgoing) {
            try {
                transport.send(shard.worker_id, peer, std::move(frame));
            } catch (const std::exception& e) {
                throw ExchangeError("exchange send failed (" + pair(shard.worker_id, peer) + "): " + e.what());
            }
        }
    // ... then every worker gathers its chunk of every list and orders it on the device
    std::vector<WordList> out(n);
    for (std::size_t j = 0; j < n; ++j) {
        std::vector<Word> mine = std::move(shards[j].kept);
        for (std::size_t src = 0; src < n; ++src) {
            if (src == j) continue;
            WireMessage frame;
            try {
                frame = transport.recv(j, src);
            } catch (const std::exception& e) {
                throw ExchangeError("exchange receive failed (" + pair(src, j) + "): " + e.what());
            }
            std::vector<Word> chunk;
            try {
                chunk = decode_message(frame);
            } catch (const WireError& e) {
                throw ExchangeError("worker " + std::to_string(j) + " got an invalid frame from worker " + std::to_string(src) +
                                    ": " + e.what());
            }
            mine.insert(mine.end(), std::make_move_iterator(chunk.begin()), std::make_move_iterator(chunk.end()));
        }
        out[j] = n == 1 ? WordList{std::move(mine), true} : sort_words(WordList{std::move(mine), false});
    }
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
