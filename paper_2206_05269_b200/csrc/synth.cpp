// synth.cpp -- deterministic synthetic Zipf corpora for BASELINE.json configs 3-5
// (generator pinned in SURVEY.md 8(d)); host-side C++, exported through the C ABI
// so the bench, the tests and the CPU baseline all consume the same bytes.
//
//   vocabulary  word(r) = prefix(r) + base26_W(r), lower-case a-z, W = ceil(log26 V),
//               prefix length = splitmix64(seed, r) mod 5  -> W..W+4 letters, unique by
//               construction (the last W letters encode r);
//               speaker k > 0 rewrites 1 % of the ranks as word(r) + digit k, which
//               gives every speaker distinctive words (config 5);
//   tokens      rank by inverse CDF of Zipf(s) over V (fp64 CDF, exact lower_bound
//               through a 65536-entry guide table); 1/16 capitalised; 1/16 followed
//               by one of . , ; ! ? ; separator '\n' with probability 1/16 else ' ';
//   documents   exactly doc_bytes bytes, tokens never cut, tail padded with spaces,
//               last byte '\n'.  Document d depends only on (seed, d, vocab, s, speaker).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

namespace wfcu {

static inline uint64_t splitmix64(uint64_t& x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t hash64(uint64_t v) {
    uint64_t x = v;
    return splitmix64(x);
}

struct Vocabulary {
    uint32_t vocab = 0;
    std::vector<uint8_t> text;   // 16 bytes per word
    std::vector<uint8_t> len;
    std::vector<double> cdf;
    std::vector<uint32_t> guide; // guide[b] = first rank with cdf >= b / 65536
};

static std::shared_ptr<const Vocabulary> get_vocabulary(uint64_t seed, uint32_t vocab, double s, uint32_t speaker) {
    static std::mutex mu;
    static std::map<std::tuple<uint64_t, uint32_t, double, uint32_t>, std::shared_ptr<const Vocabulary>> cache;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(seed, vocab, s, speaker);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;

    auto v = std::make_shared<Vocabulary>();
    v->vocab = vocab;
    uint32_t W = 1;
    for (uint64_t p = 26; p < vocab; p *= 26) ++W;
    v->text.assign(size_t(vocab) * 16, 0);
    v->len.assign(vocab, 0);
    for (uint32_t r = 0; r < vocab; ++r) {
        const uint64_t h = hash64(seed * 0x100000001B3ull + r);
        const uint32_t plen = uint32_t(h % 5);
        uint8_t* w = &v->text[size_t(r) * 16];
        uint32_t n = 0;
        for (uint32_t k = 0; k < plen; ++k) w[n++] = uint8_t('a' + ((h >> (8 + 6 * k)) % 26));
        uint32_t q = r;
        for (uint32_t k = 0; k < W; ++k) {
            w[n + W - 1 - k] = uint8_t('a' + q % 26);
            q /= 26;
        }
        n += W;
        if (speaker > 0 && hash64(seed ^ 0x5EA4E5ull ^ (uint64_t(r) << 20)) % 100 == 0) w[n++] = uint8_t('0' + speaker % 10);
        v->len[r] = uint8_t(n);
    }
    v->cdf.resize(vocab);
    double total = 0.0;
    for (uint32_t r = 0; r < vocab; ++r) total += std::pow(double(r) + 1.0, -s);
    double acc = 0.0;
    for (uint32_t r = 0; r < vocab; ++r) {
        acc += std::pow(double(r) + 1.0, -s) / total;
        v->cdf[r] = acc;
    }
    v->cdf[vocab - 1] = 1.0;
    v->guide.resize(65537);
    for (uint32_t b = 0; b <= 65536; ++b) {
        const double u = double(b) / 65536.0;
        v->guide[b] = uint32_t(std::lower_bound(v->cdf.begin(), v->cdf.end(), u) - v->cdf.begin());
    }
    cache[key] = v;
    return v;
}

static void make_document(const Vocabulary& v, uint64_t seed, uint64_t doc, uint8_t* out, uint64_t doc_bytes) {
    if (doc_bytes == 0) return;
    uint64_t state = hash64(seed ^ (doc + 1) * 0xD6E8FEB86659FD93ull);
    uint64_t pos = 0;
    const uint64_t limit = doc_bytes - 1;   // last byte is the closing '\n'
    static const char kPunct[5] = {'.', ',', ';', '!', '?'};
    for (;;) {
        const uint64_t a = splitmix64(state), b = splitmix64(state);
        const double u = double(a >> 11) * (1.0 / 9007199254740992.0);
        const uint32_t bucket = uint32_t(u * 65536.0);
        uint32_t lo = v.guide[bucket], hi = std::min<uint32_t>(v.guide[bucket + 1], v.vocab - 1);
        const uint32_t r = uint32_t(std::lower_bound(v.cdf.begin() + lo, v.cdf.begin() + hi, u) - v.cdf.begin());
        const uint8_t* w = &v.text[size_t(r) * 16];
        const uint32_t wl = v.len[r];
        const bool caps = (b & 15u) == 0, punct = ((b >> 4) & 15u) == 0, newline = ((b >> 12) & 15u) == 0;
        const uint32_t need = wl + (punct ? 1u : 0u) + 1u;
        if (pos + need > limit) break;
        std::memcpy(out + pos, w, wl);
        if (caps) out[pos] = uint8_t(out[pos] - 0x20);
        pos += wl;
        if (punct) out[pos++] = uint8_t(kPunct[(b >> 8) % 5]);
        out[pos++] = newline ? '\n' : ' ';
    }
    std::memset(out + pos, ' ', size_t(limit - pos));
    out[limit] = '\n';
}

int synth_document(uint64_t seed, uint64_t doc, uint32_t vocab, double s, uint32_t speaker, uint8_t* out,
                   uint64_t doc_bytes) {
    if (vocab == 0 || !out) return -1;
    const auto v = get_vocabulary(seed, vocab, s, speaker);
    make_document(*v, seed + 0x1000003ull * speaker, doc, out, doc_bytes);
    return 0;
}

// documents doc_begin, doc_begin + stride, ... (n_docs of them), back to back
int synth_corpus_strided(uint64_t seed, uint64_t doc_begin, uint64_t doc_stride, uint64_t n_docs, uint32_t vocab,
                         double s, uint32_t speaker, uint64_t doc_bytes, uint8_t* out, int threads) {
    if (vocab == 0 || !out || doc_stride == 0) return -1;
    const auto v = get_vocabulary(seed, vocab, s, speaker);
    unsigned nt = threads > 0 ? unsigned(threads) : std::max(1u, std::thread::hardware_concurrency());
    if (nt > n_docs) nt = unsigned(std::max<uint64_t>(1, n_docs));
    auto work = [&](unsigned t) {
        for (uint64_t d = t; d < n_docs; d += nt)
            make_document(*v, seed + 0x1000003ull * speaker, doc_begin + d * doc_stride, out + d * doc_bytes, doc_bytes);
    };
    if (nt <= 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nt; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    return 0;
}

int synth_corpus(uint64_t seed, uint64_t doc_begin, uint64_t doc_end, uint32_t vocab, double s, uint32_t speaker,
                 uint64_t doc_bytes, uint8_t* out, int threads) {
    if (doc_end < doc_begin) return -1;
    return synth_corpus_strided(seed, doc_begin, 1, doc_end - doc_begin, vocab, s, speaker, doc_bytes, out, threads);
}

// The reference bench's input recipe (/root/reference/proj/src/cli.cpp:120-125):
// std::mt19937_64(seed) + std::uniform_real_distribution<double>(0,1).  MT19937-64 is
// the published Matsumoto-Nishimura generator; libstdc++'s generate_canonical<double,53>
// with a 64-bit engine is double(x) / 2^64, clamped below 1.  (tests check this against
// the real std:: classes through oracle/ref_capi.cpp.)
int synth_uniform(uint64_t seed, uint64_t n, int as_f64, void* out) {
    if (!out && n) return -1;
    constexpr int NN = 312, MM = 156;
    constexpr uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull, MATRIX = 0xB5026F5AA96619E9ull;
    std::vector<uint64_t> mt(NN);
    mt[0] = seed;
    for (int i = 1; i < NN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
    int idx = NN;
    for (uint64_t k = 0; k < n; ++k) {
        if (idx >= NN) {
            for (int i = 0; i < NN; ++i) {
                const uint64_t x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM);
                mt[i] = mt[(i + MM) % NN] ^ (x >> 1) ^ ((x & 1ull) ? MATRIX : 0ull);
            }
            idx = 0;
        }
        uint64_t x = mt[idx++];
        x ^= (x >> 29) & 0x5555555555555555ull;
        x ^= (x << 17) & 0x71D67FFFEDA60000ull;
        x ^= (x << 37) & 0xFFF7EEE000000000ull;
        x ^= (x >> 43);
        double u = double(x) * (1.0 / 18446744073709551616.0);
        if (u >= 1.0) u = std::nextafter(1.0, 0.0);
        if (as_f64) static_cast<double*>(out)[k] = u;
        else static_cast<float*>(out)[k] = float(u);
    }
    return 0;
}

}  // namespace wfcu
