// wfc_unicode.cpp -- the per-code-point accessors of wfc/unicode.hpp (proj/src/unicode.cpp:11-44, 72-121) for source
// compatibility: single-value helpers, table driven.  No data path of this library goes through them -- tokenize,
// normalize_word, utf8_sanitize and the counting kernels classify bytes on the device.
#include <cstddef>

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

}  // namespace wfc
