// wc_count.cu -- fused tokenizer + counting map for sm_100a, third generation.
//
// Replaces, on the device, the reference's  tokenize -> normalize_word -> ++counts[word]
// loop (/root/reference/proj/src/text.cpp:9-57, proj/src/unicode.cpp:90-121,
// proj/src/pipeline.cpp:131-139).  Bytes are read from HBM once; tokens never reach HBM.
//
// The kernel is bound by instruction issue and by the shared-memory pipe, not by HBM (DESIGN.md
// section 4.1), so every choice below is about warp-instructions and shared-memory wavefronts
// per corpus byte:
//   * a ROW is 1 KiB = two interleaved 512-byte halves; lane l owns bytes [16l,16l+16) of
//     each half, so both 16-byte global loads of a warp are fully coalesced and both
//     16-byte shared stores are conflict free, while the per-row bookkeeping (shuffles,
//     prefix sum, loop control) is paid once per 1 KiB;
//   * phase 1 classifies 4 bytes per operation (SWAR range tests, answer in bit 7 of each
//     byte lane), folds A-Z in the same registers, and gathers the flag bits into 16-bit
//     masks with dp4a -- integer dot products run on the FMA pipe, which byte work leaves idle;
//     the FOLDED bytes are what the warp's shared-memory ring keeps;
//   * token boundaries are found bit-parallel: with N = non-space bits and A = alnum bits
//     of the fragments that END in the lane's chunk, F = A & ~(N + A) is the first word
//     character of every fragment (the carry of the addition runs along each fragment),
//     and the same expression on the bit-reversed masks gives the last one.  The k-th F
//     pairs with the k-th L: a token is (position, length), no per-byte loop, no look-ahead
//     (everything is resolved backwards from the whitespace byte that ends the fragment);
//   * phase 2 takes one queued token per lane: unaligned fetch of the folded bytes from
//     the ring, length mask from a table, multiply hash, one 16-byte load of a two-key
//     bucket of the CTA-wide combiner, shared-memory atomic count; two tokens per lane per
//     trip.  Misses are buffered per warp; every lane owns a drain slot whose global slot key
//     arrives by cp.async while the passes go on, then one RED.ADD.64 (table_add --
//     ATOMG.CAS.128 -- only for a first occurrence or a long probe sequence);
//   * whatever byte-class logic cannot decide exactly -- a byte >= 0x80 in the fragment (the HI
//     variant keeps two-byte letters and the E2 80 xx punctuation), a fragment whose start is
//     out of sight, a token longer than 16 bytes -- is appended to the deferred list and handled
//     by wc_slow_kernel (wordcount.cu), an exact restatement of the reference's UTF-8 rules.
#include <cstdlib>
#include <type_traits>

#include "wc_count_common.cuh"

namespace wfcu {

namespace cnt3 {
using namespace cntc;

constexpr int kHalf = 512;                         // 32 lanes x 16 bytes
constexpr int kRow = 2 * kHalf;
constexpr int kGuard = 32;                         // bytes in front of a ring slot; the last 16 mirror the previous row's tail
constexpr int kSlotStride = kGuard + kRow;         // 1056
constexpr int kRingBytes = 2 * kSlotStride + 32;   // two slots + slack for the unaligned fetch
constexpr int kQueueCap = 512;                     // u16 entries per warp: (len-1) << 12 | ring position, 0 = dead
constexpr int kMissCap = 64;

// Chunks with bytes >= 0x80.  Two-byte sequences C3..DF 80..BF (U+00C0..U+07FF: Latin-1 letters,
// Latin Extended, Greek, Cyrillic, ...) stay on the fast path: every such code point is a word
// character except U+00D7 and U+00F7, none is whitespace, and the only case fold in the range
// (U+00C0..U+00DE -> +0x20, proj/src/unicode.cpp:117-121) is "second byte | 0x20 after C3", which
// keeps the length.  This function produces the per-byte flags; pairing leads with continuation
// bytes is done on the gathered masks (hi_masks_finish).  prev_c3: 0x80000000 if the byte in front
// of the chunk is 0xC3.
//
// The same for the General Punctuation block's E2 80 90..A7 / B0..BF (U+2010..U+2027, U+2030..U+203F:
// typographic apostrophes and quotes, dashes, ellipsis ...): valid, never word characters, never
// whitespace, so their three bytes behave like ASCII punctuation (kept inside a token, trimmed at
// its edges) and need not defer the fragment.
//
// Round 2: three-byte LETTERS too.  A sequence  lead second third  with lead in E0, E1, E3..EE (E2 and EF hold the
// punctuation, whitespace and specials the reference's is_word_char / is_unicode_space single out,
// proj/src/unicode.cpp:90-115) is a word character that nothing folds, provided it is strict UTF-8 (E0 needs a second
// byte >= A0, ED one <= 9F) and is not one of the two pinned exceptions inside those leads: E1 9A xx (U+1680 OGHAM
// SPACE MARK is whitespace; its whole 64-code-point block is left to the slow path) and E3 80 xx (U+3000..U+303F).
// Devanagari, Hangul, Georgian, Vietnamese tone letters (E1 BA/BB xx), kana, ideographs ...: their fragments used to
// go to the one-thread-per-fragment slow kernel.  l3 flags those leads, b2 the continuation bytes that may NOT follow
// the lead in front of them; the pairing is done on the gathered masks like the rest.
struct HiMasks { u32 s7, a7, h7, c7, l7, x7, e7, z7, k7, l3, b2; };   // whitespace, ASCII alnum, >= 0x80, continuation, lead C3..DF,
                                                                      // x / division sign, == E2, == 80, third byte of the punctuation
                                                                      // above, three-byte letter lead, bad second byte
// prev_byte: the byte in front of the chunk (0 if unknown / none).  U3 = false: the three-byte-letter flags are not
// computed (rows without such a lead: accented Latin, Greek, Cyrillic, typographic punctuation keep their round-1 cost).
template <bool U3>
__device__ __forceinline__ HiMasks classify16_hi(const uint4& x, u32 prev_byte, uint4& f) {
    const u32 M = 0x80808080u;
    const u32 xs[4] = {x.x, x.y, x.z, x.w};
    u32 fs[4];
    u32 acc[11][2];       // 128 * (8-bit mask) of words {0,1} and {2,3}, per class
    u32 c3_prev = prev_byte == 0xC3u ? 0x80000000u : 0u;
    u32 e0_prev = prev_byte == 0xE0u ? 0x80000000u : 0u, ed_prev = prev_byte == 0xEDu ? 0x80000000u : 0u;
    u32 e1_prev = prev_byte == 0xE1u ? 0x80000000u : 0u, e3_prev = prev_byte == 0xE3u ? 0x80000000u : 0u;
#pragma unroll
    for (int pair = 0; pair < 2; ++pair) {       // two words at a time keeps the live flag words few
        u32 fl[11][2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int w = 2 * pair + k;
            const u32 xw = xs[w], v = xw & 0x7F7F7F7Fu, y = v | 0x20202020u, nx = ~xw;
            const u32 t = (y + 0x1F1F1F1Fu) & ~(y + 0x05050505u) & M & nx;          // ASCII letters
            const u32 u = (v + 0x50505050u) & ~(v + 0x46464646u) & M & nx;          // ASCII digits
            const u32 z = (v ^ 0x20202020u) + 0x7F7F7F7Fu;
            fl[0][k] = (~z | ((v + 0x77777777u) & ~(v + 0x72727272u))) & M & nx;    // whitespace
            fl[1][k] = t | u;                                                         // ASCII alnum
            fl[2][k] = xw & M;                                                        // >= 0x80
            const u32 co = xw & ~(xw << 1) & M;                                       // 10xxxxxx
            fl[3][k] = co;
            fl[4][k] = xw & (v + 0x3D3D3D3Du) & ~(v + 0x20202020u) & M;              // C3..DF
            const u32 c3 = xw & ~((v ^ 0x43434343u) + 0x7F7F7F7Fu) & M;              // == 0xC3
            const u32 after_c3 = __funnelshift_l(c3_prev, c3, 8);                     // the byte in front is 0xC3
            c3_prev = c3;
            const u32 lat = co & after_c3;                                            // second byte of U+00C0..U+00FF
            const u32 fold_hi = lat & ~(v + 0x61616161u);                             // 80..9E -> A0..BE (97 is deferred anyway)
            fl[5][k] = lat & ~(((v & 0x5F5F5F5Fu) ^ 0x17171717u) + 0x7F7F7F7Fu);      // C3 97 (x) and C3 B7 (division sign)
            fs[w] = xw | ((t | fold_hi) >> 2);
            fl[6][k] = xw & ~((v ^ 0x62626262u) + 0x7F7F7F7Fu) & M;                   // == 0xE2
            fl[7][k] = xw & ~(v + 0x7F7F7F7Fu) & M;                                   // == 0x80
            fl[8][k] = co & (((v + 0x70707070u) & ~(v + 0x58585858u)) | (v + 0x50505050u));   // 90..A7 or B0..BF
            fl[9][k] = 0;
            fl[10][k] = 0;
            if (!U3) continue;
            fl[9][k] = xw & (v + 0x20202020u) & ~(v + 0x11111111u) & ~fl[6][k] & M;           // E0..EE without E2
            const u32 e0 = xw & ~((v ^ 0x60606060u) + 0x7F7F7F7Fu) & M, ed = xw & ~((v ^ 0x6D6D6D6Du) + 0x7F7F7F7Fu) & M;
            const u32 e1 = xw & ~((v ^ 0x61616161u) + 0x7F7F7F7Fu) & M, e3 = xw & ~((v ^ 0x63636363u) + 0x7F7F7F7Fu) & M;
            const u32 ge_a0 = v + 0x60606060u;                                                 // bit 7: byte >= A0 (continuation bytes)
            fl[10][k] = co & ((__funnelshift_l(e0_prev, e0, 8) & ~ge_a0) | (__funnelshift_l(ed_prev, ed, 8) & ge_a0) |
                              (__funnelshift_l(e1_prev, e1, 8) & ~((v ^ 0x1A1A1A1Au) + 0x7F7F7F7Fu)) |
                              (__funnelshift_l(e3_prev, e3, 8) & fl[7][k]));
            e0_prev = e0; ed_prev = ed; e1_prev = e1; e3_prev = e3;
        }
#pragma unroll
        for (int c = 0; c < 11; ++c) acc[c][pair] = (c < 9 || U3) ? gather8(fl[c][0], fl[c][1], 0) : 0u;
    }
    f = make_uint4(fs[0], fs[1], fs[2], fs[3]);
    HiMasks m;
    m.s7 = acc[0][1] * 256u + acc[0][0];
    m.a7 = acc[1][1] * 256u + acc[1][0];
    m.h7 = acc[2][1] * 256u + acc[2][0];
    m.c7 = acc[3][1] * 256u + acc[3][0];
    m.l7 = acc[4][1] * 256u + acc[4][0];
    m.x7 = acc[5][1] * 256u + acc[5][0];
    m.e7 = acc[6][1] * 256u + acc[6][0];
    m.z7 = acc[7][1] * 256u + acc[7][0];
    m.k7 = acc[8][1] * 256u + acc[8][0];
    m.l3 = acc[9][1] * 256u + acc[9][0];
    m.b2 = acc[10][1] * 256u + acc[10][0];
    return m;
}
// Pairs leads with continuation bytes on packed masks (low 16 bits = half a, high = half b).
// lead_before: bit 0 / bit 16 set if the byte in front of half a / b is a lead C3..DF.
// tails_before: per half, bits 0,1 = "the byte two / one in front of the chunk is E2", bit 2 = "the
// byte in front is 80" (hi_tails of the chunk in front).
// Out: A gains the bytes of valid two-byte letters; H = bytes the fast path must not touch
// (anything else >= 0x80, x / division sign, a lead without its continuation byte -- that lead
// itself when it lies in the same chunk; bad_first tells the caller to flag the LAST byte of the
// chunk in front when the unmatched lead is there).  A chunk cannot know whether an E2 (80) at its
// end will be completed, so it flags them; clear_before tells the caller which of the last two
// bytes of the chunk in front the sequences completed HERE clear again.
struct HiIn { u32 Hi, C, L, X, E2, Z, K, L3, B2; };
// per half: bits 0,1 = the second-last / last byte is E2, bit 2 = the last byte is 80, bit 3 = the last byte is a
// three-byte letter lead, bit 4 = the second-last byte is one and the last byte may follow it
__device__ __forceinline__ u32 hi_tails(const HiIn& in) {
    return ((in.E2 >> 14) & 0x00030003u) | ((in.Z >> 13) & 0x00040004u) | ((in.L3 >> 12) & 0x00080008u) |
           ((in.L3 >> 10) & (in.C >> 11) & ~(in.B2 >> 11) & 0x00100010u);
}
// alnum_before: the bytes among them that are word characters (the first bytes of a three-byte letter completed here).
template <bool U3>
__device__ __forceinline__ void hi_masks_finish(const HiIn& in, u32 lead_before, u32 tails_before, u32& A, u32& H,
                                                u32& bad_first, u32& clear_before, u32& alnum_before) {
    const u32 Lsh = ((in.L << 1) & 0xFFFEFFFEu) | (lead_before & 0x00010001u);  // the byte in front is a lead
    const u32 validC = in.C & Lsh;
    const u32 badnext = Lsh & ~in.C;                                              // successor of an unmatched lead
    bad_first = badnext & 0x00010001u;
    const u32 Zsh = ((in.Z << 1) & 0xFFFEFFFEu) | ((tails_before >> 2) & 0x00010001u);   // the byte in front is 80
    const u32 Esh = ((in.E2 << 2) & 0xFFFCFFFCu) | (tails_before & 0x00030003u);          // the byte two in front is E2
    const u32 T3 = in.K & Zsh & Esh;                                              // third byte of a punctuation sequence
    const u32 P3 = T3 | ((T3 >> 1) & 0x7FFF7FFFu) | ((T3 >> 2) & 0x3FFF3FFFu);    // its bytes inside the chunk
    // three-byte letters: second = continuation after a lead that admits it, third = continuation after a second.
    // Only sequences COMPLETED here are cleared (those that began in the chunk in front through clear_before): a
    // lead or lead + second at the end of a chunk stays flagged until the next chunk sees the rest.
    u32 thr = 0;
    if (U3) {
        const u32 L3sh = ((in.L3 << 1) & 0xFFFEFFFEu) | ((tails_before >> 3) & 0x00010001u);
        const u32 sec = in.C & L3sh & ~in.B2;
        const u32 secsh = ((sec << 1) & 0xFFFEFFFEu) | ((tails_before >> 4) & 0x00010001u);
        thr = in.C & secsh;
    }
    const u32 G3 = thr | ((thr >> 1) & 0x7FFF7FFFu) | ((thr >> 2) & 0x3FFF3FFFu);
    const u32 done = T3 | thr;                                                    // third bytes of either kind
    clear_before = ((done & 0x00010001u) << 15) | ((done & 0x00010001u) << 14) | ((done & 0x00020002u) << 14);
    alnum_before = ((thr & 0x00010001u) << 15) | ((thr & 0x00010001u) << 14) | ((thr & 0x00020002u) << 14);
    H = (in.Hi & ~(validC | in.L | P3 | G3)) | in.X | badnext | ((badnext >> 1) & 0x7FFF7FFFu);
    A |= (validC | in.L | G3) & ~H;
}

template <int WARPS, int SETS, int MSLOTS>
struct __align__(1024) Smem {
    uint16_t queue[WARPS][kQueueCap];          // 1 KiB per warp, 1 KiB aligned (index wrap by OR)
    ulonglong2 sk[SETS];                       // short combiner: two keys (tokens <= 8 bytes, little-endian) per set
    uint2 scnt[SETS];                          //                 and their counts
    u64 mk0[MSLOTS];                           // medium combiner (9..16 bytes): key low, key high, count
    u64 mk1[MSLOTS];
    u64 lomask[16];                            // [len-1] -> mask of key bytes 0..7
    u64 himask[16];                            // [len-1] -> mask of key bytes 8..15
    ulonglong2 miss[WARPS][kMissCap];
    uint4 landing[WARPS][32];                  // where the global slot keys of a drain in flight arrive (cp.async)
    uint4 ring[WARPS][kRingBytes / 16];
    u32 mcnt[MSLOTS];
    u32 dummy[WARPS];                          // where the count of a token that missed goes (no branch around the atomic)
};

}  // namespace cnt3

using namespace cnt3;

// text[0..n): documents concatenated with whitespace between them by the caller.
// Position n acts as a whitespace byte, so does "position -1".
// Two variants of the body, both exact: HI = false treats every fragment with a byte >= 0x80 as
// the slow kernel's business (the ASCII corpora of the benchmarks never pay for anything else);
// HI = true keeps two-byte letters (accented Latin, Greek, Cyrillic ...) on the fast path, U3K three-byte letters
// as well, WIDE replaces the two combiners by one for tokens of up to 16 bytes.  The variant is chosen per call from
// a sample of the text (wc_count_kernel below): the choice affects speed only.
template <int WARPS, int SETS, int MSLOTS, bool HI, bool WIDE, bool U3K>
__device__ __forceinline__ void wc_count_body(const uint8_t* __restrict__ text, u64 n, u32 rows_per_warp, u32 one,
                                              const TableView& gt) {
    extern __shared__ uint8_t smem_raw[];
    typedef Smem<WARPS, SETS, MSLOTS> SM;
    const u32 sbase = (u32)__cvta_generic_to_shared(smem_raw);
    SM& sm = *reinterpret_cast<SM*>(smem_raw + ((1024u - (sbase & 1023u)) & 1023u));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u32 lt_mask = (1u << lane) - 1u;

    for (int i = tid; i < SETS; i += WARPS * 32) { sm.sk[i] = make_ulonglong2(0, 0); sm.scnt[i] = make_uint2(0, 0); }
    for (int i = tid; i < MSLOTS; i += WARPS * 32) { sm.mk0[i] = 0; sm.mk1[i] = 0; sm.mcnt[i] = 0; }
    if (tid < 16) {
        sm.lomask[tid] = tid < 8 ? (~0ull >> (56 - 8 * tid)) : ~0ull;
        sm.himask[tid] = tid < 8 ? 0ull : (~0ull >> (120 - 8 * tid));
    }
    for (int i = lane; i < kRingBytes / 16; i += 32) sm.ring[warp][i] = make_uint4(0, 0, 0, 0);
    __syncthreads();

    const u32 n_rows = (u32)(n / kRow) + 1;            // the last row holds the virtual whitespace at n
    const u32 full_rows = (u32)(n / kRow);             // rows [0, full_rows) lie entirely inside the text
    const u32 gw = blockIdx.x * WARPS + warp;
    const u64 rb64 = (u64)gw * rows_per_warp;
    const u32 r_begin = rb64 < n_rows ? (u32)rb64 : n_rows;
    const u32 r_end = (rb64 + rows_per_warp < n_rows) ? (u32)(rb64 + rows_per_warp) : n_rows;

    uint8_t* ring = reinterpret_cast<uint8_t*>(sm.ring[warp]);
    uint4* missbuf = reinterpret_cast<uint4*>(sm.miss[warp]);
    const u32 q_s = (u32)__cvta_generic_to_shared(sm.queue[warp]);   // 1 KiB aligned: index wrap is an OR
    u32 inserted = 0;             // global slots this lane claimed (first occurrences)
    u32 my_tokens = 0;            // per lane (careful rows)
    u32 warp_tokens = 0;          // warp-uniform (fast rows)
    u32 qhead = 0, qtail = 0;     // token queue (warp-uniform, free running, in entries)
    u32 qrd = lane * 2;           // byte offset of this lane's entry in the next pass (free running)
    u32 mhead = 0, mtail = 0;     // miss buffer (warp-uniform, free running)
    bool filling = true;          // look for empty combiner ways: while the combiner fills, and every 16th row after

    auto q_store = [&](u32 off2, u32 v) {
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(q_s | (off2 & (2 * kQueueCap - 2))), "r"(v) : "memory");
    };
    auto q_load = [&](u32 off2) {
        u32 v;
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(q_s | (off2 & (2 * kQueueCap - 2))) : "memory");
        return v;
    };

    // ---- misses -> global table ------------------------------------------------------
    // Keys wait in the warp's miss buffer (little-endian packed).  Every lane owns one drain
    // slot; a round (a) finishes what landed: the slot holds the lane's key -> one RED.ADD.64
    // on its count; another key -> next slot of the probe sequence, still in flight; an empty
    // slot (first global occurrence) or a long probe sequence -> table_add from scratch; and
    // (b) hands buffered keys to the free lanes: key -> registers, slot index from the hash,
    // cp.async of the slot's 16-byte key into the lane's landing word.  No register waits on
    // the L2 round trip, which overlaps the passes between two rounds.
    uint4* landing = sm.landing[warp];
    u32 dk0 = 0, dk1 = 0, dk2 = 0, dk3 = 0;         // the lane's key in flight (big-endian words)
    u32 didx = 0, dleft = 0;                        // slot being fetched; probes left (0 = lane free)
    auto drain_round = [&]() {
        const u32 dst = (u32)__cvta_generic_to_shared(landing + lane);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        if (dleft) {
            const uint4 cur = landing[lane];        // {k0 low, k0 high, k1 low, k1 high}
            if (cur.x == dk1 && cur.y == dk0 && cur.z == dk3 && cur.w == dk2) {
                atomicAdd(&gt.slots[didx].count, 1ull);
                dleft = 0;
            } else if ((cur.x | cur.y) == 0 || --dleft == 0) {
                // the synchronous insertion continues where the asynchronous probes stopped: at the empty slot just
                // seen (claimed without another load), or behind the last slot that held another key
                // (WIDE kernels only: their texts bring a million first occurrences per GB, +5 % there; in the narrow
                // kernel the extra operands cost 1 % on cfg3 -- it sits at its register limit)
                if constexpr (WIDE) {
                    const bool empty = (cur.x | cur.y) == 0;
                    table_add_from(gt, empty ? didx : ((didx + 1) & (u32)gt.mask), empty, ((u64)dk0 << 32) | dk1,
                                   ((u64)dk2 << 32) | dk3, 1ull, &inserted);
                } else {
                    table_add(gt, ((u64)dk0 << 32) | dk1, ((u64)dk2 << 32) | dk3, 1ull, &inserted);
                }
                dleft = 0;
            } else {
                didx = (didx + 1) & (u32)gt.mask;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gt.slots + didx) : "memory");
            }
        }
        __syncwarp();                               // miss-buffer entries were written by other lanes
        const u32 freem = __ballot_sync(kFull, dleft == 0);
        const u32 avail = mtail - mhead;
        const u32 rank = __popc(freem & lt_mask);
        if (dleft == 0 && rank < avail) {
            const uint4 k = missbuf[(mhead + rank) & (kMissCap - 1)];
            dk0 = bswap32(k.x); dk1 = bswap32(k.y); dk2 = bswap32(k.z); dk3 = bswap32(k.w);
            didx = mix32(((u64)dk0 << 32) | dk1, ((u64)dk2 << 32) | dk3) & (u32)gt.mask;
            dleft = 3;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gt.slots + didx) : "memory");
        }
        mhead += min((u32)__popc(freem), avail);
        asm volatile("cp.async.commit_group;" ::: "memory");
        __syncwarp();                               // the entries just read may be overwritten by the next append
    };
    // called between passes
    auto drain_step = [&]() {
        if (mtail - mhead >= 32) drain_round();
    };
    // room for `extra` more keys (rare: more than one miss in two tokens for a while)
    auto make_room = [&](u32 extra) {
        while ((mtail - mhead) + extra > (u32)kMissCap) drain_round();
    };
    // branch-free append
    auto push_misses = [&](bool miss, u32 k0, u32 k1, u32 k2, u32 k3) {
        const u32 mm = __ballot_sync(kFull, miss);
        if ((mtail - mhead) + __popc(mm) > (u32)kMissCap) make_room(__popc(mm));
        const u32 at = (mtail + __popc(mm & lt_mask)) & (kMissCap - 1);
        if (miss) missbuf[at] = make_uint4(k0, k1, k2, k3);
        mtail += __popc(mm);
    };

    // Two candidate slots in one 16-byte bucket; straight-line hit path, claims behind a
    // warp-uniform branch (only while the table fills).  A key present in two places (two
    // buckets can never hold it, but the global table may) is harmless: the flush adds.
    const u32 sk_s = (u32)__cvta_generic_to_shared(sm.sk);
    auto short_add = [&](u32 b0, u32 b1, u32 h, bool live) -> bool {
        const u32 set = __umulhi(h, (u32)SETS);
        u32 c0l, c0h, c1l, c1h;   // one LDS.128; a stale value only costs a redundant claim attempt (keys never change once set)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c0l), "=r"(c0h), "=r"(c1l), "=r"(c1h) : "r"(sk_s + set * 16u));
        const bool hit0 = c0l == b0 && c0h == b1, hit1 = c1l == b0 && c1h == b1;
        const bool found = (hit0 || hit1) && live;
        if (found) atomicAdd(reinterpret_cast<u32*>(sm.scnt) + set * 2u + (hit1 ? 1u : 0u), 1u);   // ATOMS.POPC.INC
        // Claim an empty slot for FUTURE occurrences (a valid key never has a zero low word:
        // its first byte is a word character).  This occurrence still goes to the global table,
        // so nothing flows out of the rare branch and the hit path stays straight-line.
        const bool can_claim = live && !found && (c0l == 0 || c1l == 0);
        if (__any_sync(kFull, can_claim)) {
            if (can_claim) {
                const u64 key = ((u64)b1 << 32) | b0;
                u64* slot = reinterpret_cast<u64*>(&sm.sk[set]);
                u64 old = 1;
                if (c0l == 0) old = atomicCAS(slot, 0ull, key);
                if (old != 0 && old != key) atomicCAS(slot + 1, 0ull, key);
            }
        }
        return found;
    };

    // one pass of phase 2: `count` (<= 32) queued tokens, one per lane.  general = some
    // queued token may be longer than 8 bytes (warp-uniform, decided per row).
    auto token_pass = [&](auto full, u32 count, bool general) {
        u32 e = q_load(qrd);
        if (!decltype(full)::value && lane >= count) e = 0;
        qrd += 2 * count;
        qhead += count;
        const bool live = e != 0;
        const u32* wp = reinterpret_cast<const u32*>(ring + (e & 0xFFCu));
        const u32 sh = e << 3;                       // funnel shifts use the low 5 bits: (pos & 3) * 8
        const u32 li = (e >> 9) & 0x78u;             // (len-1) * 8
        const u32 w0 = wp[0], w1 = wp[1], w2 = wp[2];
        u32 b0 = __funnelshift_r(w0, w1, sh);
        u32 b1 = __funnelshift_r(w1, w2, sh);
        const uint2 lm = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(sm.lomask) + li);
        b0 &= lm.x; b1 &= lm.y;
        if (!general) {
            // every token of this pass fits 8 bytes
            const u32 h = b0 * 0x9E3779B1u + b1 * 0x85EBCA77u;
            const bool ok = short_add(b0, b1, h, live);
            push_misses(live && !ok, b0, b1, 0u, 0u);
        } else {
            const u32 w3 = wp[3], w4 = wp[4];
            u32 b2 = __funnelshift_r(w2, w3, sh);
            u32 b3 = __funnelshift_r(w3, w4, sh);
            const uint2 hm = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(sm.himask) + li);
            b2 &= hm.x; b3 &= hm.y;
            const bool is_medium = e >= 0x8000u;
            u32 h = b0 * 0x9E3779B1u + b1 * 0x85EBCA77u;
            bool ok = short_add(b0, b1, h, live && !is_medium);      // votes across the warp: every lane calls it
            if (is_medium) {
                h += b2 * 0xC2B2AE3Du + b3 * 0x27D4EB2Fu;
                h ^= h >> 16;
                h *= 0x2C1B3C6Du;
                ok = medium_add(sm.mk0, sm.mk1, sm.mcnt, MSLOTS - 1, ((u64)b1 << 32) | b0, ((u64)b3 << 32) | b2, h);
            }
            push_misses(live && !ok, b0, b1, b2, b3);
        }
    };
    // Two full passes at once (64 queued tokens, two per lane), short tokens only: the two
    // dependency chains (queue -> ring -> bucket -> atomic) interleave, which is worth more
    // than occupancy on this latency-bound stretch of the kernel.
    auto token_pass2 = [&]() {
        const u32 e0 = q_load(qrd), e1 = q_load(qrd + 64);
        qrd += 128;
        qhead += 64;
        const u32* wp0 = reinterpret_cast<const u32*>(ring + (e0 & 0xFFCu));
        const u32* wp1 = reinterpret_cast<const u32*>(ring + (e1 & 0xFFCu));
        const u32 x0 = wp0[0], x1 = wp0[1], x2 = wp0[2];
        const u32 y0 = wp1[0], y1 = wp1[1], y2 = wp1[2];
        const uint2 lm0 = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(sm.lomask) + ((e0 >> 9) & 0x78u));
        const uint2 lm1 = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(sm.lomask) + ((e1 >> 9) & 0x78u));
        const u32 a0 = __funnelshift_r(x0, x1, e0 << 3) & lm0.x, a1 = __funnelshift_r(x1, x2, e0 << 3) & lm0.y;
        const u32 b0 = __funnelshift_r(y0, y1, e1 << 3) & lm1.x, b1 = __funnelshift_r(y1, y2, e1 << 3) & lm1.y;
        const u32 seta = __umulhi(a0 * 0x9E3779B1u + a1 * 0x85EBCA77u, (u32)SETS);
        const u32 setb = __umulhi(b0 * 0x9E3779B1u + b1 * 0x85EBCA77u, (u32)SETS);
        u32 p0, p1, p2, p3, r0, r1, r2, r3;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(p0), "=r"(p1), "=r"(p2), "=r"(p3) : "r"(sk_s + seta * 16u));
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(sk_s + setb * 16u));
        const bool ha0 = p0 == a0 && p1 == a1, ha1 = p2 == a0 && p3 == a1;
        const bool hb0 = r0 == b0 && r1 == b1, hb1 = r2 == b0 && r3 == b1;
        const bool live0 = e0 != 0, live1 = e1 != 0;
        const bool fa = (ha0 || ha1) && live0, fb = (hb0 || hb1) && live1;
        // round 2 (from the fourth-generation experiment, +1.9 %): a token that missed counts into the warp's dummy word
        // -- no branch around the two ATOMS.POPC.INC -- and empty ways are only looked for while the combiner fills
        atomicAdd(fa ? reinterpret_cast<u32*>(sm.scnt) + seta * 2u + (ha1 ? 1u : 0u) : &sm.dummy[warp], 1u);
        atomicAdd(fb ? reinterpret_cast<u32*>(sm.scnt) + setb * 2u + (hb1 ? 1u : 0u) : &sm.dummy[warp], 1u);
        const bool ca = live0 && !fa && (p0 == 0 || p2 == 0), cb = live1 && !fb && (r0 == 0 || r2 == 0);
        if (filling && __any_sync(kFull, ca || cb)) {
            if (ca) {
                const u64 key = ((u64)a1 << 32) | a0;
                u64* slot = reinterpret_cast<u64*>(&sm.sk[seta]);
                u64 old = 1;
                if (p0 == 0) old = atomicCAS(slot, 0ull, key);
                if (old != 0 && old != key) atomicCAS(slot + 1, 0ull, key);
            }
            if (cb) {
                const u64 key = ((u64)b1 << 32) | b0;
                u64* slot = reinterpret_cast<u64*>(&sm.sk[setb]);
                u64 old = 1;
                if (r0 == 0) old = atomicCAS(slot, 0ull, key);
                if (old != 0 && old != key) atomicCAS(slot + 1, 0ull, key);
            }
        }
        // both miss lists in one append
        const bool m0 = live0 && !fa, m1 = live1 && !fb;
        const u32 mm0 = __ballot_sync(kFull, m0), mm1 = __ballot_sync(kFull, m1);
        const u32 n0 = __popc(mm0);
        if ((mtail - mhead) + n0 + __popc(mm1) > (u32)kMissCap) make_room(n0 + __popc(mm1));
        if (m0) missbuf[(mtail + __popc(mm0 & lt_mask)) & (kMissCap - 1)] = make_uint4(a0, a1, 0u, 0u);
        if (m1) missbuf[(mtail + n0 + __popc(mm1 & lt_mask)) & (kMissCap - 1)] = make_uint4(b0, b1, 0u, 0u);
        mtail += n0 + __popc(mm1);
    };
    // WIDE variant (round 2): text where words of 9..16 bytes are common (English prose, the 1 M-word corpus) sent every
    // pass through the one-token general form above -- 170 instructions per 32 tokens against 125 per 64 for the
    // two-token short form.  Here ONE direct-mapped combiner of 16-byte keys (the medium table, instantiated with
    // most of the shared memory) takes every token of up to 16 bytes, two per lane and pass: fetch of five words,
    // both length masks, one hash over the four key words, key low / key high by two 8-byte loads (low first: a
    // published low word implies the high word is in place, medium_add's claim protocol), one shared atomic.
    auto wide_pass = [&](u32 count) {      // count <= 64
        u32 e0 = q_load(qrd), e1 = q_load(qrd + 64);
        if ((u32)lane >= count) e0 = 0;
        if ((u32)lane + 32u >= count) e1 = 0;
        qrd += 2 * count;
        qhead += count;
        const bool live0 = e0 != 0, live1 = e1 != 0;
        const u32* wp0 = reinterpret_cast<const u32*>(ring + (e0 & 0xFFCu));
        const u32* wp1 = reinterpret_cast<const u32*>(ring + (e1 & 0xFFCu));
        const u32 x0 = wp0[0], x1 = wp0[1], x2 = wp0[2], x3 = wp0[3], x4 = wp0[4];
        const u32 y0 = wp1[0], y1 = wp1[1], y2 = wp1[2], y3 = wp1[3], y4 = wp1[4];
        const u32 li0 = (e0 >> 9) & 0x78u, li1 = (e1 >> 9) & 0x78u;
        const uint2 lm0 = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(sm.lomask) + li0);
        const uint2 hm0 = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(sm.himask) + li0);
        const uint2 lm1 = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(sm.lomask) + li1);
        const uint2 hm1 = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(sm.himask) + li1);
        const u32 a0 = __funnelshift_r(x0, x1, e0 << 3) & lm0.x, a1 = __funnelshift_r(x1, x2, e0 << 3) & lm0.y;
        const u32 a2 = __funnelshift_r(x2, x3, e0 << 3) & hm0.x, a3 = __funnelshift_r(x3, x4, e0 << 3) & hm0.y;
        const u32 b0 = __funnelshift_r(y0, y1, e1 << 3) & lm1.x, b1 = __funnelshift_r(y1, y2, e1 << 3) & lm1.y;
        const u32 b2 = __funnelshift_r(y2, y3, e1 << 3) & hm1.x, b3 = __funnelshift_r(y3, y4, e1 << 3) & hm1.y;
        u32 ha = a0 * 0x9E3779B1u + a1 * 0x85EBCA77u + a2 * 0xC2B2AE3Du + a3 * 0x27D4EB2Fu;
        u32 hb = b0 * 0x9E3779B1u + b1 * 0x85EBCA77u + b2 * 0xC2B2AE3Du + b3 * 0x27D4EB2Fu;
        ha ^= ha >> 16; ha *= 0x2C1B3C6Du;
        hb ^= hb >> 16; hb *= 0x2C1B3C6Du;
        const u32 ia = __umulhi(ha, (u32)MSLOTS), ib = __umulhi(hb, (u32)MSLOTS);
        const u64 ka0 = *reinterpret_cast<volatile u64*>(sm.mk0 + ia), kb0 = *reinterpret_cast<volatile u64*>(sm.mk0 + ib);
        const u64 ka1 = *reinterpret_cast<volatile u64*>(sm.mk1 + ia), kb1 = *reinterpret_cast<volatile u64*>(sm.mk1 + ib);
        const u64 wa0 = ((u64)a1 << 32) | a0, wa1 = ((u64)a3 << 32) | a2, wb0 = ((u64)b1 << 32) | b0, wb1 = ((u64)b3 << 32) | b2;
        const bool fa = live0 && ka0 == wa0 && ka1 == wa1, fb = live1 && kb0 == wb0 && kb1 == wb1;
        atomicAdd(fa ? sm.mcnt + ia : &sm.dummy[warp], 1u);
        atomicAdd(fb ? sm.mcnt + ib : &sm.dummy[warp], 1u);
        const bool ca = live0 && !fa && ka0 == 0, cb = live1 && !fb && kb0 == 0;
        if (filling && __any_sync(kFull, ca || cb)) {       // claims for FUTURE occurrences; this one still goes out
            if (ca && atomicCAS(sm.mk0 + ia, 0ull, kSlotLocked) == 0) {
                atomicExch(sm.mk1 + ia, wa1);      // (an atomic: other warps read the high word before they know whether the low one matches)
                __threadfence_block();
                atomicExch(sm.mk0 + ia, wa0);
            }
            if (cb && atomicCAS(sm.mk0 + ib, 0ull, kSlotLocked) == 0) {
                atomicExch(sm.mk1 + ib, wb1);
                __threadfence_block();
                atomicExch(sm.mk0 + ib, wb0);
            }
        }
        const bool m0 = live0 && !fa, m1 = live1 && !fb;
        const u32 mm0 = __ballot_sync(kFull, m0), mm1 = __ballot_sync(kFull, m1);
        const u32 n0 = __popc(mm0);
        if ((mtail - mhead) + n0 + __popc(mm1) > (u32)kMissCap) make_room(n0 + __popc(mm1));
        if (m0) missbuf[(mtail + __popc(mm0 & lt_mask)) & (kMissCap - 1)] = make_uint4(a0, a1, a2, a3);
        if (m1) missbuf[(mtail + n0 + __popc(mm1 & lt_mask)) & (kMissCap - 1)] = make_uint4(b0, b1, b2, b3);
        mtail += n0 + __popc(mm1);
    };
    const std::true_type kFullPass{};
    const std::false_type kPartialPass{};

    if (r_begin < r_end) {
        // lane's two chunks of a row: bytes [16l,16l+16) of each half; zero past n
        auto load_row = [&](u32 row, uint4& xa, uint4& xb) {
            if (row < full_rows) {
                const uint4* p = reinterpret_cast<const uint4*>(text + (u64)row * kRow) + lane;
                xa = ldg_stream(p);
                xb = ldg_stream(p + 32);
            } else {
                xa = make_uint4(0, 0, 0, 0);
                xb = xa;
                if (row < r_end) {      // the last row of the text
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const u64 g = (u64)row * kRow + (u64)half * kHalf + (u64)lane * 16;
                        uint4 v = make_uint4(0, 0, 0, 0);
                        if (g + 16 <= n) {
                            v = *reinterpret_cast<const uint4*>(text + g);
                        } else if (g < n) {
                            u32 w[4] = {0, 0, 0, 0};
                            for (u32 k = 0; k < (u32)(n - g); ++k) w[k >> 2] |= (u32)text[g + k] << (8 * (k & 3));
                            v = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                        if (half == 0) xa = v; else xb = v;
                    }
                }
            }
        };

        // masks of the chunk in front of the strip (16 bits): "position -1" is whitespace
        u32 carryS = 0xFFFFu, carryA = 0, carryH = 0;
        u32 carryL = 0, carryC3 = 0;   // HI: lead mask of that chunk; its last byte
        u32 carryT = 0;                // HI: hi_tails of that chunk (E2 / 80 in its last two bytes)
        bool general_prev = false;
        if (r_begin > 0) {
            // the 16 bytes in front of the strip: predecessor masks for lane 0, folded bytes for the guard
            const uint4 x = *reinterpret_cast<const uint4*>(text + (u64)r_begin * kRow - 16);
            uint4 f;
            if constexpr (HI) {
                // what lies in front of THEM is unknown: a leading continuation byte is flagged (conservative)
                const HiMasks m = classify16_hi<U3K>(x, 0u, f);
                u32 A = m.a7 >> 7, H, bad_first, clear_before, alnum_before;
                const HiIn in{m.h7 >> 7, m.c7 >> 7, m.l7 >> 7, m.x7 >> 7, m.e7 >> 7, m.z7 >> 7, m.k7 >> 7, m.l3 >> 7, m.b2 >> 7};
                hi_masks_finish<U3K>(in, 0u, 0u, A, H, bad_first, clear_before, alnum_before);
                carryS = m.s7 >> 7; carryA = A & 0xFFFFu; carryH = H & 0xFFFFu; carryL = (m.l7 >> 7) & 0xFFFFu;
                carryT = hi_tails(in) & 0xFFFFu;
                carryC3 = x.w >> 24;
            } else {
                const Masks m = classify16<false>(x, one, f);
                carryS = m.s7 >> 7; carryA = m.a7 >> 7; carryH = m.h7 >> 7;
            }
            if (lane == 0) *reinterpret_cast<uint4*>(ring + (r_begin & 1u) * kSlotStride + 16) = f;
        }
        uint4 nxa, nxb;
        load_row(r_begin, nxa, nxb);

        for (u32 row = r_begin; row < r_end; ++row) {
            const uint4 xa = nxa, xb = nxb;
            filling = row - r_begin < 64u || (row & 15u) == 0;
            const u32 slotpos = (row & 1u) * kSlotStride;

            // ------------------------------ phase 1 ------------------------------
            u32 S, A, H = 0;
            uint4 fa, fb;
            const u32 anyhi = (xa.x | xa.y | xa.z | xa.w | xb.x | xb.y | xb.z | xb.w) & 0x80808080u;
            const bool ascii_row = !__any_sync(kFull, anyhi != 0) && (carryH | carryL) == 0;
            u32 pH_fix = 0, pH_clear = 0, pA_set = 0, H_open = 0;
            if (ascii_row) {
                const Masks ma = classify16<true>(xa, one, fa), mb = classify16<true>(xb, one, fb);
                S = pack7(ma.s7, mb.s7);
                A = pack7(ma.a7, mb.a7);
                carryC3 = 0;
            } else if constexpr (HI) {
                // is the byte in front of each chunk 0xC3 (chunk a: lane-1's a, lane 0: the previous row's
                // last chunk; chunk b: lane-1's b, lane 0: this row's a of lane 31)
                // (the last byte of the chunk in front decides what its successor may be: C3 folds, E0 / ED / E1 / E3
                // restrict the second byte of a three-byte letter)
                const u32 last_bytes = (xa.w >> 24) | ((xb.w >> 24) << 8);
                const u32 l31 = __shfl_sync(kFull, last_bytes, 31);
                u32 pc3 = __shfl_up_sync(kFull, last_bytes, 1);
                if (lane == 0) pc3 = (carryC3 & 0xFFu) | ((l31 & 0xFFu) << 8);
                carryC3 = l31 >> 8;
                // U3K: the call's sample saw three-byte letter leads -> the flags for them are compiled in (a kernel of
                // its own: the flags cost the other HI kernel registers and 10-20 % even when a branch skips them)
                u32 tails = 0;
                auto classify_row = [&](auto u3_) {
                    constexpr bool U3 = decltype(u3_)::value;
                const HiMasks ma = classify16_hi<U3>(xa, pc3 & 0xFFu, fa);
                asm volatile("" ::: "memory");     // one chunk after the other: fewer live flag words
                const HiMasks mb = classify16_hi<U3>(xb, pc3 >> 8, fb);
                S = pack7(ma.s7, mb.s7);
                A = pack7(ma.a7, mb.a7);
                const u32 L = pack7(ma.l7, mb.l7);
                // is the byte in front of each chunk a lead C3..DF
                const u32 L31 = __shfl_sync(kFull, L, 31);
                u32 pL = __shfl_up_sync(kFull, L, 1);
                if (lane == 0) pL = __byte_perm(carryL, L31, 0x5410);
                carryL = L31 >> 16;
                const HiIn in{pack7(ma.h7, mb.h7), pack7(ma.c7, mb.c7), L, pack7(ma.x7, mb.x7),
                              pack7(ma.e7, mb.e7), pack7(ma.z7, mb.z7), pack7(ma.k7, mb.k7), pack7(ma.l3, mb.l3), pack7(ma.b2, mb.b2)};
                // E2 / 80 / an open three-byte letter in the last two bytes of the chunk in front
                tails = hi_tails(in);
                const u32 t31 = __shfl_sync(kFull, tails, 31);
                u32 pT = __shfl_up_sync(kFull, tails, 1);
                if (lane == 0) pT = __byte_perm(carryT, t31, 0x5410);
                carryT = t31 >> 16;
                u32 bad_first;
                hi_masks_finish<U3>(in, pL >> 15, pT, A, H, bad_first, pH_clear, pA_set);
                pH_fix = bad_first << 15;     // an unmatched lead at the end of the chunk in front
                // Sequences left open at the end of a chunk stay flagged in H until the chunk behind completes them:
                // what THAT chunk cleared (lane + 1 for both halves; for lane 31's first half, lane 0's second) must
                // not send this row to the careful loop, nor must the open tail of the row's very last chunk -- no
                // fragment that ends in this row can hold it, and the next row sees it through carryH.
                };
                classify_row(std::integral_constant<bool, U3K>{});
                const u32 nclr = __shfl_down_sync(kFull, pH_clear, 1), clr0 = __shfl_sync(kFull, pH_clear, 0);
                const u32 tb = tails >> 16;                     // what the row's last chunk leaves open (lane 31)
                const u32 open_end = ((tb & 0x10u) || ((tb & 0x1u) && (tb & 0x4u))) ? 0xC0000000u : ((tb & 0xAu) ? 0x80000000u : 0u);
                H_open = lane == 31 ? ((clr0 >> 16) | open_end) : nclr;
            } else {
                const Masks ma = classify16<false>(xa, one, fa), mb = classify16<false>(xb, one, fb);
                S = pack7(ma.s7, mb.s7);
                A = pack7(ma.a7, mb.a7);
                H = pack7(ma.h7, mb.h7);
            }
            if (row >= full_rows) {   // last row (warp-uniform): bytes at and beyond n are whitespace
                const u64 ga = (u64)row * kRow + (u64)lane * 16, gb = ga + kHalf;
                const u32 va = ga >= n ? 0u : (n - ga >= 16 ? 16u : (u32)(n - ga));
                const u32 vb = gb >= n ? 0u : (n - gb >= 16 ? 16u : (u32)(n - gb));
                S |= ((0xFFFFu << va) & 0xFFFFu) | (((0xFFFFu << vb) & 0xFFFFu) << 16);
            }
            uint4* slot = reinterpret_cast<uint4*>(ring + slotpos + kGuard);
            slot[lane] = fa;
            slot[32 + lane] = fb;
            if (lane == 31) *reinterpret_cast<uint4*>(ring + (slotpos ^ kSlotStride) + 16) = fb;   // next row's guard

            // predecessor chunks: low half = chunk in front of a, high half = chunk in front of b
            const u32 s31 = __shfl_sync(kFull, S, 31), a31 = __shfl_sync(kFull, A, 31);
            u32 pS = __shfl_up_sync(kFull, S, 1), pA = __shfl_up_sync(kFull, A, 1), pH = 0;
            if (lane == 0) { pS = __byte_perm(carryS, s31, 0x5410); pA = __byte_perm(carryA, a31, 0x5410); }
            carryS = s31 >> 16; carryA = a31 >> 16;
            if (!ascii_row) {
                const u32 h31 = __shfl_sync(kFull, H, 31);
                pH = __shfl_up_sync(kFull, H, 1);
                if (lane == 0) pH = carryH | (h31 << 16);
                pH = (pH & ~pH_clear) | pH_fix;
                pA |= pA_set;
                carryH = h31 >> 16;
            }
            // fragment ends: whitespace byte whose predecessor is not whitespace
            const u32 E = S & ~(((S << 1) & 0xFFFEFFFEu) | ((pS >> 15) & 0x00010001u));
            // 32-bit views, bit i = byte (chunk start - 16 + i)
            const u32 VSa = __byte_perm(pS, S, 0x5410), VSb = __byte_perm(pS, S, 0x7632);
            const u32 VAa = __byte_perm(pA, A, 0x5410), VAb = __byte_perm(pA, A, 0x7632);
            const u32 Ta = E << 16, Tb = E & 0xFFFF0000u;           // ends in view coordinates
            const u32 prev_a = pS & 0xFFFFu, prev_b = pS >> 16;     // whitespace of the 16 bytes in front of each chunk
            const u32 base_a = slotpos + kGuard + lane * 16 - 16;   // ring position of view bit 0
            const u32 base_b = base_a + kHalf;

            // A fragment that ends in the chunk but has no whitespace in the 16 bytes in front
            // of the chunk may start out of sight: the careful loop decides end by end.
            // (HI: rows whose bytes >= 0x80 are all two-byte letters stay on the bit-parallel emission)
            bool careful = (HI ? __any_sync(kFull, ((H & ~H_open) | pH) != 0) : !ascii_row) ||
                           __any_sync(kFull, (Ta != 0 && prev_a == 0) || (Tb != 0 && prev_b == 0));
            bool general_row = true;
            u32 total;
            for (;;) {
                u32 Fra = 0, Lra = 0, Frb = 0, Lrb = 0, cnt;
                if (!careful) {
                    // first / last word character of every fragment that ends in the chunk
                    auto first_last = [](u32 VS, u32 VA, u32 T, u32 prev16, u32& F, u32& Lr) {
                        const u32 mt = shr_clamp(0x7FFFFFFFu, __clz(T));        // below the highest end (0 if none)
                        const u32 ml = shr_clamp(0xFFFFFFFFu, __clz(prev16));   // up to the last whitespace in front
                        const u32 K = mt & ~ml;
                        const u32 NK = ~VS & K, AK = VA & K;
                        F = AK & ~(NK + AK);                                    // first word characters, view order
                        const u32 Nr = __brev(NK), Ar = __brev(AK);
                        Lr = Ar & ~(Nr + Ar);                                   // last word characters, bit-reversed
                    };
                    first_last(VSa, VAa, Ta, prev_a, Fra, Lra);
                    first_last(VSb, VAb, Tb, prev_b, Frb, Lrb);
                    cnt = __popc(Fra) + __popc(Frb);
                } else {
                    cnt = __popc(E);
                }
                const u32 incl = warp_inclusive_sum(cnt);
                total = __shfl_sync(kFull, incl, 31);
                if ((qtail - qhead) + total > (u32)kQueueCap) {   // pathological row (tokens of 1-2 bytes): make room first
                    if constexpr (WIDE) wide_pass(qtail - qhead);
                    else token_pass(kPartialPass, qtail - qhead, true);
                    __syncwarp();
                }
                u32 qwr = (qtail + incl - cnt) * 2;               // byte offset of this lane's first entry
                if (!careful) {
                    // One token of each half per trip (two independent chains, half the branches):
                    // the k-th lowest bit of F pairs with the k-th highest bit of Lr.
                    u32 mx = 0;
                    u32 qa = qwr, qb = qwr + 2 * __popc(Fra);
                    while (Fra | Frb) {
                        const u32 lba = Fra & (0u - Fra), lbb = Frb & (0u - Frb);       // lowest set bits
                        const u32 fpa = 31 - __clz(lba), fpb = 31 - __clz(lbb);        // view position of the first word character
                        const u32 hla = 31 - __clz(Lra), hlb = 31 - __clz(Lrb);        // 31 - view position of the last one
                        const u32 ta = Fra ? 31u - hla - fpa : 0u;                     // length - 1
                        const u32 tb = Frb ? 31u - hlb - fpb : 0u;
                        if (Fra) { q_store(qa, ta * 4096u + (base_a + fpa)); qa += 2; }
                        if (Frb) { q_store(qb, tb * 4096u + (base_a + kHalf + fpb)); qb += 2; }
                        mx = max(mx, max(ta, tb));
                        Fra ^= lba;
                        Frb ^= lbb;
                        Lra ^= shl_clamp(1u, hla);
                        Lrb ^= shl_clamp(1u, hlb);
                    }
                    const u32 longest = __reduce_max_sync(kFull, mx);
                    if (longest <= 15) {
                        general_row = longest > 7;
                        warp_tokens += total;
                        break;
                    }
                    careful = true;      // a token longer than 16 bytes: redo the row end by end
                    continue;
                }
                auto emit_careful = [&](u32 VS, u32 VA, u32 VH, u32 T, u32 base, u64 gchunk) {
                    u32 Ew = T >> 16;
                    while (Ew) {
                        const u32 j = __ffs(Ew) - 1;
                        Ew &= Ew - 1;
                        const u32 below = (0x10000u << j) - 1u;            // bits below the end
                        const u32 sp = VS & below;
                        const u32 start = 32 - __clz(sp);                   // first byte of the fragment (0 if sp == 0)
                        const u32 frag = below & ~((1u << start) - 1u);
                        const u32 a = VA & frag;
                        u32 entry = 0;                                      // dead: no word character, or deferred
                        bool defer = (sp == 0) || (VH & frag);
                        if (!defer && a) {
                            const u32 first = __ffs(a) - 1;
                            const u32 tlen = 32 - __clz(a) - first;
                            if (tlen > 16) defer = true;
                            else { entry = ((tlen - 1) << 12) | (base + first); ++my_tokens; }
                        }
                        if (defer) {
                            const u64 slot_i = atomicAdd(gt.n_deferred, 1ull);
                            if (slot_i < gt.deferred_cap) gt.deferred[slot_i] = gchunk + j;
                            else atomicOr(gt.status, kStatusDeferredFull);
                        }
                        q_store(qwr, entry);
                        qwr += 2;
                    }
                };
                const u64 ga = (u64)row * kRow + (u64)lane * 16;
                emit_careful(VSa, VAa, __byte_perm(pH, H, 0x5410), Ta, base_a, ga);
                emit_careful(VSb, VAb, __byte_perm(pH, H, 0x7632), Tb, base_b, ga + kHalf);
                break;
            }
            const u32 still_carried = qtail - qhead;    // 0 if room had to be made
            qtail += total;
            __syncwarp();

            // the next row's bytes are requested here, not at the top of the loop: phase 2 (thousands of
            // cycles) covers the latency, and phase 1 -- the register peak -- does not carry them
            load_row(row + 1, nxa, nxb);

            // ------------------------------ phase 2 ------------------------------
            // full 32-token passes; the remainder waits for the next row's tokens ...
            const bool general = general_row || general_prev;   // leftovers are at most one row old
            general_prev = general_row;
            u32 consumed = 0;
            if constexpr (WIDE) {
                while (qtail - qhead >= 64) { wide_pass(64u); consumed += 64; drain_step(); }
                if (still_carried > consumed) wide_pass(qtail - qhead);
            } else {
                if (!general) {
                    while (qtail - qhead >= 64) { token_pass2(); consumed += 64; drain_step(); }
                }
                while (qtail - qhead >= 32) { token_pass(kFullPass, 32u, general); consumed += 32; drain_step(); }
                // ... unless it would outlive its bytes in the ring (the next row overwrites the
                // slot of the previous one)
                if (still_carried > consumed) token_pass(kPartialPass, qtail - qhead, general);
            }
            __syncwarp();
        }
        if (qtail != qhead) {
            if constexpr (WIDE) wide_pass(qtail - qhead);
            else token_pass(kPartialPass, qtail - qhead, true);
        }
        __syncwarp();
        while (mtail != mhead || __any_sync(kFull, dleft != 0)) drain_round();
    }

    // token total: one atomic per warp
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) my_tokens += __shfl_xor_sync(kFull, my_tokens, d);
    if (lane == 0 && (my_tokens + warp_tokens)) atomicAdd(gt.n_tokens, (u64)my_tokens + warp_tokens);

    // flush the combiners into the global table
    __syncthreads();
    for (int i = tid; i < 2 * SETS; i += WARPS * 32) {
        const u64 k = reinterpret_cast<const u64*>(sm.sk)[i];
        const u32 c = reinterpret_cast<const u32*>(sm.scnt)[i];
        if (k != 0 && c) table_add(gt, le_to_be(k), 0ull, (u64)c, &inserted);
    }
    for (int i = tid; i < MSLOTS; i += WARPS * 32) {
        const u64 k = sm.mk0[i];
        const u32 c = sm.mcnt[i];
        if (k > kSlotLocked && c) table_add(gt, le_to_be(k), le_to_be(sm.mk1[i]), (u64)c, &inserted);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) inserted += __shfl_xor_sync(kFull, inserted, d);
    if (lane == 0) table_note_inserted(gt, inserted);
}

// One kernel per variant (a kernel holding two bodies compiles the ASCII one measurably worse); every CTA runs in
// exactly one of the launched kernels, the same one for all CTAs of a call (variant_of_text, wc_count_common.cuh).
template <int WARPS, int SETS, int MSLOTS, int VARIANT>
__global__ void __launch_bounds__(WARPS * 32, 1)
wc_count_kernel(const uint8_t* __restrict__ text, u64 n, u32 rows_per_warp, int force, u32 one, TableView gt) {
    const int v = variant_of_text(text, n, force, gt.launched, VARIANT == kVarNarrow ? gt.wanted : nullptr);
    if (v != VARIANT) return;
    wc_count_body<WARPS, SETS, MSLOTS, variant_is_hi(VARIANT), variant_is_wide(VARIANT), variant_is_u3(VARIANT)>(
        text, n, rows_per_warp, one, gt);
}

// ---- host-side launcher (called from wordcount.cu) ---------------------------------
#ifndef WFCU_COUNT_SETS
#define WFCU_COUNT_SETS 3840
#endif
#ifndef WFCU_COUNT_MED_SLOTS
#define WFCU_COUNT_MED_SLOTS 256
#endif
#ifndef WFCU_WIDE_SLOTS
#define WFCU_WIDE_SLOTS 4800
#endif
constexpr int kCountWarps = kCountVariantWarps;
constexpr int kCountSets = WFCU_COUNT_SETS;             // two 8-byte keys + two counts per set (24 bytes)
constexpr int kCountMedSlots = WFCU_COUNT_MED_SLOTS;    // 20 bytes each
constexpr int kWideSets = 64, kWideSlots = WFCU_WIDE_SLOTS;   // WIDE variant: (almost) all of the combiner memory is the 16-byte-key table
typedef Smem<kCountWarps, kCountSets, kCountMedSlots> CountSmem;
typedef Smem<kCountWarps, kWideSets, kWideSlots> WideSmem;
static_assert(sizeof(CountSmem) + 1024 <= 227 * 1024, "shared memory budget");
static_assert(sizeof(WideSmem) + 1024 <= 227 * 1024, "shared memory budget");
static_assert(2 * kSlotStride + 20 <= 4096, "queue entries keep ring positions in 12 bits");

// wc_count4.cu: the fourth-generation ASCII body (bulk-TMA rows, tokens counted straight from the masks).  Exact, but
// measured slower than this file's on every corpus (cfg3 934 against 1014 GB/s), so it only
// runs when WFCU_COUNT_KERNEL=4 is set in the environment (A/B runs, tests).
cudaError_t wc_count4_launch(const uint8_t* text, u64 n, u32 rows_per_warp, unsigned grid, int force, const TableView& gt,
                             cudaStream_t stream);

// hint: variants the counter's recent texts asked for (bit per variant; the narrow one is always launched)
cudaError_t wc_count_launch(const uint8_t* text, u64 n, const TableView& gt_in, int sm_count, cudaStream_t stream, u64* launches,
                            u32 hint) {
    const size_t smem = sizeof(CountSmem) + 1024, smem_wide = sizeof(WideSmem) + 1024;   // + slack for the 1 KiB alignment
    auto k_narrow = wc_count_kernel<kCountWarps, kCountSets, kCountMedSlots, kVarNarrow>;
    typedef void (*Kernel)(const uint8_t*, u64, u32, int, u32, TableView);
    static const Kernel kernels[kVarCount] = {      // indexed by variant
        k_narrow,
        wc_count_kernel<kCountWarps, kCountSets, kCountMedSlots, kVarHi>,
        wc_count_kernel<kCountWarps, kWideSets, kWideSlots, kVarWide>,
        wc_count_kernel<kCountWarps, kWideSets, kWideSlots, kVarHiWide>,
        wc_count_kernel<kCountWarps, kCountSets, kCountMedSlots, kVarHi3>,
        wc_count_kernel<kCountWarps, kWideSets, kWideSlots, kVarHiWide3>,
    };
    static const cudaError_t attr = [&] {
        cudaError_t e = cudaSuccess;
        for (int v = 0; v < kVarCount && e == cudaSuccess; ++v)
            e = cudaFuncSetAttribute(kernels[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(variant_is_wide(v) ? smem_wide : smem));
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    cudaError_t e = cudaSuccess;
    const u64 n_rows = n / kRow + 1;
    u64 grid = (u64)sm_count;
    if (grid * kCountWarps > n_rows) grid = (n_rows + kCountWarps - 1) / kCountWarps;   // at least one row per warp
    if (grid == 0) grid = 1;
    const u64 rows_per_warp = (n_rows + grid * kCountWarps - 1) / (grid * kCountWarps);
    static const int force = [] { const char* v = getenv("WFCU_COUNT_VARIANT"); return v ? atoi(v) : -1; }();   // tests: 0..5
    static const bool gen4_ascii = [] { const char* v = getenv("WFCU_COUNT_KERNEL"); return v && v[0] == '4'; }();
    TableView gt = gt_in;
    gt.launched = (force >= 0 && force < kVarCount) ? (1u << force) : ((hint & ((1u << kVarCount) - 1u)) | 1u);
    // narrow first (it publishes the choice), the others in any order: all but one return after the sample
    for (int v = 0; v < kVarCount; ++v) {
        if (!((gt.launched >> v) & 1u)) continue;
        if (v == kVarNarrow && gen4_ascii) {
            e = wc_count4_launch(text, n, (u32)rows_per_warp, (unsigned)grid, force, gt, stream);
            if (e != cudaSuccess) return e;
        } else {
            kernels[v]<<<(unsigned)grid, kCountWarps * 32, variant_is_wide(v) ? smem_wide : smem, stream>>>(
                text, n, (u32)rows_per_warp, force, 1u, gt);
        }
        *launches += 1;
    }
    return cudaGetLastError();
}

}  // namespace wfcu
