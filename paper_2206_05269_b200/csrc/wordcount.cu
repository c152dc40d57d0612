// wordcount.cu -- fused tokenizer + counting map for sm_100a.
//
// Replaces, on the device, the reference's  tokenize -> normalize_word -> ++counts[word]
// loop (/root/reference/proj/src/text.cpp:9-57, proj/src/unicode.cpp:11-121,
// proj/src/pipeline.cpp:131-139).  Tokens never reach HBM: bytes are read once,
// classified, cut into tokens and counted in the same kernel.
//
// Kernel K1+K2 (wc_fast_kernel): HBM-bound byte scan.
//   * every warp owns a contiguous strip of 512-byte rows and streams it through
//     a private shared-memory ring with 16-byte cp.async (LDGSTS) copies,
//     RING_ROWS-2 rows ahead -- no CTA-wide barrier in steady state;
//   * phase 1, one 16-byte chunk per lane: SWAR byte classes (ASCII whitespace,
//     alphanumeric, >=0x80) -> 16-bit masks; fragment ENDS are found from the
//     whitespace mask and resolved BACKWARDS against the previous chunk's masks
//     (shuffle), so no look-ahead is ever needed; the edge trim (first..last
//     word character) falls out of the alnum mask; a warp prefix sum packs the
//     resolved (start,len) pairs into a per-warp queue;
//   * phase 2, one token per lane: unaligned fetch from the ring (3-5 LDS.32 +
//     funnel shifts), case fold in registers, big-endian pack into the 128-bit
//     key, then a CTA-wide shared-memory combiner table (the Zipf head: >80 % of
//     all tokens) with the global table (ATOMG.CAS.128 / RED.ADD.64) behind it.
//   * anything the byte-class logic cannot decide exactly -- fragments with a
//     byte >= 0x80, fragments or tokens longer than 16 bytes -- is appended to a
//     deferred list and handled by wc_slow_kernel, an exact restatement of the
//     reference's UTF-8 rules (one thread per fragment).
#include <cstdlib>

#include "wfcu_dev.cuh"
#include "wc_count_common.cuh"

namespace wfcu {

constexpr int kRowBytes = 512;              // 32 lanes x 16 bytes
constexpr int kRingRows = 4;
constexpr int kRingBytes = kRowBytes * kRingRows;   // per warp
constexpr int kRingWords = kRingBytes / 4;
constexpr int kPrefetch = kRingRows - 2;    // rows in flight ahead of the current one
constexpr int kQueueCap = 512;              // >= 256 = most fragment ends in one row
constexpr u64 kSlotLocked = 1ull;           // smem slot being claimed (never a valid k0)

// ---- SWAR byte classes: bit 7 of each byte lane is the answer ------------------
__device__ __forceinline__ u32 space4(u32 x) {
    const u32 x7 = x & 0x7F7F7F7Fu;
    const u32 z = (x7 ^ 0x20202020u) + 0x7F7F7F7Fu;  // bit7 clear <=> byte == 0x20
    const u32 a = x7 + 0x77777777u;                  // bit7 set   <=> byte >= 0x09
    const u32 b = x7 + 0x72727272u;                  // bit7 set   <=> byte >= 0x0E
    return (~z | (a & ~b)) & ~x & 0x80808080u;
}
__device__ __forceinline__ u32 alnum4(u32 x) {
    const u32 x7 = x & 0x7F7F7F7Fu;
    const u32 y = x7 | 0x20202020u;
    const u32 a1 = y + 0x1F1F1F1Fu;   // >= 'a'
    const u32 a2 = y + 0x05050505u;   // >  'z'
    const u32 d1 = x7 + 0x50505050u;  // >= '0'
    const u32 d2 = x7 + 0x46464646u;  // >  '9'
    return ((a1 & ~a2) | (d1 & ~d2)) & ~x & 0x80808080u;
}
// bytes known to be ASCII: 0x80 where 'A'..'Z'
__device__ __forceinline__ u32 upper4(u32 x) {
    const u32 u1 = x + 0x3F3F3F3Fu;   // >= 'A'
    const u32 u2 = x + 0x25252525u;   // >  'Z'
    return u1 & ~u2 & 0x80808080u;
}
// gather bit 7 of the four byte lanes into a nibble
__device__ __forceinline__ u32 nib(u32 m) { return (m * 0x00204081u) >> 28; }
__device__ __forceinline__ u32 mask16(u32 m0, u32 m1, u32 m2, u32 m3) {
    return nib(m0) | (nib(m1) << 4) | (nib(m2) << 8) | (nib(m3) << 12);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, u32 src_bytes) {
    const u32 d = (u32)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- CTA-shared combiner tables --------------------------------------------------
// Two tables so that the common case never touches a second key word:
//   short  : tokens of <= 8 bytes, key = the bytes, little-endian packed (u64)
//   medium : tokens of 9..16 bytes, key = two u64
// Both are 2-way (two candidate slots from one hash), probed with straight-line
// code.  A key that lands in two slots, or in a slot and the global table, is
// harmless: the flush adds every slot's count into the global table.  What must
// never happen is a count credited to a different key, hence the publish order
// of the medium table (k1 first, then k0 behind a fence).
// Straight-line hit path: two candidate slots, both loaded up front, slot chosen by
// selects.  Claiming an empty slot is the rare case (only while the table fills) and is
// entered through a warp-uniform branch so that the steady state carries no divergence
// bookkeeping.  live = this lane holds a token.
__device__ __forceinline__ bool short_add(u64* __restrict__ keys, u32* __restrict__ cnt, u32 mask, u64 key, u32 h,
                                          bool live) {
    const u32 i0 = (h >> 19) & mask, i1 = (h >> 6) & mask;   // best-mixed bits of a multiplicative hash
    const u64 c0 = *reinterpret_cast<volatile u64*>(keys + i0);
    const u64 c1 = *reinterpret_cast<volatile u64*>(keys + i1);
    const bool hit0 = c0 == key, hit1 = c1 == key;
    u32 slot = hit0 ? i0 : i1;
    bool found = (hit0 || hit1) && live;
    const bool can_claim = live && !found && (c0 == 0 || c1 == 0);
    if (__any_sync(0xFFFFFFFFu, can_claim)) {
        if (can_claim) {
            if (c0 == 0) {
                const u64 old = atomicCAS(keys + i0, 0ull, key);
                if (old == 0 || old == key) { slot = i0; found = true; }
            }
            if (!found && c1 == 0) {
                const u64 old = atomicCAS(keys + i1, 0ull, key);
                if (old == 0 || old == key) { slot = i1; found = true; }
            }
        }
    }
    if (found) atomicAdd(cnt + slot, 1u);
    return found;
}

__device__ __forceinline__ bool medium_add(u64* __restrict__ k0s, u64* __restrict__ k1s, u32* __restrict__ cnt,
                                           u32 mask, u64 k0, u64 k1, u32 h) {
    u32 i = h & mask;
#pragma unroll 1
    for (int way = 0; way < 2; ++way) {
        u64 c0 = *reinterpret_cast<volatile u64*>(k0s + i);
        if (c0 == 0) {
            c0 = atomicCAS(k0s + i, 0ull, kSlotLocked);
            if (c0 == 0) {
                *reinterpret_cast<volatile u64*>(k1s + i) = k1;
                __threadfence_block();
                atomicExch(k0s + i, k0);   // publish: readers that see k0 also see k1
                atomicAdd(cnt + i, 1u);
                return true;
            }
        }
        if (c0 == kSlotLocked) return false;   // being claimed: the global table is always safe
        if (c0 == k0 && *reinterpret_cast<volatile u64*>(k1s + i) == k1) {
            atomicAdd(cnt + i, 1u);
            return true;
        }
        i = (h >> 16) & mask;
    }
    return false;
}

__device__ __forceinline__ u32 bswap32(u32 v) { return __byte_perm(v, 0, 0x0123); }
// little-endian packed token word pair -> big-endian table key word
__device__ __forceinline__ u64 le_to_be(u64 v) { return ((u64)bswap32((u32)v) << 32) | bswap32((u32)(v >> 32)); }

constexpr int kMissCap = 64;   // per-warp buffer of keys that go to the global table

template <int WARPS, int NSLOTS, int MSLOTS>
struct FastSmem {
    u64 sk[NSLOTS];
    u32 scnt[NSLOTS];
    u64 mk0[MSLOTS];
    u64 mk1[MSLOTS];
    u32 mcnt[MSLOTS];
    uint4 ring[WARPS][kRingBytes / 16];
    ulonglong2 miss[WARPS][kMissCap];
    uint16_t queue[WARPS][kQueueCap];   // tlen << 11 | ring position
};

// text[0..n): one document (documents are concatenated with whitespace between
// them by the caller).  Position n acts as a whitespace byte, so does "position -1".
// EMIT = false: count into the tables.  EMIT = true: stand-alone tokenizer, every
// token becomes a TokenRec appended to `em` (order restored later by sorting on pos).
template <int WARPS, int NSLOTS, int MSLOTS, bool EMIT>
__global__ void __launch_bounds__(WARPS * 32, 1)
wc_fast_kernel(const uint8_t* __restrict__ text, u64 n, u64 rows_per_warp, TableView gt, EmitView em) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    FastSmem<WARPS, NSLOTS, MSLOTS>& sm = *reinterpret_cast<FastSmem<WARPS, NSLOTS, MSLOTS>*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u32 lt_mask = (1u << lane) - 1u;

    for (int i = tid; i < NSLOTS; i += WARPS * 32) { sm.sk[i] = 0; sm.scnt[i] = 0; }
    for (int i = tid; i < MSLOTS; i += WARPS * 32) { sm.mk0[i] = 0; sm.mk1[i] = 0; sm.mcnt[i] = 0; }
    __syncthreads();

    const u64 n_rows = n / kRowBytes + 1;   // the last row holds the virtual whitespace at n
    const u64 gw = (u64)blockIdx.x * WARPS + warp;
    const u64 row_begin = gw * rows_per_warp;
    u64 row_end = row_begin + rows_per_warp;
    if (row_end > n_rows) row_end = n_rows;

    uint8_t* ring = reinterpret_cast<uint8_t*>(sm.ring[warp]);
    const u32* ringw = reinterpret_cast<const u32*>(ring);
    uint16_t* queue = sm.queue[warp];
    ulonglong2* missbuf = sm.miss[warp];
    u32 my_tokens = 0;
    u32 qhead = 0, qtail = 0;     // token queue (warp-uniform)
    u32 mhead = 0, mtail = 0;     // miss buffer (warp-uniform)
    // compact emission (EmitView::keys): the warp's current key tile
    u64 ktile = ~0ull;            // warp-uniform; ~0 = none yet
    u32 kused = 0, ktotal = 0;    // keys in the tile / written by this warp (warp-uniform)
    u64 kor = 0, kand = ~0ull;    // per lane

    // 32 buffered keys -> global table, one key per lane
    auto drain_misses = [&](u32 count) {
        if (lane < count) {
            const ulonglong2 k = missbuf[(mhead + lane) & (kMissCap - 1)];
            table_add(gt, k.x, k.y, 1ull);
        }
        mhead += count;
    };

    // one pass of phase 2: `count` (<= 32) queued tokens, one per lane; `row_end_off`
    // is the global offset just past the row being processed
    auto token_pass = [&](u32 count, u64 row_end_off) {
        const u32 entry = (lane < count) ? queue[(qhead + lane) & (kQueueCap - 1)] : 0u;
        qhead += count;
        const u32 tlen = entry >> 11;               // 0: dead entry
        const u32 sp = entry & (kRingBytes - 1);
        const u32 wi = sp >> 2, sh = (sp & 3u) * 8u;
        const u32 w0 = ringw[wi & (kRingWords - 1)];
        const u32 w1 = ringw[(wi + 1) & (kRingWords - 1)];
        const u32 w2 = ringw[(wi + 2) & (kRingWords - 1)];
        u32 b0 = __funnelshift_r(w0, w1, sh);
        u32 b1 = __funnelshift_r(w1, w2, sh);
        b0 |= upper4(b0 & 0x7F7F7F7Fu) >> 2;   // fold A-Z (bytes past the token are masked off below)
        b1 |= upper4(b1 & 0x7F7F7F7Fu) >> 2;
        bool miss = false;
        u64 mk0 = 0, mk1 = 0;
        if (EMIT) {
            const u32 w3 = ringw[(wi + 3) & (kRingWords - 1)];
            const u32 w4 = ringw[(wi + 4) & (kRingWords - 1)];
            u32 b2 = __funnelshift_r(w2, w3, sh);
            u32 b3 = __funnelshift_r(w3, w4, sh);
            b2 |= upper4(b2 & 0x7F7F7F7Fu) >> 2;
            b3 |= upper4(b3 & 0x7F7F7F7Fu) >> 2;
            u64 lo = ((u64)b1 << 32) | b0, hi = ((u64)b3 << 32) | b2;
            if (tlen <= 8) { lo &= ~0ull >> ((64u - 8u * tlen) & 63u); hi = 0; }
            else hi &= ~0ull >> ((128u - 8u * tlen) & 63u);
            bool as_record = tlen != 0;
            if (em.keys) {
                const bool is_key = tlen != 0 && tlen <= 8;
                const u32 mk = __ballot_sync(0xFFFFFFFFu, is_key), cnt = __popc(mk);
                if (cnt) {
                    if (ktile == ~0ull || kused + cnt > kKeyTile) {       // next tile (the old one keeps its gap)
                        if (ktile != ~0ull && ktile < em.key_tiles && lane == 0) em.tile_counts[ktile] = kused;
                        u64 t = 0;
                        if (lane == 0) t = atomicAdd(em.kc + 0, 1ull);
                        ktile = __shfl_sync(0xFFFFFFFFu, t, 0);
                        kused = 0;
                    }
                    if (is_key) {
                        const u64 key = le_to_be(lo);
                        if (ktile < em.key_tiles) em.keys[ktile * kKeyTile + kused + __popc(mk & lt_mask)] = key;
                        kor |= key;
                        kand &= key;
                        ++my_tokens;
                    }
                    kused += cnt;
                    ktotal += cnt;
                }
                as_record = tlen > 8;
            }
            const u32 live = __ballot_sync(0xFFFFFFFFu, as_record);
            u64 base = 0;
            if (lane == 0 && live) base = atomicAdd(em.n_out, (u64)__popc(live));
            base = __shfl_sync(0xFFFFFFFFu, base, 0);
            if (as_record) {
                const u64 at = base + __popc(live & lt_mask);
                // token start: within one ring length before the end of the current row
                const u32 back = ((u32)row_end_off - sp) & (kRingBytes - 1);
                if (at < em.cap) em.out[at] = TokenRec{le_to_be(lo), le_to_be(hi), 0ull, row_end_off - (back ? back : kRingBytes)};
                ++my_tokens;
            }
            return;
        }
        if (!__any_sync(0xFFFFFFFFu, tlen > 8)) {
            // every token of this pass fits 8 bytes
            const u64 key = (((u64)b1 << 32) | b0) & (~0ull >> ((64u - 8u * tlen) & 63u));
            // multiplies run on the FMA pipe, which this ALU-bound kernel leaves mostly idle
            u32 h = (u32)key * 0x9E3779B1u + (u32)(key >> 32) * 0x85EBCA77u;
            h ^= h >> 16;
            h *= 0x2C1B3C6Du;
            const bool live = tlen != 0;
            if (!short_add(sm.sk, sm.scnt, NSLOTS - 1, key, h, live) && live) { miss = true; mk0 = le_to_be(key); }
            my_tokens += live;
        } else {
            const u32 w3 = ringw[(wi + 3) & (kRingWords - 1)];
            const u32 w4 = ringw[(wi + 4) & (kRingWords - 1)];
            u32 b2 = __funnelshift_r(w2, w3, sh);
            u32 b3 = __funnelshift_r(w3, w4, sh);
            b2 |= upper4(b2 & 0x7F7F7F7Fu) >> 2;
            b3 |= upper4(b3 & 0x7F7F7F7Fu) >> 2;
            u64 lo = ((u64)b1 << 32) | b0, hi = ((u64)b3 << 32) | b2;
            if (tlen <= 8) { lo &= ~0ull >> ((64u - 8u * tlen) & 63u); hi = 0; }
            else hi &= ~0ull >> ((128u - 8u * tlen) & 63u);
            u32 h = (u32)lo * 0x9E3779B1u + (u32)(lo >> 32) * 0x85EBCA77u;
            h += (u32)hi * 0xC2B2AE3Du + (u32)(hi >> 32) * 0x27D4EB2Fu;
            h ^= h >> 16;
            h *= 0x2C1B3C6Du;
            // short_add votes across the warp: every lane calls it, medium lanes as idle
            const bool is_short = tlen != 0 && tlen <= 8;
            bool ok = short_add(sm.sk, sm.scnt, NSLOTS - 1, lo, h, is_short);
            if (tlen > 8) ok = medium_add(sm.mk0, sm.mk1, sm.mcnt, MSLOTS - 1, lo, hi, h);
            if (tlen) {
                if (!ok) { miss = true; mk0 = le_to_be(lo); mk1 = le_to_be(hi); }
                ++my_tokens;
            }
        }
        const u32 mm = __ballot_sync(0xFFFFFFFFu, miss);
        if (mm) {
            if (miss) missbuf[(mtail + __popc(mm & lt_mask)) & (kMissCap - 1)] = make_ulonglong2(mk0, mk1);
            mtail += __popc(mm);
            __syncwarp();
            if (mtail - mhead >= 32) drain_misses(32);
        }
    };

    if (row_begin < row_end) {
        // issue one row: lane copies its 16-byte chunk, zero-filled past n
        // rows are indexed in 32 bits inside the loop (the launcher caps n at 2^40 bytes)
        const u32 r_begin = (u32)row_begin, r_end = (u32)row_end;
        const u32 full_rows = (u32)(n / kRowBytes);        // rows [0, full_rows) lie entirely inside the text
        const uint8_t* lane_src = text + lane * 16;
        uint8_t* lane_dst = ring + lane * 16;
        auto issue_row = [&](u32 row) {
            if (row < r_end) {
                uint8_t* dst = lane_dst + (row & (kRingRows - 1)) * kRowBytes;
                if (row < full_rows) {                     // interior row (warp-uniform): no clamping
                    cp_async16(dst, lane_src + (u64)row * kRowBytes, 16u);
                } else {
                    const u64 g = (u64)row * kRowBytes + (u64)lane * 16;
                    u32 nbytes = 0;
                    const uint8_t* src = text;
                    if (g < n) {
                        nbytes = (n - g >= 16) ? 16u : (u32)(n - g);
                        src = text + g;
                    }
                    cp_async16(dst, src, nbytes);
                }
            }
            cp_async_commit();
        };

        // masks of the chunk that precedes this lane's chunk (lane 0: carried from the previous row)
        u32 carryS = 0xFFFFu, carryA = 0, carryH = 0;   // "position -1" is whitespace
        if (row_begin > 0) {
            // history row: gives lane 0 its predecessor masks and keeps the bytes in the ring
            issue_row(r_begin - 1);   // row_begin-1 < row_end always
            cp_async_wait<0>();
            __syncwarp();
            const u64 g = (row_begin - 1) * kRowBytes + (u64)lane * 16;
            const uint4 w = *reinterpret_cast<const uint4*>(ring + (g & (kRingBytes - 1)));
            const u32 S = mask16(space4(w.x), space4(w.y), space4(w.z), space4(w.w));
            const u32 A = mask16(alnum4(w.x), alnum4(w.y), alnum4(w.z), alnum4(w.w));
            const u32 H = mask16(w.x & 0x80808080u, w.y & 0x80808080u, w.z & 0x80808080u, w.w & 0x80808080u);
            carryS = __shfl_sync(0xFFFFFFFFu, S, 31);
            carryA = __shfl_sync(0xFFFFFFFFu, A, 31);
            carryH = __shfl_sync(0xFFFFFFFFu, H, 31);
        }
#pragma unroll
        for (int p = 0; p < kPrefetch; ++p) issue_row(r_begin + p);

        for (u32 row = r_begin; row < r_end; ++row) {
            cp_async_wait<kPrefetch - 1>();
            __syncwarp();

            // ------------------------------ phase 1 ------------------------------
            const uint4 w = *reinterpret_cast<const uint4*>(lane_dst + (row & (kRingRows - 1)) * kRowBytes);
            u32 S = mask16(space4(w.x), space4(w.y), space4(w.z), space4(w.w));
            const u32 A = mask16(alnum4(w.x), alnum4(w.y), alnum4(w.z), alnum4(w.w));
            u32 H = 0;
            const u32 anyhi = (w.x | w.y | w.z | w.w) & 0x80808080u;
            if (__any_sync(0xFFFFFFFFu, anyhi != 0) || carryH) {
                H = mask16(w.x & 0x80808080u, w.y & 0x80808080u, w.z & 0x80808080u, w.w & 0x80808080u);
            }
            if (row >= full_rows) {   // last row (warp-uniform): bytes at and beyond n are whitespace
                const u64 g = (u64)row * kRowBytes + (u64)lane * 16;
                if (g + 16 > n) {
                    const u32 valid = (g < n) ? (u32)(n - g) : 0u;
                    S |= (0xFFFFu << valid) & 0xFFFFu;
                }
            }
            u32 pS = __shfl_up_sync(0xFFFFFFFFu, S, 1);
            u32 pA = __shfl_up_sync(0xFFFFFFFFu, A, 1);
            u32 pH = __shfl_up_sync(0xFFFFFFFFu, H, 1);
            if (lane == 0) { pS = carryS; pA = carryA; pH = carryH; }
            carryS = __shfl_sync(0xFFFFFFFFu, S, 31);
            carryA = __shfl_sync(0xFFFFFFFFu, A, 31);
            carryH = __shfl_sync(0xFFFFFFFFu, H, 31);

            // bit i of the 32-bit views = byte (g - 16 + i)
            const u32 S32 = pS | (S << 16);
            const u32 A32 = pA | (A << 16);
            const u32 H32 = pH | (H << 16);
            // fragment ends: whitespace byte whose predecessor is not whitespace
            u32 E = S & ~((S << 1) | (pS >> 15)) & 0xFFFFu;
            const u32 cnt = __popc(E);
            // warp exclusive prefix sum of cnt
            u32 incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u32 v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += v;
            }
            const u32 total = __shfl_sync(0xFFFFFFFFu, incl, 31);
            const u32 carried = qtail - qhead;          // entries left over from the previous row
            u32 qi = qtail + incl - cnt;
            const u32 gbase = row * kRowBytes + lane * 16 - 16u;   // ring positions only need the low bits
            // Slow-path candidates are decided once per warp: a byte >= 0x80 nearby, no
            // whitespace at all in the previous chunk, or a first fragment that reaches more
            // than 16 bytes back (only the FIRST end of a chunk can: later fragments start
            // inside the chunk).  Ordinary text takes the check-free loop.
            const u32 hbS = 31 - __clz(pS | 1u);                       // highest whitespace bit of the previous chunk
            const bool lane_rare = (H32 != 0) || (E != 0 && (pS == 0 || (u32)(__ffs(E) - 1) > hbS + 1));
            if (!__any_sync(0xFFFFFFFFu, lane_rare)) {
                while (E) {
                    const u32 j = __ffs(E) - 1;
                    E &= E - 1;
                    const u32 below = (0x10000u << j) - 1;             // bits below the end (32-bit view)
                    const u32 start = 32 - __clz(S32 & below);         // first byte of the fragment
                    const u32 a = A32 & below & ~((1u << start) - 1);
                    u32 entry = 0;                                     // dead: no word character
                    if (a) {
                        const u32 first = __ffs(a) - 1;
                        const u32 tlen = 32 - __clz(a) - first;        // <= 16 by the test above
                        entry = (tlen << 11) | ((gbase + first) & (kRingBytes - 1));
                    }
                    queue[(qi++) & (kQueueCap - 1)] = (uint16_t)entry;
                }
            } else {
                while (E) {
                    const u32 j = __ffs(E) - 1;
                    E &= E - 1;
                    const u32 pos = 16 + j;                    // end position in the 32-bit view
                    const u32 below = (1u << pos) - 1;
                    const u32 sp = S32 & below;
                    u32 entry = 0;                              // dead entry: fragment without a word character
                    const u32 start = 32 - __clz(sp);          // first byte of the fragment (0 if sp == 0)
                    const u32 frag = below & ~((1u << start) - 1);
                    const u32 a = A32 & frag;
                    bool defer = (sp == 0) || (H32 & frag);
                    if (!defer && a) {
                        const u32 first = __ffs(a) - 1;
                        const u32 tlen = 32 - __clz(a) - first;
                        if (tlen > 16) defer = true;
                        else entry = (tlen << 11) | ((gbase + first) & (kRingBytes - 1));
                    }
                    if (defer) {
                        const u64 slot = atomicAdd(gt.n_deferred, 1ull);
                        if (slot < gt.deferred_cap) gt.deferred[slot] = (u64)row * kRowBytes + (u64)lane * 16 + j;
                        else atomicOr(gt.status, kStatusDeferredFull);
                    }
                    queue[(qi++) & (kQueueCap - 1)] = (uint16_t)entry;
                }
            }
            qtail += total;
            __syncwarp();

            // ------------------------------ phase 2 ------------------------------
            // full 32-token passes; the remainder waits for the next row's tokens
            u32 consumed = 0;
            const u64 row_end_off = EMIT ? ((u64)row + 1) * kRowBytes : 0;   // only the tokenizer needs positions
            while (qtail - qhead >= 32) { token_pass(32, row_end_off); consumed += 32; }
            // ... unless it would outlive its bytes in the ring (entries of row-1 may
            // reach back into row-2, which the next copy overwrites)
            if (carried > consumed) token_pass(qtail - qhead, row_end_off);
            __syncwarp();   // everyone is done with the ring slot the next copy overwrites
            issue_row(row + kPrefetch);
        }
        cp_async_wait<0>();
        if (qtail != qhead) token_pass(qtail - qhead, row_end * kRowBytes);
        __syncwarp();
        while (mtail != mhead) drain_misses(min(mtail - mhead, 32u));
    }

    // token total: one atomic per warp
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) my_tokens += __shfl_xor_sync(0xFFFFFFFFu, my_tokens, d);
    if (lane == 0 && my_tokens) atomicAdd(gt.n_tokens, (u64)my_tokens);

    if constexpr (EMIT) {
        if (em.keys) {                                         // close the warp's key tile, publish its totals
            if (ktile != ~0ull && ktile < em.key_tiles && lane == 0) em.tile_counts[ktile] = kused;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                kor |= __shfl_xor_sync(0xFFFFFFFFu, kor, d);
                kand &= __shfl_xor_sync(0xFFFFFFFFu, kand, d);
            }
            if (lane == 0 && ktotal) {
                atomicAdd(em.kc + 1, (u64)ktotal);
                atomicOr(em.kc + 2, kor);
                atomicAnd(em.kc + 3, kand);
            }
        }
    }

    // flush the combiners into the global table
    __syncthreads();
    if constexpr (!EMIT) {
        for (int i = tid; i < NSLOTS; i += WARPS * 32) {
            const u64 k = sm.sk[i];
            const u32 c = sm.scnt[i];
            if (k != 0 && c) table_add(gt, le_to_be(k), 0ull, (u64)c);
        }
        for (int i = tid; i < MSLOTS; i += WARPS * 32) {
            const u64 k = sm.mk0[i];
            const u32 c = sm.mcnt[i];
            if (k > kSlotLocked && c) table_add(gt, le_to_be(k), le_to_be(sm.mk1[i]), (u64)c);
        }
    }
}

// ---------------------------------------------------------------------------------
// Slow path: exact restatement of the reference's UTF-8 rules, one thread per
// deferred fragment.  (/root/reference/proj/src/unicode.cpp:11-121, text.cpp:9-57)
// ---------------------------------------------------------------------------------
struct Dec { u32 cp; u32 len; bool valid; };

__device__ __forceinline__ Dec utf8_dec(const uint8_t* s, u64 pos, u64 end) {
    const Dec bad{0xFFFDu, 1u, false};
    const u32 b0 = s[pos];
    if (b0 < 0x80) return Dec{b0, 1u, true};
    u32 extra, cp, lo = 0x80, hi = 0xBF;
    if (b0 >= 0xC2 && b0 <= 0xDF) { extra = 1; cp = b0 & 0x1F; }
    else if (b0 >= 0xE0 && b0 <= 0xEF) {
        extra = 2; cp = b0 & 0x0F;
        if (b0 == 0xE0) lo = 0xA0;
        if (b0 == 0xED) hi = 0x9F;
    } else if (b0 >= 0xF0 && b0 <= 0xF4) {
        extra = 3; cp = b0 & 0x07;
        if (b0 == 0xF0) lo = 0x90;
        if (b0 == 0xF4) hi = 0x8F;
    } else return bad;
    if (pos + extra >= end) return bad;
    const u32 b1 = s[pos + 1];
    if (b1 < lo || b1 > hi) return bad;
    cp = (cp << 6) | (b1 & 0x3F);
    for (u32 k = 2; k <= extra; ++k) {
        const u32 b = s[pos + k];
        if ((b & 0xC0) != 0x80) return bad;
        cp = (cp << 6) | (b & 0x3F);
    }
    return Dec{cp, extra + 1, true};
}

__device__ __forceinline__ bool uni_space(u32 cp) {
    if (cp >= 0x09 && cp <= 0x0D) return true;
    if (cp >= 0x2000 && cp <= 0x200A) return true;
    return cp == 0x20 || cp == 0x85 || cp == 0xA0 || cp == 0x1680 || cp == 0x2028 || cp == 0x2029 ||
           cp == 0x202F || cp == 0x205F || cp == 0x3000;
}
__device__ __forceinline__ bool word_char(u32 cp) {
    if (cp < 0x80) {
        const u32 l = cp | 0x20;
        return (cp >= '0' && cp <= '9') || (l >= 'a' && l <= 'z');
    }
    if (cp == 0xFFFD) return false;
    if (cp >= 0xA1 && cp <= 0xBF) return cp == 0xAA || cp == 0xB5 || cp == 0xBA;
    if (cp == 0xD7 || cp == 0xF7) return false;
    if ((cp >= 0x2000 && cp <= 0x206F) || (cp >= 0x3000 && cp <= 0x303F)) return false;
    if ((cp >= 0xFF01 && cp <= 0xFF0F) || (cp >= 0xFF1A && cp <= 0xFF20)) return false;
    if ((cp >= 0xFF3B && cp <= 0xFF40) || (cp >= 0xFF5B && cp <= 0xFF65)) return false;
    return !uni_space(cp);
}
__device__ __forceinline__ u32 lower_cp(u32 cp) {
    if (cp >= 'A' && cp <= 'Z') return cp + 0x20;
    if (cp >= 0xC0 && cp <= 0xDE && cp != 0xD7) return cp + 0x20;
    return cp;
}
__device__ __forceinline__ u32 enc_len(u32 cp) { return cp < 0x80 ? 1 : cp < 0x800 ? 2 : cp < 0x10000 ? 3 : 4; }
__device__ __forceinline__ u32 enc_byte(u32 cp, u32 n, u32 i) {
    // byte i of the n-byte UTF-8 encoding of cp
    if (n == 1) return cp;
    const u32 shift = 6 * (n - 1 - i);
    if (i == 0) return ((0xF00u >> n) & 0xFF) | (cp >> shift);
    return 0x80 | ((cp >> shift) & 0x3F);
}

// normalize_word over one whitespace-free piece of the text, fed one decoded character at a time so that the
// caller's own walk over the fragment (which looks for Unicode whitespace) is the only one: normalised offsets of
// the first / last word character, and the first 16 normalised bytes from the first word character on (what lies
// behind the last word character is masked off at the end).
struct Piece {
    u64 noff, nfirst, nlast_end, first_b, last_e, k0, k1;
    bool any;      // a word character was seen
};
__device__ __forceinline__ void piece_reset(Piece& p) {
    p.noff = p.nfirst = p.nlast_end = p.first_b = p.last_e = p.k0 = p.k1 = 0;
    p.any = false;
}
__device__ __forceinline__ void piece_feed(Piece& p, u64 pos, const Dec& d) {
    const u32 cp = lower_cp(d.cp);
    const u32 el = enc_len(cp);
    if (word_char(cp)) {
        if (!p.any) { p.any = true; p.first_b = pos; p.nfirst = p.noff; }
        p.last_e = pos + d.len;
        p.nlast_end = p.noff + el;
    }
    if (p.any) {
        const u64 at = p.noff - p.nfirst;
        for (u32 k = 0; k < el && at + k < 16; ++k) {
            const u64 byte = enc_byte(cp, el, k), i = at + k;
            if (i < 8) p.k0 |= byte << (56 - 8 * i);
            else p.k1 |= byte << (56 - 8 * (i - 8));
        }
    }
    p.noff += el;
}
// Counts (or, when em != nullptr, emits) the token of the piece.  Returns 1 if there is one (the caller
// accounts the tokens: one atomic per warp, not per token).
__device__ u32 piece_finish(const uint8_t* text, const Piece& p, const TableView& gt, const EmitView* em, u32* inserted) {
    if (!p.any) return 0;
    const u64 nlen = p.nlast_end - p.nfirst;
    if (nlen <= 16) {
        u64 k0 = p.k0, k1 = p.k1;
        if (nlen <= 8) { k0 &= ~0ull << (64 - 8 * nlen); k1 = 0; }
        else if (nlen < 16) k1 &= ~0ull << (128 - 8 * nlen);
        if (em) {
            const u64 at = atomicAdd(em->n_out, 1ull);
            if (at < em->cap) em->out[at] = TokenRec{k0, k1, 0ull, p.first_b};
        } else {
            table_add(gt, k0, k1, 1ull, inserted);
        }
        return 1;
    }
    if (nlen > 0xFFFFFFFFull) { atomicOr(gt.status, kStatusArenaFull); return 1; }
    const u64 rec = arena_alloc(gt, (u32)nlen);
    if (!rec) return 1;
    uint8_t* out = gt.arena + rec + 8;
    u32 h = 2166136261u;
    u64 i = 0, p0 = 0, p1 = 0;
    for (u64 pos = p.first_b; pos < p.last_e;) {      // every sequence in [first_b, last_e) is complete
        const Dec d = utf8_dec(text, pos, p.last_e);
        const u32 cp = lower_cp(d.cp);
        const u32 el = enc_len(cp);
        for (u32 k = 0; k < el; ++k, ++i) {
            const u32 byte = enc_byte(cp, el, k);
            out[i] = (uint8_t)byte;
            h = (h ^ byte) * 16777619u;
            if (i < 8) p0 |= (u64)byte << (56 - 8 * i);
            else if (i < 16) p1 |= (u64)byte << (56 - 8 * (i - 8));
        }
        pos += d.len;
    }
    *reinterpret_cast<u32*>(gt.arena + rec) = (u32)nlen;
    *reinterpret_cast<u32*>(gt.arena + rec + 4) = h;
    if (em) {
        const u64 at = atomicAdd(em->n_out, 1ull);
        if (at < em->cap) em->out[at] = TokenRec{p0, p1, rec, p.first_b};
        return 1;
    }
    __threadfence();
    long_add(gt, rec, 1ull);
    return 1;
}

// the piece [a,b) on its own (normalize_word of a caller-supplied fragment)
__device__ u32 slow_count_piece(const uint8_t* text, u64 a, u64 b, const TableView& gt, const EmitView* em,
                                u32* inserted = nullptr) {
    Piece p;
    piece_reset(p);
    for (u64 pos = a; pos < b;) {
        const Dec d = utf8_dec(text, pos, b);
        piece_feed(p, pos, d);
        pos += d.len;
    }
    return piece_finish(text, p, gt, em, inserted);
}

__device__ __forceinline__ bool ascii_space(u32 b) { return b == 0x20 || (b >= 0x09 && b <= 0x0D); }

// One thread per deferred fragment END (offset of the terminating ASCII
// whitespace byte, or n).  The fragment start is found by scanning backwards.
// The deferred list is consumed: the last CTA to finish empties it for the next call (one launch less per count than
// a reset kernel of its own; every CTA has read the count before it takes its ticket).
__device__ __forceinline__ void slow_kernel_done(const TableView& gt) {
    if (!gt.ticket) return;
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(gt.ticket, 1u) + 1 == gridDim.x;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        *gt.n_deferred = 0;
        *gt.ticket = 0;
    }
}

// One forward walk over the fragment [s, e): a valid non-ASCII whitespace code point ends a piece (text.cpp:45-55),
// anything else feeds the piece's normalisation.  Decoding against the end of the fragment instead of the end of the
// piece changes nothing: the byte that follows a piece is the lead of the whitespace character, which no sequence
// accepts as a continuation byte.
__device__ void slow_fragment(const uint8_t* text, u64 s, u64 e, const TableView& gt, const EmitView* emp, u32& tokens,
                              u32& inserted) {
    Piece p;
    piece_reset(p);
    for (u64 pos = s; pos < e;) {
        const Dec d = utf8_dec(text, pos, e);
        if (d.valid && uni_space(d.cp)) {
            tokens += piece_finish(text, p, gt, emp, &inserted);
            piece_reset(p);
        } else {
            piece_feed(p, pos, d);
        }
        pos += d.len;
    }
    tokens += piece_finish(text, p, gt, emp, &inserted);
}

// ---- giant fragments ------------------------------------------------------------------------------------
// A whitespace-free run is ONE fragment however long it is (a base64 blob, a hex dump, minified code), and one thread
// walks a fragment byte by byte at ~2 MB/s: 64 MiB of 'a' took 32 s.  A fragment whose start is not found within
// kGiantBytes of its end is handed to the whole warp instead: 16 bytes per lane and step for the backwards search
// for its start and for one forward pass (any byte >= 0x80?  first / last word character), then -- pure ASCII, the
// case that occurs -- a parallel copy of the folded bytes into the arena; only the FNV hash of the record stays
// serial (one lane, 8 bytes per load).  A giant fragment with bytes >= 0x80 falls back to the one-thread walk.
constexpr u64 kGiantBytes = 4096;

__device__ __forceinline__ uint4 load16_clipped(const uint8_t* text, u64 n, u64 g) {
    if (g + 16 <= n) return *reinterpret_cast<const uint4*>(text + g);
    u32 w[4] = {0, 0, 0, 0};
    for (u64 k = g; k < n; ++k) w[(k - g) >> 2] |= (u32)text[k] << (8 * ((k - g) & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ void giant_fragment(const uint8_t* text, u64 n, u64 e, const TableView& gt, const EmitView* emp, u32& tokens,
                               u32& inserted) {
    const u32 kFull = 0xFFFFFFFFu;
    const u32 lane = threadIdx.x & 31;
    // the start: one behind the last ASCII whitespace in front of e (0 if there is none)
    u64 s = 0;
    for (u64 pos = e; pos > 0;) {
        const u64 wb = (pos - 1) & ~511ull;
        const u64 g = wb + 16 * lane;
        u32 ws = 0;
        if (g < pos) {
            uint4 f;
            ws = cntc::classify16<false>(load16_clipped(text, n, g), 1u, f).s7 >> 7;
            if (g + 16 > pos) ws &= (1u << (u32)(pos - g)) - 1u;
        }
        const u32 m = __ballot_sync(kFull, ws != 0);
        if (m) {
            const int hl = 31 - __clz(m);
            const u32 w = __shfl_sync(kFull, ws, hl);
            s = wb + 16 * (u64)hl + (u64)(31 - __clz(w)) + 1;
            break;
        }
        pos = wb;
    }
    // one pass over [s, e): bytes >= 0x80, first and last ASCII word character
    u32 hi = 0;
    u64 first = ~0ull, last = 0;
    for (u64 wb = s & ~511ull; wb < e; wb += 512) {
        const u64 g = wb + 16 * lane;
        if (g < e && g + 16 > s) {
            uint4 f;
            const cntc::Masks m = cntc::classify16<false>(load16_clipped(text, n, g), 1u, f);
            u32 keep = 0xFFFFu;
            if (g < s) keep &= ~((1u << (u32)(s - g)) - 1u);
            if (g + 16 > e) keep &= (1u << (u32)(e - g)) - 1u;
            const u32 a = (m.a7 >> 7) & keep;
            hi |= (m.h7 >> 7) & keep;
            if (a) {
                const u64 lo = g + (u64)(__ffs(a) - 1), up = g + (u64)(31 - __clz(a));
                first = first < lo ? first : lo;
                last = last > up ? last : up;
            }
        }
    }
    hi = __any_sync(kFull, hi != 0);
    for (int d = 16; d > 0; d >>= 1) {
        const u64 of = __shfl_xor_sync(kFull, first, d), ol = __shfl_xor_sync(kFull, last, d);
        first = first < of ? first : of;
        last = last > ol ? last : ol;
    }
    if (hi) {                           // not the ASCII case: the exact one-thread walk
        if (lane == 0) slow_fragment(text, s, e, gt, emp, tokens, inserted);
        __syncwarp();
        return;
    }
    if (first == ~0ull) return;         // no word character
    const u64 len = last + 1 - first;
    if (len <= 16) {
        if (lane == 0) tokens += slow_count_piece(text, first, last + 1, gt, emp, &inserted);
        __syncwarp();
        return;
    }
    u64 rec = 0;
    if (lane == 0) {
        if (len > 0xFFFFFFFFull) atomicOr(gt.status, kStatusArenaFull);
        else rec = arena_alloc(gt, (u32)len);
        tokens += 1;                    // as piece_finish: the token exists even if the arena cannot hold it
    }
    rec = __shfl_sync(kFull, rec, 0);
    if (!rec) return;
    uint8_t* out = gt.arena + rec + 8;
    // four bytes per lane and step (the record is 8-byte aligned, the source is not), two steps in flight
    const u64 len4 = len & ~3ull;
    auto fold4 = [&](u64 i) {
        const uint8_t* src = text + first + i;
        u32 w = (u32)src[0] | ((u32)src[1] << 8) | ((u32)src[2] << 16) | ((u32)src[3] << 24);
        const u32 y = w | 0x20202020u;
        const u32 upper = (y + 0x1F1F1F1Fu) & ~(y + 0x05050505u) & ~w & 0x80808080u & ~((w & 0x20202020u) << 2);
        return w | (upper >> 2);        // 'A'..'Z' -> 'a'..'z' (all bytes are < 0x80 here)
    };
    u64 i = 4ull * lane;
    for (; i + 128 < len4; i += 256) {
        const u32 w0 = fold4(i), w1 = fold4(i + 128);
        *reinterpret_cast<u32*>(out + i) = w0;
        *reinterpret_cast<u32*>(out + i + 128) = w1;
    }
    for (; i < len4; i += 128) *reinterpret_cast<u32*>(out + i) = fold4(i);
    for (u64 k = len4 + lane; k < len; k += 32) {
        u32 c = text[first + k];
        if (c >= 'A' && c <= 'Z') c |= 0x20u;
        out[k] = (uint8_t)c;
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) {
        u32 h = 2166136261u;            // fnv32 of the record's bytes (wfcu_dev.cuh), eight bytes per load
        u64 i = 0;
        for (; i + 8 <= len; i += 8) {
            u64 w = *reinterpret_cast<const volatile u64*>(out + i);
#pragma unroll
            for (int k = 0; k < 8; ++k) { h = (h ^ (u32)(w & 0xFF)) * 16777619u; w >>= 8; }
        }
        for (; i < len; ++i) h = (h ^ *reinterpret_cast<const volatile uint8_t*>(out + i)) * 16777619u;
        u64 p0 = 0, p1 = 0;
        for (u32 k = 0; k < 16; ++k) {
            const u64 byte = *reinterpret_cast<const volatile uint8_t*>(out + k);
            if (k < 8) p0 |= byte << (56 - 8 * k);
            else p1 |= byte << (56 - 8 * (k - 8));
        }
        *reinterpret_cast<u32*>(gt.arena + rec) = (u32)len;
        *reinterpret_cast<u32*>(gt.arena + rec + 4) = h;
        if (emp) {
            const u64 at = atomicAdd(emp->n_out, 1ull);
            if (at < emp->cap) emp->out[at] = TokenRec{p0, p1, rec, first};
        } else {
            __threadfence();
            long_add(gt, rec, 1ull);
        }
    }
    __syncwarp();
}

__global__ void wc_slow_kernel(const uint8_t* __restrict__ text, u64 n, TableView gt, EmitView em, int emit) {
    u64 count = *gt.n_deferred;
    if (count > gt.deferred_cap) count = gt.deferred_cap;
    if (count == 0) return;     // nothing to consume, nothing to reset: every CTA sees the same zero (no ticket traffic)
    u32 tokens = 0, inserted = 0;
    const EmitView* emp = emit ? &em : nullptr;
    const u32 lane = threadIdx.x & 31;
    // warp-uniform trip count: a lane whose fragment turns out to be a giant brings it back to the whole warp
    for (u64 base = (u64)blockIdx.x * blockDim.x + (threadIdx.x - lane); base < count; base += (u64)gridDim.x * blockDim.x) {
        const u64 idx = base + lane;
        u64 e = 0;
        bool giant = false;
        if (idx < count) {
            e = gt.deferred[idx];
            const u64 stop = e > kGiantBytes ? e - kGiantBytes : 0;
            u64 s = e;
            while (s > stop && !ascii_space(text[s - 1])) --s;
            giant = s == stop && s > 0 && !ascii_space(text[s - 1]);
            if (!giant) slow_fragment(text, s, e, gt, emp, tokens, inserted);
        }
        u32 gm = __ballot_sync(0xFFFFFFFFu, giant);
        while (gm) {
            const int src = __ffs(gm) - 1;
            gm &= gm - 1;
            giant_fragment(text, n, __shfl_sync(0xFFFFFFFFu, e, src), gt, emp, tokens, inserted);
        }
    }
    // token and claimed-slot totals: one atomic per warp (a per-token atomic on one address was most of this kernel's time)
    for (int d = 16; d > 0; d >>= 1) {
        tokens += __shfl_xor_sync(0xFFFFFFFFu, tokens, d);
        inserted += __shfl_xor_sync(0xFFFFFFFFu, inserted, d);
    }
    if ((threadIdx.x & 31) == 0) table_note_inserted(gt, inserted);
    if ((threadIdx.x & 31) == 0 && tokens) atomicAdd(gt.n_tokens, (u64)tokens);
    slow_kernel_done(gt);
}

__global__ void wc_reset_deferred_kernel(TableView gt) { *gt.n_deferred = 0; }

// normalize_word (proj/src/text.cpp:9-30) for a batch of fragments: fragment f is
// text[offsets[f] .. offsets[f+1]).  One thread per fragment; a fragment that keeps a
// token emits one TokenRec whose pos lies inside the fragment.
__global__ void wc_normalize_kernel(const uint8_t* __restrict__ text, const u64* __restrict__ offsets, u64 n_frag,
                                    TableView gt, EmitView em) {
    for (u64 f = (u64)blockIdx.x * blockDim.x + threadIdx.x; f < n_frag; f += (u64)gridDim.x * blockDim.x)
        if (slow_count_piece(text, offsets[f], offsets[f + 1], gt, &em)) atomicAdd(gt.n_tokens, 1ull);
}

// ---- host-side launchers (called from capi.cu) -----------------------------------
static_assert(kRingBytes == 2048, "queue entries keep ring positions in 11 bits");
#ifndef WFCU_FAST_WARPS
#define WFCU_FAST_WARPS 28
#endif
#ifndef WFCU_FAST_SLOTS
#define WFCU_FAST_SLOTS 8192
#endif
#ifndef WFCU_FAST_MED_SLOTS
#define WFCU_FAST_MED_SLOTS 512
#endif
constexpr int kFastWarps = WFCU_FAST_WARPS;
constexpr int kFastSlots = WFCU_FAST_SLOTS;         // short-token combiner slots (12 bytes each)
constexpr int kFastMedSlots = WFCU_FAST_MED_SLOTS;  // medium-token combiner slots (20 bytes each)
static_assert(sizeof(FastSmem<kFastWarps, kFastSlots, kFastMedSlots>) <= 227 * 1024, "shared memory budget");

size_t wc_fast_smem_bytes() { return sizeof(FastSmem<kFastWarps, kFastSlots, kFastMedSlots>); }

// wc_count.cu: the counting kernel (third generation).  wc_fast_kernel<.., EMIT = false> stays
// selectable (WFCU_COUNT_KERNEL=2 in the environment) for A/B runs on the same box.
cudaError_t wc_count_launch(const uint8_t* text, u64 n, const TableView& gt, int sm_count, cudaStream_t stream, u64* launches,
                            u32 hint);
static bool use_gen2_count_kernel() {
    static const bool v = [] { const char* e = getenv("WFCU_COUNT_KERNEL"); return e && e[0] == '2'; }();
    return v;
}

template <bool EMIT>
static cudaError_t wc_launch_impl(const uint8_t* text, u64 n, const TableView& gt, const EmitView& em, int sm_count,
                                  cudaStream_t stream, u64* launches, cudaEvent_t* ev_before_fast,
                                  cudaEvent_t* ev_after_fast, u32 variant_hint) {
    const size_t smem = wc_fast_smem_bytes();
    auto kernel = wc_fast_kernel<kFastWarps, kFastSlots, kFastMedSlots, EMIT>;
    {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const u64 n_rows = n / kRowBytes + 1;
    u64 grid = (u64)sm_count;
    const u64 total_warps_needed = n_rows;   // at least one row per warp
    if (grid * kFastWarps > total_warps_needed) grid = (total_warps_needed + kFastWarps - 1) / kFastWarps;
    if (grid == 0) grid = 1;
    const u64 rows_per_warp = (n_rows + grid * kFastWarps - 1) / (grid * kFastWarps);
    if (ev_before_fast) cudaEventRecord(*ev_before_fast, stream);
    if (!EMIT && !use_gen2_count_kernel()) {
        cudaError_t e = wc_count_launch(text, n, gt, sm_count, stream, launches, variant_hint);
        if (e != cudaSuccess) return e;
    } else {
        kernel<<<(unsigned)grid, kFastWarps * 32, smem, stream>>>(text, n, rows_per_warp, gt, em);
        *launches += 1;
    }
    if (ev_after_fast) cudaEventRecord(*ev_after_fast, stream);
    wc_slow_kernel<<<sm_count * 16, 128, 0, stream>>>(text, n, gt, em, EMIT ? 1 : 0);
    *launches += 1;
    if (!gt.ticket) {
        wc_reset_deferred_kernel<<<1, 1, 0, stream>>>(gt);
        *launches += 1;
    }
    return cudaGetLastError();
}

// count text[0..n) into the tables of gt
cudaError_t wc_launch(const uint8_t* text, u64 n, const TableView& gt, int sm_count, cudaStream_t stream,
                      u64* launches, cudaEvent_t* ev_before_fast, cudaEvent_t* ev_after_fast, u32 variant_hint) {
    return wc_launch_impl<false>(text, n, gt, EmitView{}, sm_count, stream, launches,
                                 ev_before_fast, ev_after_fast, variant_hint);
}

cudaError_t wc_normalize_launch(const uint8_t* text, const u64* offsets, u64 n_frag, const TableView& gt,
                                const EmitView& em, int sm_count, cudaStream_t stream, u64* launches) {
    if (n_frag == 0) return cudaSuccess;
    u64 g = (n_frag + 127) / 128;
    if (g > (u64)sm_count * 8) g = (u64)sm_count * 8;
    wc_normalize_kernel<<<(unsigned)g, 128, 0, stream>>>(text, offsets, n_frag, gt, em);
    *launches += 1;
    return cudaGetLastError();
}

// stand-alone tokenizer: append every token of text[0..n) to em (gt supplies the
// deferred list, the long-token arena and the status word; its tables stay untouched)
cudaError_t wc_tokenize_launch(const uint8_t* text, u64 n, const TableView& gt, const EmitView& em, int sm_count,
                               cudaStream_t stream, u64* launches) {
    return wc_launch_impl<true>(text, n, gt, em, sm_count, stream, launches, nullptr, nullptr, 63u);
}

}  // namespace wfcu
