// wc_count4.cu -- fused tokenizer + counting map for sm_100a, fourth generation (ASCII body).
//
// Replaces, on the device, the reference's  tokenize -> normalize_word -> ++counts[word]
// loop (/root/reference/proj/src/text.cpp:9-57, proj/src/unicode.cpp:90-121,
// proj/src/pipeline.cpp:131-139).  Bytes are read from HBM once; tokens never reach HBM.
//
// The third generation (wc_count.cu) spent 196 lane-instructions per token: 34 on the byte classes,
// 47 on turning the masks into a token queue (prefix sum, emission loop), 62 on the queued passes.
// This one removes the queue from the common case and the register staging of the rows:
//   * a ROW is 1 KiB; lane l owns its bytes [32l, 32l+32).  Rows arrive by 1-D bulk TMA
//     (cp.async.bulk + mbarrier, one instruction of lane 0 per row) in a two-slot ring per warp,
//     one row ahead; nothing is staged in registers.  The lane reads its two 16-byte units in an
//     order that keeps the 16-byte shared loads / stores free of bank conflicts (lanes 4..7 of
//     every group of eight start with their upper unit; the masks are rotated by 16 instead);
//   * SWAR classes (4 bytes per operation, answer in bit 7 of every byte), dp4a gathers into
//     32-bit masks W (whitespace) and A (word characters); A-Z are folded in the same registers
//     and the folded bytes replace the raw ones in the slot;
//   * with 32 contiguous bytes per lane, the fragments that lie between two whitespace bytes of
//     the lane need nothing from the neighbours: first word characters  F = A & ~(N + A)  (the
//     carry of the addition runs along each fragment), last ones by the same expression on the
//     bit-reversed masks; the k-th F pairs with the k-th L.  Only the fragment that crosses into
//     the lane from the left needs the neighbour's tail (two shuffles per row): its first / last
//     word character replace the positions of the lane's first token;
//   * tokens are counted straight from the masks, two per lane per trip (lowest and highest token
//     of the lane: two independent chains), then one per trip for the odd ones: unaligned fetch of
//     the folded bytes, length mask, multiply hash, one 16-byte load of a two-key bucket of the
//     CTA-wide combiner, shared-memory atomic count.  Misses go to the global table through the
//     asynchronous drain of the third generation (cp.async landing words, RED.ADD.64);
//   * everything else -- tokens of 9..16 bytes, rows with a byte >= 0x80, fragments that start
//     out of sight -- goes through a small per-warp queue and a general one-token pass, or to the
//     deferred list of wc_slow_kernel (tokens longer than 16 bytes, fragments with bytes >= 0x80).
// Text with letters >= 0x80 or long words runs on the third generation's other variants (wc_count.cu); the
// variant is chosen per call from one sample of the text (variant_of_text).
#include "wc_count_common.cuh"

namespace wfcu {
namespace cnt4 {
using namespace cntc;

constexpr int kRow = 1024;                         // 32 lanes x 32 bytes
constexpr int kGuard = 32;                         // in front of a slot: the previous row's last 32 folded bytes
constexpr int kSlotStride = kGuard + kRow;         // 1056
constexpr int kRingBytes = 2 * kSlotStride + 32;   // two slots + slack for the unaligned fetch
constexpr int kMissCap = 64;
constexpr int kQueueCap = 128;                     // u16 entries: ((len-1) << 12 | ring offset) + 1

// Shared memory, 1 KiB aligned.  Every hot access is  base register + compile-time offset  (ptxas otherwise
// rebuilds a shared address per field from the generic pointer, inside the loops).
struct __align__(16) WarpArea {                // 4 KiB per warp
    uint4 miss[kMissCap];                      // keys for the global table (little-endian words); 1 KiB aligned
    uint4 ring[kRingBytes / 16];
    uint4 landing[32];                         // where the global slot keys of a drain in flight arrive (cp.async)
    u64 mbar[2];
    u32 qtail;                                 // general-pass queue: entries written so far (free running)
    u32 dummy;                                 // where the count of a token that missed goes
    u32 pad0[2];
    uint16_t queue[kQueueCap];
    u32 pad1[32];
};
static_assert(sizeof(WarpArea) == 4096, "per-warp area");
template <int SETS, int MSLOTS>
struct __align__(16) Tables {
    ulonglong2 sk[SETS];                       // short combiner: two keys (tokens <= 8 bytes, little-endian) per set
    uint2 scnt[SETS];                          //                 and their counts
    u64 lomask[16];                            // [len-1] -> mask of key bytes 0..7
    u64 himask[16];                            // [len-1] -> mask of key bytes 8..15
    u64 pad[48];                               // reads of lomask[len-1] by dead lanes (len-1 up to 63) stay inside
    u64 mk0[MSLOTS];                           // medium combiner (9..16 bytes): key low, key high, count
    u64 mk1[MSLOTS];
    u32 mcnt[MSLOTS];
};
template <int WARPS, int SETS, int MSLOTS>
struct __align__(1024) Smem {
    WarpArea w[WARPS];
    Tables<SETS, MSLOTS> t;
};

__device__ __forceinline__ uint4 lds128(u32 a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts128(u32 a, const uint4& v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ u32 lds32(u32 a) {
    u32 v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint2 lds64(u32 a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}

__device__ __forceinline__ u32 bfind(u32 v) {      // index of the highest set bit, 0xFFFFFFFF if none
    u32 r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ void red_inc(u32 a) {
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a) : "memory");
}
__device__ __forceinline__ void sts128_if(u32 a, bool p, u32 x, u32 y, u32 z, u32 w) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q st.shared.v4.u32 [%0], {%2,%3,%4,%5};\n\t}"
                 ::"r"(a), "r"((u32)p), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// ---- 1-D bulk TMA into the warp's ring -------------------------------------------------
__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t"
        "}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_row(u32 dst, const uint8_t* src, u32 bytes, u32 bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <int WARPS, int SETS, int MSLOTS>
__device__ __forceinline__ void wc_count4_body(const uint8_t* __restrict__ text, u64 n, u32 rows_per_warp, const TableView& gt) {
    extern __shared__ uint8_t smem_raw[];
    typedef Smem<WARPS, SETS, MSLOTS> SM;
    typedef Tables<SETS, MSLOTS> TB;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u32 lt_mask = (1u << lane) - 1u;
    const u32 raw_s = (u32)__cvta_generic_to_shared(smem_raw);
    u32 base_s = (raw_s + 1023u) & ~1023u;             // shared address of the Smem
    SM& sm = *reinterpret_cast<SM*>(smem_raw + (base_s - raw_s));
    u32 wb = base_s + (u32)warp * (u32)sizeof(WarpArea);   // ... of the warp's area
    asm volatile("" : "+r"(base_s), "+r"(wb));           // opaque: one register each, offsets are immediates
    constexpr u32 kT = WARPS * (u32)sizeof(WarpArea);    // offset of the tables from base_s
    constexpr u32 oSk = kT + (u32)offsetof(TB, sk), oCnt = kT + (u32)offsetof(TB, scnt);
    constexpr u32 oLo = kT + (u32)offsetof(TB, lomask), oHi = kT + (u32)offsetof(TB, himask);
    constexpr u32 oMiss = (u32)offsetof(WarpArea, miss), oRing = (u32)offsetof(WarpArea, ring);
    constexpr u32 oLand = (u32)offsetof(WarpArea, landing), oBar = (u32)offsetof(WarpArea, mbar);
    constexpr u32 oQtail = (u32)offsetof(WarpArea, qtail), oDummy = (u32)offsetof(WarpArea, dummy);
    constexpr u32 oQueue = (u32)offsetof(WarpArea, queue);
    static_assert(oMiss == 0, "the miss buffer is 1 KiB aligned: index wrap by OR");

    for (int i = tid; i < SETS; i += WARPS * 32) { sm.t.sk[i] = make_ulonglong2(0, 0); sm.t.scnt[i] = make_uint2(0, 0); }
    for (int i = tid; i < MSLOTS; i += WARPS * 32) { sm.t.mk0[i] = 0; sm.t.mk1[i] = 0; sm.t.mcnt[i] = 0; }
    if (tid < 16) {
        sm.t.lomask[tid] = tid < 8 ? (~0ull >> (56 - 8 * tid)) : ~0ull;
        sm.t.himask[tid] = tid < 8 ? 0ull : (~0ull >> (120 - 8 * tid));
    }
    if (tid < 48) sm.t.pad[tid] = 0;
    for (int i = lane; i < (int)(sizeof(WarpArea) / 16); i += 32) reinterpret_cast<uint4*>(&sm.w[warp])[i] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    const u32 ring_s = wb + oRing;
    const u32 bar_s = wb + oBar;
    if (lane == 0) {
        mbar_init(bar_s, 1);
        mbar_init(bar_s + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const u32 n_rows = (u32)(n / kRow) + 1;            // the last row holds the virtual whitespace at n
    const u32 full_rows = (u32)(n / kRow);             // rows [0, full_rows) lie entirely inside the text
    const u32 gw = blockIdx.x * WARPS + warp;
    const u64 rb64 = (u64)gw * rows_per_warp;
    const u32 r_begin = rb64 < n_rows ? (u32)rb64 : n_rows;
    const u32 r_end = (rb64 + rows_per_warp < n_rows) ? (u32)(rb64 + rows_per_warp) : n_rows;
    const u32 tma_end = r_end < full_rows ? r_end : full_rows;   // rows [r_begin, tma_end) arrive by TMA

    const u32 queue_s = wb + oQueue;
    auto qtail_now = [&]() { return lds32(wb + oQtail); };
    u32 inserted = 0;             // global slots this lane claimed (first occurrences)
    u32 my_tokens = 0;            // per lane
    u32 qhead = 0;                // general-pass queue (warp-uniform, free running; the tail lives in shared memory)
    u32 mhead = 0, mtail = 0;     // miss buffer (warp-uniform, free running)

    // ---- misses -> global table (the third generation's asynchronous drain) ----------------
    u32 dk0 = 0, dk1 = 0, dk2 = 0, dk3 = 0;         // the lane's key in flight (big-endian words)
    u32 didx = 0, dleft = 0;                        // slot being fetched; probes left (0 = lane free)
    auto drain_round = [&]() {
        const u32 dst = wb + oLand + lane * 16u;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        if (dleft) {
            const uint4 cur = lds128(dst);          // {k0 low, k0 high, k1 low, k1 high}
            if (cur.x == dk1 && cur.y == dk0 && cur.z == dk3 && cur.w == dk2) {
                atomicAdd(&gt.slots[didx].count, 1ull);
                dleft = 0;
            } else if ((cur.x | cur.y) == 0 || --dleft == 0) {
                table_add(gt, ((u64)dk0 << 32) | dk1, ((u64)dk2 << 32) | dk3, 1ull, &inserted);
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
            const uint4 k = lds128(wb + (((mhead + rank) * 16u) & (kMissCap * 16u - 16u)));
            dk0 = bswap32(k.x); dk1 = bswap32(k.y); dk2 = bswap32(k.z); dk3 = bswap32(k.w);
            didx = mix32(((u64)dk0 << 32) | dk1, ((u64)dk2 << 32) | dk3) & (u32)gt.mask;
            dleft = 3;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gt.slots + didx) : "memory");
        }
        mhead += min((u32)__popc(freem), avail);
        asm volatile("cp.async.commit_group;" ::: "memory");
        __syncwarp();                               // the entries just read may be overwritten by the next append
    };
    auto drain_step = [&]() {
        if (mtail - mhead >= 32) drain_round();
    };
    auto make_room = [&](u32 extra) {
        while ((mtail - mhead) + extra > (u32)kMissCap) drain_round();
    };
    auto push_misses = [&](bool miss, u32 k0, u32 k1, u32 k2, u32 k3) {
        const u32 mm = __ballot_sync(kFull, miss);
        if ((mtail - mhead) + __popc(mm) > (u32)kMissCap) make_room(__popc(mm));
        const u32 at = (mtail + __popc(mm & lt_mask)) & (kMissCap - 1);
        sts128_if(wb + at * 16u, miss, k0, k1, k2, k3);
        mtail += __popc(mm);
    };


    // claim an empty way of the bucket for FUTURE occurrences (this one still goes to the global table)
    auto claim = [&](u32 set, u32 w0l, u32 w1l, u32 b0, u32 b1) {
        const u64 key = ((u64)b1 << 32) | b0;
        u64* slot = reinterpret_cast<u64*>(&sm.t.sk[set]);
        u64 old = 1;
        if (w0l == 0) old = atomicCAS(slot, 0ull, key);
        if (old != 0 && old != key && w1l == 0) atomicCAS(slot + 1, 0ull, key);
    };

    // general pass: `count` (<= 32) queued tokens of up to 16 bytes, one per lane
    auto general_pass = [&](u32 count) {
        u32 e = 0;
        if ((u32)lane < count) {
            asm volatile("ld.shared.u16 %0, [%1];" : "=r"(e) : "r"(queue_s + ((qhead + lane) & (kQueueCap - 1)) * 2u) : "memory");
        }
        qhead += count;
        const bool live = e != 0;
        e -= live ? 1u : 0u;
        const u32 pa = ring_s + (e & 0xFFFu);
        const u32 l1 = e >> 12;
        const u32 aa = pa & ~3u;
        const u32 w0 = lds32(aa), w1 = lds32(aa + 4), w2 = lds32(aa + 8), w3 = lds32(aa + 12), w4 = lds32(aa + 16);
        const uint2 lm = lds64(base_s + oLo + l1 * 8u), hm = lds64(base_s + oHi + l1 * 8u);
        const u32 sh = pa << 3;
        const u32 b0 = __funnelshift_r(w0, w1, sh) & lm.x, b1 = __funnelshift_r(w1, w2, sh) & lm.y;
        const u32 b2 = __funnelshift_r(w2, w3, sh) & hm.x, b3 = __funnelshift_r(w3, w4, sh) & hm.y;
        const bool is_medium = l1 > 7;
        u32 h = b0 * 0x9E3779B1u + b1 * 0x85EBCA77u;
        bool ok = false;
        {
            const u32 set = __umulhi(h, (u32)SETS);
            const uint4 c = lds128(base_s + oSk + set * 16u);
            const bool h0 = c.x == b0 && c.y == b1, h1 = c.z == b0 && c.w == b1;
            ok = (h0 || h1) && live && !is_medium;
            if (ok) atomicAdd(reinterpret_cast<u32*>(sm.t.scnt) + set * 2u + (h1 ? 1u : 0u), 1u);
            if (live && !is_medium && !ok && (c.x == 0 || c.z == 0)) claim(set, c.x, c.z, b0, b1);
        }
        if (live && is_medium) {
            h += b2 * 0xC2B2AE3Du + b3 * 0x27D4EB2Fu;
            h ^= h >> 16;
            h *= 0x2C1B3C6Du;
            ok = medium_add(sm.t.mk0, sm.t.mk1, sm.t.mcnt, MSLOTS - 1, ((u64)b1 << 32) | b0, ((u64)b3 << 32) | b2, h);
        }
        __syncwarp();
        push_misses(live && !ok, b0, b1, b2, b3);
    };
    auto run_queue = [&](u32 keep_below) {     // passes until fewer than keep_below entries wait
        __syncwarp();
        u32 waiting = qtail_now() - qhead;
        while (waiting >= keep_below && waiting != 0) {
            general_pass(waiting < 32u ? waiting : 32u);
            drain_step();
            waiting = qtail_now() - qhead;
        }
    };
    // divergent callers: one token of up to 16 bytes for the general pass (ring offset of its first byte)
    auto enqueue = [&](u32 ring_off, u32 l1) {
        const u32 at = atomicAdd(&sm.w[warp].qtail, 1u);
        const u32 v = ((l1 << 12) | ring_off) + 1u;
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(queue_s + (at & (kQueueCap - 1)) * 2u), "r"(v) : "memory");
    };
    auto defer = [&](u64 end_pos) {
        const u64 slot_i = atomicAdd(gt.n_deferred, 1ull);
        if (slot_i < gt.deferred_cap) gt.deferred[slot_i] = end_pos;
        else atomicOr(gt.status, kStatusDeferredFull);
    };

    if (r_begin < r_end) {
        // lanes 4..7 of every group of eight read their upper 16-byte unit first: conflict-free 16-byte accesses
        const u32 sw = (lane >> 2) & 1u;
        const u32 unit0 = (2u * lane + sw) * 16u, unit1 = (2u * lane + 1u - sw) * 16u;
        const u32 rot = sw * 16u;
        const u32 src_lane = (lane + 31) & 31;
        const bool flip = (lane & 16) != 0;

        // masks of the 32 bytes in front of the strip ("position -1" is whitespace)
        u32 oldW = 0xFFFFFFFFu, oldAt = 0;        // what lane 31 saw in the previous row (every lane keeps its own)
        bool carry_hi = false;                    // ... and whether its chunk held a byte >= 0x80
        if (r_begin > 0) {
            const uint4* p = reinterpret_cast<const uint4*>(text + (u64)r_begin * kRow - 32);
            const uint4 x0 = p[0], x1 = p[1];
            uint4 f0, f1;
            const Masks m0 = classify16<false>(x0, 1u, f0), m1 = classify16<false>(x1, 1u, f1);
            const u32 W = pack7(m0.s7, m1.s7), A = pack7(m0.a7, m1.a7), H = pack7(m0.h7, m1.h7);
            oldW = W;
            oldAt = A & ~shr_clamp(0xFFFFFFFFu, __clz(W));
            carry_hi = H != 0;
            if (lane == 0) {
                sts128(ring_s + (r_begin & 1u) * kSlotStride, f0);
                sts128(ring_s + (r_begin & 1u) * kSlotStride + 16, f1);
            }
        }
        if (lane == 0) {
            if (r_begin < tma_end) tma_row(ring_s + (r_begin & 1u) * kSlotStride + kGuard, text + (u64)r_begin * kRow, kRow, bar_s + (r_begin & 1u) * 8u);
            if (r_begin + 1 < tma_end) tma_row(ring_s + ((r_begin + 1) & 1u) * kSlotStride + kGuard, text + (u64)(r_begin + 1) * kRow, kRow, bar_s + ((r_begin + 1) & 1u) * 8u);
        }
        __syncwarp();

        for (u32 row = r_begin; row < r_end; ++row) {
            const u32 slotpos = (row & 1u) * kSlotStride;
            const u32 slot_s = ring_s + slotpos + kGuard;
            if (row < full_rows) {
                mbar_wait(bar_s + (row & 1u) * 8u, ((row - r_begin) >> 1) & 1u);
            } else {
                // the last row of the text: bytes at and beyond n are zero here and whitespace below
                u32 w[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) w[k] = 0;
                const u64 g = (u64)row * kRow + (u64)lane * 32;
                for (u32 k = 0; k < 32 && g + k < n; ++k) w[k >> 2] |= (u32)text[g + k] << (8 * (k & 3));
                sts128(slot_s + lane * 32u, make_uint4(w[0], w[1], w[2], w[3]));
                sts128(slot_s + lane * 32u + 16u, make_uint4(w[4], w[5], w[6], w[7]));
                __syncwarp();
            }
            const uint4 xa = lds128(slot_s + unit0), xb = lds128(slot_s + unit1);

            // ------------------------------ byte classes ------------------------------
            u32 W, A, H = 0;
            uint4 fa, fb;
            const u32 anyhi = (xa.x | xa.y | xa.z | xa.w | xb.x | xb.y | xb.z | xb.w) & 0x80808080u;
            const bool ascii_row = !__any_sync(kFull, anyhi != 0);
            if (ascii_row) {
                const Masks ma = classify16<true>(xa, 1u, fa), mb = classify16<true>(xb, 1u, fb);
                W = pack7(ma.s7, mb.s7);
                A = pack7(ma.a7, mb.a7);
            } else {
                const Masks ma = classify16<false>(xa, 1u, fa), mb = classify16<false>(xb, 1u, fb);
                W = pack7(ma.s7, mb.s7);
                A = pack7(ma.a7, mb.a7);
                H = pack7(ma.h7, mb.h7);
                H = __funnelshift_r(H, H, rot);
            }
            W = __funnelshift_r(W, W, rot);      // text order: bit i = byte i of the lane's chunk
            A = __funnelshift_r(A, A, rot);
            if (row >= full_rows) {
                const u64 g = (u64)row * kRow + (u64)lane * 32;
                const u32 valid = g >= n ? 0u : (n - g >= 32 ? 32u : (u32)(n - g));
                W |= shl_clamp(0xFFFFFFFFu, valid);
            }
            sts128(slot_s + unit0, fa);
            sts128(slot_s + unit1, fb);
            if (lane == 31) {                    // the next row's guard: this row's last 32 folded bytes (lane 31: sw = 1)
                const u32 g = ring_s + (slotpos ^ kSlotStride);
                sts128(g + 16u, fa);
                sts128(g, fb);
            }

            // the chunk in front: lane l-1's masks; lane 0 gets what lane 31 saw in the previous row
            const u32 clzW = __clz(W);
            const u32 mt1 = shr_clamp(0xFFFFFFFFu, clzW);      // bits up to the highest whitespace (0 if none)
            const u32 At = A & ~mt1;                            // word characters of the fragment left open at the end
            const u32 pW = __shfl_sync(kFull, lane == 31 ? oldW : W, src_lane);
            const u32 pAt = __shfl_sync(kFull, lane == 31 ? oldAt : At, src_lane);
            oldW = W;
            oldAt = At;
            const bool crossing = (int)pW >= 0 && W != 0;      // a fragment that ends here starts in the chunk in front
            bool careful = !ascii_row || carry_hi || __any_sync(kFull, crossing && pW == 0);
            carry_hi = false;
            __syncwarp();                                      // folded bytes and guard are in place

            u32 lane_s = slot_s + lane * 32u;                  // shared address of the chunk's first byte
            asm volatile("" : "+r"(lane_s));                    // keep it in a register
            const bool filling = row - r_begin < 64u || (row & 15u) == 0;
            if (!careful) {
                // first / last word character of every fragment that ends at a whitespace byte of the chunk
                const u32 NK = ~W & mt1, AK = A & mt1;
                u32 Fm = AK & ~(NK + AK);
                const u32 Nr = __brev(NK), Ar = __brev(AK);
                u32 Lr = Ar & ~(Nr + Ar);                       // bit-reversed
                // the fragment that crosses in from the left: its first word character may lie in the chunk in
                // front (then it replaces the first F), so may its last one (then both are placeholders at byte 0)
                const bool has_head = crossing && pAt != 0;
                const u32 loW = W & (0u - W);
                const bool head_all_left = has_head && (A & (loW - 1u)) == 0;
                const u32 hfp = (u32)__ffs(pAt) - 33u;          // relative to the chunk (negative)
                const u32 hlp = (u32)(31 - __clz(pAt)) - 32u;
                if (head_all_left) { Fm |= 1u; Lr |= 0x80000000u; }
                my_tokens += __popc(Fm);

                // rare lanes of a trip: tokens of 9..16 bytes wait for the general pass, longer ones are deferred
                auto long_token = [&](u32 fp, u32 l1) {
                    if (l1 > 15) {
                        const int lp1 = (int)(fp + l1) + 1;                       // byte behind the last word character
                        const u32 above = W & shl_clamp(0xFFFFFFFFu, lp1 > 0 ? (u32)lp1 : 0u);
                        defer((u64)row * kRow + (u64)lane * 32 + (u32)(__ffs(above) - 1));
                        --my_tokens;
                    } else {
                        enqueue(lane_s + fp - ring_s, l1);
                    }
                };
                // One trip: the lowest token of the lane's list (X) and, if TWO, the highest one (Y) -- two
                // independent chains.  Dead lanes (list empty) read valid shared addresses and a length of 34
                // bytes, which no predicate below accepts.
                auto trip = [&](auto two_, auto first_) {
                    constexpr bool TWO = decltype(two_)::value, FIRST = decltype(first_)::value;
                    const u32 lbx = Fm & (0u - Fm);
                    u32 fpx = bfind(lbx);
                    const u32 hlx = bfind(Lr);
                    bool livex = lbx != 0;
                    Fm ^= lbx;
                    Lr &= ~shl_clamp(1u, hlx);
                    u32 l1x = 31u - hlx - fpx;
                    if (FIRST) {
                        fpx = has_head ? hfp : fpx;
                        l1x = (head_all_left ? hlp : 31u - hlx) - fpx;
                    }
                    u32 fpy = 0, l1y = 64;
                    bool livey = false;
                    if (TWO) {
                        fpy = bfind(Fm);
                        const u32 lby = Lr & (0u - Lr);
                        livey = lby != 0;
                        l1y = 31u - bfind(lby) - fpy;
                        Fm &= ~shl_clamp(1u, fpy);
                        Lr ^= lby;
                    }
                    if (TWO && flip) {      // half of the lanes start from the other end: fewer bank conflicts in the fetches
                        const u32 t0 = fpx, t1 = l1x;
                        fpx = fpy; l1x = l1y; fpy = t0; l1y = t1;
                    }
                    const bool sx = l1x <= 7, sy = TWO && l1y <= 7;
                    const u32 pax = lane_s + fpx, pay = lane_s + fpy;
                    const u32 aax = pax & ~3u, aay = pay & ~3u;
                    u32 x0, x1, x2, y0 = 0, y1 = 0, y2 = 0;
                    uint2 lmx, lmy = make_uint2(0, 0);
                    x0 = lds32(aax); x1 = lds32(aax + 4); x2 = lds32(aax + 8);
                    if (TWO) { y0 = lds32(aay); y1 = lds32(aay + 4); y2 = lds32(aay + 8); }
                    lmx = lds64(base_s + oLo + l1x * 8u);
                    if (TWO) lmy = lds64(base_s + oLo + l1y * 8u);
                    const u32 a0 = __funnelshift_r(x0, x1, pax << 3) & lmx.x;
                    const u32 a1 = __funnelshift_r(x1, x2, pax << 3) & lmx.y;
                    const u32 b0 = __funnelshift_r(y0, y1, pay << 3) & lmy.x;
                    const u32 b1 = __funnelshift_r(y1, y2, pay << 3) & lmy.y;
                    const u32 seta = __umulhi(a0 * 0x9E3779B1u + a1 * 0x85EBCA77u, (u32)SETS);
                    const u32 setb = __umulhi(b0 * 0x9E3779B1u + b1 * 0x85EBCA77u, (u32)SETS);
                    const uint4 p = lds128(base_s + oSk + seta * 16u);
                    uint4 r = make_uint4(0, 0, 0, 0);
                    if (TWO) r = lds128(base_s + oSk + setb * 16u);
                    const bool ha0 = p.x == a0 && p.y == a1, ha1 = p.z == a0 && p.w == a1;
                    const bool hb0 = r.x == b0 && r.y == b1, hb1 = r.z == b0 && r.w == b1;
                    const bool fa_ = (ha0 || ha1) && sx, fb_ = (hb0 || hb1) && sy;
                    // a token that missed counts into the warp's dummy word: no branch around the atomic
                    red_inc(fa_ ? base_s + oCnt + seta * 8u + (ha1 ? 4u : 0u) : wb + oDummy);
                    if (TWO) red_inc(fb_ ? base_s + oCnt + setb * 8u + (hb1 ? 4u : 0u) : wb + oDummy);
                    const bool m0 = sx && !fa_, m1 = sy && !fb_;
                    if (filling) {      // empty ways are only looked for while the combiner fills (and every 16th row)
                        const bool ca = m0 && (p.x == 0 || p.z == 0), cb = m1 && (r.x == 0 || r.z == 0);
                        if (__any_sync(kFull, ca || cb)) {
                            if (ca) claim(seta, p.x, p.z, a0, a1);
                            if (cb) claim(setb, r.x, r.z, b0, b1);
                        }
                    }
                    if (TWO && flip) { const bool t = livex; livex = livey; livey = t; }
                    if ((livex && !sx) || (livey && !sy)) {
                        if (livex && !sx) long_token(fpx, l1x);
                        if (livey && !sy) long_token(fpy, l1y);
                    }
                    // both miss lists in one append
                    const u32 mm0 = __ballot_sync(kFull, m0), mm1 = TWO ? __ballot_sync(kFull, m1) : 0u;
                    const u32 n0 = __popc(mm0), n01 = n0 + __popc(mm1);
                    if ((mtail - mhead) + n01 > (u32)kMissCap) make_room(n01);
                    sts128_if(wb | (((mtail + __popc(mm0 & lt_mask)) * 16u) & (kMissCap * 16u - 16u)), m0, a0, a1, 0u, 0u);
                    if (TWO) sts128_if(wb | (((mtail + n0 + __popc(mm1 & lt_mask)) * 16u) & (kMissCap * 16u - 16u)), m1, b0, b1, 0u, 0u);
                    mtail += n01;
                };
                const std::true_type kYes{};
                const std::false_type kNo{};
                trip(kYes, kYes);
                drain_step();
                while (__any_sync(kFull, (Fm & (Fm - 1u)) != 0)) { trip(kYes, kNo); drain_step(); }
                while (__any_sync(kFull, Fm != 0)) { trip(kNo, kNo); drain_step(); }
            } else {
                // ------------------------------ careful row ------------------------------
                // end by end, on 64-bit views (bit i = byte i - 32 of the chunk); fragments with a byte >= 0x80 or
                // with no whitespace in sight are deferred, everything else goes through the queue
                u32 pA = __shfl_up_sync(kFull, A, 1), pH = __shfl_up_sync(kFull, H, 1);
                carry_hi = __shfl_sync(kFull, H, 31) != 0;
                if (lane == 0) {     // the previous row's last chunk: reclassify its folded bytes (the guard)
                    const uint4 g0 = lds128(ring_s + slotpos), g1 = lds128(ring_s + slotpos + 16);
                    uint4 t0, t1;
                    const Masks m0 = classify16<false>(g0, 1u, t0), m1 = classify16<false>(g1, 1u, t1);
                    pA = pack7(m0.a7, m1.a7);
                    pH = pack7(m0.h7, m1.h7);
                }
                const u64 VS = ((u64)W << 32) | pW, VA = ((u64)A << 32) | pA, VH = ((u64)H << 32) | pH;
                u32 Ew = W & ~((W << 1) | (pW >> 31));          // fragment ends: whitespace whose predecessor is not
                while (__any_sync(kFull, Ew != 0)) {
                    if (Ew) {
                        const u32 j = __ffs(Ew) - 1;
                        Ew &= Ew - 1;
                        const u64 below = (1ull << (32 + j)) - 1ull;       // bits below the end
                        const u64 sp = VS & below;
                        const u32 start = 64 - __clzll((long long)sp);     // first byte of the fragment (0 if sp == 0)
                        const u64 frag = below & ~((1ull << start) - 1ull);
                        const u64 a = VA & frag;
                        bool df = sp == 0 || (VH & frag) != 0;
                        if (!df && a) {
                            const u32 first = __ffsll((long long)a) - 1;
                            const u32 tlen = 64 - __clzll((long long)a) - first;
                            if (tlen > 16) df = true;
                            else { enqueue(lane_s + first - 32u - ring_s, tlen - 1); ++my_tokens; }
                        }
                        if (df) defer((u64)row * kRow + (u64)lane * 32 + j);
                    }
                    run_queue(kQueueCap - 64);
                }
            }
            // queued tokens must be counted before their bytes leave the ring
            __syncwarp();
            if (qtail_now() != qhead) run_queue(1);

            // the slot is free: request the row after next
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0 && row + 2 < tma_end)
                tma_row(slot_s, text + (u64)(row + 2) * kRow, kRow, bar_s + (row & 1u) * 8u);
        }
        while (mtail != mhead || __any_sync(kFull, dleft != 0)) drain_round();
    }

    // token total: one atomic per warp
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) my_tokens += __shfl_xor_sync(kFull, my_tokens, d);
    if (lane == 0 && my_tokens) atomicAdd(gt.n_tokens, (u64)my_tokens);

    // flush the combiners into the global table
    __syncthreads();
    for (int i = tid; i < 2 * SETS; i += WARPS * 32) {
        const u64 k = reinterpret_cast<const u64*>(sm.t.sk)[i];
        const u32 c = reinterpret_cast<const u32*>(sm.t.scnt)[i];
        if (k != 0 && c) table_add(gt, le_to_be(k), 0ull, (u64)c, &inserted);
    }
    for (int i = tid; i < MSLOTS; i += WARPS * 32) {
        const u64 k = sm.t.mk0[i];
        const u32 c = sm.t.mcnt[i];
        if (k > kSlotLocked && c) table_add(gt, le_to_be(k), le_to_be(sm.t.mk1[i]), (u64)c, &inserted);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) inserted += __shfl_xor_sync(kFull, inserted, d);
    if (lane == 0) table_note_inserted(gt, inserted);
}

template <int WARPS, int SETS, int MSLOTS>
__global__ void __launch_bounds__(WARPS * 32, 1)
wc_count4_kernel(const uint8_t* __restrict__ text, u64 n, u32 rows_per_warp, int force, TableView gt) {
    if (variant_of_text(text, n, force, gt.launched, gt.wanted) != kVarNarrow)
        return;
    wc_count4_body<WARPS, SETS, MSLOTS>(text, n, rows_per_warp, gt);
}

}  // namespace cnt4

#ifndef WFCU_COUNT4_SETS
#define WFCU_COUNT4_SETS 3840
#endif
#ifndef WFCU_COUNT4_MED_SLOTS
#define WFCU_COUNT4_MED_SLOTS 256
#endif

// the ASCII body for texts whose sample asks for the narrow variant; warps and the partition of the text are the
// third generation's, whose other variants take the other texts (wc_count.cu)
cudaError_t wc_count4_launch(const uint8_t* text, u64 n, u32 rows_per_warp, unsigned grid, int force, const TableView& gt,
                             cudaStream_t stream) {
    typedef cnt4::Smem<cntc::kCountVariantWarps, WFCU_COUNT4_SETS, WFCU_COUNT4_MED_SLOTS> SM;
    static_assert(sizeof(SM) + 1024 <= 227 * 1024, "shared memory budget");
    static_assert(cnt4::kRingBytes + 16 <= 4096, "queue entries keep ring offsets in 12 bits");
    const size_t smem = sizeof(SM) + 1024;   // + slack for the 1 KiB alignment
    auto k = cnt4::wc_count4_kernel<cntc::kCountVariantWarps, WFCU_COUNT4_SETS, WFCU_COUNT4_MED_SLOTS>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, cntc::kCountVariantWarps * 32, smem, stream>>>(text, n, rows_per_warp, force, gt);
    return cudaGetLastError();
}

}  // namespace wfcu
