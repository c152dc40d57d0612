// wc_count_common.cuh -- SWAR byte classes and small helpers shared by the counting kernels
// (wc_count.cu: third generation, kept for the two-byte-letter variant; wc_count4.cu: fourth generation).
#pragma once
#include <cstdlib>
#include <type_traits>

#include "wfcu_dev.cuh"

namespace wfcu {
namespace cntc {

constexpr u32 kFull = 0xFFFFFFFFu;
constexpr u64 kSlotLocked = 1ull;

// ---- SWAR byte classes: bit 7 of each byte lane is the answer ----------------------
// ASCII = true: caller guarantees no byte has bit 7 set.
// The range-test additions can run on the FMA pipe as v * one + K (IMAD R, R, Rone, imm) with a 1 the
// compiler cannot see through (a kernel argument): the integer ALU pipe is the busiest unit of the kernel.
// WFCU_FMA_ADDS: bit i = addition i of classify4 goes to the FMA pipe.
#ifndef WFCU_FMA_ADDS
#define WFCU_FMA_ADDS 0
#endif
template <u32 K, int BIT>
__device__ __forceinline__ u32 add_k(u32 v, u32 one) {
    if ((WFCU_FMA_ADDS >> BIT) & 1) return v * one + K;
    return v + K;
}
template <bool ASCII>
__device__ __forceinline__ void classify4(u32 x, u32 one, u32& s, u32& t, u32& u, u32& f) {
    const u32 M = 0x80808080u;
    const u32 v = ASCII ? x : (x & 0x7F7F7F7Fu);
    const u32 y = v | 0x20202020u;
    t = add_k<0x1F1F1F1Fu, 0>(y, one) & ~add_k<0x05050505u, 1>(y, one) & M;          // 'a'..'z' after folding
    u = add_k<0x50505050u, 2>(v, one) & ~add_k<0x46464646u, 3>(v, one) & M;          // '0'..'9'
    const u32 z = add_k<0x7F7F7F7Fu, 4>(v ^ 0x20202020u, one);                       // bit 7 clear <=> byte == 0x20
    s = (~z | (add_k<0x77777777u, 5>(v, one) & ~add_k<0x72727272u, 6>(v, one))) & M; // 0x20 or 0x09..0x0D
    if (!ASCII) { t &= ~x; u &= ~x; s &= ~x; }
    f = x | (t >> 2);                                        // A-Z -> a-z (a-z unchanged)
}

// flags (0x80 per byte) of two words -> 128 * (8-bit mask), accumulated on the FMA pipe
__device__ __forceinline__ u32 gather8(u32 f0, u32 f1, u32 acc) {
    return __dp4a(f0, 0x08040201u, __dp4a(f1, 0x80402010u, acc));
}

struct Masks { u32 s7, a7, h7; };   // 16-bit masks of one 16-byte chunk, scaled by 128

template <bool ASCII>
__device__ __forceinline__ Masks classify16(const uint4& x, u32 one, uint4& f) {
    u32 s0, s1, s2, s3, t0, t1, t2, t3, u0, u1, u2, u3;
    classify4<ASCII>(x.x, one, s0, t0, u0, f.x);
    classify4<ASCII>(x.y, one, s1, t1, u1, f.y);
    classify4<ASCII>(x.z, one, s2, t2, u2, f.z);
    classify4<ASCII>(x.w, one, s3, t3, u3, f.w);
    Masks m;
    m.s7 = gather8(s2, s3, 0) * 256u + gather8(s0, s1, 0);
    m.a7 = gather8(t2, t3, gather8(u2, u3, 0)) * 256u + gather8(t0, t1, gather8(u0, u1, 0));
    m.h7 = 0;
    if (!ASCII) {
        const u32 M = 0x80808080u;
        m.h7 = gather8(x.z & M, x.w & M, 0) * 256u + gather8(x.x & M, x.y & M, 0);
    }
    return m;
}
// pack the masks of the lane's two chunks: low 16 bits = half a, high 16 bits = half b
__device__ __forceinline__ u32 pack7(u32 a7, u32 b7) { return (b7 << 9) | (a7 >> 7); }

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// PTX shifts clamp: a shift amount >= 32 gives 0 (C++ leaves it undefined)
__device__ __forceinline__ u32 shr_clamp(u32 v, u32 s) {
    u32 r;
    asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(s));
    return r;
}
__device__ __forceinline__ u32 shl_clamp(u32 v, u32 s) {
    u32 r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(s));
    return r;
}
// warp inclusive prefix sum; the shuffle's own predicate replaces the lane compare
__device__ __forceinline__ u32 warp_inclusive_sum(u32 v) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        asm volatile("{ .reg .pred p; .reg .u32 t; shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff; @p add.u32 %0, %0, t; }"
                     : "+r"(v) : "r"(d));
    }
    return v;
}

__device__ __forceinline__ u32 bswap32(u32 v) { return __byte_perm(v, 0, 0x0123); }
__device__ __forceinline__ u64 le_to_be(u64 v) { return ((u64)bswap32((u32)v) << 32) | bswap32((u32)(v >> 32)); }

// Medium tokens (9..16 bytes): 2-way, k1 is written before k0 is published.
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
                atomicExch(k0s + i, k0);
                atomicAdd(cnt + i, 1u);
                return true;
            }
        }
        if (c0 == kSlotLocked) return false;
        if (c0 == k0 && *reinterpret_cast<volatile u64*>(k1s + i) == k1) {
            atomicAdd(cnt + i, 1u);
            return true;
        }
        i = (h >> 16) & mask;
    }
    return false;
}

// ---- which kernel variant counts a text ------------------------------------------------------------
// Every counting kernel has kCountVariantWarps warps and the same partition of the text (a strip of
// rows_per_warp KiB rows per warp).  Every CTA of every launched kernel reads the SAME sample -- one 16-byte chunk per
// thread, spread evenly over the whole text -- and so reaches the same answer without communicating:
//   kVarHi     (two-byte letters on the fast path) as soon as two chunks hold a byte >= 0x80,
//   kVarHi3    (two- and three-byte letters) when two chunks hold a lead byte E0..EE other than E2,
//   kVarWide   (one combiner for all tokens of up to 16 bytes) when 20 of the 896 chunks hold a run of nine or more
//              word characters (non-whitespace bytes in chunks with bytes >= 0x80): words longer than 8 bytes are
//              common -- English prose, the 1 M-word corpus,
//   kVarHiWide / kVarHiWide3 when that holds too,
//   kVarNarrow otherwise.
// The CTAs of the other kernels return.  The choice affects speed only.  It is one choice per call, not per CTA: the
// kernels of a call run one after the other, each with one CTA per SM, so CTAs that disagreed (a sample near a
// threshold, a mixed corpus) would leave SMs idle in every kernel -- measured: text with 13 % kana words at 194 GB/s
// when its CTAs split between two variants, 400 GB/s under either of them.  Callers that stream a corpus in chunks
// (wfcu_counter_count_host: 32 MiB) get one choice per chunk.
// Not every variant is launched every time (TableView::launched: the host launches what the counter's recent texts
// asked for, TableView::wanted): a text whose variant is missing runs the nearest HI kernel that was launched, else
// the narrow body, which is always there.
// force (WFCU_COUNT_VARIANT, tests): the variant number 0..5; else sample.
#ifndef WFCU_COUNT_WARPS
#define WFCU_COUNT_WARPS 28
#endif
constexpr int kCountVariantWarps = WFCU_COUNT_WARPS;
constexpr int kVarNarrow = 0, kVarHi = 1, kVarWide = 2, kVarHiWide = 3, kVarHi3 = 4, kVarHiWide3 = 5, kVarCount = 6;
__host__ __device__ constexpr bool variant_is_hi(int v) { return v == kVarHi || v == kVarHiWide || v == kVarHi3 || v == kVarHiWide3; }
__host__ __device__ constexpr bool variant_is_wide(int v) { return v == kVarWide || v == kVarHiWide || v == kVarHiWide3; }
__host__ __device__ constexpr bool variant_is_u3(int v) { return v == kVarHi3 || v == kVarHiWide3; }
__device__ __forceinline__ int variant_of_text(const uint8_t* __restrict__ text, u64 n, int force, u32 launched,
                                               unsigned int* wanted_word) {
    int want = kVarNarrow;
    if (force >= 0 && force < kVarCount) {
        want = force;
    } else {
        const u64 at = ((u64)threadIdx.x * (n / (u64)(kCountVariantWarps * 32))) & ~15ull;
        bool hit = false, hit3 = false, hit9 = false;
        if (at + 16 <= n) {
            const uint4 q = *reinterpret_cast<const uint4*>(text + at);
            hit = ((q.x | q.y | q.z | q.w) & 0x80808080u) != 0;
            if (hit) {
                const u32 w4[4] = {q.x, q.y, q.z, q.w};
                u32 any = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const u32 xw = w4[k], v = xw & 0x7F7F7F7Fu;
                    any |= xw & (v + 0x20202020u) & ~(v + 0x11111111u) & ((v ^ 0x62626262u) + 0x7F7F7F7Fu);   // E0..EE, not E2
                }
                hit3 = (any & 0x80808080u) != 0;
            }
            // a run of nine: of word characters in an ASCII chunk (a token longer than 8 bytes for certain), of
            // non-whitespace bytes in a chunk with bytes >= 0x80 (what is a letter there is the kernels' business)
            uint4 f;
            const Masks m = classify16<false>(q, 1u, f);
            const u32 N = (hit ? ~(m.s7 >> 7) : (m.a7 >> 7)) & 0xFFFFu;
            u32 r = N & (N >> 1);
            r &= r >> 2;
            r &= r >> 4;
            hit9 = (r & (N >> 8)) != 0;
        }
        const int c_hi = __syncthreads_count(hit), c3 = __syncthreads_count(hit3), c9 = __syncthreads_count(hit9);
        const bool wide = c9 >= 20;
        want = c_hi < 2 ? (wide ? kVarWide : kVarNarrow)
                        : c3 >= 2 ? (wide ? kVarHiWide3 : kVarHi3) : (wide ? kVarHiWide : kVarHi);
    }
    if (wanted_word && threadIdx.x == 0 && blockIdx.x == 0) atomicOr(wanted_word, 1u << want);
    // the wanted kernel, else the nearest launched one that is exact AND fast on the same kind of text, else narrow
    // (four candidates per wanted variant, one per nibble, first choice lowest)
    const u32 prefer = want == kVarHi ? 0x5341u : want == kVarHiWide ? 0x4153u : want == kVarHi3 ? 0x3154u
                     : want == kVarHiWide3 ? 0x1345u : (u32)want * 0x1111u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int cand = (int)((prefer >> (4 * k)) & 15u);
        if ((launched >> cand) & 1u) return cand;
    }
    return kVarNarrow;
}

}  // namespace cntc
}  // namespace wfcu
