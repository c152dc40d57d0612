// wfcu_dev.cuh -- device-side building blocks shared by the kernels of libwfcu.
//
// Data layout in HBM:
//   * count table: open addressing, 32-byte slots {k0,k1,count,aux}.  A token of
//     at most 16 bytes IS its key: k0 = bytes 0..7, k1 = bytes 8..15, first byte
//     most significant, zero padded.  A normalised token ends in a word
//     character, so it never ends in NUL and the padding is unambiguous; k0 == 0
//     marks an empty slot.  Integer order on (k0,k1) is unsigned byte-wise
//     lexicographic order, i.e. std::map<std::string,...> order
//     (/root/reference/proj/include/wfc/reduce.hpp:15).  No 64-bit hash stands in
//     for a key, so counts are exact by construction (SURVEY.md hard part H2).
//   * tokens longer than 16 bytes live in a byte arena and a second table whose
//     slots point at arena records; equality there is full string equality.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace wfcu {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr int kStatusTableFull = 1;
constexpr int kStatusDeferredFull = 2;
constexpr int kStatusArenaFull = 4;
constexpr int kStatusLongFull = 8;
constexpr int kStatusNotSorted = 16;

struct __align__(32) Slot {
    u64 k0, k1, count, aux;
};

// Device view of a counter (all pointers are device addresses).
struct TableView {
    Slot* slots;
    u64 mask;           // slots - 1
    u64 max_used;       // load limit
    u64* n_used;        // distinct inline keys
    u64* n_tokens;      // total tokens counted (fast path adds per CTA)
    // slow path
    u64* deferred;      // global end offsets of fragments the fast path skipped
    u64 deferred_cap;
    u64* n_deferred;
    // long tokens
    u64* long_ref;      // arena offset of the record, 0 = empty
    u64* long_count;
    u64 long_mask;
    u64* n_long;
    uint8_t* arena;     // records {u32 len, u32 hash, bytes..., pad to 8}; offset 0 unused
    u64 arena_cap;
    u64* arena_used;
    int* status;
    unsigned int* ticket = nullptr;   // a zeroed word for "last CTA" decisions (null: the caller launches the follow-up itself)
    unsigned int* wanted = nullptr;   // OR of (1 << variant) the CTAs of the counting kernels asked for (a hint for later launches)
    unsigned int launched = 63;       // variants launched in this call: a CTA whose variant is missing runs the narrow body
};

// One token of a device-resident token list (wfcu_tokens), 32 bytes.
//   k0,k1 : first 16 bytes of the token, big-endian packed, zero padded
//   ext   : 0 for tokens of <= 16 bytes; otherwise the arena offset of the full
//           record {u32 len, u32 hash, bytes...}
//   pos   : byte offset of the token in the text (text order = pos order)
struct __align__(32) TokenRec {
    u64 k0, k1, ext, pos;
};

// Where the kernels put tokens when they run as a stand-alone tokenizer.
struct EmitView {
    TokenRec* out;
    u64 cap;
    u64* n_out;
    // Compact mode (counting by sort + RLE, where text order does not matter): a token of at most 8 bytes
    // is written as its 64-bit key into a tile of kKeyTile keys that its warp owns (one atomic per tile
    // instead of one per 32 tokens); only the longer tokens become records.  keys == nullptr: off.
    u64* keys = nullptr;
    u64 key_tiles = 0;           // capacity in tiles
    u32* tile_counts = nullptr;  // keys written to each tile
    u64* kc = nullptr;           // [0] tiles handed out, [1] keys written, [2] OR of the keys, [3] AND of the keys
};
constexpr u32 kKeyTile = 2048;   // == the radix sort's tile (tokens.cu)

// ---- hashing -----------------------------------------------------------------
// 32-bit mix of the 128-bit key.  Only used to pick a slot / an owner, never as
// an identity.
__host__ __device__ __forceinline__ u32 mix32(u64 k0, u64 k1) {
    u32 a = (u32)k0, b = (u32)(k0 >> 32), c = (u32)k1, d = (u32)(k1 >> 32);
    u32 h = a * 0x9E3779B1u;
    h ^= b * 0x85EBCA77u;
    h ^= c * 0xC2B2AE3Du;
    h ^= d * 0x27D4EB2Fu;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 13;
    return h;
}
// second, independent mix for the owner GPU of the exchange
__host__ __device__ __forceinline__ u32 owner_mix32(u64 k0, u64 k1) {
    u32 h = mix32(k0 ^ 0xA5A5A5A5A5A5A5A5ull, k1 + 0x9E3779B97F4A7C15ull);
    h *= 0x165667B1u;
    h ^= h >> 16;
    return h;
}
__host__ __device__ __forceinline__ u32 fnv32(const uint8_t* p, u64 n) {
    u32 h = 2166136261u;
    for (u64 i = 0; i < n; ++i) { h ^= p[i]; h *= 16777619u; }
    return h;
}

// ---- 128-bit compare-and-swap on a slot key ------------------------------------
#ifdef __CUDACC__
__device__ __forceinline__ ulonglong2 cas128(Slot* s, u64 k0, u64 k1) {
    // if (slot key == {0,0}) slot key = {k0,k1}; returns the previous key
    ulonglong2 old;
    asm volatile(
        "{\n\t"
        ".reg .b128 cmp, swp, res;\n\t"
        "mov.b128 cmp, {%2, %3};\n\t"
        "mov.b128 swp, {%4, %5};\n\t"
        "atom.relaxed.gpu.global.cas.b128 res, [%6], cmp, swp;\n\t"
        "mov.b128 {%0, %1}, res;\n\t"
        "}"
        : "=l"(old.x), "=l"(old.y)
        : "l"(0ull), "l"(0ull), "l"(k0), "l"(k1), "l"(s)
        : "memory");
    return old;
}

__device__ __forceinline__ ulonglong2 ld_key(const Slot* s) {
    ulonglong2 v;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(s));
    return v;
}

// counts[key] += add in the global table.  Exact: a slot is claimed with one
// 128-bit CAS, and a plain (possibly torn) read that matches k0 but not k1 is
// re-read through the CAS before the probe moves on.
// inserted != nullptr: a newly claimed slot is counted there instead of in t.n_used; the caller adds its total
// with table_note_inserted (a million first occurrences are a million atomics on ONE address otherwise).
// Probing gives up after kMaxProbes slots: below the load limit a probe sequence is orders of magnitude shorter, and
// a table that is filling up beyond it (a vocabulary larger than the caller sized the table for) would otherwise
// make every insertion walk the whole table before the call fails -- minutes instead of a prompt WFCU_ERR_TABLE_FULL.
constexpr u64 kMaxProbes = 8192;
// table_add_from: the probe sequence is entered at slot i, which the caller has SEEN -- every slot between the key's
// home and i holds another key (keys never change or leave) -- and, if assume_empty, saw empty: the claim is tried
// without loading the slot first (one dependent L2 round trip less for a first occurrence; a stale observation only
// makes the CAS return the key that took the slot meanwhile, and the walk goes on as usual).
__device__ __forceinline__ void table_add_from(const TableView& t, u64 i, bool assume_empty, u64 k0, u64 k1, u64 add,
                                               u32* inserted = nullptr) {
    const u64 limit = t.mask < kMaxProbes ? t.mask : kMaxProbes;
    for (u64 probes = 0; probes <= limit; ++probes) {
        Slot* s = t.slots + i;
        ulonglong2 cur = (probes == 0 && assume_empty) ? make_ulonglong2(0ull, 0ull) : ld_key(s);
        if (cur.x == 0 || (cur.x == k0 && cur.y != k1)) {
            cur = cas128(s, k0, k1);
            if (cur.x == 0 && cur.y == 0) {
                if (inserted) {
                    ++*inserted;
                } else {
                    const u64 used = atomicAdd(t.n_used, 1ull) + 1;
                    if (used > t.max_used) atomicOr(t.status, kStatusTableFull);
                }
                cur.x = k0; cur.y = k1;
            }
        }
        if (cur.x == k0 && cur.y == k1) {
            atomicAdd(&s->count, add);
            return;
        }
        i = (i + 1) & t.mask;
    }
    atomicOr(t.status, kStatusTableFull);
}

// (spelled out rather than forwarded to table_add_from: the narrow counting kernel sits at its register limit and
// measured 0.6 % slower through the forwarding form)
__device__ __forceinline__ void table_add(const TableView& t, u64 k0, u64 k1, u64 add, u32* inserted = nullptr) {
    u64 i = mix32(k0, k1) & t.mask;
    const u64 limit = t.mask < kMaxProbes ? t.mask : kMaxProbes;
    for (u64 probes = 0; probes <= limit; ++probes) {
        Slot* s = t.slots + i;
        ulonglong2 cur = ld_key(s);
        if (cur.x == 0 || (cur.x == k0 && cur.y != k1)) {
            cur = cas128(s, k0, k1);
            if (cur.x == 0 && cur.y == 0) {
                if (inserted) {
                    ++*inserted;
                } else {
                    const u64 used = atomicAdd(t.n_used, 1ull) + 1;
                    if (used > t.max_used) atomicOr(t.status, kStatusTableFull);
                }
                cur.x = k0; cur.y = k1;
            }
        }
        if (cur.x == k0 && cur.y == k1) {
            atomicAdd(&s->count, add);
            return;
        }
        i = (i + 1) & t.mask;
    }
    atomicOr(t.status, kStatusTableFull);
}

// n slots were claimed through table_add(..., &inserted): one atomic for all of them.  An over-full table is
// noticed here instead of at the insertion that crossed the limit (probing terminates either way).
__device__ __forceinline__ void table_note_inserted(const TableView& t, u64 n) {
    if (n == 0) return;
    const u64 used = atomicAdd(t.n_used, n) + n;
    if (used > t.max_used) atomicOr(t.status, kStatusTableFull);
}

// Long tokens: `rec` is the arena offset of a complete record of this token
// (already written and fenced).  Either publishes it or adds to the equal one.
__device__ __forceinline__ void long_add(const TableView& t, u64 rec, u64 add) {
    const u32 len = *reinterpret_cast<const u32*>(t.arena + rec);
    const u32 hash = *reinterpret_cast<const u32*>(t.arena + rec + 4);
    u64 i = hash & t.long_mask;
    const u64 limit = t.long_mask < kMaxProbes ? t.long_mask : kMaxProbes;
    for (u64 probes = 0; probes <= limit; ++probes) {
        u64 r = *reinterpret_cast<volatile u64*>(t.long_ref + i);
        if (r == 0) {
            r = atomicCAS(t.long_ref + i, 0ull, rec);
            if (r == 0) {
                const u64 used = atomicAdd(t.n_long, 1ull) + 1;
                if (used * 2 > t.long_mask + 1) atomicOr(t.status, kStatusLongFull);
                atomicAdd(t.long_count + i, add);
                return;
            }
        }
        // r is a published record: compare strings
        const u32 rlen = *reinterpret_cast<const u32*>(t.arena + r);
        const u32 rhash = *reinterpret_cast<const u32*>(t.arena + r + 4);
        if (rlen == len && rhash == hash) {
            const uint8_t* a = t.arena + r + 8;
            const uint8_t* b = t.arena + rec + 8;
            bool same = true;
            u32 k = 0;
            for (; k + 8 <= len && same; k += 8)      // records are 8-byte aligned
                same = *reinterpret_cast<const u64*>(a + k) == *reinterpret_cast<const u64*>(b + k);
            for (; k < len && same; ++k) same = a[k] == b[k];
            if (same) {
                atomicAdd(t.long_count + i, add);
                return;
            }
        }
        i = (i + 1) & t.long_mask;
    }
    atomicOr(t.status, kStatusLongFull);
}

// Reserves an arena record for a token of `len` bytes; returns 0 on overflow.
__device__ __forceinline__ u64 arena_alloc(const TableView& t, u32 len) {
    const u64 need = 8 + ((u64(len) + 7) & ~7ull);
    const u64 off = atomicAdd(t.arena_used, need);
    if (off + need > t.arena_cap) {
        atomicOr(t.status, kStatusArenaFull);
        return 0;
    }
    return off;
}
#endif  // __CUDACC__

// ---- key <-> bytes (host and device) ------------------------------------------
__host__ __device__ __forceinline__ void key_from_bytes(const uint8_t* p, u32 len, u64* k0, u64* k1) {
    u64 a = 0, b = 0;
    for (u32 i = 0; i < 8; ++i) a = (a << 8) | (i < len ? p[i] : 0);
    for (u32 i = 8; i < 16; ++i) b = (b << 8) | (i < len ? p[i] : 0);
    *k0 = a; *k1 = b;
}
__host__ __device__ __forceinline__ u32 key_len(u64 k0, u64 k1) {
    // number of bytes up to the last non-zero byte
    u32 n = 0;
    for (u32 i = 0; i < 8; ++i) if ((k0 >> (56 - 8 * i)) & 0xFF) n = i + 1;
    for (u32 i = 0; i < 8; ++i) if ((k1 >> (56 - 8 * i)) & 0xFF) n = 9 + i;
    return n;
}
__host__ __device__ __forceinline__ void key_to_bytes(u64 k0, u64 k1, uint8_t* out /*16*/) {
    for (u32 i = 0; i < 8; ++i) out[i] = (uint8_t)(k0 >> (56 - 8 * i));
    for (u32 i = 0; i < 8; ++i) out[8 + i] = (uint8_t)(k1 >> (56 - 8 * i));
}

}  // namespace wfcu
