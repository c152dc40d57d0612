// tokens.cu -- device-resident token lists: the stand-alone tokenizer, the stable
// byte-wise sort and the run-length-encode reduce, i.e. the reference's
//   tokenize      /root/reference/proj/src/text.cpp:32-57
//   sort_words    proj/src/text.cpp:59-63      (std::stable_sort of std::string)
//   reduce_sorted proj/src/reduce.cpp:8-21     (RLE into the count map)
// kept as the alternative to the hash-count path for high-cardinality vocabularies.
//
// A token is a 32-byte TokenRec: its first 16 bytes big-endian packed (so unsigned
// integer order on (k0,k1) IS byte-wise lexicographic order), an arena reference for
// the rare token longer than 16 bytes, and its text position.
//   * sort: hand-written stable LSD radix sort, 8-bit digits, keys (is_long, k1, k0);
//     one OR/AND reduction over the keys finds the byte positions that vary at all and
//     only those passes run (k1 is all zero for corpora of short words: 8 passes gone);
//     ties between long tokens that share a 16-byte prefix are ordered by an exact
//     string fix-up pass.
//   * RLE: head flags by adjacent comparison -> exclusive scan -> run starts ->
//     counts[key] += run length in the table.
#include "wfcu_dev.cuh"

namespace wfcu {

// ---------------------------------------------------------------------------------
// exclusive scan of u64 (three-phase, up to 2^30 elements)
// ---------------------------------------------------------------------------------
constexpr int kScanBlock = 1024;

__global__ void scan_reduce_kernel(const u64* __restrict__ in, u64 n, u64* __restrict__ block_sums) {
    __shared__ u64 warp_sums[32];
    const u64 i = (u64)blockIdx.x * kScanBlock + threadIdx.x;
    u64 v = i < n ? in[i] : 0;
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, d);
    if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = warp_sums[threadIdx.x];
        for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, d);
        if (threadIdx.x == 0) block_sums[blockIdx.x] = v;
    }
}

// exclusive scan inside each block of kScanBlock elements, plus block_offsets[block]
__global__ void scan_block_kernel(const u64* __restrict__ in, u64 n, const u64* __restrict__ block_offsets,
                                  u64* __restrict__ out) {
    __shared__ u64 warp_sums[32];
    const u64 i = (u64)blockIdx.x * kScanBlock + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const u64 x = i < n ? in[i] : 0;
    u64 v = x;
    for (int d = 1; d < 32; d <<= 1) {
        const u64 t = __shfl_up_sync(0xFFFFFFFFu, v, d);
        if (lane >= d) v += t;
    }
    if (lane == 31) warp_sums[warp] = v;
    __syncthreads();
    if (warp == 0) {
        u64 w = warp_sums[lane];
        for (int d = 1; d < 32; d <<= 1) {
            const u64 t = __shfl_up_sync(0xFFFFFFFFu, w, d);
            if (lane >= d) w += t;
        }
        warp_sums[lane] = w;
    }
    __syncthreads();
    const u64 base = (block_offsets ? block_offsets[blockIdx.x] : 0) + (warp ? warp_sums[warp - 1] : 0);
    if (i < n) out[i] = base + v - x;
}

// out = exclusive_scan(in) ; tmp must hold ceil(n/1024) + ceil(n/1024^2) + 2 u64.  in may alias out.
cudaError_t exclusive_scan_u64(const u64* in, u64* out, u64 n, u64* tmp, cudaStream_t s, u64* launches) {
    if (n == 0) return cudaSuccess;
    const u64 nb = (n + kScanBlock - 1) / kScanBlock;
    if (nb == 1) {
        scan_block_kernel<<<1, kScanBlock, 0, s>>>(in, n, nullptr, out);
        *launches += 1;
        return cudaGetLastError();
    }
    u64* sums = tmp;
    scan_reduce_kernel<<<(unsigned)nb, kScanBlock, 0, s>>>(in, n, sums);
    *launches += 1;
    cudaError_t e = exclusive_scan_u64(sums, sums, nb, tmp + nb, s, launches);
    if (e != cudaSuccess) return e;
    scan_block_kernel<<<(unsigned)nb, kScanBlock, 0, s>>>(in, n, sums, out);
    *launches += 1;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------
// stable LSD radix sort of TokenRec
// ---------------------------------------------------------------------------------
constexpr int kSortWarps = 4;          // warps per CTA, one tile each
constexpr int kTileItems = 2048;       // records per warp tile

// pass: 0..7 -> byte of k1 (least significant first), 8..15 -> byte of k0, 16 -> pos bytes via separate kernel mode
__device__ __forceinline__ u32 digit_of(const TokenRec& r, int mode, int pass) {
    if (mode == 0) return (u32)((pass < 8 ? r.k1 >> (8 * pass) : r.k0 >> (8 * (pass - 8))) & 0xFF);
    if (mode == 1) return (u32)((r.pos >> (8 * pass)) & 0xFF);   // text order
    return r.ext ? 1u : 0u;                                      // mode 2: long tokens after equal inline ones
}

// hist[digit * n_tiles + tile]
__global__ void sort_hist_kernel(const TokenRec* __restrict__ in, u64 n, u64 n_tiles, int mode, int pass,
                                 u64* __restrict__ hist) {
    __shared__ u32 sh[kSortWarps][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u64 tile = (u64)blockIdx.x * kSortWarps + warp;
    for (int d = lane; d < 256; d += 32) sh[warp][d] = 0;
    __syncwarp();
    if (tile < n_tiles) {
        const u64 lo = tile * kTileItems;
        const u64 hi = min(lo + (u64)kTileItems, n);
        for (u64 i = lo + lane; i < hi; i += 32) atomicAdd(&sh[warp][digit_of(in[i], mode, pass)], 1u);
    }
    __syncwarp();
    if (tile < n_tiles)
        for (int d = lane; d < 256; d += 32) hist[(u64)d * n_tiles + tile] = sh[warp][d];
}

// offs = exclusive scan of hist (digit-major), scatter keeps the tile order inside a digit
__global__ void sort_scatter_kernel(const TokenRec* __restrict__ in, TokenRec* __restrict__ out, u64 n, u64 n_tiles,
                                    int mode, int pass, const u64* __restrict__ offs) {
    __shared__ u64 sh[kSortWarps][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u64 tile = (u64)blockIdx.x * kSortWarps + warp;
    if (tile >= n_tiles) return;
    for (int d = lane; d < 256; d += 32) sh[warp][d] = offs[(u64)d * n_tiles + tile];
    __syncwarp();
    const u64 lo = tile * kTileItems;
    const u64 hi = min(lo + (u64)kTileItems, n);
    const u32 lt = (1u << lane) - 1u;
    for (u64 base = lo; base < hi; base += 32) {
        const u64 i = base + lane;
        const bool live = i < hi;
        TokenRec r{};
        u32 d = 0xFFFFFFFFu;
        if (live) {
            r = in[i];
            d = digit_of(r, mode, pass);
        }
        const u32 peers = __match_any_sync(0xFFFFFFFFu, d);
        u64 dst = 0;
        if (live) dst = sh[warp][d] + __popc(peers & lt);
        __syncwarp();
        if (live && (peers & lt) == 0) sh[warp][d] += __popc(peers);   // lowest lane of each digit group
        __syncwarp();
        if (live) out[dst] = r;
    }
}

// OR / AND of every key word over all records: a byte position whose OR equals its AND is
// constant and its radix pass can be skipped without being launched.
// out[0..3] = OR(k0), AND(k0), OR(k1), AND(k1); out[4] = #records with ext != 0; out[5] = OR/AND of pos (two words)
__global__ void sort_key_range_kernel(const TokenRec* __restrict__ in, u64 n, u64* __restrict__ out) {
    u64 o0 = 0, a0 = ~0ull, o1 = 0, a1 = ~0ull, op = 0, ap = ~0ull, nl = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const TokenRec r = in[i];
        o0 |= r.k0; a0 &= r.k0; o1 |= r.k1; a1 &= r.k1; op |= r.pos; ap &= r.pos;
        nl += r.ext != 0;
    }
    for (int d = 16; d > 0; d >>= 1) {
        o0 |= __shfl_xor_sync(0xFFFFFFFFu, o0, d); a0 &= __shfl_xor_sync(0xFFFFFFFFu, a0, d);
        o1 |= __shfl_xor_sync(0xFFFFFFFFu, o1, d); a1 &= __shfl_xor_sync(0xFFFFFFFFu, a1, d);
        op |= __shfl_xor_sync(0xFFFFFFFFu, op, d); ap &= __shfl_xor_sync(0xFFFFFFFFu, ap, d);
        nl += __shfl_xor_sync(0xFFFFFFFFu, nl, d);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(out + 0, o0); atomicAnd(out + 1, a0); atomicOr(out + 2, o1); atomicAnd(out + 3, a1);
        atomicAdd(out + 4, nl); atomicOr(out + 5, op); atomicAnd(out + 6, ap);
    }
}

// ---- long-token tie fix-up ---------------------------------------------------------
__device__ __forceinline__ int long_compare(const uint8_t* arena, u64 a, u64 b) {
    const u32 la = *reinterpret_cast<const u32*>(arena + a), lb = *reinterpret_cast<const u32*>(arena + b);
    const uint8_t* pa = arena + a + 8;
    const uint8_t* pb = arena + b + 8;
    const u32 m = la < lb ? la : lb;
    u32 i = 16;                      // the first 16 bytes are known equal
    for (; i + 8 <= m; i += 8)       // records are 8-byte aligned: a word at a time up to the first difference
        if (*reinterpret_cast<const u64*>(pa + i) != *reinterpret_cast<const u64*>(pb + i)) break;
    for (; i < m; ++i) {
        if (pa[i] != pb[i]) return pa[i] < pb[i] ? -1 : 1;
    }
    return la < lb ? -1 : (la > lb ? 1 : 0);
}

// Long tokens (ext != 0) are ordered among themselves by the bytes behind their 16-byte prefix with the same LSD radix
// sort, window by window: the `pos` field, which only means something in text order, is overwritten with the sort
// key of the current window -- bytes [16 + 8w, 24 + 8w) of the string, big-endian, zero padded -- or, for the least
// significant pass of all, with the length (a string sorts behind its own prefixes; zero padding alone cannot tell
// "ab" from "ab\0").  range[5] / range[6] collect OR / AND of the key so that constant digit positions are skipped,
// range[4] the longest string (window < 0 only).
__device__ __forceinline__ u64 long_window_key(const uint8_t* arena, u64 ext, int window);
__global__ void sort_fill_window_kernel(TokenRec* __restrict__ recs, u64 n, const uint8_t* __restrict__ arena, int window,
                                        u64* __restrict__ range) {
    u64 o = 0, a = ~0ull, longest = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 ext = recs[i].ext;
        u64 key = 0;
        if (ext) {
            const u32 len = *reinterpret_cast<const u32*>(arena + ext);
            if (window < 0) {
                key = len;
                longest = longest > len ? longest : len;
            } else {
                key = long_window_key(arena, ext, window);
            }
        }
        recs[i].pos = key;
        o |= key; a &= key;
    }
    for (int d = 16; d > 0; d >>= 1) {
        o |= __shfl_xor_sync(0xFFFFFFFFu, o, d);
        a &= __shfl_xor_sync(0xFFFFFFFFu, a, d);
        const u64 other = __shfl_xor_sync(0xFFFFFFFFu, longest, d);
        longest = longest > other ? longest : other;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(range + 5, o);
        atomicAnd(range + 6, a);
        if (window < 0) atomicMax(reinterpret_cast<unsigned long long*>(range + 4), (unsigned long long)longest);
    }
}

// OR / AND of the window keys of windows [w0, w0 + count) over all long records: out[2 * j] |= key, out[2 * j + 1] &= key
// for window w0 + j.  One launch and one host read decide for a batch of windows which of them need a pass at all
// (a pair of identical 8 MiB tokens is 4096 windows in which nothing varies).
constexpr int kWindowBatch = 64;
__device__ __forceinline__ u64 long_window_key(const uint8_t* arena, u64 ext, int window) {
    const u32 len = *reinterpret_cast<const u32*>(arena + ext);
    const uint8_t* p = arena + ext + 8;
    const u32 lo = 16u + 8u * (u32)window;
    const u32 hi = len < lo + 8u ? len : lo + 8u;
    u64 key = 0;
    for (u32 j = lo; j < hi; ++j) key |= (u64)p[j] << (8 * (lo + 7 - j));
    return key;
}
__global__ void sort_window_range_kernel(const TokenRec* __restrict__ recs, u64 n, const uint8_t* __restrict__ arena, int w0,
                                         int count, u64* __restrict__ out) {
    for (int j = 0; j < count; ++j) {
        u64 o = 0, a = ~0ull;
        for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
            const u64 ext = recs[i].ext;
            const u64 key = ext ? long_window_key(arena, ext, w0 + j) : 0;
            o |= key; a &= key;
        }
        for (int d = 16; d > 0; d >>= 1) {
            o |= __shfl_xor_sync(0xFFFFFFFFu, o, d);
            a &= __shfl_xor_sync(0xFFFFFFFFu, a, d);
        }
        if ((threadIdx.x & 31) == 0) { atomicOr(out + 2 * j, o); atomicAnd(out + 2 * j + 1, a); }
    }
}

// out[0] = longest length below `longest`, out[1] = records whose length equals `longest`: windows behind the end of
// the SECOND longest string cannot order anything (at most one record has bytes there), so one 30 KB token in a list
// does not cost 3 700 window rounds.
__global__ void sort_second_longest_kernel(const TokenRec* __restrict__ recs, u64 n, const uint8_t* __restrict__ arena,
                                           u64 longest, u64* __restrict__ out) {
    u64 below = 0, equal = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 ext = recs[i].ext;
        if (!ext) continue;
        const u64 len = *reinterpret_cast<const u32*>(arena + ext);
        if (len == longest) ++equal;
        else below = below > len ? below : len;
    }
    for (int d = 16; d > 0; d >>= 1) {
        const u64 ob = __shfl_xor_sync(0xFFFFFFFFu, below, d);
        below = below > ob ? below : ob;
        equal += __shfl_xor_sync(0xFFFFFFFFu, equal, d);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)below);
        atomicAdd(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)equal);
    }
}

// Safety net behind the window passes (which stop at kLongWindows * 8 bytes): every long record compares itself with
// its predecessor, in parallel, and only if some pair with the same prefix descends (*descents != 0 -- strings that
// agree in their first 32 KiB) does the fix-up run: a stable insertion sort by the full string, one thread per run.
// (Round 1 ran the insertion sort unconditionally after sorting by the 16-byte prefix alone: a corpus whose most
// frequent word is longer than 16 bytes spent 28 ms per list in ONE thread walking its 23 000 equal records -- 89 % of
// wfc::run_wordcount -- and two such words with a common prefix, interleaved, took 87 SECONDS for 26 000 records.)
__global__ void sort_long_check_kernel(const TokenRec* __restrict__ recs, u64 n, const uint8_t* __restrict__ arena,
                                       u64* __restrict__ descents) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += (u64)gridDim.x * blockDim.x) {
        const TokenRec r = recs[i];
        if (!r.ext) continue;
        const TokenRec p = recs[i - 1];
        if (p.ext && p.k0 == r.k0 && p.k1 == r.k1 && long_compare(arena, p.ext, r.ext) > 0) {
            atomicOr(descents, 1ull);
            return;
        }
    }
}
__global__ void sort_long_fixup_kernel(TokenRec* __restrict__ recs, u64 n, const uint8_t* __restrict__ arena,
                                       const u64* __restrict__ descents) {
    if (*descents == 0) return;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const TokenRec r = recs[i];
        if (!r.ext) continue;
        if (i > 0) {
            const TokenRec p = recs[i - 1];
            if (p.ext && p.k0 == r.k0 && p.k1 == r.k1) continue;   // not a run head
        }
        u64 end = i + 1;
        while (end < n && recs[end].ext && recs[end].k0 == r.k0 && recs[end].k1 == r.k1) ++end;
        for (u64 a = i + 1; a < end; ++a) {
            const TokenRec x = recs[a];
            u64 b = a;
            while (b > i && long_compare(arena, recs[b - 1].ext, x.ext) > 0) {
                recs[b] = recs[b - 1];
                --b;
            }
            recs[b] = x;
        }
    }
}

// ---------------------------------------------------------------------------------
// run-length encode
// ---------------------------------------------------------------------------------
__device__ __forceinline__ int rec_compare(const TokenRec& a, const TokenRec& b, const uint8_t* arena) {
    if (a.k0 != b.k0) return a.k0 < b.k0 ? -1 : 1;
    if (a.k1 != b.k1) return a.k1 < b.k1 ? -1 : 1;
    if (!a.ext && !b.ext) return 0;
    if (!a.ext) return -1;   // a 16-byte token sorts before a longer one with that prefix
    if (!b.ext) return 1;
    return long_compare(arena, a.ext, b.ext);
}

// flags[i] = 1 when record i starts a run; sets kStatusNotSorted in *status on a descent
__global__ void rle_flags_kernel(const TokenRec* __restrict__ recs, u64 n, const uint8_t* __restrict__ arena,
                                 u64* __restrict__ flags, int* __restrict__ status) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 f = 1;
        if (i > 0) {
            const int c = rec_compare(recs[i - 1], recs[i], arena);
            if (c > 0) atomicOr(status, kStatusNotSorted);
            f = c != 0;
        }
        flags[i] = f;
    }
}

// run_start[scan[i]] = i for heads; n_runs = scan[n-1] + flags[n-1]
__global__ void rle_starts_kernel(const u64* __restrict__ flags_scan, const TokenRec* __restrict__ recs, u64 n,
                                  const uint8_t* __restrict__ arena, u64* __restrict__ run_start) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const bool head = (i == 0) || rec_compare(recs[i - 1], recs[i], arena) != 0;
        if (head) run_start[flags_scan[i]] = i;
    }
}

// counts[key of run r] += length of run r
__global__ void rle_insert_kernel(const TokenRec* __restrict__ recs, u64 n, const uint8_t* __restrict__ arena,
                                  const u64* __restrict__ run_start, const u64* __restrict__ flags_scan, TableView t) {
    // heads before the last record, plus the last record's own run
    const bool last_is_head = (n == 1) || rec_compare(recs[n - 2], recs[n - 1], arena) != 0;
    const u64 n_runs = flags_scan[n - 1] + (last_is_head ? 1 : 0);
    u64 tokens = 0;
    u32 inserted = 0;
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n_runs; r += (u64)gridDim.x * blockDim.x) {
        const u64 lo = run_start[r];
        const u64 hi = (r + 1 < n_runs) ? run_start[r + 1] : n;
        const TokenRec rec = recs[lo];
        const u64 len = hi - lo;
        tokens += len;
        if (!rec.ext) {
            table_add(t, rec.k0, rec.k1, len, &inserted);
        } else {
            const u32 blen = *reinterpret_cast<const u32*>(arena + rec.ext);
            const u64 dst = arena_alloc(t, blen);
            if (dst) {
                *reinterpret_cast<u32*>(t.arena + dst) = blen;
                *reinterpret_cast<u32*>(t.arena + dst + 4) = *reinterpret_cast<const u32*>(arena + rec.ext + 4);
                for (u32 k = 0; k < blen; ++k) t.arena[dst + 8 + k] = arena[rec.ext + 8 + k];
                __threadfence();
                long_add(t, dst, len);
            }
        }
    }
    for (int d = 16; d > 0; d >>= 1) {
        tokens += __shfl_xor_sync(0xFFFFFFFFu, tokens, d);
        inserted += __shfl_xor_sync(0xFFFFFFFFu, inserted, d);
    }
    if ((threadIdx.x & 31) == 0) table_note_inserted(t, inserted);
    if ((threadIdx.x & 31) == 0 && tokens) atomicAdd(t.n_tokens, tokens);
}

// ---------------------------------------------------------------------------------
// host-side drivers
// ---------------------------------------------------------------------------------
static inline unsigned blocks_for(u64 items, int threads, int sm) {
    u64 g = (items + threads - 1) / threads;
    const u64 cap = (u64)sm * 16;
    if (g > cap) g = cap;
    if (g == 0) g = 1;
    return (unsigned)g;
}

constexpr int kLongWindows = 4096;   // windows of 8 bytes behind the 16-byte prefix that the radix passes order (32 KiB + 16)

struct SortScratch {
    TokenRec* alt;   // n records
    u64* hist;       // 256 * n_tiles
    u64* tmp;        // scan scratch
};

u64 sort_n_tiles(u64 n) { return (n + kTileItems - 1) / kTileItems; }
u64 sort_hist_words(u64 n) { return 256 * sort_n_tiles(n); }
u64 scan_tmp_words(u64 n) { return (n / kScanBlock + 2) + (n / ((u64)kScanBlock * kScanBlock) + 2) + 16; }

// One stable radix pass; data ends up in `b` (either scattered or copied).
static cudaError_t radix_pass(TokenRec* a, TokenRec* b, u64 n, int mode, int pass, const SortScratch& sc, int sm,
                              cudaStream_t s, u64* launches) {
    const u64 n_tiles = sort_n_tiles(n);
    const unsigned grid = (unsigned)((n_tiles + kSortWarps - 1) / kSortWarps);
    sort_hist_kernel<<<grid, kSortWarps * 32, 0, s>>>(a, n, n_tiles, mode, pass, sc.hist);
    *launches += 1;
    cudaError_t e = exclusive_scan_u64(sc.hist, sc.hist, 256 * n_tiles, sc.tmp + 8, s, launches);
    if (e != cudaSuccess) return e;
    sort_scatter_kernel<<<grid, kSortWarps * 32, 0, s>>>(a, b, n, n_tiles, mode, pass, sc.hist);
    *launches += 1;
    return cudaGetLastError();
}

// mode 1: restore text order (sort by pos); mode 0: sort_words order.  Result in `recs`.
// sc.tmp doubles as the 8-word scratch of the key-range reduction (synchronises the stream once).
cudaError_t tokens_sort(TokenRec* recs, u64 n, bool by_position, const uint8_t* arena, const SortScratch& sc, int sm,
                        cudaStream_t s, u64* launches) {
    if (n < 2) return cudaSuccess;
    // which digit positions vary at all?
    const u64 init[8] = {0, ~0ull, 0, ~0ull, 0, 0, ~0ull, 0};
    cudaError_t e = cudaMemcpyAsync(sc.tmp, init, sizeof(init), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    sort_key_range_kernel<<<blocks_for(n, 256, sm), 256, 0, s>>>(recs, n, sc.tmp);
    *launches += 1;
    u64 range[8];
    e = cudaMemcpyAsync(range, sc.tmp, sizeof(range), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    const u64 vary_k0 = range[0] ^ range[1], vary_k1 = range[2] ^ range[3], vary_pos = range[5] ^ range[6];
    const bool mixed_long = range[4] != 0 && range[4] != n;

    TokenRec* a = recs;
    TokenRec* b = sc.alt;
    auto run = [&](int mode, int pass) {
        if (e != cudaSuccess) return;
        e = radix_pass(a, b, n, mode, pass, sc, sm, s, launches);
        TokenRec* t = a; a = b; b = t;
    };
    if (by_position) {
        for (int p = 0; p < 8; ++p)
            if ((vary_pos >> (8 * p)) & 0xFF) run(1, p);
    } else {
        const u64 m = range[4];                         // long tokens
        if (m != 0) {
            // inline tokens to the front, long ones behind them (stable): the relative order of the two kinds is
            // settled -- inline before long under equal prefixes -- and the long ones form a sub-array of their own
            if (mixed_long) run(2, 0);
            // order the sub-array by what follows the prefix: LSD over the length, then the 8-byte windows from the
            // last one to the first; the stable passes over k1 / k0 below keep that order inside equal prefixes
            TokenRec* sa = a + (n - m);
            TokenRec* sb = b + (n - m);
            auto fill = [&](int w, u64* r3) {              // keys of window w into pos; r3 (if asked for): longest, OR, AND
                const u64 init2[3] = {0, 0, ~0ull};
                e = cudaMemcpyAsync(sc.tmp + 4, init2, sizeof(init2), cudaMemcpyHostToDevice, s);
                if (e != cudaSuccess) return;
                sort_fill_window_kernel<<<blocks_for(m, 256, sm), 256, 0, s>>>(sa, m, arena, w, sc.tmp);
                *launches += 1;
                if (!r3) return;
                e = cudaMemcpyAsync(r3, sc.tmp + 4, 3 * sizeof(u64), cudaMemcpyDeviceToHost, s);
                if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            };
            auto passes = [&](u64 vary) {
                for (int p = 0; p < 8 && e == cudaSuccess; ++p) {
                    if (!((vary >> (8 * p)) & 0xFF)) continue;
                    e = radix_pass(sa, sb, m, 1, p, sc, sm, s, launches);
                    TokenRec* t = sa; sa = sb; sb = t;
                }
            };
            u64 r3[3] = {0, 0, 0};
            fill(-1, r3);                                   // least significant: the length
            if (e == cudaSuccess) passes(r3[1] ^ r3[2]);
            int windows = 0;
            if (e == cudaSuccess) {
                const u64 longest = r3[0];
                const u64 zero2[2] = {0, 0};
                e = cudaMemcpyAsync(sc.tmp + 4, zero2, sizeof(zero2), cudaMemcpyHostToDevice, s);
                if (e == cudaSuccess) {
                    sort_second_longest_kernel<<<blocks_for(m, 256, sm), 256, 0, s>>>(sa, m, arena, longest, sc.tmp + 4);
                    *launches += 1;
                    u64 r2[2];
                    e = cudaMemcpyAsync(r2, sc.tmp + 4, sizeof(r2), cudaMemcpyDeviceToHost, s);
                    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                    const u64 second = r2[1] >= 2 ? longest : r2[0];     // where two strings can still differ
                    windows = (int)std::min<u64>((second > 16 ? (second - 16 + 7) / 8 : 0), (u64)kLongWindows);
                }
            }
            // the windows from the last one to the first, a batch at a time: which of them vary at all is one launch
            // and one host read per batch (sc.hist is free between passes)
            for (int hi = windows; hi > 0 && e == cudaSuccess; hi -= kWindowBatch) {
                const int lo = hi > kWindowBatch ? hi - kWindowBatch : 0;
                u64 init[2 * kWindowBatch], got[2 * kWindowBatch];
                for (int j = 0; j < kWindowBatch; ++j) { init[2 * j] = 0; init[2 * j + 1] = ~0ull; }
                e = cudaMemcpyAsync(sc.hist, init, sizeof(init), cudaMemcpyHostToDevice, s);
                if (e != cudaSuccess) break;
                sort_window_range_kernel<<<blocks_for(m, 256, sm), 256, 0, s>>>(sa, m, arena, lo, hi - lo, sc.hist);
                *launches += 1;
                e = cudaMemcpyAsync(got, sc.hist, sizeof(got), cudaMemcpyDeviceToHost, s);
                if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                for (int w = hi - 1; w >= lo && e == cudaSuccess; --w) {
                    const u64 vary = got[2 * (w - lo)] ^ got[2 * (w - lo) + 1];
                    if (!vary) continue;
                    fill(w, nullptr);
                    passes(vary);
                }
            }
            if (e == cudaSuccess && sa != a + (n - m))
                e = cudaMemcpyAsync(a + (n - m), sa, sizeof(TokenRec) * m, cudaMemcpyDeviceToDevice, s);
        }
        for (int p = 0; p < 8; ++p)
            if ((vary_k1 >> (8 * p)) & 0xFF) run(0, p);
        for (int p = 0; p < 8; ++p)
            if ((vary_k0 >> (8 * p)) & 0xFF) run(0, 8 + p);
    }
    if (e != cudaSuccess) return e;
    if (a != recs) {
        e = cudaMemcpyAsync(recs, a, sizeof(TokenRec) * n, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return e;
    }
    if (!by_position && range[4] != 0) {
        sort_long_check_kernel<<<blocks_for(n, 256, sm), 256, 0, s>>>(recs, n, arena, sc.tmp + 7);
        sort_long_fixup_kernel<<<blocks_for(n, 256, sm), 256, 0, s>>>(recs, n, arena, sc.tmp + 7);
        *launches += 2;
    }
    return cudaGetLastError();
}

// step 1: head flags + sortedness check (status gets kStatusNotSorted on a descent)
cudaError_t tokens_rle_flags(const TokenRec* recs, u64 n, const uint8_t* arena, u64* flags, int* status, int sm,
                             cudaStream_t s, u64* launches) {
    if (n == 0) return cudaSuccess;
    rle_flags_kernel<<<blocks_for(n, 256, sm), 256, 0, s>>>(recs, n, arena, flags, status);
    *launches += 1;
    return cudaGetLastError();
}

// step 2: flags (from step 1) / run_start: n u64 each; tmp: scan scratch
cudaError_t tokens_rle_insert(const TokenRec* recs, u64 n, const uint8_t* arena, u64* flags, u64* run_start, u64* tmp,
                              const TableView& t, int sm, cudaStream_t s, u64* launches) {
    if (n == 0) return cudaSuccess;
    const unsigned g = blocks_for(n, 256, sm);
    cudaError_t e = exclusive_scan_u64(flags, flags, n, tmp, s, launches);
    if (e != cudaSuccess) return e;
    rle_starts_kernel<<<g, 256, 0, s>>>(flags, recs, n, arena, run_start);
    rle_insert_kernel<<<g, 256, 0, s>>>(recs, n, arena, run_start, flags, t);
    *launches += 2;
    return cudaGetLastError();
}


// ---------------------------------------------------------------------------------
// Compact form of the sort + RLE alternative (reduce_sorted over sort_words, proj/src/text.cpp:59-63,
// proj/src/reduce.cpp:8-21) for COUNTING: a token of at most 8 bytes is its own 64-bit key, so the
// bulk of the tokens is sorted as 8-byte keys instead of 32-byte records (a quarter of the traffic
// per radix pass); the few longer tokens keep the record path above.
// ---------------------------------------------------------------------------------
// tile_counts != nullptr: `in` is the tokenizer's tiled layout (EmitView::keys), tile t holds tile_counts[t] keys
static_assert(kTileItems == (int)kKeyTile, "the tokenizer's key tiles are the sort's tiles");
#ifndef WFCU_DENSE_TILE
#define WFCU_DENSE_TILE 32768
#endif
constexpr u32 kDenseTile = WFCU_DENSE_TILE;   // most keys a warp tile holds once the keys are dense
__global__ void ck_hist_kernel(const u64* __restrict__ in, u64 n, u64 n_tiles, int shift, u64* __restrict__ hist,
                               const u32* __restrict__ tile_counts, u32 tile_items) {
    __shared__ u32 sh[kSortWarps][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u64 tile = (u64)blockIdx.x * kSortWarps + warp;
    for (int d = lane; d < 256; d += 32) sh[warp][d] = 0;
    __syncwarp();
    if (tile < n_tiles) {
        const u64 lo = tile * tile_items;
        const u64 hi = tile_counts ? lo + tile_counts[tile] : min(lo + (u64)tile_items, n);
        for (u64 i = lo + lane; i < hi; i += 32) atomicAdd(&sh[warp][(u32)(in[i] >> shift) & 0xFF], 1u);
    }
    __syncwarp();
    if (tile < n_tiles)
        for (int d = lane; d < 256; d += 32) hist[(u64)d * n_tiles + tile] = sh[warp][d];
}

__global__ void ck_scatter_kernel(const u64* __restrict__ in, u64* __restrict__ out, u64 n, u64 n_tiles, int shift,
                                  const u64* __restrict__ offs, const u32* __restrict__ tile_counts, u32 tile_items) {
    __shared__ u64 sh[kSortWarps][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u64 tile = (u64)blockIdx.x * kSortWarps + warp;
    if (tile >= n_tiles) return;
    for (int d = lane; d < 256; d += 32) sh[warp][d] = offs[(u64)d * n_tiles + tile];
    __syncwarp();
    const u64 lo = tile * tile_items;
    const u64 hi = tile_counts ? lo + tile_counts[tile] : min(lo + (u64)tile_items, n);
    const u32 lt = (1u << lane) - 1u;
    for (u64 base = lo; base < hi; base += 32) {
        const u64 i = base + lane;
        const bool live = i < hi;
        u64 k = 0;
        u32 d = 0xFFFFFFFFu;
        if (live) {
            k = in[i];
            d = (u32)(k >> shift) & 0xFF;
        }
        const u32 peers = __match_any_sync(0xFFFFFFFFu, d);
        u64 dst = 0;
        if (live) dst = sh[warp][d] + __popc(peers & lt);
        __syncwarp();
        if (live && (peers & lt) == 0) sh[warp][d] += __popc(peers);
        __syncwarp();
        if (live) out[dst] = k;
    }
}

__global__ void ck_heads_kernel(const u64* __restrict__ keys, u64 n, u64* __restrict__ flags) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}
__global__ void ck_starts_kernel(const u64* __restrict__ keys, u64 n, const u64* __restrict__ flags_scan, u64* __restrict__ run_start) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        if (i == 0 || keys[i] != keys[i - 1]) run_start[flags_scan[i]] = i;
}
__global__ void ck_insert_kernel(const u64* __restrict__ keys, u64 n, const u64* __restrict__ run_start,
                                 const u64* __restrict__ flags_scan, TableView t) {
    const bool last_is_head = (n == 1) || keys[n - 2] != keys[n - 1];
    const u64 n_runs = flags_scan[n - 1] + (last_is_head ? 1 : 0);
    u64 tokens = 0;
    u32 inserted = 0;
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n_runs; r += (u64)gridDim.x * blockDim.x) {
        const u64 lo = run_start[r];
        const u64 hi = (r + 1 < n_runs) ? run_start[r + 1] : n;
        table_add(t, keys[lo], 0ull, hi - lo, &inserted);
        tokens += hi - lo;
    }
    for (int d = 16; d > 0; d >>= 1) {
        tokens += __shfl_xor_sync(0xFFFFFFFFu, tokens, d);
        inserted += __shfl_xor_sync(0xFFFFFFFFu, inserted, d);
    }
    if ((threadIdx.x & 31) == 0) table_note_inserted(t, inserted);
    if ((threadIdx.x & 31) == 0 && tokens) atomicAdd(t.n_tokens, tokens);
}

// Radix sort of the nk keys on the byte positions that vary, run-length encode, add to the table.
// keys_a / keys_b: nk u64 each; hist: sort_hist_words(nk); tmp: max(scan_tmp_words(hist words), scan_tmp_words(nk));
// flags / run_start: nk u64 each.  tile_counts / tiled_tiles: keys_a is the tokenizer's tiled layout (hist and tmp
// sized for max(tiled_tiles, sort_n_tiles(nk)) tiles), keys_b holds nk keys.
cudaError_t tokens_compact_count(u64* keys_a, u64* keys_b, u64 nk, u64 vary, u64* hist, u64* tmp, u64* flags, u64* run_start,
                                 const TableView& t, int sm, cudaStream_t s, u64* launches, const u32* tile_counts,
                                 u64 tiled_tiles) {
    if (nk == 0) return cudaSuccess;
    u64* a = keys_a;
    u64* b = keys_b;
    // tiled input (straight from the tokenizer): the first pass reads the tiles and writes nk dense keys; if no
    // byte position varies it still runs, on position 0, to make the keys dense
    bool tiled = tile_counts != nullptr;
    if (tiled && !vary) vary = 0xFF;
    for (int p = 0; p < 8; ++p) {
        if (!((vary >> (8 * p)) & 0xFF)) continue;
        // dense passes use larger tiles per warp (fewer histogram rows to scan: 83 -> 97 GB/s at 1 GB), as
        // large as leaves 4096 warps of work
        u32 dense_items = kTileItems;
        while (dense_items < kDenseTile && nk / (2 * dense_items) >= 4096) dense_items *= 2;
        const u32 items = tiled ? (u32)kTileItems : dense_items;
        const u64 n_tiles = tiled ? tiled_tiles : (nk + items - 1) / items;
        const unsigned grid = (unsigned)((n_tiles + kSortWarps - 1) / kSortWarps);
        const u32* tc = tiled ? tile_counts : nullptr;
        ck_hist_kernel<<<grid, kSortWarps * 32, 0, s>>>(a, nk, n_tiles, 8 * p, hist, tc, items);
        *launches += 1;
        cudaError_t e = exclusive_scan_u64(hist, hist, 256 * n_tiles, tmp, s, launches);
        if (e != cudaSuccess) return e;
        ck_scatter_kernel<<<grid, kSortWarps * 32, 0, s>>>(a, b, nk, n_tiles, 8 * p, hist, tc, items);
        *launches += 1;
        u64* x = a; a = b; b = x;
        tiled = false;
    }
    const unsigned g = blocks_for(nk, 256, sm);
    ck_heads_kernel<<<g, 256, 0, s>>>(a, nk, flags);
    *launches += 1;
    cudaError_t e = exclusive_scan_u64(flags, flags, nk, tmp, s, launches);
    if (e != cudaSuccess) return e;
    ck_starts_kernel<<<g, 256, 0, s>>>(a, nk, flags, run_start);
    ck_insert_kernel<<<g, 256, 0, s>>>(a, nk, run_start, flags, t);
    *launches += 2;
    return cudaGetLastError();
}

}  // namespace wfcu
