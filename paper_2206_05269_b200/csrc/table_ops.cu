// table_ops.cu -- kernels that move count-table entries around: export compaction,
// hash partition by owner GPU (the exchange step that replaces the reference's
// range-partition shuffle, /root/reference/proj/src/shuffle.cpp:9-168, see
// SURVEY.md D2), merge-insert of received entries (merge_counts,
// proj/src/reduce.cpp:83-89) and the long-token record stream.
#include "wfcu_dev.cuh"

namespace wfcu {

// Dense list of the non-empty inline slots (order unspecified).
__global__ void tb_compact_kernel(TableView t, Slot* __restrict__ out, u64 out_cap, u64* __restrict__ out_count) {
    const u32 lane = threadIdx.x & 31;                    // one atomic per warp, not per entry
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 <= t.mask; i0 += (u64)gridDim.x * blockDim.x) {
        const u64 i = i0 + lane;
        Slot s{};
        if (i <= t.mask) s = t.slots[i];
        const bool live = s.k0 != 0;
        const u32 m = __ballot_sync(0xFFFFFFFFu, live);
        u64 base = 0;
        if (lane == 0 && m) base = atomicAdd(out_count, (u64)__popc(m));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        const u64 j = base + __popc(m & ((1u << lane) - 1u));
        if (live && j < out_cap) out[j] = Slot{s.k0, s.k1, s.count, 0};
    }
}

// Same, as TokenRec {k0,k1,ext=0,pos=count}: the radix sort of tokens.cu then orders the
// table by key on the device and carries the count along.
__global__ void tb_compact_recs_kernel(TableView t, TokenRec* __restrict__ out, u64 out_cap, u64* __restrict__ out_count) {
    const u32 lane = threadIdx.x & 31;                    // one atomic per warp, not per entry
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 <= t.mask; i0 += (u64)gridDim.x * blockDim.x) {
        const u64 i = i0 + lane;
        Slot s{};
        if (i <= t.mask) s = t.slots[i];
        const bool live = s.k0 != 0;
        const u32 m = __ballot_sync(0xFFFFFFFFu, live);
        u64 base = 0;
        if (lane == 0 && m) base = atomicAdd(out_count, (u64)__popc(m));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        const u64 j = base + __popc(m & ((1u << lane) - 1u));
        if (live && j < out_cap) out[j] = TokenRec{s.k0, s.k1, 0ull, s.count};
    }
}

// recs sorted by pos ascending: *out = first index whose pos >= value (single thread, log n steps)
__global__ void tb_lower_bound_pos_kernel(const TokenRec* __restrict__ recs, u64 n, u64 value, u64* __restrict__ out) {
    if (blockIdx.x || threadIdx.x) return;
    u64 lo = 0, hi = n;
    while (lo < hi) {
        const u64 mid = (lo + hi) / 2;
        if (recs[mid].pos < value) lo = mid + 1; else hi = mid;
    }
    *out = lo;
}

// Export of the ordered table, packed on the device: key length of every record ...
__device__ __forceinline__ u32 key_len_fast(u64 k0, u64 k1) {
    // bytes are packed first-byte-most-significant and zero padded; a key never ends in NUL
    return k1 ? 16u - ((u32)(__ffsll((long long)k1) - 1) >> 3) : 8u - ((u32)(__ffsll((long long)k0) - 1) >> 3);
}
__global__ void tb_export_lens_kernel(const TokenRec* __restrict__ recs, u64 n, u64* __restrict__ lens) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        lens[i] = key_len_fast(recs[i].k0, recs[i].k1);
}
// ... then, with the exclusive scan of the lengths, the key bytes back to back, the lengths and the counts
__global__ void tb_export_pack_kernel(const TokenRec* __restrict__ recs, u64 n, const u64* __restrict__ offs,
                                      uint8_t* __restrict__ bytes, u32* __restrict__ lens32, u64* __restrict__ counts,
                                      u64* __restrict__ total_bytes) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const TokenRec r = recs[i];
        const u32 len = key_len_fast(r.k0, r.k1);
        uint8_t* out = bytes + offs[i];
        for (u32 b = 0; b < len; ++b) out[b] = (uint8_t)((b < 8 ? r.k0 >> (56 - 8 * b) : r.k1 >> (120 - 8 * b)) & 0xFF);
        lens32[i] = len;
        counts[i] = r.pos;
        if (i + 1 == n) *total_bytes = offs[i] + len;
    }
}

// sum of key lengths (inline keys + long records) -> *out_bytes
__global__ void tb_key_bytes_kernel(TableView t, u64* __restrict__ out_bytes) {
    u64 local = 0;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= t.mask; i += stride) {
        const Slot s = t.slots[i];
        if (s.k0 != 0) local += key_len(s.k0, s.k1);
    }
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= t.long_mask; i += stride) {
        const u64 r = t.long_ref[i];
        if (r) local += *reinterpret_cast<const u32*>(t.arena + r);
    }
    for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xFFFFFFFFu, local, d);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(out_bytes, local);
}

// ---- hash partition ---------------------------------------------------------------
// pass 1: part_counts[owner] += 1 for every inline entry
__global__ void tb_partition_count_kernel(TableView t, u32 n_parts, u64* __restrict__ part_counts) {
    extern __shared__ u32 s_hist[];
    for (u32 p = threadIdx.x; p < n_parts; p += blockDim.x) s_hist[p] = 0;
    __syncthreads();
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= t.mask; i += (u64)gridDim.x * blockDim.x) {
        const Slot s = t.slots[i];
        if (s.k0 != 0) atomicAdd(&s_hist[owner_mix32(s.k0, s.k1) % n_parts], 1u);
    }
    __syncthreads();
    for (u32 p = threadIdx.x; p < n_parts; p += blockDim.x)
        if (s_hist[p]) atomicAdd(&part_counts[p], (u64)s_hist[p]);
}
// exclusive scan of the (few) partition sizes -> cursors
__global__ void tb_partition_scan_kernel(const u64* __restrict__ part_counts, u32 n_parts, u64* __restrict__ cursors) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        u64 acc = 0;
        for (u32 p = 0; p < n_parts; ++p) { cursors[p] = acc; acc += part_counts[p]; }
    }
}
// A cursor per partition is a handful of addresses for up to millions of entries: the lanes of a warp that
// go to the same partition take their places with ONE atomic (match_any), not one each.
__device__ __forceinline__ u64 warp_claim(u64* __restrict__ cursors, u32 p, bool live) {
    const u32 lane = threadIdx.x & 31;
    const u32 peers = __match_any_sync(0xFFFFFFFFu, live ? p : 0xFFFFFFFFu);
    const u32 leader = __ffs(peers) - 1;
    u64 base = 0;
    if (live && lane == leader) base = atomicAdd(&cursors[p], (u64)__popc(peers));
    base = __shfl_sync(0xFFFFFFFFu, base, leader);
    return base + __popc(peers & ((1u << lane) - 1u));
}
// pass 2: scatter entries into their partition's region
__global__ void tb_partition_scatter_kernel(TableView t, u32 n_parts, u64* __restrict__ cursors,
                                            Slot* __restrict__ out, u64 out_cap) {
    const u32 lane = threadIdx.x & 31;
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 <= t.mask; i0 += (u64)gridDim.x * blockDim.x) {
        const u64 i = i0 + lane;
        Slot s{};
        if (i <= t.mask) s = t.slots[i];
        const bool live = s.k0 != 0;
        const u32 p = live ? owner_mix32(s.k0, s.k1) % n_parts : 0u;
        const u64 j = warp_claim(cursors, p, live);
        if (live && j < out_cap) out[j] = Slot{s.k0, s.k1, s.count, 0};
    }
}

// One-pass form for the synchronisation-free exchange: partition p owns the fixed region
// out[p * cap, (p+1) * cap); counts[p] = entries written, counts[n_parts] += long tokens in
// the table, counts[n_parts + 1] += entries that did not fit (both sticky flags for the host).
// hdr = 1: the first entry of every region is left free for a header (tb_region_headers_kernel): the region then
// describes itself and the exchange needs no separate all-to-all of the sizes.
__global__ void tb_partition_fixed_kernel(TableView t, u32 n_parts, u64 cap, u32 hdr, Slot* __restrict__ out,
                                          u64* __restrict__ counts) {
    const u32 lane = threadIdx.x & 31;
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 <= t.mask; i0 += (u64)gridDim.x * blockDim.x) {
        const u64 i = i0 + lane;
        Slot s{};
        if (i <= t.mask) s = t.slots[i];
        const bool live = s.k0 != 0;
        const u32 p = live ? owner_mix32(s.k0, s.k1) % n_parts : 0u;
        const u64 j = warp_claim(counts, p, live);
        if (live) {
            if (j + hdr < cap) out[(u64)p * cap + hdr + j] = Slot{s.k0, s.k1, s.count, 0};
            else atomicAdd(&counts[n_parts + 1], 1ull);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && *t.n_long) atomicAdd(&counts[n_parts], *t.n_long);
}
// header of region p: {0, 0, entries that follow, 0}
__global__ void tb_region_headers_kernel(Slot* __restrict__ out, u32 n_parts, u64 cap, const u64* __restrict__ counts) {
    const u32 p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n_parts) out[(u64)p * cap] = Slot{0ull, 0ull, counts[p] < cap - 1 ? counts[p] : cap - 1, 0ull};
}
// counts[key] += count for the first min(region_counts[p], cap) entries of every region
// region_counts == nullptr: the regions carry their own header (first entry, count field)
__global__ void tb_merge_regions_kernel(TableView t, const Slot* __restrict__ in, u32 n_parts, u64 cap,
                                        const u64* __restrict__ region_counts) {
    u64 tokens = 0;
    u32 inserted = 0;
    const u64 total = (u64)n_parts * cap;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (u64)gridDim.x * blockDim.x) {
        const u64 p = i / cap, j = i - p * cap;
        const bool mine = region_counts ? j < region_counts[p] : (j >= 1 && j - 1 < in[p * cap].count);
        if (mine) {
            const Slot s = in[i];
            if (s.k0 != 0 && s.count != 0) {
                table_add(t, s.k0, s.k1, s.count, &inserted);
                tokens += s.count;
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

// counts[key] += count for n received entries; also accounts the tokens
__global__ void tb_merge_entries_kernel(TableView t, const Slot* __restrict__ in, u64 n) {
    u64 tokens = 0;
    u32 inserted = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const Slot s = in[i];
        if (s.k0 != 0 && s.count != 0) {
            table_add(t, s.k0, s.k1, s.count, &inserted);
            tokens += s.count;
        }
    }
    for (int d = 16; d > 0; d >>= 1) {
        tokens += __shfl_xor_sync(0xFFFFFFFFu, tokens, d);
        inserted += __shfl_xor_sync(0xFFFFFFFFu, inserted, d);
    }
    if ((threadIdx.x & 31) == 0) table_note_inserted(t, inserted);
    if ((threadIdx.x & 31) == 0 && tokens) atomicAdd(t.n_tokens, tokens);
}

// dst += src for whole tables (inline part)
__global__ void tb_merge_table_kernel(TableView dst, TableView src) {
    u64 tokens = 0;
    u32 inserted = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= src.mask; i += (u64)gridDim.x * blockDim.x) {
        const Slot s = src.slots[i];
        if (s.k0 != 0 && s.count != 0) {
            table_add(dst, s.k0, s.k1, s.count, &inserted);
            tokens += s.count;
        }
    }
    for (int d = 16; d > 0; d >>= 1) {
        tokens += __shfl_xor_sync(0xFFFFFFFFu, tokens, d);
        inserted += __shfl_xor_sync(0xFFFFFFFFu, inserted, d);
    }
    if ((threadIdx.x & 31) == 0) table_note_inserted(dst, inserted);
    if ((threadIdx.x & 31) == 0 && tokens) atomicAdd(dst.n_tokens, tokens);
}

// ---- long-token record stream -----------------------------------------------------
// record: {u64 count, u32 len, u32 hash, bytes..., pad to 8}
__device__ __forceinline__ u64 long_record_bytes(u32 len) { return 16 + ((u64(len) + 7) & ~7ull); }

// Serialises the long table.  out == nullptr: only sizes (*out_bytes).
__global__ void tb_long_serialize_kernel(TableView t, uint8_t* __restrict__ out, u64 out_cap, u64* __restrict__ out_bytes) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= t.long_mask; i += (u64)gridDim.x * blockDim.x) {
        const u64 r = t.long_ref[i];
        if (!r) continue;
        const u32 len = *reinterpret_cast<const u32*>(t.arena + r);
        const u64 need = long_record_bytes(len);
        const u64 off = atomicAdd(out_bytes, need);
        if (out && off + need <= out_cap) {
            *reinterpret_cast<u64*>(out + off) = t.long_count[i];
            *reinterpret_cast<u32*>(out + off + 8) = len;
            *reinterpret_cast<u32*>(out + off + 12) = *reinterpret_cast<const u32*>(t.arena + r + 4);
            for (u32 k = 0; k < len; ++k) out[off + 16 + k] = t.arena[r + 8 + k];
            for (u64 k = 16 + len; k < need; ++k) out[off + k] = 0;
        }
    }
}

// Walks a record stream (single thread per CTA-strided record is impossible
// without an index, so one thread walks; long tokens are rare) and inserts the
// records owned by `part`.
__global__ void tb_long_merge_kernel(TableView t, const uint8_t* __restrict__ recs, u64 n_bytes, u32 part, u32 n_parts) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    u64 off = 0;
    while (off + 16 <= n_bytes) {
        const u64 count = *reinterpret_cast<const u64*>(recs + off);
        const u32 len = *reinterpret_cast<const u32*>(recs + off + 8);
        const u32 hash = *reinterpret_cast<const u32*>(recs + off + 12);
        const u64 need = long_record_bytes(len);
        if (off + need > n_bytes) break;
        const bool mine = (n_parts <= 1) || ((hash * 0x9E3779B1u) >> 7) % n_parts == part;
        // a token the table already holds only adds its count: no arena record is spent on it (repeated merges used
        // to leak one record per incoming token until ARENA_FULL)
        bool known = false;
        if (mine && count) {
            u64 i = hash & t.long_mask;
            const u64 limit = t.long_mask < kMaxProbes ? t.long_mask : kMaxProbes;      // long_add's bound
            for (u64 probes = 0; probes <= limit; ++probes) {
                const u64 r = *reinterpret_cast<volatile u64*>(t.long_ref + i);
                if (r == 0) break;
                if (*reinterpret_cast<const u32*>(t.arena + r) == len && *reinterpret_cast<const u32*>(t.arena + r + 4) == hash) {
                    bool same = true;
                    for (u32 k = 0; k < len && same; ++k) same = t.arena[r + 8 + k] == recs[off + 16 + k];
                    if (same) {
                        atomicAdd(t.long_count + i, count);
                        atomicAdd(t.n_tokens, count);
                        known = true;
                        break;
                    }
                }
                i = (i + 1) & t.long_mask;
            }
        }
        if (mine && count && !known) {
            const u64 rec = arena_alloc(t, len);
            if (rec) {
                *reinterpret_cast<u32*>(t.arena + rec) = len;
                *reinterpret_cast<u32*>(t.arena + rec + 4) = hash;
                for (u32 k = 0; k < len; ++k) t.arena[rec + 8 + k] = recs[off + 16 + k];
                __threadfence();
                long_add(t, rec, count);
                atomicAdd(t.n_tokens, count);
            }
        }
        off += need;
    }
}


// ---- distinctive_words on the device (proj/src/analysis.cpp:77-132) ---------------------------------------
// counts[key] of the table, 0 if the key is absent (read only: the table is not being written)
__device__ __forceinline__ bool table_find(const TableView& t, u64 k0, u64 k1, u64* count) {
    u64 i = mix32(k0, k1) & t.mask;
    const u64 limit = t.mask < kMaxProbes ? t.mask : kMaxProbes;      // table_add never places a key further from home
    for (u64 probes = 0; probes <= limit; ++probes) {
        const Slot s = t.slots[i];
        if (s.k0 == 0) return false;
        if (s.k0 == k0 && s.k1 == k1) { *count = s.count; return true; }
        i = (i + 1) & t.mask;
    }
    return false;
}
// Union of two tables as dense rows: every word of `a` (with its count in `b`), and -- second launch, swapped,
// only_missing -- every word of `b` that `a` does not hold.  recs[i] = {k0,k1,ext=i,pos=0}, ca[i] / cb[i] = the two
// counts; cursor[0] = rows written, cursor[1] += words found in both tables (first launch only).
__global__ void tb_union_rows_kernel(TableView a, TableView b, bool only_missing, TokenRec* __restrict__ recs,
                                     u64* __restrict__ ca, u64* __restrict__ cb, u64 cap, u64* __restrict__ cursor) {
    const u32 lane = threadIdx.x & 31;
    u32 both = 0;
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x - lane; i0 <= a.mask; i0 += (u64)gridDim.x * blockDim.x) {
        const u64 i = i0 + lane;
        Slot s{};
        if (i <= a.mask) s = a.slots[i];
        bool live = s.k0 != 0;
        u64 other = 0;
        if (live) {
            const bool found = table_find(b, s.k0, s.k1, &other);
            if (found && !only_missing) ++both;
            if (found && only_missing) live = false;
        }
        const u32 m = __ballot_sync(0xFFFFFFFFu, live);
        u64 base = 0;
        if (lane == 0 && m) base = atomicAdd(cursor, (u64)__popc(m));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        const u64 j = base + __popc(m & ((1u << lane) - 1u));
        if (live && j < cap) {
            recs[j] = TokenRec{s.k0, s.k1, j, 0ull};
            ca[j] = only_missing ? 0ull : s.count;
            cb[j] = only_missing ? s.count : other;
        }
    }
    for (int d = 16; d > 0; d >>= 1) both += __shfl_xor_sync(0xFFFFFFFFu, both, d);
    if (lane == 0 && both) atomicAdd(cursor + 1, (u64)both);
}
// ascending order of the key = ascending order of the double
__device__ __forceinline__ u64 double_sort_key(double v) {
    const u64 b = (u64)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
// recs[i].pos = sort key of the score  log((ct+1)/(Tt+V)) - log((co+1)/(To+V)),  V = rows + extra_vocab.  The device's
// log is within a few ulp of the host's: the caller only uses these scores to find which rows CAN make the cut
// (with a margin), the reported scores are computed on the host with the reference's expression.
__global__ void tb_score_rows_kernel(TokenRec* __restrict__ recs, const u64* __restrict__ ct, const u64* __restrict__ co,
                                     const u64* __restrict__ n_rows, u64 extra_vocab, u64 t_total, u64 o_total) {
    const u64 n = *n_rows;
    const double v = (double)(n + extra_vocab);
    const double t_den = (double)t_total + v, o_den = (double)o_total + v;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const double sc = log(((double)ct[i] + 1.0) / t_den) - log(((double)co[i] + 1.0) / o_den);
        recs[i].pos = double_sort_key(sc);
    }
}
// the two counts of the candidate rows recs[first, n), in that order
__global__ void tb_gather_counts_kernel(const TokenRec* __restrict__ recs, u64 first, u64 n, const u64* __restrict__ ct,
                                        const u64* __restrict__ co, u64* __restrict__ out_ct, u64* __restrict__ out_co) {
    for (u64 i = first + (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        out_ct[i - first] = ct[recs[i].ext];
        out_co[i - first] = co[recs[i].ext];
    }
}

// records moved into a list whose arena holds the source arena `delta` bytes further on
__global__ void tk_rebase_ext_kernel(TokenRec* __restrict__ recs, u64 n, u64 delta) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        if (recs[i].ext) recs[i].ext += delta;
}

// Reset of everything but the inline table: the long-token table is only cleared when it holds something (the
// common corpus has no token longer than 16 bytes: two 8 MB memsets per reset for nothing), then the counters.
// The grid cooperates on the clear; the last CTA to finish resets the counters (they hold n_long, which every CTA
// has to read first).
__global__ void tb_reset_aux_kernel(TableView t, u64* __restrict__ counters, unsigned int* __restrict__ done) {
    __shared__ bool last;
    if (*t.n_long != 0) {
        for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= t.long_mask; i += (u64)gridDim.x * blockDim.x) {
            t.long_ref[i] = 0;
            t.long_count[i] = 0;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) + 1 == gridDim.x;
    __syncthreads();
    if (last && threadIdx.x < 16) {
        counters[threadIdx.x] = threadIdx.x == 4 ? 8ull : 0ull;     // [4] arena_used: offset 0 means "empty"
        if (threadIdx.x == 0) *done = 0;
    }
}

// ---- launchers ----------------------------------------------------------------------
static inline unsigned grid_for(u64 items, int sm_count) {
    u64 g = (items + 255) / 256;
    const u64 cap = (u64)sm_count * 8;
    if (g > cap) g = cap;
    if (g == 0) g = 1;
    return (unsigned)g;
}

cudaError_t tb_compact(const TableView& t, Slot* out, u64 cap, u64* dev_count, int sm, cudaStream_t s, u64* launches) {
    cudaError_t e = cudaMemsetAsync(dev_count, 0, sizeof(u64), s);
    if (e != cudaSuccess) return e;
    tb_compact_kernel<<<grid_for(t.mask + 1, sm), 256, 0, s>>>(t, out, cap, dev_count);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t tb_compact_recs(const TableView& t, TokenRec* out, u64 cap, u64* dev_count, int sm, cudaStream_t s, u64* launches) {
    cudaError_t e = cudaMemsetAsync(dev_count, 0, sizeof(u64), s);
    if (e != cudaSuccess) return e;
    tb_compact_recs_kernel<<<grid_for(t.mask + 1, sm), 256, 0, s>>>(t, out, cap, dev_count);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t exclusive_scan_u64(const u64* in, u64* out, u64 n, u64* tmp, cudaStream_t s, u64* launches);   // tokens.cu

// recs (ordered) -> packed key bytes, lengths, counts; lens64 is scratch of n u64, tmp of scan_tmp_words(n)
cudaError_t tb_export_pack(const TokenRec* recs, u64 n, u64* lens64, u64* tmp, uint8_t* bytes, u32* lens32, u64* counts,
                           u64* dev_total_bytes, int sm, cudaStream_t s, u64* launches) {
    if (n == 0) return cudaMemsetAsync(dev_total_bytes, 0, sizeof(u64), s);
    tb_export_lens_kernel<<<grid_for(n, sm), 256, 0, s>>>(recs, n, lens64);
    *launches += 1;
    cudaError_t e = exclusive_scan_u64(lens64, lens64, n, tmp, s, launches);
    if (e != cudaSuccess) return e;
    tb_export_pack_kernel<<<grid_for(n, sm), 256, 0, s>>>(recs, n, lens64, bytes, lens32, counts, dev_total_bytes);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t tb_lower_bound_pos(const TokenRec* recs, u64 n, u64 value, u64* dev_out, cudaStream_t s, u64* launches) {
    tb_lower_bound_pos_kernel<<<1, 1, 0, s>>>(recs, n, value, dev_out);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t tb_key_bytes(const TableView& t, u64* dev_bytes, int sm, cudaStream_t s, u64* launches) {
    cudaError_t e = cudaMemsetAsync(dev_bytes, 0, sizeof(u64), s);
    if (e != cudaSuccess) return e;
    tb_key_bytes_kernel<<<grid_for(t.mask + 1, sm), 256, 0, s>>>(t, dev_bytes);
    *launches += 1;
    return cudaGetLastError();
}

// cursors: device scratch of n_parts u64
cudaError_t tb_partition(const TableView& t, u32 n_parts, Slot* out, u64 cap, u64* dev_part_counts, u64* cursors,
                         int sm, cudaStream_t s, u64* launches) {
    cudaError_t e = cudaMemsetAsync(dev_part_counts, 0, sizeof(u64) * n_parts, s);
    if (e != cudaSuccess) return e;
    const unsigned g = grid_for(t.mask + 1, sm);
    tb_partition_count_kernel<<<g, 256, n_parts * sizeof(u32), s>>>(t, n_parts, dev_part_counts);
    tb_partition_scan_kernel<<<1, 32, 0, s>>>(dev_part_counts, n_parts, cursors);
    tb_partition_scatter_kernel<<<g, 256, 0, s>>>(t, n_parts, cursors, out, cap);
    *launches += 3;
    return cudaGetLastError();
}

cudaError_t tb_partition_fixed(const TableView& t, u32 n_parts, u64 cap, bool framed, Slot* out, u64* dev_counts, int sm,
                               cudaStream_t s, u64* launches) {
    cudaError_t e = cudaMemsetAsync(dev_counts, 0, sizeof(u64) * n_parts, s);   // the two flags stay sticky
    if (e != cudaSuccess) return e;
    tb_partition_fixed_kernel<<<grid_for(t.mask + 1, sm), 256, 0, s>>>(t, n_parts, cap, framed ? 1u : 0u, out, dev_counts);
    *launches += 1;
    if (framed) {
        tb_region_headers_kernel<<<(n_parts + 127) / 128, 128, 0, s>>>(out, n_parts, cap, dev_counts);
        *launches += 1;
    }
    return cudaGetLastError();
}

cudaError_t tb_merge_regions(const TableView& t, const Slot* in, u32 n_parts, u64 cap, const u64* region_counts, int sm,
                             cudaStream_t s, u64* launches) {
    if (n_parts == 0 || cap == 0) return cudaSuccess;
    tb_merge_regions_kernel<<<grid_for((u64)n_parts * cap, sm), 256, 0, s>>>(t, in, n_parts, cap, region_counts);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t tb_merge_entries(const TableView& t, const Slot* in, u64 n, int sm, cudaStream_t s, u64* launches) {
    if (n == 0) return cudaSuccess;
    tb_merge_entries_kernel<<<grid_for(n, sm), 256, 0, s>>>(t, in, n);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t tb_merge_table(const TableView& dst, const TableView& src, int sm, cudaStream_t s, u64* launches) {
    tb_merge_table_kernel<<<grid_for(src.mask + 1, sm), 256, 0, s>>>(dst, src);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t tb_long_serialize(const TableView& t, uint8_t* out, u64 cap, u64* dev_bytes, int sm, cudaStream_t s,
                              u64* launches) {
    cudaError_t e = cudaMemsetAsync(dev_bytes, 0, sizeof(u64), s);
    if (e != cudaSuccess) return e;
    tb_long_serialize_kernel<<<grid_for(t.long_mask + 1, sm), 256, 0, s>>>(t, out, cap, dev_bytes);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t tb_long_merge(const TableView& t, const uint8_t* recs, u64 n_bytes, u32 part, u32 n_parts, cudaStream_t s,
                          u64* launches) {
    if (n_bytes == 0) return cudaSuccess;
    tb_long_merge_kernel<<<1, 32, 0, s>>>(t, recs, n_bytes, part, n_parts);
    *launches += 1;
    return cudaGetLastError();
}

// rows of the union of target and others; dev_cursor[0] = rows, dev_cursor[1] = words in both
cudaError_t tb_union_rows(const TableView& target, const TableView& others, TokenRec* recs, u64* ct, u64* co, u64 cap,
                          u64* dev_cursor, int sm, cudaStream_t s, u64* launches) {
    cudaError_t e = cudaMemsetAsync(dev_cursor, 0, 2 * sizeof(u64), s);
    if (e != cudaSuccess) return e;
    tb_union_rows_kernel<<<grid_for(target.mask + 1, sm), 256, 0, s>>>(target, others, false, recs, ct, co, cap, dev_cursor);
    // words only the others hold: written as (a = others, b = target), so the count lands in cb = `co`
    tb_union_rows_kernel<<<grid_for(others.mask + 1, sm), 256, 0, s>>>(others, target, true, recs, ct, co, cap, dev_cursor);
    *launches += 2;
    return cudaGetLastError();
}
cudaError_t tb_score_rows(TokenRec* recs, const u64* ct, const u64* co, const u64* dev_n_rows, u64 max_rows, u64 extra_vocab,
                          u64 t_total, u64 o_total, int sm, cudaStream_t s, u64* launches) {
    tb_score_rows_kernel<<<grid_for(max_rows, sm), 256, 0, s>>>(recs, ct, co, dev_n_rows, extra_vocab, t_total, o_total);
    *launches += 1;
    return cudaGetLastError();
}
cudaError_t tb_gather_counts(const TokenRec* recs, u64 first, u64 n, const u64* ct, const u64* co, u64* out_ct, u64* out_co,
                             int sm, cudaStream_t s, u64* launches) {
    if (first >= n) return cudaSuccess;
    tb_gather_counts_kernel<<<grid_for(n - first, sm), 256, 0, s>>>(recs, first, n, ct, co, out_ct, out_co);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t tk_rebase_ext(TokenRec* recs, u64 n, u64 delta, int sm, cudaStream_t s, u64* launches) {
    if (n == 0 || delta == 0) return cudaSuccess;
    tk_rebase_ext_kernel<<<grid_for(n, sm), 256, 0, s>>>(recs, n, delta);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t tb_reset_aux(const TableView& t, u64* counters, unsigned int* done, int sm, cudaStream_t s, u64* launches) {
    tb_reset_aux_kernel<<<sm, 256, 0, s>>>(t, counters, done);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace wfcu
