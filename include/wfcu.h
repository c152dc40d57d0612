/*
 * include/wfcu.h -- C ABI of libwfcu.so, the B200 (sm_100a) implementation of the
 * MapReduce word-frequency hot path of arXiv 2206.05269.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch types.
 * The reference's C++ API (/root/reference/proj/include/wfc/*.hpp) is re-implemented
 * on top of these entry points by paper_2206_05269_b200/host (libwfc_b200.so), and
 * INTEGRATION.md shows the binding a reference maintainer would add.  Each entry
 * point names the reference interface it replaces (paths relative to
 * /root/reference/).
 *
 * Conventions
 *   - every function returns WFCU_OK (0) or a negative WFCU_ERR_* code and never
 *     throws; wfcu_last_error() returns the thread-local message of the last
 *     failure (reference: exceptions, proj/include/wfc/pipeline.hpp:33-41).
 *   - there is NO CPU fallback: without a usable CUDA device every compute entry
 *     point returns WFCU_ERR_NO_DEVICE.
 *   - "host" pointers are ordinary host memory owned by the caller and borrowed
 *     for the duration of the call (reference: std::span / const& arguments);
 *     "dev" pointers are device addresses in the current CUDA context (a
 *     torch.Tensor.data_ptr() works), 16-byte aligned.
 *   - `stream` is a cudaStream_t passed as void* (NULL = default stream).
 *   - token keys are exported as packed byte strings in unsigned byte-wise
 *     lexicographic order = std::map<std::string,...> iteration order
 *     (proj/include/wfc/reduce.hpp:15).
 */
#ifndef WFCU_H
#define WFCU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WFCU_API __attribute__((visibility("default")))

#define WFCU_OK 0
#define WFCU_ERR_INVALID_ARGUMENT (-1) /* reference: std::invalid_argument                     */
#define WFCU_ERR_CUDA (-2)             /* CUDA runtime failure; shim rethrows PipelineError     */
#define WFCU_ERR_NO_DEVICE (-3)        /* no sm_100 device / driver: the product has no CPU path */
#define WFCU_ERR_TABLE_FULL (-4)       /* device count table over its load limit                 */
#define WFCU_ERR_DEFERRED_FULL (-5)    /* slow-path fragment list over capacity                  */
#define WFCU_ERR_ARENA_FULL (-6)       /* long-token arena / long table over capacity            */
#define WFCU_ERR_BUFFER_TOO_SMALL (-7) /* caller-provided output buffer too small                */
#define WFCU_ERR_NOT_SORTED (-8)       /* reduce_sorted on an unsorted list (std::invalid_argument) */
#define WFCU_ERR_FRAME_MAGIC (-9)      /* WCX1 frame: WireError::Kind::BadMagic (proj/include/wfc/wire.hpp:26-31) */
#define WFCU_ERR_FRAME_TRUNCATED (-10) /*             WireError::Kind::Truncated                                   */
#define WFCU_ERR_FRAME_TRAILING (-11)  /*             WireError::Kind::TrailingBytes                               */
#define WFCU_ERR_FRAME_ENCODING (-12)  /*             WireError::Kind::BadEncoding                                 */

/* MapKind, proj/include/wfc/engine.hpp:12-16; the first three values are the
 * reference's, `square` is appended for BASELINE.json config 2 (f(x)=x^2). */
#define WFCU_MAP_IDENTITY 0
#define WFCU_MAP_SQUARE_ROOT 1
#define WFCU_MAP_ALTERNATING_HARMONIC_TERM 2
#define WFCU_MAP_SQUARE 3

#define WFCU_DTYPE_F32 0
#define WFCU_DTYPE_F64 1

WFCU_API const char* wfcu_last_error(void);
WFCU_API const char* wfcu_version(void);

/* Number of usable CUDA devices (0 when there is none), and selection of the
 * device the calling thread works on.  One process per GPU is the intended
 * deployment (bench.py / torchrun); the library keeps per-device workspaces. */
WFCU_API int wfcu_device_count(void);
WFCU_API int wfcu_set_device(int device);
/* 148 on B200; grids are sized in multiples of this. */
WFCU_API int wfcu_sm_count(int* out);

/* Plain device-memory helpers, so that a host which does not link the CUDA runtime
 * (the C++ drop-in, a cgo/JNI binding) can stage the buffers the *_dev calls take. */
WFCU_API int wfcu_dev_alloc(void** out, uint64_t bytes);
WFCU_API void wfcu_dev_free(void* p);
WFCU_API int wfcu_dev_upload(void* dev_dst, const void* host_src, uint64_t bytes);
WFCU_API int wfcu_dev_download(void* host_dst, const void* dev_src, uint64_t bytes);

/* ------------------------------------------------------------------------- */
/* Generic map-then-reduce engine  (proj/include/wfc/engine.hpp:25-36,        */
/* proj/src/engine.cpp:15-98)                                                 */
/* ------------------------------------------------------------------------- */

/* sum_i map(values[i]) over device-resident values; positions are 1-based and
 * start at position_base+1 (so a rank holding a slice passes its slice offset).
 * Grid-stride, 16-byte vector loads, fp64 accumulation, warp-shuffle tree and a
 * fixed-order final pass: the result is bitwise reproducible run to run and
 * within 1e-5 relative (in practice ~1e-15) of map_reduce_serial
 * (proj/src/engine.cpp:82-86).  values may be NULL for
 * WFCU_MAP_ALTERNATING_HARMONIC_TERM.  *out is a HOST double; the call
 * synchronises the stream. */
WFCU_API int wfcu_map_reduce_dev(const void* dev_values, int dtype, uint64_t n, uint64_t position_base,
                        int map_kind, void* stream, double* out);

/* Same, but leaves the result in a device double (no host sync) -- what bench.py
 * times for the resident-data number and what precedes the allreduce.
 * The map-reduce entry points are NOT re-entrant per device: the per-CTA partials (and, for the synchronous forms,
 * the result word) live in one buffer per device, so at most one reduction per device may be in flight -- calls on
 * one stream, or calls separated by a synchronisation, are fine; two streams or two host threads are not. */
WFCU_API int wfcu_map_reduce_dev_async(const void* dev_values, int dtype, uint64_t n, uint64_t position_base,
                              int map_kind, void* stream, double* dev_out);

/* The reference's blocked engine, reproduced BIT FOR BIT on the device:
 * ceil(n/block_size) left-to-right block folds (fold_range, engine.cpp:15-20)
 * combined by the fixed pairwise tree (combine_tree, engine.cpp:23-34).  Equals
 * map_reduce_blocked(values, map, {block_size, any workers}) exactly
 * (proj/src/engine.cpp:88-92); block_size == 0 -> WFCU_ERR_INVALID_ARGUMENT
 * (engine.cpp:38-40). */
WFCU_API int wfcu_map_reduce_blocked_dev(const void* dev_values, int dtype, uint64_t n, uint64_t position_base,
                                int map_kind, uint64_t block_size, void* stream, double* out);

/* Host-buffer forms: what wfc::map_reduce_serial / map_reduce_blocked /
 * alternating_harmonic call (H2D copy inside). */
WFCU_API int wfcu_map_reduce_host(const void* host_values, int dtype, uint64_t n, int map_kind, double* out);
WFCU_API int wfcu_map_reduce_blocked_host(const void* host_values, int dtype, uint64_t n, int map_kind,
                                 uint64_t block_size, double* out);
WFCU_API int wfcu_alternating_harmonic(uint64_t n, uint64_t block_size, double* out);

/* ------------------------------------------------------------------------- */
/* Tokenizer + counting map  (proj/src/text.cpp:9-57, proj/src/unicode.cpp,   */
/* proj/src/pipeline.cpp:131-139  ++counts[word])                             */
/* ------------------------------------------------------------------------- */

typedef struct wfcu_counter wfcu_counter; /* device-resident word -> count table */

typedef struct wfcu_counter_config {
    uint64_t table_slots;    /* open-addressing slots (rounded up to 2^k); 0 = default 2^22   */
    uint64_t deferred_slots; /* capacity of the slow-path fragment list; 0 = default 2^22     */
    uint64_t arena_bytes;    /* arena for tokens longer than 16 bytes; 0 = default 64 MiB     */
    uint64_t long_slots;     /* slots of the long-token table; 0 = default 2^20               */
} wfcu_counter_config;

WFCU_API int wfcu_counter_create(wfcu_counter** out, const wfcu_counter_config* cfg /* NULL = defaults */);
WFCU_API void wfcu_counter_destroy(wfcu_counter* c);
/* Empties the table (async on stream). */
WFCU_API int wfcu_counter_reset(wfcu_counter* c, void* stream);

/* Tokenizes dev_text[0..n) exactly like wfc::tokenize (whitespace split, case
 * fold, edge trim, UTF-8 rules of proj/src/unicode.cpp) and adds every token to
 * the table.  The buffer is treated as one document; concatenate documents with
 * an ASCII whitespace byte between them (document ends are fragment ends,
 * proj/src/text.cpp:55).  Asynchronous on `stream`; capacity overflows are
 * reported by wfcu_counter_status / the export calls. */
WFCU_API int wfcu_counter_count_dev(wfcu_counter* c, const uint8_t* dev_text, uint64_t n, void* stream);

/* Host-buffer form (what wfc::serial_wordcount / run_wordcount call): packs the
 * documents with '\n' separators into pinned staging memory, copies them to the
 * device in chunks overlapped with counting, and waits for completion.  Documents
 * that lie back to back in page-locked memory and end in ASCII whitespace are not
 * packed: the copy engine streams them from the caller's buffer at PCIe speed. */
WFCU_API int wfcu_counter_count_host(wfcu_counter* c, const uint8_t* const* docs, const uint64_t* doc_lens,
                            uint64_t n_docs);

/* Measurement hook: with timing enabled every wfcu_counter_count_dev brackets its
 * dominant kernel (wc_count_kernel) with CUDA events on the launching stream;
 * take_kernel_ms waits for them and returns the summed device time and the
 * number of launches since the last call. */
WFCU_API int wfcu_counter_set_timing(wfcu_counter* c, int enabled);
WFCU_API int wfcu_counter_take_kernel_ms(wfcu_counter* c, double* sum_ms, uint64_t* launches);

/* Synchronises and reports overflow conditions (WFCU_ERR_TABLE_FULL, ...). */
WFCU_API int wfcu_counter_status(wfcu_counter* c, void* stream);

/* Distinct tokens, total tokens and total key bytes currently in the table. */
WFCU_API int wfcu_counter_stats(wfcu_counter* c, void* stream, uint64_t* distinct, uint64_t* total_tokens,
                       uint64_t* key_bytes);

/* Exports the table in std::map order: key_bytes (>= key_bytes from stats),
 * key_lens[distinct], counts[distinct].  Capacities are in elements/bytes. */
WFCU_API int wfcu_counter_export(wfcu_counter* c, void* stream, uint8_t* key_bytes, uint64_t key_bytes_cap,
                        uint32_t* key_lens, uint64_t* counts, uint64_t entries_cap);

/* top_k (proj/src/analysis.cpp:58-75) without exporting the table: rows by count
 * descending, ties by word ascending, at most k; rel_freq = count / total words of the
 * WHOLE table.  The table is ordered by count on the device and only rows that can make
 * the cut are downloaded.  key_bytes_cap >= 16 * k covers tables without long tokens. */
WFCU_API int wfcu_counter_top_k(wfcu_counter* c, uint64_t k, void* stream, uint8_t* key_bytes, uint64_t key_bytes_cap,
                                uint32_t* key_lens, uint64_t* counts, double* rel_freq, uint64_t rows_cap,
                                uint64_t* n_rows, uint64_t* total_words);

/* distinctive_words (proj/src/analysis.cpp:77-132; the per-speaker report of cli.cpp:213-221) on two device-resident
 * tables, without exporting either: score = log((c_t+1)/(T_t+V)) - log((c_o+1)/(T_o+V)), V = size of the union
 * vocabulary, rows by score descending (exact double compare), ties by word ascending, at most k.  The tables are
 * joined and scored on the device; only the rows that can make the cut are downloaded and ranked with the
 * reference's expression in host doubles, so words and scores are bit-identical to the reference's.  Both
 * counters must live on the same device.  key_bytes_cap >= 16 * k covers tables without long tokens. */
WFCU_API int wfcu_counter_distinctive(wfcu_counter* target, wfcu_counter* others, uint64_t k, void* stream,
                                      uint8_t* key_bytes, uint64_t key_bytes_cap, uint32_t* key_lens, double* scores,
                                      uint64_t rows_cap, uint64_t* n_rows);

/* dst[word] += src[word]  (merge_counts, proj/src/reduce.cpp:83-89), on device. */
WFCU_API int wfcu_counter_merge(wfcu_counter* dst, const wfcu_counter* src, void* stream);

/* Adds explicit (word, count) pairs -- the inverse of export; used to rebuild a
 * table from a CountMap. */
WFCU_API int wfcu_counter_add_words(wfcu_counter* c, const uint8_t* key_bytes, const uint32_t* key_lens,
                           const uint64_t* counts, uint64_t n_words);

/* ------------------------------------------------------------------------- */
/* Hash-partitioned exchange (replaces the range-partition shuffle,           */
/* proj/src/shuffle.cpp:9-168, as BASELINE.json asks)           */
/* ------------------------------------------------------------------------- */

/* Fixed-width wire entry of the all-to-all: 32 bytes.  Keys of at most 16
 * bytes travel inline (big-endian packed, zero padded); longer tokens travel
 * in a separate byte stream (wfcu_counter_long_records). */
typedef struct wfcu_entry {
    uint64_t k0, k1; /* token bytes 0..7 / 8..15, first byte most significant */
    uint64_t count;
    uint64_t aux;    /* reserved (0) */
} wfcu_entry;

/* owner(word) in [0, n_parts): the partition function of the exchange. */
WFCU_API uint32_t wfcu_owner_of(const uint8_t* word, uint32_t len, uint32_t n_parts);

/* Groups the table's inline entries by owner: dev_entries receives them
 * partition by partition, dev_part_counts (device uint64, n_parts + 1 slots) the size
 * of each partition and, in the last slot, the byte length of the long-token record
 * stream.  entries_cap >= distinct (wfcu_counter_max_entries is always enough).
 * Asynchronous: nothing here synchronises the stream. */
WFCU_API int wfcu_counter_partition(wfcu_counter* c, uint32_t n_parts, wfcu_entry* dev_entries,
                           uint64_t entries_cap, uint64_t* dev_part_counts, void* stream);

/* Upper bound of the number of inline entries the table can hold (its load limit). */
WFCU_API uint64_t wfcu_counter_max_entries(const wfcu_counter* c);

/* Synchronisation-free form of the same exchange step (replaces, like wfcu_counter_partition,
 * plan_partition + encode_outgoing of proj/src/shuffle.cpp:9-66): partition p owns the fixed
 * region dev_entries[p * cap_per_part, (p+1) * cap_per_part), so the all-to-all needs no sizes
 * from the host.  dev_counts has n_parts + 2 words: [p] = entries of partition p (reset by the
 * call); [n_parts] += long tokens in the table and [n_parts + 1] += entries that did not fit --
 * sticky flags the caller reads once, after any number of steps.  Asynchronous on `stream`. */
WFCU_API int wfcu_counter_partition_fixed(wfcu_counter* c, uint32_t n_parts, wfcu_entry* dev_entries,
                                 uint64_t cap_per_part, uint64_t* dev_counts, void* stream);
/* Same, self-describing: entry 0 of every region is a header {0, 0, entries that follow, 0} and at most
 * cap_per_part - 1 entries follow, so ONE all-to-all of the regions is the whole exchange (the n x 8-byte all-to-all
 * of the sizes was pure latency).  dev_counts as above.  Asynchronous on `stream`. */
WFCU_API int wfcu_counter_partition_framed(wfcu_counter* c, uint32_t n_parts, wfcu_entry* dev_entries,
                                  uint64_t cap_per_part, uint64_t* dev_counts, void* stream);
/* The receiving side (replaces merge_sorted + reduce_sorted + merge_counts, proj/src/shuffle.cpp:75-96,
 * proj/src/reduce.cpp:8-21,83-89): adds the first min(dev_region_counts[p], cap_per_part) entries of
 * every region; the counts are read on the device.  dev_region_counts == NULL: the regions are framed
 * (wfcu_counter_partition_framed) and carry their own counts.  Asynchronous on `stream`. */
WFCU_API int wfcu_counter_merge_regions(wfcu_counter* c, const wfcu_entry* dev_entries, uint32_t n_parts,
                               uint64_t cap_per_part, const uint64_t* dev_region_counts, void* stream);

/* Inserts n received entries (summing counts of equal keys). Asynchronous. */
WFCU_API int wfcu_counter_merge_entries(wfcu_counter* c, const wfcu_entry* dev_entries, uint64_t n, void* stream);

/* Long tokens (> 16 bytes) as a self-describing device byte stream of records
 * {u64 count, u32 len, u32 hash, bytes..., pad to 8}.  *n_bytes (host) gets the
 * stream length; dev_out may be NULL to query the size. */
WFCU_API int wfcu_counter_long_records(wfcu_counter* c, uint8_t* dev_out, uint64_t out_cap, uint64_t* n_bytes,
                              void* stream);
/* Inserts the records of a stream whose owner (wfcu_owner_of) is `part` of
 * n_parts (n_parts == 1 keeps everything). */
WFCU_API int wfcu_counter_merge_long_records(wfcu_counter* c, const uint8_t* dev_records, uint64_t n_bytes,
                                    uint32_t part, uint32_t n_parts, void* stream);

/* ------------------------------------------------------------------------- */
/* Tokenizer as a stand-alone stage and the sort + run-length-encode reduce   */
/* (proj/src/text.cpp:32-63, proj/src/reduce.cpp:8-21)                        */
/* ------------------------------------------------------------------------- */

typedef struct wfcu_tokens wfcu_tokens; /* device-resident token list in text order */

/* utf8_sanitize (proj/src/unicode.cpp:56-70; the ingest step, proj/src/analysis.cpp:53): every byte
 * that strict UTF-8 decoding (unicode.cpp:11-44) rejects becomes U+FFFD (EF BF BD), one replacement
 * per byte; valid sequences are copied.  The output is at most 3*n bytes; *out_len receives its
 * length (also when WFCU_ERR_BUFFER_TOO_SMALL reports that out_cap was not enough).  The device form
 * needs a 16-byte aligned dev_text, runs on `stream` and waits for it. */
WFCU_API int wfcu_utf8_sanitize_dev(const uint8_t* dev_text, uint64_t n, uint8_t* dev_out, uint64_t out_cap,
                           uint64_t* out_len, void* stream);
WFCU_API int wfcu_utf8_sanitize_host(const uint8_t* text, uint64_t n, uint8_t* out, uint64_t out_cap, uint64_t* out_len);

/* normalize_word (proj/src/text.cpp:9-30) over a batch of whitespace-free fragments:
 * case fold, strip non-word characters from both ends, U+FFFD for invalid bytes.
 * Fragment f is bytes[sum(lens[0..f)) ..]; the normalised words are written back to
 * back into out_bytes (capacity >= 3 * total input bytes is always enough) and
 * out_lens[f] = 0 means nothing remains (the reference's nullopt). */
WFCU_API int wfcu_normalize_words_host(const uint8_t* bytes, const uint32_t* lens, uint64_t n_frag,
                                       uint8_t* out_bytes, uint64_t out_cap, uint32_t* out_lens);

/* wfc::tokenize on a device buffer: tokens in text order.  dev_text is 16-byte aligned and its last, partial 16-byte
 * chunk lies inside the allocation (any cudaMalloc'd buffer does; only the bytes below n are read). */
WFCU_API int wfcu_tokenize_dev(const uint8_t* dev_text, uint64_t n, void* stream, wfcu_tokens** out);
WFCU_API int wfcu_tokenize_host(const uint8_t* text, uint64_t n, wfcu_tokens** out);
/* The tokens of several documents as ONE list (a worker's map stage, proj/src/pipeline.cpp:25-33: the tokens of its
 * documents back to back): document d is docs[d][0 .. doc_lens[d]); the documents are gathered on the device with a
 * whitespace byte behind each (a document's end is a fragment's end, text.cpp:55), no host-side concatenation. */
WFCU_API int wfcu_tokenize_docs_host(const uint8_t* const* docs, const uint64_t* doc_lens, uint64_t n_docs, wfcu_tokens** out);
WFCU_API void wfcu_tokens_destroy(wfcu_tokens* t);
WFCU_API int wfcu_tokens_stats(const wfcu_tokens* t, uint64_t* n_tokens, uint64_t* n_bytes);
/* Packed copy-out: token bytes concatenated + per-token lengths. */
WFCU_API int wfcu_tokens_export(const wfcu_tokens* t, uint8_t* bytes, uint64_t bytes_cap, uint32_t* lens,
                       uint64_t lens_cap);
/* Builds a device token list from packed host words (WordList -> device). */
WFCU_API int wfcu_tokens_from_words(const uint8_t* bytes, const uint32_t* lens, uint64_t n_tokens,
                           wfcu_tokens** out);
/* The exchange of the paper's range-partitioned pipeline in device memory (proj/src/shuffle.cpp:98-130: chunk c of
 * every worker's sorted list goes to worker c): a new list made of the slices [begin[i], end[i]) of n_src lists, in
 * that order.  Device-to-device copies (peer copies between GPUs); no frame, no host string. */
WFCU_API int wfcu_tokens_concat_slices(const wfcu_tokens* const* src, const uint64_t* begin, const uint64_t* end,
                                       uint32_t n_src, wfcu_tokens** out);
/* WCX1 frames in device memory (the paper's exchange with an NCCL-backed transport).
 * encode_message (proj/src/wire.cpp:27-48) of the slice [begin, end) of a device token list: "WCX1", u32-LE word
 * count, u32-LE length of every word, the payloads.  dev_frame == NULL: only *frame_bytes.  The frame never exists in
 * host memory; dev_frame must be 4-byte aligned. */
WFCU_API int wfcu_tokens_encode_frame(const wfcu_tokens* t, uint64_t begin, uint64_t end, uint8_t* dev_frame,
                                      uint64_t frame_cap, uint64_t* frame_bytes, void* stream);
/* decode_message (proj/src/wire.cpp:50-87) of a frame in device memory into a device token list: the reference's
 * checks in its order -- WFCU_ERR_FRAME_MAGIC / _TRUNCATED / _TRAILING / _ENCODING map WireError::Kind one to one
 * (the UTF-8 check is one device pass over the payload).  A frame with an empty word is not a token list
 * (WFCU_ERR_INVALID_ARGUMENT). */
WFCU_API int wfcu_tokens_decode_frame(const uint8_t* dev_frame, uint64_t frame_bytes, wfcu_tokens** out, void* stream);
/* sort_words (proj/src/text.cpp:59-63): stable byte-wise sort, in place. */
WFCU_API int wfcu_tokens_sort(wfcu_tokens* t, void* stream);
/* reduce_sorted (proj/src/reduce.cpp:8-21): run-length encodes a sorted list
 * into the counter; WFCU_ERR_NOT_SORTED if the list is not in order. */
WFCU_API int wfcu_tokens_reduce_sorted(const wfcu_tokens* t, wfcu_counter* into, void* stream);
/* The sort + RLE alternative end to end on a device buffer: tokenize, sort,
 * run-length encode, add the runs to the counter. */
WFCU_API int wfcu_counter_count_dev_sorted(wfcu_counter* c, const uint8_t* dev_text, uint64_t n, void* stream);

/* ------------------------------------------------------------------------- */
/* run_wordcount over n workers on the GPUs of one box                         */
/* (proj/src/pipeline.cpp:61-123, proj/include/wfc/pipeline.hpp:15-51)         */
/* ------------------------------------------------------------------------- */

/* A pair of CUDA events on the current device: the device time between start and stop on the legacy default stream,
 * which is what the reference's timed_stage (proj/src/pipeline.cpp:48-57) becomes when the stage runs on the GPU. */
typedef struct wfcu_timer wfcu_timer;
WFCU_API int wfcu_timer_create(wfcu_timer** out);
WFCU_API int wfcu_timer_start(wfcu_timer* t);
WFCU_API int wfcu_timer_stop_ns(wfcu_timer* t, uint64_t* elapsed_ns);   /* waits for the device */
WFCU_API void wfcu_timer_destroy(wfcu_timer* t);

/* StageTimings (proj/include/wfc/pipeline.hpp:15-23), filled from CUDA events: maximum over the workers. */
typedef struct wfcu_stage_ns {
    uint64_t map_ns;       /* H2D + fused tokenize / count kernels */
    uint64_t sort_ns;      /* 0: the hash-count path does not sort */
    uint64_t encode_ns;    /* partition of the local table by owner */
    uint64_t exchange_ns;  /* device-to-device delivery of the regions + merge-insert */
    uint64_t reduce_ns;    /* 0 here: the caller exports the owner tables */
    uint64_t repair_ns;    /* 0: every key has exactly one owner */
    uint64_t total_ns;     /* host wall clock of the call */
} wfcu_stage_ns;

/* Worker j (0 <= j < n_workers) lives on device j mod wfcu_device_count(), counts the documents d = j (mod n_workers)
 * (the reference's rule, pipeline.cpp:83) and ends up owning the keys whose owner hash is j: out_shards[j] is that
 * table, resident on its device (the caller destroys it).  One host thread per worker; regions travel device to
 * device (cudaMemcpyPeerAsync: NVLink between GPUs).  The union of the shards is serial_wordcount's map and no key
 * has two holders (count_unreduced_words == 0).  cfg sizes every table (NULL: defaults).  On failure nothing is
 * returned and the message names the lowest-indexed worker that failed. */
WFCU_API int wfcu_wordcount_multi(const uint8_t* const* docs, const uint64_t* lens, uint64_t n_docs, uint32_t n_workers,
                                  const wfcu_counter_config* cfg, wfcu_counter** out_shards, wfcu_stage_ns* timings);

/* ------------------------------------------------------------------------- */
/* top_k / distinctive_words over exported tables                            */
/* (proj/src/analysis.cpp:58-132).  Tables are (key_bytes, key_lens, counts) */
/* in std::map order, as wfcu_counter_export writes them.                    */
/* ------------------------------------------------------------------------- */

/* Rows ordered by count descending, ties by word ascending, truncated to k.
 * out_idx[r] indexes the input table, out_rel[r] = count / total over the WHOLE table. */
WFCU_API int wfcu_top_k(const uint8_t* key_bytes, const uint32_t* key_lens, const uint64_t* counts, uint64_t n,
                        uint64_t k, uint64_t* out_idx, double* out_rel, uint64_t* total, uint64_t* n_rows);

/* score = log((c_t+1)/(T_t+V)) - log((c_o+1)/(T_o+V)), V = |union vocabulary|; rows by
 * score descending (exact double compare), ties by word ascending.  out_src[r] = 0: the
 * word is row out_idx[r] of the target table, 1: of the others table. */
WFCU_API int wfcu_distinctive(const uint8_t* t_bytes, const uint32_t* t_lens, const uint64_t* t_counts, uint64_t nt,
                              const uint8_t* o_bytes, const uint32_t* o_lens, const uint64_t* o_counts, uint64_t no,
                              uint64_t k, int32_t* out_src, uint64_t* out_idx, double* out_score, uint64_t* n_rows);

/* ------------------------------------------------------------------------- */
/* Synthetic corpora for BASELINE.json configs 3-5; host-side */
/* generator, deterministic for (seed, doc index).                            */
/* ------------------------------------------------------------------------- */

/* Fills out[0..doc_bytes) with document `doc` of a Zipf(s) corpus over a
 * `vocab`-word vocabulary.  `speaker` permutes 1 % of the ranks (config 5). */
WFCU_API int wfcu_synth_document(uint64_t seed, uint64_t doc, uint32_t vocab, double zipf_s, uint32_t speaker,
                        uint8_t* out, uint64_t doc_bytes);
/* Documents [doc_begin, doc_end) back to back ('\n' ends every document), using
 * `threads` host threads (0 = all). */
WFCU_API int wfcu_synth_corpus(uint64_t seed, uint64_t doc_begin, uint64_t doc_end, uint32_t vocab,
                      double zipf_s, uint32_t speaker, uint64_t doc_bytes, uint8_t* out, int threads);

/* Documents doc_begin, doc_begin + doc_stride, ... (n_docs of them): the shard of the
 * rank that owns documents d = doc_begin (mod doc_stride). */
WFCU_API int wfcu_synth_corpus_strided(uint64_t seed, uint64_t doc_begin, uint64_t doc_stride, uint64_t n_docs,
                                       uint32_t vocab, double zipf_s, uint32_t speaker, uint64_t doc_bytes,
                                       uint8_t* out, int threads);

/* The reference bench's input recipe (proj/src/cli.cpp:120-125): n draws of
 * std::mt19937_64(seed) through std::uniform_real_distribution<double>(0,1),
 * stored as double (WFCU_DTYPE_F64) or rounded to float (WFCU_DTYPE_F32). */
WFCU_API int wfcu_synth_uniform(uint64_t seed, uint64_t n, int dtype, void* out);

/* Number of kernels this library has launched in this process (bench.py's
 * gpu_launches evidence). */
WFCU_API uint64_t wfcu_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* WFCU_H */
