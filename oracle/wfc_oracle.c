/*
 * oracle/wfc_oracle.c -- CPU restatement of the reference word-frequency hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may build, load or call it, and only as the checker / the timed CPU
 * baseline.  The product path (paper_2206_05269_b200/) never links or calls it.
 *
 * Parity is PINNED: oracle/Makefile also compiles the unmodified reference
 * sources from /root/reference/proj/src into oracle/_ref/libwfc_ref.so (behind
 * oracle/ref_capi.cpp) and tests/test_oracle_vs_ref.py checks this restatement
 * against it, next to the reference's own golden vectors (tests/golden/).
 *
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/).  Plain C11, no dependencies beyond libc/libm.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define WFO_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ */
/* a1: UTF-8 decode + character classes (proj/src/unicode.cpp:11-121)  */
/* ------------------------------------------------------------------ */

typedef struct {
    uint32_t cp;    /* code point, U+FFFD when invalid          */
    uint32_t len;   /* bytes consumed (always 1 when invalid)   */
    int32_t valid;
} wfo_decoded;

/* proj/src/unicode.cpp:11-44: strict decode; overlong, surrogate, >U+10FFFF,
 * stray continuation and truncated sequences are invalid and eat one byte. */
WFO_API wfo_decoded wfo_utf8_decode(const uint8_t* s, uint64_t n, uint64_t pos) {
    const wfo_decoded bad = {0xFFFDu, 1u, 0};
    if (pos >= n) return bad;
    const uint8_t lead = s[pos];
    if (lead < 0x80) {
        wfo_decoded ok = {lead, 1u, 1};
        return ok;
    }
    uint32_t extra, cp;
    uint8_t lo = 0x80, hi = 0xBF; /* window for the first continuation byte */
    if (lead >= 0xC2 && lead <= 0xDF) {
        extra = 1; cp = lead & 0x1Fu;
    } else if (lead >= 0xE0 && lead <= 0xEF) {
        extra = 2; cp = lead & 0x0Fu;
        if (lead == 0xE0) lo = 0xA0;      /* no overlong 3-byte forms */
        if (lead == 0xED) hi = 0x9F;      /* no surrogates            */
    } else if (lead >= 0xF0 && lead <= 0xF4) {
        extra = 3; cp = lead & 0x07u;
        if (lead == 0xF0) lo = 0x90;      /* no overlong 4-byte forms */
        if (lead == 0xF4) hi = 0x8F;      /* nothing above U+10FFFF   */
    } else {
        return bad;                       /* 80..C1, F5..FF */
    }
    if (pos + extra >= n) return bad;     /* truncated */
    for (uint32_t k = 1; k <= extra; ++k) {
        const uint8_t b = s[pos + k];
        const uint8_t l = (k == 1) ? lo : 0x80, h = (k == 1) ? hi : 0xBF;
        if (b < l || b > h) return bad;
        cp = (cp << 6) | (b & 0x3Fu);
    }
    wfo_decoded ok = {cp, extra + 1u, 1};
    return ok;
}

/* proj/src/unicode.cpp:90-99 */
WFO_API int wfo_is_space(uint32_t cp) {
    if (cp >= 0x09 && cp <= 0x0D) return 1;
    if (cp >= 0x2000 && cp <= 0x200A) return 1;
    return cp == 0x20 || cp == 0x85 || cp == 0xA0 || cp == 0x1680 || cp == 0x2028 ||
           cp == 0x2029 || cp == 0x202F || cp == 0x205F || cp == 0x3000;
}

/* proj/src/unicode.cpp:101-115 */
WFO_API int wfo_is_word_char(uint32_t cp) {
    if (cp < 0x80) {
        const uint32_t l = cp | 0x20u;
        return (cp >= '0' && cp <= '9') || (l >= 'a' && l <= 'z');
    }
    if (cp == 0xFFFD) return 0;
    if (cp >= 0xA1 && cp <= 0xBF) return cp == 0xAA || cp == 0xB5 || cp == 0xBA;
    if (cp == 0xD7 || cp == 0xF7) return 0;
    if ((cp >= 0x2000 && cp <= 0x206F) || (cp >= 0x3000 && cp <= 0x303F)) return 0;
    if ((cp >= 0xFF01 && cp <= 0xFF0F) || (cp >= 0xFF1A && cp <= 0xFF20)) return 0;
    if ((cp >= 0xFF3B && cp <= 0xFF40) || (cp >= 0xFF5B && cp <= 0xFF65)) return 0;
    return !wfo_is_space(cp);
}

/* proj/src/unicode.cpp:117-121 */
WFO_API uint32_t wfo_simple_lower(uint32_t cp) {
    if (cp >= 'A' && cp <= 'Z') return cp + 0x20;
    if (cp >= 0xC0 && cp <= 0xDE && cp != 0xD7) return cp + 0x20;
    return cp;
}

/* proj/src/unicode.cpp:72-88; returns bytes written (1..4) */
static uint32_t put_utf8(uint8_t* out, uint32_t cp) {
    if (cp < 0x80) { out[0] = (uint8_t)cp; return 1; }
    if (cp < 0x800) {
        out[0] = (uint8_t)(0xC0 | (cp >> 6));
        out[1] = (uint8_t)(0x80 | (cp & 0x3F));
        return 2;
    }
    if (cp < 0x10000) {
        out[0] = (uint8_t)(0xE0 | (cp >> 12));
        out[1] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
        out[2] = (uint8_t)(0x80 | (cp & 0x3F));
        return 3;
    }
    out[0] = (uint8_t)(0xF0 | (cp >> 18));
    out[1] = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
    out[2] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
    out[3] = (uint8_t)(0x80 | (cp & 0x3F));
    return 4;
}

/* proj/src/unicode.cpp:46-54 */
WFO_API int wfo_utf8_valid(const uint8_t* s, uint64_t n) {
    for (uint64_t pos = 0; pos < n;) {
        const wfo_decoded d = wfo_utf8_decode(s, n, pos);
        if (!d.valid) return 0;
        pos += d.len;
    }
    return 1;
}

/* proj/src/unicode.cpp:56-70; out must hold 3*n bytes; returns bytes written */
WFO_API uint64_t wfo_utf8_sanitize(const uint8_t* s, uint64_t n, uint8_t* out) {
    uint64_t w = 0;
    for (uint64_t pos = 0; pos < n;) {
        const wfo_decoded d = wfo_utf8_decode(s, n, pos);
        if (d.valid) {
            memcpy(out + w, s + pos, d.len);
            w += d.len;
        } else {
            w += put_utf8(out + w, 0xFFFD);
        }
        pos += d.len;
    }
    return w;
}

/* ------------------------------------------------------------------ */
/* a2/a3: normalize_word + tokenize (proj/src/text.cpp:9-57)           */
/* ------------------------------------------------------------------ */

/* proj/src/text.cpp:9-30.  The reference decodes the fragment against ITS OWN
 * end (string_view), so a sequence truncated by the fragment end is invalid.
 * Writes the normalised token to out (capacity >= 3*n) and returns its length;
 * 0 means "nothing remains" (nullopt). */
WFO_API uint64_t wfo_normalize_word(const uint8_t* frag, uint64_t n, uint8_t* out) {
    /* pass 1: byte ranges [first_b, last_e) of the kept code points */
    uint64_t first_b = n, last_e = 0;
    for (uint64_t pos = 0; pos < n;) {
        const wfo_decoded d = wfo_utf8_decode(frag, n, pos);
        if (wfo_is_word_char(wfo_simple_lower(d.cp))) {
            if (first_b == n) first_b = pos;
            last_e = pos + d.len;
        }
        pos += d.len;
    }
    if (first_b == n) return 0;
    /* pass 2: fold + re-encode the kept middle (invalid bytes become EF BF BD) */
    uint64_t w = 0;
    for (uint64_t pos = first_b; pos < last_e;) {
        const wfo_decoded d = wfo_utf8_decode(frag, n, pos);
        w += put_utf8(out + w, wfo_simple_lower(d.cp));
        pos += d.len;
    }
    return w;
}

typedef void (*wfo_token_fn)(void* ctx, const uint8_t* tok, uint64_t len);

/* proj/src/text.cpp:32-57: fragments are maximal runs without a VALID
 * whitespace code point; decode happens against the whole document. */
static void tokenize_cb(const uint8_t* text, uint64_t n, wfo_token_fn fn, void* ctx,
                        uint8_t** scratch, uint64_t* scratch_cap) {
    uint64_t start = 0;
    int in_frag = 0;
    for (uint64_t pos = 0; pos <= n;) {
        wfo_decoded d = {0, 1, 0};
        int boundary = (pos == n);
        if (!boundary) {
            d = wfo_utf8_decode(text, n, pos);
            boundary = d.valid && wfo_is_space(d.cp);
        }
        if (boundary) {
            if (in_frag) {
                const uint64_t flen = pos - start;
                if (*scratch_cap < 3 * flen + 4) {
                    *scratch_cap = 3 * flen + 64;
                    *scratch = (uint8_t*)realloc(*scratch, *scratch_cap);
                }
                const uint64_t tl = wfo_normalize_word(text + start, flen, *scratch);
                if (tl) fn(ctx, *scratch, tl);
                in_frag = 0;
            }
        } else if (!in_frag) {
            start = pos;
            in_frag = 1;
        }
        pos += d.len;
    }
}

typedef struct {
    uint8_t* bytes; uint64_t bytes_cap, nbytes;
    uint32_t* lens; uint64_t lens_cap, ntok;
    int overflow;
} tok_sink;

static void sink_token(void* ctx, const uint8_t* tok, uint64_t len) {
    tok_sink* s = (tok_sink*)ctx;
    if (s->ntok >= s->lens_cap || s->nbytes + len > s->bytes_cap) {
        s->overflow = 1;
        s->ntok++; s->nbytes += len;   /* keep counting so callers can size buffers */
        return;
    }
    memcpy(s->bytes + s->nbytes, tok, len);
    s->lens[s->ntok++] = (uint32_t)len;
    s->nbytes += len;
}

/* Tokens in text order: concatenated bytes + per-token lengths.
 * Returns 0 ok, 1 if a capacity was too small (n_tokens/n_bytes still exact). */
WFO_API int wfo_tokenize(const uint8_t* text, uint64_t n, uint8_t* out_bytes, uint64_t bytes_cap,
                         uint32_t* out_lens, uint64_t lens_cap, uint64_t* n_tokens,
                         uint64_t* n_bytes) {
    tok_sink s = {out_bytes, bytes_cap, 0, out_lens, lens_cap, 0, 0};
    uint8_t* scratch = NULL; uint64_t cap = 0;
    tokenize_cb(text, n, sink_token, &s, &scratch, &cap);
    free(scratch);
    *n_tokens = s.ntok; *n_bytes = s.nbytes;
    return s.overflow;
}

/* ------------------------------------------------------------------ */
/* a4: the counting map  (proj/src/pipeline.cpp:131-139)               */
/*     ++counts[word] over every document; exported in std::map order  */
/*     = unsigned byte-wise lexicographic (proj/include/wfc/reduce.hpp:15) */
/* ------------------------------------------------------------------ */

typedef struct {
    uint64_t off;   /* into arena */
    uint32_t len;
    uint32_t used;
    uint64_t count;
    uint64_t hash;
} wfo_slot;

typedef struct wfo_counts {
    wfo_slot* slots; uint64_t cap, size;
    uint8_t* arena; uint64_t arena_cap, arena_len;
    uint64_t total;
    uint8_t* scratch; uint64_t scratch_cap;
} wfo_counts;

static uint64_t fnv1a(const uint8_t* p, uint64_t n) {
    uint64_t h = 1469598103934665603ull;
    for (uint64_t i = 0; i < n; ++i) { h ^= p[i]; h *= 1099511628211ull; }
    return h ^ (h >> 29);
}

WFO_API wfo_counts* wfo_counts_new(void) {
    wfo_counts* c = (wfo_counts*)calloc(1, sizeof(wfo_counts));
    c->cap = 1u << 12;
    c->slots = (wfo_slot*)calloc(c->cap, sizeof(wfo_slot));
    c->arena_cap = 1u << 16;
    c->arena = (uint8_t*)malloc(c->arena_cap);
    return c;
}

WFO_API void wfo_counts_free(wfo_counts* c) {
    if (!c) return;
    free(c->slots); free(c->arena); free(c->scratch); free(c);
}

static void counts_grow(wfo_counts* c) {
    const uint64_t ncap = c->cap * 2;
    wfo_slot* ns = (wfo_slot*)calloc(ncap, sizeof(wfo_slot));
    for (uint64_t i = 0; i < c->cap; ++i) {
        if (!c->slots[i].used) continue;
        uint64_t j = c->slots[i].hash & (ncap - 1);
        while (ns[j].used) j = (j + 1) & (ncap - 1);
        ns[j] = c->slots[i];
    }
    free(c->slots);
    c->slots = ns; c->cap = ncap;
}

WFO_API void wfo_counts_add(wfo_counts* c, const uint8_t* tok, uint64_t len, uint64_t by) {
    const uint64_t h = fnv1a(tok, len);
    uint64_t j = h & (c->cap - 1);
    for (;;) {
        wfo_slot* s = &c->slots[j];
        if (!s->used) break;
        if (s->hash == h && s->len == len && memcmp(c->arena + s->off, tok, len) == 0) {
            s->count += by; c->total += by;
            return;
        }
        j = (j + 1) & (c->cap - 1);
    }
    if (c->arena_len + len > c->arena_cap) {
        while (c->arena_len + len > c->arena_cap) c->arena_cap *= 2;
        c->arena = (uint8_t*)realloc(c->arena, c->arena_cap);
    }
    memcpy(c->arena + c->arena_len, tok, len);
    wfo_slot* s = &c->slots[j];
    s->off = c->arena_len; s->len = (uint32_t)len; s->used = 1; s->count = by; s->hash = h;
    c->arena_len += len; c->size++; c->total += by;
    if (c->size * 10 > c->cap * 6) counts_grow(c);
}

static void count_token(void* ctx, const uint8_t* tok, uint64_t len) {
    wfo_counts_add((wfo_counts*)ctx, tok, len, 1);
}

/* one document of serial_wordcount (proj/src/pipeline.cpp:133-137) */
WFO_API void wfo_counts_add_document(wfo_counts* c, const uint8_t* text, uint64_t n) {
    tokenize_cb(text, n, count_token, c, &c->scratch, &c->scratch_cap);
}

WFO_API uint64_t wfo_counts_distinct(const wfo_counts* c) { return c->size; }
WFO_API uint64_t wfo_counts_total(const wfo_counts* c) { return c->total; }
WFO_API uint64_t wfo_counts_key_bytes(const wfo_counts* c) { return c->arena_len; }

static const uint8_t* g_sort_arena;
static int slot_cmp(const void* a, const void* b) {
    const wfo_slot* x = (const wfo_slot*)a; const wfo_slot* y = (const wfo_slot*)b;
    const uint32_t m = x->len < y->len ? x->len : y->len;
    const int r = memcmp(g_sort_arena + x->off, g_sort_arena + y->off, m);
    if (r) return r;
    return (x->len > y->len) - (x->len < y->len);
}

/* Export in std::map iteration order.  key_bytes: concatenated keys
 * (wfo_counts_key_bytes), key_lens / counts: wfo_counts_distinct entries. */
WFO_API void wfo_counts_export(const wfo_counts* c, uint8_t* key_bytes, uint32_t* key_lens,
                               uint64_t* counts) {
    wfo_slot* v = (wfo_slot*)malloc((c->size ? c->size : 1) * sizeof(wfo_slot));
    uint64_t k = 0;
    for (uint64_t i = 0; i < c->cap; ++i) if (c->slots[i].used) v[k++] = c->slots[i];
    g_sort_arena = c->arena;
    qsort(v, k, sizeof(wfo_slot), slot_cmp);
    uint64_t w = 0;
    for (uint64_t i = 0; i < k; ++i) {
        memcpy(key_bytes + w, c->arena + v[i].off, v[i].len);
        w += v[i].len; key_lens[i] = v[i].len; counts[i] = v[i].count;
    }
    free(v);
}

/* merge_counts (proj/src/reduce.cpp:83-89): dst[word] += src[word] */
WFO_API void wfo_counts_merge(wfo_counts* dst, const wfo_counts* src) {
    for (uint64_t i = 0; i < src->cap; ++i) {
        const wfo_slot* s = &src->slots[i];
        if (s->used) wfo_counts_add(dst, src->arena + s->off, s->len, s->count);
    }
}

/* ------------------------------------------------------------------ */
/* a5: sort_words + reduce_sorted  (proj/src/text.cpp:59-63,           */
/*     proj/src/reduce.cpp:8-21) on the packed token representation    */
/* ------------------------------------------------------------------ */

typedef struct { const uint8_t* p; uint32_t len; uint32_t idx; } tokref;
static int tokref_cmp(const void* a, const void* b) {
    const tokref* x = (const tokref*)a; const tokref* y = (const tokref*)b;
    const uint32_t m = x->len < y->len ? x->len : y->len;
    const int r = memcmp(x->p, y->p, m);
    if (r) return r;
    if (x->len != y->len) return (x->len > y->len) - (x->len < y->len);
    return (x->idx > y->idx) - (x->idx < y->idx); /* stable */
}

/* Sorts the packed token list (bytes+lens) byte-wise, stably; writes the
 * sorted packed list to out_bytes/out_lens (same sizes as the input). */
WFO_API void wfo_sort_words(const uint8_t* bytes, const uint32_t* lens, uint64_t ntok,
                            uint8_t* out_bytes, uint32_t* out_lens) {
    tokref* v = (tokref*)malloc((ntok ? ntok : 1) * sizeof(tokref));
    uint64_t off = 0;
    for (uint64_t i = 0; i < ntok; ++i) { v[i].p = bytes + off; v[i].len = lens[i]; v[i].idx = (uint32_t)i; off += lens[i]; }
    qsort(v, ntok, sizeof(tokref), tokref_cmp);
    uint64_t w = 0;
    for (uint64_t i = 0; i < ntok; ++i) { memcpy(out_bytes + w, v[i].p, v[i].len); out_lens[i] = v[i].len; w += v[i].len; }
    free(v);
}

/* Run-length encode a SORTED packed list.  Returns the number of runs; run r
 * is described by run_first[r] (index of its first token) and run_count[r].
 * Returns UINT64_MAX if the list is not sorted (the reference throws
 * std::invalid_argument when the sorted flag is missing). */
WFO_API uint64_t wfo_reduce_sorted(const uint8_t* bytes, const uint32_t* lens, uint64_t ntok,
                                   uint64_t* run_first, uint64_t* run_count) {
    uint64_t runs = 0, off = 0, prev_off = 0;
    for (uint64_t i = 0; i < ntok; ++i) {
        int same = 0;
        if (i > 0) {
            const uint32_t pl = lens[i - 1], cl = lens[i];
            const uint32_t m = pl < cl ? pl : cl;
            const int r = memcmp(bytes + prev_off, bytes + off, m);
            if (r > 0 || (r == 0 && pl > cl)) return UINT64_MAX;
            same = (r == 0 && pl == cl);
        }
        if (same) run_count[runs - 1]++;
        else { run_first[runs] = i; run_count[runs] = 1; runs++; }
        prev_off = off; off += lens[i];
    }
    return runs;
}

/* ------------------------------------------------------------------ */
/* a7: plan_partition  (proj/src/shuffle.cpp:9-46)                     */
/* ------------------------------------------------------------------ */

/* boundaries must hold n_workers+1 entries. returns 0 ok, -1 bad args */
WFO_API int wfo_plan_partition(uint64_t k, uint64_t worker_id, uint64_t n_workers,
                               uint64_t* boundaries) {
    if (n_workers == 0 || worker_id >= n_workers) return -1;
    const uint64_t keep = k / n_workers;
    uint64_t base = 0, extra = 0;
    if (n_workers > 1) {
        base = (k - keep) / (n_workers - 1);
        extra = (k - keep) % (n_workers - 1);
    }
    boundaries[0] = 0;
    for (uint64_t c = 0; c < n_workers; ++c) {
        uint64_t size;
        if (c == worker_id) size = keep;
        else { size = base + (extra ? 1 : 0); if (extra) --extra; }
        boundaries[c + 1] = boundaries[c] + size;
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* a9: map-then-reduce engine  (proj/src/engine.cpp:15-98)             */
/* kinds: 0 identity, 1 square_root, 2 alternating_harmonic_term       */
/*        (proj/include/wfc/engine.hpp:12-16) and 3 = square, appended */
/*        for BASELINE.json config 2 (no reference counterpart; the    */
/*        oracle is fold_range over double(x)*double(x)).              */
/* ------------------------------------------------------------------ */

static inline double map_term(double v, uint64_t position, int kind) {
    switch (kind) {
        case 0: return v;
        case 1: return sqrt(v);
        case 2: return ((position & 1u) ? 1.0 : -1.0) / (double)position;
        default: return v * v;
    }
}

#define FOLD_BODY(LOAD)                                                     \
    double acc = 0.0;                                                       \
    for (uint64_t i = begin; i < end; ++i) acc += map_term(LOAD, i + 1, kind); \
    return acc;

/* fold_range, proj/src/engine.cpp:15-20 (left-to-right, starting from 0.0) */
static double fold_f64(const double* v, uint64_t begin, uint64_t end, int kind) { FOLD_BODY(v ? v[i] : 0.0) }
static double fold_f32(const float* v, uint64_t begin, uint64_t end, int kind) { FOLD_BODY(v ? (double)v[i] : 0.0) }

/* combine_tree, proj/src/engine.cpp:23-34: pairwise rounds, odd tail carried */
static double combine_tree(double* level, uint64_t m) {
    if (m == 0) return 0.0;
    while (m > 1) {
        uint64_t out = 0;
        for (uint64_t i = 0; i + 1 < m; i += 2) level[out++] = level[i] + level[i + 1];
        if (m & 1u) level[out++] = level[m - 1];
        m = out;
    }
    return level[0];
}

/* map_reduce_serial, proj/src/engine.cpp:82-86 */
WFO_API double wfo_map_reduce_serial_f64(const double* v, uint64_t n, int kind) { return fold_f64(v, 0, n, kind); }
WFO_API double wfo_map_reduce_serial_f32(const float* v, uint64_t n, int kind) { return fold_f32(v, 0, n, kind); }

/* map_reduce_blocked / blocked_sum, proj/src/engine.cpp:36-66,88-92.  The
 * worker count only changes scheduling, never the value, so it is not a
 * parameter here.  Returns NaN-free -1.0 via *err=1 when block_size==0. */
WFO_API double wfo_map_reduce_blocked_f64(const double* v, uint64_t n, int kind, uint64_t block, int* err) {
    if (err) *err = 0;
    if (block == 0) { if (err) *err = 1; return 0.0; }
    const uint64_t nb = (n + block - 1) / block;
    double* part = (double*)malloc((nb ? nb : 1) * sizeof(double));
    for (uint64_t b = 0; b < nb; ++b) {
        const uint64_t lo = b * block, hi = (lo + block < n) ? lo + block : n;
        part[b] = fold_f64(v, lo, hi, kind);
    }
    const double r = combine_tree(part, nb);
    free(part);
    return r;
}

WFO_API double wfo_map_reduce_blocked_f32(const float* v, uint64_t n, int kind, uint64_t block, int* err) {
    if (err) *err = 0;
    if (block == 0) { if (err) *err = 1; return 0.0; }
    const uint64_t nb = (n + block - 1) / block;
    double* part = (double*)malloc((nb ? nb : 1) * sizeof(double));
    for (uint64_t b = 0; b < nb; ++b) {
        const uint64_t lo = b * block, hi = (lo + block < n) ? lo + block : n;
        part[b] = fold_f32(v, lo, hi, kind);
    }
    const double r = combine_tree(part, nb);
    free(part);
    return r;
}

/* alternating_harmonic, proj/src/engine.cpp:94-98 */
WFO_API double wfo_alternating_harmonic(uint64_t n, uint64_t block, int* err) {
    return wfo_map_reduce_blocked_f64(NULL, n, 2, block, err);
}

/* ------------------------------------------------------------------ */
/* a10: top_k / distinctive_words  (proj/src/analysis.cpp:58-132)      */
/* Inputs are count tables in std::map order (sorted packed keys).     */
/* ------------------------------------------------------------------ */

typedef struct { const uint8_t* p; uint32_t len; int32_t src; uint64_t count; uint64_t other; double score; uint64_t idx; } rowref;

static int key_cmp(const uint8_t* a, uint32_t al, const uint8_t* b, uint32_t bl) {
    const uint32_t m = al < bl ? al : bl;
    const int r = memcmp(a, b, m);
    if (r) return r;
    return (al > bl) - (al < bl);
}

static int topk_cmp(const void* a, const void* b) {
    const rowref* x = (const rowref*)a; const rowref* y = (const rowref*)b;
    if (x->count != y->count) return x->count > y->count ? -1 : 1;
    return key_cmp(x->p, x->len, y->p, y->len);
}

/* top_k, proj/src/analysis.cpp:58-75.  Writes min(k, n) row indices (into the
 * input table) to out_idx and count/total to out_rel; returns rows written;
 * *total gets the sum over the WHOLE table. */
WFO_API uint64_t wfo_top_k(const uint8_t* key_bytes, const uint32_t* key_lens, const uint64_t* counts,
                           uint64_t n, uint64_t k, uint64_t* out_idx, double* out_rel, uint64_t* total) {
    rowref* v = (rowref*)malloc((n ? n : 1) * sizeof(rowref));
    uint64_t off = 0, tot = 0;
    for (uint64_t i = 0; i < n; ++i) {
        v[i].p = key_bytes + off; v[i].len = key_lens[i]; v[i].count = counts[i]; v[i].idx = i; v[i].score = 0; v[i].src = 0; v[i].other = 0;
        off += key_lens[i]; tot += counts[i];
    }
    qsort(v, n, sizeof(rowref), topk_cmp);   /* keys are distinct: total order, stability moot */
    const uint64_t m = k < n ? k : n;
    for (uint64_t i = 0; i < m; ++i) { out_idx[i] = v[i].idx; out_rel[i] = (double)v[i].count / (double)tot; }
    *total = tot;
    free(v);
    return m;
}

static int score_cmp(const void* a, const void* b) {
    const rowref* x = (const rowref*)a; const rowref* y = (const rowref*)b;
    if (x->score != y->score) return x->score > y->score ? -1 : 1;
    return key_cmp(x->p, x->len, y->p, y->len);
}

/* distinctive_words, proj/src/analysis.cpp:77-132.
 * score = log((c_t+1)/(T_t+V)) - log((c_o+1)/(T_o+V)), V = |union vocabulary|.
 * Output row r: out_src[r] = 0 (key lives in target table) or 1 (others table),
 * out_idx[r] = index into that table, out_score[r].  Returns rows written. */
WFO_API uint64_t wfo_distinctive(const uint8_t* t_bytes, const uint32_t* t_lens, const uint64_t* t_counts, uint64_t nt,
                                 const uint8_t* o_bytes, const uint32_t* o_lens, const uint64_t* o_counts, uint64_t no,
                                 uint64_t k, int32_t* out_src, uint64_t* out_idx, double* out_score) {
    if (nt == 0 && no == 0) return 0;
    uint64_t Tt = 0, To = 0;
    for (uint64_t i = 0; i < nt; ++i) Tt += t_counts[i];
    for (uint64_t i = 0; i < no; ++i) To += o_counts[i];
    rowref* v = (rowref*)malloc((nt + no) * sizeof(rowref));
    /* merge walk over the two sorted tables = union vocabulary (:88-103) */
    uint64_t i = 0, j = 0, toff = 0, ooff = 0, rows = 0;
    while (i < nt || j < no) {
        int c;
        if (j >= no) c = -1;
        else if (i >= nt) c = 1;
        else c = key_cmp(t_bytes + toff, t_lens[i], o_bytes + ooff, o_lens[j]);
        rowref* r = &v[rows++];
        if (c <= 0) {   /* word present in target (maybe in others too) */
            r->p = t_bytes + toff; r->len = t_lens[i]; r->src = 0; r->idx = i;
            r->count = t_counts[i]; r->other = (c == 0) ? o_counts[j] : 0;
            toff += t_lens[i]; ++i;
            if (c == 0) { ooff += o_lens[j]; ++j; }
        } else {        /* others only */
            r->p = o_bytes + ooff; r->len = o_lens[j]; r->src = 1; r->idx = j;
            r->count = 0; r->other = o_counts[j];
            ooff += o_lens[j]; ++j;
        }
    }
    /* scores need V = rows, known only now (:105-110) */
    const double dt = (double)Tt + (double)rows, dn = (double)To + (double)rows;
    for (uint64_t r = 0; r < rows; ++r)
        v[r].score = log(((double)v[r].count + 1.0) / dt) - log(((double)v[r].other + 1.0) / dn);
    qsort(v, rows, sizeof(rowref), score_cmp);
    const uint64_t m = k < rows ? k : rows;
    for (uint64_t r = 0; r < m; ++r) {
        out_src[r] = v[r].src;
        out_idx[r] = v[r].idx;
        out_score[r] = v[r].score;
    }
    free(v);
    return m;
}
