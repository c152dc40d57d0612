// capi.cu -- the extern "C" surface declared in include/wfcu.h.
// Thin host logic only: argument checks, workspace ownership, launches.  Every
// compute step is a kernel in wordcount.cu / mapreduce.cu / table_ops.cu /
// tokens.cu; there is no CPU implementation of the path behind any entry point.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <map>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/wfcu.h"
#include "wfcu_dev.cuh"

namespace wfcu {
// wordcount.cu
cudaError_t wc_launch(const uint8_t* text, u64 n, const TableView& gt, int sm_count, cudaStream_t stream, u64* launches,
                      cudaEvent_t* ev_before_fast, cudaEvent_t* ev_after_fast, u32 variant_hint);
// mapreduce.cu
cudaError_t mr_launch(const void* values, int is_f64, u64 n, u64 base, int kind, int grid, double* partials,
                      double* dev_out, cudaStream_t s, u64* launches);
cudaError_t mr_blocked_launch(const void* values, int is_f64, u64 n, u64 base, int kind, u64 block, double* buf_a,
                              double* buf_b, double* dev_out, int sm_count, cudaStream_t s, u64* launches);
// table_ops.cu
cudaError_t tb_compact(const TableView& t, Slot* out, u64 cap, u64* dev_count, int sm, cudaStream_t s, u64* launches);
cudaError_t tb_compact_recs(const TableView& t, TokenRec* out, u64 cap, u64* dev_count, int sm, cudaStream_t s, u64* launches);
cudaError_t tb_lower_bound_pos(const TokenRec* recs, u64 n, u64 value, u64* dev_out, cudaStream_t s, u64* launches);
cudaError_t tb_union_rows(const TableView& target, const TableView& others, TokenRec* recs, u64* ct, u64* co, u64 cap,
                          u64* dev_cursor, int sm, cudaStream_t s, u64* launches);
cudaError_t tb_score_rows(TokenRec* recs, const u64* ct, const u64* co, const u64* dev_n_rows, u64 max_rows, u64 extra_vocab,
                          u64 t_total, u64 o_total, int sm, cudaStream_t s, u64* launches);
cudaError_t tb_reset_aux(const TableView& t, u64* counters, unsigned int* done, int sm, cudaStream_t s, u64* launches);
cudaError_t tk_rebase_ext(TokenRec* recs, u64 n, u64 delta, int sm, cudaStream_t s, u64* launches);
cudaError_t tb_gather_counts(const TokenRec* recs, u64 first, u64 n, const u64* ct, const u64* co, u64* out_ct, u64* out_co,
                             int sm, cudaStream_t s, u64* launches);
cudaError_t tb_export_pack(const TokenRec* recs, u64 n, u64* lens64, u64* tmp, uint8_t* bytes, u32* lens32, u64* counts,
                           u64* dev_total_bytes, int sm, cudaStream_t s, u64* launches);
cudaError_t tb_key_bytes(const TableView& t, u64* dev_bytes, int sm, cudaStream_t s, u64* launches);
cudaError_t tb_partition(const TableView& t, u32 n_parts, Slot* out, u64 cap, u64* dev_part_counts, u64* cursors,
                         int sm, cudaStream_t s, u64* launches);
cudaError_t tb_merge_entries(const TableView& t, const Slot* in, u64 n, int sm, cudaStream_t s, u64* launches);
cudaError_t tb_partition_fixed(const TableView& t, u32 n_parts, u64 cap, bool framed, Slot* out, u64* dev_counts, int sm,
                               cudaStream_t s, u64* launches);
cudaError_t tb_merge_regions(const TableView& t, const Slot* in, u32 n_parts, u64 cap, const u64* region_counts, int sm,
                             cudaStream_t s, u64* launches);
cudaError_t tb_merge_table(const TableView& dst, const TableView& src, int sm, cudaStream_t s, u64* launches);
cudaError_t tb_long_serialize(const TableView& t, uint8_t* out, u64 cap, u64* dev_bytes, int sm, cudaStream_t s,
                              u64* launches);
cudaError_t tb_long_merge(const TableView& t, const uint8_t* recs, u64 n_bytes, u32 part, u32 n_parts, cudaStream_t s,
                          u64* launches);
// wordcount.cu (stand-alone tokenizer) and tokens.cu
cudaError_t wc_tokenize_launch(const uint8_t* text, u64 n, const TableView& gt, const EmitView& em, int sm_count,
                               cudaStream_t stream, u64* launches);
cudaError_t wc_normalize_launch(const uint8_t* text, const u64* offsets, u64 n_frag, const TableView& gt,
                                const EmitView& em, int sm_count, cudaStream_t stream, u64* launches);
struct SortScratch {
    TokenRec* alt;
    u64* hist;
    u64* tmp;
};
u64 sort_hist_words(u64 n);
u64 sort_n_tiles(u64 n);
u64 scan_tmp_words(u64 n);
cudaError_t tokens_sort(TokenRec* recs, u64 n, bool by_position, const uint8_t* arena, const SortScratch& sc, int sm,
                        cudaStream_t s, u64* launches);
cudaError_t tokens_rle_flags(const TokenRec* recs, u64 n, const uint8_t* arena, u64* flags, int* status, int sm,
                             cudaStream_t s, u64* launches);
cudaError_t tokens_rle_insert(const TokenRec* recs, u64 n, const uint8_t* arena, u64* flags, u64* run_start, u64* tmp,
                              const TableView& t, int sm, cudaStream_t s, u64* launches);
// sanitize.cu
u64 sanitize_scratch_bytes(u64 n);
cudaError_t sanitize_launch(const uint8_t* text, u64 n, uint8_t* out, u64 out_cap, void* scratch, u64* dev_total,
                            int sm_count, cudaStream_t s, u64* launches);
cudaError_t tokens_compact_count(u64* keys_a, u64* keys_b, u64 nk, u64 vary, u64* hist, u64* tmp, u64* flags, u64* run_start,
                                 const TableView& t, int sm, cudaStream_t s, u64* launches, const u32* tile_counts,
                                 u64 tiled_tiles);
cudaError_t exclusive_scan_u64(const u64* in, u64* out, u64 n, u64* tmp, cudaStream_t s, u64* launches);   // tokens.cu
// frames.cu
cudaError_t frame_lengths(const TokenRec* recs, u64 m, const uint8_t* arena, u64* lens_scan, u64* tmp, int sm, cudaStream_t s,
                          u64* launches);
cudaError_t frame_pack(const TokenRec* recs, u64 m, const uint8_t* arena, const u64* offs, uint8_t* frame, int sm, cudaStream_t s,
                       u64* launches);
cudaError_t frame_read_lens(const uint8_t* frame, u64 m, u64* lens, u64* arena_need, int sm, cudaStream_t s, u64* launches);
cudaError_t frame_build(const uint8_t* frame, u64 m, const u64* offs, const u64* arena_offs, TokenRec* recs, uint8_t* arena,
                        int* flags, int sm, cudaStream_t s, u64* launches);
// analysis.cpp
uint64_t analysis_top_k(const uint8_t* bytes, const uint32_t* lens, const uint64_t* counts, uint64_t n, uint64_t k,
                        uint64_t* out_idx, double* out_rel, uint64_t* total);
uint64_t analysis_distinctive(const uint8_t* t_bytes, const uint32_t* t_lens, const uint64_t* t_counts, uint64_t nt,
                              const uint8_t* o_bytes, const uint32_t* o_lens, const uint64_t* o_counts, uint64_t no,
                              uint64_t k, int32_t* out_src, uint64_t* out_idx, double* out_score);
struct ScoredRow {
    const uint8_t* key;
    uint32_t len;
    uint64_t in_target, in_others, tag;
    double score;
};
uint64_t analysis_rank_rows(std::vector<ScoredRow>& rows, uint64_t vocab, uint64_t t_total, uint64_t o_total, uint64_t k);
// synth.cpp
int synth_document(uint64_t seed, uint64_t doc, uint32_t vocab, double s, uint32_t speaker, uint8_t* out, uint64_t doc_bytes);
int synth_corpus(uint64_t seed, uint64_t doc_begin, uint64_t doc_end, uint32_t vocab, double s, uint32_t speaker,
                 uint64_t doc_bytes, uint8_t* out, int threads);
int synth_corpus_strided(uint64_t seed, uint64_t doc_begin, uint64_t doc_stride, uint64_t n_docs, uint32_t vocab,
                         double s, uint32_t speaker, uint64_t doc_bytes, uint8_t* out, int threads);
int synth_uniform(uint64_t seed, uint64_t n, int as_f64, void* out);
}  // namespace wfcu

using namespace wfcu;

// ---- error plumbing -------------------------------------------------------------
static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}
#define CUDA_TRY(expr)                                                                           \
    do {                                                                                         \
        cudaError_t _e = (expr);                                                                 \
        if (_e != cudaSuccess) return fail(WFCU_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

struct LaunchTally {   // adds to the global launch counter on scope exit
    u64 n = 0;
    ~LaunchTally() { g_launches += n; }
};

// ---- device state -----------------------------------------------------------------
namespace {
// Device-memory cache.  cudaMalloc + cudaFree of the library's buffers cost more host time than the kernels that use
// them -- gigabyte-sized scratch of the token / export paths, but also the 240 MB of a default counter (38 ms per
// create + destroy on the virtualised B200 hosts) and the staging buffer of every *_host call.  Every device
// allocation of the library comes from here: freed blocks are kept (per device, up to kScratchKeepBytes in all,
// WFCU_CACHE_KEEP_MB overrides) and handed out again to requests they fit within a factor of two; an allocation
// that fails gives the cached blocks back to the driver and tries once more.  scratch_free waits for the block's
// device like cudaFree does, so callers keep cudaFree's ordering guarantees; blocks that did not come from here
// (wfcu_dev_free of a foreign pointer) go to cudaFree.
struct ScratchBlock { void* p; size_t bytes; int device; };
std::mutex g_scratch_mu;
std::vector<ScratchBlock> g_scratch_free;
std::vector<ScratchBlock> g_scratch_live;
size_t scratch_keep_bytes() {
    static const size_t keep = [] {
        const char* v = getenv("WFCU_CACHE_KEEP_MB");
        return v ? (size_t)strtoull(v, nullptr, 10) << 20 : size_t(24) << 30;
    }();
    return keep;
}

cudaError_t scratch_alloc(void** out, size_t bytes) {
    if (bytes == 0) bytes = 16;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lock(g_scratch_mu);
        size_t best = g_scratch_free.size();
        for (size_t i = 0; i < g_scratch_free.size(); ++i) {
            const ScratchBlock& b = g_scratch_free[i];
            if (b.device == dev && b.bytes >= bytes && b.bytes <= 2 * bytes + 4096 &&
                (best == g_scratch_free.size() || b.bytes < g_scratch_free[best].bytes))
                best = i;
        }
        if (best != g_scratch_free.size()) {
            *out = g_scratch_free[best].p;
            g_scratch_live.push_back(g_scratch_free[best]);
            g_scratch_free.erase(g_scratch_free.begin() + best);
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaMalloc(out, bytes);
    if (e != cudaSuccess) {   // give the cached blocks back and try once more
        cudaGetLastError();
        std::lock_guard<std::mutex> lock(g_scratch_mu);
        for (const ScratchBlock& b : g_scratch_free) cudaFree(b.p);
        g_scratch_free.clear();
        e = cudaMalloc(out, bytes);
        if (e != cudaSuccess) return e;
    }
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    g_scratch_live.push_back({*out, bytes, dev});
    return cudaSuccess;
}
template <typename T>
cudaError_t scratch_alloc(T** out, size_t bytes) { return scratch_alloc(reinterpret_cast<void**>(out), bytes); }

void scratch_free(void* p) {
    if (!p) return;
    ScratchBlock blk{nullptr, 0, -1};
    {
        std::lock_guard<std::mutex> lock(g_scratch_mu);
        for (size_t i = 0; i < g_scratch_live.size(); ++i) {
            if (g_scratch_live[i].p != p) continue;
            blk = g_scratch_live[i];
            g_scratch_live.erase(g_scratch_live.begin() + i);
            break;
        }
    }
    if (!blk.p) {
        cudaFree(p);                  // not ours
        return;
    }
    int cur = 0;                      // what cudaFree would have done: wait for the device that owns the block
    cudaGetDevice(&cur);
    if (cur != blk.device) cudaSetDevice(blk.device);
    cudaDeviceSynchronize();
    if (cur != blk.device) cudaSetDevice(cur);
    std::vector<void*> release;
    {
        std::lock_guard<std::mutex> lock(g_scratch_mu);
        g_scratch_free.push_back(blk);
        size_t kept = 0;
        for (const ScratchBlock& b : g_scratch_free) kept += b.bytes;
        while (kept > scratch_keep_bytes() && !g_scratch_free.empty()) {   // oldest first
            kept -= g_scratch_free.front().bytes;
            release.push_back(g_scratch_free.front().p);
            g_scratch_free.erase(g_scratch_free.begin());
        }
    }
    for (void* q : release) cudaFree(q);
}


// The same for page-locked host staging (cudaHostAlloc of 2 x 32 MiB costs tens of milliseconds): exact-size reuse,
// at most 1 GiB kept.  A buffer is only released by its counter after the copies out of it have completed.
struct PinnedBlock { void* p; size_t bytes; };
std::vector<PinnedBlock> g_pinned_free;
std::vector<PinnedBlock> g_pinned_live;
cudaError_t pinned_alloc(void** out, size_t bytes) {
    {
        std::lock_guard<std::mutex> lock(g_scratch_mu);
        for (size_t i = 0; i < g_pinned_free.size(); ++i) {
            if (g_pinned_free[i].bytes != bytes) continue;
            *out = g_pinned_free[i].p;
            g_pinned_live.push_back(g_pinned_free[i]);
            g_pinned_free.erase(g_pinned_free.begin() + i);
            return cudaSuccess;
        }
    }
    const cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    g_pinned_live.push_back({*out, bytes});
    return cudaSuccess;
}
void pinned_free(void* p) {
    if (!p) return;
    std::vector<void*> release;
    {
        std::lock_guard<std::mutex> lock(g_scratch_mu);
        for (size_t i = 0; i < g_pinned_live.size(); ++i) {
            if (g_pinned_live[i].p != p) continue;
            g_pinned_free.push_back(g_pinned_live[i]);
            g_pinned_live.erase(g_pinned_live.begin() + i);
            size_t kept = 0;
            for (const PinnedBlock& b : g_pinned_free) kept += b.bytes;
            while (kept > (size_t(1) << 30) && !g_pinned_free.empty()) {
                kept -= g_pinned_free.front().bytes;
                release.push_back(g_pinned_free.front().p);
                g_pinned_free.erase(g_pinned_free.begin());
            }
            p = nullptr;
            break;
        }
    }
    if (p) release.push_back(p);      // not ours
    for (void* q : release) cudaFreeHost(q);
}
}  // namespace

struct DeviceState {
    bool ready = false;
    int sm_count = 0;
    double* mr_partials = nullptr;   // kMrGridMax doubles
    double* mr_out = nullptr;        // device result
    u64* scratch = nullptr;          // 64 u64 of device scratch (counts, cursors)
    void* sn_scratch = nullptr;      // grow-only scratch of utf8_sanitize
    u64 sn_cap = 0;
};
static constexpr int kMaxDevices = 64;
static DeviceState g_dev[kMaxDevices];
static std::mutex g_dev_mu;

static int current_device_state(DeviceState** out) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count <= 0) {
        cudaGetLastError();
        return fail(WFCU_ERR_NO_DEVICE, "no CUDA device available (%s); libwfcu has no CPU path",
                    e == cudaSuccess ? "device count 0" : cudaGetErrorString(e));
    }
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= kMaxDevices) return fail(WFCU_ERR_NO_DEVICE, "device index %d out of range", dev);
    std::lock_guard<std::mutex> lock(g_dev_mu);
    DeviceState& d = g_dev[dev];
    if (!d.ready) {
        cudaDeviceProp prop;
        CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
        if (prop.major != 10)
            return fail(WFCU_ERR_NO_DEVICE, "device %d is sm_%d%d; libwfcu is built for sm_100a only", dev, prop.major,
                        prop.minor);
        d.sm_count = prop.multiProcessorCount;
        CUDA_TRY(cudaMalloc(&d.mr_partials, sizeof(double) * 8192));
        CUDA_TRY(cudaMalloc(&d.mr_out, sizeof(double)));
        CUDA_TRY(cudaMalloc(&d.scratch, sizeof(u64) * 64));
        d.ready = true;
    }
    *out = &d;
    return WFCU_OK;
}

extern "C" const char* wfcu_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* wfcu_version(void) { return "wfcu 0.1 (sm_100a)"; }
extern "C" uint64_t wfcu_launch_count(void) { return g_launches.load(); }

extern "C" int wfcu_device_count(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return count;
}
extern "C" int wfcu_set_device(int device) {
    CUDA_TRY(cudaSetDevice(device));
    return WFCU_OK;
}
extern "C" int wfcu_sm_count(int* out) {
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    *out = d->sm_count;
    return WFCU_OK;
}

// ---- map-then-reduce ----------------------------------------------------------------
static int check_map_args(int dtype, int kind, const void* values, uint64_t n) {
    if (dtype != WFCU_DTYPE_F32 && dtype != WFCU_DTYPE_F64) return fail(WFCU_ERR_INVALID_ARGUMENT, "unknown dtype %d", dtype);
    if (kind < 0 || kind > WFCU_MAP_SQUARE) return fail(WFCU_ERR_INVALID_ARGUMENT, "unknown map kind");
    if (!values && n && kind != WFCU_MAP_ALTERNATING_HARMONIC_TERM)
        return fail(WFCU_ERR_INVALID_ARGUMENT, "values is null");
    if (values && (reinterpret_cast<uintptr_t>(values) & 15u))
        return fail(WFCU_ERR_INVALID_ARGUMENT, "device values must be 16-byte aligned");
    return WFCU_OK;
}

// NOT re-entrant per device: the per-CTA partials live in one buffer per device (and the synchronous forms share one
// result word), so two reductions of one device must not be in flight at the same time -- neither on two streams nor
// from two host threads.  include/wfcu.h says so; callers that need overlap serialise on their side.
extern "C" int wfcu_map_reduce_dev_async(const void* dev_values, int dtype, uint64_t n, uint64_t position_base,
                                         int map_kind, void* stream, double* dev_out) {
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (int rc = check_map_args(dtype, map_kind, dev_values, n)) return rc;
    if (!dev_out) return fail(WFCU_ERR_INVALID_ARGUMENT, "dev_out is null");
    // grid: a multiple of the SM count, never more CTAs than 16-byte vectors need
    const u64 vec = (dtype == WFCU_DTYPE_F64) ? 2 : 4;
    u64 want = (n / vec + 256 * 4 - 1) / (256 * 4);
    int grid = d->sm_count * 8;
    if (map_kind == WFCU_MAP_ALTERNATING_HARMONIC_TERM) want = (n + 255) / 256;
    if ((u64)grid > want) grid = (int)std::max<u64>(1, want);
    LaunchTally tally;
    CUDA_TRY(mr_launch(dev_values, dtype == WFCU_DTYPE_F64, n, position_base, map_kind, grid, d->mr_partials, dev_out,
                       (cudaStream_t)stream, &tally.n));
    return WFCU_OK;
}

extern "C" int wfcu_map_reduce_dev(const void* dev_values, int dtype, uint64_t n, uint64_t position_base, int map_kind,
                                   void* stream, double* out) {
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    if (int rc = wfcu_map_reduce_dev_async(dev_values, dtype, n, position_base, map_kind, stream, d->mr_out)) return rc;
    CUDA_TRY(cudaMemcpyAsync(out, d->mr_out, sizeof(double), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    return WFCU_OK;
}

extern "C" int wfcu_map_reduce_blocked_dev(const void* dev_values, int dtype, uint64_t n, uint64_t position_base,
                                           int map_kind, uint64_t block_size, void* stream, double* out) {
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (block_size == 0) return fail(WFCU_ERR_INVALID_ARGUMENT, "block_size and workers must be >= 1");
    if (int rc = check_map_args(dtype, map_kind, dev_values, n)) return rc;
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    const u64 nb = (n + block_size - 1) / block_size;
    double *a = nullptr, *b = nullptr;
    CUDA_TRY(scratch_alloc(&a, sizeof(double) * std::max<u64>(nb, 1)));
    if (scratch_alloc(&b, sizeof(double) * std::max<u64>(nb / 2 + 1, 1)) != cudaSuccess) {
        scratch_free(a);
        return fail(WFCU_ERR_CUDA, "cudaMalloc of the partials failed");
    }
    LaunchTally tally;
    cudaError_t e = mr_blocked_launch(dev_values, dtype == WFCU_DTYPE_F64, n, position_base, map_kind, block_size, a, b,
                                      d->mr_out, d->sm_count, (cudaStream_t)stream, &tally.n);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d->mr_out, sizeof(double), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    scratch_free(a);
    scratch_free(b);
    if (e != cudaSuccess) return fail(WFCU_ERR_CUDA, "blocked map-reduce: %s", cudaGetErrorString(e));
    return WFCU_OK;
}

static int upload(const void* host, uint64_t bytes, void** dev) {
    *dev = nullptr;
    if (bytes == 0) return WFCU_OK;
    // + 16: the tokenizer's last chunk is fetched with cp.async src-size < 16 (only the bytes below n are read, but
    // compute-sanitizer checks the full 16) -- keep the whole chunk inside the allocation
    CUDA_TRY(scratch_alloc(dev, bytes + 16));
    cudaError_t e = cudaMemcpy(*dev, host, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        scratch_free(*dev);
        *dev = nullptr;
        return fail(WFCU_ERR_CUDA, "H2D copy: %s", cudaGetErrorString(e));
    }
    return WFCU_OK;
}

extern "C" int wfcu_map_reduce_host(const void* host_values, int dtype, uint64_t n, int map_kind, double* out) {
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (!host_values && n && map_kind != WFCU_MAP_ALTERNATING_HARMONIC_TERM)
        return fail(WFCU_ERR_INVALID_ARGUMENT, "values is null");
    void* dev = nullptr;
    const uint64_t esz = dtype == WFCU_DTYPE_F64 ? 8 : 4;
    if (map_kind != WFCU_MAP_ALTERNATING_HARMONIC_TERM)
        if (int rc = upload(host_values, n * esz, &dev)) return rc;
    const int rc = wfcu_map_reduce_dev(dev, dtype, n, 0, map_kind, nullptr, out);
    scratch_free(dev);
    return rc;
}

extern "C" int wfcu_map_reduce_blocked_host(const void* host_values, int dtype, uint64_t n, int map_kind,
                                            uint64_t block_size, double* out) {
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (block_size == 0) return fail(WFCU_ERR_INVALID_ARGUMENT, "block_size and workers must be >= 1");
    if (!host_values && n && map_kind != WFCU_MAP_ALTERNATING_HARMONIC_TERM)
        return fail(WFCU_ERR_INVALID_ARGUMENT, "values is null");
    void* dev = nullptr;
    const uint64_t esz = dtype == WFCU_DTYPE_F64 ? 8 : 4;
    if (map_kind != WFCU_MAP_ALTERNATING_HARMONIC_TERM)
        if (int rc = upload(host_values, n * esz, &dev)) return rc;
    const int rc = wfcu_map_reduce_blocked_dev(dev, dtype, n, 0, map_kind, block_size, nullptr, out);
    scratch_free(dev);
    return rc;
}

extern "C" int wfcu_alternating_harmonic(uint64_t n, uint64_t block_size, double* out) {
    return wfcu_map_reduce_blocked_dev(nullptr, WFCU_DTYPE_F64, n, 0, WFCU_MAP_ALTERNATING_HARMONIC_TERM, block_size,
                                       nullptr, out);
}

// ---- counter ------------------------------------------------------------------------
struct wfcu_counter {
    int device = 0;
    int sm_count = 0;
    TableView v{};
    u64 table_slots = 0, long_slots = 0;
    u64* counters = nullptr;    // device: [0] n_used [1] n_tokens [2] n_deferred [3] n_long [4] arena_used
                                //         [5] status(int) [6..15] scratch [16] CTA ticket of the reset kernel
    bool aux_clean = false;     // the long table and the counters have been initialised once
    u32 variant_hint = 63;       // kernel variants the texts counted so far asked for (counters[17]), read at every
                                // synchronising call: later counts launch only those (and the narrow one)
    u32* wanted_host = nullptr; // page-locked mirror of counters[17]: copied back (asynchronously, never waited for)
                                // after the first two counts and every 64th, so that callers who never make a
                                // synchronising call stop paying for the kernels their texts do not use
    u64 count_calls = 0;
    // host staging for count_host
    uint8_t* pinned[2] = {nullptr, nullptr};
    uint8_t* devbuf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    u64 chunk_cap = 0;
    cudaStream_t stream = nullptr;
    // device staging for the DMA path of count_host (pinned, adjacent documents)
    uint8_t* dma_buf[2] = {nullptr, nullptr};
    cudaEvent_t copied[2] = {nullptr, nullptr}, counted[2] = {nullptr, nullptr};
    u64 dma_cap = 0;
    cudaStream_t copy_stream = nullptr;
    // grow-only scratch of the ordered export (no cudaMalloc per call)
    void* ex_buf[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    u64 ex_cap[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // optional CUDA-event timing of the dominant kernel (bench.py's roofline leg)
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;   // one pair per wc_fast launch
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> event_pool;
};

static u64 round_pow2(u64 x) {
    u64 p = 1;
    while (p < x) p <<= 1;
    return p;
}

static void counter_free(wfcu_counter* c) {
    if (!c) return;
    {   // nothing of this counter may still be running when its buffers go back to the caches
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != c->device) cudaSetDevice(c->device);
        cudaDeviceSynchronize();
        if (cur != c->device) cudaSetDevice(cur);
    }
    scratch_free(c->v.slots);
    scratch_free(c->v.deferred);
    scratch_free(c->v.long_ref);
    scratch_free(c->v.long_count);
    scratch_free(c->v.arena);
    scratch_free(c->counters);
    pinned_free(c->wanted_host);
    for (int i = 0; i < 2; ++i) {
        if (c->pinned[i]) pinned_free(c->pinned[i]);
        if (c->devbuf[i]) scratch_free(c->devbuf[i]);
        if (c->done[i]) cudaEventDestroy(c->done[i]);
    }
    for (int i = 0; i < 2; ++i) {
        if (c->dma_buf[i]) scratch_free(c->dma_buf[i]);
        if (c->copied[i]) cudaEventDestroy(c->copied[i]);
        if (c->counted[i]) cudaEventDestroy(c->counted[i]);
    }
    for (void* b : c->ex_buf) if (b) scratch_free(b);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->stream) cudaStreamDestroy(c->stream);
    for (auto& pr : c->timed) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    for (auto& pr : c->event_pool) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    delete c;
}

extern "C" int wfcu_counter_reset(wfcu_counter* c, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(c->v.slots, 0, sizeof(Slot) * c->table_slots, s));
    if (!c->aux_clean) {      // first reset: the long table and the counters are raw memory
        CUDA_TRY(cudaMemsetAsync(c->v.long_ref, 0, sizeof(u64) * c->long_slots, s));
        CUDA_TRY(cudaMemsetAsync(c->v.long_count, 0, sizeof(u64) * c->long_slots, s));
        CUDA_TRY(cudaMemsetAsync(c->counters, 0, sizeof(u64) * 18, s));
        const u64 arena_start = 8;   // offset 0 means "empty"
        CUDA_TRY(cudaMemcpyAsync(c->v.arena_used, &arena_start, sizeof(u64), cudaMemcpyHostToDevice, s));
        c->aux_clean = true;
        return WFCU_OK;
    }
    // afterwards one small kernel: clears the long table only if it holds something, then the counters
    LaunchTally tally;
    CUDA_TRY(tb_reset_aux(c->v, c->counters, reinterpret_cast<unsigned int*>(c->counters + 16), c->sm_count, s, &tally.n));
    return WFCU_OK;
}

extern "C" int wfcu_counter_create(wfcu_counter** out, const wfcu_counter_config* cfg) {
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    wfcu_counter_config k{};
    if (cfg) k = *cfg;
    auto* c = new wfcu_counter;
    cudaGetDevice(&c->device);
    c->sm_count = d->sm_count;
    c->table_slots = round_pow2(k.table_slots ? std::max<u64>(k.table_slots, 1024) : (1ull << 22));
    c->long_slots = round_pow2(k.long_slots ? std::max<u64>(k.long_slots, 1024) : (1ull << 20));
    const u64 deferred = k.deferred_slots ? k.deferred_slots : (1ull << 22);
    const u64 arena = k.arena_bytes ? std::max<u64>(k.arena_bytes, 4096) : (64ull << 20);
    cudaError_t e = cudaSuccess;
    auto alloc = [&](void** p, u64 bytes) {
        if (e == cudaSuccess) e = scratch_alloc(p, bytes);
    };
    alloc((void**)&c->v.slots, sizeof(Slot) * c->table_slots);
    alloc((void**)&c->v.deferred, sizeof(u64) * deferred);
    alloc((void**)&c->v.long_ref, sizeof(u64) * c->long_slots);
    alloc((void**)&c->v.long_count, sizeof(u64) * c->long_slots);
    alloc((void**)&c->v.arena, arena);
    alloc((void**)&c->counters, sizeof(u64) * 18);
    if (e == cudaSuccess && pinned_alloc((void**)&c->wanted_host, 64) == cudaSuccess) *c->wanted_host = 0;
    if (e != cudaSuccess) {
        counter_free(c);
        return fail(WFCU_ERR_CUDA, "counter allocation: %s", cudaGetErrorString(e));
    }
    c->v.mask = c->table_slots - 1;
    c->v.max_used = c->table_slots / 10 * 7;
    c->v.n_used = c->counters + 0;
    c->v.n_tokens = c->counters + 1;
    c->v.n_deferred = c->counters + 2;
    c->v.n_long = c->counters + 3;
    c->v.arena_used = c->counters + 4;
    c->v.status = reinterpret_cast<int*>(c->counters + 5);
    c->v.ticket = reinterpret_cast<unsigned int*>(c->counters + 16);
    c->v.wanted = reinterpret_cast<unsigned int*>(c->counters + 17);
    c->v.deferred_cap = deferred;
    c->v.long_mask = c->long_slots - 1;
    c->v.arena_cap = arena;
    if (int rc = wfcu_counter_reset(c, nullptr)) {
        counter_free(c);
        return rc;
    }
    if (cudaStreamSynchronize(nullptr) != cudaSuccess) {
        counter_free(c);
        return fail(WFCU_ERR_CUDA, "counter reset failed");
    }
    *out = c;
    return WFCU_OK;
}

extern "C" void wfcu_counter_destroy(wfcu_counter* c) {
    if (c) cudaSetDevice(c->device);
    counter_free(c);
}

extern "C" int wfcu_counter_count_dev(wfcu_counter* c, const uint8_t* dev_text, uint64_t n, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (n == 0) return WFCU_OK;
    if (!dev_text) return fail(WFCU_ERR_INVALID_ARGUMENT, "text is null");
    if (reinterpret_cast<uintptr_t>(dev_text) & 15u)
        return fail(WFCU_ERR_INVALID_ARGUMENT, "device text must be 16-byte aligned");
    if (n >= (1ull << 40)) return fail(WFCU_ERR_INVALID_ARGUMENT, "one call counts at most 2^40 bytes; split the buffer at whitespace");
    LaunchTally tally;
    cudaEvent_t* ev0 = nullptr;
    cudaEvent_t* ev1 = nullptr;
    if (c->timing) {
        std::pair<cudaEvent_t, cudaEvent_t> pr{nullptr, nullptr};
        if (!c->event_pool.empty()) {
            pr = c->event_pool.back();
            c->event_pool.pop_back();
        } else {
            CUDA_TRY(cudaEventCreate(&pr.first));
            CUDA_TRY(cudaEventCreate(&pr.second));
        }
        c->timed.push_back(pr);
        ev0 = &c->timed.back().first;
        ev1 = &c->timed.back().second;
    }
    if (c->wanted_host) {
        const u32 seen = *reinterpret_cast<volatile u32*>(c->wanted_host);     // whatever has landed so far; speed only
        if (seen) c->variant_hint = seen | 1u;
    }
    CUDA_TRY(wc_launch(dev_text, n, c->v, c->sm_count, (cudaStream_t)stream, &tally.n, ev0, ev1, c->variant_hint));
    if (c->wanted_host && (c->count_calls < 2 || (c->count_calls & 63u) == 0))
        CUDA_TRY(cudaMemcpyAsync(c->wanted_host, c->v.wanted, sizeof(u32), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    c->count_calls += 1;
    return WFCU_OK;
}

extern "C" int wfcu_counter_set_timing(wfcu_counter* c, int enabled) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    c->timing = enabled != 0;
    return WFCU_OK;
}

extern "C" int wfcu_counter_take_kernel_ms(wfcu_counter* c, double* sum_ms, uint64_t* launches) {
    if (!c || !sum_ms || !launches) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    double total = 0.0;
    for (auto& pr : c->timed) {
        CUDA_TRY(cudaEventSynchronize(pr.second));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, pr.first, pr.second));
        total += ms;
    }
    *sum_ms = total;
    *launches = c->timed.size();
    for (auto& pr : c->timed) c->event_pool.push_back(pr);
    c->timed.clear();
    return WFCU_OK;
}

static int status_to_rc(int st) {
    if (st & kStatusTableFull) return fail(WFCU_ERR_TABLE_FULL, "count table over its load limit; recreate with more table_slots");
    if (st & kStatusDeferredFull) return fail(WFCU_ERR_DEFERRED_FULL, "slow-path fragment list full; recreate with more deferred_slots");
    if (st & (kStatusArenaFull | kStatusLongFull)) return fail(WFCU_ERR_ARENA_FULL, "long-token arena/table full; recreate with more arena_bytes / long_slots");
    if (st & kStatusNotSorted) return fail(WFCU_ERR_NOT_SORTED, "reduce_sorted: word list must be sorted");
    return WFCU_OK;
}

extern "C" int wfcu_counter_status(wfcu_counter* c, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    int st = 0;
    u32 wanted = 0;
    CUDA_TRY(cudaMemcpyAsync(&st, c->v.status, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CUDA_TRY(cudaMemcpyAsync(&wanted, c->v.wanted, sizeof(u32), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    if (wanted) c->variant_hint = wanted | 1u;
    return status_to_rc(st);
}

extern "C" int wfcu_counter_stats(wfcu_counter* c, void* stream, uint64_t* distinct, uint64_t* total_tokens,
                                  uint64_t* key_bytes) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    cudaStream_t s = (cudaStream_t)stream;
    LaunchTally tally;
    CUDA_TRY(tb_key_bytes(c->v, c->counters + 6, c->sm_count, s, &tally.n));
    u64 h[8];
    u32 wanted = 0;
    CUDA_TRY(cudaMemcpyAsync(h, c->counters, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&wanted, c->v.wanted, sizeof(u32), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (wanted) c->variant_hint = wanted | 1u;
    if (int rc = status_to_rc((int)(h[5] & 0xFFFFFFFFu))) return rc;
    if (distinct) *distinct = h[0] + h[3];
    if (total_tokens) *total_tokens = h[1];
    if (key_bytes) *key_bytes = h[6];
    return WFCU_OK;
}

namespace {
struct DevBuf {   // RAII device scratch
    void* p = nullptr;
    cudaError_t alloc(size_t bytes) { return scratch_alloc(&p, bytes); }
    ~DevBuf() { scratch_free(p); }
    template <typename T> T* as() { return static_cast<T*>(p); }
};
}  // namespace

namespace {
struct HostEntry {
    std::string key;
    u64 count;
};
}

// Pulls every (word, count) pair to the host in std::map order.  The inline keys (the
// bulk) are ordered on the device by the radix sort of tokens.cu; the rare long tokens
// are ordered on the host and merged in.
static int counter_pull_sorted(wfcu_counter* c, cudaStream_t s, std::vector<HostEntry>* out) {
    u64 h[8];
    CUDA_TRY(cudaMemcpyAsync(h, c->counters, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (int rc = status_to_rc((int)(h[5] & 0xFFFFFFFFu))) return rc;
    const u64 n_inline = h[0], n_long = h[3], arena_used = h[4];
    out->clear();
    out->reserve(n_inline + n_long);
    LaunchTally tally;
    std::vector<TokenRec> hs(n_inline);
    if (n_inline) {
        DevBuf dense, alt, hist, tmp;
        const u64 hw = sort_hist_words(n_inline);
        CUDA_TRY(dense.alloc(sizeof(TokenRec) * n_inline));
        CUDA_TRY(alt.alloc(sizeof(TokenRec) * n_inline));
        CUDA_TRY(hist.alloc(sizeof(u64) * hw));
        CUDA_TRY(tmp.alloc(sizeof(u64) * scan_tmp_words(hw)));
        CUDA_TRY(tb_compact_recs(c->v, dense.as<TokenRec>(), n_inline, c->counters + 7, c->sm_count, s, &tally.n));
        SortScratch sc{alt.as<TokenRec>(), hist.as<u64>(), tmp.as<u64>()};
        CUDA_TRY(tokens_sort(dense.as<TokenRec>(), n_inline, /*by_position=*/false, nullptr, sc, c->sm_count, s, &tally.n));
        CUDA_TRY(cudaMemcpyAsync(hs.data(), dense.p, sizeof(TokenRec) * n_inline, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    std::vector<HostEntry> longs;
    if (n_long) {
        std::vector<u64> refs(c->long_slots), counts(c->long_slots);
        std::vector<uint8_t> arena(arena_used);
        CUDA_TRY(cudaMemcpyAsync(refs.data(), c->v.long_ref, sizeof(u64) * c->long_slots, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(counts.data(), c->v.long_count, sizeof(u64) * c->long_slots, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(arena.data(), c->v.arena, arena_used, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (u64 i = 0; i < c->long_slots; ++i) {
            if (!refs[i]) continue;
            u32 len;
            std::memcpy(&len, arena.data() + refs[i], 4);
            longs.push_back({std::string(reinterpret_cast<const char*>(arena.data() + refs[i] + 8), len), counts[i]});
        }
        std::sort(longs.begin(), longs.end(), [](const HostEntry& a, const HostEntry& b) { return a.key < b.key; });
    }
    // merge the two ordered lists (std::string::compare is unsigned byte-wise = map order)
    size_t li = 0;
    for (const TokenRec& r : hs) {
        uint8_t b[16];
        key_to_bytes(r.k0, r.k1, b);
        std::string key(reinterpret_cast<const char*>(b), key_len(r.k0, r.k1));
        while (li < longs.size() && longs[li].key < key) out->push_back(std::move(longs[li++]));
        out->push_back({std::move(key), r.pos});
    }
    while (li < longs.size()) out->push_back(std::move(longs[li++]));
    return WFCU_OK;
}

// grow-only device scratch of the counter (slot i), so that an export allocates nothing in steady state
static int ex_reserve(wfcu_counter* c, int i, u64 bytes) {
    if (c->ex_cap[i] >= bytes) return WFCU_OK;
    if (c->ex_buf[i]) scratch_free(c->ex_buf[i]);
    c->ex_buf[i] = nullptr;
    c->ex_cap[i] = 0;
    const u64 want = std::max<u64>(bytes + bytes / 4, 4096);
    CUDA_TRY(scratch_alloc(&c->ex_buf[i], want));
    c->ex_cap[i] = want;
    return WFCU_OK;
}

extern "C" int wfcu_counter_export(wfcu_counter* c, void* stream, uint8_t* key_bytes, uint64_t key_bytes_cap,
                                   uint32_t* key_lens, uint64_t* counts, uint64_t entries_cap) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    cudaStream_t s = (cudaStream_t)stream;
    u64 h[8];
    CUDA_TRY(cudaMemcpyAsync(h, c->counters, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (int rc = status_to_rc((int)(h[5] & 0xFFFFFFFFu))) return rc;
    const u64 n = h[0], n_long = h[3];
    if (n_long == 0) {
        // The usual case (no token longer than 16 bytes): order AND pack on the device -- compaction,
        // radix sort by key, key lengths, scan, byte pack -- then three copies into the caller's arrays.
        if (n > entries_cap)
            return fail(WFCU_ERR_BUFFER_TOO_SMALL, "export needs %llu entries", (unsigned long long)n);
        if (n == 0) return WFCU_OK;
        const u64 hw = sort_hist_words(n);
        const u64 tmp_words = std::max(scan_tmp_words(hw), scan_tmp_words(n));
        const u64 need[8] = {sizeof(TokenRec) * n, sizeof(TokenRec) * n, sizeof(u64) * hw, sizeof(u64) * tmp_words,
                             16, sizeof(u64) * n, 16 * n, 12 * n};
        for (int i = 0; i < 8; ++i)
            if (int rc = ex_reserve(c, i, need[i])) return rc;
        TokenRec* dense = static_cast<TokenRec*>(c->ex_buf[0]);
        SortScratch sc{static_cast<TokenRec*>(c->ex_buf[1]), static_cast<u64*>(c->ex_buf[2]),
                       static_cast<u64*>(c->ex_buf[3])};
        uint8_t* d_bytes = static_cast<uint8_t*>(c->ex_buf[6]);
        u64* d_counts = static_cast<u64*>(c->ex_buf[7]);
        u32* d_lens = reinterpret_cast<u32*>(d_counts + n);
        LaunchTally tally;
        CUDA_TRY(tb_compact_recs(c->v, dense, n, c->counters + 7, c->sm_count, s, &tally.n));
        CUDA_TRY(tokens_sort(dense, n, /*by_position=*/false, nullptr, sc, c->sm_count, s, &tally.n));
        CUDA_TRY(tb_export_pack(dense, n, static_cast<u64*>(c->ex_buf[5]), static_cast<u64*>(c->ex_buf[3]), d_bytes, d_lens,
                                d_counts, c->counters + 10, c->sm_count, s, &tally.n));
        u64 total_bytes = 0;
        CUDA_TRY(cudaMemcpyAsync(&total_bytes, c->counters + 10, sizeof(u64), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(key_lens, d_lens, sizeof(u32) * n, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(counts, d_counts, sizeof(u64) * n, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (total_bytes > key_bytes_cap)
            return fail(WFCU_ERR_BUFFER_TOO_SMALL, "export needs %llu key bytes", (unsigned long long)total_bytes);
        CUDA_TRY(cudaMemcpyAsync(key_bytes, d_bytes, total_bytes, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return WFCU_OK;
    }
    std::vector<HostEntry> rows;
    if (int rc = counter_pull_sorted(c, (cudaStream_t)stream, &rows)) return rc;
    u64 total_bytes = 0;
    for (const auto& r : rows) total_bytes += r.key.size();
    if (rows.size() > entries_cap || total_bytes > key_bytes_cap)
        return fail(WFCU_ERR_BUFFER_TOO_SMALL, "export needs %llu entries / %llu key bytes",
                    (unsigned long long)rows.size(), (unsigned long long)total_bytes);
    u64 off = 0;
    for (size_t i = 0; i < rows.size(); ++i) {
        std::memcpy(key_bytes + off, rows[i].key.data(), rows[i].key.size());
        off += rows[i].key.size();
        key_lens[i] = (u32)rows[i].key.size();
        counts[i] = rows[i].count;
    }
    return WFCU_OK;
}

// top_k straight from the device table (proj/src/analysis.cpp:58-75): the compacted slots are
// ordered by count on the device, the count of the k-th row is the threshold, and only rows at
// or above it (ties included) come back to be put in the reference's exact order.
extern "C" int wfcu_counter_top_k(wfcu_counter* c, uint64_t k, void* stream, uint8_t* key_bytes, uint64_t key_bytes_cap,
                                  uint32_t* key_lens, uint64_t* counts, double* rel_freq, uint64_t rows_cap,
                                  uint64_t* n_rows, uint64_t* total_words) {
    if (!c || !n_rows || !total_words) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    u64 h[8];
    CUDA_TRY(cudaMemcpyAsync(h, c->counters, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (int rc = status_to_rc((int)(h[5] & 0xFFFFFFFFu))) return rc;
    const u64 n_inline = h[0], n_long = h[3], arena_used = h[4];
    *total_words = h[1];
    *n_rows = 0;
    std::vector<HostEntry> cand;
    LaunchTally tally;
    if (n_inline && k) {
        DevBuf dense, alt, hist, tmp;
        const u64 hw = sort_hist_words(n_inline);
        CUDA_TRY(dense.alloc(sizeof(TokenRec) * n_inline));
        CUDA_TRY(alt.alloc(sizeof(TokenRec) * n_inline));
        CUDA_TRY(hist.alloc(sizeof(u64) * hw));
        CUDA_TRY(tmp.alloc(sizeof(u64) * scan_tmp_words(hw)));
        CUDA_TRY(tb_compact_recs(c->v, dense.as<TokenRec>(), n_inline, c->counters + 7, c->sm_count, s, &tally.n));
        SortScratch sc{alt.as<TokenRec>(), hist.as<u64>(), tmp.as<u64>()};
        CUDA_TRY(tokens_sort(dense.as<TokenRec>(), n_inline, /*by_position=*/true, nullptr, sc, c->sm_count, s, &tally.n));
        // threshold = count of the k-th largest inline row (long rows can only push it up)
        const u64 kth = n_inline > k ? n_inline - k : 0;
        TokenRec pivot;
        CUDA_TRY(cudaMemcpyAsync(&pivot, dense.as<TokenRec>() + kth, sizeof(TokenRec), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        CUDA_TRY(tb_lower_bound_pos(dense.as<TokenRec>(), n_inline, pivot.pos, c->counters + 9, s, &tally.n));
        u64 first = 0;
        CUDA_TRY(cudaMemcpyAsync(&first, c->counters + 9, sizeof(u64), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        std::vector<TokenRec> hs(n_inline - first);
        CUDA_TRY(cudaMemcpyAsync(hs.data(), dense.as<TokenRec>() + first, sizeof(TokenRec) * hs.size(), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (const TokenRec& r : hs) {
            uint8_t b[16];
            key_to_bytes(r.k0, r.k1, b);
            cand.push_back({std::string(reinterpret_cast<const char*>(b), key_len(r.k0, r.k1)), r.pos});
        }
    }
    if (n_long && k) {   // rare: every long row is a candidate
        std::vector<u64> refs(c->long_slots), cnts(c->long_slots);
        std::vector<uint8_t> arena(arena_used);
        CUDA_TRY(cudaMemcpyAsync(refs.data(), c->v.long_ref, sizeof(u64) * c->long_slots, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(cnts.data(), c->v.long_count, sizeof(u64) * c->long_slots, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(arena.data(), c->v.arena, arena_used, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (u64 i = 0; i < c->long_slots; ++i) {
            if (!refs[i]) continue;
            u32 len;
            std::memcpy(&len, arena.data() + refs[i], 4);
            cand.push_back({std::string(reinterpret_cast<const char*>(arena.data() + refs[i] + 8), len), cnts[i]});
        }
    }
    const u64 keep = std::min<u64>(k, cand.size());
    std::partial_sort(cand.begin(), cand.begin() + keep, cand.end(), [](const HostEntry& a, const HostEntry& b) {
        return a.count != b.count ? a.count > b.count : a.key < b.key;
    });
    u64 off = 0;
    if (keep > rows_cap) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "top_k needs %llu rows", (unsigned long long)keep);
    for (u64 r = 0; r < keep; ++r) {
        if (off + cand[r].key.size() > key_bytes_cap) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "top_k key buffer too small");
        std::memcpy(key_bytes + off, cand[r].key.data(), cand[r].key.size());
        off += cand[r].key.size();
        key_lens[r] = (u32)cand[r].key.size();
        counts[r] = cand[r].count;
        rel_freq[r] = double(cand[r].count) / double(*total_words);
    }
    *n_rows = keep;
    return WFCU_OK;
}

// the long-token table of a counter (rare) as host strings
static int counter_pull_long(wfcu_counter* c, u64 arena_used, cudaStream_t s, std::vector<HostEntry>* out) {
    std::vector<u64> refs(c->long_slots), cnts(c->long_slots);
    std::vector<uint8_t> arena(arena_used);
    CUDA_TRY(cudaMemcpyAsync(refs.data(), c->v.long_ref, sizeof(u64) * c->long_slots, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(cnts.data(), c->v.long_count, sizeof(u64) * c->long_slots, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(arena.data(), c->v.arena, arena_used, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (u64 i = 0; i < c->long_slots; ++i) {
        if (!refs[i]) continue;
        u32 len;
        std::memcpy(&len, arena.data() + refs[i], 4);
        out->push_back({std::string(reinterpret_cast<const char*>(arena.data() + refs[i] + 8), len), cnts[i]});
    }
    return WFCU_OK;
}

static inline double sort_key_to_double(u64 key) {
    const u64 b = (key >> 63) ? (key ^ 0x8000000000000000ull) : ~key;
    double v;
    std::memcpy(&v, &b, 8);
    return v;
}
static inline u64 double_to_sort_key(double v) {
    u64 b;
    std::memcpy(&b, &v, 8);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// distinctive_words (proj/src/analysis.cpp:77-132; cli.cpp:213-221) on two device-resident tables.
//   1. the union of the two tables as dense rows {word, count in target, count in others}: every slot of one table
//      probes the other (tb_union_rows), which also gives the size V of the union vocabulary;
//   2. a score per row on the device and a radix sort by it;
//   3. only the rows whose device score is within 1e-9 of the k-th best are downloaded (the device's log may differ
//      from the host's in the last bits; ties are exact, they share both counts) and ranked by
//      analysis_rank_rows: the reference's expression in host doubles, score descending by exact compare, word
//      ascending.  Tokens longer than 16 bytes (rare) are joined and scored on the host.
extern "C" int wfcu_counter_distinctive(wfcu_counter* target, wfcu_counter* others, uint64_t k, void* stream,
                                        uint8_t* key_bytes, uint64_t key_bytes_cap, uint32_t* key_lens, double* scores,
                                        uint64_t rows_cap, uint64_t* n_rows) {
    if (!target || !others || !n_rows) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    if (target->device != others->device) return fail(WFCU_ERR_INVALID_ARGUMENT, "the two tables live on different devices");
    cudaStream_t s = (cudaStream_t)stream;
    u64 ht[8], ho[8];
    CUDA_TRY(cudaMemcpyAsync(ht, target->counters, sizeof(ht), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(ho, others->counters, sizeof(ho), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (int rc = status_to_rc((int)(ht[5] & 0xFFFFFFFFu))) return rc;
    if (int rc = status_to_rc((int)(ho[5] & 0xFFFFFFFFu))) return rc;
    *n_rows = 0;
    const u64 t_total = ht[1], o_total = ho[1];
    // long tokens: joined here
    std::vector<HostEntry> lt, lo;
    if (ht[3]) { if (int rc = counter_pull_long(target, ht[4], s, &lt)) return rc; }
    if (ho[3]) { if (int rc = counter_pull_long(others, ho[4], s, &lo)) return rc; }
    std::map<std::string, std::pair<u64, u64>> longs;
    for (const auto& e : lt) longs[e.key].first += e.count;
    for (const auto& e : lo) longs[e.key].second += e.count;

    const u64 cap = ht[0] + ho[0];
    std::vector<TokenRec> cand;
    std::vector<u64> cand_ct, cand_co;
    u64 n_union = 0;
    LaunchTally tally;
    if (cap) {
        DevBuf recs, alt, ct, co, hist, tmp, oct, oco;
        const u64 hw = sort_hist_words(cap);
        CUDA_TRY(recs.alloc(sizeof(TokenRec) * cap));
        CUDA_TRY(alt.alloc(sizeof(TokenRec) * cap));
        CUDA_TRY(ct.alloc(sizeof(u64) * cap));
        CUDA_TRY(co.alloc(sizeof(u64) * cap));
        CUDA_TRY(hist.alloc(sizeof(u64) * hw));
        CUDA_TRY(tmp.alloc(sizeof(u64) * scan_tmp_words(hw)));
        u64* cursor = target->counters + 10;     // [10] rows of the union, [11] words in both tables
        CUDA_TRY(tb_union_rows(target->v, others->v, recs.as<TokenRec>(), ct.as<u64>(), co.as<u64>(), cap, cursor,
                               target->sm_count, s, &tally.n));
        CUDA_TRY(tb_score_rows(recs.as<TokenRec>(), ct.as<u64>(), co.as<u64>(), cursor, cap, longs.size(), t_total, o_total,
                               target->sm_count, s, &tally.n));
        CUDA_TRY(cudaMemcpyAsync(&n_union, cursor, sizeof(u64), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (n_union && k) {
            SortScratch sc{alt.as<TokenRec>(), hist.as<u64>(), tmp.as<u64>()};
            CUDA_TRY(tokens_sort(recs.as<TokenRec>(), n_union, /*by_position=*/true, nullptr, sc, target->sm_count, s, &tally.n));
            const u64 kth = n_union > k ? n_union - k : 0;
            TokenRec pivot;
            CUDA_TRY(cudaMemcpyAsync(&pivot, recs.as<TokenRec>() + kth, sizeof(TokenRec), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            const double thr = sort_key_to_double(pivot.pos);
            const double low = thr - 1e-9 * std::max(1.0, std::fabs(thr));
            CUDA_TRY(tb_lower_bound_pos(recs.as<TokenRec>(), n_union, double_to_sort_key(low), target->counters + 9, s, &tally.n));
            u64 first = 0;
            CUDA_TRY(cudaMemcpyAsync(&first, target->counters + 9, sizeof(u64), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            const u64 m = n_union - first;
            CUDA_TRY(oct.alloc(sizeof(u64) * m));
            CUDA_TRY(oco.alloc(sizeof(u64) * m));
            CUDA_TRY(tb_gather_counts(recs.as<TokenRec>(), first, n_union, ct.as<u64>(), co.as<u64>(), oct.as<u64>(), oco.as<u64>(),
                                      target->sm_count, s, &tally.n));
            cand.resize(m); cand_ct.resize(m); cand_co.resize(m);
            CUDA_TRY(cudaMemcpyAsync(cand.data(), recs.as<TokenRec>() + first, sizeof(TokenRec) * m, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(cand_ct.data(), oct.p, sizeof(u64) * m, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(cand_co.data(), oco.p, sizeof(u64) * m, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
        }
    }
    // exact ranking on the host: the candidates and every long row
    std::vector<uint8_t> keybuf(16 * cand.size());
    std::vector<ScoredRow> rows;
    rows.reserve(cand.size() + longs.size());
    for (size_t i = 0; i < cand.size(); ++i) {
        key_to_bytes(cand[i].k0, cand[i].k1, keybuf.data() + 16 * i);
        rows.push_back({keybuf.data() + 16 * i, key_len(cand[i].k0, cand[i].k1), cand_ct[i], cand_co[i], 0, 0.0});
    }
    for (const auto& kv : longs)
        rows.push_back({reinterpret_cast<const uint8_t*>(kv.first.data()), (uint32_t)kv.first.size(), kv.second.first, kv.second.second, 1, 0.0});
    const u64 keep = analysis_rank_rows(rows, n_union + longs.size(), t_total, o_total, k);
    if (keep > rows_cap) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "distinctive needs %llu rows", (unsigned long long)keep);
    u64 off = 0;
    for (u64 r = 0; r < keep; ++r) {
        if (off + rows[r].len > key_bytes_cap) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "distinctive key buffer too small");
        std::memcpy(key_bytes + off, rows[r].key, rows[r].len);
        off += rows[r].len;
        key_lens[r] = rows[r].len;
        scores[r] = rows[r].score;
    }
    *n_rows = keep;
    return WFCU_OK;
}

extern "C" int wfcu_counter_merge(wfcu_counter* dst, const wfcu_counter* src, void* stream) {
    if (!dst || !src) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    cudaStream_t s = (cudaStream_t)stream;
    LaunchTally tally;
    CUDA_TRY(tb_merge_table(dst->v, src->v, dst->sm_count, s, &tally.n));
    // long tokens: serialise src, re-insert into dst
    u64 h[8];
    CUDA_TRY(cudaMemcpyAsync(h, src->counters, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (h[3]) {
        uint8_t* buf = nullptr;
        const u64 cap = h[4] + 16 * h[3] + 64;
        CUDA_TRY(scratch_alloc(&buf, cap));
        cudaError_t e = tb_long_serialize(src->v, buf, cap, dst->counters + 8, dst->sm_count, s, &tally.n);
        u64 nbytes = 0;
        if (e == cudaSuccess) e = cudaMemcpyAsync(&nbytes, dst->counters + 8, sizeof(u64), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = tb_long_merge(dst->v, buf, nbytes, 0, 1, s, &tally.n);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        scratch_free(buf);
        if (e != cudaSuccess) return fail(WFCU_ERR_CUDA, "long-token merge: %s", cudaGetErrorString(e));
    }
    return WFCU_OK;
}

extern "C" int wfcu_counter_add_words(wfcu_counter* c, const uint8_t* key_bytes, const uint32_t* key_lens,
                                      const uint64_t* counts, uint64_t n_words) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (n_words == 0) return WFCU_OK;
    if (!key_bytes || !key_lens || !counts) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    std::vector<Slot> inl;
    std::vector<uint8_t> longs;
    u64 off = 0;
    for (u64 i = 0; i < n_words; ++i) {
        const u32 len = key_lens[i];
        if (len == 0) return fail(WFCU_ERR_INVALID_ARGUMENT, "empty word");
        if (len <= 16) {
            Slot s{};
            key_from_bytes(key_bytes + off, len, &s.k0, &s.k1);
            s.count = counts[i];
            inl.push_back(s);
        } else {
            const u64 need = 16 + ((u64(len) + 7) & ~7ull);
            const size_t at = longs.size();
            longs.resize(at + need, 0);
            const u32 h = fnv32(key_bytes + off, len);
            std::memcpy(&longs[at], &counts[i], 8);
            std::memcpy(&longs[at + 8], &len, 4);
            std::memcpy(&longs[at + 12], &h, 4);
            std::memcpy(&longs[at + 16], key_bytes + off, len);
        }
        off += len;
    }
    LaunchTally tally;
    if (!inl.empty()) {
        void* dev = nullptr;
        if (int rc = upload(inl.data(), inl.size() * sizeof(Slot), &dev)) return rc;
        cudaError_t e = tb_merge_entries(c->v, static_cast<const Slot*>(dev), inl.size(), c->sm_count, nullptr, &tally.n);
        if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
        scratch_free(dev);
        if (e != cudaSuccess) return fail(WFCU_ERR_CUDA, "add_words: %s", cudaGetErrorString(e));
    }
    if (!longs.empty()) {
        void* dev = nullptr;
        if (int rc = upload(longs.data(), longs.size(), &dev)) return rc;
        cudaError_t e = tb_long_merge(c->v, static_cast<const uint8_t*>(dev), longs.size(), 0, 1, nullptr, &tally.n);
        if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
        scratch_free(dev);
        if (e != cudaSuccess) return fail(WFCU_ERR_CUDA, "add_words: %s", cudaGetErrorString(e));
    }
    return WFCU_OK;
}

// ---- host-buffer counting (the reference-facing call) ----------------------------------
static int ensure_staging(wfcu_counter* c, u64 want) {
    if (c->chunk_cap >= want) return WFCU_OK;
    if (c->chunk_cap) CUDA_TRY(cudaDeviceSynchronize());
    for (int i = 0; i < 2; ++i) {
        if (c->pinned[i]) pinned_free(c->pinned[i]);
        if (c->devbuf[i]) scratch_free(c->devbuf[i]);
        c->pinned[i] = nullptr;
        c->devbuf[i] = nullptr;
    }
    c->chunk_cap = 0;
    for (int i = 0; i < 2; ++i) {
        CUDA_TRY(pinned_alloc((void**)&c->pinned[i], want));
        CUDA_TRY(scratch_alloc((void**)&c->devbuf[i], want));
        if (!c->done[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->done[i], cudaEventDisableTiming));
    }
    if (!c->stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->chunk_cap = want;
    return WFCU_OK;
}

// two device buffers of `want` bytes, the copy stream and the events of the DMA path
static int ensure_dma(wfcu_counter* c, u64 want) {
    want = (want + 15) & ~15ull;
    if (!c->stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    if (!c->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        if (!c->copied[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->copied[i], cudaEventDisableTiming));
        if (!c->counted[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->counted[i], cudaEventDisableTiming));
    }
    if (c->dma_cap >= want) return WFCU_OK;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < 2; ++i) {
        if (c->dma_buf[i]) scratch_free(c->dma_buf[i]);
        c->dma_buf[i] = nullptr;
    }
    c->dma_cap = 0;
    for (int i = 0; i < 2; ++i) CUDA_TRY(scratch_alloc((void**)&c->dma_buf[i], want));
    c->dma_cap = want;
    return WFCU_OK;
}

extern "C" int wfcu_counter_count_host(wfcu_counter* c, const uint8_t* const* docs, const uint64_t* doc_lens,
                                       uint64_t n_docs) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (n_docs == 0) return WFCU_OK;
    if (!docs || !doc_lens) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    u64 max_doc = 0, total = 0;
    for (u64 d = 0; d < n_docs; ++d) {
        if (doc_lens[d] && !docs[d]) return fail(WFCU_ERR_INVALID_ARGUMENT, "document %llu is null", (unsigned long long)d);
        max_doc = std::max<u64>(max_doc, doc_lens[d]);
        total += doc_lens[d] + 1;
    }
    // Fast path: the documents lie back to back in page-locked host memory and each ends
    // with ASCII whitespace (so no separator is needed): DMA straight from the caller's
    // buffer, no packing pass.
    {
        bool adjacent = true;
        for (u64 d = 0; d < n_docs && adjacent; ++d) {
            if (doc_lens[d] == 0) { adjacent = false; break; }
            const uint8_t last = docs[d][doc_lens[d] - 1];
            const bool ws = last == 0x20 || (last >= 0x09 && last <= 0x0D);
            if (!ws && d + 1 < n_docs) adjacent = false;
            if (d + 1 < n_docs && docs[d] + doc_lens[d] != docs[d + 1]) adjacent = false;
        }
        cudaPointerAttributes attr{};
        if (adjacent && cudaPointerGetAttributes(&attr, docs[0]) == cudaSuccess && attr.type == cudaMemoryTypeHost) {
            // The copy engine streams chunks of whole documents straight from the caller's pinned buffer
            // into two device buffers (55 GB/s measured; a kernel reading the same memory over PCIe
            // itself reaches 49-51 GB/s) while the previous chunk is counted on a second stream.
            const u64 span = total - n_docs;   // bytes of all documents
            static const u64 chunk_mb = [] { const char* e = getenv("WFCU_DMA_CHUNK_MB"); return e ? (u64)atoi(e) : 0ull; }();
            const u64 chunk_bytes = (chunk_mb ? chunk_mb : 32ull) << 20;
            if (int rc = ensure_dma(c, std::min<u64>(std::max<u64>(max_doc, chunk_bytes), std::max<u64>(span, 16)))) return rc;
            CUDA_TRY(cudaStreamSynchronize(nullptr));
            u64 k = 0;
            for (u64 first = 0; first < n_docs;) {
                u64 last = first, len = 0;
                while (last < n_docs && (len == 0 || len + doc_lens[last] <= c->dma_cap)) len += doc_lens[last++];
                const int b = (int)(k & 1);
                if (k >= 2) CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->counted[b], 0));
                CUDA_TRY(cudaMemcpyAsync(c->dma_buf[b], docs[first], len, cudaMemcpyHostToDevice, c->copy_stream));
                CUDA_TRY(cudaEventRecord(c->copied[b], c->copy_stream));
                CUDA_TRY(cudaStreamWaitEvent(c->stream, c->copied[b], 0));
                if (int rc = wfcu_counter_count_dev(c, c->dma_buf[b], len, c->stream)) return rc;
                CUDA_TRY(cudaEventRecord(c->counted[b], c->stream));
                first = last;
                ++k;
            }
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            return wfcu_counter_status(c, c->stream);
        }
        cudaGetLastError();   // cudaPointerGetAttributes on plain malloc memory may set an error on old drivers
    }
    // chunk = whole documents, '\n' after each; 32 MiB unless one document needs more
    static const u64 pack_mb = [] { const char* e = getenv("WFCU_PACK_CHUNK_MB"); return e ? (u64)atoi(e) : 0ull; }();
    u64 chunk = std::min<u64>(std::max<u64>(total, 1 << 20), (pack_mb ? pack_mb : 32ull) << 20);
    chunk = std::max<u64>(chunk, max_doc + 1);
    chunk = (chunk + 15) & ~15ull;
    if (int rc = ensure_staging(c, chunk)) return rc;
    // default-stream work issued earlier (reset, count_dev) must be visible to our stream
    CUDA_TRY(cudaStreamSynchronize(nullptr));

    int cur = 0;
    u64 fill = 0;
    bool used[2] = {false, false};
    auto submit = [&]() -> int {
        if (fill == 0) return WFCU_OK;
        CUDA_TRY(cudaMemcpyAsync(c->devbuf[cur], c->pinned[cur], fill, cudaMemcpyHostToDevice, c->stream));
        if (int rc = wfcu_counter_count_dev(c, c->devbuf[cur], fill, c->stream)) return rc;
        CUDA_TRY(cudaEventRecord(c->done[cur], c->stream));
        used[cur] = true;
        cur ^= 1;
        fill = 0;
        if (used[cur]) CUDA_TRY(cudaEventSynchronize(c->done[cur]));   // buffer about to be refilled
        return WFCU_OK;
    };
    // documents [first, d) form one chunk; they are packed by a few host threads that live for the
    // whole call (spawning them per chunk cost ~10 % of a 64 MiB chunk's time) and take documents
    // one at a time from a shared cursor
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned n_threads = std::min(16u, hw);
    std::vector<u64> offs;
    struct PackPool {
        // Workers SPIN between chunks: on the (virtualised) GPU hosts waking 15 sleeping threads through a
        // condition variable cost 0.5-1 ms per chunk, as much as packing it.  They exist only for this call.
        std::vector<std::thread> threads;
        std::atomic<u64> generation{0};
        std::atomic<unsigned> busy{0};
        std::atomic<bool> stop{false};
        std::atomic<u64> cursor{0};
        // the chunk being packed
        uint8_t* dst = nullptr;
        const uint8_t* const* docs = nullptr;
        const uint64_t* lens = nullptr;
        const u64* offs = nullptr;
        u64 first = 0, last = 0;
        static void relax(unsigned& spins) {
            if (++spins < 4096) {
#if defined(__x86_64__) || defined(__i386__)
                __builtin_ia32_pause();
#endif
            } else {
                std::this_thread::yield();
            }
        }
        // work unit = a 256 KiB slice of the chunk's packed image, whatever documents it cuts through
        const u64 SLICE = 256u << 10;
        u64 fill = 0;    // bytes of the packed image
        void drain() {
            const u64 n_docs = last - first;
            for (;;) {
                const u64 a = cursor.fetch_add(1, std::memory_order_relaxed) * SLICE;
                if (a >= fill) return;
                const u64 b = std::min(a + SLICE, fill);
                u64 i = (u64)(std::upper_bound(offs, offs + n_docs, a) - offs) - 1;   // document holding byte a
                for (; i < n_docs && offs[i] < b; ++i) {
                    const u64 len = lens[first + i];
                    const u64 lo = std::max(a, offs[i]), hi = std::min(b, offs[i] + len);
                    if (lo < hi) std::memcpy(dst + lo, docs[first + i] + (lo - offs[i]), hi - lo);
                    if (offs[i] + len >= a && offs[i] + len < b) dst[offs[i] + len] = '\n';
                }
            }
        }
        void worker() {
            u64 seen = 0;
            for (;;) {
                unsigned spins = 0;
                while (generation.load(std::memory_order_acquire) == seen) {
                    if (stop.load(std::memory_order_acquire)) return;
                    relax(spins);
                }
                ++seen;
                drain();
                busy.fetch_sub(1, std::memory_order_release);
            }
        }
        void run(unsigned helpers) {
            if (helpers && threads.empty())
                for (unsigned t = 0; t < helpers; ++t) threads.emplace_back([this] { worker(); });
            cursor.store(0, std::memory_order_relaxed);
            if (helpers) {
                busy.store((unsigned)threads.size(), std::memory_order_relaxed);
                generation.fetch_add(1, std::memory_order_release);
            }
            drain();
            unsigned spins = 0;
            while (helpers && busy.load(std::memory_order_acquire)) relax(spins);
        }
        ~PackPool() {
            stop.store(true, std::memory_order_release);
            for (auto& th : threads) th.join();
        }
    } pool;
    pool.docs = docs;
    pool.lens = doc_lens;
    auto pack = [&](u64 first, u64 last) {
        pool.dst = c->pinned[cur];
        pool.offs = offs.data();
        pool.first = first;
        pool.last = last;
        pool.fill = fill;
        pool.run(fill >= (1u << 20) ? n_threads - 1 : 0);   // small chunks: this thread alone
    };
    u64 first = 0;
    for (u64 d = 0; d <= n_docs; ++d) {
        const u64 need = d < n_docs ? doc_lens[d] + 1 : 0;
        if (d == n_docs || fill + need > c->chunk_cap) {
            if (d > first) pack(first, d);
            if (int rc = submit()) return rc;
            first = d;
            offs.clear();
        }
        if (d < n_docs) {
            offs.push_back(fill);
            fill += need;
        }
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return wfcu_counter_status(c, c->stream);
}

// ---- exchange -------------------------------------------------------------------------
extern "C" uint32_t wfcu_owner_of(const uint8_t* word, uint32_t len, uint32_t n_parts) {
    if (n_parts <= 1 || !word) return 0;
    if (len <= 16) {
        u64 k0, k1;
        key_from_bytes(word, len, &k0, &k1);
        return owner_mix32(k0, k1) % n_parts;
    }
    return ((fnv32(word, len) * 0x9E3779B1u) >> 7) % n_parts;
}

extern "C" int wfcu_counter_partition(wfcu_counter* c, uint32_t n_parts, wfcu_entry* dev_entries, uint64_t entries_cap,
                                      uint64_t* dev_part_counts, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (n_parts == 0 || n_parts > 4096) return fail(WFCU_ERR_INVALID_ARGUMENT, "n_parts must be in 1..4096");
    if (!dev_entries || !dev_part_counts) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    static_assert(sizeof(wfcu_entry) == sizeof(Slot), "wire entry layout");
    cudaStream_t s = (cudaStream_t)stream;
    u64* cursors = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&cursors, sizeof(u64) * n_parts, s));
    LaunchTally tally;
    cudaError_t e = tb_partition(c->v, n_parts, reinterpret_cast<Slot*>(dev_entries), entries_cap,
                                 reinterpret_cast<u64*>(dev_part_counts), cursors, c->sm_count, s, &tally.n);
    cudaFreeAsync(cursors, s);
    // slot n_parts: bytes of the long-token record stream (0 for almost every corpus), so that the
    // caller learns it from the same device array and needs no extra synchronisation
    if (e == cudaSuccess)
        e = tb_long_serialize(c->v, nullptr, 0, reinterpret_cast<u64*>(dev_part_counts) + n_parts, c->sm_count, s, &tally.n);
    if (e != cudaSuccess) return fail(WFCU_ERR_CUDA, "partition: %s", cudaGetErrorString(e));
    return WFCU_OK;
}

extern "C" uint64_t wfcu_counter_max_entries(const wfcu_counter* c) { return c ? c->v.max_used + 1 : 0; }

extern "C" int wfcu_counter_partition_fixed(wfcu_counter* c, uint32_t n_parts, wfcu_entry* dev_entries,
                                            uint64_t cap_per_part, uint64_t* dev_counts, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (n_parts == 0 || n_parts > 4096) return fail(WFCU_ERR_INVALID_ARGUMENT, "n_parts must be in 1..4096");
    if (!dev_entries || !dev_counts || cap_per_part == 0) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    LaunchTally tally;
    CUDA_TRY(tb_partition_fixed(c->v, n_parts, cap_per_part, false, reinterpret_cast<Slot*>(dev_entries),
                                reinterpret_cast<u64*>(dev_counts), c->sm_count, (cudaStream_t)stream, &tally.n));
    return WFCU_OK;
}

extern "C" int wfcu_counter_partition_framed(wfcu_counter* c, uint32_t n_parts, wfcu_entry* dev_entries,
                                             uint64_t cap_per_part, uint64_t* dev_counts, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (n_parts == 0 || n_parts > 4096) return fail(WFCU_ERR_INVALID_ARGUMENT, "n_parts must be in 1..4096");
    if (!dev_entries || !dev_counts || cap_per_part < 2) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument or capacity below 2");
    LaunchTally tally;
    CUDA_TRY(tb_partition_fixed(c->v, n_parts, cap_per_part, true, reinterpret_cast<Slot*>(dev_entries),
                                reinterpret_cast<u64*>(dev_counts), c->sm_count, (cudaStream_t)stream, &tally.n));
    return WFCU_OK;
}

extern "C" int wfcu_counter_merge_regions(wfcu_counter* c, const wfcu_entry* dev_entries, uint32_t n_parts,
                                          uint64_t cap_per_part, const uint64_t* dev_region_counts, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (!dev_entries) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    LaunchTally tally;
    CUDA_TRY(tb_merge_regions(c->v, reinterpret_cast<const Slot*>(dev_entries), n_parts, cap_per_part,
                              reinterpret_cast<const u64*>(dev_region_counts), c->sm_count, (cudaStream_t)stream, &tally.n));
    return WFCU_OK;
}

extern "C" int wfcu_counter_merge_entries(wfcu_counter* c, const wfcu_entry* dev_entries, uint64_t n, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (n && !dev_entries) return fail(WFCU_ERR_INVALID_ARGUMENT, "entries is null");
    LaunchTally tally;
    CUDA_TRY(tb_merge_entries(c->v, reinterpret_cast<const Slot*>(dev_entries), n, c->sm_count, (cudaStream_t)stream, &tally.n));
    return WFCU_OK;
}

extern "C" int wfcu_counter_long_records(wfcu_counter* c, uint8_t* dev_out, uint64_t out_cap, uint64_t* n_bytes,
                                         void* stream) {
    if (!c || !n_bytes) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    LaunchTally tally;
    CUDA_TRY(tb_long_serialize(c->v, dev_out, out_cap, c->counters + 8, c->sm_count, s, &tally.n));
    CUDA_TRY(cudaMemcpyAsync(n_bytes, c->counters + 8, sizeof(u64), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (dev_out && *n_bytes > out_cap) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "long record stream needs %llu bytes", (unsigned long long)*n_bytes);
    return WFCU_OK;
}

extern "C" int wfcu_counter_merge_long_records(wfcu_counter* c, const uint8_t* dev_records, uint64_t n_bytes,
                                               uint32_t part, uint32_t n_parts, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (n_bytes && !dev_records) return fail(WFCU_ERR_INVALID_ARGUMENT, "records is null");
    LaunchTally tally;
    CUDA_TRY(tb_long_merge(c->v, dev_records, n_bytes, part, n_parts, (cudaStream_t)stream, &tally.n));
    return WFCU_OK;
}

// ---- stage timer: a pair of CUDA events ---------------------------------------------------------------------
struct wfcu_timer {
    cudaEvent_t a = nullptr, b = nullptr;
};
extern "C" int wfcu_timer_create(wfcu_timer** out) {
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    auto* t = new wfcu_timer;
    if (cudaEventCreate(&t->a) != cudaSuccess || cudaEventCreate(&t->b) != cudaSuccess) {
        wfcu_timer_destroy(t);
        return fail(WFCU_ERR_CUDA, "cudaEventCreate failed");
    }
    *out = t;
    return WFCU_OK;
}
extern "C" int wfcu_timer_start(wfcu_timer* t) {
    if (!t) return fail(WFCU_ERR_INVALID_ARGUMENT, "timer is null");
    CUDA_TRY(cudaEventRecord(t->a, nullptr));
    return WFCU_OK;
}
extern "C" int wfcu_timer_stop_ns(wfcu_timer* t, uint64_t* elapsed_ns) {
    if (!t || !elapsed_ns) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    CUDA_TRY(cudaEventRecord(t->b, nullptr));
    CUDA_TRY(cudaEventSynchronize(t->b));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, t->a, t->b));
    *elapsed_ns = uint64_t(double(ms) * 1e6);
    return WFCU_OK;
}
extern "C" void wfcu_timer_destroy(wfcu_timer* t) {
    if (!t) return;
    if (t->a) cudaEventDestroy(t->a);
    if (t->b) cudaEventDestroy(t->b);
    delete t;
}

// ---- run_wordcount over n workers on the GPUs of this box ---------------------------------------------------
// (proj/src/pipeline.cpp:61-123 with the hash-partitioned merge of BASELINE.json in place of the range shuffle.)
// One host thread per worker; worker j lives on device j mod wfcu_device_count(), counts the documents
// d = j (mod n) into a local table, partitions it by owner (tb_partition_*), then -- after a barrier -- pulls region j
// of every worker's partition straight from that worker's device memory (cudaMemcpyPeerAsync: NVLink between GPUs,
// a plain device copy when two workers share one) and merge-inserts it into the table it owns.  Long tokens (rare)
// travel as the record stream.  Stage times are CUDA-event times on each worker's device, maximum over workers.
namespace {
struct SpinBarrier {      // n threads, reusable
    explicit SpinBarrier(unsigned n) : n_(n) {}
    void wait() {
        std::unique_lock<std::mutex> lock(mu_);
        const unsigned gen = gen_;
        if (++arrived_ == n_) { arrived_ = 0; ++gen_; cv_.notify_all(); }
        else cv_.wait(lock, [&] { return gen_ != gen; });
    }
    std::mutex mu_;
    std::condition_variable cv_;
    unsigned n_, arrived_ = 0, gen_ = 0;
};
struct MultiWorker {
    int device = 0;
    wfcu_counter* local = nullptr;
    wfcu_counter* owned = nullptr;
    Slot* entries = nullptr;             // the local table partitioned by owner (on `device`)
    std::vector<u64> part_counts;        // entries per owner
    std::vector<uint8_t> long_records;   // host copy of the long-token record stream
    float map_ms = 0, encode_ms = 0, exchange_ms = 0;
    int rc = WFCU_OK;
    std::string error;
};
}  // namespace

extern "C" int wfcu_wordcount_multi(const uint8_t* const* docs, const uint64_t* lens, uint64_t n_docs, uint32_t n_workers,
                                    const wfcu_counter_config* cfg, wfcu_counter** out_shards, wfcu_stage_ns* timings) {
    if (n_workers == 0 || n_workers > 4096) return fail(WFCU_ERR_INVALID_ARGUMENT, "n_workers must be in 1..4096");
    if (!out_shards) return fail(WFCU_ERR_INVALID_ARGUMENT, "out_shards is null");
    if (n_docs && (!docs || !lens)) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    for (u32 j = 0; j < n_workers; ++j) out_shards[j] = nullptr;
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev <= 0) {
        cudaGetLastError();
        return fail(WFCU_ERR_NO_DEVICE, "no CUDA device available; libwfcu has no CPU path");
    }
    int caller_dev = 0;
    cudaGetDevice(&caller_dev);
    const auto t_start = std::chrono::steady_clock::now();
    const u32 n = n_workers;
    std::vector<MultiWorker> w(n);
    SpinBarrier barrier(n);
    auto body = [&](u32 j) {
        MultiWorker& me = w[j];
        me.device = int(j % u32(n_dev));
        auto failed = [&](int rc) { me.rc = rc; me.error = g_last_error; return rc; };
        auto cuda = [&](cudaError_t e, const char* what) {
            if (e == cudaSuccess) return WFCU_OK;
            me.rc = WFCU_ERR_CUDA;
            me.error = std::string(what) + ": " + cudaGetErrorString(e);
            return WFCU_ERR_CUDA;
        };
        cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
        u64* dev_counts = nullptr;
        Slot* recv = nullptr;
        do {   // phase 1: map + encode
            if (cuda(cudaSetDevice(me.device), "cudaSetDevice")) break;
            for (auto& e : ev) if (cuda(cudaEventCreate(&e), "cudaEventCreate")) break;
            if (me.rc) break;
            if (failed(wfcu_counter_create(&me.local, cfg))) break;
            if (failed(wfcu_counter_create(&me.owned, cfg))) break;
            std::vector<const uint8_t*> my_docs;
            std::vector<uint64_t> my_lens;
            for (u64 d = j; d < n_docs; d += n) { my_docs.push_back(docs[d]); my_lens.push_back(lens[d]); }
            cudaEventRecord(ev[0], nullptr);
            if (failed(wfcu_counter_count_host(me.local, my_docs.data(), my_lens.data(), my_docs.size()))) break;
            cudaEventRecord(ev[1], nullptr);
            uint64_t distinct = 0;
            if (failed(wfcu_counter_stats(me.local, nullptr, &distinct, nullptr, nullptr))) break;
            if (cuda(scratch_alloc((void**)&me.entries, sizeof(Slot) * std::max<u64>(distinct, 1)), "cudaMalloc entries")) break;
            if (cuda(scratch_alloc((void**)&dev_counts, sizeof(u64) * (n + 1)), "cudaMalloc counts")) break;
            if (failed(wfcu_counter_partition(me.local, n, reinterpret_cast<wfcu_entry*>(me.entries), std::max<u64>(distinct, 1),
                                              reinterpret_cast<uint64_t*>(dev_counts), nullptr))) break;
            me.part_counts.assign(n + 1, 0);
            if (cuda(cudaMemcpy(me.part_counts.data(), dev_counts, sizeof(u64) * (n + 1), cudaMemcpyDeviceToHost), "D2H counts")) break;
            if (me.part_counts[n]) {   // long-token records: serialise, keep a host copy for the owners
                uint8_t* dev_recs = nullptr;
                uint64_t bytes = me.part_counts[n];
                if (cuda(scratch_alloc((void**)&dev_recs, bytes), "cudaMalloc records")) break;
                int rc = wfcu_counter_long_records(me.local, dev_recs, bytes, &bytes, nullptr);
                me.long_records.resize(bytes);
                if (rc == WFCU_OK && cudaMemcpy(me.long_records.data(), dev_recs, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) rc = WFCU_ERR_CUDA;
                scratch_free(dev_recs);
                if (rc) { failed(rc); break; }
            }
            cudaEventRecord(ev[2], nullptr);
        } while (false);
        barrier.wait();     // every partition is complete (or its worker has failed)
        bool any_failed = false;
        for (const MultiWorker& o : w) any_failed |= o.rc != WFCU_OK;
        if (!any_failed) {
            do {   // phase 2: exchange + merge-insert of what this worker owns
                u64 most = 1;
                for (const MultiWorker& o : w) most = std::max(most, o.part_counts[j]);
                if (cuda(scratch_alloc((void**)&recv, sizeof(Slot) * most), "cudaMalloc receive buffer")) break;
                for (u32 k = 0; k < n && me.rc == WFCU_OK; ++k) {
                    const MultiWorker& o = w[(j + k) % n];        // start with the own region: spreads the peers
                    const u64 cnt = o.part_counts[j];
                    if (cnt) {
                        u64 off = 0;
                        for (u32 p = 0; p < j; ++p) off += o.part_counts[p];
                        if (cuda(cudaMemcpyPeerAsync(recv, me.device, o.entries + off, o.device, sizeof(Slot) * cnt, nullptr), "peer copy")) break;
                        if (failed(wfcu_counter_merge_entries(me.owned, reinterpret_cast<const wfcu_entry*>(recv), cnt, nullptr))) break;
                        if (cuda(cudaStreamSynchronize(nullptr), "exchange")) break;     // recv is reused
                    }
                    if (!o.long_records.empty()) {
                        uint8_t* dev_recs = nullptr;
                        if (cuda(scratch_alloc((void**)&dev_recs, o.long_records.size()), "cudaMalloc records")) break;
                        int rc = cudaMemcpy(dev_recs, o.long_records.data(), o.long_records.size(), cudaMemcpyHostToDevice) == cudaSuccess ? WFCU_OK : WFCU_ERR_CUDA;
                        if (rc == WFCU_OK) rc = wfcu_counter_merge_long_records(me.owned, dev_recs, o.long_records.size(), j, n, nullptr);
                        cudaDeviceSynchronize();
                        scratch_free(dev_recs);
                        if (rc) { failed(rc); break; }
                    }
                }
                if (me.rc) break;
                if (failed(wfcu_counter_status(me.owned, nullptr))) break;
                cudaEventRecord(ev[3], nullptr);
                if (cuda(cudaEventSynchronize(ev[3]), "exchange")) break;
                cudaEventElapsedTime(&me.map_ms, ev[0], ev[1]);
                cudaEventElapsedTime(&me.encode_ms, ev[1], ev[2]);
                cudaEventElapsedTime(&me.exchange_ms, ev[2], ev[3]);
            } while (false);
        }
        barrier.wait();     // nobody frees a partition a peer may still be reading
        scratch_free(recv);
        scratch_free(dev_counts);
        scratch_free(me.entries);
        me.entries = nullptr;
        wfcu_counter_destroy(me.local);
        me.local = nullptr;
        for (auto& e : ev) if (e) cudaEventDestroy(e);
    };
    std::vector<std::thread> threads;
    for (u32 j = 1; j < n; ++j) threads.emplace_back(body, j);
    body(0);
    for (auto& t : threads) t.join();
    cudaSetDevice(caller_dev);
    for (u32 j = 0; j < n; ++j) {     // the lowest-indexed failure is the one reported (pipeline.cpp:30-45)
        if (w[j].rc == WFCU_OK) continue;
        for (MultiWorker& o : w) { wfcu_counter_destroy(o.owned); o.owned = nullptr; }
        cudaSetDevice(caller_dev);
        return fail(w[j].rc, "worker %u: %s", j, w[j].error.c_str());
    }
    wfcu_stage_ns t{};
    for (u32 j = 0; j < n; ++j) {
        out_shards[j] = w[j].owned;
        t.map_ns = std::max<uint64_t>(t.map_ns, uint64_t(w[j].map_ms * 1e6));
        t.encode_ns = std::max<uint64_t>(t.encode_ns, uint64_t(w[j].encode_ms * 1e6));
        t.exchange_ns = std::max<uint64_t>(t.exchange_ns, uint64_t(w[j].exchange_ms * 1e6));
    }
    t.total_ns = uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_start).count());
    if (timings) *timings = t;
    return WFCU_OK;
}

// ---- synthetic corpora ------------------------------------------------------------------
extern "C" int wfcu_synth_document(uint64_t seed, uint64_t doc, uint32_t vocab, double zipf_s, uint32_t speaker,
                                   uint8_t* out, uint64_t doc_bytes) {
    if (synth_document(seed, doc, vocab, zipf_s, speaker, out, doc_bytes)) return fail(WFCU_ERR_INVALID_ARGUMENT, "bad synth arguments");
    return WFCU_OK;
}
extern "C" int wfcu_synth_corpus(uint64_t seed, uint64_t doc_begin, uint64_t doc_end, uint32_t vocab, double zipf_s,
                                 uint32_t speaker, uint64_t doc_bytes, uint8_t* out, int threads) {
    if (synth_corpus(seed, doc_begin, doc_end, vocab, zipf_s, speaker, doc_bytes, out, threads))
        return fail(WFCU_ERR_INVALID_ARGUMENT, "bad synth arguments");
    return WFCU_OK;
}
extern "C" int wfcu_synth_corpus_strided(uint64_t seed, uint64_t doc_begin, uint64_t doc_stride, uint64_t n_docs,
                                         uint32_t vocab, double zipf_s, uint32_t speaker, uint64_t doc_bytes,
                                         uint8_t* out, int threads) {
    if (synth_corpus_strided(seed, doc_begin, doc_stride, n_docs, vocab, zipf_s, speaker, doc_bytes, out, threads))
        return fail(WFCU_ERR_INVALID_ARGUMENT, "bad synth arguments");
    return WFCU_OK;
}
extern "C" int wfcu_synth_uniform(uint64_t seed, uint64_t n, int dtype, void* out) {
    if (dtype != WFCU_DTYPE_F32 && dtype != WFCU_DTYPE_F64) return fail(WFCU_ERR_INVALID_ARGUMENT, "unknown dtype %d", dtype);
    if (synth_uniform(seed, n, dtype == WFCU_DTYPE_F64, out)) return fail(WFCU_ERR_INVALID_ARGUMENT, "bad synth arguments");
    return WFCU_OK;
}

// ---- token lists: tokenize / sort_words / reduce_sorted ---------------------------------
struct wfcu_tokens {
    int device = 0;
    int sm_count = 0;
    TokenRec* recs = nullptr;
    u64 n = 0;
    uint8_t* arena = nullptr;   // long-token records {u32 len, u32 hash, bytes}, offset 0 unused
    u64 arena_used = 0;
    u64 arena_cap = 0;
    bool sorted = false;        // WordList::sorted (proj/include/wfc/text.hpp:18-21)
    // The tokenizer kernels leave the records in no particular order; text order costs a five-pass radix sort on the
    // position.  It is restored on first use (ensure_text_order) -- a list that is sorted by key right away, the map
    // stage of the paper's algorithm, never pays for it.
    bool text_order_pending = false;
    std::mutex order_mu;
};

static void tokens_free(wfcu_tokens* t) {
    if (!t) return;
    scratch_free(t->recs);
    scratch_free(t->arena);
    delete t;
}

extern "C" void wfcu_tokens_destroy(wfcu_tokens* t) {
    if (t) cudaSetDevice(t->device);
    tokens_free(t);
}

static int sort_device_tokens(wfcu_tokens* t, bool by_position, cudaStream_t s) {
    if (t->n < 2) return WFCU_OK;
    DevBuf alt, hist, tmp;
    const u64 hw = sort_hist_words(t->n);
    CUDA_TRY(alt.alloc(sizeof(TokenRec) * t->n));
    CUDA_TRY(hist.alloc(sizeof(u64) * hw));
    CUDA_TRY(tmp.alloc(sizeof(u64) * scan_tmp_words(hw)));
    SortScratch sc{alt.as<TokenRec>(), hist.as<u64>(), tmp.as<u64>()};
    LaunchTally tally;
    CUDA_TRY(tokens_sort(t->recs, t->n, by_position, t->arena, sc, t->sm_count, s, &tally.n));
    CUDA_TRY(cudaStreamSynchronize(s));
    return WFCU_OK;
}

static int ensure_text_order(const wfcu_tokens* ct, cudaStream_t s) {
    auto* t = const_cast<wfcu_tokens*>(ct);     // the order is a cache of the object, not its value
    std::lock_guard<std::mutex> lock(t->order_mu);
    if (!t->text_order_pending) return WFCU_OK;
    if (int rc = sort_device_tokens(t, /*by_position=*/true, s)) return rc;
    t->text_order_pending = false;
    return WFCU_OK;
}

// Runs the tokenizer kernels; the records come out in no particular order.
// Compact mode of tokenize_unordered (counting by sort + RLE): tokens of at most 8 bytes come back as 64-bit
// keys in the tokenizer's tiled layout, only the others as records.
struct CompactKeys {
    DevBuf keys, tile_counts;
    u64 tiles = 0;     // tiles handed out (kKeyTile keys each, tile t holds tile_counts[t])
    u64 n_keys = 0;
    u64 vary = 0;      // bits that differ between keys
};

static int tokenize_unordered(const uint8_t* dev_text, uint64_t n, cudaStream_t s, wfcu_tokens** out, CompactKeys* ck = nullptr) {
    *out = nullptr;
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (n && !dev_text) return fail(WFCU_ERR_INVALID_ARGUMENT, "text is null");
    if (reinterpret_cast<uintptr_t>(dev_text) & 15u) return fail(WFCU_ERR_INVALID_ARGUMENT, "device text must be 16-byte aligned");
    auto* t = new wfcu_tokens;
    cudaGetDevice(&t->device);
    t->sm_count = d->sm_count;
    if (n == 0) {
        *out = t;
        return WFCU_OK;
    }
    u64 cap = ck ? n / 16 + 1024 : n / 5 + 1024;   // records; grown to the exact count on overflow
    u64 key_tiles = ck ? (n / 4) / (kKeyTile - 32) + (u64)d->sm_count * 32 + 64 : 0;   // a warp leaves < 32 slots of a tile unused
    u64 deferred_cap = n / 16 + 1024;       // grown on overflow
    u64 arena_cap = std::max<u64>(1 << 20, n / 4);
    for (int attempt = 0; attempt < 4; ++attempt) {
        DevBuf recs, deferred, arena, counters;
        cudaError_t e = recs.alloc(sizeof(TokenRec) * cap);
        if (e == cudaSuccess) e = deferred.alloc(sizeof(u64) * deferred_cap);
        if (e == cudaSuccess) e = arena.alloc(arena_cap);
        if (e == cudaSuccess) e = counters.alloc(sizeof(u64) * 16);
        if (e == cudaSuccess) e = cudaMemsetAsync(counters.p, 0, sizeof(u64) * 16, s);
        const u64 arena_start = 8;
        u64* cnt = counters.as<u64>();
        if (e == cudaSuccess) e = cudaMemcpyAsync(cnt + 4, &arena_start, sizeof(u64), cudaMemcpyHostToDevice, s);
        DevBuf keys, tile_counts;
        const u64 all_ones = ~0ull;
        if (ck) {
            if (e == cudaSuccess) e = keys.alloc(sizeof(u64) * kKeyTile * key_tiles);
            if (e == cudaSuccess) e = tile_counts.alloc(sizeof(u32) * key_tiles);
            if (e == cudaSuccess) e = cudaMemsetAsync(tile_counts.p, 0, sizeof(u32) * key_tiles, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(cnt + 11, &all_ones, sizeof(u64), cudaMemcpyHostToDevice, s);   // AND of the keys
        }
        if (e != cudaSuccess) {
            tokens_free(t);
            return fail(WFCU_ERR_CUDA, "tokenize allocation: %s", cudaGetErrorString(e));
        }
        TableView v{};
        v.n_used = cnt + 0; v.n_tokens = cnt + 1; v.n_deferred = cnt + 2; v.n_long = cnt + 3; v.arena_used = cnt + 4;
        v.status = reinterpret_cast<int*>(cnt + 5);
        v.deferred = deferred.as<u64>(); v.deferred_cap = deferred_cap;
        v.arena = arena.as<uint8_t>(); v.arena_cap = arena_cap;
        EmitView em{recs.as<TokenRec>(), cap, cnt + 6};
        if (ck) {
            em.keys = keys.as<u64>();
            em.key_tiles = key_tiles;
            em.tile_counts = tile_counts.as<u32>();
            em.kc = cnt + 8;
        }
        LaunchTally tally;
        e = wc_tokenize_launch(dev_text, n, v, em, d->sm_count, s, &tally.n);
        u64 h[12];
        if (e == cudaSuccess) e = cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            tokens_free(t);
            return fail(WFCU_ERR_CUDA, "tokenize: %s", cudaGetErrorString(e));
        }
        const int st = (int)(h[5] & 0xFFFFFFFFu);
        const u64 produced = h[6];
        if (ck && h[8] > key_tiles) {             // the count of tiles asked for is exact
            key_tiles = h[8] + 64;
            if (produced > cap) cap = produced + 1024;
            continue;
        }
        if (produced > cap || (st & (kStatusDeferredFull | kStatusArenaFull))) {
            // grow what overflowed and run again (n_out keeps counting past cap, so it is exact
            // unless the deferred list or the arena cut the run short)
            if (produced > cap) cap = produced + 1024;
            if (st & kStatusDeferredFull) { deferred_cap = n / 2 + 1024; cap = std::max<u64>(cap, n / 2 + 1024); }
            // worst case per fragment: an 8-byte header + the normalised bytes (an invalid byte becomes the 3 bytes of
            // U+FFFD) padded to 8, i.e. below 3 * len + 16 for a fragment of len + 1 input bytes: 5 n + 4096 covers any text
            if (st & kStatusArenaFull) arena_cap = 5 * n + 4096;
            continue;
        }
        t->recs = recs.as<TokenRec>();
        recs.p = nullptr;
        t->arena = arena.as<uint8_t>();
        arena.p = nullptr;
        t->n = produced;
        t->arena_used = h[4];
        t->arena_cap = arena_cap;
        if (ck) {
            ck->keys.p = keys.p; keys.p = nullptr;
            ck->tile_counts.p = tile_counts.p; tile_counts.p = nullptr;
            ck->tiles = h[8];
            ck->n_keys = h[9];
            ck->vary = h[9] ? (h[10] ^ h[11]) : 0;
        }
        *out = t;
        return WFCU_OK;
    }
    tokens_free(t);
    return fail(WFCU_ERR_ARENA_FULL, "tokenize: capacities still too small after regrowing");
}

extern "C" int wfcu_tokenize_dev(const uint8_t* dev_text, uint64_t n, void* stream, wfcu_tokens** out) {
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    if (int rc = tokenize_unordered(dev_text, n, (cudaStream_t)stream, out)) return rc;
    (*out)->text_order_pending = true;      // restored by the first call that reads the order
    return WFCU_OK;
}

extern "C" int wfcu_tokenize_host(const uint8_t* text, uint64_t n, wfcu_tokens** out) {
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (n && !text) return fail(WFCU_ERR_INVALID_ARGUMENT, "text is null");
    void* dev = nullptr;
    if (int rc = upload(text, n, &dev)) return rc;
    const int rc = wfcu_tokenize_dev(static_cast<const uint8_t*>(dev), n, nullptr, out);
    scratch_free(dev);
    return rc;
}

extern "C" int wfcu_tokenize_docs_host(const uint8_t* const* docs, const uint64_t* doc_lens, uint64_t n_docs, wfcu_tokens** out) {
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (n_docs && (!docs || !doc_lens)) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    u64 total = 0;
    for (u64 i = 0; i < n_docs; ++i) {
        if (doc_lens[i] && !docs[i]) return fail(WFCU_ERR_INVALID_ARGUMENT, "document %llu is null", (unsigned long long)i);
        total += doc_lens[i] + 1;
    }
    if (total == 0) return wfcu_tokenize_dev(nullptr, 0, nullptr, out);
    DevBuf text;
    CUDA_TRY(text.alloc(total + 16));     // + 16: see upload()
    // every byte that no document overwrites is a separator
    CUDA_TRY(cudaMemsetAsync(text.p, '\n', total, nullptr));
    u64 off = 0;
    for (u64 i = 0; i < n_docs; ++i) {
        if (doc_lens[i]) CUDA_TRY(cudaMemcpyAsync(text.as<uint8_t>() + off, docs[i], doc_lens[i], cudaMemcpyHostToDevice, nullptr));
        off += doc_lens[i] + 1;
    }
    return wfcu_tokenize_dev(text.as<uint8_t>(), total, nullptr, out);     // synchronises before `text` is released
}

extern "C" int wfcu_tokens_stats(const wfcu_tokens* t, uint64_t* n_tokens, uint64_t* n_bytes) {
    if (!t) return fail(WFCU_ERR_INVALID_ARGUMENT, "tokens is null");
    if (n_tokens) *n_tokens = t->n;
    if (n_bytes) {
        // lengths are recomputed on the host from the records (cheap next to the D2H copy)
        std::vector<TokenRec> h(t->n);
        std::vector<uint8_t> arena(t->arena_used);
        if (t->n) CUDA_TRY(cudaMemcpy(h.data(), t->recs, sizeof(TokenRec) * t->n, cudaMemcpyDeviceToHost));
        if (t->arena_used > 8) CUDA_TRY(cudaMemcpy(arena.data(), t->arena, t->arena_used, cudaMemcpyDeviceToHost));
        u64 total = 0;
        for (const TokenRec& r : h) {
            if (r.ext) {
                u32 len;
                std::memcpy(&len, arena.data() + r.ext, 4);
                total += len;
            } else {
                total += key_len(r.k0, r.k1);
            }
        }
        *n_bytes = total;
    }
    return WFCU_OK;
}

extern "C" int wfcu_tokens_export(const wfcu_tokens* t, uint8_t* bytes, uint64_t bytes_cap, uint32_t* lens,
                                  uint64_t lens_cap) {
    if (!t) return fail(WFCU_ERR_INVALID_ARGUMENT, "tokens is null");
    if (t->n > lens_cap) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "export needs %llu lengths", (unsigned long long)t->n);
    if (int rc = ensure_text_order(t, nullptr)) return rc;
    std::vector<TokenRec> h(t->n);
    std::vector<uint8_t> arena(t->arena_used);
    if (t->n) CUDA_TRY(cudaMemcpy(h.data(), t->recs, sizeof(TokenRec) * t->n, cudaMemcpyDeviceToHost));
    if (t->arena_used > 8) CUDA_TRY(cudaMemcpy(arena.data(), t->arena, t->arena_used, cudaMemcpyDeviceToHost));
    u64 off = 0;
    for (u64 i = 0; i < t->n; ++i) {
        const TokenRec& r = h[i];
        if (r.ext) {
            u32 len;
            std::memcpy(&len, arena.data() + r.ext, 4);
            if (off + len > bytes_cap) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "export byte buffer too small");
            std::memcpy(bytes + off, arena.data() + r.ext + 8, len);
            lens[i] = len;
            off += len;
        } else {
            uint8_t b[16];
            key_to_bytes(r.k0, r.k1, b);
            const u32 len = key_len(r.k0, r.k1);
            if (off + len > bytes_cap) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "export byte buffer too small");
            std::memcpy(bytes + off, b, len);
            lens[i] = len;
            off += len;
        }
    }
    return WFCU_OK;
}

extern "C" int wfcu_tokens_from_words(const uint8_t* bytes, const uint32_t* lens, uint64_t n_tokens, wfcu_tokens** out) {
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (n_tokens && (!bytes || !lens)) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    std::vector<TokenRec> recs(n_tokens);
    std::vector<uint8_t> arena(8, 0);
    u64 off = 0;
    for (u64 i = 0; i < n_tokens; ++i) {
        const u32 len = lens[i];
        if (len == 0) return fail(WFCU_ERR_INVALID_ARGUMENT, "empty word at index %llu", (unsigned long long)i);
        TokenRec r{};
        key_from_bytes(bytes + off, std::min<u32>(len, 16), &r.k0, &r.k1);
        r.pos = i;
        if (len > 16) {
            const size_t at = arena.size();
            arena.resize(at + 8 + ((size_t(len) + 7) & ~size_t(7)), 0);
            const u32 h = fnv32(bytes + off, len);
            std::memcpy(&arena[at], &len, 4);
            std::memcpy(&arena[at + 4], &h, 4);
            std::memcpy(&arena[at + 8], bytes + off, len);
            r.ext = at;
        }
        recs[i] = r;
        off += len;
    }
    auto* t = new wfcu_tokens;
    cudaGetDevice(&t->device);
    t->sm_count = d->sm_count;
    t->n = n_tokens;
    t->arena_used = arena.size();
    t->arena_cap = arena.size();
    void* p = nullptr;
    if (int rc = upload(recs.data(), sizeof(TokenRec) * n_tokens, &p)) { tokens_free(t); return rc; }
    t->recs = static_cast<TokenRec*>(p);
    if (int rc = upload(arena.data(), arena.size(), &p)) { tokens_free(t); return rc; }
    t->arena = static_cast<uint8_t*>(p);
    *out = t;
    return WFCU_OK;
}

// The exchange of the paper's range-partitioned pipeline without leaving device memory (proj/src/shuffle.cpp:98-130:
// chunk c of every worker's sorted list goes to worker c): a new list made of the slices [begin[i], end[i]) of
// n_src lists, in that order.  Records move device to device (peer copies between GPUs); the long-token arenas of
// the sources are appended and the records' references rebased.
extern "C" int wfcu_tokens_concat_slices(const wfcu_tokens* const* src, const uint64_t* begin, const uint64_t* end,
                                         uint32_t n_src, wfcu_tokens** out) {
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (n_src && (!src || !begin || !end)) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    u64 total = 0, arena_total = 8;
    for (u32 i = 0; i < n_src; ++i) {
        if (!src[i] || begin[i] > end[i] || end[i] > src[i]->n)
            return fail(WFCU_ERR_INVALID_ARGUMENT, "slice %u is out of range", i);
        if (int rc = ensure_text_order(src[i], nullptr)) return rc;
        total += end[i] - begin[i];
        if (src[i]->arena_used > 8 && end[i] > begin[i]) arena_total += src[i]->arena_used - 8;
    }
    auto* t = new wfcu_tokens;
    cudaGetDevice(&t->device);
    t->sm_count = d->sm_count;
    t->n = total;
    t->arena_used = arena_total;
    t->arena_cap = arena_total;
    void* p = nullptr;
    cudaError_t e = scratch_alloc(&p, sizeof(TokenRec) * std::max<u64>(total, 1));
    if (e == cudaSuccess) { t->recs = static_cast<TokenRec*>(p); e = scratch_alloc(&p, arena_total); }
    if (e == cudaSuccess) { t->arena = static_cast<uint8_t*>(p); e = cudaMemsetAsync(t->arena, 0, 8, nullptr); }
    LaunchTally tally;
    u64 at = 0, arena_at = 8;
    for (u32 i = 0; i < n_src && e == cudaSuccess; ++i) {
        const u64 m = end[i] - begin[i];
        if (m == 0) continue;
        e = cudaMemcpyPeerAsync(t->recs + at, t->device, src[i]->recs + begin[i], src[i]->device, sizeof(TokenRec) * m, nullptr);
        if (e == cudaSuccess && src[i]->arena_used > 8) {
            const u64 bytes = src[i]->arena_used - 8;
            e = cudaMemcpyPeerAsync(t->arena + arena_at, t->device, src[i]->arena + 8, src[i]->device, bytes, nullptr);
            if (e == cudaSuccess) e = tk_rebase_ext(t->recs + at, m, arena_at - 8, t->sm_count, nullptr, &tally.n);
            arena_at += bytes;
        }
        at += m;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
    if (e != cudaSuccess) {
        tokens_free(t);
        return fail(WFCU_ERR_CUDA, "concat of token slices: %s", cudaGetErrorString(e));
    }
    *out = t;
    return WFCU_OK;
}

// ---- WCX1 frames on the device (frames.cu) ---------------------------------------------------------------------
// encode_message (proj/src/wire.cpp:27-48) of the slice [begin, end) of a device token list, into device memory.
// dev_frame == NULL: only *frame_bytes (what the frame takes).
extern "C" int wfcu_tokens_encode_frame(const wfcu_tokens* t, uint64_t begin, uint64_t end, uint8_t* dev_frame,
                                        uint64_t frame_cap, uint64_t* frame_bytes, void* stream) {
    if (!t || !frame_bytes) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    if (begin > end || end > t->n) return fail(WFCU_ERR_INVALID_ARGUMENT, "slice out of range");
    if (dev_frame && (reinterpret_cast<uintptr_t>(dev_frame) & 3u)) return fail(WFCU_ERR_INVALID_ARGUMENT, "frame buffer must be 4-byte aligned");
    const u64 m = end - begin;
    if (m > 0xFFFFFFFFull) return fail(WFCU_ERR_INVALID_ARGUMENT, "word batch exceeds 2^32-1 words");
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = ensure_text_order(t, s)) return rc;
    DevBuf offs, tmp;
    u64 payload = 0;
    LaunchTally tally;
    if (m) {
        CUDA_TRY(offs.alloc(sizeof(u64) * (m + 1)));
        CUDA_TRY(tmp.alloc(sizeof(u64) * scan_tmp_words(m)));
        CUDA_TRY(frame_lengths(t->recs + begin, m, t->arena, offs.as<u64>(), tmp.as<u64>(), t->sm_count, s, &tally.n));
        // payload bytes = offset of the last token + its length: read the last offset, add the last length on the host
        u64 last_off = 0;
        TokenRec last;
        CUDA_TRY(cudaMemcpyAsync(&last_off, offs.as<u64>() + (m - 1), sizeof(u64), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(&last, t->recs + end - 1, sizeof(TokenRec), cudaMemcpyDeviceToHost, s));
        u32 last_len = 0;
        if (true) {
            CUDA_TRY(cudaStreamSynchronize(s));
            if (last.ext) CUDA_TRY(cudaMemcpy(&last_len, t->arena + last.ext, 4, cudaMemcpyDeviceToHost));
            else last_len = key_len(last.k0, last.k1);
        }
        payload = last_off + last_len;
    }
    *frame_bytes = 8 + 4 * m + payload;
    if (!dev_frame) return WFCU_OK;
    if (frame_cap < *frame_bytes) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "frame needs %llu bytes", (unsigned long long)*frame_bytes);
    if (m == 0) {
        const uint8_t empty[8] = {0x57, 0x43, 0x58, 0x31, 0, 0, 0, 0};
        CUDA_TRY(cudaMemcpyAsync(dev_frame, empty, 8, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return WFCU_OK;
    }
    CUDA_TRY(frame_pack(t->recs + begin, m, t->arena, offs.as<u64>(), dev_frame, t->sm_count, s, &tally.n));
    CUDA_TRY(cudaStreamSynchronize(s));
    return WFCU_OK;
}

// decode_message (proj/src/wire.cpp:50-87) of a frame in device memory: the structural checks of the reference in
// its order (magic, word count, length table, payload short / trailing bytes), the UTF-8 check of the payload as one
// sanitize pass (nothing replaced) plus "no word starts with a continuation byte", and the token list.
extern "C" int wfcu_tokens_decode_frame(const uint8_t* dev_frame, uint64_t frame_bytes, wfcu_tokens** out, void* stream) {
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (frame_bytes && !dev_frame) return fail(WFCU_ERR_INVALID_ARGUMENT, "frame is null");
    if (reinterpret_cast<uintptr_t>(dev_frame) & 3u) return fail(WFCU_ERR_INVALID_ARGUMENT, "frame must be 4-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t head[8] = {0};
    if (frame_bytes) CUDA_TRY(cudaMemcpyAsync(head, dev_frame, std::min<u64>(frame_bytes, 8), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    static const uint8_t magic[4] = {0x57, 0x43, 0x58, 0x31};
    if (frame_bytes < 4 || std::memcmp(head, magic, 4) != 0) return fail(WFCU_ERR_FRAME_MAGIC, "malformed frame: bad magic");
    if (frame_bytes < 8) return fail(WFCU_ERR_FRAME_TRUNCATED, "truncated frame: missing word count");
    u32 count32;
    std::memcpy(&count32, head + 4, 4);
    const u64 m = count32;
    if ((frame_bytes - 8) / 4 < m) return fail(WFCU_ERR_FRAME_TRUNCATED, "truncated frame: missing word lengths");
    const u64 payload_bytes = frame_bytes - 8 - 4 * m;
    auto* t = new wfcu_tokens;
    cudaGetDevice(&t->device);
    t->sm_count = d->sm_count;
    t->n = m;
    struct Guard { wfcu_tokens*& t; ~Guard() { if (t) tokens_free(t); } } guard{t};
    if (m == 0) {
        if (payload_bytes) return fail(WFCU_ERR_FRAME_TRAILING, "framing error: trailing bytes after payload");
        *out = t; t = nullptr;
        return WFCU_OK;
    }
    DevBuf lens, need, tmp, flags, aligned, clean;
    CUDA_TRY(lens.alloc(sizeof(u64) * (m + 1)));
    CUDA_TRY(need.alloc(sizeof(u64) * (m + 1)));
    CUDA_TRY(tmp.alloc(sizeof(u64) * scan_tmp_words(m)));
    CUDA_TRY(flags.alloc(sizeof(int)));
    CUDA_TRY(cudaMemsetAsync(flags.p, 0, sizeof(int), s));
    LaunchTally tally;
    CUDA_TRY(frame_read_lens(dev_frame, m, lens.as<u64>(), need.as<u64>(), d->sm_count, s, &tally.n));
    u64 last[2] = {0, 0}, last_off[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(&last[0], lens.as<u64>() + (m - 1), sizeof(u64), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&last[1], need.as<u64>() + (m - 1), sizeof(u64), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(exclusive_scan_u64(lens.as<u64>(), lens.as<u64>(), m, tmp.as<u64>(), s, &tally.n));
    CUDA_TRY(exclusive_scan_u64(need.as<u64>(), need.as<u64>(), m, tmp.as<u64>(), s, &tally.n));
    CUDA_TRY(cudaMemcpyAsync(&last_off[0], lens.as<u64>() + (m - 1), sizeof(u64), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&last_off[1], need.as<u64>() + (m - 1), sizeof(u64), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const u64 declared = last_off[0] + last[0], arena_bytes = 8 + last_off[1] + last[1];
    if (declared > payload_bytes) return fail(WFCU_ERR_FRAME_TRUNCATED, "truncated frame: payload short of declared lengths");
    if (declared < payload_bytes) return fail(WFCU_ERR_FRAME_TRAILING, "framing error: trailing bytes after payload");
    void* p = nullptr;
    CUDA_TRY(scratch_alloc(&p, sizeof(TokenRec) * m));
    t->recs = static_cast<TokenRec*>(p);
    CUDA_TRY(scratch_alloc(&p, arena_bytes));
    t->arena = static_cast<uint8_t*>(p);
    t->arena_used = t->arena_cap = arena_bytes;
    CUDA_TRY(cudaMemsetAsync(t->arena, 0, 8, s));
    CUDA_TRY(frame_build(dev_frame, m, lens.as<u64>(), need.as<u64>(), t->recs, t->arena, flags.as<int>(), d->sm_count, s, &tally.n));
    int fl = 0;
    CUDA_TRY(cudaMemcpyAsync(&fl, flags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    u64 clean_len = payload_bytes;
    if (payload_bytes) {     // UTF-8: the sanitize pass replaces nothing (its input must be 16-byte aligned: copy)
        CUDA_TRY(aligned.alloc(payload_bytes + 16));
        CUDA_TRY(clean.alloc(3 * payload_bytes + 64));
        CUDA_TRY(cudaMemcpyAsync(aligned.p, dev_frame + 8 + 4 * m, payload_bytes, cudaMemcpyDeviceToDevice, s));
        uint64_t got = 0;
        if (int rc = wfcu_utf8_sanitize_dev(aligned.as<uint8_t>(), payload_bytes, clean.as<uint8_t>(), 3 * payload_bytes + 64, &got, stream)) return rc;
        clean_len = got;
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    if (fl & 1) return fail(WFCU_ERR_INVALID_ARGUMENT, "frame holds an empty word: not a token list");
    if ((fl & 2) || clean_len != payload_bytes) return fail(WFCU_ERR_FRAME_ENCODING, "encoding error: word payload is not UTF-8");
    *out = t; t = nullptr;
    return WFCU_OK;
}

extern "C" int wfcu_tokens_sort(wfcu_tokens* t, void* stream) {
    if (!t) return fail(WFCU_ERR_INVALID_ARGUMENT, "tokens is null");
    {   // sorting by key makes the text order irrelevant: a pending position sort is dropped
        std::lock_guard<std::mutex> lock(t->order_mu);
        t->text_order_pending = false;
    }
    if (int rc = sort_device_tokens(t, /*by_position=*/false, (cudaStream_t)stream)) return rc;
    t->sorted = true;
    return WFCU_OK;
}

extern "C" int wfcu_tokens_reduce_sorted(const wfcu_tokens* t, wfcu_counter* into, void* stream) {
    if (!t || !into) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    if (t->n == 0) return WFCU_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = ensure_text_order(t, s)) return rc;
    DevBuf flags, starts, tmp, status;
    CUDA_TRY(flags.alloc(sizeof(u64) * t->n));
    CUDA_TRY(starts.alloc(sizeof(u64) * t->n));
    CUDA_TRY(tmp.alloc(sizeof(u64) * scan_tmp_words(t->n)));
    CUDA_TRY(status.alloc(sizeof(int)));
    CUDA_TRY(cudaMemsetAsync(status.p, 0, sizeof(int), s));
    LaunchTally tally;
    CUDA_TRY(tokens_rle_flags(t->recs, t->n, t->arena, flags.as<u64>(), status.as<int>(), into->sm_count, s, &tally.n));
    int st = 0;
    CUDA_TRY(cudaMemcpyAsync(&st, status.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    // the reference checks the `sorted` flag (reduce.cpp:9); here the order itself is checked
    if (st & kStatusNotSorted) return fail(WFCU_ERR_NOT_SORTED, "reduce_sorted: word list must be sorted");
    CUDA_TRY(tokens_rle_insert(t->recs, t->n, t->arena, flags.as<u64>(), starts.as<u64>(), tmp.as<u64>(), into->v,
                               into->sm_count, s, &tally.n));
    CUDA_TRY(cudaStreamSynchronize(s));
    return WFCU_OK;
}

extern "C" int wfcu_counter_count_dev_sorted(wfcu_counter* c, const uint8_t* dev_text, uint64_t n, void* stream) {
    if (!c) return fail(WFCU_ERR_INVALID_ARGUMENT, "counter is null");
    if (n == 0) return WFCU_OK;
    wfcu_tokens* t = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    // Tokens of at most 8 bytes (the bulk) leave the tokenizer as 64-bit keys and are sorted and run-length
    // encoded as such; the others keep the 32-byte record path.  Counting does not care about text order, so
    // nothing is sorted by position.
    CompactKeys ck;
    if (int rc = tokenize_unordered(dev_text, n, s, &t, &ck)) return rc;
    int rc = WFCU_OK;
    if (ck.n_keys) {
        const u64 nk = ck.n_keys;
        const u64 hw = 256 * std::max(ck.tiles, sort_n_tiles(nk));
        DevBuf keys_b, hist, tmp, flags, starts;
        LaunchTally tally;
        cudaError_t e = keys_b.alloc(sizeof(u64) * nk);
        if (e == cudaSuccess) e = hist.alloc(sizeof(u64) * hw);
        if (e == cudaSuccess) e = tmp.alloc(sizeof(u64) * std::max(scan_tmp_words(hw), scan_tmp_words(nk)));
        if (e == cudaSuccess) e = flags.alloc(sizeof(u64) * nk);
        if (e == cudaSuccess) e = starts.alloc(sizeof(u64) * nk);
        if (e == cudaSuccess) e = tokens_compact_count(ck.keys.as<u64>(), keys_b.as<u64>(), nk, ck.vary, hist.as<u64>(), tmp.as<u64>(),
                                                        flags.as<u64>(), starts.as<u64>(), c->v, c->sm_count, s, &tally.n,
                                                        ck.tile_counts.as<u32>(), ck.tiles);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            tokens_free(t);
            return fail(WFCU_ERR_CUDA, "count_dev_sorted: %s", cudaGetErrorString(e));
        }
    }
    if (t->n) {   // the longer tokens: records
        rc = sort_device_tokens(t, /*by_position=*/false, s);
        if (rc == WFCU_OK) rc = wfcu_tokens_reduce_sorted(t, c, stream);
    }
    tokens_free(t);
    return rc;
}

// ---- ingest: utf8_sanitize ---------------------------------------------------------------
extern "C" int wfcu_utf8_sanitize_dev(const uint8_t* dev_text, uint64_t n, uint8_t* dev_out, uint64_t out_cap,
                                      uint64_t* out_len, void* stream) {
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (!out_len) return fail(WFCU_ERR_INVALID_ARGUMENT, "out_len is null");
    *out_len = 0;
    if (n == 0) return WFCU_OK;
    if (!dev_text || !dev_out) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    if (reinterpret_cast<uintptr_t>(dev_text) & 15u)
        return fail(WFCU_ERR_INVALID_ARGUMENT, "device text must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    const u64 need = sanitize_scratch_bytes(n);
    if (d->sn_cap < need) {
        CUDA_TRY(cudaDeviceSynchronize());
        if (d->sn_scratch) scratch_free(d->sn_scratch);
        d->sn_scratch = nullptr;
        d->sn_cap = 0;
        CUDA_TRY(scratch_alloc(&d->sn_scratch, need + need / 4));
        d->sn_cap = need + need / 4;
    }
    LaunchTally tally;
    CUDA_TRY(sanitize_launch(dev_text, n, dev_out, out_cap, d->sn_scratch, d->scratch + 32, d->sm_count, s, &tally.n));
    u64 total = 0;
    CUDA_TRY(cudaMemcpyAsync(&total, d->scratch + 32, sizeof(u64), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *out_len = total;
    if (total > out_cap)
        return fail(WFCU_ERR_BUFFER_TOO_SMALL, "utf8_sanitize needs %llu bytes of output", (unsigned long long)total);
    return WFCU_OK;
}

extern "C" int wfcu_utf8_sanitize_host(const uint8_t* text, uint64_t n, uint8_t* out, uint64_t out_cap, uint64_t* out_len) {
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (!out_len) return fail(WFCU_ERR_INVALID_ARGUMENT, "out_len is null");
    *out_len = 0;
    if (n == 0) return WFCU_OK;
    if (!text || !out) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    DevBuf din, dout;
    const u64 cap = std::min<u64>(out_cap, 3 * n);
    CUDA_TRY(din.alloc(n));
    CUDA_TRY(dout.alloc(cap));
    CUDA_TRY(cudaMemcpy(din.p, text, n, cudaMemcpyHostToDevice));
    if (int rc = wfcu_utf8_sanitize_dev(din.as<uint8_t>(), n, dout.as<uint8_t>(), cap, out_len, nullptr)) return rc;
    CUDA_TRY(cudaMemcpy(out, dout.p, *out_len, cudaMemcpyDeviceToHost));
    return WFCU_OK;
}

// normalize_word over a batch of fragments (host buffers).  Fragment f is
// bytes[sum(lens[0..f)) ...]; out_lens[f] = 0 means "nothing remains" (nullopt).
extern "C" int wfcu_normalize_words_host(const uint8_t* bytes, const uint32_t* lens, uint64_t n_frag,
                                         uint8_t* out_bytes, uint64_t out_cap, uint32_t* out_lens) {
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    if (n_frag == 0) return WFCU_OK;
    if (!lens || !out_lens || !out_bytes) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    std::vector<u64> offs(n_frag + 1, 0);
    for (u64 f = 0; f < n_frag; ++f) offs[f + 1] = offs[f] + lens[f];
    const u64 total = offs[n_frag];
    if (total && !bytes) return fail(WFCU_ERR_INVALID_ARGUMENT, "bytes is null");
    DevBuf text, doffs, recs, arena, counters;
    CUDA_TRY(text.alloc(total));
    CUDA_TRY(doffs.alloc(sizeof(u64) * (n_frag + 1)));
    CUDA_TRY(recs.alloc(sizeof(TokenRec) * n_frag));
    const u64 arena_cap = 3 * total + 16 * n_frag + 64;
    CUDA_TRY(arena.alloc(arena_cap));
    CUDA_TRY(counters.alloc(sizeof(u64) * 16));
    if (total) CUDA_TRY(cudaMemcpy(text.p, bytes, total, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(doffs.p, offs.data(), sizeof(u64) * (n_frag + 1), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemset(counters.p, 0, sizeof(u64) * 16));
    u64* cnt = counters.as<u64>();
    const u64 arena_start = 8;
    CUDA_TRY(cudaMemcpy(cnt + 4, &arena_start, sizeof(u64), cudaMemcpyHostToDevice));
    TableView v{};
    v.n_used = cnt + 0; v.n_tokens = cnt + 1; v.n_deferred = cnt + 2; v.n_long = cnt + 3; v.arena_used = cnt + 4;
    v.status = reinterpret_cast<int*>(cnt + 5);
    v.arena = arena.as<uint8_t>(); v.arena_cap = arena_cap;
    EmitView em{recs.as<TokenRec>(), n_frag, cnt + 6};
    LaunchTally tally;
    CUDA_TRY(wc_normalize_launch(text.as<uint8_t>(), doffs.as<u64>(), n_frag, v, em, d->sm_count, nullptr, &tally.n));
    u64 h[8];
    CUDA_TRY(cudaMemcpy(h, cnt, sizeof(h), cudaMemcpyDeviceToHost));
    if (int rc = status_to_rc((int)(h[5] & 0xFFFFFFFFu))) return rc;
    const u64 produced = h[6];
    std::vector<TokenRec> hr(produced);
    std::vector<uint8_t> ha(h[4]);
    if (produced) CUDA_TRY(cudaMemcpy(hr.data(), recs.p, sizeof(TokenRec) * produced, cudaMemcpyDeviceToHost));
    if (h[4] > 8) CUDA_TRY(cudaMemcpy(ha.data(), arena.p, h[4], cudaMemcpyDeviceToHost));
    // records arrive in any order: place each by the fragment its position falls in
    std::vector<const TokenRec*> by_frag(n_frag, nullptr);
    for (const TokenRec& r : hr) {
        const u64 f = u64(std::upper_bound(offs.begin(), offs.end(), r.pos) - offs.begin()) - 1;
        if (f < n_frag) by_frag[f] = &r;
    }
    u64 off = 0;
    for (u64 f = 0; f < n_frag; ++f) {
        out_lens[f] = 0;
        const TokenRec* r = by_frag[f];
        if (!r) continue;
        uint8_t b[16];
        const uint8_t* src = b;
        u32 len;
        if (r->ext) {
            std::memcpy(&len, ha.data() + r->ext, 4);
            src = ha.data() + r->ext + 8;
        } else {
            key_to_bytes(r->k0, r->k1, b);
            len = key_len(r->k0, r->k1);
        }
        if (off + len > out_cap) return fail(WFCU_ERR_BUFFER_TOO_SMALL, "normalize output buffer too small");
        std::memcpy(out_bytes + off, src, len);
        out_lens[f] = len;
        off += len;
    }
    return WFCU_OK;
}

// ---- plain device-memory helpers for hosts that do not link the CUDA runtime --------------
extern "C" int wfcu_dev_alloc(void** out, uint64_t bytes) {
    if (!out) return fail(WFCU_ERR_INVALID_ARGUMENT, "out is null");
    DeviceState* d;
    if (int rc = current_device_state(&d)) return rc;
    CUDA_TRY(scratch_alloc(out, bytes ? bytes : 16));
    return WFCU_OK;
}
extern "C" void wfcu_dev_free(void* p) {
    if (p) scratch_free(p);
}
extern "C" int wfcu_dev_upload(void* dev_dst, const void* host_src, uint64_t bytes) {
    if (bytes) CUDA_TRY(cudaMemcpy(dev_dst, host_src, bytes, cudaMemcpyHostToDevice));
    return WFCU_OK;
}
extern "C" int wfcu_dev_download(void* host_dst, const void* dev_src, uint64_t bytes) {
    if (bytes) CUDA_TRY(cudaMemcpy(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost));
    return WFCU_OK;
}

// ---- analysis over exported tables ---------------------------------------------------------
extern "C" int wfcu_top_k(const uint8_t* key_bytes, const uint32_t* key_lens, const uint64_t* counts, uint64_t n,
                          uint64_t k, uint64_t* out_idx, double* out_rel, uint64_t* total, uint64_t* n_rows) {
    if (!n_rows || !total) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    if (n && (!key_bytes || !key_lens || !counts)) return fail(WFCU_ERR_INVALID_ARGUMENT, "null table");
    if (std::min(n, k) && (!out_idx || !out_rel)) return fail(WFCU_ERR_INVALID_ARGUMENT, "null output");
    *n_rows = analysis_top_k(key_bytes, key_lens, counts, n, k, out_idx, out_rel, total);
    return WFCU_OK;
}

extern "C" int wfcu_distinctive(const uint8_t* t_bytes, const uint32_t* t_lens, const uint64_t* t_counts, uint64_t nt,
                                const uint8_t* o_bytes, const uint32_t* o_lens, const uint64_t* o_counts, uint64_t no,
                                uint64_t k, int32_t* out_src, uint64_t* out_idx, double* out_score, uint64_t* n_rows) {
    if (!n_rows) return fail(WFCU_ERR_INVALID_ARGUMENT, "null argument");
    if ((nt && (!t_bytes || !t_lens || !t_counts)) || (no && (!o_bytes || !o_lens || !o_counts)))
        return fail(WFCU_ERR_INVALID_ARGUMENT, "null table");
    if (std::min(nt + no, k) && (!out_src || !out_idx || !out_score)) return fail(WFCU_ERR_INVALID_ARGUMENT, "null output");
    *n_rows = analysis_distinctive(t_bytes, t_lens, t_counts, nt, o_bytes, o_lens, o_counts, no, k, out_src, out_idx, out_score);
    return WFCU_OK;
}
