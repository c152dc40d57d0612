// sanitize.cu -- utf8_sanitize on the device (the ingest step in front of the hot path).
//
// Replaces wfc::utf8_sanitize (/root/reference/proj/src/unicode.cpp:56-70, called by
// ingest_directory, proj/src/analysis.cpp:53): every byte that strict decoding
// (unicode.cpp:11-44) does not accept as part of a valid sequence becomes U+FFFD (EF BF BD),
// one replacement per byte; valid sequences are copied.
//
// The sequential decoder is local: a lead byte (anything that is not 10xxxxxx) is never
// consumed by an earlier sequence, so every lead is a decode position and its validity
// depends on the next three bytes only; a continuation byte is kept iff the closest lead in
// front of it starts a valid sequence that reaches it.  So:
//   pass A  one thread per 16 bytes (plus a 3-byte halo on both sides): 16-bit keep mask and
//           the output size of the chunk (16 + 2 per replaced byte);
//   scan    exclusive prefix sum of the sizes (tokens.cu);
//   pass B  every thread writes its chunk at its offset: one 16-byte store when nothing was
//           replaced in or before it (the offset is then 16-byte aligned), bytes otherwise.
// HBM traffic: 2 reads + 1 write of the text (3 bytes per input byte) + 12 bytes per 16-byte chunk.
#include "wfcu_dev.cuh"

namespace wfcu {

cudaError_t exclusive_scan_u64(const u64* in, u64* out, u64 n, u64* tmp, cudaStream_t s, u64* launches);   // tokens.cu

namespace {

// length (1..4) of the valid sequence that starts with b0 followed by b1,b2,b3; 0 if invalid.
// Bytes past the end of the text are passed as 0, which no multi-byte sequence accepts.
__device__ __forceinline__ u32 seq_len(u32 b0, u32 b1, u32 b2, u32 b3) {
    if (b0 < 0x80) return 1;
    const bool c1 = (b1 & 0xC0) == 0x80, c2 = (b2 & 0xC0) == 0x80, c3 = (b3 & 0xC0) == 0x80;
    if (b0 >= 0xC2 && b0 <= 0xDF) return c1 ? 2u : 0u;
    if (b0 >= 0xE0 && b0 <= 0xEF) {
        const u32 lo = b0 == 0xE0 ? 0xA0 : 0x80, hi = b0 == 0xED ? 0x9F : 0xBF;
        return (b1 >= lo && b1 <= hi && c2) ? 3u : 0u;
    }
    if (b0 >= 0xF0 && b0 <= 0xF4) {
        const u32 lo = b0 == 0xF0 ? 0x90 : 0x80, hi = b0 == 0xF4 ? 0x8F : 0xBF;
        return (b1 >= lo && b1 <= hi && c2 && c3) ? 4u : 0u;
    }
    return 0;
}

// the lane's 16 bytes (zero past n) and the 4 bytes on either side
struct Window {
    u32 prev, w[4], next;
};
__device__ __forceinline__ u32 load_word(const uint8_t* text, u64 n, u64 at) {   // 4 bytes at `at`, zero past n
    if (at + 4 <= n) return *reinterpret_cast<const u32*>(text + at);
    u32 v = 0;
    for (u32 k = 0; k < 4; ++k)
        if (at + k < n) v |= (u32)text[at + k] << (8 * k);
    return v;
}
__device__ __forceinline__ Window load_window(const uint8_t* __restrict__ text, u64 n, u64 chunk) {
    Window win;
    const u64 g = chunk * 16;
    if (g + 16 <= n) {
        const uint4 v = *reinterpret_cast<const uint4*>(text + g);
        win.w[0] = v.x; win.w[1] = v.y; win.w[2] = v.z; win.w[3] = v.w;
    } else {
        for (u32 k = 0; k < 4; ++k) win.w[k] = load_word(text, n, g + 4 * k);
    }
    win.prev = g ? *reinterpret_cast<const u32*>(text + g - 4) : 0u;
    win.next = load_word(text, n, g + 16);
    return win;
}
__device__ __forceinline__ u32 byte_at(const Window& win, int i) {   // i in [-4, 20)
    const u32 word = i < 0 ? win.prev : i >= 16 ? win.next : win.w[i >> 2];
    return (word >> (8 * (i & 3))) & 0xFF;
}

// bit i set <=> byte i of the chunk is copied (part of a valid sequence)
__device__ __forceinline__ u32 keep_mask(const Window& win) {
    const u32 any_hi = (win.prev | win.w[0] | win.w[1] | win.w[2] | win.w[3] | win.next) & 0x80808080u;
    if (!any_hi) return 0xFFFFu;
    u32 keep = 0;
#pragma unroll
    for (int q = -3; q < 16; ++q) {
        const u32 b0 = byte_at(win, q);
        if ((b0 & 0xC0) == 0x80) continue;     // not a lead: never a decode position that starts a sequence
        const u32 len = seq_len(b0, byte_at(win, q + 1), byte_at(win, q + 2), byte_at(win, q + 3));
        const u32 bits = ((1u << len) - 1u);   // bytes q .. q+len-1
        keep |= q >= 0 ? (bits << q) : (bits >> (-q));
    }
    return keep & 0xFFFFu;
}

__global__ void sn_sizes_kernel(const uint8_t* __restrict__ text, u64 n, u64 n_chunks, u32* __restrict__ masks,
                                u64* __restrict__ sizes) {
    for (u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x; c < n_chunks; c += (u64)gridDim.x * blockDim.x) {
        const Window win = load_window(text, n, c);
        const u64 g = c * 16;
        const u32 valid = n - g >= 16 ? 16u : (u32)(n - g);           // bytes of the chunk inside the text
        const u32 in_text = valid == 16 ? 0xFFFFu : ((1u << valid) - 1u);
        const u32 keep = keep_mask(win) & in_text;
        masks[c] = keep;
        sizes[c] = valid + 2 * (valid - __popc(keep));
    }
}

__global__ void sn_write_kernel(const uint8_t* __restrict__ text, u64 n, u64 n_chunks, const u32* __restrict__ masks,
                                const u64* __restrict__ offs, uint8_t* __restrict__ out, u64 out_cap,
                                u64* __restrict__ total) {
    for (u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x; c < n_chunks; c += (u64)gridDim.x * blockDim.x) {
        const u64 g = c * 16, at = offs[c];
        const u32 valid = n - g >= 16 ? 16u : (u32)(n - g);
        const u32 keep = masks[c];
        const u64 size = valid + 2 * (valid - __popc(keep));
        if (c + 1 == n_chunks) *total = at + size;
        if (at + size > out_cap) continue;                            // reported through *total
        if (valid == 16 && keep == 0xFFFFu && (at & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
            *reinterpret_cast<uint4*>(out + at) = *reinterpret_cast<const uint4*>(text + g);
            continue;
        }
        uint8_t* o = out + at;
        for (u32 i = 0; i < valid; ++i) {
            if ((keep >> i) & 1u) {
                *o++ = text[g + i];
            } else {
                o[0] = 0xEF; o[1] = 0xBF; o[2] = 0xBD;
                o += 3;
            }
        }
    }
}

}  // namespace

u64 sanitize_scratch_bytes(u64 n);
u64 scan_tmp_words(u64 n);

// scratch layout: sizes/offs u64[n_chunks] | scan tmp | masks u32[n_chunks]
u64 sanitize_scratch_bytes(u64 n) {
    const u64 chunks = (n + 15) / 16;
    return sizeof(u64) * chunks + sizeof(u64) * scan_tmp_words(chunks) + sizeof(u32) * chunks + 64;
}

cudaError_t sanitize_launch(const uint8_t* text, u64 n, uint8_t* out, u64 out_cap, void* scratch, u64* dev_total,
                            int sm_count, cudaStream_t s, u64* launches) {
    if (n == 0) return cudaMemsetAsync(dev_total, 0, sizeof(u64), s);
    const u64 chunks = (n + 15) / 16;
    u64* sizes = static_cast<u64*>(scratch);
    u64* tmp = sizes + chunks;
    u32* masks = reinterpret_cast<u32*>(tmp + scan_tmp_words(chunks));
    u64 g = (chunks + 255) / 256;
    if (g > (u64)sm_count * 16) g = (u64)sm_count * 16;
    sn_sizes_kernel<<<(unsigned)g, 256, 0, s>>>(text, n, chunks, masks, sizes);
    *launches += 1;
    cudaError_t e = exclusive_scan_u64(sizes, sizes, chunks, tmp, s, launches);
    if (e != cudaSuccess) return e;
    sn_write_kernel<<<(unsigned)g, 256, 0, s>>>(text, n, chunks, masks, sizes, out, out_cap, dev_total);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace wfcu
