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
//   pass A  one thread per 16 bytes (plus a 3-byte halo on both sides): 16-bit keep mask; the
//           output size (16 + 2 per replaced byte) is summed per CTA (4 KiB of input);
//   scan    exclusive prefix sum of the CTA sizes (tokens.cu);
//   pass B  every CTA rebuilds its output in shared memory, placed so that shared and global
//           addresses agree modulo 16, and writes it with 16-byte stores whatever the offset.
// HBM traffic: 2 reads + 1 write of the text + 2 bytes per 16-byte chunk: ~3.25 bytes per input byte.
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

constexpr int kSnThreads = 256;
constexpr int kSnBlockBytes = kSnThreads * 16;        // input bytes per CTA
constexpr int kSnStageBytes = 3 * kSnBlockBytes + 32; // worst case output of a CTA + alignment slack

// pass A: keep masks (16 bits per 16-byte chunk) and the output size of every 4 KiB block
__global__ void __launch_bounds__(kSnThreads)
sn_sizes_kernel(const uint8_t* __restrict__ text, u64 n, u64 n_blocks, uint16_t* __restrict__ masks,
                u64* __restrict__ block_sizes) {
    __shared__ u32 warp_sums[kSnThreads / 32];
    for (u64 b = blockIdx.x; b < n_blocks; b += gridDim.x) {
        const u64 c = b * kSnThreads + threadIdx.x;
        const u64 g = c * 16;
        u32 size = 0;
        if (g < n) {
            const Window win = load_window(text, n, c);
            const u32 valid = n - g >= 16 ? 16u : (u32)(n - g);       // bytes of the chunk inside the text
            const u32 in_text = valid == 16 ? 0xFFFFu : ((1u << valid) - 1u);
            const u32 keep = keep_mask(win) & in_text;
            masks[c] = (uint16_t)keep;
            size = valid + 2 * (valid - __popc(keep));
        }
        for (int d = 16; d > 0; d >>= 1) size += __shfl_xor_sync(0xFFFFFFFFu, size, d);
        if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = size;
        __syncthreads();
        if (threadIdx.x == 0) {
            u32 total = 0;
            for (int w = 0; w < kSnThreads / 32; ++w) total += warp_sums[w];
            block_sizes[b] = total;
        }
        __syncthreads();
    }
}

// pass B: every CTA builds the output of its 4 KiB in shared memory -- placed so that shared and
// global addresses agree modulo 16 -- and writes it with 16-byte stores (bytes at the two ends)
__global__ void __launch_bounds__(kSnThreads)
sn_write_kernel(const uint8_t* __restrict__ text, u64 n, u64 n_blocks, const uint16_t* __restrict__ masks,
                const u64* __restrict__ block_offs, uint8_t* __restrict__ out, u64 out_cap, u64* __restrict__ total) {
    __shared__ __align__(16) uint8_t stage[kSnStageBytes];
    __shared__ u32 warp_sums[kSnThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (u64 b = blockIdx.x; b < n_blocks; b += gridDim.x) {
        const u64 c = b * kSnThreads + threadIdx.x;
        const u64 g = c * 16;
        const u64 boff = block_offs[b];
        u32 valid = 0, keep = 0;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (g < n) {
            valid = n - g >= 16 ? 16u : (u32)(n - g);
            keep = masks[c];
            if (valid == 16) v = *reinterpret_cast<const uint4*>(text + g);
            else {
                u32 w[4];
                for (u32 k = 0; k < 4; ++k) w[k] = load_word(text, n, g + 4 * k);
                v = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        // a CTA whose 4 KiB hold nothing to replace (all of a valid text's) and whose output is 16-byte aligned copies
        // its registers out: no staging, no scan
        if (__syncthreads_and(valid == 16 && keep == 0xFFFFu) && ((reinterpret_cast<uintptr_t>(out) + boff) & 15) == 0) {
            if (boff + kSnBlockBytes <= out_cap) *reinterpret_cast<uint4*>(out + boff + 16 * threadIdx.x) = v;
            if (b + 1 == n_blocks && threadIdx.x == 0) *total = boff + kSnBlockBytes;
            continue;
        }
        const u32 size = valid + 2 * (valid - __popc(keep));
        // exclusive scan of the chunk sizes inside the CTA
        u32 incl = size;
        for (int d = 1; d < 32; d <<= 1) {
            const u32 t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) warp_sums[warp] = incl;
        __syncthreads();
        u32 base = 0, bsize = 0;
        for (int w = 0; w < kSnThreads / 32; ++w) {
            if (w < warp) base += warp_sums[w];
            bsize += warp_sums[w];
        }
        const u32 shift = (u32)((reinterpret_cast<uintptr_t>(out) + boff) & 15);   // stage[shift + j] = output byte j
        uint8_t* o = stage + shift + base + incl - size;
        const u32 words[4] = {v.x, v.y, v.z, v.w};
        const u32 ofs = shift + base + incl - size;
        if (keep == 0xFFFFu && (ofs & 3) == 0) {
            u32* o4 = reinterpret_cast<u32*>(o);
            o4[0] = v.x; o4[1] = v.y; o4[2] = v.z; o4[3] = v.w;
        } else if (keep == 0xFFFFu && (ofs & 1) == 0) {       // every replacement shifts the output by 2
            uint16_t* o2 = reinterpret_cast<uint16_t*>(o);
#pragma unroll
            for (u32 i = 0; i < 8; ++i) o2[i] = (uint16_t)(words[i >> 1] >> (16 * (i & 1)));
        } else {
#pragma unroll
            for (u32 i = 0; i < 16; ++i) {
                if (i < valid) {
                    if ((keep >> i) & 1u) {
                        *o++ = (uint8_t)(words[i >> 2] >> (8 * (i & 3)));
                    } else {
                        o[0] = 0xEF; o[1] = 0xBF; o[2] = 0xBD;
                        o += 3;
                    }
                }
            }
        }
        __syncthreads();
        if (b + 1 == n_blocks && threadIdx.x == 0) *total = boff + bsize;
        if (boff + bsize <= out_cap) {
            // [shift, shift + bsize) of the stage -> out[boff, boff + bsize)
            const u32 begin = shift, end = shift + bsize;
            const u32 mid_begin = min((begin + 15u) & ~15u, end), mid_end = max(end & ~15u, mid_begin);
            uint8_t* gout = out + boff - shift;                        // gout + s is the global address of stage[s]
            for (u32 s2 = begin + threadIdx.x; s2 < mid_begin; s2 += kSnThreads) gout[s2] = stage[s2];
            for (u32 s2 = mid_begin + 16 * threadIdx.x; s2 < mid_end; s2 += 16 * kSnThreads)
                *reinterpret_cast<uint4*>(gout + s2) = *reinterpret_cast<const uint4*>(stage + s2);
            for (u32 s2 = mid_end + threadIdx.x; s2 < end; s2 += kSnThreads) gout[s2] = stage[s2];
        }
        __syncthreads();
    }
}

}  // namespace

u64 sanitize_scratch_bytes(u64 n);
u64 scan_tmp_words(u64 n);

// scratch layout: block sizes/offsets u64[n_blocks] | scan tmp | masks u16[n_chunks]
u64 sanitize_scratch_bytes(u64 n) {
    const u64 blocks = (n + kSnBlockBytes - 1) / kSnBlockBytes;
    return sizeof(u64) * blocks + sizeof(u64) * scan_tmp_words(blocks) + sizeof(uint16_t) * blocks * kSnThreads + 64;
}

cudaError_t sanitize_launch(const uint8_t* text, u64 n, uint8_t* out, u64 out_cap, void* scratch, u64* dev_total,
                            int sm_count, cudaStream_t s, u64* launches) {
    if (n == 0) return cudaMemsetAsync(dev_total, 0, sizeof(u64), s);
    const u64 blocks = (n + kSnBlockBytes - 1) / kSnBlockBytes;
    u64* sizes = static_cast<u64*>(scratch);
    u64* tmp = sizes + blocks;
    uint16_t* masks = reinterpret_cast<uint16_t*>(tmp + scan_tmp_words(blocks));
    u64 g = blocks;
    if (g > (u64)sm_count * 8) g = (u64)sm_count * 8;
    sn_sizes_kernel<<<(unsigned)g, kSnThreads, 0, s>>>(text, n, blocks, masks, sizes);
    *launches += 1;
    cudaError_t e = exclusive_scan_u64(sizes, sizes, blocks, tmp, s, launches);
    if (e != cudaSuccess) return e;
    sn_write_kernel<<<(unsigned)g, kSnThreads, 0, s>>>(text, n, blocks, masks, sizes, out, out_cap, dev_total);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace wfcu
