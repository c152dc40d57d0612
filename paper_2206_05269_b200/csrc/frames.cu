// frames.cu -- WCX1 frames built and parsed ON THE DEVICE (the paper's range exchange with a
// NCCL-backed transport and the WCX1 frame as wire format).
//
// Frame layout (/root/reference/proj/include/wfc/wire.hpp, proj/src/wire.cpp:27-48): "WCX1", u32-LE word count,
// u32-LE byte length of every word, the word payloads; nothing may follow.  The reference builds frames from
// std::string vectors on the host; here a frame is the image of a slice of a device token list (TokenRec: the first
// 16 bytes of the token as a big-endian key, longer tokens in the list's arena) and never exists in host memory:
// exchange.range_partition_exchange hands the device buffers to NCCL.
#include "wfcu_dev.cuh"

namespace wfcu {

cudaError_t exclusive_scan_u64(const u64* in, u64* out, u64 n, u64* tmp, cudaStream_t s, u64* launches);   // tokens.cu

namespace {

__device__ __forceinline__ u32 rec_len(const TokenRec& r, const uint8_t* __restrict__ arena) {
    if (r.ext) return *reinterpret_cast<const u32*>(arena + r.ext);
    // bytes are packed first-byte-most-significant and zero padded; a token never ends in NUL
    return r.k1 ? 16u - ((u32)(__ffsll((long long)r.k1) - 1) >> 3) : 8u - ((u32)(__ffsll((long long)r.k0) - 1) >> 3);
}

// lens[i] = byte length of token i of the slice
__global__ void fr_lens_kernel(const TokenRec* __restrict__ recs, u64 m, const uint8_t* __restrict__ arena, u64* __restrict__ lens) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x)
        lens[i] = rec_len(recs[i], arena);
}

// header, length table and payload; offs = exclusive scan of the lengths
__global__ void fr_pack_kernel(const TokenRec* __restrict__ recs, u64 m, const uint8_t* __restrict__ arena,
                               const u64* __restrict__ offs, uint8_t* __restrict__ frame) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        frame[0] = 0x57; frame[1] = 0x43; frame[2] = 0x58; frame[3] = 0x31;
        *reinterpret_cast<u32*>(frame + 4) = (u32)m;
    }
    u32* lens = reinterpret_cast<u32*>(frame + 8);
    uint8_t* payload = frame + 8 + 4 * m;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
        const TokenRec r = recs[i];
        const u32 len = rec_len(r, arena);
        lens[i] = len;
        uint8_t* out = payload + offs[i];
        if (r.ext) {
            const uint8_t* src = arena + r.ext + 8;
            for (u32 b = 0; b < len; ++b) out[b] = src[b];
        } else {
            for (u32 b = 0; b < len; ++b) out[b] = (uint8_t)((b < 8 ? r.k0 >> (56 - 8 * b) : r.k1 >> (120 - 8 * b)) & 0xFF);
        }
    }
}

// the length table of a received frame, widened; arena_need[i] = bytes token i takes in the arena (0: inline)
__global__ void fr_read_lens_kernel(const uint8_t* __restrict__ frame, u64 m, u64* __restrict__ lens, u64* __restrict__ arena_need) {
    const u32* table = reinterpret_cast<const u32*>(frame + 8);
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
        const u32 len = table[i];
        lens[i] = len;
        arena_need[i] = len > 16 ? 8 + (((u64)len + 7) & ~7ull) : 0;
    }
}

// records (and arena records) of a received frame.  flags: bit 0 = an empty word, bit 1 = a word starts inside a
// UTF-8 sequence (its first byte is a continuation byte).
__global__ void fr_build_kernel(const uint8_t* __restrict__ frame, u64 m, const u64* __restrict__ offs,
                                const u64* __restrict__ arena_offs, TokenRec* __restrict__ recs, uint8_t* __restrict__ arena,
                                int* __restrict__ flags) {
    const u32* table = reinterpret_cast<const u32*>(frame + 8);
    const uint8_t* payload = frame + 8 + 4 * m;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
        const u32 len = table[i];
        const uint8_t* p = payload + offs[i];
        if (len == 0) { atomicOr(flags, 1); recs[i] = TokenRec{0, 0, 0, i}; continue; }
        if ((p[0] & 0xC0) == 0x80) atomicOr(flags, 2);
        TokenRec r{0, 0, 0, i};
        key_from_bytes(p, len < 16 ? len : 16, &r.k0, &r.k1);
        if (len > 16) {
            const u64 at = 8 + arena_offs[i];
            u32 h = 2166136261u;
            for (u32 b = 0; b < len; ++b) { arena[at + 8 + b] = p[b]; h = (h ^ p[b]) * 16777619u; }
            for (u64 b = len; b < (((u64)len + 7) & ~7ull); ++b) arena[at + 8 + b] = 0;
            *reinterpret_cast<u32*>(arena + at) = len;
            *reinterpret_cast<u32*>(arena + at + 4) = h;
            r.ext = at;
        }
        recs[i] = r;
    }
}

inline unsigned grid_for(u64 items, int sm_count) {
    u64 g = (items + 255) / 256;
    const u64 cap = (u64)sm_count * 8;
    if (g > cap) g = cap;
    return (unsigned)(g ? g : 1);
}

}  // namespace

// lens_scan: scratch of m u64; tmp: scan scratch.  After the call lens_scan holds the payload offsets.
cudaError_t frame_lengths(const TokenRec* recs, u64 m, const uint8_t* arena, u64* lens_scan, u64* tmp, int sm, cudaStream_t s,
                          u64* launches) {
    if (m == 0) return cudaSuccess;
    fr_lens_kernel<<<grid_for(m, sm), 256, 0, s>>>(recs, m, arena, lens_scan);
    *launches += 1;
    return exclusive_scan_u64(lens_scan, lens_scan, m, tmp, s, launches);
}
cudaError_t frame_pack(const TokenRec* recs, u64 m, const uint8_t* arena, const u64* offs, uint8_t* frame, int sm, cudaStream_t s,
                       u64* launches) {
    fr_pack_kernel<<<grid_for(m, sm), 256, 0, s>>>(recs, m, arena, offs, frame);
    *launches += 1;
    return cudaGetLastError();
}
cudaError_t frame_read_lens(const uint8_t* frame, u64 m, u64* lens, u64* arena_need, int sm, cudaStream_t s, u64* launches) {
    if (m == 0) return cudaSuccess;
    fr_read_lens_kernel<<<grid_for(m, sm), 256, 0, s>>>(frame, m, lens, arena_need);
    *launches += 1;
    return cudaGetLastError();
}
cudaError_t frame_build(const uint8_t* frame, u64 m, const u64* offs, const u64* arena_offs, TokenRec* recs, uint8_t* arena,
                        int* flags, int sm, cudaStream_t s, u64* launches) {
    if (m == 0) return cudaSuccess;
    fr_build_kernel<<<grid_for(m, sm), 256, 0, s>>>(frame, m, offs, arena_offs, recs, arena, flags);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace wfcu
