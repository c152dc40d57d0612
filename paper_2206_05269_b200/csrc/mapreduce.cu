// mapreduce.cu -- generic map-then-reduce on sm_100a.
//
// Replaces /root/reference/proj/src/engine.cpp:15-98 (fold_range, combine_tree,
// blocked_sum, map_value, map_reduce_serial/blocked, alternating_harmonic).
//
//  * mr_partial_kernel + mr_final_kernel (K6): HBM-bound streaming reduction.
//    Grid-stride over 16-byte vectors (ld.global.nc.v4), four independent fp64
//    accumulators per thread, warp-shuffle tree, per-CTA partial, then a
//    single-CTA fixed-order pass over the partials.  No floating-point atomics:
//    element -> thread assignment and every combination order are fixed by
//    (n, grid), so the result is bitwise reproducible run to run.
//  * mr_block_fold_{warp,cta}_kernel + mr_tree_level_kernel: the reference's blocked engine
//    reproduced bit for bit -- one thread folds one block left to right with
//    separately rounded operations (no FMA contraction) out of a shared tile that the
//    whole warp / CTA fills with coalesced loads, then the pairwise tree of combine_tree
//    is applied level by level.
#include <cuda_runtime.h>
#include <stdint.h>

namespace wfcu {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr int kMapIdentity = 0, kMapSqrt = 1, kMapAltHarm = 2, kMapSquare = 3;
constexpr int kMrThreads = 256;

template <int KIND>
__device__ __forceinline__ double map_term(double v, u64 position) {
    if (KIND == kMapIdentity) return v;
    if (KIND == kMapSqrt) return __dsqrt_rn(v);
    if (KIND == kMapSquare) return __dmul_rn(v, v);
    return __ddiv_rn((position & 1ull) ? 1.0 : -1.0, (double)position);
}

__device__ __forceinline__ float4 ldg_nc_f4(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ldg_nc_d2(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

__device__ __forceinline__ double block_sum(double v, double* warp_sums) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, d);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) warp_sums[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (warp == 0) {
        r = (lane < (int)(blockDim.x >> 5)) ? warp_sums[lane] : 0.0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) r += __shfl_down_sync(0xFFFFFFFFu, r, d);
    }
    return r;   // valid in thread 0
}

// T = float or double; values 16-byte aligned.
template <typename T, int KIND>
__global__ void __launch_bounds__(kMrThreads)
mr_partial_kernel(const T* __restrict__ values, u64 n, u64 position_base, double* __restrict__ partials) {
    constexpr int VEC = 16 / sizeof(T);
    __shared__ double warp_sums[kMrThreads / 32];
    const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    const u64 nthreads = (u64)gridDim.x * blockDim.x;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;

    if (KIND == kMapAltHarm) {
        // value ignored: no memory traffic at all
        for (u64 i = tid; i < n; i += nthreads) a0 += map_term<KIND>(0.0, position_base + i + 1);
    } else {
        const u64 nvec = n / VEC;
        // 4 vectors in flight per thread per iteration
        u64 v = tid;
        for (; v + 3 * nthreads < nvec; v += 4 * nthreads) {
            if (sizeof(T) == 4) {
                const float4* p = reinterpret_cast<const float4*>(values);
                const float4 x0 = ldg_nc_f4(p + v), x1 = ldg_nc_f4(p + v + nthreads);
                const float4 x2 = ldg_nc_f4(p + v + 2 * nthreads), x3 = ldg_nc_f4(p + v + 3 * nthreads);
                a0 += map_term<KIND>(x0.x, 0); a1 += map_term<KIND>(x0.y, 0); a2 += map_term<KIND>(x0.z, 0); a3 += map_term<KIND>(x0.w, 0);
                a0 += map_term<KIND>(x1.x, 0); a1 += map_term<KIND>(x1.y, 0); a2 += map_term<KIND>(x1.z, 0); a3 += map_term<KIND>(x1.w, 0);
                a0 += map_term<KIND>(x2.x, 0); a1 += map_term<KIND>(x2.y, 0); a2 += map_term<KIND>(x2.z, 0); a3 += map_term<KIND>(x2.w, 0);
                a0 += map_term<KIND>(x3.x, 0); a1 += map_term<KIND>(x3.y, 0); a2 += map_term<KIND>(x3.z, 0); a3 += map_term<KIND>(x3.w, 0);
            } else {
                const double2* p = reinterpret_cast<const double2*>(values);
                const double2 x0 = ldg_nc_d2(p + v), x1 = ldg_nc_d2(p + v + nthreads);
                const double2 x2 = ldg_nc_d2(p + v + 2 * nthreads), x3 = ldg_nc_d2(p + v + 3 * nthreads);
                a0 += map_term<KIND>(x0.x, 0); a1 += map_term<KIND>(x0.y, 0);
                a2 += map_term<KIND>(x1.x, 0); a3 += map_term<KIND>(x1.y, 0);
                a0 += map_term<KIND>(x2.x, 0); a1 += map_term<KIND>(x2.y, 0);
                a2 += map_term<KIND>(x3.x, 0); a3 += map_term<KIND>(x3.y, 0);
            }
        }
        for (; v < nvec; v += nthreads) {
#pragma unroll
            for (int k = 0; k < VEC; ++k) a0 += map_term<KIND>((double)values[v * VEC + k], 0);
        }
        // scalar tail
        for (u64 i = nvec * VEC + tid; i < n; i += nthreads) a1 += map_term<KIND>((double)values[i], 0);
    }
    const double s = block_sum((a0 + a1) + (a2 + a3), warp_sums);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// Single CTA, fixed order: thread t sums partials t, t+T, ... then the CTA tree.
__global__ void __launch_bounds__(kMrThreads)
mr_final_kernel(const double* __restrict__ partials, int n_partials, double* __restrict__ out) {
    __shared__ double warp_sums[kMrThreads / 32];
    double a = 0.0;
    for (int i = threadIdx.x; i < n_partials; i += blockDim.x) a += partials[i];
    const double s = block_sum(a, warp_sums);
    if (threadIdx.x == 0) *out = s;
}

// ---- bit-exact blocked engine ----------------------------------------------------
// partials[b] = fold_range(b*block, min((b+1)*block, n))   (engine.cpp:15-20, 44-50): every block is folded left to
// right by ONE thread with separately rounded operations -- the order of the additions is the result.  What is
// parallel is the memory side:
//  * short blocks (mr_block_fold_warp_kernel): a warp owns 32 consecutive blocks.  Per round it loads 32 elements of
//    each block with coalesced 32-lane loads into a padded shared tile (a transposition), then every lane folds the
//    32 elements of ITS block from the tile.  The first version let every thread read its own block straight from
//    global memory: 2 KiB between the lanes of a load at block_size 256, 32 sectors per instruction.
//  * long blocks (mr_block_fold_cta_kernel; map_reduce_serial is one block covering the array): a CTA per block,
//    127 threads load the next chunk and apply the map while thread 0 adds up the previous one -- the chain of
//    dependent DADDs (about 10 cycles each) is then the only thing on the critical path: 1.4 s for 2^28 values, whatever
//    the map (the square root took 12.7 s while the folding thread computed it too).  A CPU core adds in 4 cycles
//    at twice the clock: the reference's serial fold takes 0.29 s.  That gap is the price of bit-identity with a
//    sequential fp64 sum; map_reduce_blocked and map_reduce_fast are the parallel forms.
constexpr int kFoldTile = 32;
template <typename T, int KIND>
__global__ void __launch_bounds__(128)
mr_block_fold_warp_kernel(const T* __restrict__ values, u64 n, u64 position_base, u64 block, u64 n_blocks,
                          double* __restrict__ partials) {
    __shared__ double tile[4][kFoldTile][kFoldTile + 1];
    const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double (*my)[kFoldTile + 1] = tile[warp];
    const u64 warps_total = (u64)gridDim.x * 4, gw = (u64)blockIdx.x * 4 + warp;
    for (u64 b0 = gw * 32; b0 < n_blocks; b0 += warps_total * 32) {
        const u32 kmax = (u32)((n_blocks - b0 < 32) ? (n_blocks - b0) : 32);     // blocks of this warp
        const u64 lo = (b0 + lane) * block;                                        // this lane's block
        u64 hi = lo + block;
        if (hi > n || hi < lo) hi = n;
        const u64 len = (lane < kmax && hi > lo) ? hi - lo : 0;
        double acc = 0.0;
        for (u64 r = 0; r < block; r += kFoldTile) {
            if (KIND != kMapAltHarm) {
                for (u32 k = 0; k < kmax; ++k) {                                   // coalesced: 32 lanes, one block
                    const u64 i = (b0 + k) * block + r + lane;
                    const u64 end = ((b0 + k) * block + block < n) ? (b0 + k) * block + block : n;
                    my[k][lane] = (r + lane < block && i < end) ? (double)values[i] : 0.0;
                }
                __syncwarp();
            }
            const u64 left = len > r ? len - r : 0;
            const u32 m = (u32)(left < kFoldTile ? left : kFoldTile);
            for (u32 j = 0; j < m; ++j) {
                const double v = (KIND == kMapAltHarm) ? 0.0 : my[lane][j];
                acc = __dadd_rn(acc, map_term<KIND>(v, position_base + lo + r + j + 1));
            }
            __syncwarp();
        }
        if (lane < kmax) partials[b0 + lane] = acc;
    }
}

constexpr int kFoldChunk = 2048;     // elements per shared tile of the long-block kernel
template <typename T, int KIND>
__global__ void __launch_bounds__(128)
mr_block_fold_cta_kernel(const T* __restrict__ values, u64 n, u64 position_base, u64 block, u64 n_blocks,
                         double* __restrict__ partials) {
    // the MAPPED terms of two chunks: warps 1..3 load chunk c+1 (coalesced) and apply the map -- the square root
    // is a long instruction sequence, but every term is independent -- while thread 0 adds up chunk c
    __shared__ __align__(16) double term[2][kFoldChunk];
    for (u64 b = blockIdx.x; b < n_blocks; b += gridDim.x) {
        const u64 lo = b * block;
        u64 hi = lo + block;
        if (hi > n || hi < lo) hi = n;
        const u64 chunks = (hi - lo + kFoldChunk - 1) / kFoldChunk;
        double acc = 0.0;
        auto stage = [&](u64 c, u32 first_thread) {          // chunk c of the block -> term[c & 1]
            const u64 first = lo + c * kFoldChunk;
            const u32 count = (u32)((hi - first < (u64)kFoldChunk) ? hi - first : (u64)kFoldChunk);
            double* dst = term[c & 1];
            for (u32 i = threadIdx.x - first_thread; i < count; i += blockDim.x - first_thread) {
                const double v = (KIND == kMapAltHarm) ? 0.0 : (double)values[first + i];
                dst[i] = map_term<KIND>(v, position_base + first + i + 1);
            }
        };
        if (chunks) stage(0, 0);
        for (u64 c = 0; c < chunks; ++c) {
            __syncthreads();                       // chunk c is mapped, chunk c-1 has been added up
            if (threadIdx.x == 0) {
                const u64 first = lo + c * kFoldChunk;
                const u32 count = (u32)((hi - first < (u64)kFoldChunk) ? hi - first : (u64)kFoldChunk);
                const double* src = term[c & 1];
                u32 j = 0;
                for (; j + 16 <= count; j += 16) {     // the loads run ahead of the chain of additions
                    double v[16];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const double2 two = reinterpret_cast<const double2*>(src + j)[q];
                        v[2 * q] = two.x;
                        v[2 * q + 1] = two.y;
                    }
#pragma unroll
                    for (int q = 0; q < 16; ++q) acc = __dadd_rn(acc, v[q]);
                }
                for (; j < count; ++j) acc = __dadd_rn(acc, src[j]);
            } else if (threadIdx.x >= 32 && c + 1 < chunks) {     // warp 0 is the adding thread's alone: no divergent twin
                stage(c + 1, 32);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) partials[b] = acc;
    }
}

// one round of combine_tree (engine.cpp:25-32): out[i] = in[2i] + in[2i+1], odd tail carried
__global__ void mr_tree_level_kernel(const double* __restrict__ in, u64 m, double* __restrict__ out) {
    const u64 half = m / 2;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < half + (m & 1ull); i += (u64)gridDim.x * blockDim.x) {
        out[i] = (i < half) ? __dadd_rn(in[2 * i], in[2 * i + 1]) : in[m - 1];
    }
}

// ---- launchers -------------------------------------------------------------------
template <typename T>
static cudaError_t launch_partial(const T* v, u64 n, u64 base, int kind, int grid, double* partials, cudaStream_t s) {
    switch (kind) {
        case kMapIdentity: mr_partial_kernel<T, kMapIdentity><<<grid, kMrThreads, 0, s>>>(v, n, base, partials); break;
        case kMapSqrt: mr_partial_kernel<T, kMapSqrt><<<grid, kMrThreads, 0, s>>>(v, n, base, partials); break;
        case kMapAltHarm: mr_partial_kernel<T, kMapAltHarm><<<grid, kMrThreads, 0, s>>>(v, n, base, partials); break;
        case kMapSquare: mr_partial_kernel<T, kMapSquare><<<grid, kMrThreads, 0, s>>>(v, n, base, partials); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// partials: device scratch of at least `grid` doubles.  dev_out: device double.
cudaError_t mr_launch(const void* values, int is_f64, u64 n, u64 base, int kind, int grid, double* partials,
                      double* dev_out, cudaStream_t s, u64* launches) {
    cudaError_t e = is_f64 ? launch_partial(static_cast<const double*>(values), n, base, kind, grid, partials, s)
                           : launch_partial(static_cast<const float*>(values), n, base, kind, grid, partials, s);
    if (e != cudaSuccess) return e;
    mr_final_kernel<<<1, kMrThreads, 0, s>>>(partials, grid, dev_out);
    *launches += 2;
    return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_fold(const T* v, u64 n, u64 base, int kind, u64 block, u64 nb, double* partials, int sm_count,
                               cudaStream_t s) {
    const bool long_blocks = block >= 1024;     // a CTA per block pays once a block is many shared tiles long
    u64 g = long_blocks ? nb : (nb + 127) / 128;
    if (g > (u64)sm_count * 16) g = (u64)sm_count * 16;
    const unsigned grid = (unsigned)(g ? g : 1);
#define WFCU_FOLD(K)                                                                                         \
    if (long_blocks) mr_block_fold_cta_kernel<T, K><<<grid, 128, 0, s>>>(v, n, base, block, nb, partials);   \
    else mr_block_fold_warp_kernel<T, K><<<grid, 128, 0, s>>>(v, n, base, block, nb, partials)
    switch (kind) {
        case kMapIdentity: WFCU_FOLD(kMapIdentity); break;
        case kMapSqrt: WFCU_FOLD(kMapSqrt); break;
        case kMapAltHarm: WFCU_FOLD(kMapAltHarm); break;
        case kMapSquare: WFCU_FOLD(kMapSquare); break;
        default: return cudaErrorInvalidValue;
    }
#undef WFCU_FOLD
    return cudaGetLastError();
}

// buf_a/buf_b: device scratch, each >= ceil(n/block) doubles.  Result lands in *dev_out.
cudaError_t mr_blocked_launch(const void* values, int is_f64, u64 n, u64 base, int kind, u64 block, double* buf_a,
                              double* buf_b, double* dev_out, int sm_count, cudaStream_t s, u64* launches) {
    const u64 nb = (n + block - 1) / block;
    if (nb == 0) {
        *launches += 0;
        return cudaMemsetAsync(dev_out, 0, sizeof(double), s);   // empty input -> 0.0 (engine.cpp:24)
    }
    cudaError_t e = is_f64 ? launch_fold(static_cast<const double*>(values), n, base, kind, block, nb, buf_a, sm_count, s)
                           : launch_fold(static_cast<const float*>(values), n, base, kind, block, nb, buf_a, sm_count, s);
    *launches += 1;
    if (e != cudaSuccess) return e;
    u64 m = nb;
    double* in = buf_a;
    double* out = buf_b;
    while (m > 1) {
        const u64 next = m / 2 + (m & 1ull);
        u64 gl = (next + 255) / 256;
        if (gl > (u64)sm_count * 8) gl = (u64)sm_count * 8;
        mr_tree_level_kernel<<<(unsigned)gl, 256, 0, s>>>(in, m, out);
        *launches += 1;
        double* t = in; in = out; out = t;
        m = next;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(dev_out, in, sizeof(double), cudaMemcpyDeviceToDevice, s);
}

}  // namespace wfcu
