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
//  * mr_block_fold_kernel + mr_tree_level_kernel: the reference's blocked engine
//    reproduced bit for bit -- one thread folds one block left to right with
//    separately rounded operations (no FMA contraction), then the pairwise tree
//    of combine_tree is applied level by level.
#include <cuda_runtime.h>
#include <stdint.h>

namespace wfcu {

typedef unsigned long long u64;

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
// partials[b] = fold_range(b*block, min((b+1)*block, n))   (engine.cpp:15-20, 44-50)
template <typename T, int KIND>
__global__ void mr_block_fold_kernel(const T* __restrict__ values, u64 n, u64 position_base, u64 block,
                                     u64 n_blocks, double* __restrict__ partials) {
    for (u64 b = (u64)blockIdx.x * blockDim.x + threadIdx.x; b < n_blocks; b += (u64)gridDim.x * blockDim.x) {
        const u64 lo = b * block;
        u64 hi = lo + block;
        if (hi > n || hi < lo) hi = n;
        double acc = 0.0;
        for (u64 i = lo; i < hi; ++i) {
            const double v = (KIND == kMapAltHarm) ? 0.0 : (double)values[i];
            acc = __dadd_rn(acc, map_term<KIND>(v, position_base + i + 1));
        }
        partials[b] = acc;
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
static cudaError_t launch_fold(const T* v, u64 n, u64 base, int kind, u64 block, u64 nb, double* partials, int grid,
                               cudaStream_t s) {
    switch (kind) {
        case kMapIdentity: mr_block_fold_kernel<T, kMapIdentity><<<grid, 128, 0, s>>>(v, n, base, block, nb, partials); break;
        case kMapSqrt: mr_block_fold_kernel<T, kMapSqrt><<<grid, 128, 0, s>>>(v, n, base, block, nb, partials); break;
        case kMapAltHarm: mr_block_fold_kernel<T, kMapAltHarm><<<grid, 128, 0, s>>>(v, n, base, block, nb, partials); break;
        case kMapSquare: mr_block_fold_kernel<T, kMapSquare><<<grid, 128, 0, s>>>(v, n, base, block, nb, partials); break;
        default: return cudaErrorInvalidValue;
    }
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
    u64 g = (nb + 127) / 128;
    if (g > (u64)sm_count * 16) g = (u64)sm_count * 16;
    cudaError_t e = is_f64 ? launch_fold(static_cast<const double*>(values), n, base, kind, block, nb, buf_a, (int)g, s)
                           : launch_fold(static_cast<const float*>(values), n, base, kind, block, nb, buf_a, (int)g, s);
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
