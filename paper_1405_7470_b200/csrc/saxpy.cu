// saxpy: y := alpha * x + y -- Table 1's bandwidth-bound BLAS-1 row (PAPER.md
// P:670, section 3) through the same C ABI as the GEMM (include/lpy.h).
//
// Loo.py would split the single iname i into work-groups and work-items and
// vectorise (split_iname + tag "g.0"/"l.0"/"vec").  The
// B200 version of that schedule for a stream that touches every byte once:
//
//   * vec: 32-byte accesses (sm_100's LDG.256 / STG.256), so a warp moves 1 KB
//     per instruction; x is read through the non-coherent path without L1
//     allocation, both streams with an L2 evict-first hint (touched once);
//   * group/local split: a grid of 148 SMs x 8 CTAs x 256 threads (every
//     thread slot of the chip) striding over the vector, each thread keeping
//     UNR = 8 independent 32-byte loads of x and of y in flight before it stores,
//     enough bytes in flight per SM to cover HBM latency;
//   * remainders: the up-to-7 elements before y's first 32-byte
//     boundary and after its last are handled by scalar code in one thread,
//     so the vector loop carries no conditionals; if x is not 32-byte aligned
//     relative to y, x is read with scalar loads (the stores stay vectorised);
//     strided vectors (inc > 1) take a plain scalar grid-stride loop.
//
// Each element is one fmaf (fp32 RN, single rounding): DESIGN.md reading S1.
#include "lpy_internal.h"

namespace lpy {
namespace saxpy {

#ifndef LPY_SAXPY_THREADS
#define LPY_SAXPY_THREADS 256
#endif
#ifndef LPY_SAXPY_CTAS
#define LPY_SAXPY_CTAS 8
#endif
#ifndef LPY_SAXPY_UNR
#define LPY_SAXPY_UNR 8
#endif
constexpr int THREADS = LPY_SAXPY_THREADS;
constexpr int CTAS_PER_SM = LPY_SAXPY_CTAS;
constexpr int UNR = LPY_SAXPY_UNR;

// 32-byte vectors (sm_100 LDG/STG.256): 8 floats per access.
struct f8 {
    float v[8];
};
__device__ __forceinline__ f8 ld8(const float *p, bool nc) {
    f8 r;
    if (nc)
        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                       "=f"(r.v[6]), "=f"(r.v[7])
                     : "l"(p));
    else
        asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                       "=f"(r.v[6]), "=f"(r.v[7])
                     : "l"(p));
    return r;
}
__device__ __forceinline__ void st8(float *p, const f8 &r) {
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]),
                 "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
                 : "memory");
}

// XMODE 0: x 32-byte aligned with y, distinct vectors; 1: x misaligned
// (scalar loads); 2: x == y.
template <int XMODE>
__device__ __forceinline__ f8 load_x(const float *x, const float *y, int64_t v) {
    if constexpr (XMODE == 0) return ld8(x + 8 * v, true);
    if constexpr (XMODE == 1) {
        f8 r;
#pragma unroll
        for (int e = 0; e < 8; ++e) r.v[e] = __ldg(x + 8 * v + e);
        return r;
    }
    return ld8(y + 8 * v, false);
}

__device__ __forceinline__ f8 axpy8(float a, const f8 &x, const f8 &y) {
    f8 r;
#pragma unroll
    for (int e = 0; e < 8; ++e) r.v[e] = fmaf(a, x.v[e], y.v[e]);
    return r;
}

// Contiguous vectors.  x0/y0: the first element; head: scalar elements before
// y's first 32-byte boundary; nvec 8-float groups; then tail scalar elements.
template <int XMODE>
__global__ void __launch_bounds__(THREADS) saxpy_contig_kernel(int64_t head, int64_t nvec, int64_t tail,
                                                               float alpha, const float *__restrict__ x0,
                                                               float *y0) {
    const float *x = x0 + head;
    float *y = y0 + head;
    const int64_t stride = int64_t(gridDim.x) * THREADS;
    int64_t v = int64_t(blockIdx.x) * THREADS + threadIdx.x;
    for (; v + (UNR - 1) * stride < nvec; v += UNR * stride) {
        f8 xv[UNR], yv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if constexpr (XMODE != 2) yv[u] = ld8(y + 8 * (v + u * stride), false);
            xv[u] = load_x<XMODE>(x, y, v + u * stride);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            st8(y + 8 * (v + u * stride), axpy8(alpha, xv[u], XMODE == 2 ? xv[u] : yv[u]));
    }
    for (; v < nvec; v += stride) {
        const f8 xv = load_x<XMODE>(x, y, v);
        const f8 yv = XMODE == 2 ? xv : ld8(y + 8 * v, false);
        st8(y + 8 * v, axpy8(alpha, xv, yv));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int64_t i = 0; i < head; ++i) y0[i] = fmaf(alpha, x0[i], y0[i]);
        const int64_t t0 = head + 8 * nvec;
        for (int64_t i = t0; i < t0 + tail; ++i) y0[i] = fmaf(alpha, x0[i], y0[i]);
    }
}

__global__ void __launch_bounds__(THREADS) saxpy_strided_kernel(int64_t n, float alpha, const float *x,
                                                                int64_t incx, float *y, int64_t incy) {
    const int64_t stride = int64_t(gridDim.x) * THREADS;
    for (int64_t i = int64_t(blockIdx.x) * THREADS + threadIdx.x; i < n; i += stride)
        y[i * incy] = fmaf(alpha, x[i * incx], y[i * incy]);
}

static int grid_for(int64_t work, int num_sms) {
    int64_t g = (work + THREADS - 1) / THREADS;
    const int64_t cap = int64_t(num_sms) * CTAS_PER_SM;
    if (g > cap) g = cap;
    return int(g < 1 ? 1 : g);
}

}  // namespace saxpy

cudaError_t launch_saxpy(int64_t n, float alpha, const float *x, int64_t incx, float *y, int64_t incy,
                         int num_sms, cudaStream_t s) {
    using namespace saxpy;
    if (n <= 0) return cudaSuccess;
    if (incx != 1 || incy != 1) {
        saxpy_strided_kernel<<<grid_for(n, num_sms), THREADS, 0, s>>>(n, alpha, x, incx, y, incy);
        return cudaGetLastError();
    }
    const uintptr_t ya = reinterpret_cast<uintptr_t>(y);
    int64_t head = int64_t(((32 - (ya & 31)) & 31) / 4);
    if (head > n) head = n;
    const int64_t nvec = (n - head) / 8;
    const int64_t tail = n - head - 8 * nvec;
    const int grid = grid_for(nvec > 0 ? (nvec + UNR - 1) / UNR : 1, num_sms);
    if (x == y)
        saxpy_contig_kernel<2><<<grid, THREADS, 0, s>>>(head, nvec, tail, alpha, x, y);
    else if (((reinterpret_cast<uintptr_t>(x) + 4 * head) & 31) == 0)
        saxpy_contig_kernel<0><<<grid, THREADS, 0, s>>>(head, nvec, tail, alpha, x, y);
    else
        saxpy_contig_kernel<1><<<grid, THREADS, 0, s>>>(head, nvec, tail, alpha, x, y);
    return cudaGetLastError();
}

}  // namespace lpy
