// saxpy: y := alpha * x + y -- Table 1's bandwidth-bound BLAS-1 row (PAPER.md
// P:670, section 3) through the same C ABI as the GEMM (include/lpy.h).
//
// Loo.py would split the single iname i into work-groups and work-items and
// vectorise (split_iname + tag "g.0"/"l.0"/"vec").  The
// B200 version of that schedule for a stream that touches every byte once:
//
//   * vec: 16-byte accesses (LDG.128 / STG.128), so a warp moves 512 B per
//     instruction; x is read through the non-coherent path without L1
//     allocation (read once, never written by this kernel unless x == y);
//   * group/local split: a grid of 148 SMs x 8 CTAs x 256 threads (every
//     thread slot of the chip) striding over the vector, each thread keeping
//     UNR independent 16-byte loads of x and of y in flight before it stores,
//     enough bytes in flight per SM to cover HBM latency;
//   * remainders: the up-to-3 elements before y's first 16-byte
//     boundary and after its last are handled by scalar code in one thread,
//     so the vector loop carries no conditionals; if x is not 16-byte aligned
//     relative to y, x is read with scalar loads (the stores stay vectorised);
//     strided vectors (inc > 1) take a plain scalar grid-stride loop.
//
// Each element is one fmaf (fp32 RN, single rounding): DESIGN.md reading S1.
#include "lpy_internal.h"

namespace lpy {
namespace saxpy {

constexpr int THREADS = 256;
constexpr int CTAS_PER_SM = 8;
constexpr int UNR = 4;

__device__ __forceinline__ float4 ld_stream(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_rw(const float4 *p) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(float4 *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ float4 axpy4(float a, float4 x, float4 y) {
    return make_float4(fmaf(a, x.x, y.x), fmaf(a, x.y, y.y), fmaf(a, x.z, y.z), fmaf(a, x.w, y.w));
}

// XMODE 0: x 16-byte aligned with y, distinct vectors; 1: x misaligned
// (scalar loads); 2: x == y.
template <int XMODE>
__device__ __forceinline__ float4 load_x(const float *x, const float4 *y4, int64_t v) {
    if constexpr (XMODE == 0) return ld_stream(reinterpret_cast<const float4 *>(x) + v);
    if constexpr (XMODE == 1) {
        const float *p = x + 4 * v;
        return make_float4(__ldg(p), __ldg(p + 1), __ldg(p + 2), __ldg(p + 3));
    }
    return ld_rw(y4 + v);
}

// Contiguous vectors.  x0/y0: the first element; head: scalar elements before
// y's first 16-byte boundary; nvec float4 groups; then tail scalar elements.
template <int XMODE>
__global__ void __launch_bounds__(THREADS) saxpy_contig_kernel(int64_t head, int64_t nvec, int64_t tail,
                                                               float alpha, const float *__restrict__ x0,
                                                               float *y0) {
    const float *x = x0 + head;
    float4 *y4 = reinterpret_cast<float4 *>(y0 + head);
    const int64_t stride = int64_t(gridDim.x) * THREADS;
    int64_t v = int64_t(blockIdx.x) * THREADS + threadIdx.x;
    for (; v + (UNR - 1) * stride < nvec; v += UNR * stride) {
        float4 xv[UNR], yv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            yv[u] = XMODE == 2 ? float4{} : ld_rw(y4 + v + u * stride);
            xv[u] = load_x<XMODE>(x, y4, v + u * stride);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            st_stream(y4 + v + u * stride, axpy4(alpha, xv[u], XMODE == 2 ? xv[u] : yv[u]));
    }
    for (; v < nvec; v += stride) {
        const float4 xv = load_x<XMODE>(x, y4, v);
        const float4 yv = XMODE == 2 ? xv : ld_rw(y4 + v);
        st_stream(y4 + v, axpy4(alpha, xv, yv));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int64_t i = 0; i < head; ++i) y0[i] = fmaf(alpha, x0[i], y0[i]);
        const int64_t t0 = head + 4 * nvec;
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
    int64_t head = int64_t(((16 - (ya & 15)) & 15) / 4);
    if (head > n) head = n;
    const int64_t nvec = (n - head) / 4;
    const int64_t tail = n - head - 4 * nvec;
    const int grid = grid_for(nvec > 0 ? (nvec + UNR - 1) / UNR : 1, num_sms);
    if (x == y)
        saxpy_contig_kernel<2><<<grid, THREADS, 0, s>>>(head, nvec, tail, alpha, x, y);
    else if (((reinterpret_cast<uintptr_t>(x) + 4 * head) & 15) == 0)
        saxpy_contig_kernel<0><<<grid, THREADS, 0, s>>>(head, nvec, tail, alpha, x, y);
    else
        saxpy_contig_kernel<1><<<grid, THREADS, 0, s>>>(head, nvec, tail, alpha, x, y);
    return cudaGetLastError();
}

}  // namespace lpy
