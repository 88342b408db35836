// Hardware probes for the 3xTF32 design (test/diagnostic library
// liblpy_probe.so, not part of the product C-ABI):
//   * lpy_probe_umma_tf32: one 128 x N tile D = A B^T through tcgen05.mma
//     kind::tf32 with operands staged in shared memory in the canonical layouts
//     the GEMM kernels use.  Verifies descriptor encodings and measures how the
//     tensor core treats fp32 operand bits (truncate vs round) and how it rounds
//     the accumulation (readings A9, A10).
//   * lpy_probe_umma_rate: back-to-back kind::tf32 MMAs (cycles per instruction).
//   * lpy_probe_ffma_rate: FP32 FMA pipe throughput (FFMA and packed FFMA2).
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

namespace lpy {
namespace probe {

// Operand formats (R rows of the operand, k runs along Kp):
//  0: K-major, 128B swizzle, 32-wide k panels   (rows of 128 B; SBO 1024)
//  1: MN-major, 128B_BASE32B, 32-wide k panels  (32-row MN blocks of 32 k-rows x 128 B)
//  2: K-major, 64B swizzle, 16-wide k panels    (rows of 64 B; SBO 512)
//  3: MN-major, 128B_BASE32B, 16-wide k panels  (32-row MN blocks of 16 k-rows x 128 B)
__device__ __forceinline__ uint32_t offset(int fmt, int r, int k, int R) {
    switch (fmt) {
        case 0: {
            const int p = k >> 5, kk = k & 31;
            return p * R * 128 + r * 128 + (((kk >> 2) ^ (r & 7)) << 4) + (kk & 3) * 4;
        }
        case 1: {
            const int p = k >> 5, kk = k & 31, rr = r & 31;
            return p * R * 128 + (r >> 5) * 4096 + kk * 128 + (((rr >> 3) ^ (kk & 3)) << 5) + (rr & 7) * 4;
        }
        case 2: {
            const int p = k >> 4, kk = k & 15;
            return p * R * 64 + r * 64 + (((kk >> 2) ^ ((r >> 1) & 3)) << 4) + (kk & 3) * 4;
        }
        default: {
            const int p = k >> 4, kk = k & 15, rr = r & 31;
            return p * R * 64 + (r >> 5) * 2048 + kk * 128 + (((rr >> 3) ^ (kk & 3)) << 5) + (rr & 7) * 4;
        }
    }
}

// Descriptor of k-slice q (8 elements) for format fmt.
__device__ __forceinline__ uint64_t desc(int fmt, uint32_t base, int q, int R) {
    switch (fmt) {
        case 0: return umma_sdesc(base + (q >> 2) * R * 128 + (q & 3) * 32, 16, 1024, 2);
        case 1: return umma_sdesc(base + (q >> 2) * R * 128 + (q & 3) * 1024, 4096, 512, 1);
        case 2: return umma_sdesc(base + (q >> 1) * R * 64 + (q & 1) * 32, 16, 512, 4);
        default: return umma_sdesc(base + (q >> 1) * R * 64 + (q & 1) * 1024, 2048, 512, 1);
    }
}

// 128 threads.  A: 128 x Kp row-major (A(m,k)), B: N x Kp row-major (B(n,k)).
__global__ void umma_tile_kernel(const float *A, const float *B, float *D, int N, int Kp, int fa,
                                 int fb, int accumulate_first) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t *base = smem_raw + (((raw + 1023) & ~1023u) - raw);
    uint8_t *sa = base;
    uint8_t *sb = base + 128 * Kp * 4;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;

    for (int idx = threadIdx.x; idx < 128 * Kp; idx += blockDim.x)
        *reinterpret_cast<float *>(sa + offset(fa, idx / Kp, idx % Kp, 128)) = A[idx];
    for (int idx = threadIdx.x; idx < N * Kp; idx += blockDim.x)
        *reinterpret_cast<float *>(sb + offset(fb, idx / Kp, idx % Kp, N)) = B[idx];
    fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) {
        tmem_alloc(&tmem_base, 256);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;

    if (threadIdx.x == 0) {
        const uint32_t idesc = umma_idesc_tf32(128, N, fa & 1, fb & 1);
        for (int q = 0; q < Kp / 8; ++q)
            umma_tf32(tmem, desc(fa, smem_u32(sa), q, 128), desc(fb, smem_u32(sb), q, N), idesc,
                      (q > 0 || accumulate_first) ? 1u : 0u);
        umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        tmem_ld_x16(tmem + (uint32_t(warp * 32) << 16) + c0, v);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

__global__ void umma_rate_kernel(int N, int iters, long long *cycles) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t *base = smem_raw + (((raw + 1023) & ~1023u) - raw);
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    for (int i = threadIdx.x; i < (128 + 256) * 32; i += blockDim.x)
        reinterpret_cast<float *>(base)[i] = 1.0f;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) {
        tmem_alloc(&tmem_base, 256);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t idesc = umma_idesc_tf32(128, N, 0, 0);
        const uint64_t da = umma_sdesc(smem_u32(base), 16, 1024, 2);
        const uint64_t db = umma_sdesc(smem_u32(base) + 128 * 128, 16, 1024, 2);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) umma_tf32(tmem_base, da, db, idesc, i > 0 ? 1u : 0u);
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) *cycles = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem_base, 256);
}

__global__ void ffma_rate_kernel(float *out, int iters, float x, float y) {
    float a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], x, y);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += a[j];
    if (s == 12345.678f) out[0] = s;   // keep the work alive
}

__global__ void ffma2_rate_kernel(float *out, int iters, float x, float y) {
    uint64_t a[8];
    uint64_t xx, yy;
    asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
    asm("mov.b64 %0, {%1, %1};" : "=l"(yy) : "f"(y));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float lo = threadIdx.x * 1e-3f + j, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a[j]) : "f"(lo), "f"(hi));
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(xx), "l"(yy));
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[j]));
        s += lo + hi;
    }
    if (s == 12345.678f) out[0] = s;
}

}  // namespace probe
}  // namespace lpy

extern "C" {

int lpy_probe_umma_tf32(const float *A, const float *B, float *D, int N, int Kp, int fa, int fb,
                        int accumulate_first, void *stream) {
    if (N < 16 || N > 256 || N % 16 || Kp < 32 || Kp > 64 || Kp % 32 || fa < 0 || fa > 3 || fb < 0 ||
        fb > 3)
        return 1;
    if (((fa & 1) || (fb & 1)) && N % 32) return 1;
    const size_t smem = 1024 + size_t(128 + N) * Kp * 4;
    cudaFuncSetAttribute(lpy::probe::umma_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    lpy::probe::umma_tile_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(
        A, B, D, N, Kp, fa, fb, accumulate_first);
    return int(cudaGetLastError());
}

int lpy_probe_umma_rate(int N, int iters, int ctas, long long *cycles_dev, void *stream) {
    const size_t smem = 1024 + size_t(128 + 256) * 32 * 4;
    cudaFuncSetAttribute(lpy::probe::umma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    lpy::probe::umma_rate_kernel<<<ctas, 128, smem, static_cast<cudaStream_t>(stream)>>>(N, iters,
                                                                                         cycles_dev);
    return int(cudaGetLastError());
}

int lpy_probe_ffma_rate(float *out, int iters, int blocks, int threads, int pair, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (pair)
        lpy::probe::ffma2_rate_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.999f, 0.001f);
    else
        lpy::probe::ffma_rate_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.999f, 0.001f);
    return int(cudaGetLastError());
}

}  // extern "C"

// ---------------------------------------------------------------- MMA rate per operand format
// Back-to-back kind::tf32 MMAs over a 32-wide k panel in the given operand
// formats (see `offset`), single CTA (M=128) or CTA pair (M=256, cluster of 2).
namespace lpy {
namespace probe {
template <int CG>
__global__ void umma_rate_fmt_kernel(int N, int fa, int fb, int iters, long long *cycles) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t *base = smem_raw + (((raw + 1023) & ~1023u) - raw);
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int nb = N / CG;   // B rows staged per CTA
    for (int i = threadIdx.x; i < (128 + nb) * 32; i += blockDim.x)
        reinterpret_cast<float *>(base)[i] = 1.0f;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) {
        tmem_alloc_cg<CG>(&tmem_base, 256);
        tmem_relinquish_cg<CG>();
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t idesc = umma_idesc_tf32(128 * CG, N, fa & 1, fb & 1);
        const uint32_t sa = smem_u32(base), sb = smem_u32(base) + 128 * 128;
        // descriptors of the 4 k-slices, computed once (the loop must not be issue-bound)
        const uint64_t a0 = desc(fa, sa, 0, 128), a1 = desc(fa, sa, 1, 128), a2 = desc(fa, sa, 2, 128),
                       a3 = desc(fa, sa, 3, 128);
        const uint64_t b0 = desc(fb, sb, 0, nb), b1 = desc(fb, sb, 1, nb), b2 = desc(fb, sb, 2, nb),
                       b3 = desc(fb, sb, 3, nb);
        const bool same = iters < 0;          // negative iters: repeat slice 0 (operand reuse)
        if (same) iters = -iters;
        long long t0 = clock64();
        for (int i = 0; i < iters; i += 4) {
            umma_tf32_cg<CG>(tmem_base, a0, b0, idesc, i > 0 ? 1u : 0u);
            umma_tf32_cg<CG>(tmem_base, same ? a0 : a1, same ? b0 : b1, idesc, 1u);
            umma_tf32_cg<CG>(tmem_base, same ? a0 : a2, same ? b0 : b2, idesc, 1u);
            umma_tf32_cg<CG>(tmem_base, same ? a0 : a3, same ? b0 : b3, idesc, 1u);
        }
        umma_commit_cg<CG>(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) *cycles = t1 - t0;
    } else if (threadIdx.x == 0) {
        mbar_wait(&bar, 0);
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc_cg<CG>(tmem_base, 256);
}
}  // namespace probe
}  // namespace lpy

extern "C" int lpy_probe_umma_rate_fmt(int N, int fa, int fb, int iters, int ctas, int cg,
                                       long long *cycles_dev, void *stream) {
    const size_t smem = 1024 + size_t(128 + 256) * 32 * 4;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cg;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cg == 2) {
        cudaFuncSetAttribute(lpy::probe::umma_rate_fmt_kernel<2>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        return int(cudaLaunchKernelEx(&cfg, lpy::probe::umma_rate_fmt_kernel<2>, N, fa, fb, iters, cycles_dev));
    }
    cudaFuncSetAttribute(lpy::probe::umma_rate_fmt_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    return int(cudaLaunchKernelEx(&cfg, lpy::probe::umma_rate_fmt_kernel<1>, N, fa, fb, iters, cycles_dev));
}

// ---------------------------------------------------------------- launch overhead
// An empty kernel with `threads` threads and `smem` bytes of dynamic shared
// memory (touching one word so it is really allocated): how much fixed cost a
// launch with the GEMM kernels' resource shape carries.
namespace lpy {
namespace probe {
__global__ void empty_smem_kernel(int *out) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) sm[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && sm[0] == -1) out[0] = 1;
}
}  // namespace probe
}  // namespace lpy

extern "C" int lpy_probe_empty_launch(int ctas, int threads, int smem, int *out, void *stream) {
    cudaFuncSetAttribute(lpy::probe::empty_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    lpy::probe::empty_smem_kernel<<<ctas, threads, smem, static_cast<cudaStream_t>(stream)>>>(out);
    return int(cudaGetLastError());
}

// ---------------------------------------------------------------- MUFU.RSQ rate
// 16 independent rsqrt.approx chains per thread (the Coulomb kernel's bound):
// results per second over the grid = 16 * iters * blocks * threads / time.
namespace lpy {
namespace probe {
__global__ void rsqrt_rate_kernel(float *out, int iters, float x) {
    float a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = x + threadIdx.x * 1e-3f + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += a[j];
    if (s == 12345.678f) out[0] = s;
}

// Accuracy of rsqrt.approx.ftz.f32 on n inputs: out[i] = rsqrt(in[i]).
__global__ void rsqrt_eval_kernel(const float *in, float *out, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        float r;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(in[i]));
        out[i] = r;
    }
}
}  // namespace probe
}  // namespace lpy

extern "C" int lpy_probe_rsqrt_rate(float *out, int iters, int blocks, int threads, void *stream) {
    lpy::probe::rsqrt_rate_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(out, iters, 1.5f);
    return int(cudaGetLastError());
}

extern "C" int lpy_probe_rsqrt_eval(const float *in, float *out, int n, void *stream) {
    lpy::probe::rsqrt_eval_kernel<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(in, out, n);
    return int(cudaGetLastError());
}

// ---------------------------------------------------------------- f32x2 rates
// 8 independent chains per thread of one packed instruction kind:
// 0 fma.rn.f32x2, 1 add.rn.f32x2, 2 mul.rn.f32x2, 3 scalar add.f32 (16 chains),
// 4 scalar fma.f32 (16 chains).  Lane-ops per second = 16 * iters * threads / time.
namespace lpy {
namespace probe {
template <int KIND>
__global__ void x2_rate_kernel(float *out, int iters, float x) {
    unsigned long long a[8];
    float f[16];
    unsigned long long xx;
    asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float lo = threadIdx.x * 1e-3f + j, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a[j]) : "f"(lo), "f"(hi));
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if constexpr (KIND == 0) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a[j]) : "l"(xx));
            if constexpr (KIND == 1) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[j]) : "l"(xx));
            if constexpr (KIND == 2) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(a[j]) : "l"(xx));
        }
        if constexpr (KIND == 3) {
#pragma unroll
            for (int j = 0; j < 16; ++j) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(f[j]) : "f"(x));
        }
        if constexpr (KIND == 4) {
#pragma unroll
            for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[j]) : "f"(x));
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[j]));
        s += lo + hi;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) s += f[j];
    if (s == 12345.678f) out[0] = s;
}
}  // namespace probe
}  // namespace lpy

extern "C" int lpy_probe_x2_rate(int kind, float *out, int iters, int blocks, int threads, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (kind) {
        case 0: lpy::probe::x2_rate_kernel<0><<<blocks, threads, 0, s>>>(out, iters, 0.999f); break;
        case 1: lpy::probe::x2_rate_kernel<1><<<blocks, threads, 0, s>>>(out, iters, 0.999f); break;
        case 2: lpy::probe::x2_rate_kernel<2><<<blocks, threads, 0, s>>>(out, iters, 0.999f); break;
        case 3: lpy::probe::x2_rate_kernel<3><<<blocks, threads, 0, s>>>(out, iters, 0.999f); break;
        default: lpy::probe::x2_rate_kernel<4><<<blocks, threads, 0, s>>>(out, iters, 0.999f); break;
    }
    return int(cudaGetLastError());
}

// ---------------------------------------------------------------- persistent copy (diagnostics)
// dst := src over n floats by exactly `ctas` CTAs of 512 threads, each thread
// keeping four 16-byte loads in flight in a grid-stride loop: a stand-in for
// a collective's persistent channel CTAs when bench.py --emulate-bcast-gbs
// projects the row-panel step on one GPU (how many bytes `ctas` SMs move
// while the gated product holds the rest).
namespace lpy {
namespace probe {
__global__ void __launch_bounds__(512) persistent_copy_kernel(float4 *dst, const float4 *src, long long n4) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        const float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
        dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
    }
    for (; i < n4; i += stride) dst[i] = src[i];
}
}  // namespace probe
}  // namespace lpy

extern "C" int lpy_probe_persistent_copy(float *dst, const float *src, long long n, int ctas, void *stream) {
    // n must be a multiple of 4 and both pointers 16-byte aligned (diagnostics only)
    lpy::probe::persistent_copy_kernel<<<ctas, 512, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<float4 *>(dst), reinterpret_cast<const float4 *>(src), n / 4);
    return int(cudaGetLastError());
}

// ---------------------------------------------------------------- TMA bulk copy (diagnostics)
// dst := src (bytes, multiple of 16, 16-byte aligned) by `ctas` CTAs whose one
// elected thread streams 32 KB pieces global -> shared -> global with
// cp.async.bulk (4 buffers in flight): how many bytes a few SMs move when the
// copy engine of the SM (TMA) does the work instead of threads' loads/stores.
namespace lpy {
namespace probe {
constexpr int BULK_BUF = 32 * 1024, BULK_NBUF = 6;
__global__ void __launch_bounds__(32) bulk_copy_kernel(char *dst, const char *src, long long bytes) {
    extern __shared__ __align__(128) unsigned char bsm[];
    __shared__ __align__(8) unsigned long long bar[BULK_NBUF];
    if (threadIdx.x != 0) return;
    for (int b = 0; b < BULK_NBUF; ++b)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long long pieces = (bytes + BULK_BUF - 1) / BULK_BUF;
    unsigned phase[BULK_NBUF] = {0, 0, 0, 0, 0, 0};
    int issued = 0;
    long long mine[BULK_NBUF];
    for (long long p = blockIdx.x; p < pieces; p += gridDim.x) {
        const int b = issued % BULK_NBUF;
        if (issued >= BULK_NBUF) {
            // buffer b: its previous piece must be loaded and stored out before reuse
            const long long q = mine[b];
            const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar[b]);
            asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}"
                         ::"r"(sb), "r"(phase[b]) : "memory");
            phase[b] ^= 1;
            const long long qb = q * BULK_BUF, n = min((long long)BULK_BUF, bytes - qb);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(dst + qb), "r"((unsigned)__cvta_generic_to_shared(bsm + b * BULK_BUF)), "r"((unsigned)n)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
        }
        const long long pb = p * BULK_BUF, n = min((long long)BULK_BUF, bytes - pb);
        const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar[b]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"((unsigned)n) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((unsigned)__cvta_generic_to_shared(bsm + b * BULK_BUF)), "l"(src + pb), "r"((unsigned)n), "r"(sb)
                     : "memory");
        mine[b] = p;
        ++issued;
    }
    // drain
    const int live = issued < BULK_NBUF ? issued : BULK_NBUF;
    for (int j = 0; j < live; ++j) {
        const int b = (issued - live + j) % BULK_NBUF;
        const long long q = mine[b];
        const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar[b]);
        asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}"
                     ::"r"(sb), "r"(phase[b]) : "memory");
        const long long qb = q * BULK_BUF, n = min((long long)BULK_BUF, bytes - qb);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(dst + qb), "r"((unsigned)__cvta_generic_to_shared(bsm + b * BULK_BUF)), "r"((unsigned)n)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
}  // namespace probe
}  // namespace lpy

extern "C" int lpy_probe_bulk_copy(void *dst, const void *src, long long bytes, int ctas, void *stream) {
    const int smem = lpy::probe::BULK_BUF * lpy::probe::BULK_NBUF;
    cudaFuncSetAttribute(lpy::probe::bulk_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    lpy::probe::bulk_copy_kernel<<<ctas, 32, smem, static_cast<cudaStream_t>(stream)>>>(
        static_cast<char *>(dst), static_cast<const char *>(src), bytes);
    return int(cudaGetLastError());
}

// ---------------------------------------------------------------- MMA rate with commits
// As umma_rate_fmt_kernel (A K-major 64B-swizzled format 2, B MN-major format 3),
// plus a tcgen05.commit to one of 8 rotating mbarriers after every `every`
// groups of six MMAs (0: none), and optionally (`wait` != 0) the issuing thread waiting for each
// commit `lag` commits later -- the 3xTF32 kernel's per-k-block pattern
// (six MMAs, a commit freeing the stage).  Does a commit cost the pipe?
namespace lpy {
namespace probe {
template <int CG>
__global__ void umma_rate_commit_kernel(int N, int iters, int every, int lag, int pattern, long long *cycles) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t *base = smem_raw + (((raw + 1023) & ~1023u) - raw);
    __shared__ uint64_t bars[8];
    __shared__ uint64_t done;              // completed once, before the loop
    __shared__ uint32_t tmem_base;
    const int nb = N / CG;
    for (int i = threadIdx.x; i < (128 + nb) * 32; i += blockDim.x)
        reinterpret_cast<float *>(base)[i] = 1.0f;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
        mbar_init(&done, 1);
        fence_mbar_init();
        mbar_arrive(&done);
    }
    if (threadIdx.x < 32) {
        tmem_alloc_cg<CG>(&tmem_base, 512);
        tmem_relinquish_cg<CG>();
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    if (threadIdx.x < 32 && rank == 0) {
        // the whole warp runs the loop converged (descriptors in uniform registers), one
        // elected lane issues -- as the 3xTF32 kernel's MMA warp does; 6 MMAs per "k-block"
        const uint32_t idesc = umma_idesc_tf32(128 * CG, N, 0, 1);
        const uint32_t sa = smem_u32(base), sb = smem_u32(base) + 128 * 128;
        const uint64_t a0 = desc(2, sa, 0, 128), a1 = desc(2, sa, 1, 128);
        const uint64_t b0 = desc(3, sb, 0, nb), b1 = desc(3, sb, 1, nb);
        const int kblocks = iters / 6;
        long long t0 = clock64();
        for (int kb = 0; kb < kblocks; ++kb) {
            if (elect_one()) {
                if (CG == 2 && pattern > 0) {
                    // the 3xTF32 kernel's k-block: per k-slice of 8, A_big x B_small and A_big x B_big
                    // through the A collector (fill / lastuse), then A_small x B_big from shared
                    // memory (pattern 1) or from TMEM columns 256.. (pattern 2, the TS form)
#pragma unroll
                    for (int sub = 0; sub < 2; ++sub) {
                        const uint64_t a = sub ? a1 : a0, b = sub ? b1 : b0, bs = sub ? b0 : b1;
                        umma_tf32_cg2_coll<ACollector::Fill>(tmem_base, a, bs, idesc, (kb > 0 || sub) ? 1u : 0u);
                        umma_tf32_cg2_coll<ACollector::LastUse>(tmem_base, a, b, idesc, 1u);
                        if (pattern == 2) umma_tf32_ts_cg2(tmem_base, tmem_base + 256 + 8 * sub, b, idesc, 1u);
                        else              umma_tf32_cg<CG>(tmem_base, sub ? a0 : a1, b, idesc, 1u);
                    }
                } else {
                umma_tf32_cg<CG>(tmem_base, a0, b0, idesc, kb > 0 ? 1u : 0u);
                umma_tf32_cg<CG>(tmem_base, a0, b1, idesc, 1u);
                umma_tf32_cg<CG>(tmem_base, a1, b0, idesc, 1u);
                umma_tf32_cg<CG>(tmem_base, a1, b1, idesc, 1u);
                umma_tf32_cg<CG>(tmem_base, a0, b0, idesc, 1u);
                umma_tf32_cg<CG>(tmem_base, a1, b1, idesc, 1u);
                }
                if (every > 0 && (kb + 1) % every == 0) umma_commit_cg<CG>(&bars[(kb / every) & 7]);
            }
            __syncwarp();
            // mode (lag < 0): -1 fence only, -2 wait on an always-complete barrier + fence,
            // -3 that wait without the fence; lag in 1..7: wait on the commit `lag` back + fence,
            // lag in 9..15: the same wait (lag - 8 back) without the fence
            if (lag == -1) {
                tc_fence_after();
            } else if (lag == -2 || lag == -3) {
                mbar_wait(&done, 0);
                if (lag == -2) tc_fence_after();
            } else if (every > 0 && lag > 0 && (kb + 1) % every == 0 && kb / every >= (lag & 7)) {
                const int w = kb / every - (lag & 7);
                mbar_wait(&bars[w & 7], uint32_t((w >> 3) & 1));
                if (lag < 8) tc_fence_after();
            }
        }
        __shared__ uint64_t fin;
        if (elect_one()) {
            mbar_init(&fin, 1);
            fence_mbar_init();
            umma_commit_cg<CG>(&fin);
        }
        __syncwarp();
        mbar_wait(&fin, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = t1 - t0;
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc_cg<CG>(tmem_base, 512);
}
}  // namespace probe
}  // namespace lpy

extern "C" int lpy_probe_umma_rate_commit(int N, int iters, int every, int lag, int pattern, int ctas, int cg,
                                          long long *cycles_dev, void *stream) {
    const size_t smem = 1024 + size_t(128 + 256) * 32 * 4;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cg;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cg == 2) {
        cudaFuncSetAttribute(lpy::probe::umma_rate_commit_kernel<2>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        return int(cudaLaunchKernelEx(&cfg, lpy::probe::umma_rate_commit_kernel<2>, N, iters, every, lag, pattern,
                                      cycles_dev));
    }
    cudaFuncSetAttribute(lpy::probe::umma_rate_commit_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    return int(cudaLaunchKernelEx(&cfg, lpy::probe::umma_rate_commit_kernel<1>, N, iters, every, lag, pattern,
                                  cycles_dev));
}
