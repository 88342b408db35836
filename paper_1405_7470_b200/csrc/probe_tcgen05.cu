// Hardware probes for the 3xTF32 design (test/diagnostic library
// liblpy_probe.so, not part of the product C-ABI):
//   * lpy_probe_umma_tf32: one 128 x N tile D = A B^T through tcgen05.mma
//     kind::tf32 with operands staged in shared memory in the exact canonical
//     layouts the GEMM kernel uses (K-major SW128 or MN-major SW128, 32-wide
//     k panels).  Verifies descriptor encodings and measures how the tensor
//     core treats fp32 operand bits (truncate vs round) and how it rounds the
//     accumulation (reading A10).
//   * lpy_probe_umma_rate: back-to-back kind::tf32 MMAs to measure cycles per
//     instruction (the TF32 tensor roofline per SM).
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

namespace lpy {
namespace probe {

// Byte offset of element (r, k) of an R x Kp operand tile in the canonical
// layouts used by the GEMM: 32-wide k panels of R*128 bytes each.
__device__ __forceinline__ uint32_t kmajor_off(int r, int k, int R) {
    const int p = k >> 5, kk = k & 31;
    return p * R * 128 + r * 128 + ((((kk >> 2) ^ (r & 7))) << 4) + (kk & 3) * 4;
}
__device__ __forceinline__ uint32_t mnmajor_off(int r, int k, int R) {
    const int p = k >> 5, kk = k & 31, b = r >> 5, rr = r & 31;
    return p * R * 128 + b * 4096 + (kk >> 3) * 1024 + (kk & 7) * 128 +
           ((((rr >> 2) ^ (kk & 7))) << 4) + (rr & 3) * 4;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;                 // version (sm100)
    d |= uint64_t(2) << 61;                 // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
           (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// 128 threads.  A: 128 x Kp row-major (A(m,k)), B: N x Kp row-major (B(n,k)).
__global__ void umma_tile_kernel(const float *A, const float *B, float *D, int N, int Kp, int a_mn,
                                 int b_mn, int accumulate_first) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t *base = smem_raw + (((raw + 1023) & ~1023u) - raw);
    uint8_t *sa = base;
    uint8_t *sb = base + 128 * Kp * 4;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;

    for (int idx = threadIdx.x; idx < 128 * Kp; idx += blockDim.x) {
        const int r = idx / Kp, k = idx % Kp;
        const uint32_t off = a_mn ? mnmajor_off(r, k, 128) : kmajor_off(r, k, 128);
        *reinterpret_cast<float *>(sa + off) = A[idx];
    }
    for (int idx = threadIdx.x; idx < N * Kp; idx += blockDim.x) {
        const int r = idx / Kp, k = idx % Kp;
        const uint32_t off = b_mn ? mnmajor_off(r, k, N) : kmajor_off(r, k, N);
        *reinterpret_cast<float *>(sb + off) = B[idx];
    }
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
        const uint32_t idesc = idesc_tf32(128, N, a_mn, b_mn);
        for (int q = 0; q < Kp / 8; ++q) {
            const int p = q >> 2, sub = q & 3;
            uint64_t da, db;
            if (a_mn) da = sdesc(smem_u32(sa) + p * 128 * 128 + sub * 1024, 4096, 1024);
            else      da = sdesc(smem_u32(sa) + p * 128 * 128 + sub * 32, 16, 1024);
            if (b_mn) db = sdesc(smem_u32(sb) + p * N * 128 + sub * 1024, 4096, 1024);
            else      db = sdesc(smem_u32(sb) + p * N * 128 + sub * 32, 16, 1024);
            umma_tf32(tmem, da, db, idesc, (q > 0 || accumulate_first) ? 1u : 0u);
        }
        umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                       "=r"(v[6]), "=r"(v[7])
                     : "r"(tmem + (uint32_t(warp * 32) << 16) + c0));
        tmem_ld_wait();
        for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
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
        const uint32_t idesc = idesc_tf32(128, N, 0, 0);
        const uint64_t da = sdesc(smem_u32(base), 16, 1024);
        const uint64_t db = sdesc(smem_u32(base) + 128 * 128, 16, 1024);
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

}  // namespace probe
}  // namespace lpy

extern "C" {

int lpy_probe_umma_tf32(const float *A, const float *B, float *D, int N, int Kp, int a_mn, int b_mn,
                        int accumulate_first, void *stream) {
    if (N < 16 || N > 256 || N % 16 || Kp < 8 || Kp > 64 || Kp % 32) return 1;
    const size_t smem = 1024 + size_t(128 + N) * Kp * 4;
    cudaFuncSetAttribute(lpy::probe::umma_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    lpy::probe::umma_tile_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(
        A, B, D, N, Kp, a_mn, b_mn, accumulate_first);
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

}  // extern "C"

// ---------------------------------------------------------------- FFMA pipe rate
namespace lpy {
namespace probe {
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

extern "C" int lpy_probe_ffma_rate(float *out, int iters, int blocks, int threads, int pair, void *stream) {
    if (pair)
        lpy::probe::ffma2_rate_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(out, iters, 0.999f, 0.001f);
    else
        lpy::probe::ffma_rate_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(out, iters, 0.999f, 0.001f);
    return int(cudaGetLastError());
}
