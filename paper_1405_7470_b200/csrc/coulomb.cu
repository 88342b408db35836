// 3D Coulomb potential -- Table 1's third workload (section 3):
//
//     phi[i] = sum_{j : r_ij != 0} q[j] / r_ij          (reading C1)
//
// for every target i over all sources j, reported in pairs/s.  It is an
// all-pairs loop nest {[i, j]} with one reduction, the same shape as the GEMM's
// but with an rsqrt per term instead of a product, so it is bound by
// arithmetic, not memory: per pair 3 subtractions, 3 multiply-adds for r^2, one
// MUFU.RSQ, one select (coincident points) and one multiply-add into the sum.
// The B200 realisation of the paper's split_iname / local prefetch / ilp
// schedule:
//
//   * sources are packed once into float4 (x, y, z, q) and streamed through
//     shared memory in tiles of 256 (one 16-byte broadcast LDS per source per
//     thread), double-buffered;
//   * coincident points (r = 0, excluded) are masked only where they can occur
//     for sure -- the tiles holding a CTA's own targets in a self-potential --
//     and any other coincidence shows up as a non-finite sum, which sends that
//     target down a scalar masked path: the hot loop carries no select;
//   * each thread owns 4 targets held as two packed pairs, so the r^2 and
//     accumulation arithmetic runs as FADD2 / FMUL2 / FFMA2 (two fp32 RN ops per
//     instruction), leaving the 16-per-clock-per-SM MUFU.RSQ as the bound;
//   * the sum over sources is taken in fp32 over chunks of 32 sources and the
//     chunk sums are added with Kahan compensation, which keeps the error bound
//     independent of the number of sources (reading C2);
//   * under-filled grids (few targets) split the sources into S slices (fixed by
//     the shape and SM count); slice partials land in scratch and a second
//     kernel adds them in slice order, so results are deterministic.
#include "lpy_internal.h"

namespace lpy {
namespace coulomb {

constexpr int THREADS = 256;
constexpr int TPT = 4;                 // targets per thread (TPT/2 f32x2 pairs; 2 and 8 measured equal)
constexpr int TILE = 256;              // sources per shared-memory tile
constexpr int CHUNK = 32;              // sources per plain fp32 partial sum
constexpr int CTAS_PER_SM = 4;
constexpr float FAR = 3.0e18f;         // padding sources (q = 0) sit here: r^2 stays finite

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(u64 v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64 sub2s(u64 a, float b) {      // a - (b, b)
    u64 r;
    asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%2, %2};\n\tsub.rn.f32x2 %0, %1, t;\n\t}" : "=l"(r) : "l"(a), "f"(b));
    return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ u64 fma2s(float a, u64 b, u64 c) {   // (a, a) * b + c
    u64 r;
    asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%1, %1};\n\tfma.rn.f32x2 %0, t, %2, %3;\n\t}"
        : "=l"(r) : "f"(a), "l"(b), "l"(c));
    return r;
}
// 1/sqrt(r2) with the hardware approximation, 0 where r2 == 0 (coincident).
__device__ __forceinline__ float rinv(float r2) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(r2));
    return r2 > 0.f ? r : 0.f;
}
// Kahan step on pairs: (sum, comp) += x.
__device__ __forceinline__ void kahan2(u64 &sum, u64 &comp, u64 x) {
    const u64 y = sub2(x, comp);
    const u64 t = add2(sum, y);
    comp = sub2(sub2(t, sum), y);
    sum = t;
}

// One chunk of CHUNK sources from shared memory into the pair accumulators.
// MASK: exclude coincident points with a select (FSETP + FSEL per target);
// without it a coincident pair yields inf / NaN, which the caller detects.
template <bool MASK, int NP>
__device__ __forceinline__ void chunk_pass(const float4 *__restrict__ src, const u64 (&xp)[NP],
                                           const u64 (&yp)[NP], const u64 (&zp)[NP], u64 (&ap)[NP]) {
#pragma unroll 8
    for (int j = 0; j < CHUNK; ++j) {
        const float4 sj = src[j];
#pragma unroll
        for (int h = 0; h < NP; ++h) {
            const u64 dx = sub2s(xp[h], sj.x), dy = sub2s(yp[h], sj.y), dz = sub2s(zp[h], sj.z);
            u64 r2 = mul2(dx, dx);
            r2 = fma2(dy, dy, r2);
            r2 = fma2(dz, dz, r2);
            float q0, q1;
            upk(r2, q0, q1);
            float r0, r1;
            asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(q0));
            asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(q1));
            if constexpr (MASK) {
                r0 = q0 > 0.f ? r0 : 0.f;
                r1 = q1 > 0.f ? r1 : 0.f;
            }
            ap[h] = fma2s(sj.w, pk(r0, r1), ap[h]);
        }
    }
}

// The same sum for one target, scalar and masked, over source tiles
// [tile0, tile1) read from global memory: the rare path for a target that
// coincides with a source outside the tiles the main loop masks.  Every
// operation is the lane-wise equivalent of the packed one, so the result is
// bitwise the one the masked packed loop gives.
__device__ __noinline__ float target_sum_masked(float x, float y, float z, const float4 *__restrict__ src4, int tile0,
                                   int tile1) {
    float sum = 0.f, comp = 0.f;
    for (int tl = tile0; tl < tile1; ++tl) {
        for (int c0 = 0; c0 < TILE; c0 += CHUNK) {
            float a = 0.f;
            for (int j = 0; j < CHUNK; ++j) {
                const float4 sj = src4[int64_t(tl) * TILE + c0 + j];
                const float dx = x - sj.x, dy = y - sj.y, dz = z - sj.z;
                float r2 = __fmul_rn(dx, dx);
                r2 = __fmaf_rn(dy, dy, r2);
                r2 = __fmaf_rn(dz, dz, r2);
                a = __fmaf_rn(sj.w, rinv(r2), a);
            }
            const float yk = __fsub_rn(a, comp);
            const float tk = __fadd_rn(sum, yk);
            comp = __fsub_rn(__fsub_rn(tk, sum), yk);
            sum = tk;
        }
    }
    return __fsub_rn(sum, comp);
}

// Packed sources: src4[j] = (x, y, z, q); entries ns .. ns_pad-1 are q = 0 at FAR.
__global__ void pack_kernel(int64_t ns, int64_t ns_pad, const float *__restrict__ s, int64_t lds,
                            const float *__restrict__ q, float4 *__restrict__ src4) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < ns_pad;
         j += int64_t(gridDim.x) * blockDim.x)
        src4[j] = j < ns ? make_float4(s[j * lds], s[j * lds + 1], s[j * lds + 2], q[j])
                         : make_float4(FAR, FAR, FAR, 0.f);
}

// One CTA = 1024 targets x one slice of the source tiles.  splits == 1: phi is
// written directly; else partial[slice][i].
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM)
    potential_kernel(int64_t nt, const float *__restrict__ t, int64_t ldt, const float4 *__restrict__ src4,
                     int ntiles, int splits, int self, float *__restrict__ phi, float *__restrict__ partial) {
    __shared__ float4 tile[2][TILE];
    const int tb = blockIdx.x / splits, sl = blockIdx.x - tb * splits;
    const int tile0 = int((int64_t(sl) * ntiles) / splits), tile1 = int((int64_t(sl + 1) * ntiles) / splits);

    // targets i = base + threadIdx.x + k * THREADS (coalesced), as pairs (0,1) and (2,3)
    const int64_t base = int64_t(tb) * THREADS * TPT + threadIdx.x;
    float tx[TPT], ty[TPT], tz[TPT];
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
        const int64_t i = base + int64_t(k) * THREADS;
        const int64_t ic = i < nt ? i : nt - 1;     // out-of-range lanes compute a copy, never stored
        tx[k] = t[ic * ldt];
        ty[k] = t[ic * ldt + 1];
        tz[k] = t[ic * ldt + 2];
    }
    constexpr int NP = TPT / 2;                      // target pairs per thread
    u64 xp[NP], yp[NP], zp[NP];
#pragma unroll
    for (int h = 0; h < NP; ++h) {
        xp[h] = pk(tx[2 * h], tx[2 * h + 1]);
        yp[h] = pk(ty[2 * h], ty[2 * h + 1]);
        zp[h] = pk(tz[2 * h], tz[2 * h + 1]);
    }
    u64 sp[NP], cp[NP];                              // Kahan sums of the chunk partials
#pragma unroll
    for (int h = 0; h < NP; ++h) sp[h] = cp[h] = 0;

    if (tile0 < tile1) tile[0][threadIdx.x] = src4[int64_t(tile0) * TILE + threadIdx.x];
    __syncthreads();
    // self-potential (targets are the sources): this CTA's own targets sit in
    // source tiles [diag0, diag1); only those need the coincidence mask
    const int diag0 = self ? tb * (THREADS * TPT / TILE) : 0;
    const int diag1 = self ? diag0 + THREADS * TPT / TILE : 0;
    for (int tl = tile0; tl < tile1; ++tl) {
        const int b = (tl - tile0) & 1;
        if (tl + 1 < tile1) tile[b ^ 1][threadIdx.x] = src4[int64_t(tl + 1) * TILE + threadIdx.x];
        const bool masked = tl >= diag0 && tl < diag1;
#pragma unroll 1
        for (int c0 = 0; c0 < TILE; c0 += CHUNK) {
            u64 ap[NP];
#pragma unroll
            for (int h = 0; h < NP; ++h) ap[h] = 0;
            if (masked) chunk_pass<true, NP>(&tile[b][c0], xp, yp, zp, ap);
            else        chunk_pass<false, NP>(&tile[b][c0], xp, yp, zp, ap);
#pragma unroll
            for (int h = 0; h < NP; ++h) kahan2(sp[h], cp[h], ap[h]);
        }
        __syncthreads();   // tile b fully read; tile b^1 fully written
    }

    float r[TPT];
#pragma unroll
    for (int h = 0; h < NP; ++h) upk(sub2(sp[h], cp[h]), r[2 * h], r[2 * h + 1]);
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
        const int64_t i = base + int64_t(k) * THREADS;
        if (i >= nt) continue;
        // a coincident point outside the masked tiles made this sum inf / NaN:
        // redo the target with the mask everywhere (bitwise what the masked loop gives)
        if (!isfinite(r[k])) r[k] = target_sum_masked(tx[k], ty[k], tz[k], src4, tile0, tile1);
        if (splits == 1) phi[i] = r[k];
        else             partial[int64_t(sl) * nt + i] = r[k];
    }
}

// phi[i] = the slice partials added in slice order (Kahan-compensated).
__global__ void reduce_kernel(int64_t nt, int splits, const float *__restrict__ partial, float *__restrict__ phi) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nt; i += int64_t(gridDim.x) * blockDim.x) {
        float sum = 0.f, comp = 0.f;
        for (int sl = 0; sl < splits; ++sl) {
            const float y = partial[int64_t(sl) * nt + i] - comp;
            const float tt = sum + y;
            comp = (tt - sum) - y;
            sum = tt;
        }
        phi[i] = sum - comp;
    }
}

}  // namespace coulomb

cudaError_t launch_coulomb(int64_t nt, const float *t, int64_t ldt, int64_t ns, const float *s, int64_t lds,
                           const float *q, float *phi, int num_sms, cudaStream_t st) {
    using namespace coulomb;
    if (nt <= 0) return cudaSuccess;
    const int64_t ntiles = ns > 0 ? (ns + TILE - 1) / TILE : 0;
    const int64_t blocks_t = (nt + int64_t(THREADS) * TPT - 1) / (int64_t(THREADS) * TPT);
    // source slices for an under-filled grid: fill CTAS_PER_SM CTAs on every SM
    // (choose_splits as for the GEMM; >= 4 tiles per slice)
    int splits = 1;
    if (ntiles > 0 && blocks_t < (int64_t(1) << 30))
        splits = choose_splits(int(blocks_t), int(ntiles), num_sms * CTAS_PER_SM, 4, 32);
    char *scratch = nullptr;
    const size_t src_bytes = size_t(ntiles > 0 ? ntiles : 1) * TILE * sizeof(float4);
    const size_t part_bytes = splits > 1 ? size_t(splits) * size_t(nt) * 4 : 0;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&scratch), src_bytes + part_bytes, st);
    if (e != cudaSuccess) return e;
    float4 *src4 = reinterpret_cast<float4 *>(scratch);
    float *partial = splits > 1 ? reinterpret_cast<float *>(scratch + src_bytes) : nullptr;
    if (ntiles > 0) {
        const int64_t ns_pad = ntiles * TILE;
        int64_t g = (ns_pad + 255) / 256;
        if (g > int64_t(num_sms) * 8) g = int64_t(num_sms) * 8;
        pack_kernel<<<unsigned(g), 256, 0, st>>>(ns, ns_pad, s, lds, q, src4);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        const int self = (t == s && ldt == lds && nt == ns) ? 1 : 0;
        potential_kernel<<<unsigned(blocks_t * splits), THREADS, 0, st>>>(nt, t, ldt, src4, int(ntiles), splits,
                                                                         self, phi, partial);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && splits > 1) {
        int64_t g = (nt + 255) / 256;
        if (g > int64_t(num_sms) * 8) g = int64_t(num_sms) * 8;
        reduce_kernel<<<unsigned(g), 256, 0, st>>>(nt, splits, partial, phi);
        e = cudaGetLastError();
    }
    cudaFreeAsync(scratch, st);
    return e;
}

}  // namespace lpy
