// FFMA (SIMT) path of C = A*B -- the paper's reduction `sum(k, a[i,k]*b[k,j])`
// scheduled the B200 way.
//
// Loo.py reaches a fast GEMM by split_iname into group/local axes
// (P:499-507), add_prefetch of A/B tiles into local memory
// (P:621-632), unrolling ("unr") and instruction-level parallelism
// ("ilp").  The sm_100a realisation:
//
//   * split i -> (tile_m, m in tile), j -> (tile_n, n in tile): 128x128 output
//     tiles, distributed over a PERSISTENT grid (one CTA per SM) in grouped
//     raster order so concurrently running tiles share A/B panels in L2;
//   * split k -> (k_block, k in block), BK = 32: the "prefetch" of A[tile,kb]
//     and B[kb,tile] is one TMA (cp.async.bulk.tensor) per operand per k-block
//     into a 4-stage shared-memory ring guarded by full/empty mbarriers
//     (producer warp <-> 8 consumer warps) instead of work-group barriers;
//   * ilp + unr: each consumer thread owns an 8x8 register micro-tile and runs
//     the k loop unrolled; operands come from shared memory as LDS.128
//     fragments with in-warp broadcast (8 lanes share each A fragment, 8 each
//     B fragment);
//   * ragged edges: TMA zero-fills out-of-range rows/columns/k of a
//     box, so the mainloop carries no conditionals; only the epilogue stores
//     are predicated.
//
// Layouts: for each operand the tile lands in shared memory in its
// storage orientation -- "MN-major" ([k][m] / [k][n], no swizzle) or
// "K-major" ([m][k] / [n][k], 128-byte TMA swizzle) -- and the fragment loader
// is specialised per orientation so every LDS.128 is bank-conflict-free.
// Accumulation is fp32 FFMA (RN) with k ascending per element.
#include <cstdio>
#include "lpy_internal.h"
#include "ptx.cuh"

namespace lpy {
namespace ffma {

constexpr int BN = 128, BK = 32;   // (BK = 64 with 3 stages measured no faster: 57.7 vs 58.0 TFLOP/s)
constexpr int KSUB = 32;                        // k per 128B-swizzled K-major sub-tile
constexpr int STAGES = 4;

// Per-variant geometry.  Consumer warps are laid out 4 along n (32 columns each)
// and CWARPS/4 along m (64 rows each).  (12 warps / 192 x 128 tiles was measured
// for the row-major layout and was slower: 55.6 vs 58 TFLOP/s, math-pipe
// throttle instead of latency was then the top stall.)
template <bool AK, bool BKM>
struct Geo {
    static constexpr int CWARPS = 8;                       // consumer warps
    static constexpr int BM = CWARPS / 4 * 64;
    static constexpr int THREADS = (CWARPS + 1) * 32;      // + 1 TMA producer warp
    static constexpr int A_TILE = BM * BK;                 // floats
    static constexpr int B_TILE = BN * BK;
    static constexpr uint32_t STAGE_BYTES = (A_TILE + B_TILE) * 4;
    static constexpr size_t SMEM_BYTES = 1024 + STAGES * size_t(STAGE_BYTES) + 2 * STAGES * 8;
};

struct Params {
    int M, N, K;
    float *C;
    int64_t ldc;
    int tiles_m, tiles_n, num_tiles, k_blocks, group;
    int c_vec;  // C base and ldc allow 16-byte stores
};

// Packed fp32 pairs for FFMA2.  c += a * b with c, b packed (lo, hi) pairs and
// the scalar a broadcast: fma.rn.f32x2 = two fp32 RN fused multiply-adds,
// bit-identical to two FFMAs, in half the issue slots.
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ void ffma2(unsigned long long &c, float a, unsigned long long b) {
    asm("{\n\t.reg .b64 x;\n\t"
        "mov.b64 x, {%1, %1};\n\t"
        "fma.rn.f32x2 %0, x, %2, %0;\n\t}"
        : "+l"(c)
        : "f"(a), "l"(b));
}

__device__ __forceinline__ void tile_coords(int t, const Params &p, int &tm, int &tn) {
    const int per_group = p.group * p.tiles_n;
    const int g = t / per_group;
    const int first = g * p.group;
    const int gsize = min(p.group, p.tiles_m - first);
    const int r = t - g * per_group;
    tm = first + r % gsize;
    tn = r / gsize;
}

// Row (within the 128-row tile) of this thread's i-th accumulator row.
template <bool AK>
__device__ __forceinline__ int a_row(int wm, int lm, int i) {
    return AK ? wm * 64 + lm + 8 * i : wm * 64 + (i >> 2) * 32 + lm * 4 + (i & 3);
}
template <bool BKM>
__device__ __forceinline__ int b_col(int wn, int ln, int j) {
    return BKM ? wn * 32 + ln + 4 * j : wn * 32 + (j >> 2) * 16 + ln * 4 + (j & 3);
}

// a[k][i] = A(tile row a_row(i), k-block column 4*kq + k)
template <bool AK, int BM>
__device__ __forceinline__ void load_a(const float *sa, int kq, int wm, int lm, float (&a)[4][8]) {
    if constexpr (AK) {
        // K-major tile: BK/KSUB sub-tiles of BM rows x 32 floats (128 B); 16-byte chunk c of
        // row m stored at c ^ (m & 7)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int m = wm * 64 + lm + 8 * i;
            const float4 v = *reinterpret_cast<const float4 *>(sa + (kq >> 3) * BM * KSUB + m * KSUB +
                                                                ((((kq & 7) ^ (m & 7))) << 2));
            a[0][i] = v.x; a[1][i] = v.y; a[2][i] = v.z; a[3][i] = v.w;
        }
    } else {
        // MN-major tile: k-row holds BM=128 floats
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float *row = sa + (kq * 4 + k) * BM + wm * 64 + lm * 4;
            const float4 v0 = *reinterpret_cast<const float4 *>(row);
            const float4 v1 = *reinterpret_cast<const float4 *>(row + 32);
            a[k][0] = v0.x; a[k][1] = v0.y; a[k][2] = v0.z; a[k][3] = v0.w;
            a[k][4] = v1.x; a[k][5] = v1.y; a[k][6] = v1.z; a[k][7] = v1.w;
        }
    }
}

template <bool BKM>
__device__ __forceinline__ void load_b(const float *sb, int kq, int wn, int ln, float (&b)[4][8]) {
    if constexpr (BKM) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int n = wn * 32 + ln + 4 * j;
            const float4 v = *reinterpret_cast<const float4 *>(sb + (kq >> 3) * BN * KSUB + n * KSUB +
                                                                ((((kq & 7) ^ (n & 7))) << 2));
            b[0][j] = v.x; b[1][j] = v.y; b[2][j] = v.z; b[3][j] = v.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float *row = sb + (kq * 4 + k) * BN + wn * 32 + ln * 4;
            const float4 v0 = *reinterpret_cast<const float4 *>(row);
            const float4 v1 = *reinterpret_cast<const float4 *>(row + 16);
            b[k][0] = v0.x; b[k][1] = v0.y; b[k][2] = v0.z; b[k][3] = v0.w;
            b[k][4] = v1.x; b[k][5] = v1.y; b[k][6] = v1.z; b[k][7] = v1.w;
        }
    }
}

template <bool AK, bool BKM>
__global__ void __launch_bounds__(Geo<AK, BKM>::THREADS, 1)
    gemm_ffma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const Params p) {
    using G = Geo<AK, BKM>;
    constexpr int CWARPS = G::CWARPS, BM = G::BM, A_TILE = G::A_TILE, B_TILE = G::B_TILE;
    constexpr uint32_t STAGE_BYTES = G::STAGE_BYTES;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzled K-major tiles
    const uint32_t raw = smem_u32(smem_raw);
    float *stages = reinterpret_cast<float *>(smem_raw + (((raw + 1023) & ~1023u) - raw));
    uint64_t *full = reinterpret_cast<uint64_t *>(stages + STAGES * (A_TILE + B_TILE));
    uint64_t *empty = full + STAGES;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CWARPS);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == CWARPS) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
                int tm, tn;
                tile_coords(t, p, tm, tn);
                const int m0 = tm * BM, n0 = tn * BN;
                for (int kb = 0; kb < p.k_blocks; ++kb) {
                    mbar_wait_sleep(&empty[stage], phase ^ 1, 2000);
                    float *sa = stages + stage * (A_TILE + B_TILE);
                    float *sb = sa + A_TILE;
                    mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
                    if constexpr (AK) {
#pragma unroll
                        for (int j = 0; j < BK / KSUB; ++j)
                            tma_load_2d(sa + j * BM * KSUB, &tmA, &full[stage], kb * BK + j * KSUB, m0);
                    } else {
                        tma_load_2d(sa, &tmA, &full[stage], m0, kb * BK);
                    }
                    if constexpr (BKM) {
#pragma unroll
                        for (int j = 0; j < BK / KSUB; ++j)
                            tma_load_2d(sb + j * BN * KSUB, &tmB, &full[stage], kb * BK + j * KSUB, n0);
                    } else {
                        tma_load_2d(sb, &tmB, &full[stage], n0, kb * BK);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
        return;
    }

    // ---------------------------------------------------- consumers
    const int wm = warp >> 2, wn = warp & 3;
    const int lm = lane >> 2, ln = lane & 3;
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int tm, tn;
        tile_coords(t, p, tm, tn);
        // Accumulators as packed pairs for FFMA2, paired along the operand whose
        // fragment arrives with adjacent elements from one LDS.128:
        //   PAIR_J (B MN-major): acc2[i][jp] = (acc(i, 2jp), acc(i, 2jp+1)), a broadcast
        //   PAIR_I (A MN-major, B K-major): acc2[ip][j] = (acc(2ip, j), acc(2ip+1, j)), b broadcast
        // Both K-major: plain FFMA (pairing would cost a register move per FFMA2).
        constexpr bool PAIR_J = !BKM, PAIR_I = BKM && !AK;
        constexpr int P0 = PAIR_I ? 4 : 8, P1 = PAIR_I ? 8 : 4;
        unsigned long long acc2[P0][P1];
        float accf[8][8];
#pragma unroll
        for (int i = 0; i < P0; ++i)
#pragma unroll
            for (int j = 0; j < P1; ++j) acc2[i][j] = 0ull;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) accf[i][j] = 0.f;

        for (int kb = 0; kb < p.k_blocks; ++kb) {
            mbar_wait(&full[stage], phase);
            const float *sa = stages + stage * (A_TILE + B_TILE);
            const float *sb = sa + A_TILE;
            constexpr int UNR = BKM ? 2 : 8;   // deep unroll where registers allow
#pragma unroll UNR
            for (int kq = 0; kq < BK / 4; ++kq) {
                float a[4][8], b[4][8];
                load_a<AK, BM>(sa, kq, wm, lm, a);
                load_b<BKM>(sb, kq, wn, ln, b);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if constexpr (PAIR_J) {
                        unsigned long long bp[4];   // adjacent registers: packing is free
#pragma unroll
                        for (int jp = 0; jp < 4; ++jp) bp[jp] = pack2(b[k][2 * jp], b[k][2 * jp + 1]);
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int jp = 0; jp < 4; ++jp) ffma2(acc2[i][jp], a[k][i], bp[jp]);
                    } else if constexpr (PAIR_I) {
                        unsigned long long ap[4];
#pragma unroll
                        for (int ip = 0; ip < 4; ++ip) ap[ip] = pack2(a[k][2 * ip], a[k][2 * ip + 1]);
#pragma unroll
                        for (int ip = 0; ip < 4; ++ip)
#pragma unroll
                            for (int j = 0; j < 8; ++j) ffma2(acc2[ip][j], b[k][j], ap[ip]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int j = 0; j < 8; ++j) accf[i][j] = fmaf(a[k][i], b[k][j], accf[i][j]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }

        // ------------------------------------------------ epilogue (ragged-edge stores)
        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if constexpr (PAIR_J) {
                    if (j % 2 == 0) unpack2(acc2[i][j / 2], acc[i][j], acc[i][j + 1]);
                } else if constexpr (PAIR_I) {
                    if (i % 2 == 0) unpack2(acc2[i / 2][j], acc[i][j], acc[i + 1][j]);
                } else {
                    acc[i][j] = accf[i][j];
                }
            }
        const int m0 = tm * BM, n0 = tn * BN;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = m0 + a_row<AK>(wm, lm, i);
            if (row >= p.M) continue;
            float *crow = p.C + int64_t(row) * p.ldc;
            if constexpr (!BKM) {
#pragma unroll
                for (int jq = 0; jq < 2; ++jq) {
                    const int col = n0 + b_col<BKM>(wn, ln, jq * 4);
                    if (p.c_vec && col + 3 < p.N) {
                        *reinterpret_cast<float4 *>(crow + col) =
                            make_float4(acc[i][jq * 4 + 0], acc[i][jq * 4 + 1], acc[i][jq * 4 + 2],
                                        acc[i][jq * 4 + 3]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (col + e < p.N) crow[col + e] = acc[i][jq * 4 + e];
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int col = n0 + b_col<BKM>(wn, ln, j);
                    if (col < p.N) crow[col] = acc[i][j];
                }
            }
        }
    }
}

template <bool AK, bool BKM>
static cudaError_t launch_t(const Problem &p, const Knobs &kn, cudaStream_t s) {
    using G = Geo<AK, BKM>;
    constexpr int BM = G::BM;
    CUtensorMap ta, tb;
    cudaError_t e;
    if (AK) e = make_tmap_2d(&ta, p.A, p.K, p.M, p.lda, KSUB, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    else    e = make_tmap_2d(&ta, p.A, p.M, p.K, p.lda, BM, BK, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (e != cudaSuccess) return e;
    if (BKM) e = make_tmap_2d(&tb, p.B, p.K, p.N, p.ldb, KSUB, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    else     e = make_tmap_2d(&tb, p.B, p.N, p.K, p.ldb, BN, BK, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (e != cudaSuccess) return e;

    Params prm;
    prm.M = p.M; prm.N = p.N; prm.K = p.K;
    prm.C = p.C; prm.ldc = p.ldc;
    prm.tiles_m = (p.M + BM - 1) / BM;
    prm.tiles_n = (p.N + BN - 1) / BN;
    prm.num_tiles = prm.tiles_m * prm.tiles_n;
    prm.k_blocks = (p.K + BK - 1) / BK;
    prm.group = kn.raster_group > 0 ? kn.raster_group : 16;
    prm.c_vec = ((reinterpret_cast<uintptr_t>(p.C) & 15) == 0) && (p.ldc % 4 == 0);
    int grid = kn.num_ctas > 0 ? kn.num_ctas : kn.num_sms;
    if (grid > prm.num_tiles) grid = prm.num_tiles;
    if (grid < 1) grid = 1;

    auto kern = gemm_ffma_kernel<AK, BKM>;
    static bool attr_done = false;  // benign race: setting the attribute twice is harmless
    if (!attr_done) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(G::SMEM_BYTES));
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    kern<<<grid, G::THREADS, G::SMEM_BYTES, s>>>(ta, tb, prm);
    return cudaGetLastError();
}

}  // namespace ffma

cudaError_t launch_ffma(const Problem &p, const Knobs &kn, cudaStream_t s) {
    using namespace ffma;
    const bool AK = (p.la == 0);   // row-major A: K contiguous
    const bool BKM = (p.lb == 1);  // column-major B: K contiguous
    if (AK && BKM)  return launch_t<true, true>(p, kn, s);
    if (AK && !BKM) return launch_t<true, false>(p, kn, s);
    if (!AK && BKM) return launch_t<false, true>(p, kn, s);
    return launch_t<false, false>(p, kn, s);
}

}  // namespace lpy
