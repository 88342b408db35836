// FFMA (SIMT) path of C = A*B -- the paper's reduction `sum(k, a[i,k]*b[k,j])`
// scheduled the B200 way.
//
// Loo.py reaches a fast GEMM by split_iname into group/local axes
// (P:499-507), add_prefetch of A/B tiles into local memory
// (P:621-632), unrolling ("unr") and instruction-level parallelism
// ("ilp").  The sm_100a realisation:
//
//   * split i -> (tile_m, m in tile), j -> (tile_n, n in tile): 128 x 256 (or
//     128 x 128 when that fills the waves better) output tiles, distributed over
//     a PERSISTENT grid (one CTA per SM) in grouped raster order so
//     concurrently running tiles share A/B panels in L2;
//   * split k -> (k_block, k in block), BK = 32: the "prefetch" of A[tile,kb]
//     and B[kb,tile] is one TMA (cp.async.bulk.tensor) per operand per k-block
//     into a shared-memory ring guarded by full/empty mbarriers (producer warp
//     <-> consumer warps) instead of work-group barriers;
//   * ilp + unr: each consumer thread owns an 8 x 16 (or 8 x 8) register
//     micro-tile and runs the k loop fully unrolled; operands come from shared memory as LDS.128
//     fragments with in-warp broadcast, and the products are packed FFMA2
//     (fma.rn.f32x2: two fp32 RN FMAs per instruction, a scalar of A times a
//     pair of adjacent B columns);
//   * ragged edges: TMA zero-fills out-of-range rows/columns/k of a
//     box, so the mainloop carries no conditionals; only the epilogue stores
//     are predicated.
//
// Layouts.  The consumers always read both operands "MN-major"
// ([k][m] and [k][n]: 4 adjacent rows / columns per LDS.128), the orientation
// whose fragments feed FFMA2 without any register repacking.  An operand
// stored K-major (row-major A, column-major B) lands from TMA as [m][k] /
// [n][k] with the 128-byte swizzle, and three "transpose" warps rewrite each
// such tile into an MN-major copy (4x4 register transposes, bank-conflict-free
// on both sides) -- the paper's "precompute" into local temporaries
// used as a layout change -- before the consumers see it.
// Accumulation is fp32 FFMA (RN) with k ascending per element, identical for
// every layout.
//
// Under-filled grids (the paper's "separate code for edge and corner cases",
// P:524-528): a single wave of too few tiles splits K inside a thread-block
// cluster (DSMEM reduction); a ragged last wave is stream-K'd (its k-iterations
// dealt over every planned SM, pieces summed in k order by the last to finish,
// in the consumer warps); otherwise split-K slices and a fix-up kernel --
// whichever choose_stream_k's model says is shortest.  The producer honours
// the K-gate of lpy_gemm_f32_gated like the 3xTF32 one.
#include <cstdio>
#include <cstdlib>
#include "lpy_internal.h"
#include "ptx.cuh"

namespace lpy {
namespace ffma {

constexpr int BM = 128, BK = 32;             // tile width BN: template (128 or 256)
constexpr int KSUB = 32;                     // k per 128B-swizzled K-major TMA box (= BK)
constexpr int CWARPS = 8;                    // consumer warps: 2 along m (64 rows) x 4 along n (BN/4 cols)
constexpr int XWARPS = 3;                    // transpose warps (warps CWARPS+1 .. CWARPS+3)
constexpr int MAX_SPLITS = 8;                // split-K slices at most (choose_splits' cap; cluster size)

// Per-layout geometry.  AK: A is K-major (row-major A); BKM: B is K-major
// (column-major B).  Each stage holds the raw TMA tiles plus MN-major copies
// of the K-major ones.
template <bool AK, bool BKM, int BN, bool SPLIT = false>
struct Geo {
    static constexpr bool XA = AK, XB = BKM, X = AK || BKM;
    static constexpr int JN = BN / 32;                     // column pairs per thread (8 x 2JN micro-tile)
    static constexpr int STAGE_FLOATS_ = BM * BK + BN * BK + (XA ? BM * BK : 0) + (XB ? BN * BK : 0);
    static constexpr int STAGES_FIT = int((227 * 1024 - 1024 - 256) / (STAGE_FLOATS_ * 4));
    static constexpr int STAGES = STAGES_FIT < 4 ? STAGES_FIT : 4;
    // 8 consumer warps + a producer warpgroup (warp CWARPS: one TMA lane; the next
    // XWARPS warps: transposes).  A whole warpgroup so setmaxnreg can move its
    // registers to the consumers: launched at 168/thread (the SMSP holding 3
    // warps caps a 12-warp CTA there), consumers rise to REGS_CONS, the producer
    // group drops to REGS_PROD (2*32*224 + 32*56 <= 16384 per SMSP).
    static constexpr int THREADS = (CWARPS + 4) * 32;
    static constexpr int REGS_CONS = 224, REGS_PROD = 56;
    static constexpr int A_TILE = BM * BK, B_TILE = BN * BK;   // floats
    static constexpr int STAGE_FLOATS = A_TILE + B_TILE + (XA ? A_TILE : 0) + (XB ? B_TILE : 0);
    static constexpr uint32_t TMA_BYTES = (A_TILE + B_TILE) * 4;
    static constexpr size_t SMEM_BYTES = 1024 + STAGES * size_t(STAGE_FLOATS) * 4 + 3 * STAGES * 8;
};

struct Params {
    int M, N, K;
    float *C;
    int64_t ldc;
    int tiles_m, tiles_n, num_tiles, k_blocks, group;
    int c_vec;  // C base and ldc allow 16-byte stores
    // split-K (bulk/edge specialisation for under-filled grids): work unit
    // u = tile * splits + slice covers k-blocks [slice*KB/splits, (slice+1)*KB/splits)
    int splits, num_units;
    float *ws;       // [num_units][BM*BN] partial tiles (splits > 1, not cluster_split)
    // cluster split (a single wave, splits <= 8): the `splits` CTAs of one
    // cluster compute the slices of one tile and sum them through distributed
    // shared memory (no ws, no fix-up kernel)
    int cluster_split;
    int ws_stride;   // float4 stride between a thread's partial float4s: 256 (interleaved) or 1 (LPY_FFMA_PARTIAL=contig, A/B)
    KGate gate;      // operands arriving in chunks of K (lpy_kgate): the producer waits per k-block
    // Stream-K (sk_workers > 0; replaces the equal slices above): tiles
    // [0, full_tiles) are one unit each; the remaining tiles' sk_iters =
    // (num_tiles - full_tiles) * k_blocks k-block iterations are dealt out
    // evenly to sk_workers workers (worker w: [floor(w W / P), floor((w+1) W / P))),
    // a range at most one tile long, so it covers at most two pieces: unit
    // full_tiles + piece * sk_stride + w (empty when it does not exist).  With
    // a grid of sk_stride CTAs, CTA w runs worker w.  The pieces of a tile are
    // summed in the kernel, in k order, by the piece that finishes last
    // (tickets in sem); partials park in ws (slot = unit - full_tiles).
    int full_tiles, sk_workers, sk_stride;
    long long sk_iters;
    int *sem;        // 2 x [num_tiles - full_tiles] ticket / written counters, zero on entry and exit
};

// Stream-K: the worker whose iteration range contains tail iteration x, and
// the first iteration of worker w.
__device__ __forceinline__ int sk_worker_of(long long x, const Params &p) {
    return int(((x + 1) * p.sk_workers + p.sk_iters - 1) / p.sk_iters) - 1;
}
__device__ __forceinline__ long long sk_begin(int w, const Params &p) {
    return (static_cast<long long>(w) * p.sk_iters) / p.sk_workers;
}

// Work unit u -> tile t and k-block range [kb0, kb1) (empty when kb0 >= kb1).
__device__ __forceinline__ void unit_range(int u, const Params &p, int &t, int &kb0, int &kb1) {
    if (p.sk_workers > 0) {
        if (u < p.full_tiles) {
            t = u; kb0 = 0; kb1 = p.k_blocks;
            return;
        }
        const int su = u - p.full_tiles;
        const int piece = su / p.sk_stride, w = su - piece * p.sk_stride;
        t = p.full_tiles; kb0 = kb1 = 0;
        if (w >= p.sk_workers) return;
        const long long b0 = sk_begin(w, p), b1 = sk_begin(w + 1, p), kb = p.k_blocks;
        const long long vt = b0 / kb + piece;
        const long long lo = max(b0, vt * kb), hi = min(b1, (vt + 1) * kb);
        if (lo >= hi) return;
        t = p.full_tiles + int(vt);
        kb0 = int(lo - vt * kb);
        kb1 = int(hi - vt * kb);
        return;
    }
    t = u / p.splits;
    const int s = u - t * p.splits;
    kb0 = int((int64_t(s) * p.k_blocks) / p.splits);
    kb1 = int((int64_t(s + 1) * p.k_blocks) / p.splits);
}
// The pieces of stream-K tail tile vt in k order: count, and the unit slot
// (index past full_tiles) of the i-th.
__device__ __forceinline__ int sk_pieces(int vt, const Params &p) {
    const long long kb = p.k_blocks;
    return sk_worker_of((vt + 1) * kb - 1, p) - sk_worker_of(vt * kb, p) + 1;
}
__device__ __forceinline__ int sk_slot(int vt, int i, const Params &p) {
    const long long kb = p.k_blocks;
    const int w = sk_worker_of(vt * kb, p) + i;
    const int piece = int(sk_begin(w, p) / kb) == vt ? 0 : 1;
    return piece * p.sk_stride + w;
}

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

// Row (within the tile) of this thread's i-th accumulator row, column of its j-th:
// 8 rows (two groups of 4 adjacent, 32 apart) x 2JN columns (groups of 4
// adjacent, 16 apart) -- every fragment is one conflict-free LDS.128 per group.
__device__ __forceinline__ int a_row(int wm, int lm, int i) { return wm * 64 + (i >> 2) * 32 + lm * 4 + (i & 3); }
template <int JN>
__device__ __forceinline__ int b_col(int wn, int ln, int j) {
    return wn * (8 * JN) + (j >> 2) * 16 + ln * 4 + (j & 3);
}

// a[i] = A(a_row(i), k) from an MN-major [BK][BM] tile.
__device__ __forceinline__ void load_a(const float *sa, int k, int wm, int lm, float (&a)[8]) {
    const float *row = sa + k * BM + wm * 64 + lm * 4;
    const float4 v0 = *reinterpret_cast<const float4 *>(row);
    const float4 v1 = *reinterpret_cast<const float4 *>(row + 32);
    a[0] = v0.x; a[1] = v0.y; a[2] = v0.z; a[3] = v0.w;
    a[4] = v1.x; a[5] = v1.y; a[6] = v1.z; a[7] = v1.w;
}

// b[j] = B(k, b_col(j)) from an MN-major [BK][BN] tile.
template <int JN, int BN>
__device__ __forceinline__ void load_b(const float *sb, int k, int wn, int ln, float (&b)[2 * JN]) {
    const float *row = sb + k * BN + wn * (8 * JN) + ln * 4;
#pragma unroll
    for (int g = 0; g < JN / 2; ++g) {
        const float4 v = *reinterpret_cast<const float4 *>(row + 16 * g);
        b[4 * g] = v.x; b[4 * g + 1] = v.y; b[4 * g + 2] = v.z; b[4 * g + 3] = v.w;
    }
}

// K-major tile (128 lines x 32 k, TMA 128B swizzle: 16-byte chunk c of line r
// stored at chunk c ^ (r & 7)) -> MN-major [32 k][128] copy.  The tile is 8
// k-chunks x 32 line-groups of 4x4 blocks; one warp pass covers 4 chunks x 8
// line-groups.  128-bit shared accesses are served a quarter-warp (8 lanes) at
// a time, so each quarter must touch 8 distinct 16-byte bank groups on both
// sides: lane l = lane & 7 of quarter k takes line-group g0 + l (distinct
// groups for the STS.128 rows) and chunk c0 + ((l/2 + k) & 3) (4 chunks per
// line-group parity, whose swizzles differ in bit 2, for the LDS.128) -- 4
// wavefronts per 512 B on both sides.  (A lane = chunk + 4 * group mapping
// stored with 16 wavefronts: ncu, profiles/r02_ffma_transpose_banks.txt.)
template <int LINES>
__device__ __forceinline__ void transpose_tile(const float *src, float *dst, int xw, int lane) {
    for (int it = xw; it < LINES / 16; it += XWARPS) {
        const int l = lane & 7;
        const int c = (it & 1) * 4 + (((l >> 1) + (lane >> 3)) & 3);
        const int g = (it >> 1) * 8 + l;
        float4 r[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int line = 4 * g + q;
            r[q] = *reinterpret_cast<const float4 *>(src + line * KSUB + ((c ^ (line & 7)) << 2));
        }
        float *d = dst + (4 * c) * LINES + 4 * g;
        *reinterpret_cast<float4 *>(d + 0 * LINES) = make_float4(r[0].x, r[1].x, r[2].x, r[3].x);
        *reinterpret_cast<float4 *>(d + 1 * LINES) = make_float4(r[0].y, r[1].y, r[2].y, r[3].y);
        *reinterpret_cast<float4 *>(d + 2 * LINES) = make_float4(r[0].z, r[1].z, r[2].z, r[3].z);
        *reinterpret_cast<float4 *>(d + 3 * LINES) = make_float4(r[0].w, r[1].w, r[2].w, r[3].w);
    }
}

template <bool AK, bool BKM, int BN, bool SPLIT>
__global__ void __launch_bounds__(Geo<AK, BKM, BN, SPLIT>::THREADS, 1)
    gemm_ffma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const Params p) {
    using G = Geo<AK, BKM, BN, SPLIT>;
    constexpr int JN = G::JN;
    constexpr int STAGES = G::STAGES, A_TILE = G::A_TILE, B_TILE = G::B_TILE, SF = G::STAGE_FLOATS;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzled K-major tiles
    const uint32_t raw = smem_u32(smem_raw);
    float *stages = reinterpret_cast<float *>(smem_raw + (((raw + 1023) & ~1023u) - raw));
    uint64_t *full = reinterpret_cast<uint64_t *>(stages + STAGES * SF);  // TMA landed
    uint64_t *xfull = full + STAGES;                                      // transposes written
    uint64_t *empty = xfull + STAGES;                                     // stage free again
    // stage s: [raw A][raw B][MN-major A if AK][MN-major B if BKM]
    auto raw_a = [&](int s) { return stages + s * SF; };
    auto raw_b = [&](int s) { return stages + s * SF + A_TILE; };
    auto x_a = [&](int s) { return stages + s * SF + A_TILE + B_TILE; };
    auto x_b = [&](int s) { return stages + s * SF + A_TILE + B_TILE + (G::XA ? A_TILE : 0); };

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&xfull[s], XWARPS * 32);
            mbar_init(&empty[s], CWARPS + (G::X ? XWARPS : 0));
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp >= CWARPS) {
        setmaxnreg_dec<G::REGS_PROD>();
        if (warp == CWARPS) {
            // -------------------------------------------- TMA producer
            if (lane == 0) {
                tma_prefetch_desc(&tmA);
                tma_prefetch_desc(&tmB);
                int stage = 0;
                uint32_t phase = 0;
                int gready = -1;                           // K-gate: chunks known ready
                int glimit = kgate_limit0(p.gate);         // ... and the first k-block they do not cover
                for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
                    int t, kb0, kb1, tm, tn;
                    unit_range(u, p, t, kb0, kb1);
                    tile_coords(t, p, tm, tn);
                    const int m0 = tm * BM, n0 = tn * BN;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        if (kb >= glimit) glimit = kgate_admit(p.gate, gready, kb, BK, p.K);
                        mbar_wait_sleep(&empty[stage], phase ^ 1, 2000);
                        mbar_arrive_expect_tx(&full[stage], G::TMA_BYTES);
                        if constexpr (AK) tma_load_2d(raw_a(stage), &tmA, &full[stage], kb * BK, m0);
                        else              tma_load_2d(raw_a(stage), &tmA, &full[stage], m0, kb * BK);
                        if constexpr (BKM) tma_load_2d(raw_b(stage), &tmB, &full[stage], kb * BK, n0);
                        else               tma_load_2d(raw_b(stage), &tmB, &full[stage], n0, kb * BK);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        } else if constexpr (G::X) {
            // -------------------------------------------- transposes of K-major tiles
            const int xw = warp - CWARPS - 1;
            int stage = 0;
            uint32_t phase = 0;
            for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
                int t, kb0, kb1;
                unit_range(u, p, t, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    if constexpr (G::XA) transpose_tile<BM>(raw_a(stage), x_a(stage), xw, lane);
                    if constexpr (G::XB) transpose_tile<BN>(raw_b(stage), x_b(stage), xw, lane);
                    // this lane's STS of the copy (and LDS of the raw tile) must be
                    // complete before it publishes the copy and frees the raw tile
                    asm volatile("fence.acq_rel.cta;" ::: "memory");
                    mbar_arrive(&xfull[stage]);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
        if (SPLIT && p.cluster_split) {   // the consumers' two cluster barriers
            cluster_sync();
            cluster_sync();
        }
        return;
    }

    // ---------------------------------------------------- consumers
    setmaxnreg_inc<G::REGS_CONS>();
    const int wm = warp >> 2, wn = warp & 3;
    const int lm = lane >> 2, ln = lane & 3;
    int stage = 0;
    uint32_t phase = 0;
    __shared__ int sk_last;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
        int t, kb0, kb1, tm, tn;
        unit_range(u, p, t, kb0, kb1);
        if (kb0 >= kb1) continue;   // an empty stream-K unit
        tile_coords(t, p, tm, tn);
        // acc2[i][jp] = (acc(i, 2jp), acc(i, 2jp+1)): pairs along n, where one
        // LDS.128 of the MN-major B tile delivers adjacent columns
        unsigned long long acc2[8][JN];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < JN; ++j) acc2[i][j] = 0ull;

        for (int kb = kb0; kb < kb1; ++kb) {
            if constexpr (!(G::XA && G::XB)) mbar_wait(&full[stage], phase);   // reads a raw tile
            if constexpr (G::X) mbar_wait(&xfull[stage], phase);
            const float *sa = G::XA ? x_a(stage) : raw_a(stage);
            const float *sb = G::XB ? x_b(stage) : raw_b(stage);
#ifdef LPY_MUTATE_STAGE_RACE
            // MUTATION (liblpy_mutant.so, tests/test_mutation_gpu.py only): the
            // stage is released BEFORE it is read, so the producer may refill it
            // under the consumers -- the race the detector tests must catch
            mbar_arrive_after_reads(&empty[stage], lane);
#endif
#pragma unroll
            for (int k = 0; k < BK; ++k) {
                float a[8], b[2 * JN];
                load_a(sa, k, wm, lm, a);
                load_b<JN, BN>(sb, k, wn, ln, b);
                unsigned long long bp[JN];   // adjacent registers: packing is free
#pragma unroll
                for (int jp = 0; jp < JN; ++jp) bp[jp] = pack2(b[2 * jp], b[2 * jp + 1]);
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int jp = 0; jp < JN; ++jp) ffma2(acc2[i][jp], a[i], bp[jp]);
            }
#ifndef LPY_MUTATE_STAGE_RACE
            mbar_arrive_after_reads(&empty[stage], lane);
#endif
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }

        if (SPLIT && p.cluster_split) {
            // ---------------------------------------- cluster split: DSMEM sum
            // Park the partial in this CTA's operand ring (idle once every
            // consumer has read its last stage: one unit per CTA, no more TMA),
            // rows padded by 4 floats; after a cluster barrier CTA r of the
            // cluster sums rows [r*BM/S, (r+1)*BM/S) over the S slices in slice
            // order -- the fix-up kernel's order, so results are bitwise those of
            // the global-memory split -- and stores them coalesced.
            named_bar_sync(1, CWARPS * 32);
            constexpr int LDS_ = BN + 4;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int jp = 0; jp < JN; jp += 2) {
                    float lo0, hi0, lo1, hi1;
                    unpack2(acc2[i][jp], lo0, hi0);
                    unpack2(acc2[i][jp + 1], lo1, hi1);
                    *reinterpret_cast<float4 *>(stages + a_row(wm, lm, i) * LDS_ + b_col<JN>(wn, ln, 2 * jp)) =
                        make_float4(lo0, hi0, lo1, hi1);
                }
            cluster_sync();
            const int S = p.splits, r = int(cluster_ctarank());
            const int r0 = r * BM / S, r1 = (r + 1) * BM / S;
            constexpr int C4 = BN / 4;
            const int m0 = tm * BM, n0 = tn * BN;
            const uint32_t stg = smem_u32(stages);
            for (int idx = threadIdx.x; idx < (r1 - r0) * C4; idx += CWARPS * 32) {
                const int rl = r0 + idx / C4, c4 = idx % C4;
                const uint32_t off = stg + uint32_t((rl * LDS_ + c4 * 4) * 4);
                float4 v[MAX_SPLITS];
#pragma unroll
                for (int sl = 0; sl < MAX_SPLITS; ++sl)
                    if (sl < S) v[sl] = ld_dsmem_v4(mapa_shared(off, uint32_t(sl)));
#pragma unroll
                for (int sl = 1; sl < MAX_SPLITS; ++sl)
                    if (sl < S) { v[0].x += v[sl].x; v[0].y += v[sl].y; v[0].z += v[sl].z; v[0].w += v[sl].w; }
                const int row = m0 + rl, col = n0 + c4 * 4;
                if (row < p.M) {
                    float *c = p.C + int64_t(row) * p.ldc + col;
                    if (p.c_vec && col + 3 < p.N) {
                        *reinterpret_cast<float4 *>(c) = v[0];
                    } else {
                        const float o[4] = {v[0].x, v[0].y, v[0].z, v[0].w};
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (col + e < p.N) c[e] = o[e];
                    }
                }
            }
            cluster_sync();   // peers done reading this CTA's partial
            continue;
        }
        if (SPLIT && p.sk_workers > 0 && u >= p.full_tiles && !(kb0 == 0 && kb1 == p.k_blocks)) {
            // ---------------------------------------- stream-K piece: fix-up in the kernel
            // Each piece of a tail tile takes a ticket; all but the last park
            // their partial (thread-interleaved, as the split-K slices do) and
            // count themselves written; the last waits for those writes -- the
            // writers already hold tickets, so they are running and the wait is
            // bounded -- and sums the pieces in k order, its own from registers:
            // ((p0 + p1) + p2) ..., with the own piece first or second the
            // running sum starts from acc (p1 + p0 == p0 + p1 bitwise); a later
            // own piece is parked and the sum rebuilt from memory.  The order is
            // fixed by the decomposition, never by who finishes last.
            const int vt = t - p.full_tiles;
            const int npieces = sk_pieces(vt, p);
            const int su = u - p.full_tiles;
            const int me = su % p.sk_stride - sk_worker_of(static_cast<long long>(vt) * p.k_blocks, p);
            int *arrive = p.sem + vt;
            int *written = p.sem + (p.num_tiles - p.full_tiles) + vt;
            constexpr int NV = 8 * JN / 2;                    // float4s per thread
            auto slot_ptr = [&](int i) {
                return reinterpret_cast<float4 *>(p.ws + int64_t(sk_slot(vt, i, p)) * (BM * BN)) + threadIdx.x;
            };
            auto park = [&](float4 *dst) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int jp = 0; jp < JN; jp += 2) {
                        float lo0, hi0, lo1, hi1;
                        unpack2(acc2[i][jp], lo0, hi0);
                        unpack2(acc2[i][jp + 1], lo1, hi1);
                        __stcg(dst + ((i * JN + jp) / 2) * (CWARPS * 32), make_float4(lo0, hi0, lo1, hi1));
                    }
            };
            if (threadIdx.x == 0) sk_last = atomicAdd(arrive, 1) == npieces - 1;
            named_bar_sync(1, CWARPS * 32);
            if (!sk_last) {
                park(slot_ptr(me));
                __threadfence();
                named_bar_sync(1, CWARPS * 32);
                if (threadIdx.x == 0) atomicAdd(written, 1);
                continue;
            }
            if (threadIdx.x == 0) {
                while (ld_acquire_gpu(written) < npieces - 1) __nanosleep(64);
                *arrive = 0;      // ready for the next launch (nobody else touches them now)
                *written = 0;
            }
            named_bar_sync(1, CWARPS * 32);
            __threadfence();
            float acc[8][2 * JN];
            int i0 = 0;
            if (me >= 2) {
                park(slot_ptr(me));
                __threadfence_block();
                const float4 *src = slot_ptr(0);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float4 x = __ldcg(src + v * (CWARPS * 32));
                    const int i = (2 * v) / JN, j = (4 * v) % (2 * JN);
                    acc[i][j] = x.x; acc[i][j + 1] = x.y; acc[i][j + 2] = x.z; acc[i][j + 3] = x.w;
                }
                i0 = 1;
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int jp = 0; jp < JN; ++jp) unpack2(acc2[i][jp], acc[i][2 * jp], acc[i][2 * jp + 1]);
            }
#pragma unroll 1
            for (int q = i0; q < npieces; ++q) {
                if (q == me && me < 2) continue;
                const float4 *src = slot_ptr(q);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float4 x = __ldcg(src + v * (CWARPS * 32));
                    const int i = (2 * v) / JN, j = (4 * v) % (2 * JN);
                    acc[i][j] += x.x; acc[i][j + 1] += x.y; acc[i][j + 2] += x.z; acc[i][j + 3] += x.w;
                }
            }
            const int m0 = tm * BM, n0 = tn * BN;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int row = m0 + a_row(wm, lm, i);
                if (row >= p.M) continue;
                float *crow = p.C + int64_t(row) * p.ldc;
#pragma unroll
                for (int jq = 0; jq < JN / 2; ++jq) {
                    const int col = n0 + b_col<JN>(wn, ln, jq * 4);
                    if (p.c_vec && col + 3 < p.N) {
                        *reinterpret_cast<float4 *>(crow + col) =
                            make_float4(acc[i][jq * 4 + 0], acc[i][jq * 4 + 1], acc[i][jq * 4 + 2], acc[i][jq * 4 + 3]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (col + e < p.N) crow[col + e] = acc[i][jq * 4 + e];
                    }
                }
            }
            continue;
        }
        if (SPLIT && p.sk_workers == 0) {
            // ---------------------------------------- split-K: park the partial
            // Every slice stores its partial tile (each thread its own 8 x 2JN
            // values, contiguous) and the fix-up kernel (splitk_fixup) adds the
            // slices of each tile in slice order -- a fixed order, independent of
            // which slice finished first.
            // thread-interleaved: float4 v of thread t at [v][t], so a warp's store
            // covers 512 contiguous bytes (a per-thread-contiguous layout put
            // its 32 lanes 512 B apart: 32 sectors per instruction)
            float4 *mine = reinterpret_cast<float4 *>(p.ws + int64_t(u) * (BM * BN)) +
                           threadIdx.x * (p.ws_stride == 1 ? 8 * JN / 2 : 1);
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int jp = 0; jp < JN; jp += 2) {
                    float lo0, hi0, lo1, hi1;
                    unpack2(acc2[i][jp], lo0, hi0);
                    unpack2(acc2[i][jp + 1], lo1, hi1);
                    mine[((i * JN + jp) / 2) * p.ws_stride] = make_float4(lo0, hi0, lo1, hi1);
                }
            continue;
        }

        // ------------------------------------------------ epilogue (ragged-edge stores)
        const int m0 = tm * BM, n0 = tn * BN;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = m0 + a_row(wm, lm, i);
            if (row >= p.M) continue;
            float acc[2 * JN];
#pragma unroll
            for (int jp = 0; jp < JN; ++jp) unpack2(acc2[i][jp], acc[2 * jp], acc[2 * jp + 1]);
            float *crow = p.C + int64_t(row) * p.ldc;
#pragma unroll
            for (int jq = 0; jq < JN / 2; ++jq) {
                const int col = n0 + b_col<JN>(wn, ln, jq * 4);
                if (p.c_vec && col + 3 < p.N) {
                    *reinterpret_cast<float4 *>(crow + col) =
                        make_float4(acc[jq * 4 + 0], acc[jq * 4 + 1], acc[jq * 4 + 2], acc[jq * 4 + 3]);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (col + e < p.N) crow[col + e] = acc[jq * 4 + e];
                }
            }
        }
    }
    // the split-K fix-up (launched with programmatic dependent launch) may start
    // once every CTA's consumers are past their last unit; it waits for this
    // grid's completion (griddepcontrol.wait) before reading the partials
    if constexpr (SPLIT) pdl_launch_dependents();
}

// Split-K fix-up: FIXUP_PARTS CTAs of 256 threads per output tile, part r
// taking micro-tile rows i in [r * 8 / FIXUP_PARTS, (r + 1) * 8 / FIXUP_PARTS);
// thread ctid owns the elements consumer thread ctid of the GEMM kernel owned
// (same a_row / b_col map), adds the tile's slice partials in slice order and
// stores C with the same ragged-edge predicates.  Several CTAs per tile: one
// SM pulls only ~50 GB/s of partials from L2 (bytes in flight / latency), so
// the fix-up is spread over more SMs than there are tiles.
constexpr int FIXUP_PARTS = 8;   // 8 vs 4: ragged config 103.3 -> 102.5 us, others equal (profiles/r01_ffma_partial_layout.txt)
template <int BN>
__global__ void __launch_bounds__(CWARPS * 32) splitk_fixup_kernel(const Params p) {
    pdl_wait();                 // the slices' partials (the split-K grid) are complete and visible
    constexpr int JN = BN / 32;
    const int IPART = 8 / int(gridDim.y);   // gridDim.y = parts per tile (1, 2, 4 or 8)
    const int t = blockIdx.x;
    const int i0 = blockIdx.y * IPART;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp >> 2, wn = warp & 3, lm = lane >> 2, ln = lane & 3;
    int tm, tn;
    tile_coords(t, p, tm, tn);
    const float4 *base = reinterpret_cast<const float4 *>(p.ws + int64_t(t) * p.splits * (BM * BN)) +
                         threadIdx.x * (p.ws_stride == 1 ? 8 * JN / 2 : 1);   // [v][thread] within each slice's tile
    const int m0 = tm * BM, n0 = tn * BN;
    for (int ii = 0; ii < IPART; ++ii) {
        const int i = i0 + ii;
        const int row = m0 + a_row(wm, lm, i);
        float acc[2 * JN];
#pragma unroll
        for (int h = 0; h < JN / 2; ++h) {
            float4 s0 = base[(i * (JN / 2) + h) * p.ws_stride];
#pragma unroll
            for (int sl = 1; sl < MAX_SPLITS; ++sl) {   // unrolled: every slice's load in flight
                if (sl < p.splits) {
                    const float4 q = base[int64_t(sl) * (BM * BN / 4) + (i * (JN / 2) + h) * p.ws_stride];
                    s0.x += q.x; s0.y += q.y; s0.z += q.z; s0.w += q.w;
                }
            }
            acc[4 * h] = s0.x; acc[4 * h + 1] = s0.y; acc[4 * h + 2] = s0.z; acc[4 * h + 3] = s0.w;
        }
        if (row >= p.M) continue;
        float *crow = p.C + int64_t(row) * p.ldc;
#pragma unroll
        for (int jq = 0; jq < JN / 2; ++jq) {
            const int col = n0 + b_col<JN>(wn, ln, jq * 4);
            if (p.c_vec && col + 3 < p.N) {
                *reinterpret_cast<float4 *>(crow + col) =
                    make_float4(acc[jq * 4 + 0], acc[jq * 4 + 1], acc[jq * 4 + 2], acc[jq * 4 + 3]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (col + e < p.N) crow[col + e] = acc[jq * 4 + e];
            }
        }
    }
}

// Stream-K for a ragged or under-filled last wave (the paper's "separate code
// for edge and corner cases", as a fractional split): tiles
// [0, (waves - 1) P) run whole, the last wave's rem tiles are dealt out as
// rem * k_blocks k-block iterations over P' = min(P, iterations / 12) workers,
// so it lasts rem / P' of a tile instead of a whole one.  Taken when its
// modelled length -- the fix-up costs the last piece of a tile the reads of
// the others' 128 KB partials and every other piece one write, ~2.6 us each
// at the ~50 GB/s one SM pulls from L2 (round-1 measurement) -- beats the
// split-K choice `splits` (with its fix-up kernel) by >= 3%.  Fixed by the shape and the planned SM
// count (never by opts.num_ctas).  LPY_FFMA_STREAMK=0 disables it, =2 takes it
// whenever it applies (A/B).
struct StreamK { int full_tiles, workers; long long iters; };
static StreamK choose_stream_k(int tiles, int k_blocks, int P, int splits, int bn) {
    static const int mode = [] {
        const char *e = getenv("LPY_FFMA_STREAMK");
        return e ? atoi(e) : 1;
    }();
    StreamK r{tiles, 0, 0};
    if (mode == 0 || tiles <= 0 || P <= 0 || k_blocks < 8) return r;
    const int waves = (tiles + P - 1) / P;
    const int rem = tiles - (waves - 1) * P;
    if (rem == P) return r;
    const long long iters = static_cast<long long>(rem) * k_blocks;
    long long workers = P;
    // >= 12 k-blocks per worker: shorter pieces lose to split-K -- config 5 at
    // BN = 128 (7.4 k-blocks per worker) ran 110 us stream-K'd vs 107 us split
    // (profiles/r02_ffma_schedule.txt); n = 2048 (47 per worker) 304 vs 312
    if (workers > iters / 12) workers = iters / 12;
    if (workers <= rem) return r;
    const double kb_us = bn == 256 ? 4.2 : 2.1;               // one k-block of one tile at full FMA rate
    const double tile_us = k_blocks * kb_us;
    const double pieces = double(rem) * k_blocks / double(workers) < k_blocks ? 2.0 : 1.0;
    const double fix = 2.6 * pieces / tile_us;                 // fix-up, in tiles
    const double t_sk = (waves - 1) + double(rem) / double(workers) + fix;
    const long long units = static_cast<long long>(tiles) * splits;
    double t_split = double((units + P - 1) / P) / double(splits);
    // the split-K alternative's own fix-up: none for a cluster split (a single
    // wave, DSMEM), else the fix-up kernel re-reading every slice's partial
    // (measured ~3 us + bytes at ~5 TB/s: 24 us at n = 2048 with 8 slices,
    // 11 us on the ragged config with 3; profiles/r02_ffma_streamk.txt)
    if (splits > 1 && units > P) t_split += (3.0 + double(units) * BM * bn * 4 / 5e6) / tile_us;
    if (mode != 2 && t_sk > 0.97 * t_split) return r;
    r.full_tiles = (waves - 1) * P;
    r.workers = int(workers);
    r.iters = iters;
    return r;
}

template <bool AK, bool BKM, int BN>
static cudaError_t launch_t(const Problem &p, const Knobs &kn, cudaStream_t s) {
    using G = Geo<AK, BKM, BN>;
    static_assert(G::STAGES >= 2, "stage ring does not fit");
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
    // k-blocks per slice at least: 1 -- a 128^3 product (one tile, 4 k-blocks)
    // then runs as 4 slices on 4 SMs: 13.8 -> 11.2 us, n=512 19.9 -> 17.1 us,
    // larger shapes unchanged (graph replay, profiles/r01_small_shapes.txt);
    // LPY_FFMA_MINKB overrides it for A/B runs.
    static const int min_kb = [] {
        const char *e = getenv("LPY_FFMA_MINKB");
        return e ? atoi(e) : 1;
    }();
    prm.splits = choose_splits(prm.num_tiles, prm.k_blocks, kn.num_sms, min_kb, MAX_SPLITS);
    static const int force_splits = [] {   // LPY_FFMA_SPLITS=S (A/B): split-K factor, 0 = choose_splits
        const char *e = getenv("LPY_FFMA_SPLITS");
        const int v = e ? atoi(e) : 0;
        return v >= 1 && v <= MAX_SPLITS ? v : 0;
    }();
    if (force_splits && force_splits <= prm.k_blocks) prm.splits = force_splits;   // (every slice non-empty)
    prm.num_units = prm.num_tiles * prm.splits;
    prm.ws = nullptr;
    prm.sem = nullptr;
    prm.full_tiles = prm.num_tiles;
    prm.sk_workers = prm.sk_stride = 0;
    prm.sk_iters = 0;
    {
        const StreamK sk = choose_stream_k(prm.num_tiles, prm.k_blocks, kn.num_sms, prm.splits, BN);
        if (sk.workers > 0) {
            prm.splits = 1;
            prm.full_tiles = sk.full_tiles;
            prm.sk_workers = sk.workers;
            prm.sk_stride = kn.num_sms;
            prm.sk_iters = sk.iters;
            prm.num_units = sk.full_tiles + 2 * kn.num_sms;
        }
    }
    static const int ws_stride = [] {
        const char *v = getenv("LPY_FFMA_PARTIAL");
        return (v && v[0] == 'c') ? 1 : CWARPS * 32;
    }();
    prm.ws_stride = ws_stride;
    prm.gate = kn.gate;
    int grid = kn.num_ctas > 0 ? kn.num_ctas : kn.num_sms;
    if (grid > prm.num_units) grid = prm.num_units;
    if (grid < 1) grid = 1;
    const bool split_kernel = prm.splits > 1 || prm.sk_workers > 0;
    auto kern = split_kernel ? gemm_ffma_kernel<AK, BKM, BN, true> : gemm_ffma_kernel<AK, BKM, BN, false>;
    static std::atomic<uint64_t> attr_done[2];
    e = ensure_smem_attr(kern, int(G::SMEM_BYTES), attr_done[split_kernel]);
    if (e != cudaSuccess) return e;
    // Cluster split: a single wave (one unit per CTA), S <= 8 (the portable
    // cluster size), as many tiles as clusters of S fit at once -> one cluster
    // per tile, slices summed
    // through DSMEM (no scratch, no fix-up launch).  LPY_FFMA_CLUSTER=0 keeps the
    // global-memory split (A/B).
    static const bool cluster_on = [] {
        const char *v = getenv("LPY_FFMA_CLUSTER");
        return !(v && v[0] == '0');
    }();
    auto cluster_cfg = [&](int S, cudaLaunchAttribute *attr) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(prm.num_tiles * S);
        cfg.blockDim = dim3(G::THREADS);
        cfg.dynamicSmemBytes = G::SMEM_BYTES;
        cfg.stream = s;
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = S;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cfg;
    };
    // co-resident clusters of S CTAs, once per (kernel variant, device, S)
    auto fits = [&](int S) {
        if (S < 2 || S > MAX_SPLITS || int64_t(prm.num_tiles) * S > kn.num_sms) return false;
        static std::atomic<int> fit_cache[64][MAX_SPLITS];
        static std::atomic<bool> fit_init{false};
        if (!fit_init.load()) {
            for (auto &d : fit_cache)
                for (auto &x : d) x.store(-1);
            fit_init.store(true);
        }
        int dev = 0;
        (void)cudaGetDevice(&dev);
        std::atomic<int> &slot = fit_cache[dev & 63][S - 1];
        int fit = slot.load();
        if (fit < 0) {
            cudaLaunchAttribute attr[1];
            const cudaLaunchConfig_t cfg = cluster_cfg(S, attr);
            if (cudaOccupancyMaxActiveClusters(&fit, kern, &cfg) != cudaSuccess) {
                (void)cudaGetLastError();
                fit = 0;
            }
            slot.store(fit);
        }
        return fit >= prm.num_tiles;
    };
    // The split factor, from the shape and the device only (results never depend
    // on opts.num_ctas): choose_splits' S, or S/2 when clusters of S do not fit at
    // once but clusters of S/2 do (n = 512: 16 tiles, S = 8 -> 4).
    bool cluster = prm.sk_workers == 0 && cluster_on && fits(prm.splits);
    if (cluster_on && !cluster && prm.splits >= 4 && fits(prm.splits / 2)) {
        prm.splits /= 2;
        prm.num_units = prm.num_tiles * prm.splits;
        grid = kn.num_ctas > 0 && kn.num_ctas < prm.num_units ? kn.num_ctas : prm.num_units;
        cluster = true;
    }
    prm.cluster_split = 0;
    if (cluster && (kn.num_ctas == 0 || kn.num_ctas >= prm.num_units)) {
        cudaLaunchAttribute attr[2];
        const cudaLaunchConfig_t cfg = cluster_cfg(prm.splits, attr);
        prm.cluster_split = 1;
        e = cudaLaunchKernelEx(&cfg, kern, ta, tb, prm);
        if (e == cudaSuccess) return cudaSuccess;
        (void)cudaGetLastError();   // not placed: the same split through global memory
        prm.cluster_split = 0;
    }
    if (prm.splits > 1) {
        // The split is fixed by the shape and the device's SM count (never by
        // opts.num_ctas), so results stay bitwise grid-invariant.  Scratch
        // (the partial tiles) is stream-ordered.
        const size_t ws_bytes = size_t(prm.num_units) * BM * BN * 4;
        e = cudaMallocAsync(reinterpret_cast<void **>(&prm.ws), ws_bytes, s);
        if (e != cudaSuccess) return e;
    } else if (prm.sk_workers > 0) {
        // stream-K: a partial slot per (piece, worker) and the per-tail-tile
        // ticket / written counters (zeroed here, left zero by the kernel)
        const int tail = prm.num_tiles - prm.full_tiles;
        const size_t ws_bytes = size_t(2) * prm.sk_stride * BM * BN * 4;
        char *buf = nullptr;
        e = cudaMallocAsync(reinterpret_cast<void **>(&buf), ws_bytes + size_t(tail) * 8, s);
        if (e != cudaSuccess) return e;
        prm.ws = reinterpret_cast<float *>(buf);
        prm.sem = reinterpret_cast<int *>(buf + ws_bytes);
        e = cudaMemsetAsync(prm.sem, 0, size_t(tail) * 8, s);
        if (e != cudaSuccess) { cudaFreeAsync(buf, s); return e; }
        if (grid > prm.sk_stride) grid = prm.sk_stride;
    }

    {
        cudaLaunchAttribute attr[1];
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(G::THREADS);
        cfg.dynamicSmemBytes = G::SMEM_BYTES;
        cfg.stream = s;
        // (no programmatic dependent launch on this path: measured 3% slower on
        // the ragged config with its split-K fix-up, no gain elsewhere)
        cfg.attrs = attr;
        cfg.numAttrs = 0;
        e = cudaLaunchKernelEx(&cfg, kern, ta, tb, prm);
    }
    if (e == cudaSuccess && prm.splits > 1) {
        cudaLaunchAttribute attr[1];
        cudaLaunchConfig_t cfg = {};
        static const int parts = [] {   // LPY_FFMA_FIXUP_PARTS (A/B); default FIXUP_PARTS
            const char *v = getenv("LPY_FFMA_FIXUP_PARTS");
            const int x = v ? atoi(v) : FIXUP_PARTS;
            return (x == 1 || x == 2 || x == 4 || x == 8) ? x : FIXUP_PARTS;
        }();
        cfg.gridDim = dim3(prm.num_tiles, parts);
        cfg.blockDim = dim3(CWARPS * 32);
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_attr(attr, 0);   // its launch overlaps the split grid's tail
        e = cudaLaunchKernelEx(&cfg, splitk_fixup_kernel<BN>, prm);
    }
    if (prm.ws) cudaFreeAsync(prm.ws, s);
    return e;
}

}  // namespace ffma

// Split-K factor for an under-filled grid (the paper's separate code for edge
// cases, read as "bulk tiles vs the ragged last wave"): the S in
// 1..max_splits whose (tile, slice) units fill `workers` persistent CTAs best,
// keeping at least `min_kb` k-blocks per slice; S = 1 unless it gains > 10%.
int choose_splits(int tiles, int k_blocks, int workers, int min_kb, int max_splits) {
    auto eff = [&](int s) {
        const int64_t units = int64_t(tiles) * s;
        const int64_t waves = (units + workers - 1) / workers;
        return double(units) / double(waves * workers);
    };
    int best = 1;
    double best_eff = eff(1);
    for (int s = 2; s <= max_splits && k_blocks / s >= min_kb; ++s)
        if (eff(s) > best_eff * 1.10 + 1e-9) { best = s; best_eff = eff(s); }
    return best;
}

cudaError_t launch_ffma(const Problem &p, const Knobs &kn, cudaStream_t s) {
    using namespace ffma;
    const bool AK = (p.la == 0);   // row-major A: K contiguous
    const bool BKM = (p.lb == 1);  // column-major B: K contiguous
    // Tile width: 128 x 256 tiles (8 x 16 per thread: 6 LDS.128 per 64 FFMA2)
    // run 2-5% faster per flop than 128 x 128 (8 x 8: 4 per 32) at n = 8192
    // (profiles/r01_ab_ffma_bn256.txt) but halve the tile count, so take 256
    // unless 128 fills the persistent grid's waves better by more than that.
    // (from the device's SM count, not opts.num_ctas: the split-K decision
    // follows the tile count, and results must not depend on the grid)
    const int grid = kn.num_sms;
    auto eff = [&](int bn, double kern) {
        const int64_t tiles = int64_t((p.M + BM - 1) / BM) * ((p.N + bn - 1) / bn);
        const int64_t waves = (tiles + grid - 1) / grid;
        return kern * double(tiles) / double(waves * grid) * double(p.N) / double(((p.N + bn - 1) / bn) * bn);
    };
    // The 4% per-flop edge of 256 shows only on long k loops: with K <= 2048 (<= 64
    // k-blocks per tile) 128-wide tiles -- half the partial bytes per split and
    // twice the units to balance -- measured 2-5% faster where the wave fill ties
    // (config 5 115 -> 110 us, n=2048 310 -> 304 us, 1536x2048x2048 240 -> 233 us;
    // 2048x2048x8192 and 1024x8192x8192 keep 256: profiles/r02_ffma_tile_width.txt).
    const double kern256 = p.K >= 4096 ? 1.04 : 0.98;
    if (kn.tile_n == 256 || (kn.tile_n == 0 && eff(256, kern256) >= eff(128, 1.0))) {
        if (AK && BKM)  return launch_t<true, true, 256>(p, kn, s);
        if (AK && !BKM) return launch_t<true, false, 256>(p, kn, s);
        if (!AK && BKM) return launch_t<false, true, 256>(p, kn, s);
        return launch_t<false, false, 256>(p, kn, s);
    }
    if (AK && BKM)  return launch_t<true, true, 128>(p, kn, s);
    if (AK && !BKM) return launch_t<true, false, 128>(p, kn, s);
    if (!AK && BKM) return launch_t<false, true, 128>(p, kn, s);
    return launch_t<false, false, 128>(p, kn, s);
}

}  // namespace lpy
