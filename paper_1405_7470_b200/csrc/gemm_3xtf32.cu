// 3xTF32 tensor-core path of C = A*B (the reduction sum(k, a[i,k]*b[k,j]),
// PAPER.md P:251-254) on the sm_100a 5th-generation tensor cores.
//
// Split precision (readings A9/A10).  The tensor core reads an fp32
// operand as tf32 by TRUNCATING its low 13 mantissa bits (measured:
// tests/test_numerics_tmem.py).  So each fp32 x is used as
//     big   = x                                  (the hardware sees trunc_tf32(x))
//     small = rna_tf32(x - trunc_tf32(x))        (computed here; exact residual, rounded)
// and  a*b ~= a_big*b_small + a_big*b_big + a_small*b_big  (small*small dropped;
// issued in that order so the two MMAs sharing A_big are adjacent).  Per
// product the representation error is below
// 2^-20 |a||b|.  TMEM accumulation rounds toward zero (measured), so the
// accumulator is PROMOTED: every `promote` k-blocks the MMA closes a TMEM partial
// (double-buffered, 2 x 256 columns) and the partial is added into fp32 registers
// with round-to-nearest (measured max normalised error at n=8192, uniform[0,1):
// 2.8e-6 with promote = 8, 5.3e-6 with 16; scripts/accuracy_tf32.py).
//
// Schedule (Loo.py's split_iname / group-local tags / add_prefetch / precompute,
// P:499-632, realised the Blackwell way).  CG = 1: one CTA per 128 x 256 output
// tile.  CG = 2 (default): a CTA pair (thread-block cluster of 2 on one TPC) per
// 256 x 256 tile with tcgen05.mma.cta_group::2 -- each CTA stages its own 128
// rows of A and its own 128 columns of B, the leader issues M=256 N=256 MMAs that
// read both CTAs' shared memory, and each CTA's TMEM receives its 128 rows.
// Warp roles (16 warps; registers rebalanced per warpgroup with setmaxnreg):
//   WG0  warp 0: TMA producer (A[128 x 16] + B[16 x 256/CG] fp32 per k-block,
//                "add_prefetch" into the stage ring); warp 1: tcgen05.mma issuer
//                (leader CTA; three kind::tf32 MMAs per k-slice of 8, commit to
//                free the stage / publish a partial); warps 2-3 idle.
//   WG1  warps 4-7: split transform of every stage (raw -> small in the same
//                swizzled layout, fence.proxy.async, arrive on the leader's
//                "ready" barrier) -- an elementwise "precompute".
//   WG2-3 warps 8-15: promotion + epilogue.  Each thread owns one TMEM lane (row)
//                x 128 columns as fp32 registers, folds in every finished partial,
//                and stores its row segment of C after a tile's last partial
//                (predicated 16-byte stores: ragged M/N; TMA zero-fill covers
//                ragged K).
// Operand smem layouts: K-major tiles use the 64B swizzle (16 fp32 per row);
// MN-major tf32 tiles must use SWIZZLE_128B_BASE32B (TMA "128B_ATOM_32B").
// Tile widths 128 / 176 / 192 / 256 (176 only for K-major A and B: config 5 fills 72 of
// 74 pairs).  Narrow tiles (BN <= 192) with a K-major A keep A_small in TENSOR memory: the
// transform warps write each row's 16 small values with tcgen05.st and the
// a_small * b_big MMA reads A from TMEM (TS form), so that tile never crosses
// the shared-memory port.
// Around the k loop: ragged last waves are stream-K'd (tail_split: the tail's
// k-iterations dealt over every planned pair, pieces summed in k order by the
// last to finish); a single under-filled wave is split inside a cluster and
// summed through DSMEM; and an optional K-gate (lpy_gemm_f32_gated) makes the
// producer wait for each chunk of K to be flagged as arrived before loading it
// -- the multi-GPU row-panel product consuming B while it is broadcast.
// Opt-in (LPY_TF32_MC=1, Params::mc): the two CTA pairs of a 4-CTA cluster take
// vertically adjacent tiles and multicast their shared B boxes (TMA
// .multicast::cluster), halving B's L2 -> SM traffic; off by default because
// clusters of 4 leave 16 of 148 SMs unplaced (profiles/r02_tf32_b_multicast.txt).
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include "lpy_internal.h"
#include "ptx.cuh"

namespace lpy {
namespace tf32 {

constexpr int MAX_SPLITS = 4;                // k-slices per split tile (cluster split)
constexpr int BM = 128, BK = 16;             // BM rows per CTA (the tile's BN columns: template, 128/192/256)
constexpr int THREADS = 512;                 // 16 warps = 4 warpgroups
constexpr int XFORM_WARP0 = 4, XFORM_WARPS = 4;
constexpr int EPI_WARP0 = 8, EPI_WARPS = 8;
constexpr int REGS_CTRL = 56, REGS_XFORM = 72, REGS_EPI = 192;   // 128*56 + 128*72 + 256*192 = 65536
constexpr uint32_t TMEM_COLS = 512;          // 2 partial buffers x 256 columns

template <int CG, int BN>
struct Cfg {
    static constexpr int BN_CTA = BN / CG;                       // B columns staged per CTA
    static constexpr int EC = BN / 2;                            // columns per promotion thread
    static constexpr uint32_t STAGE_BYTES_ = 2 * (BM * BK * 4 + BN_CTA * BK * 4);
    static constexpr int STAGES = CG == 2 ? int((227 * 1024 - 1024 - 256 - 64) / STAGE_BYTES_) : 4;
    static constexpr uint32_t A_BYTES = BM * BK * 4;             // 8 KB
    static constexpr uint32_t B_BYTES = BN_CTA * BK * 4;         // 16 KB / CG
    static constexpr uint32_t RAW_BYTES = A_BYTES + B_BYTES;     // TMA transaction per stage
    static constexpr uint32_t STAGE_BYTES = 2 * RAW_BYTES;       // raw + small
    static constexpr size_t SMEM_BYTES = 1024 + size_t(STAGES) * STAGE_BYTES + 256;
};

struct Params {
    int M, N, K;
    float *C;
    int64_t ldc;
    int tiles_m, tiles_n, num_tiles, k_blocks, group, promote;
    int c_vec;          // C rows 16-byte aligned (float4 stores)
    int c_vec8;         // C rows 32-byte aligned (STG.256)
    long long *trace;   // diagnostics build only (-DLPY_TRACE): per-CTA cycle counters
    // Work units.  Tiles [0, full_tiles) are one unit each.  The later tiles
    // (the ragged last wave) are cut along k in one of two ways:
    //  * stream-K (sk_workers > 0; >= 2 waves): the tail's sk_iters =
    //    (num_tiles - full_tiles) * k_blocks k-block iterations are dealt out
    //    evenly to sk_workers "workers" -- worker w takes iterations
    //    [floor(w*W/P'), floor((w+1)*W/P')) of the tail tiles in order -- so the
    //    last wave is (tail tiles / P') of a tile long for every CTA pair, a
    //    fractional split.  A worker's range is at most one tile
    //    long, so it covers at most two pieces (the end of one tile, the start
    //    of the next): unit full_tiles + piece * sk_stride + w, empty when
    //    w >= sk_workers or the range does not reach a second tile.  With the
    //    whole grid of sk_stride pairs, pair w runs worker w's pieces.
    //  * equal slices (splits > 1, sk_workers == 0): every tail tile is cut into
    //    `splits` k-slices, unit full_tiles + tail_tile * splits + slice (the
    //    cluster split's global-memory fallback for a capped grid).
    // A tile cut into several pieces has each piece park its partial in `ws`
    // (slot = the unit's index past full_tiles); the piece that finishes last
    // adds them in k order -- a fixed order, so results are deterministic and
    // independent of the grid.
    int full_tiles, splits, num_units;
    int sk_workers, sk_stride;
    long long sk_iters;
    // cluster split (a single under-filled wave): every tile is cut into
    // `splits` k-slices computed by the `splits` CTA pairs of one cluster, whose
    // partials are summed through distributed shared memory (no ws / sem)
    int cluster_split;
    // B multicast (CG = 2, row-major B, BN = 256): clusters of TWO CTA pairs.
    // Tile t (tiles_m counts pairs of 256-row tiles) is the 512 x BN block
    // whose pair q in {0, 1} computes 256-row tile 2 tm + q: both pairs need
    // the same B columns, so CTA (q, r) loads half of its pair-half's B boxes
    // and multicasts them to CTA (1 - q, r) -- every B byte crosses L2 -> SM
    // once per cluster instead of once per pair.  A stage is refilled only
    // after BOTH pairs' MMAs have released it (empty barriers count 2).
    int mc;
    float *ws;          // [(num_units - full_tiles)][CG (x2 with mc)][BM x BN] partial tiles
    int *sem;           // 2 x [(num_tiles - full_tiles)][CG] ticket / written counters, zero on entry and exit
    KGate gate;         // operands arriving in chunks of K (lpy_kgate): the producer waits per k-block
};

// Stream-K: the worker whose iteration range contains tail iteration x
// (b(w) = floor(w W / P') <= x < b(w+1)), and b(w) itself.
__device__ __forceinline__ int sk_worker_of(long long x, const Params &p) {
    return int(((x + 1) * p.sk_workers + p.sk_iters - 1) / p.sk_iters) - 1;
}
__device__ __forceinline__ long long sk_begin(int w, const Params &p) {
    return (static_cast<long long>(w) * p.sk_iters) / p.sk_workers;
}

// Work unit u -> tile t, k-block range [kb0, kb1) (empty when kb0 >= kb1), and
// for a piece of a tile cut into several its partial slot (-1 for a tile done
// by one unit).
__device__ __forceinline__ void unit_range(int u, const Params &p, int &t, int &kb0, int &kb1, int &su) {
    if (u < p.full_tiles) {
        t = u; kb0 = 0; kb1 = p.k_blocks; su = -1;
        return;
    }
    su = u - p.full_tiles;
    if (p.sk_workers > 0) {
        // (running the pieces FIRST, so that their fix-ups overlap later whole
        // tiles, measured slower: the fix-up then stalls its pair's next tile,
        // profiles/r02_streamk.txt)
        const int piece = su / p.sk_stride, w = su - piece * p.sk_stride;
        t = p.full_tiles; kb0 = kb1 = 0;
        if (w >= p.sk_workers) return;
        const long long b0 = sk_begin(w, p), b1 = sk_begin(w + 1, p), kb = p.k_blocks;
        const long long vt = b0 / kb + piece;                  // tail tile of this piece
        const long long lo = max(b0, vt * kb), hi = min(b1, (vt + 1) * kb);
        if (lo >= hi) return;
        t = p.full_tiles + int(vt);
        kb0 = int(lo - vt * kb);
        kb1 = int(hi - vt * kb);
        // a piece covering its whole tile is the tile's only unit
        if (kb0 == 0 && kb1 == p.k_blocks) su = -1;
        return;
    }
    const int v = su / p.splits, sl = su - v * p.splits;
    t = p.full_tiles + v;
    kb0 = int((int64_t(sl) * p.k_blocks) / p.splits);
    kb1 = int((int64_t(sl + 1) * p.k_blocks) / p.splits);
}

// The pieces of split tail tile vt in k order: count, and the partial slot of
// the i-th.
__device__ __forceinline__ int split_pieces(int vt, const Params &p) {
    if (p.sk_workers == 0) return p.splits;
    const long long kb = p.k_blocks;
    return sk_worker_of((vt + 1) * kb - 1, p) - sk_worker_of(vt * kb, p) + 1;
}
__device__ __forceinline__ int split_slot(int vt, int i, const Params &p) {
    if (p.sk_workers == 0) return vt * p.splits + i;
    const long long kb = p.k_blocks;
    const int w = sk_worker_of(vt * kb, p) + i;
    const int piece = int(sk_begin(w, p) / kb) == vt ? 0 : 1;
    return piece * p.sk_stride + w;
}

// Whether any unit after u (stride `units`) of this pair is non-empty.
__device__ __forceinline__ bool more_work_after(int u, int units, const Params &p) {
    for (int v = u + units; v < p.num_units; v += units) {
        int t, kb0, kb1, su;
        unit_range(v, p, t, kb0, kb1, su);
        if (kb0 < kb1) return true;
    }
    return false;
}

// Cycle accounting for the diagnostics build (liblpy_trace.so); compiled out of
// the product library.  Slots per CTA: 0 MMA total, 1 MMA wait(ready), 2 MMA
// wait(acce), 3 producer wait(empty), 4 transform wait(full), 5 epilogue
// wait(accf), 6 transform busy, 7 epilogue busy.
#ifdef LPY_TRACE
#define TR_T0(v) const long long v = clock64()
#define TR_ADD(slot, v) (tr[slot] += clock64() - (v))
// timeline of CTA 0: %globaltimer (ns) at event `slot`, after the counters
#define TL(slot)                                                                      \
    do {                                                                              \
        if (p.trace && blockIdx.x == 0) {                                             \
            unsigned long long g_;                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                    \
            p.trace[gridDim.x * 8 + (slot)] = (long long)g_;                          \
        }                                                                             \
    } while (0)
// every CTA's event times (12 slots: 0 entry, 1 exit, 2 fix-up start, 3 fix-up
// loads done, 4 MMA loop done, 5 last partial promoted, 6 first split unit's
// first MMA, 7 fix-up: other pieces written, 8 / 9 a writer's ticket / partial
// written), after the timeline
#define TLC(which)                                                                    \
    do {                                                                              \
        if (p.trace) {                                                                \
            unsigned long long g_;                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                    \
            p.trace[gridDim.x * 8 + 16 + 12 * blockIdx.x + (which)] = (long long)g_;   \
        }                                                                             \
    } while (0)
#else
#define TR_T0(v) (void)0
#define TR_ADD(slot, v) (void)0
#define TL(slot) (void)0
#define TLC(which) (void)0
#endif

__device__ __forceinline__ void tile_coords(int t, const Params &p, int &tm, int &tn) {
    const int per_group = p.group * p.tiles_n;
    const int g = t / per_group;
    const int first = g * p.group;
    const int gsize = min(p.group, p.tiles_m - first);
    const int r = t - g * per_group;
    tm = first + r % gsize;
    tn = r / gsize;
}

// UMMA descriptor of k-slice `sub` (0/1, 8 elements each) of an operand tile.
// K-major (64B swizzle): rows of 64 B, 8-row groups at 512 B; the slice starts
// 32 B into the row.  MN-major (128B_BASE32B): 32-wide MN blocks of 16 k-rows
// x 128 B (2 KB, LBO), 4-row groups at 512 B (SBO); the slice starts 8 rows in.
template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t tile, int sub) {
    if constexpr (MN) return umma_sdesc(tile + sub * 1024, 2048, 512, 1);
    else              return umma_sdesc(tile + sub * 32, 16, 512, 4);
}

// small = rna_tf32(x - trunc_tf32(x)).  The residual is exact in fp32 and finite
// for finite x, so round-to-nearest-away on its bit pattern is an integer add of
// half a tf32 ulp followed by truncation (what cvt.rna.tf32.f32 does, minus its
// NaN/Inf guard).
__device__ __forceinline__ float tf32_small(float x) {
    const float big = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);   // what the MMA sees
    const uint32_t r = __float_as_uint(x - big);
    return __uint_as_float((r + 0x1000u) & 0xFFFFE000u);
}

// C[row, col .. col+7] = v (a row pointer `crow`), clipped at N: one STG.256
// when C's rows are 32-byte aligned, else two float4 stores, else scalars.
__device__ __forceinline__ void store_row8(const Params &p, float *crow, int col, const float *v) {
    if (p.c_vec8 && col + 7 < p.N) {
        st_v8(crow + col, v);
    } else if (p.c_vec && col + 7 < p.N) {
        *reinterpret_cast<float4 *>(crow + col) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4 *>(crow + col + 4) = make_float4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (col + e < p.N) crow[col + e] = v[e];
    }
}

// Arrive (one per warp) on the leader CTA's copy of `bar`.
template <int CG>
__device__ __forceinline__ void arrive_leader(uint64_t *bar, uint32_t lead) {
    if constexpr (CG == 1) mbar_arrive(bar);
    else                   mbar_arrive_remote(mapa_shared(smem_u32(bar), lead));
}

template <int CG, bool AMN, bool BMN, int BN>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const Params p) {
    using C_ = Cfg<CG, BN>;
    constexpr int EC = C_::EC;
    constexpr int STAGES = C_::STAGES;
    static_assert(size_t(BM) * (BN + 4) * 4 <= size_t(STAGES) * C_::STAGE_BYTES,
                  "cluster-split staging must fit in the operand ring");
    // A_small in TENSOR memory (narrow tiles, K-major A): the transform warps
    // write each row's 16 small values straight into TMEM (lane = row) and the
    // a_small * b_big MMA reads A from there ("TS" form) -- the A_small tile
    // then never crosses the shared-memory port (neither the transform's write
    // nor the MMA's read), which bounds the narrow tiles.  TMEM:
    // the two partial accumulators at columns [0, BN) and [BN, 2 BN), A_small of
    // stage s at 2 BN + 16 s.
#ifdef LPY_TF32_NO_TMEMA
    constexpr bool TA = false;       // (A/B build: A_small through shared memory everywhere)
#else
    constexpr bool TA = CG == 2 && !AMN && BN <= 192;
#endif
    static_assert(!TA || 2 * BN + 16 * STAGES <= int(TMEM_COLS), "A_small stages must fit in TMEM");
    constexpr uint32_t acc_stride = TA ? uint32_t(BN) : 256u;
    constexpr uint32_t A_BYTES = C_::A_BYTES, RAW_BYTES = C_::RAW_BYTES, STAGE_BYTES = C_::STAGE_BYTES;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t *stages = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
    uint64_t *bars = reinterpret_cast<uint64_t *>(stages + STAGES * STAGE_BYTES);
    uint64_t *full = bars;                  // TMA -> transform (per CTA)
    uint64_t *ready = bars + STAGES;        // transforms of the pair -> MMA (leader)
    uint64_t *empty = bars + 2 * STAGES;    // MMA commit -> producer (per CTA)
    uint64_t *accf = bars + 3 * STAGES;     // MMA commit -> promotion (per CTA)
    uint64_t *acce = accf + 2;              // promotions of the pair -> MMA (leader)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acce + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // rank: which CTA of the pair (0 = the MMA-issuing leader); lead: the
    // leader's rank in the cluster (pairs are ranks (2q, 2q+1); a cluster
    // holds one pair, or `splits` pairs in a cluster split)
    const uint32_t crank = CG == 2 ? cluster_ctarank() : 0;
    const int rank = int(crank & 1);
    const uint32_t lead = crank & ~1u;
    const uint16_t pair_mask = uint16_t(3u << lead);
    // B multicast: pair mq of a 4-CTA cluster; a unit is the cluster's
    // 512-row block, whose pair mq computes 256-row tile 2 tm + mq (Params::mc)
    const bool mc = CG == 2 && p.mc;
    const int mq = mc ? int(crank >> 1) : 0;
    const int cl = mc ? 2 * CG : CG;                              // CTAs per unit
    const int unit0 = blockIdx.x / cl, units = gridDim.x / cl;   // this pair's first tile, stride
    // the operand stages a commit frees: this pair's, or both pairs' (a
    // multicast writes B into the other pair's stage too)
    const uint16_t empty_mask = mc ? uint16_t(0xF) : pair_mask;
    // partial slots of split tiles: one per CTA of the unit
    const int sub_id = mq * CG + rank, subs = cl;

    if (threadIdx.x == 0) {
        TL(0);
        TLC(0);
        // descriptor fetch overlaps the barrier / TMEM setup (kernel parameters:
        // not written by the previous grid, so no need to wait for it)
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], CG * XFORM_WARPS);
            mbar_init(&empty[s], mc ? 2 : 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accf[b], 1);
            mbar_init(&acce[b], CG * EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        tmem_alloc_cg<CG>(tmem_slot, TMEM_COLS);
        tmem_relinquish_cg<CG>();
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();                 // the previous grid's writes (A, B; readers of C) are done
    if (threadIdx.x == 0) TL(1);
#ifdef LPY_TRACE
    long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif

    if (warp < XFORM_WARP0) {
        setmaxnreg_dec<REGS_CTRL>();
        if (warp == 0) {
            // ------------------------------------------------ TMA producer
            if (lane == 0) {
                int s = 0;
                uint32_t ph = 0;
                int gready = -1;                           // K-gate: chunks known ready
                int glimit = kgate_limit0(p.gate);         // ... and the first k-block they do not cover
                for (int u = unit0; u < p.num_units; u += units) {
                    int t, kb0, kb1, su, tm, tn;
                    unit_range(u, p, t, kb0, kb1, su);
                    tile_coords(t, p, tm, tn);
                    const int m0 = (mc ? 2 * tm + mq : tm) * (BM * CG) + rank * BM;
                    const int n0 = tn * BN + rank * C_::BN_CTA;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        // (before the stage wait: off the critical path when the ring is full)
                        if (kb >= glimit) glimit = kgate_admit(p.gate, gready, kb, BK, p.K);
                        TR_T0(t_w);
                        mbar_wait(&empty[s], ph ^ 1);
                        TR_ADD(3, t_w);
                        uint8_t *sa = stages + s * STAGE_BYTES;
                        uint8_t *sb = sa + A_BYTES;
                        mbar_arrive_expect_tx(&full[s], RAW_BYTES);
                        const int k0 = kb * BK;
                        if constexpr (AMN) {
#pragma unroll
                            for (int j = 0; j < BM / 32; ++j)
                                tma_load_2d(sa + j * 2048, &tmA, &full[s], m0 + 32 * j, k0);
                        } else {
                            tma_load_2d(sa, &tmA, &full[s], k0, m0);
                        }
                        if constexpr (BMN) {
                            if (mc) {
                                // this CTA's share of the boxes, to itself and its rank-mate in the other pair
                                constexpr int PER = C_::BN_CTA / 64;
                                const uint16_t to = uint16_t((1u << rank) | (1u << (2 + rank)));
#pragma unroll
                                for (int j = 0; j < PER; ++j)
                                    tma_load_2d_mc(sb + (mq * PER + j) * 2048, &tmB, &full[s],
                                                   n0 + 32 * (mq * PER + j), k0, to);
                            } else {
#pragma unroll
                                for (int j = 0; j < C_::BN_CTA / 32; ++j)
                                    tma_load_2d(sb + j * 2048, &tmB, &full[s], n0 + 32 * j, k0);
                            }
                        } else {
                            tma_load_2d(sb, &tmB, &full[s], k0, n0);
                        }
                        if (kb == kb0 && u == unit0) TL(2);
                        if (++s == STAGES) { s = 0; ph ^= 1; }
                    }
                }
            }
        } else if (warp == 1 && rank == 0) {
            // ------------------------------------------------ MMA issuer (leader CTA)
            // The whole warp runs the loop (converged, so descriptors stay in
            // uniform registers) and one elected lane issues: an issue path that
            // rebuilt descriptors per MMA through R2UR waterfalls could not keep
            // up with 128-cycle MMAs.
            constexpr uint32_t idesc = umma_idesc_tf32(BM * CG, BN, AMN ? 1 : 0, BMN ? 1 : 0);
            // stage s adds s * STAGE_BYTES >> 4 to the descriptors' start-address field
            const uint32_t sa0 = smem_u32(stages), sb0 = sa0 + A_BYTES;
            const uint64_t dab[2] = {op_desc<AMN>(sa0, 0), op_desc<AMN>(sa0, 1)};
            const uint64_t dbb[2] = {op_desc<BMN>(sb0, 0), op_desc<BMN>(sb0, 1)};
            constexpr uint64_t SMALL = RAW_BYTES >> 4, STEP = STAGE_BYTES >> 4;
            int s = 0;
            uint32_t ph = 0;
            uint32_t npart = 0;   // partials issued by this pair
            TR_T0(t_all);
            for (int u = unit0; u < p.num_units; u += units) {
                int t, kb0, kb1, su;
                unit_range(u, p, t, kb0, kb1, su);
                for (int kb = kb0; kb < kb1; ++kb) {
                    const bool first = ((kb - kb0) % p.promote) == 0;
                    const bool last = ((kb - kb0) % p.promote) == p.promote - 1 || kb == kb1 - 1;
                    const uint32_t b = npart & 1;
                    if (first) {
                        TR_T0(t_e);
                        mbar_wait(&acce[b], ((npart >> 1) & 1) ^ 1);   // buffer drained (both CTAs)
                        TR_ADD(2, t_e);
                        tc_fence_after();
                    }
                    TR_T0(t_r);
                    mbar_wait(&ready[s], ph);
                    TR_ADD(1, t_r);
                    if (kb == kb0 && u == unit0 && lane == 0) TL(4);
                    if (kb == kb0 && su >= 0 && lane == 0 && su < p.sk_stride) TLC(6);
                    tc_fence_after();
                    const uint32_t d = tmem + b * acc_stride;
                    const uint64_t off = uint64_t(s) * STEP;
                    const uint32_t a_tm = tmem + uint32_t(2 * BN + 16 * s);   // A_small of stage s (TA)
                    if (elect_one()) {
#pragma unroll
                        for (int sub = 0; sub < BK / 8; ++sub) {
                            const uint64_t a_big = dab[sub] + off, b_big = dbb[sub] + off;
                            // a_big * b_small, a_big * b_big, a_small * b_big: the two MMAs
                            // sharing A back to back measured 1-3% faster than small terms first
                            // (accuracy unchanged: every partial is promoted within 128 of K)
                            // A_big through the tensor core's collector: read from shared
                            // memory once for both of its MMAs (fill / lastuse), which
                            // eases the shared-memory port that bounds the narrow tiles
                            // (n=1024, BN=128: 27.8 -> 26.9 us; no change at n=8192;
                            // profiles/r01_tf32_collector.txt)
                            if constexpr (CG == 2) {
                                umma_tf32_cg2_coll<ACollector::Fill>(d, a_big, b_big + SMALL, idesc,
                                                                     (first && sub == 0) ? 0u : 1u);
                                umma_tf32_cg2_coll<ACollector::LastUse>(d, a_big, b_big, idesc, 1u);
                            } else {
                                umma_tf32_cg<CG>(d, a_big, b_big + SMALL, idesc, (first && sub == 0) ? 0u : 1u);
                                umma_tf32_cg<CG>(d, a_big, b_big, idesc, 1u);
                            }
                            if constexpr (TA) {
                                umma_tf32_ts_cg2(d, a_tm + 8 * sub, b_big, idesc, 1u);
                            } else {
                                umma_tf32_cg<CG>(d, a_big + SMALL, b_big, idesc, 1u);
                            }
                        }
                        umma_commit_cg<CG>(&empty[s], empty_mask);
                        if (last) umma_commit_cg<CG>(&accf[b], pair_mask);
                        TL(5);
                    }
                    __syncwarp();
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                    if (last) ++npart;
                }
            }
            TR_ADD(0, t_all);
            if (lane == 0) TLC(4);
        }
    } else if (warp < EPI_WARP0) {
        // ------------------------------------------------ split transform (WG1)
        setmaxnreg_dec<REGS_XFORM>();
        const int xt = threadIdx.x - XFORM_WARP0 * 32;   // 0..127
        constexpr int PER_THREAD = int(RAW_BYTES / 16) / (XFORM_WARPS * 32);
        int s = 0;
        uint32_t ph = 0;
        for (int u = unit0; u < p.num_units; u += units) {
            int t, kb0, kb1, su;
            unit_range(u, p, t, kb0, kb1, su);
            for (int kb = kb0; kb < kb1; ++kb) {
                TR_T0(t_f);
                mbar_wait(&full[s], ph);
                TR_ADD(4, t_f);
                if (kb == kb0 && u == unit0 && xt == 0) TL(3);
                TR_T0(t_x);
#ifdef LPY_MUTATE_STAGE_RACE
                // MUTATION (liblpy_mutant.so, tests/test_mutation_gpu.py only): the
                // stage is declared ready BEFORE its small parts are written, so the
                // MMA may read stale ones -- the race the detector tests must catch
                if (lane == 0) arrive_leader<CG>(&ready[s], lead);
#endif
                const float4 *src = reinterpret_cast<const float4 *>(stages + s * STAGE_BYTES);
                float4 *dst = reinterpret_cast<float4 *>(stages + s * STAGE_BYTES + RAW_BYTES);
                if constexpr (TA) {
                    // A: thread xt owns row xt (TMEM lane xt: warp 4 + q holds lanes
                    // 32q..32q+31).  The raw K-major tile is 128 rows x 64 B under
                    // the 64B swizzle: 16-byte chunk c of row r sits at c ^ ((r >> 1) & 3).
                    uint32_t v[16];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float4 q = src[xt * 4 + (c ^ ((xt >> 1) & 3))];
                        v[4 * c + 0] = __float_as_uint(tf32_small(q.x));
                        v[4 * c + 1] = __float_as_uint(tf32_small(q.y));
                        v[4 * c + 2] = __float_as_uint(tf32_small(q.z));
                        v[4 * c + 3] = __float_as_uint(tf32_small(q.w));
                    }
                    tmem_st_x16(tmem + (uint32_t((xt >> 5) * 32) << 16) + uint32_t(2 * BN + 16 * s), v);
                    // B: as below, over the B part of the stage only
                    constexpr int A4 = int(A_BYTES / 16), B_PER = int(C_::B_BYTES / 16) / (XFORM_WARPS * 32);
                    constexpr int B_REM = int(C_::B_BYTES / 16) % (XFORM_WARPS * 32);   // (BN = 176: 96)
#pragma unroll 4
                    for (int i = 0; i < B_PER + (B_REM ? 1 : 0); ++i) {
                        if (B_REM && i == B_PER && xt >= B_REM) break;
                        float4 w = src[A4 + xt + i * XFORM_WARPS * 32];
                        w.x = tf32_small(w.x);
                        w.y = tf32_small(w.y);
                        w.z = tf32_small(w.z);
                        w.w = tf32_small(w.w);
                        dst[A4 + xt + i * XFORM_WARPS * 32] = w;
                    }
                    tmem_st_wait();
                    tc_fence_before();
                } else {
#pragma unroll 4
                    for (int i = 0; i < PER_THREAD; ++i) {
                        float4 v = src[xt + i * XFORM_WARPS * 32];
                        v.x = tf32_small(v.x);
                        v.y = tf32_small(v.y);
                        v.z = tf32_small(v.z);
                        v.w = tf32_small(v.w);
                        dst[xt + i * XFORM_WARPS * 32] = v;
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
#ifndef LPY_MUTATE_STAGE_RACE
                if (lane == 0) arrive_leader<CG>(&ready[s], lead);
#endif
                if (++s == STAGES) { s = 0; ph ^= 1; }
                TR_ADD(6, t_x);
            }
        }
    } else {
        // ------------------------------------------------ promotion + epilogue (WG2, WG3)
        setmaxnreg_inc<REGS_EPI>();
        const int quad = warp & 3;                       // TMEM lanes 32*quad .. +31 (hardware rule)
        const int half = (warp - EPI_WARP0) >> 2;        // columns 128*half .. +127
        const uint32_t lane_base = uint32_t(quad * 32) << 16;
        const int ept = threadIdx.x - EPI_WARP0 * 32;   // 0..255
        __shared__ int last_flag;
        uint32_t np = 0;                                 // partials promoted so far
        for (int u = unit0; u < p.num_units; u += units) {
            int t, kb0, kb1, su;
            unit_range(u, p, t, kb0, kb1, su);
            if (kb0 >= kb1) continue;
            const int parts_per_tile = (kb1 - kb0 + p.promote - 1) / p.promote;
            float acc[EC];
#pragma unroll
            for (int j = 0; j < EC; ++j) acc[j] = 0.f;
            for (int part = 0; part < parts_per_tile; ++part, ++np) {
                const uint32_t b = np & 1;
                TR_T0(t_w);
                mbar_wait(&accf[b], (np >> 1) & 1);
                TR_ADD(5, t_w);
                if (np == 0 && ept == 0) TL(6);
                TR_T0(t_b);
                tc_fence_after();
                const uint32_t base = tmem + lane_base + b * acc_stride + half * EC;
#pragma unroll
                for (int c = 0; c + 32 <= EC; c += 32) {
                    uint32_t v0[16], v1[16];
                    tmem_ld_x16(base + c, v0);
                    tmem_ld_x16(base + c + 16, v1);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        acc[c + j] += __uint_as_float(v0[j]);
                        acc[c + 16 + j] += __uint_as_float(v1[j]);
                    }
                }
                if constexpr (EC % 32 >= 16) {            // (BN = 176: columns 64..79 of 88)
                    constexpr int c = EC / 32 * 32;
                    uint32_t v0[16];
                    tmem_ld_x16(base + c, v0);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc[c + j] += __uint_as_float(v0[j]);
                }
                if constexpr (EC % 16 == 8) {             // (BN = 176: columns 80..87)
                    constexpr int c = EC - 8;
                    uint32_t v0[8];
                    tmem_ld_x8(base + c, v0);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[c + j] += __uint_as_float(v0[j]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_leader<CG>(&acce[b], lead);
                TR_ADD(7, t_b);
            }
            // one row per thread (TMEM lane = row), written with 32-byte stores so
            // each instruction writes whole sectors of 32 rows
            // (computed where used: live across the partial's write they cost
            // the BN = 256 variants register spills)
            if (ept == 0) { TL(9); TLC(5); }
            auto row_of = [&]() {
                int tm, tn;
                tile_coords(t, p, tm, tn);
                return (mc ? 2 * tm + mq : tm) * (BM * CG) + rank * BM + quad * 32 + lane;
            };
            auto col0_of = [&]() {
                int tm, tn;
                tile_coords(t, p, tm, tn);
                return tn * BN + half * EC;
            };
            if (p.cluster_split) {
                // cluster split: park this slice's partial in this CTA's own shared
                // memory (the operand ring is idle: the accf commit covers every MMA
                // of the pair, so nothing reads it any more); rows padded by 4
                // floats so a warp's float4 stores (32 rows) hit distinct banks.
                // Summed across the cluster's slices after the cluster barrier.
                float *dst = reinterpret_cast<float *>(stages) + (quad * 32 + lane) * (BN + 4) + half * EC;
#pragma unroll
                for (int j = 0; j < EC; j += 4)
                    *reinterpret_cast<float4 *>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
                continue;
            }
            if (su >= 0) {
                // A tile cut into pieces.  Each piece takes a ticket per (tile,
                // CTA); all but the last park their partial as thread-
                // interleaved 32-byte vectors (a warp writes and later reads
                // 1 KB contiguous) and count themselves written.  The last
                // waits for those writes -- the writers already hold tickets,
                // so they are running and the wait is bounded (no spin on a
                // CTA that may not be resident) -- and sums the pieces in k
                // order with its own partial taken from registers: it neither
                // writes nor re-reads it, and reads the others with 32-byte
                // loads.  The order of the additions is fixed
                // by the decomposition, never by who finishes last.
                constexpr int TILE8 = BM * BN / 8;
                const int vt = t - p.full_tiles;
                const int npieces = split_pieces(vt, p);
                const int me = p.sk_workers > 0
                                   ? su % p.sk_stride - sk_worker_of(static_cast<long long>(vt) * p.k_blocks, p)
                                   : su - vt * p.splits;
                int *arrive = p.sem + vt * subs + sub_id;
                int *written = p.sem + (p.num_tiles - p.full_tiles + vt) * subs + sub_id;
                if (ept == 0) last_flag = atomicAdd(arrive, 1) == npieces - 1;
                named_bar_sync(1, EPI_WARPS * 32);
                if (!last_flag) {
                    if (ept == 0) TLC(8);
                    float *mine = p.ws + ((int64_t(su) * subs + sub_id) * TILE8 + ept) * 8;
#pragma unroll
                    for (int j = 0; j < EC; j += 8) st_cg_v8(mine + (j / 8) * 256 * 8, &acc[j]);
                    if (ept == 0) TL(10);
                    __threadfence();
                    named_bar_sync(1, EPI_WARPS * 32);
                    if (ept == 0) { atomicAdd(written, 1); TLC(9); }
                    continue;
                }
                if (ept == 0) {
                    TLC(2);
                    while (ld_acquire_gpu(written) < npieces - 1) __nanosleep(64);
                    TLC(7);
                    *arrive = 0;      // ready for the next launch (nobody else touches them now)
                    *written = 0;
                }
                named_bar_sync(1, EPI_WARPS * 32);
                __threadfence();
                // Sum in k order, ((p0 + p1) + p2) + ...  With the own piece
                // first or second, acc (= p_me) is the running sum from the
                // start (p1 + p0 == p0 + p1 bitwise: addition commutes).  A
                // later own piece (rare: the last to finish is usually the
                // tile's first or second piece) is written out and the sum
                // rebuilt from memory in order.
                auto slot_ptr = [&](int i) {
                    return p.ws + ((int64_t(split_slot(vt, i, p)) * subs + sub_id) * TILE8 + ept) * 8;
                };
                int i0 = 0;
                if (me >= 2) {
                    float *mine = slot_ptr(me);
#pragma unroll
                    for (int j = 0; j < EC; j += 8) st_cg_v8(mine + (j / 8) * 256 * 8, &acc[j]);
                    const float *src = slot_ptr(0);
#pragma unroll
                    for (int j = 0; j < EC; j += 8) ld_cg_v8(src + (j / 8) * 256 * 8, &acc[j]);
                    i0 = 1;
                }
#pragma unroll 1
                for (int i = i0; i < npieces; ++i) {
                    if (i == me && me < 2) continue;
                    // (the own piece re-read when me >= 2 was written by this
                    // thread: the volatile load keeps it after that store)
                    const float *src = slot_ptr(i) + opaque_zero();
                    const bool own = i == me;
#pragma unroll
                    for (int j = 0; j < EC; j += 8) {
                        float v[8];
                        if (own) ld_cg_v8(src + (j / 8) * 256 * 8, v);
                        else     ld_cg_v8_nv(src + (j / 8) * 256 * 8, v);
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc[j + e] += v[e];
                    }
                }
                if (ept == 0) { TL(12); TLC(3); }
            }
            if (!more_work_after(u, units, p)) {
                // This CTA's last tile: the operand ring is idle (the final accf
                // commit covers every MMA of the pair), so the tile goes through
                // it and leaves row-contiguous -- a warp stores 512 consecutive
                // bytes per instruction instead of 32 bytes of 32 rows, which
                // halves the exposed epilogue of small products.
                float *dst = reinterpret_cast<float *>(stages) + (quad * 32 + lane) * (BN + 4) + half * EC;
#pragma unroll
                for (int j = 0; j < EC; j += 4)
                    *reinterpret_cast<float4 *>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
                named_bar_sync(1, EPI_WARPS * 32);
                int tm, tn;
                tile_coords(t, p, tm, tn);
                const int row0 = (mc ? 2 * tm + mq : tm) * (BM * CG) + rank * BM, colt = tn * BN;
                constexpr int C4 = BN / 4;
                const float *stg = reinterpret_cast<const float *>(stages);
#pragma unroll 4
                for (int idx = ept; idx < BM * C4; idx += EPI_WARPS * 32) {
                    const int rl = idx / C4, c4 = idx % C4;
                    const float4 v = *reinterpret_cast<const float4 *>(stg + rl * (BN + 4) + c4 * 4);
                    const int row = row0 + rl, col = colt + c4 * 4;
                    if (row < p.M) {
                        float *c = p.C + int64_t(row) * p.ldc + col;
                        if (p.c_vec && col + 3 < p.N) {
                            *reinterpret_cast<float4 *>(c) = v;
                        } else {
                            const float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (col + e < p.N) c[e] = o[e];
                        }
                    }
                }
                continue;
            }
            const int row = row_of(), col0 = col0_of();
            float *crow = p.C + int64_t(row) * p.ldc;
            if (row < p.M) {
#pragma unroll
                for (int j = 0; j < EC; j += 8) store_row8(p, crow, col0 + j, &acc[j]);
            }
        }
    }
#ifdef LPY_TRACE
    if (p.trace && lane == 0 && (warp <= 1 || warp == XFORM_WARP0 || warp == EPI_WARP0))
        for (int i = 0; i < 8; ++i)
            if (tr[i]) atomicAdd(reinterpret_cast<unsigned long long *>(&p.trace[blockIdx.x * 8 + i]),
                                 (unsigned long long)tr[i]);
#endif

    if (threadIdx.x == EPI_WARP0 * 32) TL(7);
    // The next grid in the stream may launch once every CTA is here (its
    // prologue then overlaps this grid's reduction / teardown; triggered at the
    // start instead, its waiting CTAs slowed this grid by up to 8%).
    pdl_launch_dependents();
    if constexpr (CG == 2) {
        if (p.cluster_split) {
            // every slice's partial parked (all threads of the cluster arrive)
            cluster_sync();
            if (warp >= EPI_WARP0) {
                // This CTA sums rows [q*RPS, (q+1)*RPS) of its half of the tile
                // (q = its pair's slice) over the cluster's slices in slice order,
                // reading each slice's partial from the same half's CTA through
                // distributed shared memory, and stores them to C coalesced
                // (consecutive threads take consecutive float4s of a row).
                const int ks = p.splits;
                const int q = unit0 % ks, t = unit0 / ks;
                int tm, tn;
                tile_coords(t, p, tm, tn);
                const int rps = BM / ks;
                const int row0 = tm * (BM * CG) + rank * BM;
                const int col0 = tn * BN;
                const uint32_t stg = smem_u32(stages);
                constexpr int C4 = BN / 4;
                const int items = rps * C4;
#pragma unroll 4
                for (int idx = threadIdx.x - EPI_WARP0 * 32; idx < items; idx += EPI_WARPS * 32) {
                    const int rl = q * rps + idx / C4, c4 = idx % C4;
                    const uint32_t off = stg + uint32_t((rl * (BN + 4) + c4 * 4) * 4);
                    float4 v[MAX_SPLITS];
#pragma unroll
                    for (int sl = 0; sl < MAX_SPLITS; ++sl)
                        if (sl < ks) v[sl] = ld_dsmem_v4(mapa_shared(off, uint32_t(2 * sl + rank)));
#pragma unroll
                    for (int sl = 1; sl < MAX_SPLITS; ++sl)
                        if (sl < ks) { v[0].x += v[sl].x; v[0].y += v[sl].y; v[0].z += v[sl].z; v[0].w += v[sl].w; }
                    const int row = row0 + rl, col = col0 + c4 * 4;
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
            }
        }
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    if (warp == 1) tmem_dealloc_cg<CG>(tmem, TMEM_COLS);
    if (threadIdx.x == 32) { TL(8); TLC(1); }
}

template <int CG, bool AMN, bool BMN, int BN>
static cudaError_t launch_t(const CUtensorMap &ta, const CUtensorMap &tb, const Params &prm, int grid,
                            cudaStream_t s) {
    using C_ = Cfg<CG, BN>;
    static_assert(C_::EC % 8 == 0 && C_::SMEM_BYTES <= 227 * 1024, "tile does not fit");
    // 32-column MN-major B boxes, whole float4 shares of the transform outside the TMEM-A path
    static_assert(BN % 64 == 0 || (!AMN && !BMN), "BN = 176 needs K-major A and B");
    auto kern = gemm_3xtf32_kernel<CG, AMN, BMN, BN>;
    static std::atomic<uint64_t> attr_done{0};
    if (cudaError_t e = ensure_smem_attr(kern, int(C_::SMEM_BYTES), attr_done); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = C_::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG * (prm.cluster_split ? prm.splits : prm.mc ? 2 : 1);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_attr(attr, 1);
    return cudaLaunchKernelEx(&cfg, kern, ta, tb, prm);
}

static long long *g_trace = nullptr;   // set by lpy_trace_set_buffer (diagnostics build)

// Split of the last wave along k, fixed by the shape and the device (never by
// opts.num_ctas, so results stay bitwise grid-invariant):
//  * >= 2 waves with a partial last one: stream-K over the last wave's `rem`
//    tiles.  Their rem * k_blocks iterations are dealt out evenly to
//    P' = min(pairs, 4 rem, rem k_blocks / 16) workers (<= 4 pieces per tile
//    + 1, >= 16 k-blocks per worker), so the last wave takes rem / P' of a
//    tile instead of a whole one -- a fractional split (the paper's "separate
//    code for edge and corner cases").  Used when it shortens the
//    last wave by >= 10% and K >= 4096.  (Round 1 cut the tail tiles into S = floor(pairs /
//    rem) equal slices: at 128 tiles on 74 pairs, S = 1, no gain.)
//  * a single under-filled wave (tiles < pairs, e.g. n = 1024): every tile is
//    cut into S = 2 or 4 k-slices (S * tiles <= pairs, >= 8 k-blocks each)
//    computed by the S CTA pairs of one cluster (2S CTAs), which sum their
//    partials through distributed shared memory, each CTA reducing and
//    storing 1/S of its rows (`cluster_split`).  The global-memory variant of
//    this split (last arriver re-reads S partials of 128 KB through one SM at
//    ~50 GB/s) was slower than no split (profiles/r01_tf32_split1.txt); the
//    cluster's barrier is safe where a global spin-wait is not, since the
//    hardware co-schedules a cluster's CTAs.  LPY_TF32_SPLIT1=0 disables it.
//    S = 4 needs clusters of 8 CTAs, of which only `caps.max8` fit on the chip
//    at once (a cluster lives in one GPC), so S follows what fits in one wave.
// LPY_TF32_STREAMK=0 disables the stream-K tail (diagnostics / A-B).
struct ClusterCaps { int max4, max8; };   // co-resident clusters of 4 / 8 CTAs
struct TailSplit {
    int splits, full_tiles, num_units, cluster;
    int sk_workers, sk_stride;
    long long sk_iters;
    double waves;          // modelled length of the schedule in whole-tile waves
};
constexpr int SK_MAX_PIECES = 4;        // workers per tail tile (fix-up reads)
constexpr int SK_MIN_KB = 16;           // k-blocks per stream-K worker
constexpr int SK_MIN_TILE_KB = 256;     // stream-K only for K >= 4096
static TailSplit tail_split(int num_tiles, int k_blocks, int pairs, const ClusterCaps &caps) {
    static const bool split1 = [] {
        const char *e = getenv("LPY_TF32_SPLIT1");
        return !(e && e[0] == '0');
    }();
    static const bool streamk = [] {
        const char *e = getenv("LPY_TF32_STREAMK");
        return !(e && e[0] == '0');
    }();
    TailSplit r{1, num_tiles, num_tiles, 0, 0, 0, 0, 0.0};
    if (num_tiles <= 0 || pairs <= 0) return r;
    const int waves = (num_tiles + pairs - 1) / pairs;
    r.waves = waves;
    const int rem = num_tiles - (waves - 1) * pairs;
    if (waves < 2) {
        int S = pairs / rem;
        if (S > MAX_SPLITS) S = MAX_SPLITS;
        while (S > 1 && k_blocks / S < 8) --S;
        if (S == 3) S = 2;   // clusters of 2S CTAs: 4 or 8
        if (S == 4 && num_tiles > caps.max8) S = 2;
        if (S == 2 && num_tiles > caps.max4) S = 1;
        if (S < 2 || !split1) return r;
        r.splits = S;
        r.full_tiles = 0;
        r.num_units = num_tiles * S;
        r.cluster = 1;
        r.waves = 1.0 / S;
        return r;
    }
    // Only for long k loops: a split tile costs its pieces a 128 KB partial
    // write per CTA and the last piece the reads of the others, ~30 GB/s per
    // SM while the pair's TMA traffic shares the port (~5 us per partial,
    // scripts/trace_tf32.py, profiles/r02_streamk.txt) -- at K = 1024 (64
    // k-blocks, ~34 us per tile) that ate the whole gain.
    static const int min_tile_kb = [] {    // LPY_TF32_SK_MINKB (A/B): shortest k loop worth stream-K
        const char *e = getenv("LPY_TF32_SK_MINKB");
        return e ? atoi(e) : SK_MIN_TILE_KB;
    }();
    if (!streamk || rem == pairs || k_blocks < min_tile_kb) return r;
    static const int force_workers = [] {   // LPY_TF32_SKW=n: n stream-K workers (diagnostics / A-B)
        const char *e = getenv("LPY_TF32_SKW");
        return e ? atoi(e) : 0;
    }();
    const long long iters = static_cast<long long>(rem) * k_blocks;
    long long workers = pairs;
    if (workers > static_cast<long long>(rem) * SK_MAX_PIECES) workers = static_cast<long long>(rem) * SK_MAX_PIECES;
    if (workers > iters / SK_MIN_KB) workers = iters / SK_MIN_KB;
    if (force_workers > rem && force_workers <= pairs && force_workers <= rem * SK_MAX_PIECES)
        workers = force_workers;
    const double tail = double(rem) / double(workers > 0 ? workers : 1);
    static const double max_tail = [] {     // LPY_TF32_SK_TAIL (A/B): largest tail worth splitting
        const char *e = getenv("LPY_TF32_SK_TAIL");
        return e ? atof(e) : 0.9;
    }();
    if (workers <= rem || tail > max_tail) return r;
    r.full_tiles = (waves - 1) * pairs;
    r.sk_workers = int(workers);
    r.sk_stride = pairs;
    r.sk_iters = iters;
    r.num_units = r.full_tiles + 2 * pairs;
    // + the fix-up: the last piece of a tile re-reads its tile's partials
    r.waves = (waves - 1) + tail + 0.05;
    return r;
}

// Tile width for a CTA-pair product (256-row tiles): the BN in {256, 192, 128}
// minimising the modelled time of the schedule it gives on `pairs` persistent
// CTA pairs: (unit waves) x (k-blocks per unit) x BN / (the kernel's measured
// per-flop efficiency at that width relative to 256: 0.94 for 192, 0.80 for
// 128 at n = 8192 -- narrower MMAs leave the fixed per-k-block work (the A
// tile's TMA and split) less time to hide in; profiles/r02_tf32_bn_sweep.txt,
// with A_small in TMEM for the narrow widths; round 1 measured 0.86 / 0.69),
// over the useful columns; narrower wins only by > 3%.  n >= 4096 -> 256;
// n = 1024 -> 128 (32 tiles instead of 16); the ragged config -> 192 (64 tiles
// instead of 48).
int choose_bn(int M, int N, int K, int pairs, const ClusterCaps &caps, bool kmajor_ab) {
    const int64_t tm = (M + 2 * BM - 1) / (2 * BM);
    const int kb = (K + BK - 1) / BK;
    auto cost = [&](int bn) {
        const int64_t tn = (N + bn - 1) / bn, tiles = tm * tn;
        const TailSplit ts = tail_split(int(tiles), kb, pairs, caps);
        const double kern = bn == 256 ? 1.0 : bn == 192 ? 0.94 : bn == 176 ? 0.92 : 0.80;
        return ts.waves * bn / kern * double(tn * bn) / double(N);
    };
    int best = 256;
    double best_cost = cost(256);
    for (int bn : {192, 176, 128}) {
        if (bn == 176 && !kmajor_ab) continue;   // 176-wide tiles exist for K-major A and B only
        if (cost(bn) * 1.03 < best_cost) { best = bn; best_cost = cost(bn); }
    }
    return best;
}

template <int CG, int BN>
static cudaError_t launch_cg(const Problem &p, const Knobs &kn, const ClusterCaps &caps, cudaStream_t s) {
    const bool AMN = (p.la == 1);   // column-major A: M contiguous
    const bool BMN = (p.lb == 0);   // row-major B: N contiguous
    constexpr int BN_CTA = Cfg<CG, BN>::BN_CTA;
    CUtensorMap ta, tb;
    cudaError_t e;
    if (AMN) e = make_tmap_2d(&ta, p.A, p.M, p.K, p.lda, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    else     e = make_tmap_2d(&ta, p.A, p.K, p.M, p.lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_64B);
    if (e != cudaSuccess) return e;
    if (BMN) e = make_tmap_2d(&tb, p.B, p.N, p.K, p.ldb, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    else     e = make_tmap_2d(&tb, p.B, p.K, p.N, p.ldb, BK, BN_CTA, CU_TENSOR_MAP_SWIZZLE_64B);
    if (e != cudaSuccess) return e;

    Params prm{};
    prm.M = p.M; prm.N = p.N; prm.K = p.K;
    prm.C = p.C; prm.ldc = p.ldc;
    prm.tiles_m = (p.M + BM * CG - 1) / (BM * CG);
    prm.tiles_n = (p.N + BN - 1) / BN;   // (template BN)
    prm.num_tiles = prm.tiles_m * prm.tiles_n;
    prm.k_blocks = (p.K + BK - 1) / BK;
    prm.group = kn.raster_group > 0 ? kn.raster_group : 16 / CG;
    prm.promote = kn.promote_kblocks > 0 ? kn.promote_kblocks : 8;   // 128 of K per TMEM partial
    prm.c_vec = ((reinterpret_cast<uintptr_t>(p.C) & 15) == 0) && (p.ldc % 4 == 0);
    prm.c_vec8 = ((reinterpret_cast<uintptr_t>(p.C) & 31) == 0) && (p.ldc % 8 == 0);
    prm.trace = g_trace;
    prm.gate = kn.gate;
    // B multicast across the two pairs of a 4-CTA cluster (Params::mc):
    // full-width tiles of a row-major B, an even number of 256-row tiles, and
    // a schedule of >= 2 waves of clusters (a single under-filled wave takes
    // the cluster split instead).  LPY_TF32_MC=0 / 1 forces it off / on.
#ifndef LPY_TF32_MC_DEFAULT
#define LPY_TF32_MC_DEFAULT 0
#endif
    static const int mc_env = [] {
        const char *e = getenv("LPY_TF32_MC");
        return e ? atoi(e) : LPY_TF32_MC_DEFAULT;
    }();
    const int clusters = std::min(kn.num_sms / (2 * CG), caps.max4);
    bool mc = CG == 2 && BN == 256 && BMN && mc_env == 1 && kn.num_ctas == 0 && prm.tiles_m % 2 == 0 && clusters > 0 &&
              prm.num_tiles / 2 >= 2 * clusters;
    if (mc) {
        prm.mc = 1;
        prm.tiles_m /= 2;
        prm.num_tiles = prm.tiles_m * prm.tiles_n;
        prm.group = std::max(1, prm.group / 2);
    }
    const int subs = mc ? 2 * CG : CG;   // CTAs per unit
    {
        const TailSplit ts = tail_split(prm.num_tiles, prm.k_blocks, mc ? clusters : kn.num_sms / CG, caps);
        prm.splits = ts.splits;
        prm.full_tiles = ts.full_tiles;
        prm.num_units = ts.num_units;
        prm.sk_workers = ts.sk_workers;
        prm.sk_stride = ts.sk_stride;
        prm.sk_iters = ts.sk_iters;
        prm.cluster_split = CG == 2 ? ts.cluster : 0;
        if (CG == 1 && ts.cluster) {   // (single-CTA diagnostics variant: no cluster split)
            prm.splits = 1;
            prm.full_tiles = prm.num_units = prm.num_tiles;
        }
    }
    prm.ws = nullptr;
    prm.sem = nullptr;
    int units = (kn.num_ctas > 0 ? kn.num_ctas : kn.num_sms) / subs;  // pairs (clusters with mc) in the grid
    if (mc && units > clusters) units = clusters;
    if (units > prm.num_units) units = prm.num_units;
    if (units < 1) units = 1;
    // cluster split: one cluster per tile, every pair runs exactly one unit.
    // A grid capped by opts.num_ctas below that (dist.py's concurrent block
    // products share the GPU) runs the same k-slices through the global-memory
    // fix-up instead -- the same slice-order sums, so the same bits.
    if (prm.cluster_split) {
        if (kn.num_ctas > 0 && kn.num_ctas / CG < prm.num_units) prm.cluster_split = 0;
        else units = prm.num_units;
    }
    const int grid = units * subs;
    if ((prm.splits > 1 && !prm.cluster_split) || prm.sk_workers > 0) {
        const int split_tiles = prm.num_tiles - prm.full_tiles;
        const size_t slots = prm.sk_workers > 0 ? size_t(2) * prm.sk_stride : size_t(split_tiles) * prm.splits;
        const size_t ws_bytes = slots * subs * BM * BN * 4;
        char *buf = nullptr;
        e = cudaMallocAsync(reinterpret_cast<void **>(&buf), ws_bytes + size_t(split_tiles) * subs * 8, s);
        if (e != cudaSuccess) return e;
        prm.ws = reinterpret_cast<float *>(buf);
        prm.sem = reinterpret_cast<int *>(buf + ws_bytes);
        e = cudaMemsetAsync(prm.sem, 0, size_t(split_tiles) * subs * 8, s);
        if (e != cudaSuccess) { cudaFreeAsync(buf, s); return e; }
    }

    auto launch = [&](const Params &q, int g) {
        if constexpr (BN % 64 != 0) {   // (176: K-major A and B only, choose_bn's contract)
            return (AMN || BMN) ? cudaErrorInvalidValue : launch_t<CG, false, false, BN>(ta, tb, q, g, s);
        } else {
            if (AMN && BMN)  return launch_t<CG, true, true, BN>(ta, tb, q, g, s);
            if (AMN && !BMN) return launch_t<CG, true, false, BN>(ta, tb, q, g, s);
            if (!AMN && BMN) return launch_t<CG, false, true, BN>(ta, tb, q, g, s);
            return launch_t<CG, false, false, BN>(ta, tb, q, g, s);
        }
    };
    e = launch(prm, grid);
    if (e != cudaSuccess && prm.cluster_split) {
        // a cluster of 2S CTAs this size could not be placed (configuration
        // error, nothing enqueued): run the tiles whole instead
        (void)cudaGetLastError();
        Params q = prm;
        q.cluster_split = 0;
        q.splits = 1;
        q.sk_workers = 0;
        q.full_tiles = q.num_units = q.num_tiles;
        const int g = CG * (q.num_units < kn.num_sms / CG ? q.num_units : kn.num_sms / CG);
        e = launch(q, g > 0 ? g : CG);
    }
    if (prm.ws) cudaFreeAsync(prm.ws, s);
    return e;
}

// Co-resident clusters of 4 and 8 CTAs of the (one CTA per SM) kernel on the
// current device, queried once per device.
static ClusterCaps cluster_caps(int num_sms) {
    static std::mutex mu;
    static ClusterCaps cache[64];
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return ClusterCaps{0, 0};
    std::lock_guard<std::mutex> g(mu);
    if (done[dev]) return cache[dev];
    using C_ = Cfg<2, 256>;
    auto kern = gemm_3xtf32_kernel<2, false, true, 256>;
    static std::atomic<uint64_t> attr_done{0};
    ClusterCaps c{0, 0};
    if (ensure_smem_attr(kern, int(C_::SMEM_BYTES), attr_done) == cudaSuccess) {
        for (int size : {4, 8}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(size * (num_sms / size > 0 ? num_sms / size : 1));
            cfg.blockDim = dim3(THREADS);
            cfg.dynamicSmemBytes = C_::SMEM_BYTES;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = size;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
                (void)cudaGetLastError();
                n = 0;
            }
            (size == 4 ? c.max4 : c.max8) = n;
        }
    }
    cache[dev] = c;
    done[dev] = true;
    return c;
}

}  // namespace tf32

bool tf32_available() { return true; }
bool tf32_supported(const Problem &) { return true; }

cudaError_t launch_3xtf32(const Problem &p, const Knobs &kn, cudaStream_t s) {
    // LPY_TF32_CG=1 selects the single-CTA variant (diagnostics / A-B comparison).
    static const int cg = [] {
        const char *e = getenv("LPY_TF32_CG");
        return (e && e[0] == '1') ? 1 : 2;
    }();
    const tf32::ClusterCaps caps = tf32::cluster_caps(kn.dev_sms);
    if (cg == 1) return tf32::launch_cg<1, 256>(p, kn, caps, s);
    // LPY_TF32_BN=128|192|256 forces the tile width (diagnostics / A-B comparison).
    static const int force_bn = [] {
        const char *e = getenv("LPY_TF32_BN");
        return e ? atoi(e) : 0;
    }();
    // the tile width comes from the shape and the device (the tail split
    // follows the tile count, and results must not depend on opts.num_ctas),
    // or from opts.tile_n (dist.py's per-chunk products, which share the GPU,
    // ask for full-width tiles)
    const int pairs = kn.num_sms / 2;
    const bool kmajor_ab = p.la == 0 && p.lb == 1;   // row-major A, column-major B
    const int bn = kn.tile_n ? kn.tile_n : force_bn ? force_bn : tf32::choose_bn(p.M, p.N, p.K, pairs > 0 ? pairs : 1, caps,
                                                                                kmajor_ab);
    switch (bn) {
        case 128: return tf32::launch_cg<2, 128>(p, kn, caps, s);
        case 176: return kmajor_ab ? tf32::launch_cg<2, 176>(p, kn, caps, s) : cudaErrorInvalidValue;
        case 192: return tf32::launch_cg<2, 192>(p, kn, caps, s);
        default:  return tf32::launch_cg<2, 256>(p, kn, caps, s);
    }
}

}  // namespace lpy

#ifdef LPY_TRACE
// Diagnostics build only: device buffer of 8 counters per CTA, accumulated by
// every subsequent 3xTF32 launch (zero it between runs).
extern "C" void lpy_trace_set_buffer(long long *dev) { lpy::tf32::g_trace = dev; }
#endif
