/*
 * lpy.h -- C ABI of the B200-native fp32 GEMM after Loo.py (Kloeckner,
 * "Loo.py: transformation-based code generation for GPUs and CPUs",
 * ARRAY'14, arXiv:1405.7470).  Citations "P:n" are lines of the paper text
 * (/root/reference/PAPER.md); "S:n" lines of SPEC.md.  Implementation:
 * paper_1405_7470_b200/csrc/.  Python binding with the same names:
 * paper_1405_7470_b200/__init__.py.
 *
 * THE OPERATION.  The paper's reduction example
 *
 *     c[i,j] = sum(k, a[i,k]*b[k,j])                  (section 2.1)
 *
 * over the loop domain {[i,j,k]: 0<=i<M, 0<=j<N, 0<=k<K} whose parameters
 * M, N, K are passed by value at call time.  fp32 inputs give
 * fp32 outputs (type inference).  C is OVERWRITTEN (pure
 * assignment, no alpha/beta: the instruction is a plain assignment).
 * The order of the k summation is unspecified (unordered semantics,
 * P:395-401); results are accurate to
 *     max_ij |C_ij - Cexact_ij| / sum_k |A_ik||B_kj|  <=  1e-5
 * on either path for FINITE inputs (with promote_kblocks <= 16, the largest
 * value lpy_gemm_f32_ex accepts), and exact when every input and partial sum
 * is an integer representable in fp32 and tf32 (readings A1, A2).
 * Non-finite inputs: the FFMA path propagates Inf/NaN as IEEE fp32 FMAs do;
 * the 3xTF32 path turns Inf into NaN (see LPY_PATH_3XTF32).
 *
 * LAYOUT.  Every operand carries a stride tag (P:278-280, P:313-315,
 * P:594-601, sections 2.1 and 2.4.3):
 *     LPY_ROW_MAJOR:  X(r,c) = X[r*ld + c],  ld >= max(1, cols)
 *     LPY_COL_MAJOR:  X(r,c) = X[r + c*ld],  ld >= max(1, rows)
 * A is M x K, B is K x N, C is M x N (logical shapes).  Leading dimensions
 * and element counts are in ELEMENTS (floats), not bytes.  Padding between
 * lines (ld > minor extent, "padding") is never read or written.
 *
 * OWNERSHIP.  The caller owns A, B, C.  For the device entry points they are
 * device memory of the CURRENT CUDA device (e.g. torch tensors); the library
 * never frees, reallocates or retains them beyond the enqueued work.  Internal
 * scratch (the aligned repack of an operand whose base is not 16-byte aligned
 * or whose ld is not a multiple of 4) is stream-ordered (cudaMallocAsync /
 * cudaFreeAsync on the caller's stream).
 *
 * ASYNCHRONY.  Device entry points enqueue on `stream` (a cudaStream_t passed
 * as void*; NULL = legacy default stream) and return without synchronising,
 * like the paper's `evt, (out,) = knl(queue, a=x_dev)`.  Faults in
 * enqueued work surface at the caller's next synchronisation.
 *
 * ERRORS.  Every argument is validated BEFORE anything is enqueued; on any
 * error return C is untouched and nothing was enqueued (except LPY_ERR_CUDA
 * raised by a failed launch).  Nothing is thrown across the ABI.  Reentrant;
 * safe to call from several host threads on different streams.
 *
 * DEGENERATE SIZES.  M == 0 or N == 0: empty domain, no-op returning LPY_OK
 * (S:295).  K == 0: C := 0, the identity of `sum`.
 *
 * DETERMINISM.  For a given shape, path, operand values, tile width and device
 * (its SM count), the result is bitwise reproducible and independent of the
 * lpy_gemm_opts scheduling knobs num_ctas and raster_group, of the layouts of
 * A and B, and of the stream: every element's k order is fixed by the shape
 * (split-K slices, however scheduled -- persistent tiles, global-memory
 * fix-up, or a thread-block cluster's distributed-shared-memory reduction --
 * are summed in slice order).
 *
 * CAPTURE AND CHAINING.  Calls are stream-capturable into CUDA graphs.  The
 * 3xTF32 and repack kernels use programmatic dependent launch: they may start
 * their prologue while the preceding kernel in the stream finishes, but wait
 * for it (griddepcontrol.wait) before reading A/B or writing C, so stream
 * order semantics are unchanged.
 */
#ifndef LPY_H
#define LPY_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LPY_VERSION 5

typedef enum { LPY_ROW_MAJOR = 0, LPY_COL_MAJOR = 1 } lpy_layout;

/* Which kernel computes the product.
 *  LPY_PATH_FFMA   : fp32 FFMA on the SIMT pipes -- TMA-staged tiles in shared
 *                    memory ("add_prefetch"), mbarrier producer /
 *                    consumer ring, per-thread register micro-tile ("ilp" +
 *                    "unr").  Each product and sum is an fp32 RN op.
 *  LPY_PATH_3XTF32 : tcgen05 tensor cores, kind::tf32.  The tensor core reads
 *                    an fp32 operand as tf32 by TRUNCATING its 13 low mantissa
 *                    bits (measured, reading A9), so each fp32 x is
 *                    used as big = x (seen as trunc_tf32(x)) plus
 *                    small = rna_tf32(x - trunc_tf32(x)), and
 *                    C += A_big B_small + A_big B_big + A_small B_big
 *                    (small*small dropped; issued in that order) accumulated in
 *                    TMEM, which rounds toward zero, and promoted into fp32
 *                    registers (round-to-nearest) every promote_kblocks k-blocks.
 *                    INPUTS MUST BE FINITE on this path: an Inf operand makes
 *                    x - trunc(x) = Inf - Inf = NaN, so the result is NaN where
 *                    the FFMA path would give Inf (reading A11).
 *  LPY_PATH_AUTO   : the library picks (lpy_select_path says which). */
typedef enum { LPY_PATH_AUTO = 0, LPY_PATH_FFMA = 1, LPY_PATH_3XTF32 = 2 } lpy_path;

typedef enum {
    LPY_OK = 0,
    LPY_ERR_INVALID_VALUE = 1,      /* M/N/K < 0 or > 2^31 - 1024, bad enum value, an    */
                                    /* operand spanning >= 2^62 elements, or an opts     */
                                    /* field out of range                                */
    LPY_ERR_INVALID_LD = 2,         /* ld below the minimum stated under LAYOUT          */
    LPY_ERR_NULL_POINTER = 3,       /* NULL operand with a nonzero footprint             */
    LPY_ERR_MISALIGNED = 4,         /* operand pointer not 4-byte aligned                */
    LPY_ERR_ALIAS = 5,              /* C's footprint overlaps A's or B's ("restrict",    */
                                    /* P:354)                                            */
    LPY_ERR_UNSUPPORTED_DEVICE = 6, /* current device is not compute capability 10.0     */
    LPY_ERR_OUT_OF_MEMORY = 7,      /* scratch allocation failed                         */
    LPY_ERR_CUDA = 8,               /* CUDA runtime/driver error: lpy_last_cuda_error()  */
    LPY_ERR_NOT_SUPPORTED = 9       /* requested path cannot run this problem            */
} lpy_status;

/* Tuning / test knobs for lpy_gemm_f32_ex.  Zero-initialise for defaults. */
typedef struct lpy_gemm_opts {
    int32_t num_ctas;        /* persistent grid size; 0 = one CTA (pair) per SM      */
    int32_t raster_group;    /* output-tile rows per rasterisation group; 0 = auto   */
    int32_t promote_kblocks; /* 3xTF32: k-blocks (16 of K each) per TMEM partial     */
                             /* before promotion; 0 = auto (8); 1..16, larger values */
                             /* are LPY_ERR_INVALID_VALUE (32 measured 1.05e-5 on    */
                             /* uniform[0,1) at K = 8192: beyond the contract)       */
    int32_t tile_n;          /* output-tile width: 0 = auto (from shape and device;  */
                             /* auto may also pick 176 on 3xTF32 for row-major A     */
                             /* with column-major B, a width not selectable here),   */
                             /* else 128 or 256 (both paths) or 192 (3xTF32 only;    */
                             /* LPY_ERR_NOT_SUPPORTED on FFMA); other values are     */
                             /* LPY_ERR_INVALID_VALUE.  Results do not depend on the  */
                             /* grid (num_ctas); a different tile width can change   */
                             /* the k-split of under-filled grids and so the last    */
                             /* bits (always within the 1e-5 bound)                  */
    int32_t plan_sms;        /* SMs the schedule is planned for: 0 = the device's    */
                             /* (all of them), else 1..device SMs.  Sets the tile    */
                             /* width, the split-K / stream-K decomposition and the  */
                             /* default grid; the result depends on it (like tile_n) */
                             /* but never on num_ctas.  A product sharing the GPU    */
                             /* with concurrent work (the row-panel product beside   */
                             /* its broadcast, lpy_gemm_f32_gated) plans for the SMs */
                             /* it will actually get                                 */
    int32_t reserved[3];     /* must be 0                                            */
} lpy_gemm_opts;

/* C := A * B on the device, enqueued on `stream` (see header comment).
 * Returns LPY_OK or an lpy_status error. */
lpy_status lpy_gemm_f32(int64_t M, int64_t N, int64_t K,
                        const float *A, int64_t lda, lpy_layout layout_a,
                        const float *B, int64_t ldb, lpy_layout layout_b,
                        float *C, int64_t ldc, lpy_layout layout_c,
                        void *stream);

/* As lpy_gemm_f32 with an explicit path and optional knobs (opts may be NULL). */
lpy_status lpy_gemm_f32_ex(int64_t M, int64_t N, int64_t K,
                           const float *A, int64_t lda, lpy_layout layout_a,
                           const float *B, int64_t ldb, lpy_layout layout_b,
                           float *C, int64_t ldc, lpy_layout layout_c,
                           void *stream, lpy_path path, const lpy_gemm_opts *opts);

/* ---------------------------------------------------------------- K-gated product
 * The row-panel product of the multi-GPU step (BASELINE north_star: C's row
 * panels sharded over the GPUs, B broadcast once over NVLink)
 * starts while B is still arriving.  Every output tile walks K in order, so
 * the k-th rows of B are needed only when the tiles reach k: B is broadcast in
 * chunks of K rows (contiguous in row-major B) and ONE persistent product
 * consumes each chunk as soon as it has landed -- the paper's reduction
 * sum(k, a[i,k]*b[k,j]) with its k loop split into chunks
 * (split_iname) whose prefetch (add_prefetch) waits for
 * the chunk's arrival.
 *
 * lpy_kgate describes the arrival flags: chunk c = k in [c*chunk_k,
 * min(K, (c+1)*chunk_k)), published by setting flags[c] to `epoch` (e.g. with
 * lpy_kgate_signal after the chunk's broadcast, stream-ordered).  The product
 * reads NO element of A or B with k in chunk c before (int32_t)(flags[c] -
 * epoch) >= 0, i.e. flags compare wrap-aware, so a caller reuses one flag
 * array across steps by raising the epoch (no reset).  Chunks must be published
 * in increasing c (the kernels poll the next chunk only).
 *   flags      : device memory of the current device, ceil(K / chunk_k) words,
 *                owned by the caller, read (never written) by the product.
 *   chunk_k    : K indices per chunk, >= 32 (a k-block of 32 spans at most two
 *                chunks) and <= 2^31 - 1024.
 *   epoch      : the value that marks a chunk ready in this call.
 *   timeout_ms : a chunk not ready this long after the kernel first polls it
 *                traps the kernel (a deadlock detector: the error surfaces at
 *                the next synchronisation as a CUDA launch failure and the
 *                context is lost); 0 = 10000 ms.
 * SCHEDULING CONTRACT.  The product spins on the flags while occupying its
 * grid, so whatever sets them (the broadcast's NCCL kernels and the signal
 * kernel) must be able to run beside it: plan the product for fewer SMs than
 * the device has (opts.plan_sms; dist.py leaves 32 free) or set the flags from
 * a copy engine / the host.  Every kernel that sets flags must also be LOADED
 * before the product is launched: under CUDA's lazy module loading a kernel's
 * first launch loads its code and waits for the device, i.e. for the spinning
 * product (this call loads lpy_kgate_signal's kernel itself; a caller's own
 * kernels -- NCCL's included -- must have run once, or be enqueued before the
 * product as dist.py does).  Operands that would need the aligned repack
 * (base not 16-byte aligned or ld not a multiple of 4) are LPY_ERR_NOT_SUPPORTED
 * here: the repack would read them before they arrive.  Otherwise the
 * arguments, errors and result are those of lpy_gemm_f32_ex with the same opts
 * (bitwise: the gate changes when operands are read, not the arithmetic). */
typedef struct lpy_kgate {
    const uint32_t *flags;
    int64_t chunk_k;
    uint32_t epoch;
    uint32_t timeout_ms;
} lpy_kgate;

lpy_status lpy_gemm_f32_gated(int64_t M, int64_t N, int64_t K,
                              const float *A, int64_t lda, lpy_layout layout_a,
                              const float *B, int64_t ldb, lpy_layout layout_b,
                              float *C, int64_t ldc, lpy_layout layout_c,
                              void *stream, lpy_path path, const lpy_gemm_opts *opts,
                              const lpy_kgate *gate);

/* Enqueue on `stream`: once all work before it in the stream has completed,
 * *flag := value with release semantics at GPU scope (the writes of that
 * earlier work -- e.g. a broadcast's received bytes -- are visible to a
 * product that acquires the flag).  flag: device memory of the current
 * device, 4-byte aligned (LPY_ERR_NULL_POINTER / LPY_ERR_MISALIGNED).  One
 * 32-thread kernel launch; needs one free SM while a gated product runs. */
lpy_status lpy_kgate_signal(uint32_t *flag, uint32_t value, void *stream);

/* End-to-end variant on HOST buffers: copies the logical extents of A and B to
 * device scratch (stream-ordered, repacked to 16-byte-aligned leading
 * dimensions on the way), runs lpy_gemm_f32_ex, copies the logical extent of C
 * back (padding of host C untouched) and SYNCHRONISES `stream` before
 * returning.  Pinned (page-locked) host buffers give full PCIe bandwidth;
 * pageable ones work but are slower. */
lpy_status lpy_gemm_f32_host(int64_t M, int64_t N, int64_t K,
                             const float *A, int64_t lda, lpy_layout layout_a,
                             const float *B, int64_t ldb, lpy_layout layout_b,
                             float *C, int64_t ldc, lpy_layout layout_c,
                             void *stream, lpy_path path);

/* ---------------------------------------------------------------- saxpy
 * y := alpha * x + y over n elements: Table 1's "saxpy" row (section 3),
 * the paper's bandwidth-bound BLAS-1 workload, through the same boundary.
 * Element i lives at x[i*incx] and y[i*incy] (incx, incy >= 1, in ELEMENTS).
 * Each result is fl32(alpha*x_i + y_i) rounded ONCE (one fused multiply-add,
 * round-to-nearest-even); inputs finite (reading S1).
 * x and y are device memory of the current device, owned by the caller; y is
 * overwritten in place, nothing else is written.  x and y must either not
 * overlap or be the same vector (x == y, incx == incy: y := alpha*y + y);
 * any other overlap is LPY_ERR_ALIAS.  n == 0 is a no-op.  Enqueued on
 * `stream` (NULL = legacy default stream), asynchronous like lpy_gemm_f32.
 * Errors: LPY_ERR_INVALID_VALUE (n < 0, inc < 1, n*inc beyond 2^62),
 * LPY_ERR_NULL_POINTER, LPY_ERR_MISALIGNED (not 4-byte aligned), LPY_ERR_ALIAS,
 * LPY_ERR_UNSUPPORTED_DEVICE, LPY_ERR_CUDA; validated before anything runs. */
lpy_status lpy_saxpy_f32(int64_t n, float alpha, const float *x, int64_t incx, float *y,
                         int64_t incy, void *stream);

/* End-to-end saxpy on HOST buffers: copies x and y to device scratch, runs
 * lpy_saxpy_f32, copies y back and SYNCHRONISES `stream` before returning.
 * Same argument rules as lpy_saxpy_f32 (pinned host memory for full PCIe
 * bandwidth). */
lpy_status lpy_saxpy_f32_host(int64_t n, float alpha, const float *x, int64_t incx, float *y,
                              int64_t incy, void *stream);

/* ---------------------------------------------------------------- Coulomb
 * phi[i] := sum_{j : r_ij != 0} q[j] / r_ij for i < nt: the 3D Coulomb
 * potential of ns point charges at nt targets, Table 1's third workload
 * (section 3), reported in pairs/s (nt * ns per call).
 *   targets: t[i*ldt + 0..2] = (x, y, z) of target i, ldt >= 3 (ELEMENTS);
 *   sources: s[j*lds + 0..2] = (x, y, z) of source j, lds >= 3; q[j] its charge;
 *   phi:     nt floats, OVERWRITTEN (ns == 0 gives zeros).
 * r_ij = |t_i - s_j|.  A source exactly at a target (r_ij == 0, e.g. the
 * target itself when the two sets are the same array) contributes nothing
 * (reading C1).  fp32 in, fp32 out; accuracy (reading C2):
 *     |phi_i - phi_exact_i| <= 5e-6 * sum_j |q_j| / r_ij
 * for finite inputs whose nonzero coordinate differences have squares in the
 * fp32 normal range (|d| in [2^-63, 2^63]).  Deterministic (fixed summation
 * order for a given shape and device).  Device memory of the current device,
 * owned by the caller; internal scratch (packed sources, slice partials) is
 * stream-ordered on `stream`.  phi must not overlap t, s or q
 * (LPY_ERR_ALIAS).  nt == 0 is a no-op.  Errors as for lpy_gemm_f32:
 * LPY_ERR_INVALID_VALUE (nt/ns < 0), LPY_ERR_INVALID_LD (ldt/lds < 3),
 * LPY_ERR_NULL_POINTER, LPY_ERR_MISALIGNED, LPY_ERR_ALIAS,
 * LPY_ERR_UNSUPPORTED_DEVICE, LPY_ERR_OUT_OF_MEMORY, LPY_ERR_CUDA. */
lpy_status lpy_coulomb_f32(int64_t nt, const float *t, int64_t ldt,
                           int64_t ns, const float *s, int64_t lds, const float *q,
                           float *phi, void *stream);

/* End-to-end Coulomb on HOST buffers: uploads targets, sources and charges,
 * runs lpy_coulomb_f32, downloads phi and SYNCHRONISES `stream`. */
lpy_status lpy_coulomb_f32_host(int64_t nt, const float *t, int64_t ldt,
                                int64_t ns, const float *s, int64_t lds, const float *q,
                                float *phi, void *stream);

/* Host-only: the path `requested` resolves to for this problem shape (no CUDA
 * calls).  Returns LPY_ERR_INVALID_VALUE for bad enum/sizes. */
lpy_status lpy_select_path(int64_t M, int64_t N, int64_t K, lpy_path requested,
                           lpy_path *chosen);

/* Static description of an lpy_status value (never NULL). */
const char *lpy_status_string(lpy_status s);

/* cudaError_t of this thread's most recent LPY_ERR_CUDA (0 if none). */
int lpy_last_cuda_error(void);

/* LPY_VERSION of the loaded library. */
int lpy_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LPY_H */
