// Internal interface between the C-ABI front end (lpy_api.cu) and the kernels.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace lpy {

// A canonical problem: C is row-major (lpy_api.cu maps a column-major C to
// the transposed problem C^T = B^T A^T first).  Operand layouts: 0 = row-major,
// 1 = column-major, as in lpy.h.  After the front end's repack step every
// operand pointer is 16-byte aligned and every ld a multiple of 4 (TMA).
struct Problem {
    int M, N, K;
    const float *A;
    int64_t lda;
    int la;
    const float *B;
    int64_t ldb;
    int lb;
    float *C;
    int64_t ldc;
};

// cudaFuncAttributeMaxDynamicSharedMemorySize for `kern` on the current
// device, once per device (function attributes are per device context; a
// process-wide "done" flag would skip the second GPU of a multi-GPU process).
// `done` is a per-kernel bitmask of devices already configured.
template <class F>
inline cudaError_t ensure_smem_attr(F kern, int bytes, std::atomic<uint64_t> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// Programmatic dependent launch for the library's kernels (every kernel
// launched with it calls griddepcontrol.wait before its first global memory
// access): on unless LPY_PDL=0.  Appends the attribute to attrs[n], returns
// the new count.
int pdl_attr(cudaLaunchAttribute *attrs, int n);

// K-gate of a product whose operands arrive in chunks of K (lpy_kgate in
// lpy.h; waited on by the kernels' TMA producers, ptx.cuh kgate_wait): no
// operand element with k in chunk c = [c*chunk_k, (c+1)*chunk_k) is read
// before flags[c] - epoch >= 0 (wrap-aware).
struct KGate {
    const uint32_t *flags;   // nullptr: ungated
    int chunk_k;             // K indices per flag (>= 32, so a k-block spans <= 2 chunks)
    uint32_t epoch;
    uint64_t timeout_ns;     // per wait; exceeded -> __trap() (a deadlock detector)
    int nchunks;             // ceil(K / chunk_k)
};

struct Knobs {
    int num_ctas;         // 0 = auto
    int raster_group;     // 0 = auto
    int promote_kblocks;  // 0 = auto
    int num_sms;          // SMs the schedule is PLANNED for: opts.plan_sms, else the device's
                          // (tile width, split-K / stream-K decomposition, default grid)
    int tile_n;           // 0 = auto; else the output-tile width (validated by the front end)
    int dev_sms;          // multiprocessor count of the current device (co-residency queries)
    KGate gate;           // flags == nullptr: ungated
};

// 2-D tensor map over a strided matrix: `inner` contiguous elements per line,
// `outer` lines at stride `ld` elements; box = box_inner x box_outer elements.
// `swizzle` is the smem swizzle mode TMA applies to the box.
cudaError_t make_tmap_2d(CUtensorMap *tm, const float *base, uint64_t inner, uint64_t outer,
                         uint64_t ld, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swizzle);

cudaError_t launch_ffma(const Problem &p, const Knobs &k, cudaStream_t s);
// flag := value (release, GPU scope) once the stream's earlier work is done (kgate.cu)
cudaError_t launch_kgate_signal(uint32_t *flag, uint32_t value, cudaStream_t s);
cudaError_t preload_kgate_signal();   // load its module now (lazy loading vs a spinning product)
// split-K slices for `tiles` output tiles of `k_blocks` k-blocks on `workers`
// persistent CTAs (pairs); >= min_kb k-blocks per slice, <= max_splits (gemm_ffma.cu)
int choose_splits(int tiles, int k_blocks, int workers, int min_kb, int max_splits);
cudaError_t launch_3xtf32(const Problem &p, const Knobs &k, cudaStream_t s);
bool tf32_supported(const Problem &p);
bool tf32_available();  // the 3xTF32 kernel is compiled in

// y := alpha * x + y (saxpy.cu); n > 0 handled, n <= 0 is a no-op.
cudaError_t launch_saxpy(int64_t n, float alpha, const float *x, int64_t incx, float *y, int64_t incy,
                         int num_sms, cudaStream_t s);

// phi := Coulomb potential of (s, q) at t (coulomb.cu); nt <= 0 is a no-op.
cudaError_t launch_coulomb(int64_t nt, const float *t, int64_t ldt, int64_t ns, const float *s, int64_t lds,
                           const float *q, float *phi, int num_sms, cudaStream_t st);

// dst[line*ld_dst + e] = src[line*ld_src + e] for line < lines, e < inner
// (pad columns zeroed), for njobs (1 or 2) operands in one launch.
struct RepackJob {
    const float *src;
    int64_t ld_src;
    float *dst;
    int64_t ld_dst, lines, inner;
};
cudaError_t launch_repack(const RepackJob *jobs, int njobs, int num_sms, cudaStream_t s);

}  // namespace lpy
