// C-ABI front end (include/lpy.h): validation, layout canonicalisation,
// degenerate sizes, aligned repack, path selection, launch, and the host-buffer
// end-to-end entry point.  No torch types anywhere; plain pointers and sizes.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/lpy.h"
#include "lpy_internal.h"

namespace {

thread_local int g_last_cuda_error = 0;

lpy_status cuda_fail(cudaError_t e) {
    g_last_cuda_error = static_cast<int>(e);
    if (e == cudaErrorMemoryAllocation) return LPY_ERR_OUT_OF_MEMORY;
    return LPY_ERR_CUDA;
}

// M, N, K <= 2^31 - 1024: the kernels round dimensions up to whole tiles and
// k-blocks in 32-bit int arithmetic, which must not overflow (include/lpy.h).
constexpr int64_t kMaxDim = INT32_MAX - 1023;
constexpr int64_t kMaxLd = (int64_t(1) << 40) / 4 - 1;  // TMA: global strides < 2^40 bytes
constexpr int64_t kMaxFootprint = int64_t(1) << 62;      // elements an operand may span
constexpr int kMaxPromote = 16;                          // 3xTF32 partial length bound (1e-5 contract)

struct Operand {
    const float *p;
    int64_t rows, cols, ld;
    int layout;
    int64_t lines() const { return layout == LPY_ROW_MAJOR ? rows : cols; }
    int64_t inner() const { return layout == LPY_ROW_MAJOR ? cols : rows; }
    // footprint in elements: (lines-1)*ld + inner, or 0 for an empty matrix
    int64_t extent() const { return (rows == 0 || cols == 0) ? 0 : (lines() - 1) * ld + inner(); }
};

bool valid_layout(int l) { return l == LPY_ROW_MAJOR || l == LPY_COL_MAJOR; }

lpy_status validate_operand(const Operand &o) {
    const int64_t need = o.inner() > 1 ? o.inner() : 1;
    if (o.ld < need || o.ld > kMaxLd) return LPY_ERR_INVALID_LD;
    // (lines-1)*ld + inner must stay far from int64 overflow before extent()
    // multiplies it out (lines <= 2^31, ld < 2^38, so the product can pass 2^63)
    if (o.rows > 0 && o.cols > 0 && o.lines() - 1 > (kMaxFootprint - o.inner()) / o.ld)
        return LPY_ERR_INVALID_VALUE;
    if (o.extent() > 0) {
        if (o.p == nullptr) return LPY_ERR_NULL_POINTER;
        if (reinterpret_cast<uintptr_t>(o.p) & 3) return LPY_ERR_MISALIGNED;
    }
    return LPY_OK;
}

bool overlaps(const Operand &a, const Operand &b) {
    if (a.extent() == 0 || b.extent() == 0) return false;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(a.p), a1 = a0 + uintptr_t(a.extent()) * 4;
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(b.p), b1 = b0 + uintptr_t(b.extent()) * 4;
    return a0 < b1 && b0 < a1;
}

lpy_status validate_all(int64_t M, int64_t N, int64_t K, const Operand &A, const Operand &B,
                        const Operand &C, int path, const lpy_gemm_opts *opts) {
    if (M < 0 || N < 0 || K < 0 || M > kMaxDim || N > kMaxDim || K > kMaxDim)
        return LPY_ERR_INVALID_VALUE;
    if (!valid_layout(A.layout) || !valid_layout(B.layout) || !valid_layout(C.layout))
        return LPY_ERR_INVALID_VALUE;
    if (path != LPY_PATH_AUTO && path != LPY_PATH_FFMA && path != LPY_PATH_3XTF32)
        return LPY_ERR_INVALID_VALUE;
    if (opts) {
        if (opts->num_ctas < 0 || opts->raster_group < 0 || opts->promote_kblocks < 0 ||
            opts->promote_kblocks > kMaxPromote)
            return LPY_ERR_INVALID_VALUE;
        if (opts->tile_n != 0 && opts->tile_n != 128 && opts->tile_n != 192 && opts->tile_n != 256)
            return LPY_ERR_INVALID_VALUE;
        if (opts->plan_sms < 0) return LPY_ERR_INVALID_VALUE;   // (upper bound: the device's, checked at launch)
        for (int i = 0; i < 3; ++i)
            if (opts->reserved[i] != 0) return LPY_ERR_INVALID_VALUE;
    }
    lpy_status s;
    if ((s = validate_operand(A)) != LPY_OK) return s;
    if ((s = validate_operand(B)) != LPY_OK) return s;
    if ((s = validate_operand(C)) != LPY_OK) return s;
    if (overlaps(C, A) || overlaps(C, B)) return LPY_ERR_ALIAS;
    return LPY_OK;
}

struct DeviceInfo {
    int major = 0, minor = 0, sms = 0;
    bool ok = false;
};

lpy_status device_info(DeviceInfo &out) {
    static std::mutex mu;
    static DeviceInfo cache[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    if (dev < 0 || dev >= 64) return LPY_ERR_UNSUPPORTED_DEVICE;
    std::lock_guard<std::mutex> g(mu);
    if (!cache[dev].ok) {
        DeviceInfo d;
        if ((e = cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess ||
            (e = cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev)) != cudaSuccess ||
            (e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
            return cuda_fail(e);
        d.ok = true;
        cache[dev] = d;
        // Keep freed stream-ordered scratch in the device's default pool instead of
        // returning it to the driver at every synchronisation: the end-to-end entry
        // point allocates and frees ~800 MB per call at n = 8192, and re-mapping it
        // each time cost more than the copies themselves.
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    out = cache[dev];
    // The kernels are built for sm_100a only (tcgen05 / TMA); anything else would
    // fail at launch with "no kernel image", so refuse up front.
    if (!(out.major == 10 && out.minor == 0)) return LPY_ERR_UNSUPPORTED_DEVICE;
    return LPY_OK;
}

// Copy `lines` lines of `inner` floats between pitched buffers; one linear DMA
// when both sides are packed (2-D copies of very tall matrices run far below
// PCIe bandwidth).
cudaError_t copy_lines(void *dst, int64_t ld_dst, const void *src, int64_t ld_src, int64_t inner,
                       int64_t lines, cudaMemcpyKind kind, cudaStream_t s) {
    if (ld_dst == inner && ld_src == inner)
        return cudaMemcpyAsync(dst, src, size_t(inner * lines) * 4, kind, s);
    return cudaMemcpy2DAsync(dst, size_t(ld_dst) * 4, src, size_t(ld_src) * 4, size_t(inner) * 4,
                             size_t(lines), kind, s);
}

lpy_path resolve_path(int64_t M, int64_t N, int64_t K, lpy_path requested) {
    if (requested != LPY_PATH_AUTO) return requested;
    // 3xTF32 on the tensor cores wins once there is enough work to fill the
    // machine; tiny problems are launch-latency bound either way.
    const double work = double(M) * double(N) * double(K);
    return (lpy::tf32_available() && work >= double(1 << 27)) ? LPY_PATH_3XTF32 : LPY_PATH_FFMA;
}

}  // namespace

namespace lpy {

using PFN_encodeTiled = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                     const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                     const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    return fn;
}

// Encoded descriptors are cached (a call re-using the buffers of an earlier one
// -- a training or benchmark loop -- skips cuTensorMapEncodeTiled, which costs
// about as much host time as the launch).  A descriptor holds only the address
// and geometry, so an entry stays valid whatever happens to the memory behind
// it; the cache is a small direct-mapped table under a mutex.
namespace {
struct TmapKey {
    const float *base;
    uint64_t inner, outer, ld;
    uint32_t box_inner, box_outer;
    int swizzle;
    bool operator==(const TmapKey &o) const {
        return base == o.base && inner == o.inner && outer == o.outer && ld == o.ld && box_inner == o.box_inner &&
               box_outer == o.box_outer && swizzle == o.swizzle;
    }
};
struct TmapEntry {
    bool used = false;
    TmapKey key{};
    CUtensorMap map{};
};
constexpr int kTmapCache = 64;
std::mutex tmap_mu;
TmapEntry tmap_cache[kTmapCache];

size_t tmap_slot(const TmapKey &k) {
    uint64_t h = reinterpret_cast<uintptr_t>(k.base) >> 8;
    for (uint64_t v : {k.inner, k.outer, k.ld, uint64_t(k.box_inner) << 32 | k.box_outer, uint64_t(k.swizzle)})
        h = (h ^ v) * 0x9E3779B97F4A7C15ull;
    return size_t(h >> 58) % kTmapCache;
}
}  // namespace

int pdl_attr(cudaLaunchAttribute *attrs, int n) {
    static const bool on = [] {
        const char *e = getenv("LPY_PDL");
        return !(e && e[0] == '0');
    }();
    if (!on) return n;
    attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[n].val.programmaticStreamSerializationAllowed = 1;
    return n + 1;
}

cudaError_t make_tmap_2d(CUtensorMap *tm, const float *base, uint64_t inner, uint64_t outer, uint64_t ld,
                         uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swizzle) {
    const TmapKey key{base, inner, outer, ld, box_inner, box_outer, int(swizzle)};
    const size_t slot = tmap_slot(key);
    {
        std::lock_guard<std::mutex> g(tmap_mu);
        if (tmap_cache[slot].used && tmap_cache[slot].key == key) {
            *tm = tmap_cache[slot].map;
            return cudaSuccess;
        }
    }
    PFN_encodeTiled enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * sizeof(float)};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swizzle,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(tmap_mu);
    tmap_cache[slot].used = true;
    tmap_cache[slot].key = key;
    tmap_cache[slot].map = *tm;
    return cudaSuccess;
}

}  // namespace lpy

extern "C" {

const char *lpy_status_string(lpy_status s) {
    switch (s) {
        case LPY_OK: return "LPY_OK";
        case LPY_ERR_INVALID_VALUE: return "LPY_ERR_INVALID_VALUE: bad size or enum argument";
        case LPY_ERR_INVALID_LD: return "LPY_ERR_INVALID_LD: leading dimension below the minor extent";
        case LPY_ERR_NULL_POINTER: return "LPY_ERR_NULL_POINTER: NULL operand with nonzero extent";
        case LPY_ERR_MISALIGNED: return "LPY_ERR_MISALIGNED: operand not 4-byte aligned";
        case LPY_ERR_ALIAS: return "LPY_ERR_ALIAS: C overlaps A or B";
        case LPY_ERR_UNSUPPORTED_DEVICE: return "LPY_ERR_UNSUPPORTED_DEVICE: need compute capability 10.0 (B200)";
        case LPY_ERR_OUT_OF_MEMORY: return "LPY_ERR_OUT_OF_MEMORY: scratch allocation failed";
        case LPY_ERR_CUDA: return "LPY_ERR_CUDA: CUDA error (see lpy_last_cuda_error)";
        case LPY_ERR_NOT_SUPPORTED: return "LPY_ERR_NOT_SUPPORTED: path cannot run this problem";
    }
    return "LPY_ERR_UNKNOWN";
}

int lpy_last_cuda_error(void) { return g_last_cuda_error; }

int lpy_version(void) { return LPY_VERSION; }

lpy_status lpy_select_path(int64_t M, int64_t N, int64_t K, lpy_path requested, lpy_path *chosen) {
    if (M < 0 || N < 0 || K < 0 || M > kMaxDim || N > kMaxDim || K > kMaxDim || chosen == nullptr)
        return LPY_ERR_INVALID_VALUE;
    if (requested != LPY_PATH_AUTO && requested != LPY_PATH_FFMA && requested != LPY_PATH_3XTF32)
        return LPY_ERR_INVALID_VALUE;
    *chosen = resolve_path(M, N, K, requested);
    return LPY_OK;
}

}  // extern "C"

namespace {

// lpy_gemm_f32_ex and lpy_gemm_f32_gated (gate == nullptr: ungated).
lpy_status gemm_impl(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, lpy_layout layout_a,
                     const float *B, int64_t ldb, lpy_layout layout_b, float *C, int64_t ldc,
                     lpy_layout layout_c, void *stream, lpy_path path, const lpy_gemm_opts *opts,
                     const lpy_kgate *gate) {
    Operand oa{A, M, K, lda, int(layout_a)}, ob{B, K, N, ldb, int(layout_b)}, oc{C, M, N, ldc, int(layout_c)};
    lpy_status st = validate_all(M, N, K, oa, ob, oc, int(path), opts);
    if (st != LPY_OK) return st;
    if (gate) {
        if (gate->flags == nullptr) return LPY_ERR_NULL_POINTER;
        if (reinterpret_cast<uintptr_t>(gate->flags) & 3) return LPY_ERR_MISALIGNED;
        if (gate->chunk_k < 32 || gate->chunk_k > kMaxDim) return LPY_ERR_INVALID_VALUE;
    }

    // Column-major C: C^T (N x M, row-major, ld = ldc) = B^T A^T, where the
    // transpose of a stored matrix is the same memory with the other layout tag.
    if (layout_c == LPY_COL_MAJOR) {
        Operand na{B, N, K, ldb, 1 - int(layout_b)};
        Operand nb{A, K, M, lda, 1 - int(layout_a)};
        std::swap(M, N);
        oa = na;
        ob = nb;
    }
    if (M == 0 || N == 0) return LPY_OK;  // empty domain

    DeviceInfo dev;
    if ((st = device_info(dev)) != LPY_OK) return st;
    if (opts && opts->plan_sms > dev.sms) return LPY_ERR_INVALID_VALUE;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;

    if (K == 0) {  // identity of sum: C := 0 (row-major after canonicalisation)
        e = cudaMemset2DAsync(C, size_t(ldc) * 4, 0, size_t(N) * 4, size_t(M), s);
        return e == cudaSuccess ? LPY_OK : cuda_fail(e);
    }

    const lpy_path chosen = resolve_path(M, N, K, path);

    // a tile width only the 3xTF32 kernel has: refused before anything is enqueued
    if (opts && opts->tile_n == 192 && (chosen == LPY_PATH_FFMA || !lpy::tf32_available()))
        return LPY_ERR_NOT_SUPPORTED;

    // Aligned repack (reading A7) of any operand TMA cannot describe directly:
    // one stream-ordered scratch allocation and one launch for both operands.
    lpy::RepackJob jobs[2];
    int njobs = 0;
    size_t scratch_floats = 0;
    Operand *ops[2] = {&oa, &ob};
    int64_t ld2[2] = {0, 0};
    size_t off[2] = {0, 0};
    for (int i = 0; i < 2; ++i) {
        const Operand &o = *ops[i];
        if ((reinterpret_cast<uintptr_t>(o.p) & 15) == 0 && (o.ld & 3) == 0) continue;
        if (gate) return LPY_ERR_NOT_SUPPORTED;   // the repack would read the operand before it arrives
        ld2[i] = (o.inner() + 3) & ~int64_t(3);
        off[i] = scratch_floats;
        scratch_floats += size_t(o.lines() * ld2[i]);
    }
    float *scratch = nullptr;
    if (scratch_floats > 0) {
        e = cudaMallocAsync(reinterpret_cast<void **>(&scratch), scratch_floats * 4, s);
        if (e != cudaSuccess) return cuda_fail(e);
        for (int i = 0; i < 2; ++i) {
            Operand &o = *ops[i];
            if (ld2[i] == 0) continue;
            jobs[njobs++] = lpy::RepackJob{o.p, o.ld, scratch + off[i], ld2[i], o.lines(), o.inner()};
            o.p = scratch + off[i];
            o.ld = ld2[i];
        }
        e = lpy::launch_repack(jobs, njobs, dev.sms, s);
        if (e != cudaSuccess) {
            cudaFreeAsync(scratch, s);
            return cuda_fail(e);
        }
    }

    lpy::Problem prob{int(M), int(N), int(K), oa.p, oa.ld, oa.layout, ob.p, ob.ld, ob.layout, C, ldc};
    lpy::Knobs kn{opts ? opts->num_ctas : 0, opts ? opts->raster_group : 0, opts ? opts->promote_kblocks : 0,
                  (opts && opts->plan_sms > 0) ? opts->plan_sms : dev.sms, opts ? opts->tile_n : 0, dev.sms,
                  lpy::KGate{nullptr, 0, 0, 0, 0}};
    if (gate) {
        if ((e = lpy::preload_kgate_signal()) != cudaSuccess) {
            if (scratch) cudaFreeAsync(scratch, s);
            return cuda_fail(e);
        }
        kn.gate.flags = gate->flags;
        kn.gate.chunk_k = int(gate->chunk_k);
        kn.gate.epoch = gate->epoch;
        kn.gate.timeout_ns = uint64_t(gate->timeout_ms ? gate->timeout_ms : 10000u) * 1000000ull;
        kn.gate.nchunks = int((K + gate->chunk_k - 1) / gate->chunk_k);
    }
    if (chosen == LPY_PATH_3XTF32 && !lpy::tf32_supported(prob)) {
        st = (path == LPY_PATH_3XTF32) ? LPY_ERR_NOT_SUPPORTED : LPY_OK;
        if (st == LPY_OK) e = lpy::launch_ffma(prob, kn, s);
    } else {
        e = chosen == LPY_PATH_3XTF32 ? lpy::launch_3xtf32(prob, kn, s) : lpy::launch_ffma(prob, kn, s);
    }
    if (scratch) cudaFreeAsync(scratch, s);
    if (st != LPY_OK) return st;
    return e == cudaSuccess ? LPY_OK : cuda_fail(e);
}

}  // namespace

extern "C" {

lpy_status lpy_gemm_f32_ex(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                           lpy_layout layout_a, const float *B, int64_t ldb, lpy_layout layout_b,
                           float *C, int64_t ldc, lpy_layout layout_c, void *stream, lpy_path path,
                           const lpy_gemm_opts *opts) {
    return gemm_impl(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc, layout_c, stream, path, opts, nullptr);
}

lpy_status lpy_gemm_f32_gated(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                              lpy_layout layout_a, const float *B, int64_t ldb, lpy_layout layout_b,
                              float *C, int64_t ldc, lpy_layout layout_c, void *stream, lpy_path path,
                              const lpy_gemm_opts *opts, const lpy_kgate *gate) {
    if (gate == nullptr) return LPY_ERR_NULL_POINTER;
    return gemm_impl(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc, layout_c, stream, path, opts, gate);
}

lpy_status lpy_kgate_signal(uint32_t *flag, uint32_t value, void *stream) {
    if (flag == nullptr) return LPY_ERR_NULL_POINTER;
    if (reinterpret_cast<uintptr_t>(flag) & 3) return LPY_ERR_MISALIGNED;
    DeviceInfo dev;
    lpy_status st = device_info(dev);
    if (st != LPY_OK) return st;
    const cudaError_t e = lpy::launch_kgate_signal(flag, value, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? LPY_OK : cuda_fail(e);
}

lpy_status lpy_gemm_f32(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, lpy_layout layout_a,
                        const float *B, int64_t ldb, lpy_layout layout_b, float *C, int64_t ldc,
                        lpy_layout layout_c, void *stream) {
    return lpy_gemm_f32_ex(M, N, K, A, lda, layout_a, B, ldb, layout_b, C, ldc, layout_c, stream,
                           LPY_PATH_AUTO, nullptr);
}

lpy_status lpy_gemm_f32_host(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                             lpy_layout layout_a, const float *B, int64_t ldb, lpy_layout layout_b,
                             float *C, int64_t ldc, lpy_layout layout_c, void *stream, lpy_path path) {
    Operand oa{A, M, K, lda, int(layout_a)}, ob{B, K, N, ldb, int(layout_b)}, oc{C, M, N, ldc, int(layout_c)};
    lpy_status st = validate_all(M, N, K, oa, ob, oc, int(path), nullptr);
    if (st != LPY_OK) return st;
    if (M == 0 || N == 0) return LPY_OK;
    DeviceInfo dev;
    if ((st = device_info(dev)) != LPY_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);

    // Device copies with 16-byte-aligned leading dimensions (the H2D copy does
    // the repack for free), allocated stream-ordered on the caller's stream.
    Operand *ops[3] = {&oa, &ob, &oc};
    float *dev_buf[3] = {nullptr, nullptr, nullptr};
    int64_t dev_ld[3] = {1, 1, 1};
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
        const Operand &o = *ops[i];
        dev_ld[i] = o.inner() > 0 ? (o.inner() + 3) & ~int64_t(3) : 4;
        if (o.extent() == 0) continue;
        e = cudaMallocAsync(reinterpret_cast<void **>(&dev_buf[i]), size_t(o.lines() * dev_ld[i]) * 4, s);
    }

    // Row-panel pipeline over three internal streams: H2D of B then of each A
    // panel, the panel products as their inputs land, and D2H of each C panel
    // as soon as it is computed -- so the C download and the products hide
    // under the A upload (PCIe is full duplex).  Panels are multiples of 128
    // rows (the output tile).  At n = 8192 the call is upload-bound: 537 MB at
    // the measured 53 GB/s (47.5 each way while the C download runs) is
    // ~10.7 ms of the ~11.8 ms measured; 16 vs 8 panels measured equal.
    constexpr int kMaxPanels = 16;
    // panels of >= 512 rows (multiples of 128), at most kMaxPanels: the last
    // panel's product and download are the exposed tail after the upload ends
    const int64_t prow = M <= 1024 ? M
                                   : std::max<int64_t>(512, ((M + kMaxPanels - 1) / kMaxPanels + 127) / 128 * 128);
    // Panel q covers rows [pb[q], pb[q + 1]).  The last regular panel is cut
    // into halving pieces (L/2, L/4, L/4; multiples of 128): its product and
    // download are the exposed tail after the last upload, so the tail is
    // the smallest piece's, not a whole panel's.
    int64_t pb[kMaxPanels + 3];
    int npanel = 0;
    pb[0] = 0;
    for (int64_t r = 0; r < M; r += prow) {
        const int64_t len = std::min(prow, M - r);
        if (r + len == M && M > 1024 && len >= 512) {
            const int64_t h1 = (len / 2 + 127) / 128 * 128, h2 = ((len - h1) / 2 + 127) / 128 * 128;
            pb[++npanel] = r + h1;
            pb[++npanel] = r + h1 + h2;
            pb[++npanel] = M;
        } else {
            pb[++npanel] = r + len;
        }
    }
    cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_b = nullptr, ev_done = nullptr;
    cudaEvent_t ev_a[kMaxPanels + 2] = {}, ev_c[kMaxPanels + 2] = {};
    auto mk_stream = [&](cudaStream_t *x) {
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(x, cudaStreamNonBlocking);
    };
    auto mk_event = [&](cudaEvent_t *x) {
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(x, cudaEventDisableTiming);
    };
    mk_stream(&sh); mk_stream(&sc); mk_stream(&sd);
    mk_event(&ev_fork); mk_event(&ev_b); mk_event(&ev_done);
    for (int q = 0; q < npanel; ++q) { mk_event(&ev_a[q]); mk_event(&ev_c[q]); }

    // Copy rows [r0, r1) of an M-row operand (A or C) between host and device.
    auto copy_rows = [&](int i, int64_t r0, int64_t r1, cudaMemcpyKind kind, cudaStream_t st_) {
        const Operand &o = *ops[i];
        float *host = const_cast<float *>(o.p);
        const bool row = o.layout == LPY_ROW_MAJOR;
        const int64_t cols = i == 0 ? K : N;
        if (cols == 0 || r1 <= r0) return cudaSuccess;
        float *h = host + (row ? r0 * o.ld : r0);
        float *d = dev_buf[i] + (row ? r0 * dev_ld[i] : r0);
        const int64_t inner = row ? cols : r1 - r0, lines = row ? r1 - r0 : cols;
        return kind == cudaMemcpyHostToDevice
                   ? copy_lines(d, dev_ld[i], h, o.ld, inner, lines, kind, st_)
                   : copy_lines(h, o.ld, d, dev_ld[i], inner, lines, kind, st_);
    };

    if (e == cudaSuccess) e = cudaEventRecord(ev_fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sh, ev_fork, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sc, ev_fork, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, ev_fork, 0);
    if (e == cudaSuccess && ob.extent() > 0)
        e = copy_lines(dev_buf[1], dev_ld[1], ob.p, ob.ld, ob.inner(), ob.lines(), cudaMemcpyHostToDevice, sh);
    if (e == cudaSuccess) e = cudaEventRecord(ev_b, sh);
    for (int q = 0; q < npanel && e == cudaSuccess; ++q) {
        const int64_t r0 = pb[q], r1 = pb[q + 1];
        e = copy_rows(0, r0, r1, cudaMemcpyHostToDevice, sh);
        if (e == cudaSuccess) e = cudaEventRecord(ev_a[q], sh);
    }
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sc, ev_b, 0);
    for (int q = 0; q < npanel && e == cudaSuccess && st == LPY_OK; ++q) {
        const int64_t r0 = pb[q], r1 = pb[q + 1];
        e = cudaStreamWaitEvent(sc, ev_a[q], 0);
        if (e != cudaSuccess) break;
        const bool arow = layout_a == LPY_ROW_MAJOR, crow = layout_c == LPY_ROW_MAJOR;
        const float *ap = dev_buf[0] ? dev_buf[0] + (arow ? r0 * dev_ld[0] : r0) : nullptr;
        float *cp = dev_buf[2] + (crow ? r0 * dev_ld[2] : r0);
        st = lpy_gemm_f32_ex(r1 - r0, N, K, ap, dev_ld[0], layout_a, dev_buf[1], dev_ld[1], layout_b, cp,
                             dev_ld[2], layout_c, sc, path, nullptr);
        if (st == LPY_OK) e = cudaEventRecord(ev_c[q], sc);
        if (e == cudaSuccess && st == LPY_OK) e = cudaStreamWaitEvent(sd, ev_c[q], 0);
        if (e == cudaSuccess && st == LPY_OK) e = copy_rows(2, r0, r1, cudaMemcpyDeviceToHost, sd);
    }
    // join everything back onto the caller's stream, then free and synchronise
    cudaStream_t side[3] = {sh, sc, sd};
    for (cudaStream_t x : side) {
        if (x && ev_done && cudaEventRecord(ev_done, x) == cudaSuccess) cudaStreamWaitEvent(s, ev_done, 0);
    }
    for (int i = 0; i < 3; ++i)
        if (dev_buf[i]) cudaFreeAsync(dev_buf[i], s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = e2;
    for (cudaStream_t x : side)
        if (x) cudaStreamDestroy(x);
    for (cudaEvent_t x : {ev_fork, ev_b, ev_done})
        if (x) cudaEventDestroy(x);
    for (int q = 0; q < npanel; ++q) {
        if (ev_a[q]) cudaEventDestroy(ev_a[q]);
        if (ev_c[q]) cudaEventDestroy(ev_c[q]);
    }
    if (st != LPY_OK) return st;
    return e == cudaSuccess ? LPY_OK : cuda_fail(e);
}

}  // extern "C"

// ------------------------------------------------------------------ saxpy
namespace {

constexpr int64_t kMaxSpan = int64_t(1) << 62;

// Validation shared by the device and host entry points (include/lpy.h).
lpy_status validate_saxpy(int64_t n, const float *x, int64_t incx, const float *y, int64_t incy) {
    if (n < 0 || incx < 1 || incy < 1) return LPY_ERR_INVALID_VALUE;
    if (n == 0) return LPY_OK;
    if ((n - 1) > (kMaxSpan - 1) / incx || (n - 1) > (kMaxSpan - 1) / incy) return LPY_ERR_INVALID_VALUE;
    if (x == nullptr || y == nullptr) return LPY_ERR_NULL_POINTER;
    if ((reinterpret_cast<uintptr_t>(x) & 3) || (reinterpret_cast<uintptr_t>(y) & 3)) return LPY_ERR_MISALIGNED;
    if (x == y && incx == incy) return LPY_OK;  // the same vector: y := alpha*y + y
    const uintptr_t x0 = reinterpret_cast<uintptr_t>(x), x1 = x0 + uintptr_t((n - 1) * incx + 1) * 4;
    const uintptr_t y0 = reinterpret_cast<uintptr_t>(y), y1 = y0 + uintptr_t((n - 1) * incy + 1) * 4;
    if (x0 < y1 && y0 < x1) return LPY_ERR_ALIAS;
    return LPY_OK;
}

}  // namespace

extern "C" {

lpy_status lpy_saxpy_f32(int64_t n, float alpha, const float *x, int64_t incx, float *y, int64_t incy,
                         void *stream) {
    lpy_status st = validate_saxpy(n, x, incx, y, incy);
    if (st != LPY_OK || n == 0) return st;
    DeviceInfo dev;
    if ((st = device_info(dev)) != LPY_OK) return st;
    cudaError_t e = lpy::launch_saxpy(n, alpha, x, incx, y, incy, dev.sms, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? LPY_OK : cuda_fail(e);
}

lpy_status lpy_saxpy_f32_host(int64_t n, float alpha, const float *x, int64_t incx, float *y, int64_t incy,
                              void *stream) {
    lpy_status st = validate_saxpy(n, x, incx, y, incy);
    if (st != LPY_OK || n == 0) return st;
    DeviceInfo dev;
    if ((st = device_info(dev)) != LPY_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool same = (x == y && incx == incy);
    // Packed device copies (a strided host vector is gathered by a 2-D copy of
    // 4-byte rows), in chunks pipelined over two internal streams: the upload
    // of chunk c+1 overlaps chunk c's kernel and download (PCIe is full duplex).
    float *dx = nullptr, *dy = nullptr;
    cudaError_t e = cudaSuccess;
    if (!same) e = cudaMallocAsync(reinterpret_cast<void **>(&dx), size_t(n) * 4, s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void **>(&dy), size_t(n) * 4, s);
    const int64_t nchunk = n < (int64_t(1) << 20) ? 1 : 8;
    const int64_t per = ((n + nchunk - 1) / nchunk + 3) / 4 * 4;
    cudaStream_t su = nullptr, sd = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_done = nullptr, ev_up[8] = {}, ev_k[8] = {};
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&su, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming);
    for (int c = 0; c < nchunk && e == cudaSuccess; ++c) {
        e = cudaEventCreateWithFlags(&ev_up[c], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_k[c], cudaEventDisableTiming);
    }
    auto copy = [&](float *dst, int64_t dinc, const float *src, int64_t sinc, int64_t cnt, cudaMemcpyKind kind,
                    cudaStream_t st_) {
        if (dinc == 1 && sinc == 1) return cudaMemcpyAsync(dst, src, size_t(cnt) * 4, kind, st_);
        return cudaMemcpy2DAsync(dst, size_t(dinc) * 4, src, size_t(sinc) * 4, 4, size_t(cnt), kind, st_);
    };
    if (e == cudaSuccess) e = cudaEventRecord(ev_fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(su, ev_fork, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, ev_fork, 0);
    for (int64_t c = 0; c < nchunk && e == cudaSuccess; ++c) {
        const int64_t i0 = c * per, cnt = std::min(n, i0 + per) - i0;
        if (cnt <= 0) break;
        if (!same) e = copy(dx + i0, 1, x + i0 * incx, incx, cnt, cudaMemcpyHostToDevice, su);
        if (e == cudaSuccess) e = copy(dy + i0, 1, y + i0 * incy, incy, cnt, cudaMemcpyHostToDevice, su);
        if (e == cudaSuccess) e = cudaEventRecord(ev_up[c], su);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, ev_up[c], 0);
        if (e == cudaSuccess)
            e = lpy::launch_saxpy(cnt, alpha, same ? dy + i0 : dx + i0, 1, dy + i0, 1, dev.sms, sd);
        if (e == cudaSuccess) e = copy(y + i0 * incy, incy, dy + i0, 1, cnt, cudaMemcpyDeviceToHost, sd);
    }
    for (cudaStream_t x_ : {su, sd})
        if (x_ && ev_done && cudaEventRecord(ev_done, x_) == cudaSuccess) cudaStreamWaitEvent(s, ev_done, 0);
    if (dx) cudaFreeAsync(dx, s);
    if (dy) cudaFreeAsync(dy, s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = e2;
    for (cudaStream_t x_ : {su, sd})
        if (x_) cudaStreamDestroy(x_);
    for (cudaEvent_t x_ : {ev_fork, ev_done})
        if (x_) cudaEventDestroy(x_);
    for (int c = 0; c < 8; ++c) {
        if (ev_up[c]) cudaEventDestroy(ev_up[c]);
        if (ev_k[c]) cudaEventDestroy(ev_k[c]);
    }
    return e == cudaSuccess ? LPY_OK : cuda_fail(e);
}

}  // extern "C"

// ------------------------------------------------------------------ Coulomb
namespace {

lpy_status validate_coulomb(int64_t nt, const float *t, int64_t ldt, int64_t ns, const float *s, int64_t lds,
                            const float *q, const float *phi) {
    if (nt < 0 || ns < 0 || nt > kMaxSpan / 64 || ns > kMaxSpan / 64) return LPY_ERR_INVALID_VALUE;
    if (ldt < 3 || lds < 3 || ldt > kMaxSpan / 64 || lds > kMaxSpan / 64) return LPY_ERR_INVALID_LD;
    struct Span { const float *p; int64_t n; };
    const Span spans[4] = {{t, nt > 0 ? (nt - 1) * ldt + 3 : 0}, {s, ns > 0 ? (ns - 1) * lds + 3 : 0},
                           {q, ns}, {phi, nt}};
    for (const Span &sp : spans) {
        if (sp.n == 0) continue;
        if (sp.p == nullptr) return LPY_ERR_NULL_POINTER;
        if (reinterpret_cast<uintptr_t>(sp.p) & 3) return LPY_ERR_MISALIGNED;
    }
    if (nt > 0) {
        const uintptr_t o0 = reinterpret_cast<uintptr_t>(phi), o1 = o0 + uintptr_t(nt) * 4;
        for (int k = 0; k < 3; ++k) {
            if (spans[k].n == 0) continue;
            const uintptr_t a0 = reinterpret_cast<uintptr_t>(spans[k].p), a1 = a0 + uintptr_t(spans[k].n) * 4;
            if (a0 < o1 && o0 < a1) return LPY_ERR_ALIAS;
        }
    }
    return LPY_OK;
}

}  // namespace

extern "C" {

lpy_status lpy_coulomb_f32(int64_t nt, const float *t, int64_t ldt, int64_t ns, const float *s, int64_t lds,
                           const float *q, float *phi, void *stream) {
    lpy_status st = validate_coulomb(nt, t, ldt, ns, s, lds, q, phi);
    if (st != LPY_OK || nt == 0) return st;
    DeviceInfo dev;
    if ((st = device_info(dev)) != LPY_OK) return st;
    cudaError_t e = lpy::launch_coulomb(nt, t, ldt, ns, s, lds, q, phi, dev.sms, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? LPY_OK : cuda_fail(e);
}

lpy_status lpy_coulomb_f32_host(int64_t nt, const float *t, int64_t ldt, int64_t ns, const float *s,
                                int64_t lds, const float *q, float *phi, void *stream) {
    lpy_status st = validate_coulomb(nt, t, ldt, ns, s, lds, q, phi);
    if (st != LPY_OK || nt == 0) return st;
    DeviceInfo dev;
    if ((st = device_info(dev)) != LPY_OK) return st;
    cudaStream_t sm = static_cast<cudaStream_t>(stream);
    const size_t tb = size_t(nt > 0 ? (nt - 1) * ldt + 3 : 0) * 4, sb = size_t(ns > 0 ? (ns - 1) * lds + 3 : 0) * 4;
    const size_t qb = size_t(ns) * 4, pb = size_t(nt) * 4;
    char *buf = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&buf), tb + sb + qb + pb + 64, sm);
    if (e != cudaSuccess) return cuda_fail(e);
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    float *dt = reinterpret_cast<float *>(buf);
    float *ds = reinterpret_cast<float *>(buf + al(tb));
    float *dq = reinterpret_cast<float *>(buf + al(tb) + al(sb));
    float *dp = reinterpret_cast<float *>(buf + al(tb) + al(sb) + al(qb));
    if (tb) e = cudaMemcpyAsync(dt, t, tb, cudaMemcpyHostToDevice, sm);
    if (e == cudaSuccess && sb) e = cudaMemcpyAsync(ds, s, sb, cudaMemcpyHostToDevice, sm);
    if (e == cudaSuccess && qb) e = cudaMemcpyAsync(dq, q, qb, cudaMemcpyHostToDevice, sm);
    if (e == cudaSuccess) e = lpy::launch_coulomb(nt, dt, ldt, ns, ds, lds, dq, dp, dev.sms, sm);
    if (e == cudaSuccess) e = cudaMemcpyAsync(phi, dp, pb, cudaMemcpyDeviceToHost, sm);
    cudaFreeAsync(buf, sm);
    cudaError_t e2 = cudaStreamSynchronize(sm);
    if (e == cudaSuccess) e = e2;
    return e == cudaSuccess ? LPY_OK : cuda_fail(e);
}

}  // extern "C"
