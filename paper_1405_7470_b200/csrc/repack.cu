// Aligned repack of one operand (reading A7).  TMA needs a 16-byte
// aligned base and a leading dimension that is a multiple of 16 bytes; an
// operand violating either (e.g. the packed ragged config, ld = 777) is copied
// line by line into stream-ordered scratch with ld rounded up to a multiple of
// 4 floats -- the paper's "padding" data-layout transformation
// applied on the fly.  Bytes only: no arithmetic of the method happens here.
#include "lpy_internal.h"
#include "ptx.cuh"

namespace lpy {

// One thread per destination float4, flattened over both jobs' lines: the
// four source floats of a 16-byte destination chunk are scalar loads (the
// source line is only 4-byte aligned), the store is one STG.128.  REPACK_VEC
// chunks per thread, strided by the grid, put 4 * REPACK_VEC independent loads
// in flight per thread.  (The previous one-warp-per-line loop left each warp
// two dependent load/store rounds per 777-float line: 10.4 us cold for the
// ragged config's 12.4 MB, 1.2 TB/s.)  The pad columns of dst are zeroed (TMA
// never reads them: the descriptors carry the logical extent).
constexpr int REPACK_VEC = 2;
__global__ void __launch_bounds__(256) repack_kernel(RepackJob j0, RepackJob j1, int njobs) {
    pdl_wait();                 // the operands' producer (the previous grid) is done
    const int64_t n0 = j0.lines * (j0.ld_dst / 4);
    const int64_t total = n0 + (njobs > 1 ? j1.lines * (j1.ld_dst / 4) : 0);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; base < total; base += stride * REPACK_VEC) {
        float4 v[REPACK_VEC];
        float *dst[REPACK_VEC];
#pragma unroll
        for (int u = 0; u < REPACK_VEC; ++u) {
            const int64_t i = base + u * stride;
            dst[u] = nullptr;
            if (i >= total) continue;
            const bool first = i < n0;
            const RepackJob &j = first ? j0 : j1;
            const int64_t q = first ? i : i - n0, c4 = j.ld_dst / 4;
            const int64_t line = q / c4, col = (q - line * c4) * 4;
            const float *s = j.src + line * j.ld_src + col;
            v[u].x = col + 0 < j.inner ? __ldg(s + 0) : 0.f;
            v[u].y = col + 1 < j.inner ? __ldg(s + 1) : 0.f;
            v[u].z = col + 2 < j.inner ? __ldg(s + 2) : 0.f;
            v[u].w = col + 3 < j.inner ? __ldg(s + 3) : 0.f;
            dst[u] = j.dst + line * j.ld_dst + col;
        }
#pragma unroll
        for (int u = 0; u < REPACK_VEC; ++u)
            if (dst[u]) *reinterpret_cast<float4 *>(dst[u]) = v[u];
    }
    pdl_launch_dependents();
}

// Both operands' repacks (njobs = 1 or 2) in one launch.
cudaError_t launch_repack(const RepackJob *jobs, int njobs, int num_sms, cudaStream_t s) {
    int64_t chunks = 0;
    for (int i = 0; i < njobs; ++i) chunks += jobs[i].lines * (jobs[i].ld_dst / 4);
    if (njobs <= 0 || chunks <= 0) return cudaSuccess;
    int64_t blocks = (chunks + 256 * REPACK_VEC - 1) / (256 * REPACK_VEC);
    if (blocks > int64_t(num_sms) * 32) blocks = int64_t(num_sms) * 32;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(blocks));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_attr(attr, 0);
    return cudaLaunchKernelEx(&cfg, repack_kernel, jobs[0], njobs > 1 ? jobs[1] : jobs[0], njobs);
}

}  // namespace lpy
