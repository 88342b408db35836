// Aligned repack of one operand (reading A7).  TMA needs a 16-byte
// aligned base and a leading dimension that is a multiple of 16 bytes; an
// operand violating either (e.g. the packed ragged config, ld = 777) is copied
// line by line into stream-ordered scratch with ld rounded up to a multiple of
// 4 floats -- the paper's "padding" data-layout transformation
// applied on the fly.  Bytes only: no arithmetic of the method happens here.
#include "lpy_internal.h"
#include "ptx.cuh"

namespace lpy {

// One warp per line (grid-stride over lines): 32 consecutive 4-byte loads and
// stores per instruction, so even short lines (the ragged config's 777 floats)
// move at full coalescing, and UNROLL loads in flight per lane before their
// stores (a load / store chain per element would leave each warp waiting one
// memory latency per 128 bytes).  The pad columns of dst are zeroed (TMA never
// reads them: the descriptors carry the logical extent).
constexpr int REPACK_UNROLL = 16;
__global__ void __launch_bounds__(256) repack_kernel(RepackJob j0, RepackJob j1, int njobs) {
    pdl_wait();                 // the operands' producer (the previous grid) is done
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    const int64_t total = j0.lines + (njobs > 1 ? j1.lines : 0);
    for (int64_t gl = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); gl < total; gl += warps) {
        const bool first = gl < j0.lines;
        const RepackJob &j = first ? j0 : j1;
        const int64_t line = first ? gl : gl - j0.lines;
        const float *s = j.src + line * j.ld_src;
        float *d = j.dst + line * j.ld_dst;
        for (int64_t e0 = lane; e0 < j.ld_dst; e0 += 32 * REPACK_UNROLL) {
            float v[REPACK_UNROLL];
#pragma unroll
            for (int k = 0; k < REPACK_UNROLL; ++k) {
                const int64_t e = e0 + 32 * k;
                v[k] = e < j.inner ? __ldg(s + e) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < REPACK_UNROLL; ++k) {
                const int64_t e = e0 + 32 * k;
                if (e < j.ld_dst) d[e] = v[k];
            }
        }
    }
    pdl_launch_dependents();
}

// Both operands' repacks (njobs = 1 or 2) in one launch.
cudaError_t launch_repack(const RepackJob *jobs, int njobs, int num_sms, cudaStream_t s) {
    int64_t lines = 0;
    for (int i = 0; i < njobs; ++i) lines += jobs[i].lines;
    if (njobs <= 0 || lines <= 0) return cudaSuccess;
    int64_t blocks = (lines + 7) / 8;
    if (blocks > int64_t(num_sms) * 8) blocks = int64_t(num_sms) * 8;
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
