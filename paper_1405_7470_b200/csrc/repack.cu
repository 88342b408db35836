// Aligned repack of one operand (reading A7).  TMA needs a 16-byte
// aligned base and a leading dimension that is a multiple of 16 bytes; an
// operand violating either (e.g. the packed ragged config, ld = 777) is copied
// line by line into stream-ordered scratch with ld rounded up to a multiple of
// 4 floats -- the paper's "padding" data-layout transformation
// applied on the fly.  Bytes only: no arithmetic of the method happens here.
#include "lpy_internal.h"

namespace lpy {

// One warp per line (grid-stride over lines): 32 consecutive 4-byte loads and
// stores per instruction, so even short lines (the ragged config's 777 floats)
// move at full coalescing; the grid fills every SM once.
__global__ void __launch_bounds__(256) repack_kernel(const float *__restrict__ src, int64_t ld_src,
                                                     float *__restrict__ dst, int64_t ld_dst, int64_t lines,
                                                     int64_t inner) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t line = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); line < lines;
         line += warps) {
        const float *s = src + line * ld_src;
        float *d = dst + line * ld_dst;
        for (int64_t e = lane; e < ld_dst; e += 32) d[e] = e < inner ? s[e] : 0.f;   // zero the pad
    }
}

cudaError_t launch_repack(const float *src, int64_t ld_src, float *dst, int64_t ld_dst, int64_t lines,
                          int64_t inner, cudaStream_t s) {
    if (lines <= 0 || inner <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (lines + 7) / 8;
    if (blocks > int64_t(sms) * 8) blocks = int64_t(sms) * 8;
    repack_kernel<<<unsigned(blocks), 256, 0, s>>>(src, ld_src, dst, ld_dst, lines, inner);
    return cudaGetLastError();
}

}  // namespace lpy
