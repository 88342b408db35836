// Aligned repack of one operand (reading A7).  TMA needs a 16-byte
// aligned base and a leading dimension that is a multiple of 16 bytes; an
// operand violating either (e.g. the packed ragged config, ld = 777) is copied
// line by line into stream-ordered scratch with ld rounded up to a multiple of
// 4 floats -- the paper's "padding" data-layout transformation
// applied on the fly.  Bytes only: no arithmetic of the method happens here.
#include "lpy_internal.h"

namespace lpy {

__global__ void repack_kernel(const float *__restrict__ src, int64_t ld_src, float *__restrict__ dst,
                              int64_t ld_dst, int64_t lines, int64_t inner) {
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        const float *s = src + line * ld_src;
        float *d = dst + line * ld_dst;
        for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < ld_dst;
             e += int64_t(gridDim.x) * blockDim.x)
            d[e] = e < inner ? s[e] : 0.f;   // pad the tail of each line with zeros
    }
}

cudaError_t launch_repack(const float *src, int64_t ld_src, float *dst, int64_t ld_dst, int64_t lines,
                          int64_t inner, cudaStream_t s) {
    if (lines <= 0 || inner <= 0) return cudaSuccess;
    const int threads = 256;
    int64_t gx = (ld_dst + threads - 1) / threads;
    if (gx > 64) gx = 64;
    int64_t gy = lines < 65535 ? lines : 65535;
    repack_kernel<<<dim3(unsigned(gx), unsigned(gy)), threads, 0, s>>>(src, ld_src, dst, ld_dst, lines,
                                                                       inner);
    return cudaGetLastError();
}

}  // namespace lpy
