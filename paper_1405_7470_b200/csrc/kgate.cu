// lpy_kgate_signal (include/lpy.h): publish "chunk c of K has arrived" for a
// K-gated product (the row-panel product consuming B while it is broadcast,
// DESIGN.md 8).  Stream order makes every write of the work before this kernel
// (the chunk's broadcast) visible to it; the release store then publishes them
// to the product's producer warps, which acquire the flag (ptx.cuh kgate_wait).
#include "lpy_internal.h"

namespace lpy {

__global__ void kgate_signal_kernel(uint32_t *flag, uint32_t value) {
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
    }
}

// Load the signal kernel's module on the current device now.  With CUDA's lazy
// module loading a kernel's first launch loads its code, and that load waits
// for the device -- so a first signal launched while a gated product already
// spins on the flag it would set blocks until the product's deadlock detector
// traps (measured: scripts/gate_probe.py).  lpy_gemm_f32_gated calls this
// before launching the product.
cudaError_t preload_kgate_signal() {
    static std::atomic<uint64_t> done{0};   // devices already loaded
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    cudaFuncAttributes a;
    e = cudaFuncGetAttributes(&a, kgate_signal_kernel);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

cudaError_t launch_kgate_signal(uint32_t *flag, uint32_t value, cudaStream_t s) {
    kgate_signal_kernel<<<1, 32, 0, s>>>(flag, value);
    return cudaGetLastError();
}

}  // namespace lpy
