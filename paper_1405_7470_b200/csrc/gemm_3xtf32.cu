// 3xTF32 tcgen05 path -- placeholder until the kernel lands.
#include "lpy_internal.h"

namespace lpy {
bool tf32_supported(const Problem &) { return false; }
bool tf32_available() { return false; }
cudaError_t launch_3xtf32(const Problem &, const Knobs &, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace lpy
