// decode_fast.cu — placeholder until the persistent sm_100a kernel lands.
#include "decode_common.cuh"

namespace df11 {
bool fast_supports(const df11_device_tensor &) { return false; }
cudaError_t launch_fast(const Batch &, int, cudaStream_t, uint64_t *) { return cudaErrorNotSupported; }
}  // namespace df11
