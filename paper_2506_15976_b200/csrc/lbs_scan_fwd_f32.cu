// Instantiation unit of the fused forward for io=float, B/C=float (parallel build).
#include "lbs_scan_fwd.cuh"

namespace lbs {
cudaError_t launch_fwd_f32(const FwdParams& p, cudaStream_t st) { return launch_fwd_v<float, float>(p, st); }
}  // namespace lbs
