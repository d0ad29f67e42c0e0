// Instantiation unit of the fused backward for io=float, B/C=float (parallel build).
#include "lbs_scan_bwd.cuh"

namespace lbs {
cudaError_t launch_bwd_f32(const BwdParams& p, cudaStream_t st) { return launch_bwd_v<float, float>(p, st); }
}  // namespace lbs
