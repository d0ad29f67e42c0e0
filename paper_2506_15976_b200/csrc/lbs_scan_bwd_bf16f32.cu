// Instantiation unit of the fused backward for io=__nv_bfloat16, B/C=float (parallel build).
#include "lbs_scan_bwd.cuh"

namespace lbs {
cudaError_t launch_bwd_bf16f32(const BwdParams& p, cudaStream_t st) { return launch_bwd_v<__nv_bfloat16, float>(p, st); }
}  // namespace lbs
