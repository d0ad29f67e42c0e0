// Instantiation unit of the fused forward for io=__nv_bfloat16, B/C=float (parallel build).
#include "lbs_scan_fwd.cuh"

namespace lbs {
cudaError_t launch_fwd_bf16f32(const FwdParams& p, cudaStream_t st) { return launch_fwd_v<__nv_bfloat16, float>(p, st); }
}  // namespace lbs
