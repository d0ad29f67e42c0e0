// Instantiation unit of the fused forward for io=__nv_bfloat16, B/C=__nv_bfloat16 (parallel build).
#include "lbs_scan_fwd.cuh"

namespace lbs {
cudaError_t launch_fwd_bf16(const FwdParams& p, cudaStream_t st) { return launch_fwd_v<__nv_bfloat16, __nv_bfloat16>(p, st); }
}  // namespace lbs
