// Instantiation unit of the fused backward for io=__nv_bfloat16, B/C=__nv_bfloat16 (parallel build).
#include "lbs_scan_bwd.cuh"

namespace lbs {
cudaError_t launch_bwd_bf16(const BwdParams& p, cudaStream_t st) { return launch_bwd_v<__nv_bfloat16, __nv_bfloat16>(p, st); }
}  // namespace lbs
