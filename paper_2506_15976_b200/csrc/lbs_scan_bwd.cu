// Fused LB selective scan backward: dtype dispatch (kernels in lbs_scan_bwd.cuh,
// one instantiation unit per dtype combination).
#include "lbs_internal.h"
#include "../../include/lbscan_b200.h"

namespace lbs {
cudaError_t launch_bwd_f32(const BwdParams& p, cudaStream_t st);
cudaError_t launch_bwd_bf16(const BwdParams& p, cudaStream_t st);
cudaError_t launch_bwd_bf16f32(const BwdParams& p, cudaStream_t st);

// backward chunk = whole LB tiles fitting the 8- (m <= 8) or 16-step register window
int bwd_chunk_len(int m) {
  const int kt = m <= 8 ? 8 : 16;
  return (kt / m) * m;
}

cudaError_t launch_bwd(const BwdParams& p, int io_dtype, int bc_dtype, cudaStream_t st) {
  if (io_dtype == LBS_F32 && bc_dtype == LBS_F32) return launch_bwd_f32(p, st);
  if (io_dtype == LBS_BF16 && bc_dtype == LBS_BF16) return launch_bwd_bf16(p, st);
  if (io_dtype == LBS_BF16 && bc_dtype == LBS_F32) return launch_bwd_bf16f32(p, st);
  return cudaErrorInvalidValue;
}
}  // namespace lbs
