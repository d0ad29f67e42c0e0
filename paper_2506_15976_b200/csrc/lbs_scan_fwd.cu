// Fused LB selective scan forward: dtype dispatch (kernels in lbs_scan_fwd.cuh,
// one instantiation unit per dtype combination so nvcc runs them in parallel).
#include "lbs_internal.h"
#include "../../include/lbscan_b200.h"

#ifndef LBS_FWD_TMA
#define LBS_FWD_TMA 1
#endif
#define LBS_FWD_TMA_ENABLED (LBS_FWD_TMA != 0)

namespace lbs {
cudaError_t launch_fwd_f32(const FwdParams& p, cudaStream_t st);
cudaError_t launch_fwd_bf16(const FwdParams& p, cudaStream_t st);
cudaError_t launch_fwd_bf16f32(const FwdParams& p, cudaStream_t st);

bool fwd_tma_enabled() { return LBS_FWD_TMA_ENABLED; }

cudaError_t launch_fwd(const FwdParams& p, int io_dtype, int bc_dtype, cudaStream_t st) {
  if (io_dtype == LBS_F32 && bc_dtype == LBS_F32) return launch_fwd_f32(p, st);
  if (io_dtype == LBS_BF16 && bc_dtype == LBS_BF16) return launch_fwd_bf16(p, st);
  if (io_dtype == LBS_BF16 && bc_dtype == LBS_F32) return launch_fwd_bf16f32(p, st);
  return cudaErrorInvalidValue;
}
}  // namespace lbs
