// vtrace_ct_host.h -- host entry points of the column-task kernels, defined in
// vtrace_ct_launch.cu (a separate translation unit, compiled in parallel).
#pragma once
#include <cuda_runtime.h>

#include "vtrace_kernels.cuh"
#include "vtrace_ct.cuh"

namespace vtb200 {

// The balanced (one 16-warp CTA per SM) work split for C.tasks / C.K / C.warp_bytes
// on S SMs; false if it does not apply (then one-warp CTAs are used).
bool ct_plan_balanced(CtParams& C, int S);

int ct_num_sms();  // SM count of the current device (cached)

// Launch the column-task kernel (balanced or one-warp CTAs) for bf16 / fp32 logits,
// loss or from_logits mode, on stream st.
vt_status ct_launch_bf16(bool loss, const Params& P, const CtParams& C, const TmaMaps& maps,
                         cudaStream_t st);
vt_status ct_launch_f32(bool loss, const Params& P, const CtParams& C, const TmaMaps& maps,
                        cudaStream_t st);
inline vt_status ct_launch(bool bf16, bool loss, const Params& P, const CtParams& C,
                           const TmaMaps& maps, cudaStream_t st) {
  return bf16 ? ct_launch_bf16(loss, P, C, maps, st) : ct_launch_f32(loss, P, C, maps, st);
}

}  // namespace vtb200
