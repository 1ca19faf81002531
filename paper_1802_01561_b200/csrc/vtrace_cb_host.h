// vtrace_cb_host.h -- host entry points of the column-block kernel, defined in
// vtrace_cb_launch.cu (a separate translation unit, compiled in parallel).
#pragma once
#include <cuda_runtime.h>

#include "vtrace_kernels.cuh"
#include "vtrace_cb.cuh"

namespace vtb200 {

struct CbPlan {
  int g, ncg, nts, Bc, Ts, J, nstage, grid;
  unsigned pi, mu, a, r, gm, v, dv, vs, pg, lr, lp, lm, stage, tx_bytes, out_mask, ebuf;
  size_t smem;
  int plain;  // 1: plain-load producer (no TMA)
};

// Dynamic shared memory of one column-block CTA: the stages (+ ~9 KB of static arrays,
// within the 227 KB per-CTA opt-in limit)
constexpr size_t kCbMaxDynSmem = kMaxSmem - 12 * 1024;

// Compile-time action counts the column-block kernel is instantiated for.
inline bool cb_supported_a(long long A) { return A == 3 || A == 4 || A == 6 || A == 9 || A == 18; }

// Work split for (T, B, A, elem) on `sms` SMs; false if the kernel does not apply.
bool cb_plan(long long T, long long B, int A, int elem, bool mu_lp, unsigned out_mask, int sms,
             CbPlan& p, bool plain = false);

int cb_num_sms(int dev);  // SM count of device `dev` (cached per device)

// Validation of the method parameters shared by every V-trace entry point (vtrace_api.cu).
vt_status check_params(const vt_vtrace_params* p);

vt_status cb_launch_bf16(bool loss, bool plain, const Params& P, const CbParams& C,
                         const CbMaps& maps, int grid, size_t smem, int dev, cudaStream_t st);
vt_status cb_launch_f32(bool loss, bool plain, const Params& P, const CbParams& C,
                        const CbMaps& maps, int grid, size_t smem, int dev, cudaStream_t st);

}  // namespace vtb200
