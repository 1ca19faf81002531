// vtrace_ct_launch.cu -- the column-task kernels (vtrace_ct.cuh) and their launch.
// Compiled twice, in parallel with vtrace_api.cu: -DVT_CT_PART=0 (bf16 logits, and
// the shared host helpers) and -DVT_CT_PART=1 (fp32 logits).
#ifndef VT_CT_PART
#define VT_CT_PART 0
#endif
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "../../include/vtrace.h"
#include "vtrace_kernels.cuh"
#include "vtrace_rows.cuh"
#include "vtrace_ct.cuh"
#include "vtrace_ct_host.h"

namespace vtb200 {

#if VT_CT_PART == 0
int ct_num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// Work split of the balanced kernel (one CTB_WARPS-warp CTA per SM): f whole tasks
// per SM sub-partition (f4 = 4 f warps per CTA), the remaining R tasks cut into
// `segs` time segments, `tpc` cut tasks per CTA; chosen to minimise the largest
// per-sub-partition load f + ceil(segs tpc / 4) / segs.  False if it does not fit.
bool ct_plan_balanced(CtParams& C, int S) {
  const char* e = getenv("VTRACE_CT_BALANCED");  // "0": one-warp CTAs (A/B, tests)
  if ((e && e[0] == '0') || S <= 0) return false;
  if ((size_t)CTB_WARPS * C.warp_bytes > kMaxSmem) return false;  // e.g. fp32 logits, A = 18
  const long long N = C.tasks;
  const int f = (int)std::min<long long>(N / (4LL * S), 4);
  if (f < 1) return false;
  const long long R = N - 4LL * f * S;
  if (R == 0) {
    C.f4 = 4 * f; C.segs = 1; C.seg_len = C.K; C.tpc = 0;
    return true;
  }
  const int tpc = (int)((R + S - 1) / S);
  // one-warp CTAs put ceil(N / S) tasks on an SM, i.e. ceil(that / 4) on its busiest
  // sub-partition: the balanced split must beat that; and a task is cut into at most
  // 2 segments (a longer chain serialises its segments' hand-overs; measured slower)
  const double one_warp_max = (double)((((N + S - 1) / S) + 3) / 4);
  double best = one_warp_max - 0.01;
  int best_p = 0;
  for (int segs = 1; segs <= 2 && segs <= C.K; ++segs) {
    if (4 * f + segs * tpc > CTB_WARPS) continue;
    // every segment non-empty (a later one waits for the carry of an earlier one)
    const int sl = (C.K + segs - 1) / segs;
    if ((segs - 1) * sl >= C.K) continue;
    const double load = f + (double)((segs * tpc + 3) / 4) / segs;
    if (load < best - 1e-9) { best = load; best_p = segs; }
  }
  if (best_p == 0) return false;
  C.f4 = 4 * f; C.segs = best_p; C.tpc = tpc;
  C.seg_len = (C.K + best_p - 1) / best_p;
  return true;
}

#endif

// Launch, as a programmatic dependent of the previous kernel on the stream when
// `pdl` (vt_vtrace_params.overlap_previous): the kernel waits (griddepcontrol.wait)
// before its first global write.
template <typename Kern>
static vt_status launch_maybe_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                  bool pdl, const Params& P, const CtParams& C,
                                  const TmaMaps& maps) {
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, kern, P, C, maps) != cudaSuccess) return VT_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}

// VTRACE_RESERVE_SMS=r: the balanced kernel uses S - r SMs (leaves r for a concurrent
// collective, e.g. the per-step NCCL all-reduce with overlapped steps; bench.py, N > 1)
static int reserve_sms() {
  const char* e = getenv("VTRACE_RESERVE_SMS");
  const int r = (e && *e) ? atoi(e) : 0;
  return r < 0 ? 0 : (r > 16 ? 16 : r);
}

template <typename LT, int A_CT, bool LOSS, int MODE, bool GEN, bool MULP>
static vt_status ct_launch_one(const Params& P, CtParams C, const TmaMaps& maps,
                               cudaStream_t st) {
  const int S = ct_num_sms() - reserve_sms();
  if (ct_plan_balanced(C, S)) {
    auto kern = vtrace_ctb_kernel<LT, A_CT, LOSS, MODE, GEN, MULP>;
    const size_t smem = (size_t)CTB_WARPS * C.warp_bytes;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
      attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
    });
    if (attr_err != cudaSuccess || smem > kMaxSmem) return VT_ERR_CUDA;
    return launch_maybe_pdl(kern, dim3(S), dim3(CTB_WARPS * 32), smem, st, P.pdl != 0, P, C,
                            maps);
  }
  auto kern = vtrace_ct_kernel<LT, A_CT, LOSS, MODE, GEN, MULP>;
  const size_t smem = (size_t)CT_WARPS * C.warp_bytes;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
    // one-warp CTAs: occupancy is set by shared memory, so take the largest carveout
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      cudaSharedmemCarveoutMaxShared);
  });
  if (attr_err != cudaSuccess || smem > kMaxSmem) return VT_ERR_CUDA;
  const unsigned grid = (unsigned)((C.tasks + CT_WARPS - 1) / CT_WARPS);
  return launch_maybe_pdl(kern, dim3(grid), dim3(CT_WARPS * 32), smem, st, P.pdl != 0, P, C,
                          maps);
}

template <typename LT, bool LOSS, int MODE, bool GEN, bool MULP>
static vt_status ct_dispatch_a(const Params& P, const CtParams& C, const TmaMaps& maps,
                               cudaStream_t st) {
  if (P.A == 18) return ct_launch_one<LT, 18, LOSS, MODE, GEN, MULP>(P, C, maps, st);
  if (P.A == 9) return ct_launch_one<LT, 9, LOSS, MODE, GEN, MULP>(P, C, maps, st);
  return ct_launch_one<LT, 0, LOSS, MODE, GEN, MULP>(P, C, maps, st);
}

template <typename LT, bool LOSS>
static vt_status ct_dispatch(const Params& P, const CtParams& C, const TmaMaps& maps,
                             cudaStream_t st) {
  // plain V-trace with behaviour logits takes the instantiation with the variant
  // logic compiled out; behaviour log-probs (MULP) come with the general one
  const bool gen = P.correction != VT_CORRECTION_VTRACE || P.q_values != 0 || P.mu_lp != 0;
  if (exp_mode() == EXP_MUFU) {
    if (P.mu_lp) return ct_dispatch_a<LT, LOSS, EXP_MUFU, true, true>(P, C, maps, st);
    if (gen) return ct_dispatch_a<LT, LOSS, EXP_MUFU, true, false>(P, C, maps, st);
    return ct_dispatch_a<LT, LOSS, EXP_MUFU, false, false>(P, C, maps, st);
  }
  if (P.mu_lp) return ct_dispatch_a<LT, LOSS, EXP_F64, true, true>(P, C, maps, st);
  return ct_dispatch_a<LT, LOSS, EXP_F64, true, false>(P, C, maps, st);
}

// each object instantiates one logits dtype (VT_CT_PART 0: bf16, 1: fp32)
#if VT_CT_PART == 0
vt_status ct_launch_bf16(bool loss, const Params& P, const CtParams& C, const TmaMaps& maps,
                         cudaStream_t st) {
  return loss ? ct_dispatch<__nv_bfloat16, true>(P, C, maps, st)
              : ct_dispatch<__nv_bfloat16, false>(P, C, maps, st);
}
#else
vt_status ct_launch_f32(bool loss, const Params& P, const CtParams& C, const TmaMaps& maps,
                        cudaStream_t st) {
  return loss ? ct_dispatch<float, true>(P, C, maps, st) : ct_dispatch<float, false>(P, C, maps, st);
}
#endif

}  // namespace vtb200
