// vtrace_cb_launch.cu -- plan, tensor maps and launch of the column-block kernel
// (vtrace_cb.cuh).  Compiled twice, in parallel with vtrace_api.cu:
// -DVT_CB_PART=0 (bf16 logits, and the host plan) and -DVT_CB_PART=1 (fp32 logits).
#ifndef VT_CB_PART
#define VT_CB_PART 0
#endif
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/vtrace.h"
#include "vtrace_kernels.cuh"
#include "vtrace_rows.cuh"
#include "vtrace_cb.cuh"
#include "vtrace_cb_host.h"

namespace vtb200 {

#if VT_CB_PART == 0
// Work split of the column-block kernel on `sms` SMs (trajectories are
// independent, so blocks of columns need no exchange but the partial sums).
//   g    column groups (of 4) per logits TMA segment: 4 g A elem must be a multiple
//        of 16 bytes (bf16 with odd A: g = 2)
//   ncg  column groups per CTA = ceil(B/4 / sms) rounded up to g: one CTA per SM
//   nts  warps per column group (time slots): as many as cb_max_warps allows, at most the
//        number of 8-step chunks, spread so that the iterations are evenly filled
// False if the shape does not fit the kernel (then the look-back kernel runs).
bool cb_plan(long long T, long long B, int A, int elem, bool mu_lp, unsigned out_mask, int sms,
             CbPlan& p, bool plain) {
  std::memset(&p, 0, sizeof(p));
  if (sms <= 0 || T <= 0 || B <= 0) return false;
  int g = 1;
  if (plain) {
    // plain loads: no alignment constraint, small problems only (one warp copies the tiles)
    if (T * B * A > (1LL << 20)) return false;
  } else {
    g = ((4 * A * elem) % 16 == 0) ? 1 : (((8 * A * elem) % 16 == 0) ? 2 : 4);
    if (g > 2) return false;
    if (4 * g * A > 256) return false;           // TMA box inner dimension
    if (B % (4 * g) != 0) return false;          // the [T][B/(4g)][4gA] view is exact
  }
  if ((T + 256) * B >= (1LL << 31)) return false;  // 32-bit row arithmetic
  if (!cb_supported_a(A)) return false;
  const long long G4 = (B + 3) / 4;
  const int maxw = cb_max_warps(elem);  // the instantiation's compute warps (its register cap)
  int ncg = (int)std::min<long long>((G4 + sms - 1) / sms, maxw);
  ncg = (ncg + g - 1) / g * g;
  if (ncg > maxw) ncg -= g;
  const long long grid = (G4 + ncg - 1) / ncg;
  if (grid > (1LL << 20)) return false;
  const long long K8 = (T + 7) / 8;  // 8-step chunks
#ifndef CB_MAXNTS
#define CB_MAXNTS 14  // A/B: cap on the time slots per column group
#endif
  int nts = (int)std::max<long long>(1, std::min<long long>(std::min(maxw / ncg, CB_MAXNTS), K8));
  const long long J0 = (K8 + nts - 1) / nts;
  nts = (int)((K8 + J0 - 1) / J0);  // same number of iterations, fewest idle slots
  const int Bc = 4 * ncg;
  const auto stage_bytes = [&](int nts_) {
    const size_t Ts = 8 * (size_t)nts_;
    const size_t logit = a128((size_t)Bc * A * elem * Ts);
    const size_t step = a128((size_t)Bc * 4 * Ts);
    size_t off = 0;
    p.pi = (unsigned)off; off += logit;
    p.mu = (unsigned)off; off += mu_lp ? step : logit;
    p.a = (unsigned)off; off += step;
    p.r = (unsigned)off; off += step;
    p.gm = (unsigned)off; off += step;
    p.v = (unsigned)off; off += a128((size_t)Bc * 4 * (Ts + 1));
    const unsigned outs[6] = {OUT_DV, OUT_VS, OUT_PG, OUT_LR, OUT_LP, OUT_LM};
    unsigned* dst[6] = {&p.dv, &p.vs, &p.pg, &p.lr, &p.lp, &p.lm};
    for (int k = 0; k < 6; ++k) {
      *dst[k] = (unsigned)off;
      if (out_mask & outs[k]) off += step;
    }
    p.tx_bytes = (unsigned)((mu_lp ? Bc * A * elem * Ts + Bc * 4 * Ts : 2 * Bc * A * elem * Ts) +
                            3 * Bc * 4 * Ts + Bc * 4 * (Ts + 1));
    return off;
  };
  // shared memory: the stages, the compute warps' exps buffers (2 per warp, NP float2
  // per lane), plus ~3.5 KB of static arrays
  const size_t budget = kCbMaxDynSmem;
  const auto ebuf_bytes = [&](int nts_) {
    return CB_EBUF ? (size_t)ncg * nts_ * 2 * ((A + 1) / 2) * 32 * 8 : (size_t)0;
  };
  size_t st = stage_bytes(nts);
  while (nts > 1 && 2 * st + ebuf_bytes(nts) > budget) st = stage_bytes(--nts);
  if (2 * st + ebuf_bytes(nts) > budget) return false;
  int nstage = 4;
  while (nstage > 2 && nstage * st + ebuf_bytes(nts) > budget) --nstage;
  p.g = g; p.ncg = ncg; p.nts = nts; p.Bc = Bc; p.Ts = 8 * nts;
  p.J = (int)((T + p.Ts - 1) / p.Ts);
  p.nstage = nstage; p.grid = (int)grid; p.stage = (unsigned)st;
  p.ebuf = (unsigned)(nstage * st);
  p.smem = nstage * st + ebuf_bytes(nts);
  p.out_mask = out_mask;
  p.plain = plain ? 1 : 0;
  return true;
}

int cb_num_sms(int dev) {
  static std::atomic<int> cache[64];
  if (dev < 0 || dev >= 64) return 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}
#endif

template <typename LT, int A_CT, bool LOSS, bool GEN, bool MULP, bool PLAIN>
static vt_status cb_launch_one(const Params& P, const CbParams& C, const CbMaps& maps, int grid,
                               size_t smem, int dev, cudaStream_t st) {
  auto kern = vtrace_cb_kernel<LT, A_CT, LOSS, GEN, MULP, PLAIN>;
  // the dynamic shared-memory limit is a per-device function attribute: set once per device
  static std::atomic<unsigned long long> attr_set{0};
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kCbMaxDynSmem) != cudaSuccess)
      return VT_ERR_CUDA;
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)((C.ncg * C.nts + 1) * 32));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = P.pdl ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, kern, P, C, maps) != cudaSuccess) return VT_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}

template <typename LT, bool LOSS, bool GEN, bool MULP, bool PLAIN>
static vt_status cb_dispatch_a(const Params& P, const CbParams& C, const CbMaps& maps, int grid,
                               size_t smem, int dev, cudaStream_t st) {
  switch (P.A) {
    case 18: return cb_launch_one<LT, 18, LOSS, GEN, MULP, PLAIN>(P, C, maps, grid, smem, dev, st);
    case 9: return cb_launch_one<LT, 9, LOSS, GEN, MULP, PLAIN>(P, C, maps, grid, smem, dev, st);
    case 6: return cb_launch_one<LT, 6, LOSS, GEN, MULP, PLAIN>(P, C, maps, grid, smem, dev, st);
    case 4: return cb_launch_one<LT, 4, LOSS, GEN, MULP, PLAIN>(P, C, maps, grid, smem, dev, st);
    case 3: return cb_launch_one<LT, 3, LOSS, GEN, MULP, PLAIN>(P, C, maps, grid, smem, dev, st);
    default: return VT_ERR_SHAPE;
  }
}

template <typename LT, bool LOSS, bool GEN, bool MULP>
static vt_status cb_dispatch_p(bool plain, const Params& P, const CbParams& C, const CbMaps& maps,
                               int grid, size_t smem, int dev, cudaStream_t st) {
  return plain ? cb_dispatch_a<LT, LOSS, GEN, MULP, true>(P, C, maps, grid, smem, dev, st)
               : cb_dispatch_a<LT, LOSS, GEN, MULP, false>(P, C, maps, grid, smem, dev, st);
}

template <typename LT>
static vt_status cb_dispatch(bool loss, bool plain, const Params& P, const CbParams& C,
                             const CbMaps& maps, int grid, size_t smem, int dev, cudaStream_t st) {
  // plain V-trace from logits takes the instantiation with the variant logic compiled
  // out; behaviour log-probs (MULP) come with the general one
  const bool gen = P.correction != VT_CORRECTION_VTRACE || P.q_values != 0 || P.mu_lp != 0;
  if (loss) {
    if (P.mu_lp) return cb_dispatch_p<LT, true, true, true>(plain, P, C, maps, grid, smem, dev, st);
    if (gen) return cb_dispatch_p<LT, true, true, false>(plain, P, C, maps, grid, smem, dev, st);
    return cb_dispatch_p<LT, true, false, false>(plain, P, C, maps, grid, smem, dev, st);
  }
  if (P.mu_lp) return cb_dispatch_p<LT, false, true, true>(plain, P, C, maps, grid, smem, dev, st);
  if (gen) return cb_dispatch_p<LT, false, true, false>(plain, P, C, maps, grid, smem, dev, st);
  return cb_dispatch_p<LT, false, false, false>(plain, P, C, maps, grid, smem, dev, st);
}

#if VT_CB_PART == 0
#ifdef CB_TIMING
// timing build only (not part of the ABI): copy the per-CTA stamps of the last launch
extern "C" int vtrace_debug_cb_stamps(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, cb_stamps, sizeof(unsigned long long) * 8 * n);
}
#endif
vt_status cb_launch_bf16(bool loss, bool plain, const Params& P, const CbParams& C,
                         const CbMaps& maps, int grid, size_t smem, int dev, cudaStream_t st) {
  return cb_dispatch<__nv_bfloat16>(loss, plain, P, C, maps, grid, smem, dev, st);
}
#else
vt_status cb_launch_f32(bool loss, bool plain, const Params& P, const CbParams& C,
                        const CbMaps& maps, int grid, size_t smem, int dev, cudaStream_t st) {
  return cb_dispatch<float>(loss, plain, P, C, maps, grid, smem, dev, st);
}
#endif

}  // namespace vtb200
