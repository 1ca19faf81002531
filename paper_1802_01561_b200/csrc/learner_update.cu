// learner_update.cu -- the learner's parameter update after the network backward
// (SURVEY.md 8(f) NEXT #4): global-norm clip and RMSProp with momentum 0
// (P:838), TF form with epsilon inside the square root (DESIGN.md r9):
//     g' = g * c / max(||g||_2, c)            (c = max_global_norm; reading r10)
//     ms <- decay * ms + (1 - decay) * g'^2
//     theta <- theta - lr * g' / sqrt(ms + epsilon)
//
// One cooperative launch, one CTA per SM (co-resident by construction):
//   phase 1  every CTA sums g^2 of its contiguous slice in fp64 (fixed strides, a
//            fixed tree) and publishes it as an epoch-tagged 16-byte record; every
//            CTA then reads all records in index order -> the same ||g|| bitwise in
//            every CTA, no second pass over memory and no atomics on the data path;
//   phase 2  the clip scale and the RMSProp update of the slice (its g re-read hits
//            L2: the slice was streamed moments ago), IEEE sqrt and division.
// HBM traffic per parameter: g 4 B read, ms 4+4 B, theta 4+4 B = 20 B.
// Data-parallel learners: the caller all-reduces (SUM) the gradient first
// (paper_1802_01561_b200/learner.py, NCCL); every learner then applies the same
// update to its replica (reading r11).

#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "vtrace.h"
#include "vtrace_kernels.cuh"

namespace vtb200 {

constexpr int RMS_THREADS = 512;
constexpr int RMS_MAX_CTAS = 1024;
constexpr size_t RMS_RECS_OFF = 256;

struct RmsHeader {  // workspace bytes [0, 8); vtrace_workspace_init zeroes it
  unsigned int epoch;   // calls completed (tags this call's records with epoch + 1)
  unsigned int ticket;  // CTAs done with phase 1 (the last one bumps the epoch)
};

struct RmsArgs {
  long long n;
  float* theta;
  float* ms;
  const float* g;
  float lr, decay, eps, clip;
  double* norm_out;
  unsigned char* ws;
};

__device__ __forceinline__ void rms_update(float& th, float& m, float gv, float scale,
                                           const RmsArgs& a) {
  const float gg = gv * scale;
  m = fmaf(a.decay, m, (1.f - a.decay) * (gg * gg));
  th = th - __fdiv_rn(a.lr * gg, __fsqrt_rn(m + a.eps));
}

template <bool VEC>
__global__ void __launch_bounds__(RMS_THREADS, 1) rmsprop_kernel(const RmsArgs a) {
  __shared__ double red[RMS_THREADS / 32];
  __shared__ double s_total;
  RmsHeader* hdr = reinterpret_cast<RmsHeader*>(a.ws);
  TagRec* recs = reinterpret_cast<TagRec*>(a.ws + RMS_RECS_OFF);
  const int S = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const unsigned int epoch = *reinterpret_cast<volatile unsigned int*>(&hdr->epoch);
  const unsigned long long tag = (unsigned long long)epoch + 1ull;
  // the CTA's slice [lo, hi) in units of float4 (VEC) or floats; the n % 4 tail of
  // the vector path belongs to the last CTA
  const long long units = VEC ? a.n / 4 : a.n;
  const long long per = (units + S - 1) / S;
  const long long lo = min(units, (long long)cta * per), hi = min(units, lo + per);
  const long long tail0 = VEC ? units * 4 : a.n;
  const bool has_tail = VEC && cta == S - 1;

  // ---- phase 1: sum of squares (fp64; "global gradient norm") ----
  double ss = 0.0;
  if constexpr (VEC) {
    const float4* g4 = reinterpret_cast<const float4*>(a.g);
#pragma unroll 4
    for (long long i = lo + tid; i < hi; i += RMS_THREADS) {
      const float4 v = __ldg(g4 + i);
      ss = fma((double)v.x, (double)v.x, ss);
      ss = fma((double)v.y, (double)v.y, ss);
      ss = fma((double)v.z, (double)v.z, ss);
      ss = fma((double)v.w, (double)v.w, ss);
    }
  } else {
    for (long long i = lo + tid; i < hi; i += RMS_THREADS) {
      const double v = (double)__ldg(a.g + i);
      ss = fma(v, v, ss);
    }
  }
  if (has_tail) {
    for (long long i = tail0 + tid; i < a.n; i += RMS_THREADS) {
      const double v = (double)__ldg(a.g + i);
      ss = fma(v, v, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) red[w] = ss;
  __syncthreads();
  if (w == 0) {
    double x = lane < RMS_THREADS / 32 ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) st_tag16(recs + cta, x, tag);  // (value, tag) in one 16-byte store
    // every CTA adds all CTAs' sums in index order (lane l: l, l + 32, ...), then a
    // fixed tree: the same total in every CTA
    double tot = 0.0;
    for (int c = lane; c < S; c += 32) {
      double v;
      unsigned long long t;
      while (true) {
        ld_tag16(recs + c, v, t);
        if (t == tag) break;
        __nanosleep(64);
      }
      tot += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) {
      s_total = tot;
      // re-arm: every CTA has published (we read all records), so all have read
      // the epoch; the last to get here starts the next call's epoch
      const unsigned int prev = atomicAdd(&hdr->ticket, 1u);
      if (prev == (unsigned int)(S - 1)) {
        hdr->ticket = 0u;
        hdr->epoch = epoch + 1u;
      }
    }
  }
  __syncthreads();
  const double norm = sqrt(s_total);
  // clip scale c / max(||g||, c) in fp64 (reading r10); 1 when disabled
  const float scale =
      (a.clip > 0.f && norm > (double)a.clip) ? (float)((double)a.clip / norm) : 1.f;
  if (cta == 0 && tid == 0 && a.norm_out) *a.norm_out = norm;

  // ---- phase 2: RMSProp, momentum 0 ----
  if constexpr (VEC) {
    const float4* g4 = reinterpret_cast<const float4*>(a.g);
    float4* t4 = reinterpret_cast<float4*>(a.theta);
    float4* m4 = reinterpret_cast<float4*>(a.ms);
#pragma unroll 2
    for (long long i = lo + tid; i < hi; i += RMS_THREADS) {
      const float4 gv = __ldg(g4 + i);
      float4 th = __ldcs(t4 + i), m = __ldcs(m4 + i);
      rms_update(th.x, m.x, gv.x, scale, a);
      rms_update(th.y, m.y, gv.y, scale, a);
      rms_update(th.z, m.z, gv.z, scale, a);
      rms_update(th.w, m.w, gv.w, scale, a);
      __stcs(t4 + i, th);
      __stcs(m4 + i, m);
    }
  } else {
    for (long long i = lo + tid; i < hi; i += RMS_THREADS) {
      float th = a.theta[i], m = a.ms[i];
      rms_update(th, m, __ldg(a.g + i), scale, a);
      a.theta[i] = th;
      a.ms[i] = m;
    }
  }
  if (has_tail) {
    for (long long i = tail0 + tid; i < a.n; i += RMS_THREADS) {
      float th = a.theta[i], m = a.ms[i];
      rms_update(th, m, __ldg(a.g + i), scale, a);
      a.theta[i] = th;
      a.ms[i] = m;
    }
  }
}

static int rms_num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

static bool al(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

}  // namespace vtb200

using namespace vtb200;

extern "C" {

size_t vtrace_rmsprop_workspace_bytes(int64_t n) {
  if (n < 0) return 0;
  return RMS_RECS_OFF + (size_t)RMS_MAX_CTAS * sizeof(TagRec);
}

vt_status vtrace_rmsprop_step(int64_t n, float* params, float* mean_square, const float* grads,
                              const vt_rmsprop_params* prm, double* global_norm_out,
                              void* workspace, size_t workspace_bytes, vt_stream_t stream) {
  if (!prm || (n > 0 && (!params || !mean_square || !grads))) return VT_ERR_INVALID_ARG;
  if (n < 0) return VT_ERR_SHAPE;
  const float lr = prm->learning_rate, decay = prm->decay, eps = prm->epsilon,
              clip = prm->max_global_norm;
  if (!(lr > 0.f) || !isfinite(lr) || !(decay >= 0.f && decay < 1.f) || !(eps > 0.f) ||
      !isfinite(eps) || !(clip >= 0.f) || !isfinite(clip))
    return VT_ERR_PARAM;
  if (!al(params, 4) || !al(mean_square, 4) || !al(grads, 4) ||
      (global_norm_out && !al(global_norm_out, 8)))
    return VT_ERR_ALIGNMENT;
  if (!workspace || !al(workspace, 256) || workspace_bytes < vtrace_rmsprop_workspace_bytes(n))
    return VT_ERR_WORKSPACE;
  int dev = 0, maj = 0, mnr = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
    return VT_ERR_CUDA;
  if (!(maj == 10 && mnr == 0)) return VT_ERR_DEVICE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (n == 0) {  // nothing to update; the norm of an empty gradient is 0
    if (global_norm_out && cudaMemsetAsync(global_norm_out, 0, sizeof(double), st) != cudaSuccess)
      return VT_ERR_CUDA;
    return VT_OK;
  }
  const bool vec = al(params, 16) && al(mean_square, 16) && al(grads, 16);
  const long long units = vec ? n / 4 : n;
  const int sms = rms_num_sms();
  if (sms <= 0) return VT_ERR_CUDA;
  // at least 4 units per thread before a CTA is added; at most one CTA per SM
  long long want = (units + (long long)RMS_THREADS * 4 - 1) / ((long long)RMS_THREADS * 4);
  const int S = (int)std::max(1LL, std::min<long long>(want, std::min(sms, RMS_MAX_CTAS)));
  RmsArgs a;
  a.n = n; a.theta = params; a.ms = mean_square; a.g = grads;
  a.lr = lr; a.decay = decay; a.eps = eps; a.clip = clip;
  a.norm_out = global_norm_out;
  a.ws = static_cast<unsigned char*>(workspace);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S);
  cfg.blockDim = dim3(RMS_THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (phase-1 exchange)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = vec ? cudaLaunchKernelEx(&cfg, rmsprop_kernel<true>, a)
                            : cudaLaunchKernelEx(&cfg, rmsprop_kernel<false>, a);
  return e == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}

}  // extern "C"
