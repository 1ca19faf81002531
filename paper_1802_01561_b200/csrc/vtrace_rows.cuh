// vtrace_rows.cuh -- row arithmetic shared by the look-back kernel (vtrace_api.cu)
// and the column-block kernel (vtrace_cb.cuh), plus small shared constants.
#pragma once

#include "../../include/vtrace.h"
#include "vtrace_kernels.cuh"

namespace vtb200 {

__host__ __device__ inline size_t a128(size_t x) { return (x + 127) & ~size_t(127); }
__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

constexpr size_t kMaxSmem = 220 * 1024;  // dynamic shared memory bound of every launch

// ---------------------------------------------------------------------------
// Row arithmetic.  Each thread owns one row
// (t, b) of the unit for the whole unit: it keeps the target row in registers
// from the statistics phase to the gradient epilogue.

template <typename T>
__device__ __forceinline__ T store_cvt(float x);
template <>
__device__ __forceinline__ float store_cvt<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 store_cvt<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// A logits row held in registers as fp32 (compile-time A, unpacked once) or
// read from shared memory (A_CT == 0).
template <typename LT, int A_CT>
struct RowRegs {
  static constexpr bool kPacked = (sizeof(LT) == 2) && (A_CT % 2 == 0) && (A_CT > 0);
  static constexpr int kN = A_CT > 0 ? A_CT : 1;
  float z[kN];
  const LT* src;
  __device__ __forceinline__ void load(const LT* row) {
    src = row;
    if constexpr (kPacked) {
      const uint32_t* p = reinterpret_cast<const uint32_t*>(row);
#pragma unroll
      for (int k = 0; k < A_CT / 2; ++k) {
        const uint32_t x = p[k];
        z[2 * k] = __uint_as_float(x << 16);
        z[2 * k + 1] = __uint_as_float(x & 0xffff0000u);
      }
    } else if constexpr (A_CT > 0) {
      if constexpr (sizeof(LT) == 4 && (A_CT % 2) == 0) {
        const float2* p = reinterpret_cast<const float2*>(row);
#pragma unroll
        for (int k = 0; k < A_CT / 2; ++k) {
          const float2 x = p[k];
          z[2 * k] = x.x;
          z[2 * k + 1] = x.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < A_CT; ++j) z[j] = Elem<LT>::get(row, j);
      }
    }
  }
  __device__ __forceinline__ float get(int j) const {  // j compile-time in unrolled loops
    if constexpr (A_CT > 0) {
      return z[j];
    } else {
      return Elem<LT>::get(src, j);
    }
  }
};

// Statistics of one logits row: m = max z, S = sum_j exp(z_j - m) (accurate to
// ~1e-8 relative), xa = z_a - m (exact, fp64), ea_f = exp(z_a - m) (fp32; it is
// exactly 1 when a is the argmax), and sed = sum_j e_j (z_j - m) (for the
// entropy, fp32).
template <typename LT, int A_CT, int MODE>
__device__ __forceinline__ void row_stats(const RowRegs<LT, A_CT>& R, int A, int a, float& m,
                                          double& S, double& xa, float& ea_f, float& sed,
                                          bool& finite) {
  constexpr bool EXACT_DIFF = (sizeof(LT) == 2);  // bf16: 8-bit significands
  constexpr int NA = A_CT > 0 ? A_CT : 1;
  const int nA = A_CT > 0 ? A_CT : A;
  m = R.get(0);
#pragma unroll
  for (int j = 1; j < NA; ++j) m = fmaxf(m, R.get(j));
  if constexpr (A_CT == 0)
    for (int j = 1; j < nA; ++j) m = fmaxf(m, R.get(j));
  // MUFU mode: e_j = 2^{y_j} with one rounding of the exponent y_j = (z_j - m) L'.
  //  bf16 logits: y_j = fma(z_j, L16, -m L16) with a 16-bit log2 e, so z L16 and
  //    m L16 are exact and the max term is exactly 2^0 = 1;
  //  fp32 logits: y_j = fl(z_j - m) * L32 (the max term again exactly 1).
  // The truncation of log2 e is a first-order factor 2^{(z_j - m)(log2 e - L')},
  // applied once per row through sed = sum_j e_j (z_j - m).  The e_j are summed
  // exactly: Fast2Sum in fp32 (s_hi starts at 1 >= every term), or, with
  // -DVTRACE_SUM_F64, fp32 -> fp64 conversions and two fp64 accumulators.
  constexpr float L16 = 1.44268798828125f;          // log2 e to 16 bits
  constexpr float L32 = 1.44269502f;                // fp32(log2 e)
  constexpr float CORR16 = 4.8884952e-06f;          // ln2 (log2 e - L16)
  constexpr float CORR32 = 1.3349930e-08f;          // ln2 (log2 e - L32)
  const float mL = m * L16;                         // exact for bf16 m
  double S64a = 0.0;
  [[maybe_unused]] double S64b = 0.0;
  float s_hi = 1.f, s_lo = 0.f, sd = 0.f, chk = 0.f, cw = 0.f;
  auto term = [&](float z, int j) {
    if constexpr (MODE == EXP_F64) {
      const double e = exp64((double)z - (double)m);
      S64a += e;
      sd = fmaf((float)e, z - m, sd);
      chk = __fmaf_rn(z, 0.f, chk);
    } else {
      float e, d;
      if constexpr (EXACT_DIFF) {
        e = ex2_approx(fmaf(z, L16, -mL));
        d = z - m;
      } else {
        d = z - m;
        const float y = d * L32;
        e = ex2_approx(y);
        // exact errors of d = z - m (TwoSum) and of y = d L32 (FMA residual)
        const float bb = d - z;
        const float dlo = (z - (d - bb)) + (-m - bb);
        cw = fmaf(e, fmaf(dlo, L32, fmaf(d, L32, -y)), cw);
      }
      sd = fmaf(e, d, sd);  // NaN if some z is inf/nan (0 * inf for -inf)
#ifdef VTRACE_SUM_F64
      if (j & 1) S64b += (double)e; else S64a += (double)e;
#else
      const float sum = s_hi + e;
      s_lo += (s_hi - sum) + e;
      s_hi = sum;
#endif
    }
  };
  if constexpr (A_CT > 0) {
#pragma unroll
    for (int j = 0; j < A_CT; ++j) term(R.get(j), j);
  } else {
    for (int j = 0; j < nA; ++j) term(R.get(j), j);
  }
  const float za = Elem<LT>::get(R.src, a);
  xa = (double)za - (double)m;  // z_a - m, exact
  ea_f = ex2_approx((za - m) * 1.44269504088896341f);  // exp(z_a - m), fp32 (exactly 1 at the max)
  sed = sd;
  if constexpr (MODE == EXP_F64) {
    S = S64a;
    finite = (chk == 0.f) && (m == m);
  } else {
#ifdef VTRACE_SUM_F64
    const double S0 = S64a + S64b;
#else
    const double S0 = (double)(s_hi - 1.f) + (double)s_lo;
#endif
    S = S0 + (double)(sd * (EXACT_DIFF ? CORR16 : CORR32));
    if constexpr (!EXACT_DIFF) S += (double)(cw * 0.693147182f);  // first order in the errors
    finite = isfinite(S) && isfinite(sd) && isfinite(m);
  }
}

// Both policies' statistics of one row in one interleaved loop (MUFU mode, compile-
// time A): four independent compensated-sum chains (2 per policy, even/odd j)
// instead of two long serial ones, for instruction-level parallelism.
struct RowStat {
  float m, sed, ea_f;
  double S, xa;
  bool finite;
};

template <typename LT, int A_CT>
__device__ __forceinline__ void row_stats2(const RowRegs<LT, A_CT>& Rp, const RowRegs<LT, A_CT>& Rm,
                                           int a, RowStat& sp, RowStat& sm) {
  static_assert(A_CT > 0, "compile-time A only");
  constexpr bool EXACT_DIFF = (sizeof(LT) == 2);
  constexpr float L16 = 1.44268798828125f;
  constexpr float L32 = 1.44269502f;
  constexpr float CORR = EXACT_DIFF ? 4.8884952e-06f : 1.3349930e-08f;
  float mp = Rp.get(0), mm = Rm.get(0);
#pragma unroll
  for (int j = 1; j < A_CT; ++j) {
    mp = fmaxf(mp, Rp.get(j));
    mm = fmaxf(mm, Rm.get(j));
  }
  const float mLp = mp * L16, mLm = mm * L16;
  float hp[2] = {1.f, 1.f}, lp[2] = {0.f, 0.f}, hm[2] = {1.f, 1.f}, lm[2] = {0.f, 0.f};
  float sdp = 0.f, sdm = 0.f;
#pragma unroll
  for (int j = 0; j < A_CT; ++j) {
    const int q = j & 1;
    const float zp = Rp.get(j), zm = Rm.get(j);
    float ep, em;
    if constexpr (EXACT_DIFF) {
      ep = ex2_approx(fmaf(zp, L16, -mLp));
      em = ex2_approx(fmaf(zm, L16, -mLm));
      sdp = fmaf(ep, zp, sdp);  // sum e z; (z - m) applied once per row below
      sdm = fmaf(em, zm, sdm);
    } else {
      const float dp = zp - mp, dm = zm - mm;
      ep = ex2_approx(dp * L32);
      em = ex2_approx(dm * L32);
      sdp = fmaf(ep, dp, sdp);
      sdm = fmaf(em, dm, sdm);
    }
    const float np = hp[q] + ep, nm = hm[q] + em;  // Fast2Sum: h >= 1 >= e
    lp[q] += (hp[q] - np) + ep;
    lm[q] += (hm[q] - nm) + em;
    hp[q] = np;
    hm[q] = nm;
  }
  // each chain started at 1: h - 1 is exact
  const float Sp_hi = (hp[0] - 1.f) + (hp[1] - 1.f), Sm_hi = (hm[0] - 1.f) + (hm[1] - 1.f);
  if constexpr (EXACT_DIFF) {  // sum e (z - m) = sum e z - m sum e (entropy/correction only)
    sdp = fmaf(-mp, Sp_hi, sdp);
    sdm = fmaf(-mm, Sm_hi, sdm);
  }
  const double Sp = ((double)(hp[0] - 1.f) + (double)(hp[1] - 1.f)) +
                    ((double)lp[0] + (double)lp[1]) + (double)(sdp * CORR);
  const double Sm = ((double)(hm[0] - 1.f) + (double)(hm[1] - 1.f)) +
                    ((double)lm[0] + (double)lm[1]) + (double)(sdm * CORR);
  const float zap = Elem<LT>::get(Rp.src, a), zam = Elem<LT>::get(Rm.src, a);
  sp.m = mp; sp.sed = sdp; sp.S = Sp; sp.xa = (double)zap - (double)mp;
  sp.ea_f = ex2_approx((zap - mp) * 1.44269504088896341f);
  sp.finite = isfinite(Sp) && isfinite(sdp) && isfinite(mp);
  sm.m = mm; sm.sed = sdm; sm.S = Sm; sm.xa = (double)zam - (double)mm;
  sm.ea_f = 1.f;
  sm.finite = isfinite(Sm) && isfinite(sdm) && isfinite(mm);
}

__device__ __forceinline__ double reward_transform(float r, int mode) {
  if (mode == 1) return (double)fminf(1.f, fmaxf(-1.f, r));  // P:944 (exact in fp32)
  double x = (double)r;
  if (mode == 2) {
    double th = tanh(x);
    return 0.3 * fmin(th, 0.0) + 5.0 * fmax(th, 0.0);
  }
  return x;
}

__device__ __forceinline__ void record_bad(WsHeader* ws, long long row, int kind) {
  unsigned long long key = ((unsigned long long)row << 8) | (unsigned long long)kind;
  atomicMin(&ws->status, key);
}

}  // namespace vtb200
