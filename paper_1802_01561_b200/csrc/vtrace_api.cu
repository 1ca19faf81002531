// vtrace_api.cu -- the fused sm_100a kernel and the C ABI of include/vtrace.h.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared
//        -Xcompiler -fPIC (see paper_1802_01561_b200/_build.py).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/vtrace.h"
#include "vtrace_kernels.cuh"

namespace vtb200 {

// ---------------------------------------------------------------------------
// Per-row statistics of one logits row:
//   m = max_j z_j, S = sum_j exp(z_j - m), ea = exp(z_a - m), finite flag.
// m is only a shift for range (reading c14); S and ea are accurate to ~1e-9.

template <typename LT, int A_CT, int MODE, bool EXACT_DIFF>
__device__ __forceinline__ void row_stats(const LT* zrow, int A, int a, float& m, double& S,
                                          double& ea, bool& finite) {
  float chk = 0.f;
  if constexpr (A_CT > 0) {
    float z[A_CT];
    load_row<LT, A_CT>(zrow, z);
    m = z[0];
#pragma unroll
    for (int j = 0; j < A_CT; ++j) {
      m = fmaxf(m, z[j]);
      chk = __fmaf_rn(z[j], 0.f, chk);  // NaN iff some z_j is inf/nan
    }
    if constexpr (MODE == EXP_F64) {
      const double m64 = (double)m;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < A_CT; ++j) acc += exp64_nonpos((double)z[j] - m64);
      S = acc;
    } else {
      float s_hi = 1.f, s_lo = 0.f;  // s_hi starts at 1 >= every term: Fast2Sum is exact
#pragma unroll
      for (int j = 0; j < A_CT; ++j) {
        float e = exp_mufu<EXACT_DIFF>(z[j], m);
        float s = s_hi + e;
        s_lo += (s_hi - s) + e;
        s_hi = s;
      }
      S = (double)(s_hi - 1.f) + (double)s_lo;
    }
  } else {
    m = Elem<LT>::get(zrow, 0);
    for (int j = 0; j < A; ++j) {
      float zj = Elem<LT>::get(zrow, j);
      m = fmaxf(m, zj);
      chk = __fmaf_rn(zj, 0.f, chk);
    }
    const double m64 = (double)m;
    double acc = 0.0;
    if constexpr (MODE == EXP_F64) {
      for (int j = 0; j < A; ++j) acc += exp64_nonpos((double)Elem<LT>::get(zrow, j) - m64);
      S = acc;
    } else {
      float s_hi = 1.f, s_lo = 0.f;
      for (int j = 0; j < A; ++j) {
        float e = exp_mufu<EXACT_DIFF>(Elem<LT>::get(zrow, j), m);
        float s = s_hi + e;
        s_lo += (s_hi - s) + e;
        s_hi = s;
      }
      S = (double)(s_hi - 1.f) + (double)s_lo;
    }
  }
  // the gathered term in fp64 in both modes (it enters the ratio undamped)
  ea = exp64_nonpos((double)Elem<LT>::get(zrow, a) - (double)m);
  finite = (chk == 0.f) && (m == m);
}

// Gradient epilogue of one row, fp32:
//   logp_j = z_j - lse, pi_j = exp(logp_j), H = -sum pi_j logp_j,
//   dz_j = pi_j (pg + c_e (logp_j + H))            for j != a
//   dz_a = -pg sum_{j != a} pi_j + c_e pi_a (logp_a + H)
// (pi_a - 1 is formed as -sum of the other pi_j: no cancellation).
// Writes dz to dzrow; returns H, log pi(a), sum dz^2.
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

template <typename LT, int A_CT>
__device__ __forceinline__ void row_epilogue(const LT* zrow, LT* dzrow, int A, int a, float lse,
                                             float pg, float ce, float& H_out, float& lpa_out,
                                             float& sq_out) {
  const float L = 1.44269504088896341f;
  if constexpr (A_CT > 0) {
    float z[A_CT];
    load_row<LT, A_CT>(zrow, z);
    float lp[A_CT], p[A_CT];
    float H = 0.f, rest = 0.f, lpa = 0.f, pa = 0.f;
#pragma unroll
    for (int j = 0; j < A_CT; ++j) {
      lp[j] = z[j] - lse;
      p[j] = ex2_approx(lp[j] * L);
      H = fmaf(-p[j], lp[j], H);
      const bool isa = (j == a);
      rest += isa ? 0.f : p[j];
      lpa = isa ? lp[j] : lpa;
      pa = isa ? p[j] : pa;
    }
    float sq = 0.f;
    if constexpr (sizeof(LT) == 2 && (A_CT % 2) == 0) {
      uint32_t* w = reinterpret_cast<uint32_t*>(dzrow);
#pragma unroll
      for (int k = 0; k < A_CT / 2; ++k) {
        float d0 = p[2 * k] * fmaf(ce, lp[2 * k] + H, pg);
        float d1 = p[2 * k + 1] * fmaf(ce, lp[2 * k + 1] + H, pg);
        if (2 * k == a) d0 = fmaf(-pg, rest, ce * pa * (lpa + H));
        if (2 * k + 1 == a) d1 = fmaf(-pg, rest, ce * pa * (lpa + H));
        sq = fmaf(d0, d0, sq);
        sq = fmaf(d1, d1, sq);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(d0, d1);
        w[k] = *reinterpret_cast<uint32_t*>(&h2);
      }
    } else {
#pragma unroll
      for (int j = 0; j < A_CT; ++j) {
        float d = p[j] * fmaf(ce, lp[j] + H, pg);
        if (j == a) d = fmaf(-pg, rest, ce * pa * (lpa + H));
        sq = fmaf(d, d, sq);
        dzrow[j] = store_cvt<LT>(d);
      }
    }
    H_out = H;
    lpa_out = lpa;
    sq_out = sq;
  } else {
    float H = 0.f, rest = 0.f;
    for (int j = 0; j < A; ++j) {
      float lpj = Elem<LT>::get(zrow, j) - lse;
      float pj = ex2_approx(lpj * L);
      H = fmaf(-pj, lpj, H);
      rest += (j == a) ? 0.f : pj;
    }
    const float lpa = Elem<LT>::get(zrow, a) - lse;
    const float pa = ex2_approx(lpa * L);
    float sq = 0.f;
    for (int j = 0; j < A; ++j) {
      float lpj = Elem<LT>::get(zrow, j) - lse;
      float pj = ex2_approx(lpj * L);
      float d = pj * fmaf(ce, lpj + H, pg);
      if (j == a) d = fmaf(-pg, rest, ce * pa * (lpa + H));
      sq = fmaf(d, d, sq);
      dzrow[j] = store_cvt<LT>(d);
    }
    H_out = H;
    lpa_out = lpa;
    sq_out = sq;
  }
}

__device__ __forceinline__ double reward_transform(float r, int mode) {
  double x = (double)r;
  if (mode == 1) return fmin(1.0, fmax(-1.0, x));
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

__device__ __forceinline__ size_t align128(size_t x) { return (x + 127) & ~size_t(127); }

// ---------------------------------------------------------------------------
// Shared-memory layout of one CTA (host and device agree on it).
//   NSTAGE input stages: z^pi, z^mu [Tc][8*A] (logits dtype), a, r, gamma, V [Tc][8]
//   per-unit row statistics: ratio (f64), lse, vs, pg_adv (f32)
//   one dlogits staging tile [Tc][8*A] (TMA-stored while the next unit runs)

constexpr int NSTAGE = 2;

struct Layout {
  size_t pi, mu, a, r, g, v, stage, ratio, lse, vs, pg, dz, total;
};

__host__ __device__ inline size_t a128(size_t x) { return (x + 127) & ~size_t(127); }

__host__ __device__ inline Layout make_layout(int nrow, int A, int elem) {
  Layout L;
  size_t off = 0;
  L.pi = off; off = a128(off + (size_t)nrow * A * elem);
  L.mu = off; off = a128(off + (size_t)nrow * A * elem);
  L.a = off;  off = a128(off + (size_t)nrow * 4);
  L.r = off;  off = a128(off + (size_t)nrow * 4);
  L.g = off;  off = a128(off + (size_t)nrow * 4);
  L.v = off;  off = a128(off + (size_t)nrow * 4);
  L.stage = off;
  off = NSTAGE * L.stage;
  L.ratio = off; off = a128(off + (size_t)nrow * 8);
  L.lse = off;   off = a128(off + (size_t)nrow * 4);
  L.vs = off;    off = a128(off + (size_t)nrow * 4);
  L.pg = off;    off = a128(off + (size_t)nrow * 4);
  L.dz = off;    off = a128(off + (size_t)nrow * A * elem);
  L.total = off;
  return L;
}

// ---------------------------------------------------------------------------
// The fused kernel.  Persistent CTAs loop over work units handed out by an
// atomic ticket (reverse time order); a 2-stage TMA ring prefetches the next
// unit's tiles while the current unit is computed.  Template: logits type,
// compile-time A (0 = runtime), LOSS (loss_and_grad) vs targets only, TMA
// staging vs plain loads, exp mode.

template <typename LT, int A_CT, bool LOSS, bool USE_TMA, int MODE>
__global__ void __launch_bounds__(NTHREADS)
    vtrace_fused_kernel(const Params P, const __grid_constant__ TmaMaps maps) {
  constexpr bool EXACT_DIFF = (sizeof(LT) == 2);  // z - m exact in fp32 for bf16 inputs
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[NSTAGE];
  __shared__ int s_unit[NSTAGE];
  __shared__ unsigned int s_epoch;
  __shared__ int s_last;
  __shared__ double s_red[NWARPS][NPART];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int A = (A_CT > 0) ? A_CT : P.A;
  const int Tc = P.Tc;
  const int nrow = Tc * BC;
  const long long T = P.T, B = P.B;
  const Layout L = make_layout(nrow, A, (int)sizeof(LT));
  double* ratio_s = reinterpret_cast<double*>(smem + L.ratio);
  float* lse_s = reinterpret_cast<float*>(smem + L.lse);
  float* vs_s = reinterpret_cast<float*>(smem + L.vs);
  float* pg_s = reinterpret_cast<float*>(smem + L.pg);
  LT* dz_t = reinterpret_cast<LT*>(smem + L.dz);

  // thread 0: claim the next unit for stage `st` and start its TMA loads
  auto claim_and_load = [&](int st) {
    const int u = (int)atomicAdd(&P.ws->ticket, 1u);
    s_unit[st] = u;
    if constexpr (USE_TMA) {
      if (u < P.units) {
        const int kc = P.K - 1 - u / P.G;
        const int t0 = kc * Tc;
        const int b0 = (u % P.G) * BC;
        unsigned char* sb = smem + (size_t)st * L.stage;
        const uint32_t bytes =
            (uint32_t)(2 * (size_t)nrow * A * sizeof(LT) + 4 * (size_t)nrow * 4);
        mbar_expect_tx(&bar[st], bytes);
        tma_load_2d(sb + L.pi, &maps.pi, b0 * A, t0, &bar[st]);
        tma_load_2d(sb + L.mu, &maps.mu, b0 * A, t0, &bar[st]);
        tma_load_2d(sb + L.a, &maps.a, b0, t0, &bar[st]);
        tma_load_2d(sb + L.r, &maps.r, b0, t0, &bar[st]);
        tma_load_2d(sb + L.g, &maps.g, b0, t0, &bar[st]);
        tma_load_2d(sb + L.v, &maps.v, b0, t0, &bar[st]);
      }
    }
  };

  if (tid == 0) {
    s_epoch = *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch);
    if constexpr (USE_TMA) {
      for (int st = 0; st < NSTAGE; ++st) mbar_init(&bar[st], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int st = 0; st < NSTAGE; ++st) claim_and_load(st);
  }
  __syncthreads();
  const unsigned int epoch = s_epoch & 0x3fffffffu;
  const float ce = (float)P.c_e;
  const float cv = (float)P.c_v;

  for (int it = 0;; ++it) {
    const int st = it % NSTAGE;
    const int u = s_unit[st];
    if (u >= P.units) break;  // CTA-uniform
    unsigned char* sb = smem + (size_t)st * L.stage;
    LT* pi_t = reinterpret_cast<LT*>(sb + L.pi);
    LT* mu_t = reinterpret_cast<LT*>(sb + L.mu);
    int* a_t = reinterpret_cast<int*>(sb + L.a);
    float* r_t = reinterpret_cast<float*>(sb + L.r);
    float* g_t = reinterpret_cast<float*>(sb + L.g);
    float* v_t = reinterpret_cast<float*>(sb + L.v);
    const int kchunk = P.K - 1 - u / P.G;  // reverse time order of tickets
    const int grp = u % P.G;
    const int t0 = kchunk * Tc;
    const int tlen = (int)min((long long)Tc, T - t0);
    const long long b0 = (long long)grp * BC;
    const int blen = (int)min((long long)BC, B - b0);

    // ---- a1: the unit's tiles ------------------------------------------------------
    if constexpr (USE_TMA) {
      mbar_wait(&bar[st], (uint32_t)((it / NSTAGE) & 1));
    } else {
      const LT* gpi = reinterpret_cast<const LT*>(P.pi);
      const LT* gmu = reinterpret_cast<const LT*>(P.mu);
      const int rowlen = BC * A;
      for (int i = tid; i < nrow * A; i += NTHREADS) {
        const int tl = i / rowlen, rem = i - tl * rowlen, bl = rem / A, j = rem - bl * A;
        LT zp = store_cvt<LT>(0.f), zm = store_cvt<LT>(0.f);
        if (tl < tlen && bl < blen) {
          const long long gi = (((long long)(t0 + tl)) * B + b0 + bl) * A + j;
          zp = gpi[gi];
          zm = gmu[gi];
        }
        pi_t[i] = zp;
        mu_t[i] = zm;
      }
      for (int i = tid; i < nrow; i += NTHREADS) {
        const int tl = i / BC, bl = i - tl * BC;
        int av = 0;
        float rv = 0.f, gv = 0.f, vv = 0.f;
        if (tl < tlen && bl < blen) {
          const long long gi = ((long long)(t0 + tl)) * B + b0 + bl;
          av = P.actions[gi];
          rv = P.rew[gi];
          gv = P.disc[gi];
          vv = P.val[gi];
        }
        a_t[i] = av;
        r_t[i] = rv;
        g_t[i] = gv;
        v_t[i] = vv;
      }
      __syncthreads();
    }

    double acc_pg = 0, acc_v = 0, acc_H = 0, acc_dz = 0, acc_dv = 0, acc_rho = 0, acc_clip = 0;

    // ---- a3-a5: per-row statistics of both policies -------------------------------
    for (int r = tid; r < nrow; r += NTHREADS) {
      const int tl = r >> 3, bl = r & 7;
      if (tl >= tlen || bl >= blen) continue;
      const long long row = (long long)(t0 + tl) * B + b0 + bl;
      const int a_raw = a_t[r];
      const int a = min(max(a_raw, 0), A - 1);
      float m_p, m_m;
      double S_p, S_m, ea_p, ea_m;
      bool fin_p, fin_m;
      row_stats<LT, A_CT, MODE, EXACT_DIFF>(pi_t + (size_t)r * A, A, a, m_p, S_p, ea_p, fin_p);
      row_stats<LT, A_CT, MODE, EXACT_DIFF>(mu_t + (size_t)r * A, A, a, m_m, S_m, ea_m, fin_m);
      // pi(a)/mu(a) = (ea_p / S_p) / (ea_m / S_m)
      const double ratio = (ea_p * S_m) / (ea_m * S_p);
      ratio_s[r] = ratio;
      lse_s[r] = m_p + logf((float)S_p);
      acc_rho += fmin(P.rho_bar, ratio);
      acc_clip += (ratio > P.rho_bar) ? 1.0 : 0.0;
      if (P.has_lr) P.log_rhos[row] = (float)log(ratio);
      if (P.has_lp)
        P.lp_out[row] =
            (float)(((double)Elem<LT>::get(pi_t + (size_t)r * A, a) - (double)m_p) - log(S_p));
      if (P.has_lm)
        P.lm_out[row] =
            (float)(((double)Elem<LT>::get(mu_t + (size_t)r * A, a) - (double)m_m) - log(S_m));
      if (a_raw != a) record_bad(P.ws, row, VT_DATA_ACTION);
      if (!(fin_p && fin_m)) record_bad(P.ws, row, VT_DATA_LOGITS);
      if (!isfinite(r_t[r])) record_bad(P.ws, row, VT_DATA_REWARD);
      if (!isfinite(v_t[r])) record_bad(P.ws, row, VT_DATA_VALUE);
      const float gm = g_t[r];
      if (!(gm >= 0.f && gm <= 1.f)) record_bad(P.ws, row, VT_DATA_DISCOUNT);
    }
    __syncthreads();

    // ---- a2, a7-a9: reverse V-trace recursion, warp per column --------------------
    if (warp < blen) {
      const int bl = warp;
      const long long b = b0 + bl;
      const int kk = (tlen + 31) >> 5;  // steps per lane
      const int s_beg = min(lane * kk, tlen), s_end = min(s_beg + kk, tlen);
      const bool last_chunk = (kchunk == P.K - 1);
      double V_after;  // V(x) just after this chunk: next chunk's first value or bootstrap
      if (last_chunk) {
        V_after = (double)__ldg(P.boot + b);
        if (lane == 0 && !isfinite((float)V_after)) record_bad(P.ws, T * B + b, VT_DATA_VALUE);
      } else {
        V_after = (double)__ldg(P.val + (long long)(t0 + tlen) * B + b);
      }
      // local affine aggregate of this lane's segment: A_beg = D + G * A_end
      double Gl = 1.0, Dl = 0.0;
      for (int s = s_end - 1; s >= s_beg; --s) {
        const int r = s * BC + bl;
        const double ratio = ratio_s[r];
        const double rho = fmin(P.rho_bar, ratio);
        const double c = P.lambda * fmin(P.c_bar, ratio);
        const double gam = (double)g_t[r];
        const double Vt = (double)v_t[r];
        const double Vn = (s + 1 < tlen) ? (double)v_t[r + BC] : V_after;
        const double delta = rho * (reward_transform(r_t[r], P.reward_mode) + gam * Vn - Vt);
        Dl = fma(gam * c, Dl, delta);
        Gl = gam * c * Gl;
      }
      // inclusive suffix scan over lanes: lane l <- composition of segments l..31
      double Gi = Gl, Di = Dl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double Go = shfl_down_d(Gi, o), Do = shfl_down_d(Di, o);
        if (lane + o < 32) {
          Di = fma(Gi, Do, Di);
          Gi = Gi * Go;
        }
      }
      double Ge = shfl_down_d(Gi, 1), De = shfl_down_d(Di, 1);  // exclusive: l+1..31
      if (lane == 31) {
        Ge = 1.0;
        De = 0.0;
      }
      const double Gc = __shfl_sync(0xffffffffu, Gi, 0), Dc = __shfl_sync(0xffffffffu, Di, 0);
      double carry = 0.0;  // A at the end of this chunk; A_T = 0 (v_T = V(x_T), reading c2)
      if (P.K > 1) {
        ColRec* rec = P.recs + (size_t)u * BC + bl;
        if (lane == 0) {
          if (last_chunk) {
            rec->incl = Dc;
            st_release_u32(&rec->flag, (epoch << 2) | 2u);
          } else {
            rec->G = Gc;
            rec->D = Dc;
            st_release_u32(&rec->flag, (epoch << 2) | 1u);
            double aG = 1.0, aD = 0.0;  // composition of the later chunks seen so far
            int up = u - P.G;
            while (true) {
              const ColRec* pr = P.recs + (size_t)up * BC + bl;
              unsigned int f = ld_acquire_u32(&pr->flag);
              int spins = 0;
              while ((f >> 2) != epoch || (f & 3u) == 0u) {
                if (++spins > 8) __nanosleep(64);
                f = ld_acquire_u32(&pr->flag);
              }
              if ((f & 3u) == 2u) {
                carry = fma(aG, __ldcg(&pr->incl), aD);
                break;
              }
              const double Gp = __ldcg(&pr->G), Dp = __ldcg(&pr->D);
              aD = fma(aG, Dp, aD);
              aG = aG * Gp;
              up -= P.G;
            }
            rec->incl = fma(Gc, carry, Dc);
            st_release_u32(&rec->flag, (epoch << 2) | 2u);
          }
        }
        carry = __shfl_sync(0xffffffffu, carry, 0);
      }
      // second pass over the segment: v_t, q_t, pg_adv_t
      double A_next = fma(Ge, carry, De);  // A at s_end
      double V_next = (s_end < tlen) ? (double)v_t[s_end * BC + bl] : V_after;
      for (int s = s_end - 1; s >= s_beg; --s) {
        const int r = s * BC + bl;
        const double ratio = ratio_s[r];
        const double rho = fmin(P.rho_bar, ratio);
        const double c = P.lambda * fmin(P.c_bar, ratio);
        const double rho_pg = fmin(P.pg_rho_bar, ratio);
        const double gam = (double)g_t[r];
        const double Vt = (double)v_t[r];
        const double rr = reward_transform(r_t[r], P.reward_mode);
        const double delta = rho * (rr + gam * V_next - Vt);
        const double A_t = fma(gam * c, A_next, delta);
        const double v_next = V_next + A_next;  // v_{t+1}; v_T = V(x_T)
        const double adv = rho_pg * (rr + gam * v_next - Vt);
        vs_s[r] = (float)(Vt + A_t);
        pg_s[r] = (float)adv;
        A_next = A_t;
        V_next = Vt;
      }
    }
    if constexpr (LOSS && USE_TMA) {
      // the previous unit's dlogits store must have read dz_t before we overwrite it
      if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();

    // ---- a6, a10, a11: gradient epilogue + row outputs ----------------------------
    for (int r = tid; r < nrow; r += NTHREADS) {
      const int tl = r >> 3, bl = r & 7;
      if (tl >= tlen || bl >= blen) continue;
      const long long row = (long long)(t0 + tl) * B + b0 + bl;
      const float vsr = vs_s[r], pgr = pg_s[r], Vt = v_t[r];
      if (P.vs) P.vs[row] = vsr;
      if (P.pg_adv) P.pg_adv[row] = pgr;
      if constexpr (LOSS) {
        const int a = min(max(a_t[r], 0), A - 1);
        float H, lpa, sq;
        row_epilogue<LT, A_CT>(pi_t + (size_t)r * A, dz_t + (size_t)r * A, A, a, lse_s[r], pgr,
                               ce, H, lpa, sq);
        const float dv = cv * (Vt - vsr);
        P.dvalues[row] = dv;
        const double res = (double)vsr - (double)Vt;
        acc_pg += -(double)pgr * (double)lpa;
        acc_v += 0.5 * res * res;
        acc_H += (double)H;
        acc_dz += (double)sq;
        acc_dv += (double)dv * (double)dv;
      }
    }
    if constexpr (LOSS && USE_TMA) fence_proxy_async_smem();
    __syncthreads();  // stage st fully consumed; dz_t complete
    if (tid == 0) {
      if constexpr (LOSS && USE_TMA) {
        tma_store_2d(&maps.dz, (int)(b0 * A), t0, dz_t);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if constexpr (USE_TMA) fence_proxy_async_smem();  // generic reads before async refill
      claim_and_load(st);
    }
    if constexpr (LOSS && !USE_TMA) {
      LT* gdz = reinterpret_cast<LT*>(P.dlogits);
      const int rowlen = BC * A;
      for (int i = tid; i < nrow * A; i += NTHREADS) {
        const int tl = i / rowlen, rem = i - tl * rowlen, bl = rem / A, j = rem - bl * A;
        if (tl < tlen && bl < blen)
          gdz[(((long long)(t0 + tl)) * B + b0 + bl) * A + j] = dz_t[i];
      }
    }

    // ---- a12: this unit's partial sums (fixed order: rows -> warps -> unit) --------
    if constexpr (LOSS) {
      double part[NPART] = {acc_pg, acc_v, acc_H, 0.0, acc_dz, acc_dv, acc_rho, acc_clip};
#pragma unroll
      for (int i = 0; i < NPART; ++i) {
        double x = part[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) s_red[warp][i] = x;
      }
      __syncthreads();
      if (tid < NPART) {
        double x = 0.0;
#pragma unroll
        for (int w = 0; w < NWARPS; ++w) x += s_red[w][tid];
        P.unit_partials[(size_t)u * NPART + tid] = x;
      }
    }
    __syncthreads();  // s_unit[st] (claimed above) visible; s_red free
  }

  // ---- exit: the last CTA out reduces the unit partials and re-arms the workspace --
  if (tid == 0) {
    if constexpr (LOSS && USE_TMA) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __threadfence();
    const unsigned int prev = atomicAdd(&P.ws->exited, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (LOSS && P.partials) {
      // warp i sums partial i: lane l takes units l, l+32, ... in order, then the
      // 32 lane sums are added in lane order (a fixed tree: bitwise reproducible)
      if (warp < NPART) {
        double x = 0.0;
        for (int v = lane; v < P.units; v += 32)
          x += __ldcg(P.unit_partials + (size_t)v * NPART + warp);
        double tot = 0.0;
        for (int l = 0; l < 32; ++l) tot += __shfl_sync(0xffffffffu, x, l);
        if (lane == 0) s_red[warp][0] = tot;
      }
      __syncthreads();
      if (tid == 0) {
        double out[NPART];
        for (int i = 0; i < NPART; ++i) out[i] = s_red[i][0];
        out[VT_P_TOTAL_LOSS] = out[VT_P_PG_LOSS] + P.c_v * out[VT_P_BASELINE_LOSS] -
                               P.c_e * out[VT_P_ENTROPY_SUM];
        for (int i = 0; i < NPART; ++i) P.partials[i] = out[i];
      }
    }
    if (tid == 0) {
      P.ws->ticket = 0u;
      P.ws->exited = 0u;
      __threadfence();
      *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch) = (epoch + 1u) & 0x3fffffffu;
    }
  }
}

// ---------------------------------------------------------------------------
// host side

struct Plan {
  int Tc, K, G, units;
  size_t smem;
};

constexpr size_t kMaxSmem = 220 * 1024;

static int tc_max_for(int A, int elem) {
  const long long row_bytes = 2LL * A * elem + 16;
  long long tc = 40960 / (BC * row_bytes);
  if (tc > 64) tc = 64;
  if (tc < 1) tc = 1;
  return (int)tc;
}

static Plan make_plan(long long T, long long B, int A, int elem) {
  Plan p;
  const int tcm = tc_max_for(A, elem);
  if (T <= tcm) {
    p.Tc = (int)T;
    p.K = 1;
  } else {
    p.K = (int)((T + tcm - 1) / tcm);
    p.Tc = (int)((T + p.K - 1) / p.K);
    p.K = (int)((T + p.Tc - 1) / p.Tc);
  }
  p.G = (int)((B + BC - 1) / BC);
  p.units = p.K * p.G;
  p.smem = make_layout(p.Tc * BC, A, elem).total;
  return p;
}

static size_t ws_bytes_for(const Plan& p) {
  return 256 + (size_t)p.units * BC * sizeof(ColRec) + (size_t)p.units * NPART * sizeof(double);
}

// ---- device / driver queries ---------------------------------------------------------
static std::mutex g_mu;
static int g_dev_ok[64];  // 0 unknown, 1 ok, 2 bad
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static vt_status check_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return VT_ERR_CUDA;
  if (dev < 0 || dev >= 64) return VT_ERR_DEVICE;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_dev_ok[dev] == 0) {
    int maj = 0, mnr = 0;
    if (cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
      return VT_ERR_CUDA;
    g_dev_ok[dev] = (maj == 10 && mnr == 0) ? 1 : 2;
  }
  return g_dev_ok[dev] == 1 ? VT_OK : VT_ERR_DEVICE;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return g_encode;
}

static bool encode_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem,
                      long long inner, long long outer, int box_inner, int box_outer) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(inner * elem)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int exp_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("VTRACE_EXP_MODE");
    mode = (e && (e[0] == 'm' || e[0] == 'M' || e[0] == '1')) ? EXP_MUFU : EXP_F64;
  }
  return mode;
}

template <typename LT, int A_CT, bool LOSS, bool TMA, int MODE>
static vt_status launch_one(const Params& P, const TmaMaps& maps, const Plan& plan,
                            cudaStream_t st) {
  auto kern = vtrace_fused_kernel<LT, A_CT, LOSS, TMA, MODE>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  static int num_sms = 0;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kMaxSmem);
    int dev = 0;
    if (attr_err == cudaSuccess) attr_err = cudaGetDevice(&dev);
    if (attr_err == cudaSuccess)
      attr_err = cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  });
  if (attr_err != cudaSuccess) return VT_ERR_CUDA;
  // persistent grid: every resident CTA slot, never more CTAs than units
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTHREADS, plan.smem) !=
          cudaSuccess ||
      per_sm < 1)
    return VT_ERR_CUDA;
  const long long grid = std::min<long long>(plan.units, (long long)per_sm * num_sms);
  kern<<<(unsigned)grid, NTHREADS, plan.smem, st>>>(P, maps);
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}

template <typename LT, bool LOSS, bool TMA, int MODE>
static vt_status dispatch_a(const Params& P, const TmaMaps& maps, const Plan& plan,
                            cudaStream_t st) {
  if constexpr (TMA) {
    if (P.A == 18) return launch_one<LT, 18, LOSS, TMA, MODE>(P, maps, plan, st);
    if (P.A == 9) return launch_one<LT, 9, LOSS, TMA, MODE>(P, maps, plan, st);
  }
  return launch_one<LT, 0, LOSS, TMA, MODE>(P, maps, plan, st);
}

template <typename LT, bool LOSS>
static vt_status dispatch(const Params& P, const TmaMaps& maps, const Plan& plan, bool tma,
                          cudaStream_t st) {
  if (exp_mode() == EXP_MUFU) {
    return tma ? dispatch_a<LT, LOSS, true, EXP_MUFU>(P, maps, plan, st)
               : dispatch_a<LT, LOSS, false, EXP_MUFU>(P, maps, plan, st);
  }
  return tma ? dispatch_a<LT, LOSS, true, EXP_F64>(P, maps, plan, st)
             : dispatch_a<LT, LOSS, false, EXP_F64>(P, maps, plan, st);
}

static bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

static vt_status check_params(const vt_vtrace_params* p) {
  if (!p) return VT_ERR_INVALID_ARG;
  const float rb = p->clip_rho_threshold, cb = p->clip_c_threshold,
              pb = p->clip_pg_rho_threshold, l = p->lambda_;
  if (std::isnan(rb) || std::isnan(cb) || std::isnan(pb) || std::isnan(l)) return VT_ERR_PARAM;
  if (!(rb > 0.f) || !(cb > 0.f) || !(pb > 0.f)) return VT_ERR_PARAM;
  if (cb > rb) return VT_ERR_PARAM;  // rho_bar >= c_bar
  if (l < 0.f || l > 1.f) return VT_ERR_PARAM;
  if (p->reward_mode < 0 || p->reward_mode > 2) return VT_ERR_PARAM;
  return VT_OK;
}

static vt_status common_launch(bool loss, long long T, long long B, long long A, vt_dtype dt,
                               const void* mu, const void* pi, const int32_t* actions,
                               const float* disc, const float* rew, const float* val,
                               const float* boot, const vt_vtrace_params* prm,
                               const vt_loss_weights* w, void* dlogits, float* dvalues,
                               double* partials, float* vs, float* pg_adv, float* lr,
                               float* lp, float* lm, void* ws, size_t ws_bytes,
                               cudaStream_t st) {
  if (!mu || !pi || !actions || !disc || !rew || !val || !boot) return VT_ERR_INVALID_ARG;
  if (T <= 0 || B <= 0 || A <= 0 || A > VT_MAX_ACTIONS) return VT_ERR_SHAPE;
  if (T > (1LL << 30) || B > (1LL << 30) || T * B > (1LL << 40) || T * B * A > (1LL << 46))
    return VT_ERR_SHAPE;
  if (dt != VT_FLOAT32 && dt != VT_BFLOAT16) return VT_ERR_DTYPE;
  vt_status s = check_params(prm);
  if (s) return s;
  if (loss) {
    if (!w || !dlogits || !dvalues || !partials) return VT_ERR_INVALID_ARG;
    if (!std::isfinite(w->baseline_cost) || !std::isfinite(w->entropy_cost)) return VT_ERR_PARAM;
  } else {
    if (!vs || !pg_adv) return VT_ERR_INVALID_ARG;
  }
  const int elem = dt == VT_BFLOAT16 ? 2 : 4;
  if (!aligned(mu, elem) || !aligned(pi, elem) || !aligned(actions, 4) || !aligned(disc, 4) ||
      !aligned(rew, 4) || !aligned(val, 4) || !aligned(boot, 4) ||
      (dlogits && !aligned(dlogits, elem)) || (dvalues && !aligned(dvalues, 4)) ||
      (partials && !aligned(partials, 8)) || (vs && !aligned(vs, 4)) ||
      (pg_adv && !aligned(pg_adv, 4)) || (lr && !aligned(lr, 4)) || (lp && !aligned(lp, 4)) ||
      (lm && !aligned(lm, 4)))
    return VT_ERR_ALIGNMENT;
  const Plan plan = make_plan(T, B, (int)A, elem);
  if (!ws || !aligned(ws, 256) || ws_bytes < ws_bytes_for(plan)) return VT_ERR_WORKSPACE;
  s = check_device();
  if (s) return s;

  Params P;
  std::memset(&P, 0, sizeof(P));
  P.T = T; P.B = B; P.A = (int)A; P.Tc = plan.Tc; P.K = plan.K; P.G = plan.G;
  P.units = plan.units;
  P.has_lr = lr != nullptr; P.has_lp = lp != nullptr; P.has_lm = lm != nullptr;
  P.mu = mu; P.pi = pi; P.actions = actions; P.disc = disc; P.rew = rew; P.val = val;
  P.boot = boot;
  P.vs = vs; P.pg_adv = pg_adv; P.log_rhos = lr; P.lp_out = lp; P.lm_out = lm;
  P.dlogits = dlogits; P.dvalues = dvalues; P.partials = partials;
  P.rho_bar = (double)prm->clip_rho_threshold;
  P.c_bar = (double)prm->clip_c_threshold;
  P.pg_rho_bar = (double)prm->clip_pg_rho_threshold;
  P.lambda = (double)prm->lambda_;
  P.reward_mode = prm->reward_mode;
  P.c_v = loss ? (double)w->baseline_cost : 0.0;
  P.c_e = loss ? (double)w->entropy_cost : 0.0;
  unsigned char* wsb = static_cast<unsigned char*>(ws);
  P.ws = reinterpret_cast<WsHeader*>(wsb);
  P.recs = reinterpret_cast<ColRec*>(wsb + 256);
  P.unit_partials =
      reinterpret_cast<double*>(wsb + 256 + (size_t)plan.units * BC * sizeof(ColRec));

  // TMA eligibility: 16-byte aligned bases and row pitches, box inner <= 256 elements
  TmaMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  bool tma = (A * BC <= 256) && (B * A < (1LL << 31)) && (T < (1LL << 31)) && ((B * A * elem) % 16 == 0) && ((B * 4) % 16 == 0) &&
             aligned(mu, 16) && aligned(pi, 16) && aligned(actions, 16) && aligned(disc, 16) &&
             aligned(rew, 16) && aligned(val, 16) && (!loss || aligned(dlogits, 16)) &&
             plan.Tc <= 256 && plan.smem <= kMaxSmem;
  if (tma) {
    const CUtensorMapDataType ldt =
        dt == VT_BFLOAT16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    tma = encode_2d(&maps.mu, mu, ldt, elem, B * A, T, BC * (int)A, plan.Tc) &&
          encode_2d(&maps.pi, pi, ldt, elem, B * A, T, BC * (int)A, plan.Tc) &&
          encode_2d(&maps.a, actions, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, B, T, BC, plan.Tc) &&
          encode_2d(&maps.r, rew, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, T, BC, plan.Tc) &&
          encode_2d(&maps.g, disc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, T, BC, plan.Tc) &&
          encode_2d(&maps.v, val, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, T, BC, plan.Tc) &&
          (!loss || encode_2d(&maps.dz, dlogits, ldt, elem, B * A, T, BC * (int)A, plan.Tc));
  }
  if (plan.smem > kMaxSmem) return VT_ERR_SHAPE;
  if (dt == VT_BFLOAT16) {
    return loss ? dispatch<__nv_bfloat16, true>(P, maps, plan, tma, st)
                : dispatch<__nv_bfloat16, false>(P, maps, plan, tma, st);
  }
  return loss ? dispatch<float, true>(P, maps, plan, tma, st)
              : dispatch<float, false>(P, maps, plan, tma, st);
}

}  // namespace vtb200

using namespace vtb200;

extern "C" {

size_t vtrace_workspace_bytes(int64_t T, int64_t B, int64_t A, vt_dtype dt) {
  if (T <= 0 || B <= 0 || A <= 0 || A > VT_MAX_ACTIONS) return 0;
  if (dt != VT_FLOAT32 && dt != VT_BFLOAT16) return 0;
  const Plan p = make_plan(T, B, (int)A, dt == VT_BFLOAT16 ? 2 : 4);
  return ws_bytes_for(p);
}

vt_status vtrace_workspace_init(void* ws, size_t bytes, vt_stream_t stream) {
  if (!ws || bytes < 256 || !aligned(ws, 256)) return VT_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(ws, 0, bytes, st) != cudaSuccess) return VT_ERR_CUDA;
  if (cudaMemsetAsync(static_cast<unsigned char*>(ws) + offsetof(WsHeader, status), 0xFF, 8,
                      st) != cudaSuccess)
    return VT_ERR_CUDA;
  return VT_OK;
}

vt_status vtrace_from_logits(int64_t T, int64_t B, int64_t A, vt_dtype dt, const void* mu,
                             const void* pi, const int32_t* actions, const float* discounts,
                             const float* rewards, const float* values, const float* boot,
                             const vt_vtrace_params* params, float* vs, float* pg_adv,
                             float* log_rhos, float* lp, float* lm, void* ws, size_t ws_bytes,
                             vt_stream_t stream) {
  return common_launch(false, T, B, A, dt, mu, pi, actions, discounts, rewards, values, boot,
                       params, nullptr, nullptr, nullptr, nullptr, vs, pg_adv, log_rhos, lp, lm,
                       ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

vt_status vtrace_loss_and_grad(int64_t T, int64_t B, int64_t A, vt_dtype dt, const void* mu,
                               const void* pi, const int32_t* actions, const float* discounts,
                               const float* rewards, const float* values, const float* boot,
                               const vt_vtrace_params* params, const vt_loss_weights* weights,
                               void* dlogits, float* dvalues, double* partials, float* vs,
                               float* pg_adv, void* ws, size_t ws_bytes, vt_stream_t stream) {
  return common_launch(true, T, B, A, dt, mu, pi, actions, discounts, rewards, values, boot,
                       params, weights, dlogits, dvalues, partials, vs, pg_adv, nullptr, nullptr,
                       nullptr, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

vt_status vtrace_loss_and_grad_from_host(
    int64_t T, int64_t B, int64_t A, vt_dtype dt, const void* h_mu, const void* h_pi,
    const int32_t* h_a, const float* h_g, const float* h_r, const float* h_v,
    const float* h_boot, void* d_mu, void* d_pi, int32_t* d_a, float* d_g, float* d_r,
    float* d_v, float* d_boot, const vt_vtrace_params* params, const vt_loss_weights* weights,
    void* dlogits, float* dvalues, double* partials_device, double* partials_host, void* ws,
    size_t ws_bytes, vt_stream_t stream) {
  if (!h_mu || !h_pi || !h_a || !h_g || !h_r || !h_v || !h_boot || !partials_host)
    return VT_ERR_INVALID_ARG;
  if (T <= 0 || B <= 0 || A <= 0 || A > VT_MAX_ACTIONS) return VT_ERR_SHAPE;
  if (dt != VT_FLOAT32 && dt != VT_BFLOAT16) return VT_ERR_DTYPE;
  if (!d_mu || !d_pi || !d_a || !d_g || !d_r || !d_v || !d_boot) return VT_ERR_INVALID_ARG;
  const size_t elem = dt == VT_BFLOAT16 ? 2 : 4;
  const size_t nl = (size_t)T * B * A * elem, ns = (size_t)T * B * 4;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // validate before any copy is issued
  vt_status s = check_params(params);
  if (s) return s;
  if (!weights || !dlogits || !dvalues || !partials_device) return VT_ERR_INVALID_ARG;
  const Plan plan = make_plan(T, B, (int)A, (int)elem);
  if (!ws || !aligned(ws, 256) || ws_bytes < ws_bytes_for(plan)) return VT_ERR_WORKSPACE;
  s = check_device();
  if (s) return s;
  const cudaMemcpyKind h2d = cudaMemcpyHostToDevice;
  if (cudaMemcpyAsync(d_pi, h_pi, nl, h2d, st) != cudaSuccess ||
      cudaMemcpyAsync(d_mu, h_mu, nl, h2d, st) != cudaSuccess ||
      cudaMemcpyAsync(d_a, h_a, ns, h2d, st) != cudaSuccess ||
      cudaMemcpyAsync(d_g, h_g, ns, h2d, st) != cudaSuccess ||
      cudaMemcpyAsync(d_r, h_r, ns, h2d, st) != cudaSuccess ||
      cudaMemcpyAsync(d_v, h_v, ns, h2d, st) != cudaSuccess ||
      cudaMemcpyAsync(d_boot, h_boot, (size_t)B * 4, h2d, st) != cudaSuccess)
    return VT_ERR_CUDA;
  s = vtrace_loss_and_grad(T, B, A, dt, d_mu, d_pi, d_a, d_g, d_r, d_v, d_boot, params, weights,
                           dlogits, dvalues, partials_device, nullptr, nullptr, ws, ws_bytes,
                           stream);
  if (s) return s;
  if (cudaMemcpyAsync(partials_host, partials_device, VT_P_COUNT * sizeof(double),
                      cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return VT_ERR_CUDA;
  return VT_OK;
}

vt_status vtrace_read_device_status(void* ws, int32_t* code, int64_t* first_bad,
                                    vt_stream_t stream) {
  if (!ws || !code || !first_bad) return VT_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long key = ~0ull;
  unsigned char* p = static_cast<unsigned char*>(ws) + offsetof(WsHeader, status);
  if (cudaMemcpyAsync(&key, p, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return VT_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return VT_ERR_CUDA;
  if (key == ~0ull) {
    *code = VT_DATA_OK;
    *first_bad = -1;
  } else {
    *code = (int32_t)(key & 0xff);
    *first_bad = (int64_t)(key >> 8);
    if (cudaMemsetAsync(p, 0xFF, 8, st) != cudaSuccess) return VT_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return VT_ERR_CUDA;
  }
  return VT_OK;
}

const char* vtrace_status_string(vt_status s) {
  switch (s) {
    case VT_OK: return "ok";
    case VT_ERR_INVALID_ARG: return "invalid argument (NULL pointer)";
    case VT_ERR_SHAPE: return "invalid shape";
    case VT_ERR_DTYPE: return "unsupported logits dtype";
    case VT_ERR_PARAM: return "invalid V-trace parameter or loss weight";
    case VT_ERR_ALIGNMENT: return "misaligned pointer";
    case VT_ERR_WORKSPACE: return "workspace NULL, misaligned or too small";
    case VT_ERR_CUDA: return "CUDA runtime error";
    case VT_ERR_DEVICE: return "device is not sm_100 (B200)";
  }
  return "unknown status";
}

int32_t vtrace_version(void) { return 100; }

}  // extern "C"
