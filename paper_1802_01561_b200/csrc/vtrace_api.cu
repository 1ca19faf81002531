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
#include <atomic>
#include <mutex>
#include <type_traits>

#include "../../include/vtrace.h"
#include "vtrace_kernels.cuh"
#include "vtrace_rows.cuh"
#include "vtrace_cb_host.h"

namespace vtb200 {

// ---------------------------------------------------------------------------
// Shared-memory layout of one CTA (host and device agree on it).
//   NSTAGE input stages: z^pi, z^mu [Tc][8*A] (logits dtype); a, r, gamma [Tc][8];
//     V [Tc+1][8] (one row past the chunk); bootstrap [8].  The gradient is written
//     in place over the z^pi tile and TMA-stored from there.
//   2 row-state buffers (by unit parity): ratio pi/mu and TD error r + gamma V' - V
//     (f64), lse, lse - H, 1 - pi(a) (f32); A = v - V (f64, Tc+1 rows: the last is
//     the carry from the later chunks)

constexpr int NSTAGE = 3;
constexpr int NROWWARPS = NWARPS - 1;       // warps 0..4 own rows, warp 5 runs the scan
constexpr int NROWTHREADS = NROWWARPS * 32;  // 160 >= Tc * 8
constexpr int KSEG = (NROWTHREADS / BC + 3) / 4;  // steps per scan lane (Tc <= 20)

struct Layout {
  size_t pi, mu, a, r, g, v, boot, stage;          // offsets inside a stage
  size_t ratio[2], td[2], adv[2], lse[2], csh[2], rest[2];  // row state
  size_t total;
};


// Every TMA destination is 128-byte aligned (a tiled cp.async.bulk.tensor into a
// merely 16-byte aligned address faults with "misaligned address" on sm_100a);
// the row-state arrays, read and written by threads only, are 16-byte aligned.
__host__ __device__ inline Layout make_layout(int nrow, int A, int elem) {
  Layout L;
  size_t off = 0;
  L.pi = off;   off = a128(off + (size_t)nrow * A * elem);
  L.mu = off;   off = a128(off + std::max((size_t)nrow * A * elem, (size_t)nrow * 4));
  L.a = off;    off = a128(off + (size_t)nrow * 4);
  L.r = off;    off = a128(off + (size_t)nrow * 4);
  L.g = off;    off = a128(off + (size_t)nrow * 4);
  L.v = off;    off = a128(off + (size_t)(nrow + BC) * 4);
  L.boot = off; off = a128(off + (size_t)BC * 4);
  L.stage = off;
  off = NSTAGE * L.stage;
  for (int p = 0; p < 2; ++p) {
    L.ratio[p] = off; off = a16(off + (size_t)nrow * 8);
    L.td[p] = off;    off = a16(off + (size_t)nrow * 8);
    L.adv[p] = off;   off = a16(off + (size_t)(nrow + BC) * 8);
    L.lse[p] = off;   off = a16(off + (size_t)nrow * 4);
    L.csh[p] = off;   off = a16(off + (size_t)nrow * 4);
    L.rest[p] = off;  off = a16(off + (size_t)nrow * 4);
  }
  L.total = a128(off);
  return L;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// geometry of one work unit (T, B < 2^31: 32-bit arithmetic)
struct Unit {
  int u, kchunk, grp, t0, tlen, b0, blen;
  bool last_chunk;
  __device__ __forceinline__ void finish(const Params& P) {
    t0 = kchunk * P.Tc;
    tlen = min(P.Tc, P.T32 - t0);
    b0 = grp * BC;
    blen = min(BC, P.B32 - b0);
    last_chunk = (kchunk == P.K - 1);
  }
  __device__ __forceinline__ void set(int uu, const Params& P) {
    u = uu;
    kchunk = P.K - 1 - uu / P.G;  // unit ids run in reverse time order
    grp = uu % P.G;
    finish(P);
  }
  // u += gridDim.x without a division: gridDim.x = stride_q * G + stride_r
  __device__ __forceinline__ void advance(const Params& P, int stride) {
    u += stride;
    grp += P.stride_r;
    kchunk -= P.stride_q;
    if (grp >= P.G) {
      grp -= P.G;
      --kchunk;
    }
    finish(P);
  }
};

// ---------------------------------------------------------------------------
// The fused kernel.  A cooperative (co-resident) persistent grid; CTA c owns
// units c, c + grid, ...  (unit ids run in reverse time order, so a unit only
// ever waits, in the look-back, on units of earlier or the same rounds, all
// resident).  Warp-specialised software pipeline over the CTA's units; in
// iteration i (NWARPS = 6, 192 threads; a unit is 8 columns x Tc <= 20 steps):
//   row warps 0..4 : P1(i)   row statistics + TD errors of unit i (one row per thread)
//   scan warp 5    : SCAN(i-1) the reverse recursion of unit i-1 (affine maps on
//                    A = v - V; 4 lanes per column, each over a segment of steps),
//                    look-back on the later units' aggregates, publication
//   thread 0       : waits for the TMA store of unit i-2's gradient, reloads that
//                    stage with unit i+1
//   -- barrier 1 (192 threads) --
//   row warps      : P3(i-1) v, pg_adv, dL/dV and dL/dz of unit i-1, dz written in
//                    place over z^pi, then one TMA store
// so the latency-bound recursion overlaps the row arithmetic of the next unit.

// GEN: the call uses a Section 5.2.2 variant, the App. E.3 q estimate or behaviour
// log-probs (false: plain V-trace from logits, that logic compiled out).
template <typename LT, int A_CT, bool LOSS, bool USE_TMA, int MODE, bool GEN>
__global__ void __launch_bounds__(NTHREADS, 4)
    vtrace_fused_kernel(const Params P, const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[NSTAGE];
  __shared__ unsigned int s_epoch;
  __shared__ int s_last;
  __shared__ double s_red[NWARPS][NPART];
  __shared__ double s_fin[NPART];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int A = (A_CT > 0) ? A_CT : P.A;
  const int Tc = P.Tc;
  const int nrow = Tc * BC;
  const long long T = P.T, B = P.B;
  const KLayout& L = P.L;
  const int stride = (int)gridDim.x;
  const int n_my = (P.units - (int)blockIdx.x + stride - 1) / stride;  // units of this CTA

#ifdef VTRACE_TIMING
  if (P.timing && tid == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.timing[(size_t)blockIdx.x * P.timing_iters * 8 + (P.timing_iters - 1) * 8 + 0] = g;
  }
#endif
  if (tid == 0) {
    s_epoch = *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch);
    if constexpr (USE_TMA) {
      for (int st = 0; st < NSTAGE; ++st) mbar_init(&bar[st], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  const unsigned int epoch = s_epoch & 0x3fffffffu;

  // TMA: unit i of this CTA -> stage i % NSTAGE (thread 0 only)
  auto load_unit = [&](int i) {
    if constexpr (USE_TMA) {
      if (i < n_my) {
        Unit U;
        U.set((int)blockIdx.x + i * stride, P);
        const int st = i % NSTAGE;
        unsigned char* sb = smem + (size_t)st * L.stage;
        const uint32_t bytes = (uint32_t)((size_t)nrow * A * sizeof(LT) +
                                          ((GEN && P.mu_lp) ? (size_t)nrow * 4
                                                            : (size_t)nrow * A * sizeof(LT)) +
                                          3 * (size_t)nrow * 4 + (size_t)(nrow + BC) * 4 + BC * 4);
        mbar_expect_tx(&bar[st], bytes);
        const int xb = (int)(U.b0 * A);
        tma_load_2d(sb + L.pi, &maps.pi, xb, U.t0, &bar[st]);
        tma_load_2d(sb + L.mu, &maps.mu, (GEN && P.mu_lp) ? (int)U.b0 : xb, U.t0, &bar[st]);
        tma_load_2d(sb + L.a, &maps.a, (int)U.b0, U.t0, &bar[st]);
        tma_load_2d(sb + L.r, &maps.r, (int)U.b0, U.t0, &bar[st]);
        tma_load_2d(sb + L.g, &maps.g, (int)U.b0, U.t0, &bar[st]);
        tma_load_2d(sb + L.v, &maps.v, (int)U.b0, U.t0, &bar[st]);
        tma_load_1d(sb + L.boot, &maps.boot, (int)U.b0, &bar[st]);
      }
    }
  };
  if (USE_TMA && tid == 0) load_unit(0);

  const float ce = (float)P.c_e;
  const float cv = (float)P.c_v;
  // per-thread partial sums (fixed assignment of rows to threads: deterministic)
  float acc_pg = 0.f, acc_v = 0.f, acc_H = 0.f, acc_dz = 0.f, acc_dv = 0.f, acc_rho = 0.f,
        acc_clip = 0.f;

  Unit Ucur, Uprev;  // units i and i-1 of this CTA
  Ucur.set((int)blockIdx.x, P);
  Uprev = Ucur;
#ifdef VTRACE_TIMING
  unsigned long long* tim =
      P.timing ? P.timing + (size_t)blockIdx.x * P.timing_iters * 8 : nullptr;
#else
  constexpr unsigned long long* tim = nullptr;  // phase timing compiled out
#endif
  for (int i = 0; i <= n_my; ++i) {
    if (tim && i < P.timing_iters && (tid == 0 || tid == NROWTHREADS))
      tim[i * 8 + (tid == 0 ? 0 : 4)] = clock64();
    // ================= phase A: P1(i) on row warps || SCAN(i-1) on the scan warp ====
    if (warp < NROWWARPS) {
      if (i < n_my) {
        const Unit& U = Ucur;
        const int st = i % NSTAGE, par = i & 1;
        unsigned char* sb = smem + (size_t)st * L.stage;
        const LT* pi_t = reinterpret_cast<const LT*>(sb + L.pi);
        const LT* mu_t = reinterpret_cast<const LT*>(sb + L.mu);
        if constexpr (USE_TMA) {
          mbar_wait(&bar[st], (uint32_t)((i / NSTAGE) & 1));
#ifdef VTRACE_TIMING
          if (P.timing && tid == 0 && i == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            P.timing[(size_t)blockIdx.x * P.timing_iters * 8 + (P.timing_iters - 1) * 8 + 3] = g;
          }
#endif
        } else {
          // plain staged loads (unaligned shapes): the row warps fill the stage
          LT* wpi = reinterpret_cast<LT*>(sb + L.pi);
          LT* wmu = reinterpret_cast<LT*>(sb + L.mu);
          int* wa = reinterpret_cast<int*>(sb + L.a);
          float* wr = reinterpret_cast<float*>(sb + L.r);
          float* wg = reinterpret_cast<float*>(sb + L.g);
          float* wv = reinterpret_cast<float*>(sb + L.v);
          float* wb = reinterpret_cast<float*>(sb + L.boot);
          const LT* gpi = reinterpret_cast<const LT*>(P.pi);
          const LT* gmu = reinterpret_cast<const LT*>(P.mu);
          const int rowlen = BC * A;
          for (int k = tid; k < nrow * A; k += NROWTHREADS) {
            const int tl = k / rowlen, rem = k - tl * rowlen, bl = rem / A, j = rem - bl * A;
            LT zp = store_cvt<LT>(0.f), zm = store_cvt<LT>(0.f);
            if (tl < U.tlen && bl < U.blen) {
              const long long gi = (((long long)(U.t0 + tl)) * B + U.b0 + bl) * A + j;
              zp = gpi[gi];
              if (!(GEN && P.mu_lp)) zm = gmu[gi];
            }
            wpi[k] = zp;
            if (!(GEN && P.mu_lp)) wmu[k] = zm;
          }
          for (int k = tid; k < nrow + BC; k += NROWTHREADS) {
            const int tl = k / BC, bl = k - tl * BC;
            const long long t = (long long)U.t0 + tl;
            const bool ok = bl < U.blen && t < T && tl <= Tc;
            const long long gi = t * B + U.b0 + bl;
            if (k < nrow) {
              const bool okr = ok && tl < U.tlen;
              if (GEN && P.mu_lp)  // log mu(a_t) in the mu region
                reinterpret_cast<float*>(wmu)[k] = okr ? reinterpret_cast<const float*>(P.mu)[gi] : 0.f;
              wa[k] = okr ? P.actions[gi] : 0;
              wr[k] = okr ? P.rew[gi] : 0.f;
              wg[k] = okr ? P.disc[gi] : 0.f;
            }
            wv[k] = ok ? P.val[gi] : 0.f;
          }
          if (tid < BC) wb[tid] = tid < U.blen ? P.boot[U.b0 + tid] : 0.f;
          named_bar_sync(2, NROWTHREADS);
        }
        const int r = tid;
        const int tl = r >> 3, bl = r & 7;
        if (r < nrow && tl < U.tlen && bl < U.blen) {
          const int* a_t = reinterpret_cast<const int*>(sb + L.a);
          const float* r_t = reinterpret_cast<const float*>(sb + L.r);
          const float* g_t = reinterpret_cast<const float*>(sb + L.g);
          const float* v_t = reinterpret_cast<const float*>(sb + L.v);
          const int a_raw = a_t[r];
          const int a = min(max(a_raw, 0), A - 1);
          float m_p, m_m, sed_p, sed_m, ea_p, ea_m;
          double S_p, S_m, xa_p, xa_m;
          bool fin_p, fin_m;
          {
            RowRegs<LT, A_CT> zp;
            zp.load(pi_t + (size_t)r * A);
            row_stats<LT, A_CT, MODE>(zp, A, a, m_p, S_p, xa_p, ea_p, sed_p, fin_p);
          }
          if (GEN && P.mu_lp) {  // behaviour as log mu(a_t): ratio = pi(a) / exp(log mu(a))
            const float lmu = reinterpret_cast<const float*>(mu_t)[r];
            xa_m = (double)lmu;
            S_m = 1.0;
            fin_m = isfinite(lmu);
            m_m = ea_m = sed_m = 0.f;
          } else {
            RowRegs<LT, A_CT> zm;
            zm.load(mu_t + (size_t)r * A);
            row_stats<LT, A_CT, MODE>(zm, A, a, m_m, S_m, xa_m, ea_m, sed_m, fin_m);
          }
          // pi(a)/mu(a) = exp((z^pi_a - m_pi) - (z^mu_a - m_mu)) S_mu / S_pi
          const double ratio = exp64(xa_p - xa_m) * (S_m / S_p);
          // TD error r_t + gamma_t V(x_{t+1}) - V(x_t), V(x_T) = bootstrap
          const float rt = r_t[r], gm = g_t[r], Vt = v_t[r];
          const float Vn = (tl + 1 < U.tlen || !U.last_chunk)
                               ? v_t[r + BC]  // the V tile has Tc + 1 rows
                               : reinterpret_cast<const float*>(sb + L.boot)[bl];
          const double td =
              reward_transform(rt, P.reward_mode) + (double)gm * (double)Vn - (double)Vt;
          const float Sf = (float)S_p;
          const float inv_S = rcp_approx(Sf);
          reinterpret_cast<double*>(smem + L.ratio[par])[r] = ratio;
          reinterpret_cast<double*>(smem + L.td[par])[r] = td;
          const float lse = m_p + __logf(Sf);  // log sum_j exp(z_j)
          reinterpret_cast<float*>(smem + L.lse[par])[r] = lse;
          reinterpret_cast<float*>(smem + L.csh[par])[r] = fmaf(sed_p, inv_S, m_p);  // lse - H
          reinterpret_cast<float*>(smem + L.rest[par])[r] = (float)(S_p - (double)ea_p) * inv_S;
          acc_rho += (float)step_weights<GEN>(P, ratio).rho;  // the rho_t in delta_t (r6)
          acc_clip += ((!GEN || P.correction == VT_CORRECTION_VTRACE) && ratio > P.rho_bar) ? 1.f
                                                                                        : 0.f;
          if constexpr (!LOSS) {
            const long long row = (long long)(U.t0 + tl) * B + U.b0 + bl;
            if (P.has_lr) P.log_rhos[row] = (float)log(ratio);
            if (P.has_lp) P.lp_out[row] = (float)(xa_p - log(S_p));
            if (P.has_lm) P.lm_out[row] = (float)(xa_m - log(S_m));
          }
          // data checks (the host cannot see the data), one branch when clean
          const bool bad = (a_raw != a) || !(fin_p && fin_m) || !isfinite(rt) ||
                           !isfinite(Vt) || !isfinite(Vn) || !(gm >= 0.f && gm <= 1.f);
          if (bad) {
            const long long row = (long long)(U.t0 + tl) * B + U.b0 + bl;
            if (a_raw != a) record_bad(P.ws, row, VT_DATA_ACTION);
            if (!(fin_p && fin_m)) record_bad(P.ws, row, VT_DATA_LOGITS);
            if (!isfinite(rt)) record_bad(P.ws, row, VT_DATA_REWARD);
            if (!isfinite(Vt)) record_bad(P.ws, row, VT_DATA_VALUE);
            if (!(gm >= 0.f && gm <= 1.f)) record_bad(P.ws, row, VT_DATA_DISCOUNT);
            if (!isfinite(Vn) && U.last_chunk && tl + 1 == U.tlen)
              record_bad(P.ws, T * B + U.b0 + bl, VT_DATA_VALUE);  // the bootstrap
          }
        }
      }
      if (tid == 0) {
        // the gradient store of unit i-2 must have read its stage before the refill
        if constexpr (LOSS && USE_TMA) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if constexpr (USE_TMA) {
          fence_proxy_async_smem();  // generic reads of the stage before its async refill
          load_unit(i + 1);          // stage (i+1)%3 == (i-2)%3
        }
      }
    } else if (i >= 1) {
      // ---- SCAN(i-1): warp 7.  Lane 4c + s owns column c, segment s of 4 --------
      const Unit& U = Uprev;
      const int st = (i - 1) % NSTAGE, par = (i - 1) & 1;
      const unsigned char* sb = smem + (size_t)st * L.stage;
      const float* g_t = reinterpret_cast<const float*>(sb + L.g);
      const double* ratio_s = reinterpret_cast<const double*>(smem + L.ratio[par]);
      const double* td_s = reinterpret_cast<const double*>(smem + L.td[par]);
      double* adv_s = reinterpret_cast<double*>(smem + L.adv[par]);
      const int c = lane >> 2, sg = lane & 3;
      const bool col_ok = c < U.blen;
      const int kk = (U.tlen + 3) >> 2;  // <= KSEG
      const int s_beg = min(sg * kk, U.tlen), s_end = min(s_beg + kk, U.tlen);
      const bool need_carry = (P.K > 1) && !U.last_chunk;
      // early (speculative) look-back read: the predecessor is usually long done
      const unsigned long long tagA = ((unsigned long long)epoch << 2) | 1ull;
      const unsigned long long tagI = ((unsigned long long)epoch << 2) | 2ull;
      unsigned long long t0tag = 0ull;
      double incl0 = 0.0;
      const int up0 = U.u - P.G;
      if (need_carry && col_ok && sg == 0)
        ld_tag16(P.recs + ((size_t)up0 * BC + c) * RECS_PER_COL + 2, incl0, t0tag);
      // per step: delta_t = rho_t td_t and g_t = gamma_t c_t (Remark 2 P:225);
      // delta_t is parked in adv_s (overwritten by A_t in the second pass)
      double G = 1.0, D = 0.0;  // local affine aggregate: A_beg = D + G * A_end
#pragma unroll
      for (int k = KSEG - 1; k >= 0; --k) {
        if (col_ok && s_beg + k < s_end) {
          const int q = (s_beg + k) * BC + c;
          const double ratio = ratio_s[q];
          const StepWeights sw = step_weights<GEN>(P, ratio);  // (Section 5.2.2 variants)
          const double dl = sw.rho * td_s[q];
          const double gc = (double)g_t[q] * sw.c;
          adv_s[q] = dl;
          D = fma(gc, D, dl);
          G = gc * G;
        }
      }
      // suffix scan over the 4 segments of each column (width-4 shuffles)
      double Gi = G, Di = D;
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        const double Go = __shfl_down_sync(0xffffffffu, Gi, o, 4);
        const double Do = __shfl_down_sync(0xffffffffu, Di, o, 4);
        if (sg + o < 4) {
          Di = fma(Gi, Do, Di);
          Gi = Gi * Go;
        }
      }
      double Ge = __shfl_down_sync(0xffffffffu, Gi, 1, 4);  // exclusive: segments > sg
      double De = __shfl_down_sync(0xffffffffu, Di, 1, 4);
      if (sg == 3) {
        Ge = 1.0;
        De = 0.0;
      }
      if (tim && i < P.timing_iters && lane == 0) tim[i * 8 + 7] = clock64();
      // carry = A at the end of the chunk (A_T = 0: v_T = V(x_T), reading c2)
      double carry = 0.0;
      if (P.K > 1) {
        TagRec* my = P.recs + ((size_t)U.u * BC + c) * RECS_PER_COL;
        // publish the aggregate (chunk 0 is never looked back at)
        if (U.kchunk > 0 && !U.last_chunk && col_ok && sg == 0) {
          st_tag16(my + 0, Gi, tagA);
          st_tag16(my + 1, Di, tagA);
        }
        if (need_carry && col_ok && sg == 0) {
          if (t0tag == tagI) {
            carry = incl0;
          } else {
            double aG = 1.0, aD = 0.0;  // composition of the later chunks seen so far
            int up = up0;
            int spins = 0;
            while (true) {
              const TagRec* pr = P.recs + ((size_t)up * BC + c) * RECS_PER_COL;
              double vi, vg, vd;
              unsigned long long ti, tg, td;
              ld_tag16(pr + 2, vi, ti);
              if (ti == tagI) {
                carry = fma(aG, vi, aD);
                break;
              }
              ld_tag16(pr + 0, vg, tg);
              ld_tag16(pr + 1, vd, td);
              if (tg == tagA && td == tagA) {
                aD = fma(aG, vd, aD);
                aG = aG * vg;
                up -= P.G;
                spins = 0;
              } else if (++spins > 4) {
                __nanosleep(32);
              }
            }
          }
        }
        carry = __shfl_sync(0xffffffffu, carry, lane & ~3);
        // publish the inclusive carry: A at this chunk's first step
        if (U.kchunk > 0 && col_ok && sg == 0) st_tag16(my + 2, fma(Gi, carry, Di), tagI);
      }
      // second pass: A_t = delta_t + g_t A_{t+1}  (Remark 1)
      double A_next = fma(Ge, carry, De);  // A at s_end
      if (col_ok && sg == 0) adv_s[U.tlen * BC + c] = carry;  // A just after the chunk
#pragma unroll
      for (int k = KSEG - 1; k >= 0; --k) {
        if (col_ok && s_beg + k < s_end) {
          const int q = (s_beg + k) * BC + c;
          const double gc = (double)g_t[q] * step_weights<GEN>(P, ratio_s[q]).c;
          A_next = fma(gc, A_next, adv_s[q]);
          adv_s[q] = A_next;
        }
      }
    }
    if (tim && i < P.timing_iters && (tid == 0 || tid == NROWTHREADS))
      tim[i * 8 + (tid == 0 ? 1 : 5)] = clock64();
    named_bar_sync(1, NTHREADS);
    if (tim && i < P.timing_iters && tid == 0) tim[i * 8 + 2] = clock64();

    // ================= phase B: P3(i-1) on the row warps ============================
    if (warp < NROWWARPS && i >= 1) {
      const Unit& U = Uprev;
      const int st = (i - 1) % NSTAGE, par = (i - 1) & 1;
      unsigned char* sb = smem + (size_t)st * L.stage;
      const int r = tid;
      const int tl = r >> 3, bl = r & 7;
      if (r < nrow && tl < U.tlen && bl < U.blen) {
        const long long row = (long long)(U.t0 + tl) * B + U.b0 + bl;
        const double* adv_s = reinterpret_cast<const double*>(smem + L.adv[par]);
        const double A_t = adv_s[r], A_n = adv_s[r + BC];  // A_t and A_{t+1}
        const double ratio = reinterpret_cast<const double*>(smem + L.ratio[par])[r];
        const double td = reinterpret_cast<const double*>(smem + L.td[par])[r];
        const float gm = reinterpret_cast<const float*>(sb + L.g)[r];
        const float Vt = reinterpret_cast<const float*>(sb + L.v)[r];
        // v_t = V(x_t) + A_t;  pg_adv_t = rho_pg (r_t + gamma_t v_{t+1} - V(x_t))
        //                              = rho_pg (td_t + gamma_t A_{t+1})
        const float vsr = (float)((double)Vt + A_t);
        // (q_s = r_s + gamma V(x_{s+1}) instead with q_values: App. E.3)
        const float pgr = (float)(step_weights<GEN>(P, ratio).rho_pg *
                                  ((GEN && P.q_values) ? td : fma((double)gm, A_n, td)));
        if (P.vs) P.vs[row] = vsr;
        if (P.pg_adv) P.pg_adv[row] = pgr;
        if constexpr (LOSS) {
          const float Ar = (float)A_t;
          const float lse = reinterpret_cast<const float*>(smem + L.lse[par])[r];
          const float cshift = reinterpret_cast<const float*>(smem + L.csh[par])[r];
          const float rest = reinterpret_cast<const float*>(smem + L.rest[par])[r];
          const float pa = 1.f - rest;  // pi(a); only scaled by c_e below
          const int a = min(max(reinterpret_cast<const int*>(sb + L.a)[r], 0), A - 1);
          LT* zrow = reinterpret_cast<LT*>(sb + L.pi) + (size_t)r * A;  // dz overwrites z
          RowRegs<LT, A_CT> zp;
          zp.load(zrow);
          const float za = Elem<LT>::get(zrow, a);
          const float L2E = 1.44269504088896341f;
          const float lseL = lse * L2E;
          // epsilon-correction (readings c11, r7): the policy-gradient term uses
          // log(pi_a + eps); its logit gradient is the plain one times pi_a / (pi_a + eps)
          float pge = pgr, logpa = za - lse;
          if (GEN && P.correction == VT_CORRECTION_EPSILON) {
            const float pa_e = ex2_approx((za - lse) * L2E);  // pi(a), relative accuracy
            const float rr = P.eps / pa_e;
            logpa = pa_e > 0.f ? (za - lse) + log1pf(rr) : logf(P.eps);
            pge = pgr / (1.f + rr);
          }
          const float alpha = fmaf(-ce, cshift, pge);  // pg + c_e (z_j - cshift) = alpha + c_e z_j
          float sq = 0.f;
          // dz_j = pi_j (pg + c_e (log pi_j + H))   (j != a)
          if constexpr (RowRegs<LT, A_CT>::kPacked) {
            uint32_t* w = reinterpret_cast<uint32_t*>(zrow);
#pragma unroll
            for (int k = 0; k < A_CT / 2; ++k) {
              const float z0 = zp.get(2 * k), z1 = zp.get(2 * k + 1);
              const float d0 = ex2_approx(fmaf(z0, L2E, -lseL)) * fmaf(ce, z0, alpha);
              const float d1 = ex2_approx(fmaf(z1, L2E, -lseL)) * fmaf(ce, z1, alpha);
              sq = fmaf(d0, d0, sq);
              sq = fmaf(d1, d1, sq);
              __nv_bfloat162 h2 = __floats2bfloat162_rn(d0, d1);
              w[k] = *reinterpret_cast<uint32_t*>(&h2);
            }
          } else if constexpr (A_CT > 0) {
#pragma unroll
            for (int j = 0; j < A_CT; ++j) {
              const float z = zp.get(j);
              const float d = ex2_approx(fmaf(z, L2E, -lseL)) * fmaf(ce, z, alpha);
              sq = fmaf(d, d, sq);
              zrow[j] = store_cvt<LT>(d);
            }
          } else {
            for (int j = 0; j < A; ++j) {
              const float z = zp.get(j);
              const float d = ex2_approx(fmaf(z, L2E, -lseL)) * fmaf(ce, z, alpha);
              sq = fmaf(d, d, sq);
              zrow[j] = store_cvt<LT>(d);
            }
          }
          // the taken action: dz_a = -pg (1 - pi_a) + c_e pi_a (log pi_a + H)
          const float d_wrong = ex2_approx(fmaf(za, L2E, -lseL)) * fmaf(ce, za, alpha);
          const float d_a = fmaf(-pge, rest, ce * pa * (za - cshift));
          zrow[a] = store_cvt<LT>(d_a);
          sq = __fadd_rn(__fsub_rn(sq, __fmul_rn(d_wrong, d_wrong)), __fmul_rn(d_a, d_a));
          if (tim && i < P.timing_iters && tid == 0) tim[i * 8 + 6] = clock64();
          const float dv = -cv * Ar;  // c_v (V - v)
          P.dvalues[row] = dv;
          acc_pg = fmaf(-pgr, logpa, acc_pg);  // -pg_adv log pi(a)  (log(pi(a) + eps))
          acc_v = fmaf(0.5f * Ar, Ar, acc_v);
          acc_H += lse - cshift;  // H = lse - (lse - H)
          acc_dz += sq;
          acc_dv = fmaf(dv, dv, acc_dv);
          if constexpr (!USE_TMA) {
            LT* gdz = reinterpret_cast<LT*>(P.dlogits) + row * A;
            for (int j = 0; j < A; ++j) gdz[j] = zrow[j];
          }
        }
      }
      if constexpr (LOSS && USE_TMA) {
        fence_proxy_async_smem();
        named_bar_sync(2, NROWTHREADS);  // the gradient tile is complete
        if (tid == 0) {
          tma_store_2d(&maps.dz, (int)(U.b0 * A), U.t0, sb + L.pi);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (tim && i < P.timing_iters && tid == 0) tim[i * 8 + 3] = clock64();
    }
    Uprev = Ucur;
    Ucur.advance(P, stride);
  }

#ifdef VTRACE_TIMING
  if (P.timing && tid == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.timing[(size_t)blockIdx.x * P.timing_iters * 8 + (P.timing_iters - 1) * 8 + 1] = g;
  }
#endif
  // ---- a12: CTA partials (fixed order), then the last CTA out reduces them ---------
  {
    const double part[NPART] = {acc_pg, acc_v, acc_H, 0.0, acc_dz, acc_dv, acc_rho, acc_clip};
#pragma unroll
    for (int k = 0; k < NPART; ++k) {
      double x = part[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) s_red[warp][k] = x;
    }
    __syncthreads();
    if (tid < NPART) {
      double x = 0.0;
#pragma unroll
      for (int w = 0; w < NWARPS; ++w) x += s_red[w][tid];
      P.cta_partials[(size_t)blockIdx.x * NPART + tid] = x;
    }
  }
  __syncthreads();
  if (tid == 0) {
    // (the gradient stores must have read the CTA's shared memory; their global writes
    // complete with the grid)
    if constexpr (LOSS && USE_TMA) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __threadfence();
    const unsigned int prev = atomicAdd(&P.ws->exited, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (LOSS && P.partials) {
      for (int k = warp; k < NPART; k += NWARPS) {  // warp w: partials w, w + NWARPS
        // lanes stride the CTAs (8 independent loads in flight per lane), then the
        // 32 lane sums are added in lane order: a fixed tree, bitwise reproducible
        double x = 0.0;
        for (int v0 = 0; v0 < (int)gridDim.x; v0 += 32 * 8) {
          double buf[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int v = v0 + q * 32 + lane;
            buf[q] = v < (int)gridDim.x ? __ldcg(P.cta_partials + (size_t)v * NPART + k) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) x += buf[q];
        }
        // a fixed butterfly over the 32 lane sums (deterministic; not a serial chain)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) s_fin[k] = x;
      }
      __syncthreads();
      if (tid == 0) {
        double out[NPART];
        for (int k = 0; k < NPART; ++k) out[k] = s_fin[k];
        out[VT_P_TOTAL_LOSS] = out[VT_P_PG_LOSS] + P.c_v * out[VT_P_BASELINE_LOSS] -
                               P.c_e * out[VT_P_ENTROPY_SUM];
        for (int k = 0; k < NPART; ++k) P.partials[k] = out[k];
      }
    }
#ifdef VTRACE_TIMING
    if (P.timing && tid == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      P.timing[(size_t)blockIdx.x * P.timing_iters * 8 + (P.timing_iters - 1) * 8 + 2] = g;
    }
#endif
    if (tid == 0) {
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

constexpr int kMaxCtas = 4096;  // bound on the persistent grid (workspace sizing)

// Tc (steps per unit) depends only on (T, A, dtype): at most 20 so that a unit's
// Tc * 8 rows map one-to-one onto the 160 row threads, and small enough for the
// NSTAGE input stages plus the row-state buffers to fit in 100 KB of shared memory.
static int tc_max_for(int A, int elem) {
  for (int tc = NROWTHREADS / BC; tc > 1; --tc)
    if (make_layout(tc * BC, A, elem).total <= 100 * 1024) return tc;
  return 1;
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

struct WsLayout {
  size_t recs, cta, cb_recs, cb_count, total;
};

static WsLayout ws_layout(const Plan& p) {
  WsLayout w;
  w.recs = 256;
  w.cta = a128(w.recs + (size_t)p.units * BC * RECS_PER_COL * sizeof(TagRec));
  // column-block kernel: one record set per CTA (at most ceil(B / 4) CTAs) + a ticket
  w.cb_recs = a128(w.cta + (size_t)kMaxCtas * NPART * sizeof(double));
  const size_t ctas = ((size_t)p.G * BC + 3) / 4;  // >= ceil(B / 4)
  w.cb_count = a128(w.cb_recs + ctas * NPART * sizeof(TagRec));
  w.total = a128(w.cb_count + sizeof(unsigned int));
  return w;
}

static size_t ws_bytes_for(const Plan& p) { return ws_layout(p).total; }

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

// Logits [T][B][A] viewed as [T][B / (4g)][4gA] (column segments of 4g trajectories),
// with the segment index as the OUTER box dimension: a box {4gA, Ts, nseg_box} lands in
// shared memory as [segment][t][4gA], so one warp's 4 columns x 8 steps are 32
// consecutive rows (column-block kernel).
static bool encode_logits_3d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem,
                             int seg, long long T, long long nseg, long long row_elems, int box_t,
                             int box_seg) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)seg, (cuuint64_t)T, (cuuint64_t)nseg};
  cuuint64_t strides[2] = {(cuuint64_t)(row_elems * elem), (cuuint64_t)((long long)seg * elem)};
  cuuint32_t box[3] = {(cuuint32_t)seg, (cuuint32_t)box_t, (cuuint32_t)box_seg};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static bool encode_1d(CUtensorMap* m, const void* base, long long n, int box) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[1] = {(cuuint64_t)n};
  cuuint64_t strides[1] = {0};
  cuuint32_t bx[1] = {(cuuint32_t)box};
  cuuint32_t estr[1] = {1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, const_cast<void*>(base), dims, strides,
                   bx, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}


template <typename LT, int A_CT, bool LOSS, bool TMA, int MODE, bool GEN>
static vt_status launch_one(const Params& P, const TmaMaps& maps, const Plan& plan,
                            cudaStream_t st) {
  auto kern = vtrace_fused_kernel<LT, A_CT, LOSS, TMA, MODE, GEN>;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return VT_ERR_CUDA;
  // the dynamic shared-memory limit is a per-device function attribute: set once per device
  static std::atomic<unsigned long long> attr_set{0};
  const unsigned long long bit = 1ull << dev;
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem) !=
        cudaSuccess)
      return VT_ERR_CUDA;
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  const int num_sms = cb_num_sms(dev);
  if (num_sms <= 0) return VT_ERR_CUDA;
  // persistent, co-resident grid: every CTA slot of the device, never more CTAs
  // than units (cooperative launch guarantees co-residency for the look-back)
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTHREADS, plan.smem) !=
          cudaSuccess ||
      per_sm < 1)
    return VT_ERR_CUDA;
  const long long grid =
      std::min<long long>({(long long)plan.units, (long long)per_sm * num_sms, (long long)kMaxCtas});
  Params Pl = P;
  Pl.stride_q = (int)(grid / P.G);
  Pl.stride_r = (int)(grid % P.G);
  Pl.timing = nullptr;
  Pl.timing_iters = 0;
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = plan.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, Pl, maps) != cudaSuccess) return VT_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}

template <typename LT, bool LOSS, bool TMA, int MODE, bool GEN>
static vt_status dispatch_a(const Params& P, const TmaMaps& maps, const Plan& plan,
                            cudaStream_t st) {
  if constexpr (TMA) {
    if (P.A == 18) return launch_one<LT, 18, LOSS, TMA, MODE, GEN>(P, maps, plan, st);
    if (P.A == 9) return launch_one<LT, 9, LOSS, TMA, MODE, GEN>(P, maps, plan, st);
  }
  return launch_one<LT, 0, LOSS, TMA, MODE, GEN>(P, maps, plan, st);
}

template <typename LT, bool LOSS, int MODE, bool GEN>
static vt_status dispatch_t(const Params& P, const TmaMaps& maps, const Plan& plan, bool tma,
                            cudaStream_t st) {
  return tma ? dispatch_a<LT, LOSS, true, MODE, GEN>(P, maps, plan, st)
             : dispatch_a<LT, LOSS, false, MODE, GEN>(P, maps, plan, st);
}

template <typename LT, bool LOSS>
static vt_status dispatch(const Params& P, const TmaMaps& maps, const Plan& plan, bool tma,
                          cudaStream_t st) {
  // plain V-trace from logits takes the instantiation with the GEN logic compiled out
  const bool gen = P.correction != VT_CORRECTION_VTRACE || P.q_values != 0 || P.mu_lp != 0;
  return gen ? dispatch_t<LT, LOSS, EXP_MUFU, true>(P, maps, plan, tma, st)
             : dispatch_t<LT, LOSS, EXP_MUFU, false>(P, maps, plan, tma, st);
}

static bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

vt_status check_params(const vt_vtrace_params* p) {
  if (!p) return VT_ERR_INVALID_ARG;
  const float rb = p->clip_rho_threshold, cb = p->clip_c_threshold,
              pb = p->clip_pg_rho_threshold, l = p->lambda_;
  if (std::isnan(rb) || std::isnan(cb) || std::isnan(pb) || std::isnan(l)) return VT_ERR_PARAM;
  if (!(rb > 0.f) || !(cb > 0.f) || !(pb > 0.f)) return VT_ERR_PARAM;
  if (cb > rb) return VT_ERR_PARAM;  // rho_bar >= c_bar
  if (l < 0.f || l > 1.f) return VT_ERR_PARAM;
  if (p->reward_mode < 0 || p->reward_mode > 2) return VT_ERR_PARAM;
  if (p->correction < VT_CORRECTION_VTRACE || p->correction > VT_CORRECTION_ONE_STEP_IS)
    return VT_ERR_PARAM;
  if (p->correction == VT_CORRECTION_EPSILON && !(p->epsilon > 0.f && std::isfinite(p->epsilon)))
    return VT_ERR_PARAM;
  if (p->q_from_values != 0 && p->q_from_values != 1) return VT_ERR_PARAM;
  if (p->behaviour_log_probs != 0 && p->behaviour_log_probs != 1) return VT_ERR_PARAM;
  if (p->overlap_previous != 0 && p->overlap_previous != 1) return VT_ERR_PARAM;
  if (p->kernel < VT_KERNEL_AUTO || p->kernel > VT_KERNEL_LOOKBACK) return VT_ERR_PARAM;
  if (p->sm_budget < 0) return VT_ERR_PARAM;
  return VT_OK;
}

enum KernelChoice { K_CB = 0, K_LOOKBACK_TMA = 1, K_LOOKBACK_PLAIN = 2 };

static unsigned out_mask_for(bool loss, bool vs, bool pg, bool lr, bool lp, bool lm) {
  return (loss ? (OUT_DZ | OUT_DV) : 0u) | (vs ? OUT_VS : 0u) | (pg ? OUT_PG : 0u) |
         (lr ? OUT_LR : 0u) | (lp ? OUT_LP : 0u) | (lm ? OUT_LM : 0u);
}

// Which kernel a call takes (a pure function of the shape, the pointer alignment and the
// SM budget): the column-block kernel where its TMA boxes apply, else the look-back kernel,
// with TMA staging when pitches and bases are 16-byte aligned.
static KernelChoice choose_kernel(long long T, long long B, long long A, int elem,
                                  const Plan& plan, bool ptrs16, bool mu_lp, unsigned out_mask,
                                  int sms, int forced, CbPlan* cbp) {
  const bool tma = (A * BC <= 256) && (B * A < (1LL << 31)) && (T < (1LL << 31)) &&
                   ((B * A * elem) % 16 == 0) && ((B * 4) % 16 == 0) && ptrs16 &&
                   plan.Tc + 1 <= 256 && plan.smem <= kMaxSmem;
  CbPlan tmp;
  CbPlan& cp = cbp ? *cbp : tmp;
  if (forced != VT_KERNEL_LOOKBACK) {
    if (ptrs16 && cb_plan(T, B, (int)A, elem, mu_lp, out_mask, sms, cp, false)) return K_CB;
    // small shapes whose pitches or bases rule out TMA: the same kernel with plain loads
    if (cb_supported_a(A) && cb_plan(T, B, (int)A, elem, mu_lp, out_mask, sms, cp, true))
      return K_CB;
  }
  return tma ? K_LOOKBACK_TMA : K_LOOKBACK_PLAIN;
}

static vt_status common_launch(bool loss, long long T, long long B, long long A, vt_dtype dt,
                               const void* mu, const void* pi, const int32_t* actions,
                               const float* disc, const float* rew, const float* val,
                               const float* boot, const vt_vtrace_params* prm,
                               const vt_loss_weights* w, void* dlogits, float* dvalues,
                               double* partials, float* vs, float* pg_adv, float* lr,
                               float* lp, float* lm, void* ws, size_t ws_bytes,
                               cudaStream_t st, double* const* mboxes = nullptr,
                               int nlearn = 0, int self = 0) {
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
  const bool mu_lp = prm->behaviour_log_probs != 0;  // mu given as log mu(a_t) [T][B] fp32
  if (!aligned(mu, mu_lp ? 4 : elem) || !aligned(pi, elem) || !aligned(actions, 4) || !aligned(disc, 4) ||
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
  P.T = T; P.B = B; P.A = (int)A; P.T32 = (int)T; P.B32 = (int)B; P.Tc = plan.Tc; P.K = plan.K; P.G = plan.G;
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
  P.correction = prm->correction;
  P.q_values = prm->q_from_values;
  P.eps = prm->epsilon;
  P.mu_lp = mu_lp ? 1 : 0;
  P.pdl = prm->overlap_previous;  // honoured by the column-task kernels
  P.c_v = loss ? (double)w->baseline_cost : 0.0;
  P.c_e = loss ? (double)w->entropy_cost : 0.0;
  unsigned char* wsb = static_cast<unsigned char*>(ws);
  {
    const Layout Lh = make_layout(plan.Tc * BC, (int)A, elem);
    KLayout& K = P.L;
    K.pi = (unsigned)Lh.pi; K.mu = (unsigned)Lh.mu; K.a = (unsigned)Lh.a; K.r = (unsigned)Lh.r;
    K.g = (unsigned)Lh.g; K.v = (unsigned)Lh.v; K.boot = (unsigned)Lh.boot;
    K.stage = (unsigned)Lh.stage;
    for (int q = 0; q < 2; ++q) {
      K.ratio[q] = (unsigned)Lh.ratio[q]; K.td[q] = (unsigned)Lh.td[q];
      K.adv[q] = (unsigned)Lh.adv[q]; K.lse[q] = (unsigned)Lh.lse[q];
      K.csh[q] = (unsigned)Lh.csh[q]; K.rest[q] = (unsigned)Lh.rest[q];
    }
  }
  P.ws = reinterpret_cast<WsHeader*>(wsb);
  P.nlearn = nlearn;
  P.self = self;
  for (int r = 0; r < 16; ++r) P.mbox[r] = (mboxes && r < nlearn) ? (void*)mboxes[r] : nullptr;
  const WsLayout wl = ws_layout(plan);
  P.recs = reinterpret_cast<TagRec*>(wsb + wl.recs);
  P.cta_partials = reinterpret_cast<double*>(wsb + wl.cta);

  // TMA eligibility: 16-byte aligned bases and row pitches, box inner <= 256 elements
  const bool ptrs16 = aligned(mu, 16) && aligned(pi, 16) && aligned(actions, 16) &&
                      aligned(disc, 16) && aligned(rew, 16) && aligned(val, 16) &&
                      aligned(boot, 16) && (!loss || (aligned(dlogits, 16) && aligned(dvalues, 16))) &&
                      (!vs || aligned(vs, 16)) && (!pg_adv || aligned(pg_adv, 16)) &&
                      (!lr || aligned(lr, 16)) && (!lp || aligned(lp, 16)) && (!lm || aligned(lm, 16));
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return VT_ERR_CUDA;
  const int all_sms = cb_num_sms(dev);
  if (all_sms <= 0) return VT_ERR_CUDA;
  const int sms = prm->sm_budget > 0 ? std::min(prm->sm_budget, all_sms) : all_sms;
  const unsigned om = out_mask_for(loss, vs != nullptr, pg_adv != nullptr, lr != nullptr,
                                   lp != nullptr, lm != nullptr);
  CbPlan cp;
  const KernelChoice kc = choose_kernel(T, B, A, elem, plan, ptrs16, mu_lp, om, sms,
                                        prm->kernel, &cp);
  if (prm->kernel == VT_KERNEL_COLUMN_BLOCK && kc != K_CB) return VT_ERR_SHAPE;
  if (nlearn > 1 && kc != K_CB) return VT_ERR_SHAPE;  // (the in-kernel exchange is cb-only)
  if (kc == K_CB && cp.plain) {
    CbMaps cm;
    std::memset(&cm, 0, sizeof(cm));
    CbParams C;
    std::memset(&C, 0, sizeof(C));
    C.ncg = cp.ncg; C.nts = cp.nts; C.Ts = cp.Ts; C.J = cp.J; C.nstage = cp.nstage; C.g = cp.g;
    C.Bc = cp.Bc;
    C.pi = cp.pi; C.mu = cp.mu; C.a = cp.a; C.r = cp.r; C.gm = cp.gm; C.v = cp.v; C.dv = cp.dv;
    C.vs = cp.vs; C.pg = cp.pg; C.lr = cp.lr; C.lp = cp.lp; C.lm = cp.lm; C.stage = cp.stage;
    C.tx_bytes = cp.tx_bytes; C.out_mask = cp.out_mask;
    const WsLayout wl2 = ws_layout(plan);
    C.cta_recs = reinterpret_cast<TagRec*>(wsb + wl2.cb_recs);
    C.top_count = reinterpret_cast<unsigned int*>(wsb + wl2.cb_count);
    return dt == VT_BFLOAT16 ? cb_launch_bf16(loss, true, P, C, cm, cp.grid, cp.smem, dev, st)
                             : cb_launch_f32(loss, true, P, C, cm, cp.grid, cp.smem, dev, st);
  }
  if (kc == K_CB) {
    const CUtensorMapDataType ldt =
        dt == VT_BFLOAT16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const CUtensorMapDataType f32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CbMaps cm;
    std::memset(&cm, 0, sizeof(cm));
    const int seg = 4 * cp.g * (int)A;  // elements per logits column segment
    const long long nseg = B / (4 * cp.g);
    bool ok = encode_logits_3d(&cm.pi, pi, ldt, elem, seg, T, nseg, B * A, cp.Ts, cp.ncg / cp.g) &&
              (mu_lp ? encode_2d(&cm.mu, mu, f32, 4, B, T, cp.Bc, cp.Ts)
                     : encode_logits_3d(&cm.mu, mu, ldt, elem, seg, T, nseg, B * A, cp.Ts, cp.ncg / cp.g)) &&
              encode_2d(&cm.a, actions, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, B, T, cp.Bc, cp.Ts) &&
              encode_2d(&cm.r, rew, f32, 4, B, T, cp.Bc, cp.Ts) &&
              encode_2d(&cm.g, disc, f32, 4, B, T, cp.Bc, cp.Ts) &&
              encode_2d(&cm.v, val, f32, 4, B, T, cp.Bc, cp.Ts + 1);
    if (loss)
      ok = ok && encode_logits_3d(&cm.dz, dlogits, ldt, elem, seg, T, nseg, B * A, cp.Ts, cp.ncg / cp.g) &&
           encode_2d(&cm.dv, dvalues, f32, 4, B, T, cp.Bc, cp.Ts);
    if (vs) ok = ok && encode_2d(&cm.vs, vs, f32, 4, B, T, cp.Bc, cp.Ts);
    if (pg_adv) ok = ok && encode_2d(&cm.pg, pg_adv, f32, 4, B, T, cp.Bc, cp.Ts);
    if (lr) ok = ok && encode_2d(&cm.lr, lr, f32, 4, B, T, cp.Bc, cp.Ts);
    if (lp) ok = ok && encode_2d(&cm.lp, lp, f32, 4, B, T, cp.Bc, cp.Ts);
    if (lm) ok = ok && encode_2d(&cm.lm, lm, f32, 4, B, T, cp.Bc, cp.Ts);
    if (!ok) return VT_ERR_CUDA;
    CbParams C;
    std::memset(&C, 0, sizeof(C));
    C.ncg = cp.ncg; C.nts = cp.nts; C.Ts = cp.Ts; C.J = cp.J; C.nstage = cp.nstage; C.g = cp.g;
    C.Bc = cp.Bc;
    C.pi = cp.pi; C.mu = cp.mu; C.a = cp.a; C.r = cp.r; C.gm = cp.gm; C.v = cp.v; C.dv = cp.dv;
    C.vs = cp.vs; C.pg = cp.pg; C.lr = cp.lr; C.lp = cp.lp; C.lm = cp.lm; C.stage = cp.stage;
    C.tx_bytes = cp.tx_bytes; C.out_mask = cp.out_mask; C.ebuf = cp.ebuf;
    const WsLayout wl2 = ws_layout(plan);
    C.cta_recs = reinterpret_cast<TagRec*>(wsb + wl2.cb_recs);
    C.top_count = reinterpret_cast<unsigned int*>(wsb + wl2.cb_count);
    return dt == VT_BFLOAT16 ? cb_launch_bf16(loss, false, P, C, cm, cp.grid, cp.smem, dev, st)
                             : cb_launch_f32(loss, false, P, C, cm, cp.grid, cp.smem, dev, st);
  }
  TmaMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  bool tma = kc == K_LOOKBACK_TMA;
  if (tma) {
    const CUtensorMapDataType ldt =
        dt == VT_BFLOAT16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    tma = (mu_lp ? encode_2d(&maps.mu, mu, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, T, BC, plan.Tc)
                 : encode_2d(&maps.mu, mu, ldt, elem, B * A, T, BC * (int)A, plan.Tc)) &&
          encode_2d(&maps.pi, pi, ldt, elem, B * A, T, BC * (int)A, plan.Tc) &&
          encode_2d(&maps.a, actions, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, B, T, BC, plan.Tc) &&
          encode_2d(&maps.r, rew, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, T, BC, plan.Tc) &&
          encode_2d(&maps.g, disc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, T, BC, plan.Tc) &&
          encode_2d(&maps.v, val, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, T, BC, plan.Tc + 1) &&
          encode_1d(&maps.boot, boot, B, BC) &&
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

vt_status vtrace_loss_and_grad_learners(
    int64_t T, int64_t B, int64_t A, vt_dtype dt, const void* mu, const void* pi,
    const int32_t* actions, const float* discounts, const float* rewards, const float* values,
    const float* boot, const vt_vtrace_params* params, const vt_loss_weights* weights,
    void* dlogits, float* dvalues, double* partials, float* vs, float* pg_adv, void* ws,
    size_t ws_bytes, double* const* mailboxes, int32_t num_learners, int32_t self,
    vt_stream_t stream) {
  if (!mailboxes || num_learners < 1 || num_learners > 16 || self < 0 || self >= num_learners)
    return VT_ERR_INVALID_ARG;
  for (int r = 0; r < num_learners; ++r) {
    if (!mailboxes[r]) return VT_ERR_INVALID_ARG;
    if (!aligned(mailboxes[r], 16)) return VT_ERR_ALIGNMENT;
  }
  return common_launch(true, T, B, A, dt, mu, pi, actions, discounts, rewards, values, boot,
                       params, weights, dlogits, dvalues, partials, vs, pg_adv, nullptr, nullptr,
                       nullptr, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), mailboxes,
                       num_learners, self);
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
  const size_t nmu = (params && params->behaviour_log_probs) ? ns : nl;  // mu logits or log mu(a)
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
      cudaMemcpyAsync(d_mu, h_mu, nmu, h2d, st) != cudaSuccess ||
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

const char* vtrace_kernel_for(int64_t T, int64_t B, int64_t A, vt_dtype logits_dtype) {
  if (T <= 0 || B <= 0 || A <= 0 || A > VT_MAX_ACTIONS) return "none (invalid shape)";
  if (logits_dtype != VT_FLOAT32 && logits_dtype != VT_BFLOAT16) return "none (invalid dtype)";
  const int elem = logits_dtype == VT_BFLOAT16 ? 2 : 4;
  const Plan plan = make_plan(T, B, (int)A, elem);
  int dev = 0;
  const int sms = cudaGetDevice(&dev) == cudaSuccess ? cb_num_sms(dev) : 0;
  CbPlan cpk;
  switch (choose_kernel(T, B, A, elem, plan, true, false, OUT_DZ | OUT_DV, sms > 0 ? sms : 148,
                        VT_KERNEL_AUTO, &cpk)) {
    case K_CB: return cpk.plain ? "vtrace_cb_kernel (plain loads)" : "vtrace_cb_kernel";
    case K_LOOKBACK_TMA: return "vtrace_fused_kernel";
    default: return "vtrace_fused_kernel (plain loads)";
  }
}

}  // extern "C"
