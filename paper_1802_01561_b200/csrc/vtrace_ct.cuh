// vtrace_ct.cuh -- "column-task" fused kernel: one warp owns CT_COLS = 4
// trajectories over the whole unroll and walks it backwards in chunks of
// CT_STEPS = 8 steps (4 x 8 = 32 rows = one row per lane), carrying the
// V-trace recursion state A = v - V from chunk to chunk in registers.
//
// Used when the batch is wide enough to occupy the GPU with such tasks
// (ceil(B/4) >= a few per SM), e.g. the large-batch learner (T=100,
// B=8192): no look-back, no block barriers, no shared-memory round trip of
// row state, and the target logits row stays in registers from the log-softmax
// statistics to the gradient.  Per chunk, per lane (= row (t, b)):
//   a3-a6  m, sum exp, ratio pi/mu (fp64), lse, entropy terms
//   a7     delta_t = rho_t (r_t + gamma_t V_{t+1} - V_t), g_t = gamma_t c_t
//   a8     suffix scan of the affine maps (g, delta) over the chunk's 8 steps
//          (3 shuffle levels), A_t = D_t + G_t * carry          (Remark 1)
//   a9     q_t / pg_adv_t from A_{t+1}
//   a10-11 dL/dz written in place over the z^pi tile, one TMA store per chunk
// TMA: CT_NSTAGE-stage ring per warp (CT_NSTAGE-1 chunks in flight while one is computed).
#pragma once
// (included inside namespace vtb200 by vtrace_api.cu)

constexpr int CT_COLS = 4;
constexpr int CT_STEPS = 8;
constexpr int CT_ROWS = CT_COLS * CT_STEPS;  // 32 == warp size
#ifndef VTRACE_CT_NSTAGE
#define VTRACE_CT_NSTAGE 5
#endif
constexpr int CT_NSTAGE = VTRACE_CT_NSTAGE;  // chunks in flight + the one computed
constexpr int CT_WARPS = 1;                  // warps (tasks) per CTA
constexpr int CT_GROUP = 32;                 // tasks per partials group
static_assert(CT_ROWS == 32, "one row per lane");

struct CtLayout {
  size_t pi, mu, a, r, g, v, stage, boot, warp_bytes;
};

__host__ __device__ inline CtLayout make_ct_layout(int A, int elem) {
  CtLayout L;
  size_t off = 0;
  L.pi = off; off = a128(off + (size_t)CT_ROWS * A * elem);
  L.mu = off; off = a128(off + (size_t)CT_ROWS * A * elem);
  L.a = off;  off = a128(off + (size_t)CT_ROWS * 4);
  L.r = off;  off = a128(off + (size_t)CT_ROWS * 4);
  L.g = off;  off = a128(off + (size_t)CT_ROWS * 4);
  L.v = off;  off = a128(off + (size_t)(CT_ROWS + CT_COLS) * 4);  // one step past the chunk
  L.stage = off;
  L.boot = CT_NSTAGE * L.stage;
  L.warp_bytes = a128(L.boot + (size_t)CT_COLS * 4);
  return L;
}

struct CtParams {
  unsigned int pi, mu, a, r, g, v, stage, boot, warp_bytes;  // CtLayout, 32-bit
  int tasks, groups, K;
  double* task_partials;   // [tasks][NPART]
  double* group_partials;  // [groups][NPART]
  unsigned int* group_count;  // [groups], re-armed to 0 by the last arriver
  unsigned int* top_count;
};

template <typename LT, int A_CT, bool LOSS, int MODE>
__global__ void __launch_bounds__(CT_WARPS * 32)
    vtrace_ct_kernel(const Params P, const CtParams C, const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[CT_WARPS][CT_NSTAGE];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * CT_WARPS + warp;
  if (task >= C.tasks) return;  // warp-uniform
  const int A = (A_CT > 0) ? A_CT : P.A;
  const int T = P.T32, B = P.B32;
  const int b0 = task * CT_COLS;
  const int blen = min(CT_COLS, B - b0);
  const int K = C.K;
  unsigned char* base = smem + (size_t)warp * C.warp_bytes;
  uint64_t* wb = bar[warp];
  const uint32_t stage_bytes = (uint32_t)(2 * (size_t)CT_ROWS * A * sizeof(LT) +
                                          3 * CT_ROWS * 4 + (CT_ROWS + CT_COLS) * 4);

  // chunk of iteration `it` (reverse time): k = K - 1 - it, t0 = 8 k
  auto load_iter = [&](int it) {  // lane 0 only
    if (it >= K) return;
    const int st = it % CT_NSTAGE;
    const int t0 = (K - 1 - it) * CT_STEPS;
    unsigned char* sb = base + (size_t)st * C.stage;
    const uint32_t extra = (it == 0) ? (uint32_t)(CT_COLS * 4) : 0u;
    mbar_expect_tx(&wb[st], stage_bytes + extra);
    tma_load_2d(sb + C.pi, &maps.pi, b0 * A, t0, &wb[st]);
    tma_load_2d(sb + C.mu, &maps.mu, b0 * A, t0, &wb[st]);
    tma_load_2d(sb + C.a, &maps.a, b0, t0, &wb[st]);
    tma_load_2d(sb + C.r, &maps.r, b0, t0, &wb[st]);
    tma_load_2d(sb + C.g, &maps.g, b0, t0, &wb[st]);
    tma_load_2d(sb + C.v, &maps.v, b0, t0, &wb[st]);
    if (it == 0) tma_load_1d(base + C.boot, &maps.boot, b0, &wb[st]);
  };
  if (lane == 0) {
    for (int s = 0; s < CT_NSTAGE; ++s) mbar_init(&wb[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int it = 0; it < CT_NSTAGE; ++it) load_iter(it);
  }
  __syncwarp();

  const float ce = (float)P.c_e;
  const float cv = (float)P.c_v;
  const float rho_bar_f = (float)P.rho_bar;
  const int tl = lane >> 2, c = lane & 3;  // row (tl, c) of the [8 steps][4 columns] chunk
  float acc_pg = 0.f, acc_v = 0.f, acc_H = 0.f, acc_dz = 0.f, acc_dv = 0.f, acc_rho = 0.f,
        acc_clip = 0.f;
  double carry = 0.0;  // A = v - V just after the current chunk, for column c (A_T = 0)

  int st = 0;                 // it % CT_NSTAGE
  uint32_t phase = 0;         // (it / CT_NSTAGE) & 1
  for (int it = 0; it < K; ++it) {
    const int t0 = (K - 1 - it) * CT_STEPS;
    const int tlen = min(CT_STEPS, T - t0);
    unsigned char* sb = base + (size_t)st * C.stage;
    mbar_wait(&wb[st], phase);
    const bool row_ok = (tl < tlen) && (c < blen);
    const int r = lane;
    LT* zrow = reinterpret_cast<LT*>(sb + C.pi) + (size_t)r * A;

    // ---- a3-a7: statistics of this lane's row ----------------------------------
    // Every lane computes its row; rows past the end of the unroll (the last
    // chunk only; TMA zero-filled) are masked out of the scan and the outputs.
    RowRegs<LT, A_CT> zp;
    float lse, cshift, rest, Vt, gm;
    double ratio, td, dl, gc;
    int a;
    {
      const int a_raw = reinterpret_cast<const int*>(sb + C.a)[r];
      a = min(max(a_raw, 0), A - 1);
      float m_p, m_m, sed_p, sed_m, ea_p, ea_m;
      double S_p, S_m, xa_p, xa_m;
      bool fin_p, fin_m;
      zp.load(zrow);
      if constexpr (A_CT > 0 && MODE == EXP_MUFU) {
        RowRegs<LT, A_CT> zm;
        zm.load(reinterpret_cast<const LT*>(sb + C.mu) + (size_t)r * A);
        RowStat sp, sm;
        row_stats2<LT, A_CT>(zp, zm, a, sp, sm);
        m_p = sp.m; S_p = sp.S; xa_p = sp.xa; ea_p = sp.ea_f; sed_p = sp.sed; fin_p = sp.finite;
        m_m = sm.m; S_m = sm.S; xa_m = sm.xa; ea_m = sm.ea_f; sed_m = sm.sed; fin_m = sm.finite;
      } else {
        row_stats<LT, A_CT, MODE>(zp, A, a, m_p, S_p, xa_p, ea_p, sed_p, fin_p);
        RowRegs<LT, A_CT> zm;
        zm.load(reinterpret_cast<const LT*>(sb + C.mu) + (size_t)r * A);
        row_stats<LT, A_CT, MODE>(zm, A, a, m_m, S_m, xa_m, ea_m, sed_m, fin_m);
      }
      // pi(a)/mu(a) = exp((z^pi_a - m_pi) - (z^mu_a - m_mu)) S_mu / S_pi
      ratio = exp64(xa_p - xa_m) * (S_m / S_p);
      const float rt = reinterpret_cast<const float*>(sb + C.r)[r];
      gm = reinterpret_cast<const float*>(sb + C.g)[r];
      Vt = reinterpret_cast<const float*>(sb + C.v)[r];
      // V(x_{t+1}): the V tile has one extra step; the last step of the unroll
      // bootstraps from V(x_T)
      const float Vn = (tl + 1 < tlen || it > 0)
                           ? reinterpret_cast<const float*>(sb + C.v)[r + CT_COLS]
                           : reinterpret_cast<const float*>(base + C.boot)[c];
      td = reward_transform(rt, P.reward_mode) + (double)gm * (double)Vn - (double)Vt;
      dl = dmin_t(P.rho_bar, ratio) * td;                         // delta_t V
      gc = (double)gm * (P.lambda * dmin_t(P.c_bar, ratio));      // gamma_t c_t
      const float Sf = (float)S_p;
      const float inv_S = rcp_approx(Sf);
      lse = m_p + __logf(Sf);
      cshift = fmaf(sed_p, inv_S, m_p);  // lse - H
      rest = (float)(S_p - (double)ea_p) * inv_S;
      if (row_ok) {
        acc_rho += fminf(rho_bar_f, (float)ratio);
        acc_clip += (ratio > P.rho_bar) ? 1.f : 0.f;
      }
      const long long row = (long long)(t0 + tl) * B + b0 + c;
      if (!LOSS && row_ok) {
        if (P.has_lr) P.log_rhos[row] = (float)log(ratio);
        if (P.has_lp) P.lp_out[row] = (float)(xa_p - log(S_p));
        if (P.has_lm) P.lm_out[row] = (float)(xa_m - log(S_m));
      }
      const bool bad = row_ok && ((a_raw != a) || !(fin_p && fin_m) || !isfinite(rt) ||
                                  !isfinite(Vt) || !isfinite(Vn) || !(gm >= 0.f && gm <= 1.f));
      if (!row_ok) {
        dl = 0.0;  // identity map for steps past the end of the unroll
        gc = 1.0;
      }
      if (bad) {
        if (a_raw != a) record_bad(P.ws, row, VT_DATA_ACTION);
        if (!(fin_p && fin_m)) record_bad(P.ws, row, VT_DATA_LOGITS);
        if (!isfinite(rt)) record_bad(P.ws, row, VT_DATA_REWARD);
        if (!isfinite(Vt)) record_bad(P.ws, row, VT_DATA_VALUE);
        if (!(gm >= 0.f && gm <= 1.f)) record_bad(P.ws, row, VT_DATA_DISCOUNT);
        if (!isfinite(Vn) && it == 0 && tl + 1 == tlen)
          record_bad(P.ws, (long long)T * B + b0 + c, VT_DATA_VALUE);  // the bootstrap
      }
    }

    // ---- a8: suffix scan of the chunk's affine maps, per column ----------------
    // lanes c, c+4, ..., c+28 are steps 0..7 of column c; composing later steps:
    // (G1, D1) o (G2, D2) = (G1 G2, D1 + G1 D2)
    double Gi = gc, Di = dl;
#pragma unroll
    for (int o = CT_COLS; o < 32; o <<= 1) {
      const double Go = shfl_down_d(Gi, o), Do = shfl_down_d(Di, o);
      const bool in = lane + o < 32;  // beyond the chunk: identity map
      Di = fma(Gi, in ? Do : 0.0, Di);
      Gi = Gi * (in ? Go : 1.0);
    }
    const double A_t = fma(Gi, carry, Di);                 // A_t = v_t - V(x_t)
    double A_n = shfl_down_d(A_t, CT_COLS);                // A_{t+1}
    if (tl + 1 >= tlen) A_n = carry;
    carry = __shfl_sync(0xffffffffu, A_t, c);              // A at the chunk's first step

    // ---- a9-a11: advantages, value gradient, policy gradient ------------------
    if (row_ok) {
      const long long row = (long long)(t0 + tl) * B + b0 + c;
      // pg_adv = rho_pg (r + gamma v_{t+1} - V) = rho_pg (td + gamma A_{t+1})
      const float pgr = (float)(dmin_t(P.pg_rho_bar, ratio) * fma((double)gm, A_n, td));
      if (P.vs) P.vs[row] = (float)((double)Vt + A_t);
      if (P.pg_adv) P.pg_adv[row] = pgr;
      if constexpr (LOSS) {
        const float Ar = (float)A_t;
        const float pa = 1.f - rest;
        const float za = Elem<LT>::get(zrow, a);
        const float L2E = 1.44269504088896341f;
        const float lseL = lse * L2E;
        const float alpha = fmaf(-ce, cshift, pgr);  // pg + c_e (z_j - cshift) = alpha + c_e z_j
        float sq = 0.f;
        // dz_j = pi_j (pg + c_e (log pi_j + H))   (j != a), in place over z
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
        const float d_a = fmaf(-pgr, rest, ce * pa * (za - cshift));
        zrow[a] = store_cvt<LT>(d_a);
        sq = __fadd_rn(__fsub_rn(sq, __fmul_rn(d_wrong, d_wrong)), __fmul_rn(d_a, d_a));
        const float dv = -cv * Ar;  // c_v (V - v)
        P.dvalues[row] = dv;
        acc_pg = fmaf(-pgr, za - lse, acc_pg);  // -pg_adv log pi(a)
        acc_v = fmaf(0.5f * Ar, Ar, acc_v);
        acc_H += lse - cshift;
        acc_dz += sq;
        acc_dv = fmaf(dv, dv, acc_dv);
      }
    }
    if constexpr (LOSS) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&maps.dz, b0 * A, t0, sb + C.pi);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      __syncwarp();
    }
    if (lane == 0 && it >= 1) {
      // the stage of iteration it-1 (== that of it + NSTAGE - 1): its gradient store
      // must have read it (this iteration's store may stay in flight); then refill
      if constexpr (LOSS) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      fence_proxy_async_smem();
      load_iter(it + CT_NSTAGE - 1);
    }
    __syncwarp();
    if (++st == CT_NSTAGE) {
      st = 0;
      phase ^= 1u;
    }
  }
  if constexpr (LOSS) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    // ---- a12: partial sums: task -> group of 32 tasks -> total, fixed orders ----
    double part[NPART] = {acc_pg, acc_v, acc_H, 0.0, acc_dz, acc_dv, acc_rho, acc_clip};
#pragma unroll
    for (int k = 0; k < NPART; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part[k] += __shfl_xor_sync(0xffffffffu, part[k], o);
    }
    if (P.partials == nullptr) return;
    if (lane < NPART) {
      double v = part[0];
#pragma unroll
      for (int k = 1; k < NPART; ++k) v = (lane == k) ? part[k] : v;
      C.task_partials[(size_t)task * NPART + lane] = v;
    }
    __threadfence();
    __syncwarp();
    const int grp = task / CT_GROUP;
    const int g0 = grp * CT_GROUP, gn = min(CT_GROUP, C.tasks - g0);
    unsigned int prev = 0;
    if (lane == 0) prev = atomicAdd(C.group_count + grp, 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != (unsigned int)(gn - 1)) return;  // not the last task of the group
    __threadfence();
    // lane l holds task g0 + l; reduce the group in a fixed tree per partial
    double gp[NPART];
#pragma unroll
    for (int k = 0; k < NPART; ++k)
      gp[k] = lane < gn ? __ldcg(C.task_partials + (size_t)(g0 + lane) * NPART + k) : 0.0;
#pragma unroll
    for (int k = 0; k < NPART; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gp[k] += __shfl_xor_sync(0xffffffffu, gp[k], o);
    }
    if (lane < NPART) {
      double v = gp[0];
#pragma unroll
      for (int k = 1; k < NPART; ++k) v = (lane == k) ? gp[k] : v;
      C.group_partials[(size_t)grp * NPART + lane] = v;
    }
    if (lane == 0) C.group_count[grp] = 0u;  // re-arm for the next call
    __threadfence();
    __syncwarp();
    if (lane == 0) prev = atomicAdd(C.top_count, 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != (unsigned int)(C.groups - 1)) return;
    __threadfence();
    // the last group: lanes stride the groups (fixed order), then a fixed tree
    double tp[NPART];
#pragma unroll
    for (int k = 0; k < NPART; ++k) tp[k] = 0.0;
    for (int gi = lane; gi < C.groups; gi += 32) {
#pragma unroll
      for (int k = 0; k < NPART; ++k) tp[k] += __ldcg(C.group_partials + (size_t)gi * NPART + k);
    }
#pragma unroll
    for (int k = 0; k < NPART; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tp[k] += __shfl_xor_sync(0xffffffffu, tp[k], o);
    }
    if (lane == 0) {
      tp[VT_P_TOTAL_LOSS] =
          tp[VT_P_PG_LOSS] + P.c_v * tp[VT_P_BASELINE_LOSS] - P.c_e * tp[VT_P_ENTROPY_SUM];
#pragma unroll
      for (int k = 0; k < NPART; ++k) P.partials[k] = tp[k];
      *C.top_count = 0u;
    }
  }
}

