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
// Inputs: the two logits tiles by TMA (CT_NSTAGE-stage ring per warp); the
// per-step a, r, gamma, V, V' by plain coalesced loads one chunk ahead.

#pragma once
// (included inside namespace vtb200 by vtrace_api.cu)

constexpr int CT_COLS = 4;
constexpr int CT_STEPS = 8;
constexpr int CT_ROWS = CT_COLS * CT_STEPS;  // 32 == warp size
constexpr int CT_NSTAGE = 4;                 // logits stages: chunks in flight + the one computed
constexpr int CT_WARPS = 1;                  // warps (tasks) per CTA
constexpr int CT_GROUP = 32;                 // tasks per partials group
static_assert(CT_ROWS == 32, "one row per lane");

struct CtLayout {
  size_t pi, mu, stage, warp_bytes;
};

__host__ __device__ inline CtLayout make_ct_layout(int A, int elem) {
  CtLayout L;
  size_t off = 0;
  L.pi = off; off = a128(off + (size_t)CT_ROWS * A * elem);
  L.mu = off; off = a128(off + (size_t)CT_ROWS * A * elem);
  L.stage = off;
  L.warp_bytes = CT_NSTAGE * L.stage;
  return L;
}

struct CtParams {
  unsigned int pi, mu, stage, warp_bytes;  // CtLayout, 32-bit
  int tasks, K, groups;
  double* task_partials;   // [tasks][NPART]
  double* group_partials;  // [groups][NPART]
  unsigned int* group_count;  // [groups], re-armed to 0 by the last arriver
  unsigned int* top_count;
};

__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }

// Statistics of both policies' rows (fast path: MUFU exps, compile-time even A).
// Same scheme as row_stats2 (precision): e_j = 2^{y_j} with
// y_j = fma(z_j, L16, -m L16) for bf16 (exact products, max term exactly 1) or
// (z_j - m) L32 for fp32; Fast2Sum chains that start at 1 >= every term (one
// chain per half of the float2); the log2 e truncation corrected to first order
// through sd = sum_j e_j (z_j - m).  The target's (z_j, e_j) pairs are returned
// for the gradient.
template <typename LT, int A_CT>
struct CtStats {
  static constexpr int NP = A_CT / 2;
  float2 z[NP], e[NP];   // target row and its exps (kept for a10-a11)
  float m_p, sd_p, ea_p; // max, sum e (z - m), exp(z_a - m) (corrected)
  double S_p, S_m;       // sums (corrected)
  double xa_p, xa_m;     // z_a - m per policy (exact)
  bool finite;
};

template <typename LT, int A_CT>
__device__ __forceinline__ void ct_stats_fast(const LT* zrow, const LT* mrow, int a,
                                              CtStats<LT, A_CT>& R) {
  constexpr int NP = A_CT / 2;
  constexpr bool BF16 = sizeof(LT) == 2;
  constexpr float L16 = 1.44268798828125f;  // log2 e to 16 bits
  constexpr float L32 = 1.44269502f;        // fp32(log2 e)
  constexpr float CORR = BF16 ? 4.8884952e-06f : 1.3349930e-08f;  // ln2 (log2 e - L)
  float2 zm[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    if constexpr (BF16) {
      const uint32_t xp = reinterpret_cast<const uint32_t*>(zrow)[k];
      const uint32_t xm = reinterpret_cast<const uint32_t*>(mrow)[k];
      R.z[k] = make_float2(__uint_as_float(xp << 16), __uint_as_float(xp & 0xffff0000u));
      zm[k] = make_float2(__uint_as_float(xm << 16), __uint_as_float(xm & 0xffff0000u));
    } else {
      R.z[k] = reinterpret_cast<const float2*>(zrow)[k];
      zm[k] = reinterpret_cast<const float2*>(mrow)[k];
    }
  }
  float mp = fmaxf(R.z[0].x, R.z[0].y), mm = fmaxf(zm[0].x, zm[0].y);
#pragma unroll
  for (int k = 1; k < NP; ++k) {
    mp = fmaxf(mp, fmaxf(R.z[k].x, R.z[k].y));
    mm = fmaxf(mm, fmaxf(zm[k].x, zm[k].y));
  }
  // exponent y = z L - m L (bf16) or (z - m) L32 (fp32), two elements per instruction
  const float2 Lp = f2(BF16 ? L16 : L32);
  const float2 nmLp = f2(BF16 ? -mp * L16 : 0.f), nmLm = f2(BF16 ? -mm * L16 : 0.f);
  const float2 nmp = f2(-mp), nmm = f2(-mm);
  float2 hp = f2(1.f), lp = f2(0.f), hm = f2(1.f), lm = f2(0.f), sdp = f2(0.f), sdm = f2(0.f);
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    float2 yp, ym, dp, dm;
    if constexpr (BF16) {
      yp = __ffma2_rn(R.z[k], Lp, nmLp);
      ym = __ffma2_rn(zm[k], Lp, nmLm);
      dp = R.z[k];  // sum e z; (z - m) applied once per row below
      dm = zm[k];
    } else {
      dp = __fadd2_rn(R.z[k], nmp);
      dm = __fadd2_rn(zm[k], nmm);
      yp = __fmul2_rn(dp, Lp);
      ym = __fmul2_rn(dm, Lp);
    }
    const float2 ep = make_float2(ex2_approx(yp.x), ex2_approx(yp.y));
    const float2 em = make_float2(ex2_approx(ym.x), ex2_approx(ym.y));
    R.e[k] = ep;
    sdp = __ffma2_rn(ep, dp, sdp);  // NaN if some z is inf/nan (0 * inf for -inf)
    sdm = __ffma2_rn(em, dm, sdm);
    // Fast2Sum: h >= 1 >= e, so s = h + e and (h - s) + e is its exact error
    const float2 np = __fadd2_rn(hp, ep), nm = __fadd2_rn(hm, em);
    lp = __fadd2_rn(lp, __fadd2_rn(__fadd2_rn(hp, make_float2(-np.x, -np.y)), ep));
    lm = __fadd2_rn(lm, __fadd2_rn(__fadd2_rn(hm, make_float2(-nm.x, -nm.y)), em));
    hp = np;
    hm = nm;
  }
  // finish both policies at once (.x = pi, .y = mu): the chains started at 1, so
  // h - 1 is exact; TwoSum of the two chain heads, then the low parts
  const float2 h0 = __fadd2_rn(make_float2(hp.x, hm.x), f2(-1.f));
  const float2 h1 = __fadd2_rn(make_float2(hp.y, hm.y), f2(-1.f));
  const float2 s = __fadd2_rn(h0, h1);
  const float2 bb = __fadd2_rn(s, make_float2(-h0.x, -h0.y));
  const float2 err = __fadd2_rn(__fadd2_rn(h0, make_float2(bb.x - s.x, bb.y - s.y)),
                                __fadd2_rn(h1, make_float2(-bb.x, -bb.y)));
  float2 sd = make_float2(sdp.x + sdp.y, sdm.x + sdm.y);
  if constexpr (BF16)  // sum e (z - m) = sum e z - m sum e
    sd = __ffma2_rn(make_float2(-mp, -mm), s, sd);
  const float2 lo = __ffma2_rn(sd, f2(CORR), __fadd2_rn(err, __fadd2_rn(make_float2(lp.x, lm.x),
                                                                        make_float2(lp.y, lm.y))));
  R.S_p = (double)s.x + (double)lo.x;
  R.S_m = (double)s.y + (double)lo.y;
  R.m_p = mp;
  R.sd_p = sd.x;
  // gathered terms: z_a - m exactly (fp64), and exp(z^pi_a - m) as in the sum, corrected
  const float zap = Elem<LT>::get(zrow, a), zam = Elem<LT>::get(mrow, a);
  R.xa_p = (double)zap - (double)mp;
  R.xa_m = (double)zam - (double)mm;
  const float ya = BF16 ? fmaf(zap, L16, -mp * L16) : (zap - mp) * L32;
  const float ea = ex2_approx(ya);
  R.ea_p = fmaf(ea * CORR, zap - mp, ea);
  R.finite = isfinite(sd.x) && isfinite(sd.y) && isfinite(mp) && isfinite(mm);
}

// a12 for one task: its partial sums -> group of CT_GROUP tasks -> total, in fixed
// orders (the last arriver of a group reduces it; the last group the total).
__device__ __forceinline__ void ct_unit_partials(const Params& P, const CtParams& C, int u,
                                                 int lane, double (&part)[NPART]) {
#pragma unroll
  for (int k = 0; k < NPART; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part[k] += __shfl_xor_sync(0xffffffffu, part[k], o);
  }
  if (lane < NPART) {
    double v = part[0];
#pragma unroll
    for (int k = 1; k < NPART; ++k) v = (lane == k) ? part[k] : v;
    C.task_partials[(size_t)u * NPART + lane] = v;
  }
  __threadfence();
  __syncwarp();
  const int grp = u / CT_GROUP;
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

template <typename LT, int A_CT, bool LOSS, int MODE>
__global__ void __launch_bounds__(CT_WARPS * 32)
    vtrace_ct_kernel(const Params P, const CtParams C, const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[CT_WARPS][CT_NSTAGE];
  constexpr bool kFast = (A_CT > 0) && (A_CT % 2 == 0) && (MODE == EXP_MUFU);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * CT_WARPS + warp;
  if (task >= C.tasks) return;  // warp-uniform
  const int A = (A_CT > 0) ? A_CT : P.A;
  const int T = P.T32, B = P.B32;
  const int K = C.K;
  const int b0 = task * CT_COLS;
  const int blen = min(CT_COLS, B - b0);
  unsigned char* base = smem + (size_t)warp * C.warp_bytes;
  uint64_t* wb = bar[warp];
  const uint32_t tile_bytes = (uint32_t)((size_t)CT_ROWS * A * sizeof(LT));
  constexpr int it_begin = 0;
  const int it_end = K;

  // chunk of iteration `it` (reverse time): k = K - 1 - it, t0 = 8 k; stage it mod NSTAGE
  auto load_iter = [&](int it) {  // lane 0 only
    if (it >= it_end) return;
    const int stg = it % CT_NSTAGE;
    const int t0 = (K - 1 - it) * CT_STEPS;
    unsigned char* sb = base + (size_t)stg * C.stage;
    mbar_expect_tx(&wb[stg], 2 * tile_bytes);
    tma_load_2d(sb + C.pi, &maps.pi, b0 * A, t0, &wb[stg]);
    tma_load_2d(sb + C.mu, &maps.mu, b0 * A, t0, &wb[stg]);
  };
  if (lane == 0) {
    for (int s = 0; s < CT_NSTAGE; ++s) mbar_init(&wb[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < CT_NSTAGE; ++i) load_iter(i);
  }
  __syncwarp();
  uint32_t phase_bits = 0;  // bit s: parity of stage s's next completion

  const float ce = (float)P.c_e;
  const float cv = (float)P.c_v;
  const float rho_bar_f = (float)P.rho_bar;
  const int tl = lane >> 2, c = lane & 3;  // row (tl, c) of the [8 steps][4 columns] chunk
  const long long stepB = (long long)CT_STEPS * B;
  float acc_pg = 0.f, acc_v = 0.f, acc_H = 0.f, acc_dz = 0.f, acc_dv = 0.f, acc_rho = 0.f,
        acc_clip = 0.f;
  double carry = 0.0;  // A = v - V just after the current chunk, for column c (A_T = 0)

  // per-step inputs of one chunk (a, r, gamma, V(x_t), V(x_{t+1})), loaded one chunk
  // ahead; `off` = flat index t * B + b of this lane's row, stepped back 8 B per chunk
  struct StepIn {
    int a;
    float r, g, v, vn;
  };
  const long long off0 = (long long)((K - 1) * CT_STEPS + tl) * B + b0 + c;
  const float* const bootp = P.boot + b0 + c;
  auto load_step = [&](int it, long long off, StepIn& s) {
    const int t = (K - 1 - it) * CT_STEPS + tl;
    s.a = 0; s.r = 0.f; s.g = 0.f; s.v = 0.f; s.vn = 0.f;
    if (t < T && c < blen) {
      s.a = __ldg(P.actions + off);
      s.r = __ldg(P.rew + off);
      s.g = __ldg(P.disc + off);
      s.v = __ldg(P.val + off);
      // V(x_{t+1}); the last step of the unroll bootstraps from V(x_T)
      s.vn = __ldg((t + 1 < T) ? P.val + off + B : bootp);
    }
  };
  StepIn cur, nxt;
  load_step(0, off0, cur);
  nxt = cur;

  int st = 0;  // (it - it_begin) mod NSTAGE
  long long off = off0;  // this iteration's row
  for (int it = it_begin; it < it_end; ++it, off -= stepB) {
    if (it + 1 < it_end) load_step(it + 1, off - stepB, nxt);
    const int t0 = (K - 1 - it) * CT_STEPS;
    const int tlen = min(CT_STEPS, T - t0);
    unsigned char* sb = base + (size_t)st * C.stage;
    const bool row_ok = (tl < tlen) && (c < blen);
    LT* zrow = reinterpret_cast<LT*>(sb + C.pi) + lane * A;
    const LT* mrow = reinterpret_cast<const LT*>(sb + C.mu) + lane * A;
    const int a_raw = cur.a;
    const int a = min(max(a_raw, 0), A - 1);
    mbar_wait(&wb[st], (phase_bits >> st) & 1u);
    phase_bits ^= 1u << st;

    // ---- a3-a7: statistics of this lane's row ----------------------------------
    // Every lane computes its row; rows past the end of the unroll (the first
    // iteration only; TMA zero-filled) are masked out of the scan and the outputs.
    float m_p, sed_p, ea_p;
    double S_p, S_m, xa_p, xa_m;
    bool fin;
    [[maybe_unused]] CtStats<LT, (kFast ? A_CT : 2)> F;
    [[maybe_unused]] RowRegs<LT, A_CT> zp;
    if constexpr (kFast) {
      ct_stats_fast<LT, A_CT>(zrow, mrow, a, F);
      m_p = F.m_p; sed_p = F.sd_p; ea_p = F.ea_p; S_p = F.S_p; S_m = F.S_m;
      xa_p = F.xa_p; xa_m = F.xa_m;
      fin = F.finite;
    } else {
      float m_m, sed_m, ea_m;
      bool fin_p, fin_m;
      zp.load(zrow);
      row_stats<LT, A_CT, MODE>(zp, A, a, m_p, S_p, xa_p, ea_p, sed_p, fin_p);
      RowRegs<LT, A_CT> zm;
      zm.load(mrow);
      row_stats<LT, A_CT, MODE>(zm, A, a, m_m, S_m, xa_m, ea_m, sed_m, fin_m);
      fin = fin_p && fin_m;
    }
    // pi(a)/mu(a) = exp((z^pi_a - m_pi) - (z^mu_a - m_mu)) S_mu / S_pi
    const double ratio = exp64(xa_p - xa_m) * (S_m / S_p);
    const float rt = cur.r, gm = cur.g, Vt = cur.v, Vn = cur.vn;
    const double td = reward_transform(rt, P.reward_mode) + (double)gm * (double)Vn - (double)Vt;
    double dl = dmin_t(P.rho_bar, ratio) * td;                         // delta_t V
    double gc = (double)gm * (P.lambda * dmin_t(P.c_bar, ratio));      // gamma_t c_t
    const float Sf = (float)S_p;
    const float inv_S = rcp_approx(Sf);
    const float lse = m_p + __logf(Sf);
    const float cshift = fmaf(sed_p, inv_S, m_p);  // lse - H
    const float rest = (float)(S_p - (double)ea_p) * inv_S;  // 1 - pi(a)
    if (row_ok) {
      acc_rho += fminf(rho_bar_f, (float)ratio);
      acc_clip += (ratio > P.rho_bar) ? 1.f : 0.f;
    }
    if (!LOSS && row_ok) {
      const long long row = off;
      if (P.has_lr) P.log_rhos[row] = (float)log(ratio);
      if (P.has_lp) P.lp_out[row] = (float)(xa_p - log(S_p));
      if (P.has_lm) P.lm_out[row] = (float)(xa_m - log(S_m));
    }
    const bool bad = row_ok && ((a_raw != a) || !fin || !isfinite(rt) || !isfinite(Vt) ||
                                !isfinite(Vn) || !(gm >= 0.f && gm <= 1.f));
    if (!row_ok) {
      dl = 0.0;  // identity map for steps past the end of the unroll
      gc = 1.0;
    }
    if (bad) {
      const long long row = off;
      if (a_raw != a) record_bad(P.ws, row, VT_DATA_ACTION);
      if (!fin) record_bad(P.ws, row, VT_DATA_LOGITS);
      if (!isfinite(rt)) record_bad(P.ws, row, VT_DATA_REWARD);
      if (!isfinite(Vt)) record_bad(P.ws, row, VT_DATA_VALUE);
      if (!(gm >= 0.f && gm <= 1.f)) record_bad(P.ws, row, VT_DATA_DISCOUNT);
      if (!isfinite(Vn) && t0 + tl + 1 == T)
        record_bad(P.ws, (long long)T * B + b0 + c, VT_DATA_VALUE);  // the bootstrap
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
      const long long row = off;
      // pg_adv = rho_pg (r + gamma v_{t+1} - V) = rho_pg (td + gamma A_{t+1})
      const float pgr = (float)(dmin_t(P.pg_rho_bar, ratio) * fma((double)gm, A_n, td));
      if (P.vs) P.vs[row] = (float)((double)Vt + A_t);
      if (P.pg_adv) P.pg_adv[row] = pgr;
      if constexpr (LOSS) {
        const float Ar = (float)A_t;
        const float za = Elem<LT>::get(zrow, a);
        const float alpha = fmaf(-ce, cshift, pgr);  // pg + c_e (z_j - cshift) = alpha + c_e z_j
        float sq, d_wrong;
        // dz_j = pi_j (pg + c_e (log pi_j + H))   (j != a), in place over z
        if constexpr (kFast) {
          // pi_j = e_j (1 + CORR (z_j - m)) / S  (the exps of the statistics, same
          // first-order log2 e correction as the sum)
          constexpr bool BF16 = sizeof(LT) == 2;
          constexpr float CORR = BF16 ? 4.8884952e-06f : 1.3349930e-08f;
          const float2 u1 = f2(CORR * inv_S), u0 = f2(inv_S * fmaf(-CORR, m_p, 1.f));
          const float2 ce2 = f2(ce), al2 = f2(alpha);
          float2 sq2 = f2(0.f);
#pragma unroll
          for (int k = 0; k < A_CT / 2; ++k) {
            const float2 t2 = __ffma2_rn(ce2, F.z[k], al2);
            const float2 w2 = __ffma2_rn(u1, F.z[k], u0);
            const float2 d2 = __fmul2_rn(__fmul2_rn(F.e[k], w2), t2);
            sq2 = __ffma2_rn(d2, d2, sq2);
            if constexpr (BF16) {
              __nv_bfloat162 h2 = __floats2bfloat162_rn(d2.x, d2.y);
              reinterpret_cast<uint32_t*>(zrow)[k] = *reinterpret_cast<uint32_t*>(&h2);
            } else {
              reinterpret_cast<float2*>(zrow)[k] = d2;
            }
          }
          sq = sq2.x + sq2.y;
          // the value the loop produced for j = a (same operations, bit-identical)
          const float ya = BF16 ? fmaf(za, 1.44268798828125f, -m_p * 1.44268798828125f)
                                : (za - m_p) * 1.44269502f;
          d_wrong = (ex2_approx(ya) * fmaf(CORR * inv_S, za, inv_S * fmaf(-CORR, m_p, 1.f))) *
                    fmaf(ce, za, alpha);
        } else {
          const float L2E = 1.44269504088896341f;
          const float lseL = lse * L2E;
          sq = 0.f;
          for (int j = 0; j < A; ++j) {
            const float z = zp.get(j);
            const float d = ex2_approx(fmaf(z, L2E, -lseL)) * fmaf(ce, z, alpha);
            sq = fmaf(d, d, sq);
            zrow[j] = store_cvt<LT>(d);
          }
          d_wrong = ex2_approx(fmaf(za, L2E, -lseL)) * fmaf(ce, za, alpha);
        }
        // the taken action: dz_a = -pg (1 - pi_a) + c_e pi_a (log pi_a + H)
        const float pa = 1.f - rest;
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
    if (lane == 0 && it > it_begin) {
      // the stage of iteration it-1 (== that of it + NSTAGE - 1): its gradient store
      // must have read it (this iteration's store may stay in flight); then refill
      if constexpr (LOSS) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      fence_proxy_async_smem();
      load_iter(it + CT_NSTAGE - 1);
    }
    __syncwarp();
    cur = nxt;
    if (++st == CT_NSTAGE) st = 0;
  }
  if constexpr (LOSS) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (P.partials != nullptr) {
      double part[NPART] = {acc_pg, acc_v, acc_H, 0.0, acc_dz, acc_dv, acc_rho, acc_clip};
      ct_unit_partials(P, C, task, lane, part);
    }
  }
}
