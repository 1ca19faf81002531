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
#include <type_traits>

#include "vtrace_kernels.cuh"
#include "vtrace_rows.cuh"

namespace vtb200 {

constexpr int CT_COLS = 4;
constexpr int CT_STEPS = 8;
constexpr int CT_ROWS = CT_COLS * CT_STEPS;  // 32 == warp size
#ifndef VT_CT_NSTAGE
#define VT_CT_NSTAGE 4  // (A/B: 3 same, 5 and 6 slower -- profiles/r1_perf_analysis.md)
#endif
constexpr int CT_NSTAGE = VT_CT_NSTAGE;      // logits stages: chunks in flight + the one computed
constexpr int CT_WARPS = 1;                  // warps (tasks) per CTA
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
  int tasks, K;
  int f4, segs, seg_len, tpc;  // balanced kernel: whole-task warps per CTA, segments per
                               // cut task, chunks per segment, cut tasks per CTA
  unsigned long long* timing;  // debug: per task [start, own end, group done, exit] (ns)
  TagRec* task_recs;   // [tasks][NPART] (value, epoch tag)
  TagRec* group_recs;  // [groups][NPART]
  unsigned int* group_count;  // [groups] tickets, re-armed by the last arrival
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

// The target row's statistics alone (behaviour given as log mu(a_t): no mu row);
// same arithmetic as ct_stats_fast for pi.  S_m = 1 and xa_m are set by the caller.
template <typename LT, int A_CT>
__device__ __forceinline__ void ct_stats_fast_pi(const LT* zrow, int a, CtStats<LT, A_CT>& R) {
  constexpr int NP = A_CT / 2;
  constexpr bool BF16 = sizeof(LT) == 2;
  constexpr float L16 = 1.44268798828125f;
  constexpr float L32 = 1.44269502f;
  constexpr float CORR = BF16 ? 4.8884952e-06f : 1.3349930e-08f;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    if constexpr (BF16) {
      const uint32_t xp = reinterpret_cast<const uint32_t*>(zrow)[k];
      R.z[k] = make_float2(__uint_as_float(xp << 16), __uint_as_float(xp & 0xffff0000u));
    } else {
      R.z[k] = reinterpret_cast<const float2*>(zrow)[k];
    }
  }
  float mp = fmaxf(R.z[0].x, R.z[0].y);
#pragma unroll
  for (int k = 1; k < NP; ++k) mp = fmaxf(mp, fmaxf(R.z[k].x, R.z[k].y));
  const float2 Lp = f2(BF16 ? L16 : L32);
  const float2 nmLp = f2(BF16 ? -mp * L16 : 0.f);
  const float2 nmp = f2(-mp);
  float2 hp = f2(1.f), lp = f2(0.f), sdp = f2(0.f);
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    float2 yp, dp;
    if constexpr (BF16) {
      yp = __ffma2_rn(R.z[k], Lp, nmLp);
      dp = R.z[k];
    } else {
      dp = __fadd2_rn(R.z[k], nmp);
      yp = __fmul2_rn(dp, Lp);
    }
    const float2 ep = make_float2(ex2_approx(yp.x), ex2_approx(yp.y));
    R.e[k] = ep;
    sdp = __ffma2_rn(ep, dp, sdp);
    const float2 np = __fadd2_rn(hp, ep);  // Fast2Sum: h >= 1 >= e
    lp = __fadd2_rn(lp, __fadd2_rn(__fadd2_rn(hp, make_float2(-np.x, -np.y)), ep));
    hp = np;
  }
  const float h0 = hp.x - 1.f, h1 = hp.y - 1.f;  // exact
  const float s = h0 + h1;                         // TwoSum of the chain heads
  const float bb = s - h0;
  const float err = (h0 - (s - bb)) + (h1 - bb);
  float sd = sdp.x + sdp.y;
  if constexpr (BF16) sd = fmaf(-mp, s, sd);
  const float lo = fmaf(sd, CORR, err + (lp.x + lp.y));
  R.S_p = (double)s + (double)lo;
  R.S_m = 1.0;
  R.m_p = mp;
  R.sd_p = sd;
  const float zap = Elem<LT>::get(zrow, a);
  R.xa_p = (double)zap - (double)mp;
  R.xa_m = 0.0;
  const float ya = BF16 ? fmaf(zap, L16, -mp * L16) : (zap - mp) * L32;
  const float ea = ex2_approx(ya);
  R.ea_p = fmaf(ea * CORR, zap - mp, ea);
  R.finite = isfinite(sd) && isfinite(mp);
}

constexpr int CT_GROUP = 32;  // tasks per partials group

// Waits until the N partial-sum records at p[0 .. N) carry this call's tag (relaxed
// 16-byte loads: value and tag arrive together, so no fence on either side); all N
// loads of a poll are in flight at once.
template <int N, int SLEEP_NS = 1000>
__device__ __forceinline__ int wait_recs(const TagRec* p, unsigned long long tag,
                                         double (&v)[N]) {
  int spins = 0;
  while (true) {
    unsigned long long t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) ld_tag16(p + i, v[i], t[i]);
    bool ok = true;
#pragma unroll
    for (int i = 0; i < N; ++i) ok = ok && (t[i] == tag);
    if (ok) return spins;
    ++spins;
    __nanosleep(SLEEP_NS);
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  return g;
}

// a12: task sums -> group of CT_GROUP tasks -> total, in fixed orders.  Every task
// publishes its 8 sums as epoch-tagged 16-byte (value, tag) records (st.relaxed.v2:
// value and tag arrive together, no fence) and takes a ticket from its group's
// counter (relaxed atomic); the last to arrive reduces the group in task order,
// reading the records by index and checking their tags.  Likewise the last group to
// arrive reduces the groups, writes the result and re-arms the counters.  The sums
// are formed in index order whatever the arrival order: bitwise reproducible.
__device__ __forceinline__ void ct_partials(const Params& P, const CtParams& C, int task,
                                            int lane, unsigned long long tag,
                                            double (&part)[NPART]) {
#pragma unroll
  for (int k = 0; k < NPART; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part[k] += __shfl_xor_sync(0xffffffffu, part[k], o);
  }
  auto pick = [&](const double (&x)[NPART]) {  // x[lane] for lane < NPART
    double v = x[0];
#pragma unroll
    for (int k = 1; k < NPART; ++k) v = (lane == k) ? x[k] : v;
    return v;
  };
  const int grp = task / CT_GROUP;
  const int g0 = grp * CT_GROUP, gn = min(CT_GROUP, C.tasks - g0);
  {
    const double v = pick(part);
    if (lane < NPART) st_tag16(C.task_recs + (size_t)task * NPART + lane, v, tag);
  }
  unsigned int prev = 0;
  if (lane == 0) prev = atomicAdd(C.group_count + grp, 1u);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (C.timing && lane == 0) C.timing[(size_t)task * 4 + 1] = gtimer();
  if (prev != (unsigned int)(gn - 1)) return;
  if (lane == 0) C.group_count[grp] = 0u;  // every ticket of this group is taken: re-arm
  // the group's last arrival: lane l reads task g0 + l (its own from registers)
  double gp[NPART];
#pragma unroll
  for (int k = 0; k < NPART; ++k) gp[k] = (g0 + lane == task) ? part[k] : 0.0;
  if (lane < gn && g0 + lane != task)
    wait_recs<NPART, 32>(C.task_recs + (size_t)(g0 + lane) * NPART, tag, gp);
#pragma unroll
  for (int k = 0; k < NPART; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gp[k] += __shfl_xor_sync(0xffffffffu, gp[k], o);
  }
  {
    const double v = pick(gp);
    if (lane < NPART) st_tag16(C.group_recs + (size_t)grp * NPART + lane, v, tag);
  }
  const int ng = (C.tasks + CT_GROUP - 1) / CT_GROUP;
  if (lane == 0) prev = atomicAdd(C.top_count, 1u);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (C.timing && lane == 0) C.timing[(size_t)task * 4 + 2] = gtimer();
  if (prev != (unsigned int)(ng - 1)) return;
  if (lane == 0) *C.top_count = 0u;
  // the last group: lane l adds groups l, l + 32, ... in order, then a fixed tree
  double tp[NPART];
#pragma unroll
  for (int k = 0; k < NPART; ++k) tp[k] = 0.0;
  for (int gi = lane; gi < ng; gi += 32) {
    double x[NPART];
    if (gi == grp) {
#pragma unroll
      for (int k = 0; k < NPART; ++k) x[k] = gp[k];
    } else {
      wait_recs<NPART, 32>(C.group_recs + (size_t)gi * NPART, tag, x);
    }
#pragma unroll
    for (int k = 0; k < NPART; ++k) tp[k] += x[k];
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
    if (C.timing) C.timing[(size_t)task * 4 + 3] = gtimer();
    // every record of this call has been read: the next call uses the next tag
    *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch) =
        (unsigned int)((tag >> 2) + 1u) & 0x3fffffffu;
  }
}

// Tail / data accumulators of one warp's work.
struct CtAcc {
  float pg, v, H, dz, dv, rho, clip;
};

// GEN: the call uses a Section 5.2.2 variant or the App. E.3 q estimate (false:
// plain V-trace, the variant logic compiled out).  MULP: the behaviour is given as
// log mu(a_t) [T][B] (no mu tile, no mu statistics; implies GEN).
// One warp runs iterations [it_begin, it_end) of task `task` (4 trajectories): its
// TMA ring (`base`, barriers `wb`), the per-step loads, a3-a11 per chunk.  The
// carry A just after the segment comes from `cin` (another warp of the CTA, when
// `cin_bar` completes) or is A_T = 0; the carry at the segment's first step goes
// to `cout` / `cout_bar` for the warp running the earlier segment.
template <typename LT, int A_CT, bool LOSS, int MODE, bool GEN, bool MULP>
__device__ __forceinline__ void ct_run(const Params& P, const CtParams& C, const TmaMaps& maps,
                                       unsigned char* base, uint64_t* wb, const int lane,
                                       const int task, const int it_begin, const int it_end,
                                       const double* cin, uint64_t* cin_bar, double* cout,
                                       uint64_t* cout_bar, CtAcc& acc_out) {
  constexpr bool kFast = (A_CT > 0) && (A_CT % 2 == 0) && (MODE == EXP_MUFU);
  const int A = (A_CT > 0) ? A_CT : P.A;
  const int T = P.T32, B = P.B32;
  const int K = C.K;
  const int b0 = task * CT_COLS;
  const int blen = min(CT_COLS, B - b0);
  const uint32_t tile_bytes = (uint32_t)((size_t)CT_ROWS * A * sizeof(LT));

  // chunk of iteration `it` (reverse time): k = K - 1 - it, t0 = 8 k; stage it mod NSTAGE
  auto load_iter = [&](int it) {  // lane 0 only
#if defined(VTRACE_ABLATE) && VTRACE_ABLATE == 8
    return;  // ablation: no logits loads
#endif
    if (it >= it_end) return;
    const int stg = (it - it_begin) % CT_NSTAGE;
    const int t0 = (K - 1 - it) * CT_STEPS;
    unsigned char* sb = base + (size_t)stg * C.stage;
    mbar_expect_tx(&wb[stg], (MULP ? 1u : 2u) * tile_bytes);
    tma_load_2d(sb + C.pi, &maps.pi, b0 * A, t0, &wb[stg]);
    if constexpr (!MULP) tma_load_2d(sb + C.mu, &maps.mu, b0 * A, t0, &wb[stg]);
  };
  if (lane == 0) {
    for (int s = 0; s < CT_NSTAGE; ++s) mbar_init(&wb[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < CT_NSTAGE; ++i) load_iter(it_begin + i);
  }
  __syncwarp();
  uint32_t phase_bits = 0;  // bit s: parity of stage s's next completion

  const float ce = (float)P.c_e;
  const float cv = (float)P.c_v;
  const int tl = lane >> 2, c = lane & 3;  // row (tl, c) of the [8 steps][4 columns] chunk
  const int stepB = CT_STEPS * B;  // T * B < 2^31 on this path (host check)
  float acc_pg = 0.f, acc_v = 0.f, acc_H = 0.f, acc_dz = 0.f, acc_dv = 0.f, acc_rho = 0.f,
        acc_clip = 0.f;
  double carry = 0.0;  // A = v - V just after the current chunk, for column c (A_T = 0)

  // per-step inputs of one chunk (a, r, gamma, V(x_t), V(x_{t+1})), loaded one chunk
  // ahead; `off` = flat index t * B + b of this lane's row, stepped back 8 B per chunk
  struct StepIn {
    int a;
    float r, g, v, vn, lmu;  // lmu: log mu(a_t) (MULP only)
  };
  const int off0 = ((K - 1 - it_begin) * CT_STEPS + tl) * B + b0 + c;
  const float* const bootp = P.boot + b0 + c;
  auto load_step = [&](int it, int off, StepIn& s) {
    const int t = (K - 1 - it) * CT_STEPS + tl;
    s.a = 0; s.r = 0.f; s.g = 0.f; s.v = 0.f; s.vn = 0.f; s.lmu = 0.f;
#if defined(VTRACE_ABLATE) && (VTRACE_ABLATE == 7 || VTRACE_ABLATE == 8)
    if (false) {  // ablation: no per-step loads
#else
    if (t < T && c < blen) {
#endif
      s.a = __ldg(P.actions + off);
      s.r = __ldg(P.rew + off);
      s.g = __ldg(P.disc + off);
      s.v = __ldg(P.val + off);
      // V(x_{t+1}); the last step of the unroll bootstraps from V(x_T)
      s.vn = __ldg((t + 1 < T) ? P.val + off + B : bootp);
      if constexpr (MULP) s.lmu = __ldg(reinterpret_cast<const float*>(P.mu) + off);
    }
  };

  int st = 0;  // (it - it_begin) mod NSTAGE
  int off = off0;  // this iteration's row
  // one chunk; `cur` holds its per-step inputs, `nxt` receives those of the chunk two
  // ahead (three register sets in rotation: no copy that would wait on loads in flight)
  auto chunk = [&](const int it, const StepIn& cur, StepIn& nxt) {
    // per-step inputs two chunks ahead (three register sets in rotation)
    if (it + 2 < it_end) load_step(it + 2, off - 2 * stepB, nxt);
    const int t0 = (K - 1 - it) * CT_STEPS;
    const int tlen = min(CT_STEPS, T - t0);
    unsigned char* sb = base + (size_t)st * C.stage;
    const bool row_ok = (tl < tlen) && (c < blen);
    LT* zrow = reinterpret_cast<LT*>(sb + C.pi) + lane * A;
    const LT* mrow = reinterpret_cast<const LT*>(sb + C.mu) + lane * A;
    const int a_raw = cur.a;
    const int a = min(max(a_raw, 0), A - 1);
#if !(defined(VTRACE_ABLATE) && VTRACE_ABLATE == 8)
    mbar_wait(&wb[st], (phase_bits >> st) & 1u);
    phase_bits ^= 1u << st;
#endif

    // ---- a3-a7: statistics of this lane's row ----------------------------------
    // Every lane computes its row; rows past the end of the unroll (the first
    // iteration only; TMA zero-filled) are masked out of the scan and the outputs.
    float m_p, sed_p, ea_p;
    double S_p, S_m, xa_p, xa_m;
    bool fin;
    [[maybe_unused]] CtStats<LT, (kFast ? A_CT : 2)> F;
    [[maybe_unused]] RowRegs<LT, A_CT> zp;
#if defined(VTRACE_ABLATE) && (VTRACE_ABLATE == 1 || VTRACE_ABLATE == 5 || VTRACE_ABLATE == 6 || VTRACE_ABLATE == 7)
    if constexpr (kFast) {  // ablation: no row statistics (loads only)
      const uint32_t* zw = reinterpret_cast<const uint32_t*>(zrow);
      const uint32_t* mw = reinterpret_cast<const uint32_t*>(mrow);
      uint32_t acc = 0;
#pragma unroll
      for (int k = 0; k < A_CT / 2; ++k) {
        acc ^= zw[k] ^ mw[k];
        F.z[k] = make_float2(__uint_as_float(zw[k] << 16), 0.f);
        F.e[k] = make_float2(1.f, 1.f);
      }
      F.m_p = __uint_as_float(acc & 0x3f000000u); F.sd_p = 0.f; F.ea_p = 1.f; F.S_p = 18.0;
      F.S_m = 18.0; F.xa_p = 0.0; F.xa_m = 0.0; F.finite = true;
#else
    if constexpr (kFast) {
      if constexpr (MULP) {
        ct_stats_fast_pi<LT, A_CT>(zrow, a, F);
        F.xa_m = (double)cur.lmu;  // log mu(a_t), given (S_m = 1)
        F.finite = F.finite && isfinite(cur.lmu);
      } else {
        ct_stats_fast<LT, A_CT>(zrow, mrow, a, F);
      }
#endif
      m_p = F.m_p; sed_p = F.sd_p; ea_p = F.ea_p; S_p = F.S_p; S_m = F.S_m;
      xa_p = F.xa_p; xa_m = F.xa_m;
      fin = F.finite;
    } else if constexpr (MULP) {
      bool fin_p;
      zp.load(zrow);
      row_stats<LT, A_CT, MODE>(zp, A, a, m_p, S_p, xa_p, ea_p, sed_p, fin_p);
      xa_m = (double)cur.lmu;  // log mu(a_t), given
      S_m = 1.0;
      fin = fin_p && isfinite(cur.lmu);
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
#if defined(VTRACE_ABLATE) && (VTRACE_ABLATE == 2 || VTRACE_ABLATE == 5 || VTRACE_ABLATE == 6 || VTRACE_ABLATE == 7)
    const double ratio = 1.0 + (xa_p - xa_m) + (S_m - S_p);  // ablation: no exp64 / division
#else
    const double ratio = exp64(xa_p - xa_m) * ddiv_pos(S_m, S_p);
#endif
    const float rt = cur.r, gm = cur.g, Vt = cur.v, Vn = cur.vn;
    const double td = reward_transform(rt, P.reward_mode) + (double)gm * (double)Vn - (double)Vt;
    const StepWeights sw = step_weights<GEN>(P, ratio);  // rho, c, rho_pg (Section 5.2.2)
    double dl = sw.rho * td;                        // delta_t V
    double gc = (double)gm * sw.c;                  // gamma_t c_t
    const float Sf = (float)S_p;
    const float inv_S = rcp_approx(Sf);
    const float lse = m_p + __logf(Sf);
    const float cshift = fmaf(sed_p, inv_S, m_p);  // lse - H
    const float rest = (float)(S_p - (double)ea_p) * inv_S;  // 1 - pi(a)
    if (row_ok) {
      acc_rho += (float)sw.rho;  // the rho_t in delta_t (reading r6)
      acc_clip += ((!GEN || P.correction == VT_CORRECTION_VTRACE) && ratio > P.rho_bar) ? 1.f : 0.f;
    }
    const bool bad = row_ok && ((a_raw != a) || !fin || !isfinite(rt) || !isfinite(Vt) ||
                                !isfinite(Vn) || !(gm >= 0.f && gm <= 1.f));
    if (!row_ok) {
      dl = 0.0;  // identity map for steps past the end of the unroll
      gc = 1.0;
    }

    // ---- a8: suffix scan of the chunk's affine maps, per column ----------------
    // lanes c, c+4, ..., c+28 are steps 0..7 of column c; composing later steps:
    // (G1, D1) o (G2, D2) = (G1 G2, D1 + G1 D2)
    if (cin != nullptr && it == it_begin) {
      // A just after this segment = A at the first step of the later segment
      mbar_wait_sleep(cin_bar, 0u, 500);
      carry = cin[c];
    }
    double Gi = gc, Di = dl;
#if defined(VTRACE_ABLATE) && (VTRACE_ABLATE == 3 || VTRACE_ABLATE == 5 || VTRACE_ABLATE == 6 || VTRACE_ABLATE == 7)
    if (false)  // ablation: no scan
#else
#pragma unroll
#endif
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

    // (programmatic dependent launch: everything above only read this call's inputs;
    // the task's first global write waits for the previous kernel on the stream)
    if (P.pdl && it == it_begin) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!LOSS && row_ok) {
      const int row = off;
      if (P.has_lr) P.log_rhos[row] = (float)log(ratio);
      if (P.has_lp) P.lp_out[row] = (float)(xa_p - log(S_p));
      if (P.has_lm) P.lm_out[row] = (float)(xa_m - log(S_m));
    }
#if defined(VTRACE_ABLATE) && VTRACE_ABLATE == 8
    if (false) {  // (garbage inputs)
#else
    if (bad) {
#endif
      const int row = off;
      if (a_raw != a) record_bad(P.ws, row, VT_DATA_ACTION);
      if (!fin) record_bad(P.ws, row, VT_DATA_LOGITS);
      if (!isfinite(rt)) record_bad(P.ws, row, VT_DATA_REWARD);
      if (!isfinite(Vt)) record_bad(P.ws, row, VT_DATA_VALUE);
      if (!(gm >= 0.f && gm <= 1.f)) record_bad(P.ws, row, VT_DATA_DISCOUNT);
      if (!isfinite(Vn) && t0 + tl + 1 == T)
        record_bad(P.ws, (long long)T * B + b0 + c, VT_DATA_VALUE);  // the bootstrap
    }

    // ---- a9-a11: advantages, value gradient, policy gradient ------------------
    if (row_ok) {
      const int row = off;
      // pg_adv = rho_pg (r + gamma v_{t+1} - V) = rho_pg (td + gamma A_{t+1})
      // (q_s = r_s + gamma V(x_{s+1}) instead with q_values: App. E.3)
      const float pgr =
          (float)(sw.rho_pg * ((GEN && P.q_values) ? td : fma((double)gm, A_n, td)));
#if !(defined(VTRACE_ABLATE) && (VTRACE_ABLATE == 7 || VTRACE_ABLATE == 8))
      if (P.vs) P.vs[row] = (float)((double)Vt + A_t);
      if (P.pg_adv) P.pg_adv[row] = pgr;
#endif
      if constexpr (LOSS) {
        const float Ar = (float)A_t;
        const float za = Elem<LT>::get(zrow, a);
        // epsilon-correction (readings c11, r7): the policy-gradient term uses
        // log(pi_a + eps); its logit gradient is the plain one times pi_a / (pi_a + eps)
        float pge = pgr, logpa = za - lse;
        if (GEN && P.correction == VT_CORRECTION_EPSILON) {
          const float pa_e = ea_p * inv_S;  // pi(a), relative accuracy
          const float rr = P.eps / pa_e;
          logpa = pa_e > 0.f ? (za - lse) + log1pf(rr) : logf(P.eps);
          pge = pgr / (1.f + rr);
        }
        const float alpha = fmaf(-ce, cshift, pge);  // pg + c_e (z_j - cshift) = alpha + c_e z_j
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
#if defined(VTRACE_ABLATE) && (VTRACE_ABLATE == 4 || VTRACE_ABLATE == 5 || VTRACE_ABLATE == 6 || VTRACE_ABLATE == 7)
          if (false)  // ablation: no gradient loop
#else
#pragma unroll
#endif
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
        const float d_a = fmaf(-pge, rest, ce * pa * (za - cshift));
        zrow[a] = store_cvt<LT>(d_a);
        sq = __fadd_rn(__fsub_rn(sq, __fmul_rn(d_wrong, d_wrong)), __fmul_rn(d_a, d_a));
        const float dv = -cv * Ar;  // c_v (V - v)
#if !(defined(VTRACE_ABLATE) && (VTRACE_ABLATE == 7 || VTRACE_ABLATE == 8))
        P.dvalues[row] = dv;
#endif
        acc_pg = fmaf(-pgr, logpa, acc_pg);  // -pg_adv log pi(a)  (log(pi(a) + eps))
        acc_v = fmaf(0.5f * Ar, Ar, acc_v);
        acc_H += lse - cshift;
        acc_dz += sq;
        acc_dv = fmaf(dv, dv, acc_dv);
      }
    }
#if defined(VTRACE_ABLATE) && (VTRACE_ABLATE == 6 || VTRACE_ABLATE == 8)
    if (false) {  // ablation: no gradient store
#else
    if constexpr (LOSS) {
#endif
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
    off -= stepB;
    if (++st == CT_NSTAGE) st = 0;
  };
  StepIn sA, sB, sC;
  load_step(it_begin, off0, sA);
  if (it_begin + 1 < it_end) load_step(it_begin + 1, off0 - stepB, sB);
  for (int it = it_begin; it < it_end; it += 3) {
    chunk(it, sA, sC);
    if (it + 1 < it_end) chunk(it + 1, sB, sA);
    if (it + 2 < it_end) chunk(it + 2, sC, sB);
  }
  if (cout != nullptr) {  // hand the carry at this segment's first step on
    if (tl == 0) cout[c] = carry;
    __syncwarp();
    if (lane == 0) mbar_arrive(cout_bar);
  }
  if constexpr (LOSS) {
    // the gradient stores must have read the stages before the CTA's smem goes away
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  acc_out = CtAcc{acc_pg, acc_v, acc_H, acc_dz, acc_dv, acc_rho, acc_clip};
}

template <typename LT, int A_CT, bool LOSS, int MODE, bool GEN, bool MULP>
__global__ void __launch_bounds__(CT_WARPS * 32)
    vtrace_ct_kernel(const Params P, const CtParams C, const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[CT_NSTAGE];
  // a programmatically dependent next kernel may launch (it waits before writing)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int task = blockIdx.x;
  if (task >= C.tasks) return;
  if (C.timing && lane == 0) C.timing[(size_t)task * 4 + 0] = gtimer();
  CtAcc acc;
  ct_run<LT, A_CT, LOSS, MODE, GEN, MULP>(P, C, maps, smem, bar, lane, task, 0, C.K, nullptr, nullptr,
                               nullptr, nullptr, acc);
  if constexpr (LOSS) {
    if (P.partials != nullptr) {
      const unsigned int epoch =
          *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch) & 0x3fffffffu;
      const unsigned long long tag = ((unsigned long long)epoch << 2) | 3ull;
      double part[NPART] = {acc.pg, acc.v, acc.H, 0.0, acc.dz, acc.dv, acc.rho, acc.clip};
      ct_partials(P, C, task, lane, tag, part);
    }
  }
}

// ---------------------------------------------------------------------------
// Balanced column-task kernel: one CTA of CTB_WARPS = 16 warps per SM, so warp w
// runs on SM sub-partition w mod 4.  The first f4 = 4 f warps take whole tasks
// (f per sub-partition); the remaining tasks are cut into P time segments run by
// P consecutive warps (on different sub-partitions), the carry passed down the
// chain through shared memory and an mbarrier.  With B = 8192 on 148 SMs: 12 whole
// tasks + 4 half tasks per SM, i.e. 3.5 tasks of work per sub-partition instead of
// the 4/4/3/3 split of one-warp CTAs.  Partials: warp sums -> CTA sum (warp order)
// -> the last CTA to finish adds the CTA sums in CTA order.
constexpr int CTB_WARPS = 16;

template <typename LT, int A_CT, bool LOSS, int MODE, bool GEN, bool MULP>
__global__ void __launch_bounds__(CTB_WARPS * 32, 1)
    vtrace_ctb_kernel(const Params P, const CtParams C, const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[CTB_WARPS][CT_NSTAGE];
  __shared__ __align__(8) uint64_t hbar[CTB_WARPS];
  __shared__ double hcarry[CTB_WARPS][CT_COLS];
  __shared__ double wpart[CTB_WARPS][NPART];
  // a programmatically dependent next kernel may launch (it waits before writing)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cta = blockIdx.x, S = gridDim.x;
  if (lane == 0) {
    mbar_init(&hbar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // this warp's share: a whole task, or segment p of a task cut in C.segs.  Slots
  // are laid over the warps diagonally (slot j -> warp 4 ((j + j/4) mod 4) + j mod 4),
  // so any 4 consecutive slots fall on 4 different sub-partitions whether the
  // hardware maps warp w to sub-partition w mod 4 or w / 4; the segment slots come
  // first (j < 16 - f4), the whole tasks take the rest.
  int task = -1, it_begin = 0, it_end = C.K, p = 0;
  const int jslot = ((w >> 2) - (w & 3) + 4) & 3;  // block of the inverse diagonal map
  const int slot = 4 * jslot + (w & 3);
  const int nseg = CTB_WARPS - C.f4;  // segment slots
  if (slot >= nseg) {
    task = cta * C.f4 + (slot - nseg);
  } else {
    const int j = slot, i = j / C.segs;
    p = j - i * C.segs;
    if (i < C.tpc) {
      const int t = C.f4 * S + cta * C.tpc + i;
      if (t < C.tasks) {
        task = t;
        it_begin = p * C.seg_len;
        it_end = min(C.K, it_begin + C.seg_len);
      }
    }
  }
  CtAcc acc = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (task >= 0) {
    const bool whole = slot >= nseg;
    const bool first = whole || p == 0, last = whole || p == C.segs - 1;
    // segment hand-over slots: slot j feeds slot j + 1 (same task)
    ct_run<LT, A_CT, LOSS, MODE, GEN, MULP>(P, C, maps, smem + (size_t)w * C.warp_bytes, bar[w], lane,
                                 task, it_begin, it_end, first ? nullptr : hcarry[slot - 1],
                                 &hbar[first ? slot : slot - 1], last ? nullptr : hcarry[slot],
                                 &hbar[slot], acc);
  }
  if constexpr (LOSS) {
    if (P.partials == nullptr) return;
    if (P.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");  // (idle warps too)
    double part[NPART] = {acc.pg, acc.v, acc.H, 0.0, acc.dz, acc.dv, acc.rho, acc.clip};
#pragma unroll
    for (int k = 0; k < NPART; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part[k] += __shfl_xor_sync(0xffffffffu, part[k], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < NPART; ++k) wpart[w][k] = part[k];
    }
    __syncthreads();
    if (w != 0) return;
    double cs[NPART];  // this CTA's sums, warps in order
#pragma unroll
    for (int k = 0; k < NPART; ++k) {
      double x = 0.0;
      for (int v = 0; v < CTB_WARPS; ++v) x += wpart[v][k];
      cs[k] = x;
    }
    const unsigned int epoch =
        *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch) & 0x3fffffffu;
    const unsigned long long tag = ((unsigned long long)epoch << 2) | 3ull;
    {
      double v = cs[0];
#pragma unroll
      for (int k = 1; k < NPART; ++k) v = (lane == k) ? cs[k] : v;
      if (lane < NPART) st_tag16(C.task_recs + (size_t)cta * NPART + lane, v, tag);
    }
    unsigned int prev = 0;
    if (lane == 0) prev = atomicAdd(C.top_count, 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != (unsigned int)(S - 1)) return;
    if (lane == 0) *C.top_count = 0u;
    // the last CTA: lane l adds CTAs l, l + 32, ... in order, then a fixed tree
    double tp[NPART];
#pragma unroll
    for (int k = 0; k < NPART; ++k) tp[k] = 0.0;
    for (int ci = lane; ci < S; ci += 32) {
      double x[NPART];
      if (ci == cta) {
#pragma unroll
        for (int k = 0; k < NPART; ++k) x[k] = cs[k];
      } else {
        wait_recs<NPART, 32>(C.task_recs + (size_t)ci * NPART, tag, x);
      }
#pragma unroll
      for (int k = 0; k < NPART; ++k) tp[k] += x[k];
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
      *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch) = (epoch + 1u) & 0x3fffffffu;
    }
  }
}

}  // namespace vtb200
