// vtrace_kernels.cuh -- shared types and device helpers of the fused V-trace +
// actor-critic loss + gradient kernels for sm_100a (the look-back kernel in
// vtrace_api.cu, the column-block kernel in vtrace_cb.cuh).
//
// Look-back kernel: a work unit = (column group of BC=8 trajectories) x (time chunk
// of Tc <= 20 steps); unit ids run in REVERSE time order.  A co-resident persistent
// grid walks the units round-robin; the reverse V-trace recursion (Remark 1)
// crosses chunk boundaries through a decoupled look-back on per-unit affine
// aggregates (G, D):  A_start = D + G * A_end  with A = v - V.
//
// Phases inside a unit:
//   a1  stage: TMA 2D tile loads of z^pi, z^mu [Tc][BC*A] and a, r, gamma, V [Tc][BC]
//       into shared memory (one mbarrier), or plain loads for unaligned shapes
//   a3-a6  per row (thread per row): max, accurate sum of exp for both policies,
//       importance ratio pi/mu at a_t in fp64, lse of pi (fp32) for the epilogue
//   a2,a7-a9  per column (warp per column, lanes over time): reward transform,
//       delta_t, segment affine aggregates, warp suffix scan, look-back carry,
//       v_t, q_t, pg_adv_t -- all fp64
//   a10-a11  per row: pi_j, log pi_j, entropy, dL/dz^pi written in place over
//       the z^pi tile, then one TMA 2D store; dL/dV from the scan warps
//   a12  per-unit fp64 partials; the last CTA reduces them in a fixed order
//
// Precision: every quantity that feeds the recursion (sum_j exp, the ratio,
// delta, the scan) is carried well beyond fp32 (fp64 or compensated fp32);
// the gradient epilogue is fp32 (its outputs are fp32/bf16).  See DESIGN.md.
// The column-block kernel (vtrace_cb.cuh) follows the same steps with one warp per
// 4 trajectories x 8 steps of a CTA-wide TMA tile.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace vtb200 {

constexpr int BC = 8;          // trajectories (columns) per unit
constexpr int NWARPS = 6;      // 5 row warps + 1 scan warp
constexpr int NTHREADS = NWARPS * 32;
constexpr int NPART = 8;

enum ExpMode { EXP_F64 = 0, EXP_MUFU = 1 };

struct alignas(16) WsHeader {
  unsigned int pad_t;
  unsigned int exited;   // CTAs that have left the unit loop
  unsigned int epoch;    // call counter (tags the look-back flags)
  unsigned int pad0;
  unsigned long long status;  // (row << 8) | kind, atomicMin; ~0ull = clean
  unsigned long long pad1[5];
};

// Decoupled look-back record: a 16-byte (value, tag) pair written and read
// with single 16-byte relaxed accesses, so no fence or flag is needed; tag =
// (epoch << 2) | kind.  Per (unit, column) there are three: the chunk's affine
// aggregate G and D (kind 1) and the inclusive carry A = v - V at the chunk's
// first step (kind 2).
struct alignas(16) TagRec {
  double value;
  unsigned long long tag;
};
static_assert(sizeof(TagRec) == 16, "TagRec layout");
constexpr int RECS_PER_COL = 3;  // G, D, incl

// Shared-memory offsets of one CTA (computed on the host, read from the
// kernel's parameter space so they never occupy registers).
struct KLayout {
  unsigned int pi, mu, a, r, g, v, boot, stage;
  unsigned int ratio[2], td[2], adv[2], lse[2], csh[2], rest[2];
};

struct Params {
  long long T, B;
  int T32, B32;
  int A, Tc, K, G, units;
  int has_lr, has_lp, has_lm;
  const void* mu;
  const void* pi;
  const int* actions;
  const float* disc;
  const float* rew;
  const float* val;
  const float* boot;
  float* vs;
  float* pg_adv;
  float* log_rhos;
  float* lp_out;
  float* lm_out;
  void* dlogits;
  float* dvalues;
  double* partials;
  double rho_bar, c_bar, pg_rho_bar, lambda;
  double c_v, c_e;
  int reward_mode;
  int correction;  // vt_correction (Section 5.2.2)
  int q_values;    // 1: q_s = r_s + gamma V(x_{s+1}) (App. E.3)
  int mu_lp;       // 1: `mu` is log mu(a_t) [T][B] fp32 instead of [T][B][A] logits
  int pdl;         // 1: launched as a programmatic dependent (overlap_previous)
  float eps;       // epsilon-correction constant
  WsHeader* ws;
  TagRec* recs;          // [units][BC][RECS_PER_COL]
  double* cta_partials;
  unsigned long long* timing;  // debug: per-CTA phase timestamps (NULL = off)
  int timing_iters;
  int stride_q, stride_r;  // gridDim.x = stride_q * G + stride_r
  KLayout L;
  // learners (vtrace_loss_and_grad_learners): the column-block kernel's last CTA adds the
  // learners' partials through peer-mapped mailboxes ({value, tag} [2][nlearn][8])
  int nlearn;              // <= 1: no exchange
  int self;
  void* mbox[16];
};

struct TmaMaps {
  CUtensorMap mu, pi, a, r, g, v, boot, dz;
};

// ---------------------------------------------------------------------------
// small PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// mbar_wait for long waits: test without blocking, sleep between tests (a waiting
// warp should not take issue slots from the warps sharing its sub-partition)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase, int ns) {
  const uint32_t addr = smem_u32(bar);
#ifdef VTRACE_WAIT_HINT
  // A/B only: try_wait with a suspend-time hint parks the warp until the phase
  // completes -- no polling (the __nanosleep loop below polls every ~20 ns), but
  // measured slower at `large` (34.2 vs 33.6 us: a late wake-up of the segment warp)
  (void)ns;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITH_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITH_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase), "r"(1000000u)
      : "memory");
#else
  while (true) {
    uint32_t done;
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(addr), "r"(phase)
        : "memory");
    if (done) return;
    __nanosleep(ns);
  }
#endif
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {  // release.cta semantics
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const CUtensorMap* map, int x,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2}], [%3];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y,
                                             const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}

__device__ __forceinline__ void tma_store_commit_and_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_tag16(TagRec* p, double v, unsigned long long tag) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p),
               "l"((unsigned long long)__double_as_longlong(v)), "l"(tag)
               : "memory");
}

__device__ __forceinline__ void ld_tag16(const TagRec* p, double& v, unsigned long long& tag) {
  unsigned long long a, b;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  v = __longlong_as_double((long long)a);
  tag = b;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }

__device__ __forceinline__ double shfl_down_d(double v, int off) {
  return __shfl_down_sync(0xffffffffu, v, off);
}

// ---------------------------------------------------------------------------
// logits element access

template <typename LT>
struct Elem;
template <>
struct Elem<float> {
  static constexpr int bytes = 4;
  static __device__ __forceinline__ float get(const float* p, int i) { return p[i]; }
};
template <>
struct Elem<__nv_bfloat16> {
  static constexpr int bytes = 2;
  static __device__ __forceinline__ float get(const __nv_bfloat16* p, int i) {
    return __uint_as_float((uint32_t)reinterpret_cast<const unsigned short*>(p)[i] << 16);
  }
};

// min(bound, x) for a threshold that is never NaN (compare + select, no NaN fixups)
__device__ __forceinline__ double dmin_t(double bound, double x) { return x < bound ? x : bound; }

// Loads a row of A_CT logits from shared memory into registers (exact upcast).
template <typename LT, int A_CT>
__device__ __forceinline__ void load_row(const LT* row, float (&z)[A_CT]) {
  if constexpr (sizeof(LT) == 2 && (A_CT % 2) == 0) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(row);
#pragma unroll
    for (int k = 0; k < A_CT / 2; ++k) {
      uint32_t x = w[k];
      z[2 * k] = __uint_as_float(x << 16);
      z[2 * k + 1] = __uint_as_float(x & 0xffff0000u);
    }
  } else if constexpr (sizeof(LT) == 4 && (A_CT % 2) == 0) {
    // rows of even length start 8-byte aligned
    const float2* w = reinterpret_cast<const float2*>(row);
#pragma unroll
    for (int k = 0; k < A_CT / 2; ++k) {
      float2 x = w[k];
      z[2 * k] = x.x;
      z[2 * k + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < A_CT; ++j) z[j] = Elem<LT>::get(row, j);
  }
}

// a / b in fp64 for b in [1, 2^30] (a row sum): MUFU reciprocal seed, two Newton steps
// and one residual correction (within an ulp; no slow-path branch as in div.rn.f64).
// The short-chain form (one Newton step) pays where a kernel is bound by its warps'
// dependent chains: the bf16 column-block kernel (14 warps), the look-back and fused-head
// kernels.  The fp32 column-block unit (18 warps, VT_CB_PART == 1) is issue-bound and keeps
// two steps (stress 76.7 vs 76.1 us) -- profiles/r2_ratio_chain_ab.txt.
#if defined(VT_CB_PART) && VT_CB_PART == 1
#define VT_SHORT_CHAIN_DEFAULT 0
#else
#define VT_SHORT_CHAIN_DEFAULT 1
#endif
#ifndef VT_DDIV_NEWTON
#define VT_DDIV_NEWTON (VT_SHORT_CHAIN_DEFAULT ? 1 : 2)  // Newton steps on the reciprocal seed
#endif
__device__ __forceinline__ double ddiv_pos(double a, double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  // one step squares the seed's error (~2^-44 after it); the residual correction of the
  // quotient below squares it again, so the result is within an ulp either way (and
  // a / a == 1 exactly: the on-policy ratio), with two fewer dependent DFMAs on the chain
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
#if VT_DDIV_NEWTON > 1
  e = fma(-b, r, 1.0);
  r = fma(r, e, r);
#endif
  const double q = a * r;
  return fma(fma(-b, q, a), r, q);
}

// Weights of step t from its importance ratio under the call's correction
// (Section 5.2.2; readings r5): rho for delta_t V, c for the trace,
// rho_pg for the policy-gradient advantage.
struct StepWeights {
  double rho, c, rho_pg;
};
// GEN = false: the call is plain V-trace (a compile-time fast path, no variant logic).
template <bool GEN = true>
__device__ __forceinline__ StepWeights step_weights(const Params& P, double ratio) {
  StepWeights w;
  if (!GEN || P.correction == VT_CORRECTION_VTRACE) {
    w.rho = dmin_t(P.rho_bar, ratio);
    w.c = P.lambda * dmin_t(P.c_bar, ratio);
    w.rho_pg = dmin_t(P.pg_rho_bar, ratio);
  } else {
    w.rho = 1.0;
    w.c = P.lambda;
    w.rho_pg = (P.correction == VT_CORRECTION_ONE_STEP_IS) ? dmin_t(P.pg_rho_bar, ratio) : 1.0;
  }
  return w;
}

// fp64 exp, argument clamped to [-700, 700].  Cody-Waite reduction
// x = n ln2 + r, |r| <= ln2/2, then a degree-6 polynomial fitted to exp on
// that interval as 1 + r q(r) (max relative error 2.2e-9; the path needs ~1e-8,
// DESIGN.md; exp(0) = 1 exactly).
#ifndef VT_EXP64_ESTRIN
#define VT_EXP64_ESTRIN 0  // A/B: 1 = Estrin (faster before exp64 moved between the policies' exps,
                           // slower after: 25.77 vs 25.58 us at large, r2_ratio_chain_ab.txt)
#endif
#ifndef VT_EXP64_CW1
#define VT_EXP64_CW1 0  // A/B: 1 = one-step reduction (no gain measured)
#endif
__device__ __forceinline__ double exp64(double x) {
  const double LOG2E = 1.4426950408889634;
  const double LN2_HI = 6.93147180369123816490e-01;
  const double LN2_LO = 1.90821492927058770002e-10;
  const double MAGIC = 6755399441055744.0;  // 1.5 * 2^52: round-to-integer shifter
  x = (x < -700.0) ? -700.0 : ((x > 700.0) ? 700.0 : x);  // (NaN passes through)
  double t = fma(x, LOG2E, MAGIC);
  double n = t - MAGIC;
  int ni = __double2loint(t);
#if VT_EXP64_CW1
  // one-step reduction: |n (ln2 - fl(ln2))| <= 1010 * 2.3e-17, a relative error of 2.3e-14 in
  // the result, far inside the polynomial's 2.2e-9 -- one dependent DFMA fewer
  double r = fma(-n, 6.93147180559945286e-01, x);
  (void)LN2_HI;
  (void)LN2_LO;
#else
  double r = fma(-n, LN2_HI, x);
  r = fma(-n, LN2_LO, r);
#endif
  // p(r) = 1 + r q(r): exact at r = 0, so exp(0) == 1 bitwise (on-policy ratio).
  // q by Estrin's scheme (three independent pairs, then two steps in r^2): 3 dependent
  // DFMAs instead of Horner's 5 on the ratio's chain (the kernels are latency-bound there)
#if VT_EXP64_ESTRIN
  const double r2 = r * r;
  const double q01 = fma(4.99999953509942752e-01, r, 1.00000003609212618e+00);
  const double q23 = fma(4.16677243209218270e-02, r, 1.66664209451321627e-01);
  const double q45 = fma(1.38592910771707131e-03, r, 8.37476397493414765e-03);
  const double q = fma(fma(q45, r2, q23), r2, q01);
#else
  double q = 1.38592910771707131e-03;
  q = fma(q, r, 8.37476397493414765e-03);
  q = fma(q, r, 4.16677243209218270e-02);
  q = fma(q, r, 1.66664209451321627e-01);
  q = fma(q, r, 4.99999953509942752e-01);
  q = fma(q, r, 1.00000003609212618e+00);
#endif
  const double p = fma(q, r, 1.0);
  // scale by 2^n: add n to the exponent field (p in [0.7, 1.5], |n| <= 1010)
  int hi = __double2hiint(p) + (ni << 20);
  return __hiloint2double(hi, __double2loint(p));
}

// Compensated fp32 exp for MUFU mode: e = 2^{(z - m) log2 e} via ex2.approx,
// with the fp32 rounding of the argument (and, for fp32 logits, of z - m)
// corrected to first order.  Returns e (fp32).
template <bool EXACT_DIFF>
__device__ __forceinline__ float exp_mufu(float z, float m) {
  const float L = 1.44269502f;       // fp32(log2 e)
  const float L_LO = 1.925963e-08f;  // log2 e - L
  const float LN2 = 0.693147182f;
  float d = z - m;
  float y = d * L;
  float y_lo = fmaf(d, L, -y);
  y_lo = fmaf(d, L_LO, y_lo);
  if constexpr (!EXACT_DIFF) {
    float bb = d - z;  // TwoSum error of the fp32 difference
    float d_lo = (z - (d - bb)) + (-m - bb);
    y_lo = fmaf(d_lo, L, y_lo);
  }
  float e = ex2_approx(y);
  return fmaf(e, y_lo * LN2, e);
}

}  // namespace vtb200
