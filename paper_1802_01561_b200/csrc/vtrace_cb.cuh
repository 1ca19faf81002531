// vtrace_cb.cuh -- "column-block" fused kernel (round 2): one CTA per SM owns a
// block of Bc = 4 ncg trajectories over the whole unroll.
//
// Warp roles (one CTA = NW = ncg * nts compute warps + 1 producer warp):
//   producer (warp NW, one lane): a CTA-wide NSTAGE ring of TMA tiles.  Iteration j
//     covers Ts = 8 nts steps x Bc columns: both logits tiles as ONE 3-D box each
//     ({4 g A, Ts, ncg / g} over the [T][B/(4g)][4 g A] view -- so a warp's 32 rows
//     are contiguous in shared memory, bank-conflict free), a, r, gamma [Ts][Bc] and
//     V [Ts+1][Bc] as 2-D boxes.  When every compute warp has released iteration j
//     (mbarrier `done`, NW arrivals) it TMA-stores j's outputs from the same stage
//     (dL/dz written in place over the z^pi tile, dL/dV / vs / pg_adv tiles), waits
//     until the stores have read the stage, and refills it with iteration j + NSTAGE.
//   compute warp (cg, ts): trajectories 4 cg .. 4 cg + 3 of the block, steps
//     8 ts .. 8 ts + 7 of every iteration; lane = (tl, c) = one row (t, b):
//       a3-a6  both policies' log-sum-exp statistics (packed fp32 + MUFU ex2,
//              compensated sums; DESIGN.md precision), the gathered log-probs
//       a5,a7  ratio pi/mu (fp64), rho, c, delta_t V = rho_t (r_t + gamma_t V_{t+1} - V_t)
//       a8     suffix scan of the affine maps (gamma_t c_t, delta_t V) over the
//              warp's 8 steps (3 shuffle levels, fp64), then the carry: with nts = 1
//              it stays in registers from iteration to iteration (the reverse
//              recursion of Remark 1, walks the block's columns backwards
//              in time); with nts > 1 the nts warps of a column group swap their
//              8-step aggregates through shared memory (one named barrier per
//              iteration) and each folds the later ones into its carry
//       a9-a11 q, pg_adv, dL/dV, dL/dz (written in place over z^pi)
//       a10/12 per-lane fp64 sums -> warp -> CTA (warp order) -> epoch-tagged
//              records -> the last CTA adds the CTA sums in CTA order
// No look-back between CTAs, no per-step global loads, no CTA-wide barrier in the
// loop (nts = 1).  Shapes: SURVEY 8(d) `large` (B = 8192: 147 CTAs of 56 columns,
// 14 + 1 warps) and its strong-scaling shards (B = 4096: 28 columns, nts = 2; ...).
#pragma once

#include <cassert>

#include "vtrace_kernels.cuh"
#include "vtrace_rows.cuh"

// -DVT_DEBUG_CHECKS: device-side bounds checks of every shared-memory tile index, stage
// and record index (a build for small test runs; compute-sanitizer is closed on the pool)
#ifdef VT_DEBUG_CHECKS
#define VT_CHECK(c) assert(c)
#else
#define VT_CHECK(c) ((void)0)
#endif

// compile-time variants (A/B builds, VTRACE_DEFINES)
#ifndef CB_F32_EXACT
// 1: fp32 logits, first-order correction for the roundings of z - m and (z - m) L32 (TwoSum
// + FMA residual per element).  Off: the parity tests (hard distribution included) pass
// without it, and it costs 13% at `stress` (92.6 vs 80.8 us, profiles/r2_cb_f32_exact_ab.txt)
#define CB_F32_EXACT 0
#endif
#ifndef CB_PIPE
#define CB_PIPE 0  // 1: X(j+1) next to Y(j) (software pipeline); 0: X(j) then Y(j)
#endif
#ifndef CB_EBUF
#define CB_EBUF 0  // 1: the target exps wait in shared memory between X and Y
#endif

namespace vtb200 {

#ifndef CB_PLAIN_SUMS
#define CB_PLAIN_SUMS 0   // A/B only: plain (uncompensated) exponent sums
#endif
#ifndef CB_TD32
#define CB_TD32 0         // A/B only: r + gamma V' - V in fp32
#endif

#ifdef CB_TIMING
// timing build only: per-CTA globaltimer stamps [start, first stage landed (warp 0),
// last stage released (warp 0), partials published, exit of the last CTA's reduction]
__device__ unsigned long long cb_stamps[4096][8];
__device__ __forceinline__ unsigned long long cb_now() {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  return g;
}
#define CB_STAMP(k) (cb_stamps[blockIdx.x][k] = cb_now())
#else
#define CB_STAMP(k) ((void)0)
#endif

// Compute warps per CTA (+1 producer), per logits dtype; the register cap is
// 64K / (32 (warps + 1)): 14 -> 128 registers (bf16: `large` keeps every value in registers),
// 18 -> 107 (fp32: a few spilled bytes, but `stress` gets 9 time slots per column group
// instead of 7 -- 28 iterations instead of 36: 80.5 -> 76.1 us, profiles/r2_cb_maxw_ab.txt)
#ifndef CB_MAXW_BF16
#define CB_MAXW_BF16 14
#endif
#ifndef CB_MAXW_F32
#define CB_MAXW_F32 18
#endif
#if defined(VT_CB_PART) && VT_CB_PART == 1
constexpr int CB_MAX_WARPS = CB_MAXW_F32;
#else
constexpr int CB_MAX_WARPS = CB_MAXW_BF16;
#endif
constexpr int cb_max_warps(int elem) { return elem == 4 ? CB_MAXW_F32 : CB_MAXW_BF16; }
static_assert(CB_MAXW_BF16 <= 20 && CB_MAXW_F32 <= 20, "at most 20 compute warps (>= 97 registers)");
constexpr int CB_MAX_STAGES = 4;

struct CbParams {
  int ncg, nts, Ts, J, nstage, g, Bc;
  unsigned pi, mu, a, r, gm, v, dv, vs, pg, lr, lp, lm, stage;  // stage layout (bytes)
  unsigned tx_bytes;     // bytes the TMA loads of one stage deliver
  unsigned ebuf;         // per-warp exps buffers [warp][2][NP][32] float2, after the stages
  unsigned out_mask;     // bit k: output tile k is stored (OUT_*)
  TagRec* cta_recs;      // [grid][NPART] (value, epoch tag)
  unsigned int* top_count;
};

enum { OUT_DZ = 1, OUT_DV = 2, OUT_VS = 4, OUT_PG = 8, OUT_LR = 16, OUT_LP = 32, OUT_LM = 64 };

struct CbMaps {
  CUtensorMap pi, mu, a, r, g, v, dz, dv, vs, pg, lr, lp, lm;
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y,
                                            int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int x, int y, int z,
                                             const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
      : "memory");
}

// mbarrier operations on 32-bit shared addresses computed once (no generic-to-shared
// conversion inside the loops)
__device__ __forceinline__ void mbar_wait32(uint32_t addr, uint32_t phase) {
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

// the producer's wait for the compute warps: test, then back off (its issue slots belong
// to the compute warps of its sub-partition)
__device__ __forceinline__ void mbar_wait_sleep32(uint32_t addr, uint32_t phase) {
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(phase)
        : "memory");
    if (ok) return;
    __nanosleep(64);
  }
}

// the producer's wait for a stage's release (A/B: CB_PROD_WAIT 0 = try_wait loop,
// 1 = try_wait with a suspend-time hint of CB_PROD_HINT ns, 2 = test_wait + nanosleep)
#ifndef CB_PROD_WAIT
#define CB_PROD_WAIT 0
#endif
#ifndef CB_PROD_HINT
#define CB_PROD_HINT 500
#endif
__device__ __forceinline__ void mbar_wait_prod32(uint32_t addr, uint32_t phase) {
#if CB_PROD_WAIT == 1
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITP_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITP_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase), "r"((uint32_t)CB_PROD_HINT)
      : "memory");
#elif CB_PROD_WAIT == 2
  mbar_wait_sleep32(addr, phase);
#else
  mbar_wait32(addr, phase);
#endif
}

__device__ __forceinline__ void mbar_arrive32(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx32(uint32_t addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_3d32(uint32_t dst, const CUtensorMap* map, int x, int y,
                                              int z, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d32(uint32_t dst, const CUtensorMap* map, int x, int y,
                                              uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_store_3d32(const CUtensorMap* map, int x, int y, int z,
                                               uint32_t src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(x), "r"(y), "r"(z), "r"(src)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d32(const CUtensorMap* map, int x, int y, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(src)
               : "memory");
}

// One level of the suffix scan of affine maps over the warp's 8 steps: compose this
// lane's (G, D) with the map `o` lanes further down, (G, D) o (Go, Do) = (G Go, D + G Do);
// lanes whose partner is past the warp (steps beyond the 8) keep theirs (identity).
// The shuffle's in-range predicate guards the two fp64 ops: no selects, no branch.
__device__ __forceinline__ void scan_level(double& G, double& D, int o) {
  asm("{\n"
      ".reg .pred p;\n"
      ".reg .b32 g0, g1, d0, d1;\n"
      ".reg .f64 go, dd;\n"
      "mov.b64 {g0, g1}, %0;\n"
      "mov.b64 {d0, d1}, %1;\n"
      "shfl.sync.down.b32 g0|p, g0, %2, 31, -1;\n"
      "shfl.sync.down.b32 g1, g1, %2, 31, -1;\n"
      "shfl.sync.down.b32 d0, d0, %2, 31, -1;\n"
      "shfl.sync.down.b32 d1, d1, %2, 31, -1;\n"
      "mov.b64 go, {g0, g1};\n"
      "mov.b64 dd, {d0, d1};\n"
      "@p fma.rn.f64 %1, %0, dd, %1;\n"
      "@p mul.rn.f64 %0, %0, go;\n"
      "}\n"
      : "+d"(G), "+d"(D)
      : "r"(o));
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename T>
__device__ __forceinline__ T lds(const unsigned char* p) {
  return *reinterpret_cast<const T*>(p);
}

// Row statistics of both policies for compile-time A (any parity), rows in shared
// memory.  Same arithmetic as DESIGN.md "precision": e_j = 2^{y_j}, y_j = fma(z_j, L16,
// -m L16) for bf16 (exact products; the max term is exactly 1) or (z_j - m) L32 for
// fp32; two Fast2Sum chains per policy (one per float2 half) that start at 1 >= every
// term; the log2 e truncation corrected to first order through sd = sum_j e_j (z_j - m).
// The target's (z_j, e_j) stay in registers for the gradient.
template <typename LT, int A_CT>
struct CbRow {
  static constexpr int NP = (A_CT + 1) / 2;   // float2 pairs (odd A: the last .y is padding)
  float2 z[NP], e[NP];   // target row and its exps (padding: z = -inf, e = 0)
  float m_p;             // max of the target row
  float s_p, lo_p;       // S_pi = s_p + lo_p (s_p in [1, A], lo_p the error terms)
  float sd_p;            // sum e (z - m), target
  double S_p, S_m;       // sums (corrected), fp64
  float ea_raw;          // 2^{y_a} of the target row, bit-identical to e[a]
  bool finite;
};

template <typename LT, int A_CT>
__device__ __forceinline__ void cb_load_pairs(const LT* row, float2 (&z)[(A_CT + 1) / 2]) {
  constexpr int NP = (A_CT + 1) / 2;
  if constexpr (sizeof(LT) == 2) {
    if constexpr (A_CT % 2 == 0) {  // rows start 4-byte aligned
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        // exact bf16 -> fp32 on the ALU pipe (PRMT, LOP3): the FMA pipe carries the math
        const uint32_t x = reinterpret_cast<const uint32_t*>(row)[k];
        z[k] = make_float2(__uint_as_float(__byte_perm(x, 0u, 0x1044)),
                           __uint_as_float(x & 0xffff0000u));
      }
    } else {
      const unsigned short* h = reinterpret_cast<const unsigned short*>(row);
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const float lo = __uint_as_float((uint32_t)h[2 * k] << 16);
        const float hi = (2 * k + 1 < A_CT) ? __uint_as_float((uint32_t)h[2 * k + 1] << 16)
                                            : -INFINITY;
        z[k] = make_float2(lo, hi);
      }
    }
  } else {
    const float* f = reinterpret_cast<const float*>(row);
    if constexpr (A_CT % 2 == 0) {  // rows start 8-byte aligned
#pragma unroll
      for (int k = 0; k < NP; ++k) z[k] = reinterpret_cast<const float2*>(row)[k];
    } else {
#pragma unroll
      for (int k = 0; k < NP; ++k)
        z[k] = make_float2(f[2 * k], (2 * k + 1 < A_CT) ? f[2 * k + 1] : -INFINITY);
    }
  }
}

// max over a row held as float2 pairs: a shallow tree (3-input FMNMX) instead of a
// chain through every pair
template <int NP>
__device__ __forceinline__ float row_max(const float2 (&z)[NP]) {
  float m[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) m[k] = fmaxf(z[k].x, z[k].y);
#pragma unroll
  for (int w = 1; w < NP; w *= 3) {
#pragma unroll
    for (int k = 0; k + w < NP; k += 3 * w) {
      float x = fmaxf(m[k], m[k + w]);
      if (k + 2 * w < NP) x = fmaxf(x, m[k + 2 * w]);
      m[k] = x;
    }
  }
  return m[0];
}

// One policy's exps and compensated sums over the row in `z` (max m given).
// Returns the chain heads/tails; sdz = sum e z (bf16) or sum e (z - m) (fp32).
// fp32 logits: z - m and (z - m) L32 are rounded; their exact errors (TwoSum,
// FMA residual) w_j = d_lo L32 + (d L32 - y) are accumulated as cw = sum e_j w_j,
// so that S = sum e_j (1 + ln2 w_j) to first order (bf16: both steps exact, cw = 0).
template <typename LT, int A_CT, bool KEEP>
__device__ __forceinline__ void cb_exps(const float2 (&z)[(A_CT + 1) / 2], float m,
                                        float2 (&e)[(A_CT + 1) / 2], float2& h, float2& l,
                                        float2& sdz, float2& cw) {
  constexpr int NP = (A_CT + 1) / 2;
  constexpr bool BF16 = sizeof(LT) == 2;
  constexpr float L16 = 1.44268798828125f;  // log2 e to 16 bits
  constexpr float L32 = 1.44269502f;        // fp32(log2 e)
  const float2 Lp = f2(BF16 ? L16 : L32);
  const float2 nmL = f2(BF16 ? -m * L16 : 0.f), nm = f2(-m);
  h = f2(1.f);
  l = f2(0.f);
  sdz = f2(0.f);
  cw = f2(0.f);
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    float2 y, d, w;
    if constexpr (BF16) {
      y = __ffma2_rn(z[k], Lp, nmL);
      d = z[k];
    } else {
      d = __fadd2_rn(z[k], nm);
      y = __fmul2_rn(d, Lp);
#if CB_F32_EXACT
      // TwoSum error of d = z - m, and the FMA residual of y = d L32
      const float2 bb = __fadd2_rn(d, make_float2(-z[k].x, -z[k].y));
      const float2 t = __fadd2_rn(d, make_float2(-bb.x, -bb.y));
      const float2 dlo = __fadd2_rn(__fadd2_rn(z[k], make_float2(-t.x, -t.y)),
                                    __fadd2_rn(nm, make_float2(-bb.x, -bb.y)));
      w = __ffma2_rn(dlo, Lp, __ffma2_rn(d, Lp, make_float2(-y.x, -y.y)));
#else
      w = f2(0.f);
#endif
    }
    float2 ek = make_float2(ex2_approx(y.x), ex2_approx(y.y));
    if constexpr (A_CT % 2 == 1) {
      if (k == NP - 1) {  // padding element (z = -inf): no term
        ek.y = 0.f;
        d.y = 0.f;
        if constexpr (!BF16) w.y = 0.f;
      }
    }
    if constexpr (KEEP) e[k] = ek;
    sdz = __ffma2_rn(ek, d, sdz);  // NaN if some z is inf/nan
    if constexpr (!BF16 && CB_F32_EXACT) cw = __ffma2_rn(ek, w, cw);
#if CB_PLAIN_SUMS
    h = __fadd2_rn(h, ek);
#else
    // Fast2Sum: h >= 1 >= e, so s = h + e and (h - s) + e is its exact error
    const float2 s = __fadd2_rn(h, ek);
    l = __fadd2_rn(l, __fadd2_rn(__fadd2_rn(h, make_float2(-s.x, -s.y)), ek));
    h = s;
#endif
  }
}

#ifndef CB_EARLY_RATIO
#define CB_EARLY_RATIO 0  // 1: exp64 issued before both policies' exps (A/B; 0: between the two)
#endif
// e_delta (with_mu): exp((z^pi_a - m_pi) - (z^mu_a - m_mu)) in fp64, issued as soon as the
// behaviour row's maximum is known (between the two policies' exps) so that its dependent
// DFMA chain overlaps the behaviour exps and sums (the kernel is bound by its warps'
// dependent chains, DESIGN 6a; profiles/r2_ratio_chain_ab.txt: 26.32 -> 25.78 us at large)
template <typename LT, int A_CT>
__device__ __forceinline__ void cb_stats(const LT* zrow, const LT* mrow, int a,
                                         CbRow<LT, A_CT>& R, double& xa_p, double& xa_m,
                                         bool with_mu, double& e_delta) {
  constexpr int NP = (A_CT + 1) / 2;
  constexpr bool BF16 = sizeof(LT) == 2;
  constexpr float L16 = 1.44268798828125f;
  constexpr float L32 = 1.44269502f;
  constexpr float CORR = BF16 ? 4.8884952e-06f : 1.3349930e-08f;  // ln2 (log2 e - L)
  cb_load_pairs<LT, A_CT>(zrow, R.z);
  const float mp = row_max<NP>(R.z);
  const float zap = Elem<LT>::get(zrow, a);
  xa_p = (double)zap - (double)mp;  // z_a - m, exact
  float2 hm = f2(1.f), lm = f2(0.f), sdm = f2(0.f), cwm = f2(0.f);
  float mm = 0.f;
  float2 zm[NP], em[NP];
#if CB_EARLY_RATIO
  if (with_mu) {
    cb_load_pairs<LT, A_CT>(mrow, zm);
    mm = row_max<NP>(zm);
    const float zam = Elem<LT>::get(mrow, a);
    xa_m = (double)zam - (double)mm;
    e_delta = exp64(xa_p - xa_m);
  }
#endif
  float2 hp, lp, sdp, cwp;
  cb_exps<LT, A_CT, true>(R.z, mp, R.e, hp, lp, sdp, cwp);
  if (with_mu) {
#if !CB_EARLY_RATIO
    cb_load_pairs<LT, A_CT>(mrow, zm);
    mm = row_max<NP>(zm);
    const float zam = Elem<LT>::get(mrow, a);
    xa_m = (double)zam - (double)mm;
    e_delta = exp64(xa_p - xa_m);
#endif
    cb_exps<LT, A_CT, false>(zm, mm, em, hm, lm, sdm, cwm);
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
  if constexpr (BF16) sd = __ffma2_rn(make_float2(-mp, -mm), s, sd);  // sum e (z - m)
  float2 lo = __ffma2_rn(sd, f2(CORR), __fadd2_rn(err, __fadd2_rn(make_float2(lp.x, lm.x),
                                                                  make_float2(lp.y, lm.y))));
  if constexpr (!BF16) {  // the rounding of z - m and of (z - m) L32, first order
    constexpr float LN2 = 0.693147182f;
    lo = __ffma2_rn(make_float2(cwp.x + cwp.y, cwm.x + cwm.y), f2(LN2), lo);
  }
  R.s_p = s.x;
  R.lo_p = lo.x;
  R.S_p = (double)s.x + (double)lo.x;
  R.S_m = with_mu ? (double)s.y + (double)lo.y : 1.0;
  R.m_p = mp;
  R.sd_p = sd.x;
  R.ea_raw = ex2_approx(BF16 ? fmaf(zap, L16, -mp * L16) : (zap - mp) * L32);
  R.finite = isfinite(sd.x) && isfinite(mp) && (!with_mu || (isfinite(sd.y) && isfinite(mm)));
}

// What X(j) hands to Y(j) for one lane's row (a3-a8 results that do not need the carry).

#ifndef CB_KEEPZ
#define CB_KEEPZ 1  // keep the target row's packed bf16 words in registers for a11 (A/B: 0)
#endif
template <int A_CT>
struct CbSt {
#if !CB_EBUF
  float2 e[(A_CT + 1) / 2];  // the target row's exps (a11 reuses them)
#endif
#if CB_KEEPZ
  uint32_t zw[(A_CT + 1) / 2];  // (bf16, even A) the target row's packed words
#endif
  double G, D;               // suffix composition of this row's step with the warp's later steps
  double td, rho_pg;         // r_t + gamma_t V_{t+1} - V_t; rho_pg_t
  float gm, Vt, inv_S, cshift, logpa, rest, pa, za, ea_raw;
  int a;
  bool row_ok;
};

// Per-lane fp64 sums of one compute warp (a10, a12).
struct CbAcc {
  double pg, v2, H, dz, rho;
  unsigned int clip;
};

// The learners' sum of partial k inside the kernel: this
// learner's value goes into its slot of every learner's mailbox (value, then the call tag with
// release semantics, NVLink stores), then the learners' slots of this call are added in
// learner order from the own mailbox -- bitwise the same on every learner.  The tag is the
// workspace's call epoch + 1 (every learner makes the same calls); slots alternate parity, so
// a learner one call ahead never overwrites a slot still to be read.  A learner that never
// publishes makes its term NaN after 20 s (no hang).
__device__ __forceinline__ double learners_sum(const Params& P, double v, int k, unsigned int epoch) {
  struct Slot { double v; unsigned long long tag; };
  const unsigned long long tag = (unsigned long long)epoch + 1ull;
  const int par = (int)(tag & 1ull), n = P.nlearn;
  for (int r = 0; r < n; ++r) {
    Slot* d = reinterpret_cast<Slot*>(P.mbox[r]) + ((size_t)(par * n + P.self) * NPART + k);
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(&d->v), "d"(v) : "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&d->tag), "l"(tag) : "memory");
  }
  const Slot* own = reinterpret_cast<const Slot*>(P.mbox[P.self]) + (size_t)par * n * NPART + k;
  double s = 0.0;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < n; ++r) {
    const Slot* q = own + (size_t)r * NPART;
    bool late = false;
    while (true) {
      unsigned long long t;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(t) : "l"(&q->tag) : "memory");
      if (t == tag) break;
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 20ull * 1000 * 1000 * 1000) { late = true; break; }
      __nanosleep(20);
    }
    double x;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(x) : "l"(&q->v) : "memory");
    s += late ? __longlong_as_double(0x7ff8000000000000ll) : x;
  }
  return s;
}

// ---------------------------------------------------------------------------
// The kernel.  GEN: a Section 5.2.2 variant / App. E.3 q estimate / behaviour
// log-probs (false: plain V-trace, that logic compiled out); MULP: the behaviour is
// log mu(a_t) [T][B] (no mu tile, no mu statistics; implies GEN).  LOSS: the fused
// loss + gradients (vtrace_loss_and_grad), else vtrace_from_logits' outputs.
// Plain-load producer (PLAIN: shapes whose pitches or bases do not allow TMA boxes, e.g. the
// toy's 24-byte rows): the producer warp's 32 lanes copy the same tiles with ordinary loads
// into the same shared-memory layout (zero outside the batch), arrive on `full` (one arrival
// per lane), and copy the output tiles back with ordinary stores.  Small problems only.
template <typename LT, int A_CT, bool LOSS, bool MULP>
struct CbPlainIO {
  const Params& P;
  const CbParams& C;
  unsigned char* smem;
  int c0, lane;
  __device__ __forceinline__ void load(int j, int s) const {
    const int T = P.T32, B = P.B32, Ts = C.Ts, Bc = C.Bc;
    const int tb = (C.J - 1 - j) * Ts;
    unsigned char* sb = smem + (size_t)s * C.stage;
    LT* zp = reinterpret_cast<LT*>(sb + C.pi);
    LT* zm = reinterpret_cast<LT*>(sb + C.mu);
    const LT* gp = reinterpret_cast<const LT*>(P.pi);
    const LT* gm = reinterpret_cast<const LT*>(P.mu);
    // logits rows ((cg Ts + t) 4 + c) A + k (g = 1)
    const int nz = Ts * Bc * A_CT;
    for (int i = lane; i < nz; i += 32) {
      const int k = i % A_CT, row = i / A_CT;
      const int c = row & 3, rest = row >> 2;
      const int t = rest % Ts, cg = rest / Ts;
      const int tt = tb + t, b = c0 + 4 * cg + c;
      const bool ok = tt < T && b < B;
      const size_t gi = ((size_t)tt * B + b) * A_CT + k;
      zp[i] = ok ? gp[gi] : LT(0.f);
      if constexpr (!MULP) zm[i] = ok ? gm[gi] : LT(0.f);
    }
    const int ns = Ts * Bc;
    for (int i = lane; i < ns; i += 32) {  // [Ts][Bc] per-step tiles
      const int t = i / Bc, bl = i - t * Bc;
      const int tt = tb + t, b = c0 + bl;
      const bool ok = tt < T && b < B;
      const size_t gi = (size_t)tt * B + b;
      reinterpret_cast<int*>(sb + C.a)[i] = ok ? P.actions[gi] : 0;
      reinterpret_cast<float*>(sb + C.r)[i] = ok ? P.rew[gi] : 0.f;
      reinterpret_cast<float*>(sb + C.gm)[i] = ok ? P.disc[gi] : 0.f;
      if constexpr (MULP)
        reinterpret_cast<float*>(sb + C.mu)[i] = ok ? reinterpret_cast<const float*>(P.mu)[gi] : 0.f;
    }
    for (int i = lane; i < ns + Bc; i += 32) {  // V [Ts + 1][Bc]
      const int t = i / Bc, bl = i - t * Bc;
      const int tt = tb + t, b = c0 + bl;
      const bool ok = tt < T && b < B;
      reinterpret_cast<float*>(sb + C.v)[i] = ok ? P.val[(size_t)tt * B + b] : 0.f;
    }
  }
  __device__ __forceinline__ void store(int j, int s, unsigned om) const {
    const int T = P.T32, B = P.B32, Ts = C.Ts, Bc = C.Bc;
    const int tb = (C.J - 1 - j) * Ts;
    const unsigned char* sb = smem + (size_t)s * C.stage;
    if (om & OUT_DZ) {
      const LT* zp = reinterpret_cast<const LT*>(sb + C.pi);
      LT* gd = reinterpret_cast<LT*>(P.dlogits);
      const int nz = Ts * Bc * A_CT;
      for (int i = lane; i < nz; i += 32) {
        const int k = i % A_CT, row = i / A_CT;
        const int c = row & 3, rest = row >> 2;
        const int t = rest % Ts, cg = rest / Ts;
        const int tt = tb + t, b = c0 + 4 * cg + c;
        if (tt < T && b < B) gd[((size_t)tt * B + b) * A_CT + k] = zp[i];
      }
    }
    const int ns = Ts * Bc;
    auto out = [&](unsigned bit, unsigned off, float* g) {
      if (!(om & bit)) return;
      for (int i = lane; i < ns; i += 32) {
        const int t = i / Bc, bl = i - t * Bc;
        const int tt = tb + t, b = c0 + bl;
        if (tt < T && b < B) g[(size_t)tt * B + b] = reinterpret_cast<const float*>(sb + off)[i];
      }
    };
    out(OUT_DV, C.dv, P.dvalues);
    out(OUT_VS, C.vs, P.vs);
    out(OUT_PG, C.pg, P.pg_adv);
    out(OUT_LR, C.lr, P.log_rhos);
    out(OUT_LP, C.lp, P.lp_out);
    out(OUT_LM, C.lm, P.lm_out);
  }
};

template <typename LT, int A_CT, bool LOSS, bool GEN, bool MULP, bool PLAIN = false>
__global__ void __launch_bounds__((CB_MAX_WARPS + 1) * 32, 1)
    vtrace_cb_kernel(const Params P, const CbParams C, const __grid_constant__ CbMaps M) {
  static_assert(A_CT > 0, "compile-time A");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[CB_MAX_STAGES], done[CB_MAX_STAGES];
  __shared__ double agg[2][CB_MAX_WARPS][4][2];  // [parity][warp][column][G, D]
  __shared__ double wpart[CB_MAX_WARPS + 2][NPART];  // [warps | producer | own CTA sum]
  __shared__ unsigned int s_epoch, s_last;
  __shared__ __align__(8) uint64_t ep_bar;  // the producer has read the call's epoch

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) CB_STAMP(0);
  constexpr int A = A_CT;
  constexpr bool BF16 = sizeof(LT) == 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NW = C.ncg * C.nts;
  const int T = P.T32, B = P.B32;
  const int c0 = blockIdx.x * C.Bc;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C.nstage; ++s) {
      mbar_init(&full[s], PLAIN ? 32 : 1);
      mbar_init(&done[s], NW);
    }
    mbar_init(&ep_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (PLAIN && warp == NW) {
    // ---------------- producer, plain loads (all 32 lanes) ----------------
    const CbPlainIO<LT, A_CT, LOSS, MULP> io{P, C, smem, c0, lane};
    const uint32_t full0 = smem_u32(&full[0]), done0 = smem_u32(&done[0]);
    const int npre = min(C.nstage, C.J);
    for (int s2 = 0; s2 < npre; ++s2) {
      io.load(s2, s2);
      mbar_arrive32(full0 + 8u * s2);  // (release: this lane's tile writes)
    }
    int s = 0;
    uint32_t ph = 0;
    for (int j = 0; j < C.J; ++j) {
      mbar_wait32(done0 + 8u * s, ph);
      if (j == 0) {
        if (P.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
        if (lane == 0) {
          s_epoch = *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch) & 0x3fffffffu;
          mbar_arrive(&ep_bar);
        }
      }
      io.store(j, s, C.out_mask);
      __syncwarp();
      if (j + C.nstage < C.J) {
        io.load(j + C.nstage, s);
        mbar_arrive32(full0 + 8u * s);
      }
      if (++s == C.nstage) {
        s = 0;
        ph ^= 1u;
      }
    }
  } else if (warp == NW) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const int zc = c0 / (4 * C.g);  // first logits column segment of the block
      const uint32_t sm0 = smem_u32(smem), full0 = smem_u32(&full[0]), done0 = smem_u32(&done[0]);
      auto load = [&](int j, int s) {
        const int tb = (C.J - 1 - j) * C.Ts;
        const uint32_t sb = sm0 + (uint32_t)s * C.stage, fb = full0 + 8u * s;
#if defined(CB_ABLATE) && CB_ABLATE == 1
        if (j >= C.nstage) {  // timing ablation: compute on the stages' stale data
          mbar_arrive32(fb);
          return;
        }
#endif
        mbar_expect_tx32(fb, C.tx_bytes);
        tma_load_3d32(sb + C.pi, &M.pi, 0, tb, zc, fb);
        if constexpr (MULP) {
          tma_load_2d32(sb + C.mu, &M.mu, c0, tb, fb);
        } else {
          tma_load_3d32(sb + C.mu, &M.mu, 0, tb, zc, fb);
        }
        tma_load_2d32(sb + C.a, &M.a, c0, tb, fb);
        tma_load_2d32(sb + C.r, &M.r, c0, tb, fb);
        tma_load_2d32(sb + C.gm, &M.g, c0, tb, fb);
        tma_load_2d32(sb + C.v, &M.v, c0, tb, fb);
      };
      // the first stage alone, then the rest once it has landed: the first iteration's
      // data is not queued behind the whole ring's (all SMs fill their rings at once)
      const int npre = min(C.nstage, C.J);
      load(0, 0);
      if (npre > 1) {
        mbar_wait32(full0, 0u);
        for (int s = 1; s < npre; ++s) load(s, s);
      }
      int s = 0;
      uint32_t ph = 0;
      for (int j = 0; j < C.J; ++j) {
        mbar_wait_prod32(done0 + 8u * s, ph);
        if (j == 0) {
          // (programmatic dependent launch: the first global write waits for the previous
          // kernel on the stream).  The call's epoch (it tags the partial-sum records) is
          // final from here on: read it now, off the tail of the kernel
          if (P.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
          s_epoch = *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch) & 0x3fffffffu;
          mbar_arrive(&ep_bar);
        }
        const int tb = (C.J - 1 - j) * C.Ts;
        const uint32_t sb = sm0 + (uint32_t)s * C.stage;
#if defined(CB_ABLATE) && CB_ABLATE == 1
        const unsigned om = 0;  // timing ablation: no stores
#else
        const unsigned om = C.out_mask;
#endif
        if (om & OUT_DZ) tma_store_3d32(&M.dz, 0, tb, zc, sb + C.pi);
        if (om & OUT_DV) tma_store_2d32(&M.dv, c0, tb, sb + C.dv);
        if (om & OUT_VS) tma_store_2d32(&M.vs, c0, tb, sb + C.vs);
        if (om & OUT_PG) tma_store_2d32(&M.pg, c0, tb, sb + C.pg);
        if (om & OUT_LR) tma_store_2d32(&M.lr, c0, tb, sb + C.lr);
        if (om & OUT_LP) tma_store_2d32(&M.lp, c0, tb, sb + C.lp);
        if (om & OUT_LM) tma_store_2d32(&M.lm, c0, tb, sb + C.lm);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (j + C.nstage < C.J) {
          // the stores must have read the stage before it is refilled
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          load(j + C.nstage, s);
        }
        if (++s == C.nstage) {
          s = 0;
          ph ^= 1u;
        }
      }
      // the last stores must have read their stage before the CTA's shared memory goes
      // away (their global writes complete with the grid)
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  } else {
    // ---------------- compute warp (cg, ts) ----------------
    // Software pipeline over the iterations: X(j) is everything of iteration j that
    // does not need the recursion carry (a1-a7, the warp's local affine scan, the
    // carry-free outputs); Y(j) folds the carry in (A_t, q, pg_adv, a9-a11) and
    // releases the stage.  The body runs X(j+1) next to Y(j) (independent), so each
    // warp has two rows' worth of instruction-level parallelism.
    const int cg = warp % C.ncg, ts = warp / C.ncg;
    const int tl = lane >> 2, c = lane & 3;
    const int bl = 4 * cg + c;  // column within the block
    const int b = c0 + bl;
    const bool col_ok = b < B;
    const float boot = col_ok ? __ldg(P.boot + b) : 0.f;
    // shared-memory offsets of this lane's row inside a stage
    const int seg = cg / C.g, sub = cg - seg * C.g;
    const unsigned zoff =
        (unsigned)((((seg * C.Ts + 8 * ts + tl) * C.g + sub) * 4 + c) * A * (int)sizeof(LT));
    const unsigned soff = (unsigned)(((8 * ts + tl) * C.Bc + bl) * 4);
    const unsigned voff = soff + (unsigned)(C.Bc * 4);
    const float ce = (float)P.c_e, cv = (float)P.c_v;
    const uint32_t full0 = smem_u32(&full[0]), done0 = smem_u32(&done[0]);
    constexpr int NPc = CbRow<LT, A_CT>::NP;
    // the lane's row inside each tile of a stage (logits tile [ncg/g][Ts][4gA], step
    // tiles [Ts][Bc], V tile [Ts + 1][Bc], output tiles [Ts][Bc])
    VT_CHECK(zoff + (unsigned)(A * sizeof(LT)) <= (unsigned)(C.Bc * A * sizeof(LT) * C.Ts));
    VT_CHECK(C.pi + zoff + (unsigned)(A * sizeof(LT)) <= C.mu);
    VT_CHECK(soff + 4u <= (unsigned)(C.Bc * 4 * C.Ts) && voff + 4u <= (unsigned)(C.Bc * 4 * (C.Ts + 1)));
    VT_CHECK(C.nstage >= 2 && C.nstage <= CB_MAX_STAGES && NW <= CB_MAX_WARPS);
    // one threshold for rho, c and rho_pg (rho_bar = c_bar = pg_rho_bar, lambda = 1: the
    // paper's setting): one min instead of three
    const bool one_bar = !GEN && P.rho_bar == P.c_bar && P.rho_bar == P.pg_rho_bar && P.lambda == 1.0;
    double carry = 0.0;  // A = v - V just after the next iteration to finish (A_T = 0)
    CbAcc acc = {0.0, 0.0, 0.0, 0.0, 0.0, 0u};
    // loop-invariant switches, kept in predicates (not re-read from parameter space)
    const bool want_vs = (C.out_mask & OUT_VS) != 0, want_pg = (C.out_mask & OUT_PG) != 0;
    const bool want_lr = (C.out_mask & OUT_LR) != 0, want_lp = (C.out_mask & OUT_LP) != 0;
    const bool want_lm = (C.out_mask & OUT_LM) != 0;
    const int tdec = C.Ts;  // X(j) rows: t = t_first - j * Ts
    const int t_first = (C.J - 1) * C.Ts + 8 * ts + tl;
    int sx = 0, sy = 0;         // stages of the next X and the next Y
    uint32_t phx = 0;           // parity of full[sx]'s next completion

    // ---- X(j): a1-a7 and the local scan of this lane's row (no carry) ------------
    auto X = [&](const int j, CbSt<A_CT>& S) {
      const int t = t_first - j * tdec;
      const bool row_ok = col_ok && (t < T);
      unsigned char* sb = smem + (size_t)sx * C.stage;
      VT_CHECK(sx >= 0 && sx < C.nstage);
      mbar_wait32(full0 + 8u * sx, phx);
      if (j == 0 && threadIdx.x == 0) CB_STAMP(1);
      const int a_raw = lds<int>(sb + C.a + soff);
      const float rt = lds<float>(sb + C.r + soff);
      const float gm = lds<float>(sb + C.gm + soff);
      const float Vt = lds<float>(sb + C.v + soff);
      const float Vnt = lds<float>(sb + C.v + voff);  // (row T of the tile: zero-filled)
      const float Vn = (t + 1 < T) ? Vnt : boot;        // V(x_T) = bootstrap
      const int a = min(max(a_raw, 0), A - 1);
      VT_CHECK(a >= 0 && a < A);
      const LT* zrow = reinterpret_cast<const LT*>(sb + C.pi + zoff);
      const LT* mrow = reinterpret_cast<const LT*>(sb + C.mu + zoff);
      CbRow<LT, A_CT> R;
      double xa_p, xa_m = 0.0, e_delta = 1.0;
      cb_stats<LT, A_CT>(zrow, mrow, a, R, xa_p, xa_m, !MULP, e_delta);
      float lmu = 0.f;
      if constexpr (MULP) {
        lmu = lds<float>(sb + C.mu + soff);  // log mu(a_t), given (S_m = 1)
        xa_m = (double)lmu;
        e_delta = exp64(xa_p - xa_m);
      }
      // a5, a7: pi(a)/mu(a) = exp((z^pi_a - m_pi) - (z^mu_a - m_mu)) S_mu / S_pi
      const double ratio = e_delta * ddiv_pos(R.S_m, R.S_p);
#if CB_TD32
      const double td = (double)(fmaf(gm, Vn, (float)reward_transform(rt, P.reward_mode)) - Vt);
#else
      const double td = reward_transform(rt, P.reward_mode) + (double)gm * (double)Vn - (double)Vt;
#endif
      StepWeights sw;
      if (one_bar) {
        const double rh = dmin_t(P.rho_bar, ratio);
        sw = StepWeights{rh, rh, rh};
      } else {
        sw = step_weights<GEN>(P, ratio);
      }
      const float Sf = R.s_p + R.lo_p;
      const float inv_S = rcp_approx(Sf);
      const float lse = R.m_p + __logf(Sf);
      const float cshift = fmaf(R.sd_p, inv_S, R.m_p);  // lse - H
      const float za = BF16 ? __uint_as_float((uint32_t)reinterpret_cast<const unsigned short*>(zrow)[a] << 16)
                            : reinterpret_cast<const float*>(zrow)[a];
      constexpr float CORR = BF16 ? 4.8884952e-06f : 1.3349930e-08f;
      const float ea_c = fmaf(R.ea_raw * CORR, za - R.m_p, R.ea_raw);  // exp(z_a - m), corrected
      // a8: this row's affine map; suffix scan over the warp's 8 steps, per column:
      // lanes c, c+4, ..., c+28 are steps 0..7 of column c, (G1, D1) o (G2, D2) =
      // (G1 G2, D1 + G1 D2); steps past the unroll are identity maps
      double Gi = row_ok ? (double)gm * sw.c : 1.0;  // gamma_t c_t
      double Di = row_ok ? sw.rho * td : 0.0;        // delta_t V
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) scan_level(Gi, Di, o);
      if (C.nts > 1 && tl == 0) {  // the warp's 8-step aggregate for the column group
        agg[j & 1][warp][c][0] = Gi;
        agg[j & 1][warp][c][1] = Di;
      }
#if CB_EBUF
      {  // the target exps wait in shared memory for Y(j) (element-major: conflict-free)
        float2* eb = reinterpret_cast<float2*>(smem + C.ebuf) + ((warp * 2 + (j & 1)) * NPc) * 32 + lane;
#pragma unroll
        for (int k = 0; k < NPc; ++k) eb[k * 32] = R.e[k];
      }
#else
#pragma unroll
      for (int k = 0; k < NPc; ++k) S.e[k] = R.e[k];
#endif
      S.G = Gi;
      S.D = Di;
      S.td = td;
      S.rho_pg = sw.rho_pg;
      S.gm = gm;
      S.Vt = Vt;
      S.inv_S = inv_S;
      S.cshift = cshift;
      S.logpa = za - lse;
      S.rest = ((R.s_p - ea_c) + R.lo_p) * inv_S;  // 1 - pi(a) without cancellation
      S.pa = ea_c * inv_S;                         // pi(a), relative accuracy
      S.za = za;
      S.ea_raw = R.ea_raw;
#if CB_KEEPZ
      if constexpr (sizeof(LT) == 2 && A_CT % 2 == 0) {
#pragma unroll
        for (int k = 0; k < NPc; ++k) S.zw[k] = reinterpret_cast<const uint32_t*>(zrow)[k];
      }
#endif
      S.a = a;
      S.row_ok = row_ok;
      if constexpr (!LOSS) {  // carry-free outputs of vtrace_from_logits
        if (row_ok) {
          if (want_lr) *reinterpret_cast<float*>(sb + C.lr + soff) = (float)log(ratio);
          if (want_lp) *reinterpret_cast<float*>(sb + C.lp + soff) = (float)(xa_p - log(R.S_p));
          if (want_lm) *reinterpret_cast<float*>(sb + C.lm + soff) = (float)(xa_m - log(R.S_m));
        }
      }
      if (row_ok) {
        acc.rho += sw.rho;  // the rho_t in delta_t (reading r6)
        if ((!GEN || P.correction == VT_CORRECTION_VTRACE) && ratio > P.rho_bar) ++acc.clip;
        if constexpr (LOSS) acc.H += (double)(lse - cshift);
      }
      // data checks (reading r3): one NaN probe for r, V and V' (x * 0 is NaN for +-inf and
      // NaN), a range test for gamma, the action clamp, the row statistics' finiteness
      const float probe = fmaf(rt, 0.f, fmaf(Vt, 0.f, Vn * 0.f));
      bool bad = (a_raw != a) || !R.finite || (probe != 0.f) || !(gm >= 0.f && gm <= 1.f);
      if constexpr (MULP) bad = bad || !isfinite(lmu);
      if (row_ok && bad) {
        if (P.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
        const long long row = (long long)t * B + b;
        if (a_raw != a) record_bad(P.ws, row, VT_DATA_ACTION);
        if (!R.finite || (MULP && !isfinite(lmu))) record_bad(P.ws, row, VT_DATA_LOGITS);
        if (!isfinite(rt)) record_bad(P.ws, row, VT_DATA_REWARD);
        if (!isfinite(Vt)) record_bad(P.ws, row, VT_DATA_VALUE);
        if (!(gm >= 0.f && gm <= 1.f)) record_bad(P.ws, row, VT_DATA_DISCOUNT);
        if (!isfinite(Vn) && t + 1 == T) record_bad(P.ws, (long long)T * B + b, VT_DATA_VALUE);
      }
      sx = (sx + 1 == C.nstage) ? 0 : sx + 1;
      phx ^= (sx == 0) ? 1u : 0u;
    };

    // ---- Y(j): the carry, a9-a11, release of the stage ------------------------------
    auto Y = [&](const int j, const CbSt<A_CT>& S) {
      unsigned char* sb = smem + (size_t)sy * C.stage;
      VT_CHECK(sy >= 0 && sy < C.nstage && S.a >= 0 && S.a < A);
      double cin = carry;  // A just after this warp's 8 steps
      if (C.nts > 1) {
        // the group's aggregates of iteration j (published by X(j), before the barrier)
        const int par = j & 1;
        VT_CHECK((C.nts - 1) * C.ncg + cg < NW);
        if (tl == 0) {
          double x = carry;
          for (int q = C.nts - 1; q > ts; --q)
            x = fma(agg[par][q * C.ncg + cg][c][0], x, agg[par][q * C.ncg + cg][c][1]);
          cin = x;
          for (int q = ts; q >= 0; --q)
            x = fma(agg[par][q * C.ncg + cg][c][0], x, agg[par][q * C.ncg + cg][c][1]);
          carry = x;  // A at the iteration's first step: the next iteration's carry
        }
        cin = __shfl_sync(0xffffffffu, cin, c);
        carry = __shfl_sync(0xffffffffu, carry, c);
      }
      const double A_t = fma(S.G, cin, S.D);  // A_t = v_t - V(x_t)
      double A_n = shfl_down_d(A_t, 4);       // A_{t+1}
      if (tl == 7) A_n = cin;
      if (C.nts == 1) carry = __shfl_sync(0xffffffffu, A_t, c);  // A at the first step
      // pg_adv = rho_pg (r + gamma v_{t+1} - V) = rho_pg (td + gamma A_{t+1})
      // (q_s = r_s + gamma V(x_{s+1}) instead with q_values: App. E.3)
      const double pgd = S.rho_pg * ((GEN && P.q_values) ? S.td : fma((double)S.gm, A_n, S.td));
      const float pgr = (float)pgd;
      if (want_vs) *reinterpret_cast<float*>(sb + C.vs + soff) = (float)((double)S.Vt + A_t);
      if (want_pg) *reinterpret_cast<float*>(sb + C.pg + soff) = pgr;
      if constexpr (LOSS) {
        // epsilon-correction (readings c11, r7): the policy-gradient term uses
        // log(pi_a + eps); its logit gradient is the plain one times pi_a / (pi_a + eps)
        float pge = pgr, logpa = S.logpa;
        if (GEN && P.correction == VT_CORRECTION_EPSILON) {
          const float rr = P.eps / S.pa;
          logpa = S.pa > 0.f ? S.logpa + log1pf(rr) : logf(P.eps);
          pge = pgr / (1.f + rr);
        }
        // dz_j = pi_j (pg + c_e (log pi_j + H)) = e_j / S (alpha + c_e z_j)  (j != a;
        // P:257), alpha = pg - c_e (lse - H); in place over z^pi
        const float alpha = fmaf(-ce, S.cshift, pge);
        const float2 k1 = f2(ce * S.inv_S), k0 = f2(alpha * S.inv_S);
        LT* zw = reinterpret_cast<LT*>(sb + C.pi + zoff);
        float2 zr[NPc];
#if CB_KEEPZ
        if constexpr (sizeof(LT) == 2 && A_CT % 2 == 0) {
#pragma unroll
          for (int k = 0; k < NPc; ++k)
            zr[k] = make_float2(__uint_as_float(__byte_perm(S.zw[k], 0u, 0x1044)),
                                __uint_as_float(S.zw[k] & 0xffff0000u));
        } else {
          cb_load_pairs<LT, A_CT>(zw, zr);
        }
#else
        cb_load_pairs<LT, A_CT>(zw, zr);  // the target row again (smem)
#endif
#if CB_EBUF
        float2 er[NPc];
        {
          const float2* eb = reinterpret_cast<const float2*>(smem + C.ebuf) + ((warp * 2 + (j & 1)) * NPc) * 32 + lane;
#pragma unroll
          for (int k = 0; k < NPc; ++k) er[k] = eb[k * 32];
        }
#else
        const float2 (&er)[NPc] = S.e;
#endif
        float2 sq2 = f2(0.f);
        constexpr int NP = (A_CT + 1) / 2;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const float2 d2 = __fmul2_rn(er[k], __ffma2_rn(k1, zr[k], k0));
          if constexpr (A_CT % 2 == 1) {
            if (k == NP - 1) {
              sq2 = make_float2(fmaf(d2.x, d2.x, sq2.x), sq2.y);
              if constexpr (BF16) reinterpret_cast<__nv_bfloat16*>(zw)[2 * k] = __float2bfloat16_rn(d2.x);
              else reinterpret_cast<float*>(zw)[2 * k] = d2.x;
              continue;
            }
          }
          sq2 = __ffma2_rn(d2, d2, sq2);
          if constexpr (BF16) {
            if constexpr (A_CT % 2 == 0) {
              __nv_bfloat162 h2 = __floats2bfloat162_rn(d2.x, d2.y);
              reinterpret_cast<uint32_t*>(zw)[k] = *reinterpret_cast<uint32_t*>(&h2);
            } else {
              reinterpret_cast<__nv_bfloat16*>(zw)[2 * k] = __float2bfloat16_rn(d2.x);
              reinterpret_cast<__nv_bfloat16*>(zw)[2 * k + 1] = __float2bfloat16_rn(d2.y);
            }
          } else {
            if constexpr (A_CT % 2 == 0) {
              reinterpret_cast<float2*>(zw)[k] = d2;
            } else {
              reinterpret_cast<float*>(zw)[2 * k] = d2.x;
              reinterpret_cast<float*>(zw)[2 * k + 1] = d2.y;
            }
          }
        }
        // the taken action: dz_a = -pg (1 - pi_a) + c_e pi_a (log pi_a + H); the loop's
        // value for j = a (same operations: bit-identical) leaves the sum of squares
        const float d_wrong = S.ea_raw * fmaf(k1.x, S.za, k0.x);
        const float d_a = fmaf(-pge, S.rest, ce * (1.f - S.rest) * (S.za - S.cshift));
        if constexpr (BF16) reinterpret_cast<__nv_bfloat16*>(zw)[S.a] = __float2bfloat16_rn(d_a);
        else reinterpret_cast<float*>(zw)[S.a] = d_a;
        const float sq = fmaf(d_a, d_a, fmaf(-d_wrong, d_wrong, sq2.x + sq2.y));
        *reinterpret_cast<float*>(sb + C.dv + soff) = (float)(-(double)cv * A_t);  // c_v (V - v)
        if (S.row_ok) {
          acc.pg = fma(-pgd, (double)logpa, acc.pg);  // -pg_adv log pi(a)  (log(pi(a) + eps))
          acc.v2 = fma(A_t, A_t, acc.v2);
          acc.dz += (double)sq;
        }
      }
      // release the stage: outputs written (generic proxy) before the TMA stores read them
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive32(done0 + 8u * sy);
      if (j == C.J - 1 && threadIdx.x == 0) CB_STAMP(2);
      sy = (sy + 1 == C.nstage) ? 0 : sy + 1;
    };

    auto group_sync = [&]() {
#if defined(CB_NOSYNC)
      // timing A/B only (wrong results): no barrier between the group's X(j) and Y(j)
#else
      if (C.nts > 1) named_bar(1 + cg, 32 * C.nts);  // the group's X(j) aggregates are out
#endif
    };
#if defined(CB_STAGGER) && CB_STAGGER > 0
    // phase offset between the warps of a sub-partition (warps w and w + 4 share one):
    // odd slots start later, so the sub-partition's warps are not all in their
    // MUFU-heavy statistics (or fp64 chain) at the same time
    if ((warp >> 2) & 1) __nanosleep(CB_STAGGER);
#endif
#if defined(CB_ABLATE) && CB_ABLATE == 2
    // timing ablation: data movement only (no arithmetic; garbage outputs)
    for (int j = 0; j < C.J; ++j) {
      mbar_wait32(full0 + 8u * sx, phx);
      if (++sx == C.nstage) { sx = 0; phx ^= 1u; }
      group_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive32(done0 + 8u * sy);
      if (j == C.J - 1 && threadIdx.x == 0) CB_STAMP(2);
      if (++sy == C.nstage) sy = 0;
    }
#elif !CB_PIPE
    for (int j = 0; j < C.J; ++j) {
      CbSt<A_CT> S;
      X(j, S);
      group_sync();
      Y(j, S);
    }
#else
    CbSt<A_CT> SA, SB;
    X(0, SA);
    int j = 0;
    for (; j + 2 < C.J; j += 2) {
      group_sync();
      X(j + 1, SB);
      Y(j, SA);
      group_sync();
      X(j + 2, SA);
      Y(j + 1, SB);
    }
    if (j + 1 < C.J) {
      group_sync();
      X(j + 1, SB);
      Y(j, SA);
      group_sync();
      Y(j + 1, SB);
    } else {
      group_sync();
      Y(j, SA);
    }
#endif
    // ---- a12: per-lane fp64 sums -> warp -> CTA ---------------------------------
    double part[NPART] = {acc.pg, 0.5 * acc.v2, acc.H, 0.0, acc.dz,
                          (double)cv * (double)cv * acc.v2, acc.rho, (double)acc.clip};
#pragma unroll
    for (int k = 0; k < NPART; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part[k] += __shfl_xor_sync(0xffffffffu, part[k], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < NPART; ++k) wpart[warp][k] = part[k];
    }
  }
  if (!LOSS || P.partials == nullptr) return;
  // The producer leaves once its last stores have read shared memory: the partials tail
  // runs on the compute warps alone, in parallel with that drain (named barrier 15 over
  // the NW compute warps; the group barriers use 1..ncg <= 14)
  if (warp == NW) return;
  named_bar(15, 32 * NW);  // wpart complete
  mbar_wait32(smem_u32(&ep_bar), 0u);  // s_epoch set (the producer's first iteration)
  const int S = gridDim.x;
  const unsigned int epoch = s_epoch;
  const unsigned long long tag = ((unsigned long long)epoch << 2) | 3ull;
  if (warp == 0) {
    if (P.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    double v = 0.0;  // lane k < NPART: this CTA's sum k, warps in order
    if (lane < NPART)
      for (int w2 = 0; w2 < NW; ++w2) v += wpart[w2][lane];
    VT_CHECK((int)blockIdx.x < S);
    if (lane < NPART) st_tag16(C.cta_recs + (size_t)blockIdx.x * NPART + lane, v, tag);
    if (lane < NPART) wpart[CB_MAX_WARPS + 1][lane] = v;  // (the last CTA's own, from shared)
    unsigned int prev = 0;
    if (lane == 0) prev = atomicAdd(C.top_count, 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (lane == 0) {
      CB_STAMP(3);
      s_last = (prev == (unsigned int)(S - 1)) ? 1u : 0u;
      if (s_last) *C.top_count = 0u;  // every ticket of this call is taken: re-arm
    }
  }
  named_bar(15, 32 * NW);
  if (!s_last) return;
  if (threadIdx.x == 0) CB_STAMP(5);
  // the last CTA: all its warps request the other CTAs' records at once (warp w2 takes
  // the contiguous CTA range [w2 S / W, (w2 + 1) S / W), lane = (CTA, partial)), re-poll
  // any record whose tag is not this call's yet, add their range in CTA order; warp 0
  // then adds the warps' sums in order: a fixed tree, independent of the arrival order
  const int W = NW;
  {
    const int c_lo = warp * S / W, c_hi = (warp + 1) * S / W;
    const int k = lane & (NPART - 1), sub = lane >> 3;  // 4 CTAs per pass, one partial per lane
    double acc_k = 0.0;
    for (int cbase = c_lo; cbase < c_hi; cbase += 4 * 4) {
      double x[4];
      unsigned long long tg[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ci = cbase + 4 * q + sub;
        x[q] = 0.0;
        tg[q] = tag;
        if (ci < c_hi) {
          if (ci == (int)blockIdx.x) x[q] = wpart[CB_MAX_WARPS + 1][k];
          else ld_tag16(C.cta_recs + (size_t)ci * NPART + k, x[q], tg[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ci = cbase + 4 * q + sub;
        int spins = 0;
        while (ci < c_hi && ci != (int)blockIdx.x && tg[q] != tag) {
          if (++spins > 4) __nanosleep(32);
          ld_tag16(C.cta_recs + (size_t)ci * NPART + k, x[q], tg[q]);
        }
      }
      // CTA order inside the pass: q major, sub minor -> ci = cbase + 4 q + sub
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double y = x[q];
        // add the 4 CTAs of step q (lanes sub = 0..3 hold consecutive CTAs) in order
        const double y1 = __shfl_sync(0xffffffffu, y, (lane & 7) + 8);
        const double y2 = __shfl_sync(0xffffffffu, y, (lane & 7) + 16);
        const double y3 = __shfl_sync(0xffffffffu, y, (lane & 7) + 24);
        const double y0 = __shfl_sync(0xffffffffu, y, lane & 7);
        acc_k += ((y0 + y1) + y2) + y3;
      }
    }
    if (lane < NPART) wpart[warp][lane] = acc_k;
    if (threadIdx.x == 0) CB_STAMP(6);
  }
  named_bar(15, 32 * NW);
  if (threadIdx.x == 0) CB_STAMP(7);
  if (warp == 0) {
    // lane k < NPART adds partial k over the warps in order (one short chain per lane,
    // not one serial chain through all of them)
    double x = 0.0;
    if (lane < NPART)
      for (int w2 = 0; w2 < W; ++w2) x += wpart[w2][lane];
    const double pg = __shfl_sync(0xffffffffu, x, VT_P_PG_LOSS);
    const double bl = __shfl_sync(0xffffffffu, x, VT_P_BASELINE_LOSS);
    const double en = __shfl_sync(0xffffffffu, x, VT_P_ENTROPY_SUM);
    if (lane == VT_P_TOTAL_LOSS) x = pg + P.c_v * bl - P.c_e * en;
    if (P.nlearn > 1 && lane < NPART) x = learners_sum(P, x, lane, epoch);
    if (lane < NPART) P.partials[lane] = x;
    if (lane == 0) *reinterpret_cast<volatile unsigned int*>(&P.ws->epoch) = (epoch + 1u) & 0x3fffffffu;
    if (lane == 0) CB_STAMP(4);
  }
}

}  // namespace vtb200
