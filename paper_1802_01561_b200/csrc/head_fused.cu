// NEXT #3, second half: the learner's output layer fused with the whole
// V-trace path and its backward -- [z^pi | V] = h W + b over all folded steps (P:173-174,
// Fig. 3), the V-trace targets, loss and dL/dz, dL/dV of Section 4 as the GEMM's epilogue
// (z^pi and V never leave the SM), then the head's backward dh = dZ W^T and
// dW = h^T dZ, db = sum dZ on the same tile while h is still in shared memory.
// See include/vtrace.h (vtrace_head_loss_and_grad), reading r12.
//
// Persistent kernel, one CTA (11 warps) per SM.  A tile is 8 trajectories x 16 steps =
// 128 rows of h (MMA M = 128), row r = 16 b + t; a CTA owns blocks of 8 trajectories and
// walks each block's 16-step chunks backwards in time, so the recursion's carry stays in
// the epilogue warps' registers.
//   warp 8      producer: TMA of h (H/64 boxes of 64 x 16 x 8, 128-byte swizzle), the
//               behaviour logits, a, r, gamma of a tile into one of NS stages
//   warp 9      forward MMA: z = h W^T-tile (tcgen05, M=128 N=32 K=16, bf16 -> fp32) into
//               one of two TMEM accumulators
//   warps 0-3   the V-trace epilogue (lane = row, TMEM lanes 32w..32w+31): row statistics,
//               ratio, TD error, 16-step suffix scan of the affine maps, the carry, the
//               gradient row dZ = [dL/dz | dL/dV] written as bf16 hi + lo (dZ = hi + lo to
//               2^-17) into shared memory (64-byte swizzle), db by a butterfly over lanes
//   warp 10     backward MMA: dh = [hi|lo] W (A = dZ K-major, B = W^T MN-major, N = H)
//               and dW += h^T [hi|lo] (A = the h tile MN-major, B = dZ MN-major),
//               accumulated in TMEM over every tile of the CTA
//   warps 4-7   the dh epilogue: TMEM -> bf16 -> 128-byte-swizzled staging -> TMA store
// The CTA's dW, db and loss sums go to workspace partials; after a grid barrier (the launch
// is cooperative) every CTA adds a slice of them over all CTAs in a fixed order
// (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "../../include/vtrace.h"
#include "vtrace_cb_host.h"

namespace vthf {
using namespace vtb200;

constexpr int TB = 8;            // trajectories per tile
constexpr int TT = 16;           // steps per tile
constexpr int BM = TB * TT;      // 128 rows: MMA M and TMEM lanes
#ifndef HF_ABLATE
#define HF_ABLATE 0   // A/B only: 1 = the V-trace epilogue's arithmetic compiled out (dZ = 0)
#endif
constexpr int MAX_NS = 4;        // h stages: as many as shared memory holds (2 at H = 256, 3 at 128)
constexpr int NWARPS = 11;
constexpr int THREADS = NWARPS * 32;
constexpr int W_PROD = 8, W_FWD = 9, W_BWD = 10;
constexpr uint32_t TM_Z = 0, TM_DH = 64, TM_DW = 320, TM_COLS = 512;
constexpr int NPART = 8;
constexpr int RSLOT = THREADS / 8;  // outputs per round of the final sum (8 groups of CTAs)
constexpr uint32_t SW128 = 2, SW64 = 4;  // tcgen05 smem descriptor layout types

struct HfArgs {
  int T, B, H, A, KB, nblk, nch, ns;
  const float* bias;  // [A+1] or null
  const float* boot;  // [B]
  float* w_part;      // [grid][A+1][H]
  double* db_part;    // [grid][32]
  double* l_part;     // [grid][8]
  unsigned* gbar;     // grid barrier {count, generation} (zero-initialised once)
  float* grad_w_t;    // [A+1][H]
  float* grad_b;      // [A+1]
  double* partials;   // [8]
  Params P;           // method parameters (thresholds, lambda, costs, reward mode, correction)
  // dynamic shared memory layout (bytes from the 1024-aligned base)
  uint32_t o_w, o_h, h_stage, o_sm, sm_stage, o_mu, o_a, o_r, o_g, o_dz, o_st;
  uint32_t tx_bytes;
};

struct HfMaps {
  CUtensorMap h, w, mu, a, r, g, dh;
};

// ---------------------------------------------------------------------------
// tcgen05 helpers

// shared-memory matrix descriptor: start, leading / stride byte offsets, version 1, layout
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)layout << 61);
}

// instruction descriptor, kind::f16: D fp32, A and B bf16, majors, N >> 3, M >> 4
__device__ __forceinline__ uint32_t idesc(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id,
                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(id), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes (lane i gets row i of its quarter)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// one level of the suffix scan over a 16-lane segment (lanes tl of one trajectory):
// (G, D) o (G', D') of the lane `o` steps later; lanes past the segment keep theirs
__device__ __forceinline__ void scan_level16(double& G, double& D, int o) {
  asm("{\n"
      ".reg .pred p;\n"
      ".reg .b32 g0, g1, d0, d1;\n"
      ".reg .f64 go, dd;\n"
      "mov.b64 {g0, g1}, %0;\n"
      "mov.b64 {d0, d1}, %1;\n"
      "shfl.sync.down.b32 g0|p, g0, %2, 0x100f, -1;\n"
      "shfl.sync.down.b32 g1, g1, %2, 0x100f, -1;\n"
      "shfl.sync.down.b32 d0, d0, %2, 0x100f, -1;\n"
      "shfl.sync.down.b32 d1, d1, %2, 0x100f, -1;\n"
      "mov.b64 go, {g0, g1};\n"
      "mov.b64 dd, {d0, d1};\n"
      "@p fma.rn.f64 %1, %0, dd, %1;\n"
      "@p mul.rn.f64 %0, %0, go;\n"
      "}\n"
      : "+d"(G), "+d"(D)
      : "r"(o));
}

#ifndef HF_WAIT
#define HF_WAIT 0   // 0: try_wait loop; 1: try_wait with a suspend-time hint (HF_HINT ns)
#endif
#ifndef HF_HINT
#define HF_HINT 2000
#endif
__device__ __forceinline__ void hf_wait(uint64_t* bar, uint32_t phase) {
#if HF_WAIT == 1
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITH_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITH_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"((uint32_t)HF_HINT)
      : "memory");
#else
  mbar_wait(bar, phase);
#endif
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h2 = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h2);
}

// Statistics of one behaviour row (fp32 logits in shared memory), the same operations as
// the column-block kernel's mu half: S_mu with its compensated low part, z^mu_a - m_mu.
template <int A_CT>
__device__ __forceinline__ double2 mu_stats(const float* mrow, int a) {
  constexpr int NP = (A_CT + 1) / 2;
  constexpr float CORR = 1.3349930e-08f;
  float2 zm[NP], em[NP], hm, lm, sdm, cwm;
  cb_load_pairs<float, A_CT>(mrow, zm);
  const float mm = row_max<NP>(zm);
  cb_exps<float, A_CT, false>(zm, mm, em, hm, lm, sdm, cwm);
  const float h0 = hm.x - 1.f, h1 = hm.y - 1.f;
  const float ss = h0 + h1;
  const float bb = ss - h0;
  const float err = (h0 - (ss - bb)) + (h1 - bb);
  const float sd = sdm.x + sdm.y;
  const float lo = fmaf(sd, CORR, err + (lm.x + lm.y));
  float zam = 0.f;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    zam = (2 * k == a) ? zm[k].x : zam;
    if (2 * k + 1 < A_CT) zam = (2 * k + 1 == a) ? zm[k].y : zam;
  }
  const bool finite = isfinite(sd) && isfinite(mm);
  const double S_m = finite ? (double)ss + (double)lo : __longlong_as_double(0x7ff8000000000000ll);
  return make_double2(S_m, (double)zam - (double)mm);
}

// ---------------------------------------------------------------------------
// The fused kernel

template <int A_CT>
__global__ void __launch_bounds__(THREADS, 1)
    head_fused_kernel(const HfArgs G, const __grid_constant__ HfMaps M) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  __shared__ __align__(8) uint64_t full[MAX_NS], sfree[MAX_NS], zfull[2], zempty[2];
  __shared__ __align__(8) uint64_t mufull[MAX_NS];
  // the behaviour rows' statistics of a stage (computed by the dh warps one tile ahead):
  // S_mu (NaN if the row is not finite) and z^mu_a - m_mu, per tile row
  __shared__ double2 mus[MAX_NS][BM];
  __shared__ __align__(8) uint64_t dzfull, dzempty, dhfull, dhempty, wbar;
  __shared__ uint32_t tmem_base;
  __shared__ double wpart[4][NPART];
  __shared__ double wdb[4][32];
  __shared__ float s_bias[32];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = G.T, B = G.B, A = A_CT, KB = G.KB, NS = G.ns;
  // this CTA's tiles: blocks blockIdx.x, +gridDim.x, ...; each block's chunks backwards
  const int my_blocks = G.nblk > (int)blockIdx.x ? (G.nblk - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int ntiles = my_blocks * G.nch;
  auto tile_of = [&](int j, int& b0, int& t0) {
    const int bi = j / G.nch, ci = G.nch - 1 - (j - bi * G.nch);
    b0 = ((int)blockIdx.x + bi * (int)gridDim.x) * TB;
    t0 = ci * TT;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {  // (NS = G.ns)
      mbar_init(&full[i], 1);
      mbar_init(&sfree[i], 1);
      mbar_init(&mufull[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&zfull[i], 1);
      mbar_init(&zempty[i], 4);
    }
    mbar_init(&dzfull, 4);
    mbar_init(&dzempty, 1);
    mbar_init(&dhfull, 1);
    mbar_init(&dhempty, 4);
    mbar_init(&wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) s_bias[threadIdx.x] = (G.bias && (int)threadIdx.x <= A) ? G.bias[threadIdx.x] : 0.f;
  if (warp == W_FWD) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t s_w = sbase + G.o_w;
  auto s_h = [&](int s) { return sbase + G.o_h + (uint32_t)s * G.h_stage; };
  auto s_sm = [&](int s) { return G.o_sm + (uint32_t)s * G.sm_stage; };  // offset
  const uint32_t s_dzhi = sbase + G.o_dz, s_dzlo = s_dzhi + BM * 64;

  if (warp == W_PROD) {
    // ---------------- producer ----------------
    if (lane == 0 && ntiles > 0) {
      mbar_expect_tx(&wbar, (uint32_t)KB * 4096u);
      for (int q = 0; q < KB; ++q) tma_load_2d(smem + G.o_w + q * 4096, &M.w, q * 64, 0, &wbar);
      for (int j = 0; j < ntiles; ++j) {
        const int s = j % NS;
        if (j >= NS) hf_wait(&sfree[s], (uint32_t)((j / NS) - 1) & 1u);
        int b0, t0;
        tile_of(j, b0, t0);
        mbar_expect_tx(&full[s], G.tx_bytes);
        uint8_t* hs = smem + G.o_h + s * G.h_stage;
        for (int q = 0; q < KB; ++q) tma_load_3d(hs + q * 16384, &M.h, q * 64, t0, b0, &full[s]);
        uint8_t* sm = smem + s_sm(s);
        tma_load_3d(sm + G.o_mu, &M.mu, 0, t0, b0 / 4, &full[s]);
        tma_load_2d(sm + G.o_a, &M.a, b0, t0, &full[s]);
        tma_load_2d(sm + G.o_r, &M.r, b0, t0, &full[s]);
        tma_load_2d(sm + G.o_g, &M.g, b0, t0, &full[s]);
      }
    }
  } else if (warp == W_FWD) {
    // ---------------- forward MMA: z = h W^T ----------------
    if (lane == 0 && ntiles > 0) {
      hf_wait(&wbar, 0);
      const uint32_t id = idesc(BM, 32, false, false);
      for (int j = 0; j < ntiles; ++j) {
        const int s = j % NS, zb = j & 1;
        hf_wait(&full[s], (uint32_t)(j / NS) & 1u);
        if (j >= 2) hf_wait(&zempty[zb], (uint32_t)((j >> 1) - 1) & 1u);
        tc_fence_after();
        const uint32_t hb = s_h(s);
        for (int k = 0; k < KB * 4; ++k) {  // K = 16 per MMA: +32 B inside a 128-byte row
          const uint64_t da = sdesc(hb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, SW128);
          const uint64_t db = sdesc(s_w + (k >> 2) * 4096 + (k & 3) * 32, 16, 1024, SW128);
          umma(tmem + TM_Z + zb * 32, da, db, id, k > 0 ? 1u : 0u);
        }
        umma_commit(smem_u32(&zfull[zb]));
      }
    }
  } else if (warp == W_BWD) {
    // ---------------- backward MMAs: dh = dZ W, dW += h^T dZ ----------------
    if (lane == 0 && ntiles > 0) {
      hf_wait(&wbar, 0);
      const uint32_t id_dh = idesc(BM, G.H, false, true);
      const uint32_t id_dw = idesc(128, 32, true, true);
      for (int j = 0; j < ntiles; ++j) {
        const int s = j % NS;
        hf_wait(&dzfull, (uint32_t)j & 1u);
        tc_fence_after();
        // dW [H x 32] += h^T [H x 128] dZ [128 x 32], per 128-row half of H; A: the h tile
        // as MN-major (K = tile row, 8-row groups 1024 B apart, K = 16 -> +2048 B; M = h in
        // 64-element atoms 16384 B apart); B: dZ as MN-major (N = head column in one
        // 64-byte atom, 8-row groups 512 B apart, K = 16 -> +1024 B).  First: it is the last
        // reader of the h stage, which goes back to the producer at once.
        const uint32_t hb = s_h(s);
        for (int half = 0; half < KB / 2; ++half) {
          for (int p = 0; p < 2; ++p) {
            const uint32_t dz = p ? s_dzlo : s_dzhi;
            for (int k = 0; k < BM / 16; ++k) {
              const uint64_t da = sdesc(hb + half * 32768 + k * 2048, 16384, 1024, SW128);
              const uint64_t db = sdesc(dz + k * 1024, 64, 512, SW64);
              umma(tmem + TM_DW + half * 32, da, db, id_dw, (j | p | k) ? 1u : 0u);
            }
          }
        }
        umma_commit(smem_u32(&sfree[s]));
        // dh [128 x H] = dZ [128 x 32] W [32 x H], once the dh warps have read the previous
        // tile's; A: dZ rows of 64 B (K-major, 64-byte swizzle, 8-row groups 512 B apart,
        // K = 16 -> +32 B); B: the W^T tile as MN-major (K = head column j = its 128-byte
        // rows, 8-row groups 1024 B apart, K = 16 -> +2048 B; N = h in 64-element atoms 4096 B
        // apart)
        if (j >= 1) {
          hf_wait(&dhempty, (uint32_t)(j - 1) & 1u);
          tc_fence_after();
        }
        for (int p = 0; p < 2; ++p) {
          const uint32_t dz = p ? s_dzlo : s_dzhi;
          for (int k = 0; k < 2; ++k) {
            const uint64_t da = sdesc(dz + k * 32, 16, 512, SW64);
            const uint64_t db = sdesc(s_w + k * 2048, 4096, 1024, SW128);
            umma(tmem + TM_DH, da, db, id_dh, (p | k) ? 1u : 0u);
          }
        }
        umma_commit(smem_u32(&dhfull));
        umma_commit(smem_u32(&dzempty));
      }
    }
  } else if (warp >= 4) {
    // ---------------- dh epilogue (warps 4-7) ----------------
    const int q4 = warp - 4;
    const int r = q4 * 32 + lane;  // tile row = TMEM lane
    const bool leader = (q4 == 0 && lane == 0);
    int nst = 0;  // stores issued (staging buffer = nst & 1)
    const int c = lane >> 4, tl = lane & 15, bl = 2 * q4 + c;  // the V-trace warps' row map
    for (int jj = 0; jj <= ntiles; ++jj) {
      if (jj < ntiles) {  // the behaviour statistics of tile jj, ahead of its V-trace warps
        const int s = jj % NS;
        hf_wait(&full[s], (uint32_t)(jj / NS) & 1u);
        const uint8_t* sm = smem + s_sm(s);
        const float* mrow = reinterpret_cast<const float*>(sm + G.o_mu) +
                            (((bl >> 2) * TT + tl) * 4 + (bl & 3)) * A_CT;
        const int a = min(max(reinterpret_cast<const int*>(sm + G.o_a)[tl * TB + bl], 0), A - 1);
#if HF_ABLATE == 3
        mus[s][r] = make_double2(1.0, 0.0);
        (void)mrow;
        (void)a;
#else
        mus[s][r] = mu_stats<A_CT>(mrow, a);
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(&mufull[s]);
      }
      if (jj == 0) continue;
      const int j = jj - 1;  // the dh epilogue of the previous tile
      int b0, t0;
      tile_of(j, b0, t0);
      hf_wait(&dhfull, (uint32_t)j & 1u);
      tc_fence_after();
      for (int q = 0; q < KB; ++q, ++nst) {
        uint32_t v0[32], v1[32];
        tmem_ld32(tmem + TM_DH + q * 64 + ((uint32_t)(q4 * 32) << 16), v0);
        tmem_ld32(tmem + TM_DH + q * 64 + 32 + ((uint32_t)(q4 * 32) << 16), v1);
        tmem_wait_ld();
        if (q == KB - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dhempty);
        }
#if HF_ABLATE == 2
        continue;  // A/B only: no dh output
#endif
        // the staging buffer's previous store (two atoms ago) must have read it
        if (leader) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        named_bar(1, 128);
        uint8_t* st = smem + G.o_st + (nst & 1) * 16384 + r * 128;
#pragma unroll
        for (int cch = 0; cch < 8; ++cch) {  // 16-byte chunk cch of the row, swizzled
          const uint32_t* src = cch < 4 ? &v0[cch * 8] : &v1[(cch - 4) * 8];
          uint4 w;
          w.x = pack_bf16(__uint_as_float(src[0]), __uint_as_float(src[1]));
          w.y = pack_bf16(__uint_as_float(src[2]), __uint_as_float(src[3]));
          w.z = pack_bf16(__uint_as_float(src[4]), __uint_as_float(src[5]));
          w.w = pack_bf16(__uint_as_float(src[6]), __uint_as_float(src[7]));
          *reinterpret_cast<uint4*>(st + ((cch ^ (r & 7)) << 4)) = w;
        }
        fence_proxy_async_smem();
        named_bar(1, 128);
        if (leader) {
          tma_store_3d(&M.dh, q * 64, t0, b0, smem + G.o_st + (nst & 1) * 16384);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    // the CTA's dW partial, after the last tile's backward MMAs: TMEM lane = h row
    if (ntiles > 0) {
      hf_wait(&dzempty, (uint32_t)(ntiles - 1) & 1u);
      tc_fence_after();
      for (int half = 0; half < KB / 2; ++half) {
        uint32_t v[32];
        tmem_ld32(tmem + TM_DW + half * 32 + ((uint32_t)(q4 * 32) << 16), v);
        tmem_wait_ld();
        const int hh = half * 128 + q4 * 32 + lane;
        float* wp = G.w_part + (size_t)blockIdx.x * (A + 1) * G.H;
#pragma unroll
        for (int n = 0; n <= A_CT; ++n) wp[(size_t)n * G.H + hh] = __uint_as_float(v[n]);
      }
    } else {
      float* wp = G.w_part + (size_t)blockIdx.x * (A + 1) * G.H;
      for (int i = threadIdx.x - 128; i < (A + 1) * G.H; i += 128) wp[i] = 0.f;
    }
    if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else {
    // ---------------- V-trace epilogue (warps 0-3) ----------------
    const int c = lane >> 4, tl = lane & 15;
    const int bl = 2 * warp + c;  // trajectory within the tile
    const int r = warp * 32 + lane;
    const Params& P = G.P;
    const float ce = (float)P.c_e, cv = (float)P.c_v;
    constexpr int NP = (A_CT + 1) / 2;
    constexpr float L32 = 1.44269502f;
    constexpr float CORR = 1.3349930e-08f;
    double carry = 0.0;   // A just after this chunk (A_T = 0)
    float vnext = 0.f;    // V(x) of the step after this chunk
    CbAcc acc = {0.0, 0.0, 0.0, 0.0, 0.0, 0u};
    double db_acc = 0.0;  // lane n: sum of column n of dZ
    float dsum[A_CT + 1];
#pragma unroll
    for (int k = 0; k <= A_CT; ++k) dsum[k] = 0.f;
    float bz[A_CT + 1];
#pragma unroll
    for (int k = 0; k <= A_CT; ++k) bz[k] = s_bias[k];
    for (int j = 0; j < ntiles; ++j) {
      const int s = j % NS, zb = j & 1;
      int b0, t0;
      tile_of(j, b0, t0);
      const int b = b0 + bl, t = t0 + tl;
      const bool row_ok = b < B && t < T;
      if (t0 + TT >= T) carry = 0.0;  // a new block starts at its last chunk
      hf_wait(&zfull[zb], (uint32_t)(j >> 1) & 1u);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(tmem + TM_Z + zb * 32 + ((uint32_t)(warp * 32) << 16), v);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&zempty[zb]);
      hf_wait(&full[s], (uint32_t)(j / NS) & 1u);  // the small tiles of this stage
      const uint8_t* sm = smem + s_sm(s);
#if HF_ABLATE == 1
      if (true) {
        if (j >= 1) hf_wait(&dzempty, (uint32_t)(j - 1) & 1u);
        uint8_t* hi = smem + G.o_dz + r * 64;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          *reinterpret_cast<uint4*>(hi + q * 16) = make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(hi + BM * 64 + q * 16) = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dzfull);
        continue;
      }
#endif
      // z^pi and V of this row (+ bias)
      CbRow<float, A_CT> R;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const float x0 = __uint_as_float(v[2 * k]) + bz[2 * k];
        const float x1 = (2 * k + 1 < A_CT) ? __uint_as_float(v[2 * k + 1]) + bz[2 * k + 1] : -INFINITY;
        R.z[k] = make_float2(x0, x1);
      }
      const float Vt = __uint_as_float(v[A_CT]) + bz[A_CT];
      const int a_raw = reinterpret_cast<const int*>(sm + G.o_a)[tl * TB + bl];
      const float rt = reinterpret_cast<const float*>(sm + G.o_r)[tl * TB + bl];
      const float gm = reinterpret_cast<const float*>(sm + G.o_g)[tl * TB + bl];
      const int a = min(max(a_raw, 0), A - 1);
      // V(x_{t+1}): the next lane of the segment; past the chunk: the later chunk's first
      // step; at t = T - 1: the bootstrap value
      float Vn = __shfl_down_sync(0xffffffffu, Vt, 1, 16);
      if (tl == TT - 1) Vn = vnext;
      if (t + 1 == T) Vn = (b < B) ? __ldg(G.boot + b) : 0.f;
      // a3-a7: statistics of the target row (as the column-block kernel, fp32 logits); the
      // behaviour row's come from the dh warps (same operations, one tile ahead)
      const float mp = row_max<NP>(R.z);
      float2 hp, lp, sdp, cwp;
      cb_exps<float, A_CT, true>(R.z, mp, R.e, hp, lp, sdp, cwp);
      const float h0 = hp.x - 1.f, h1 = hp.y - 1.f;
      const float ss0 = h0 + h1;
      const float bb = ss0 - h0;
      const float err = (h0 - (ss0 - bb)) + (h1 - bb);
      const float sd0 = sdp.x + sdp.y;
      const float lo0 = fmaf(sd0, CORR, err + (lp.x + lp.y));
      const float2 ss = make_float2(ss0, 0.f), lo = make_float2(lo0, 0.f), sd = make_float2(sd0, 0.f);
      const double S_p = (double)ss0 + (double)lo0;
      float zap = 0.f;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        zap = (2 * k == a) ? R.z[k].x : zap;
        if (2 * k + 1 < A_CT) zap = (2 * k + 1 == a) ? R.z[k].y : zap;
      }
      hf_wait(&mufull[s], (uint32_t)(j / NS) & 1u);
      const double2 mst = mus[s][r];
      const double S_m = mst.x, xa_m = mst.y;
      const double xa_p = (double)zap - (double)mp;
      const float ea_raw = ex2_approx((zap - mp) * L32);
      const bool finite = isfinite(sd0) && isfinite(mp) && isfinite(S_m);
      // a5, a7: pi(a)/mu(a) = exp((z^pi_a - m_pi) - (z^mu_a - m_mu)) S_mu / S_pi
      const double ratio = exp64(xa_p - xa_m) * ddiv_pos(S_m, S_p);
      const double td = reward_transform(rt, P.reward_mode) + (double)gm * (double)Vn - (double)Vt;
      const StepWeights sw = step_weights<true>(P, ratio);
      const float Sf = ss.x + lo.x;
      const float inv_S = rcp_approx(Sf);
      const float lse = mp + __logf(Sf);
      const float cshift = fmaf(sd.x, inv_S, mp);  // lse - H
      const float ea_c = fmaf(ea_raw * CORR, zap - mp, ea_raw);
      const float rest = ((ss.x - ea_c) + lo.x) * inv_S;  // 1 - pi(a)
      const float pa = ea_c * inv_S;
      // a8: the 16-step suffix scan of (gamma_t c_t, delta_t V), then the carry
      double Gi = row_ok ? (double)gm * sw.c : 1.0;
      double Di = row_ok ? sw.rho * td : 0.0;
#pragma unroll
      for (int o = 1; o < TT; o <<= 1) scan_level16(Gi, Di, o);
      const double A_t = fma(Gi, carry, Di);  // v_t - V(x_t)
      double A_n = __shfl_down_sync(0xffffffffu, A_t, 1, 16);
      if (tl == TT - 1) A_n = carry;
      carry = __shfl_sync(0xffffffffu, A_t, c * 16);   // A at the chunk's first step
      vnext = __shfl_sync(0xffffffffu, Vt, c * 16);    // V at the chunk's first step
      // pg_adv = rho_pg (r + gamma v_{t+1} - V) (App. E.3 q variant)
      const double pgd = sw.rho_pg * (P.q_values ? td : fma((double)gm, A_n, td));
      float pge = (float)pgd, logpa = zap - lse;
      if (P.correction == VT_CORRECTION_EPSILON) {  // P:412, readings c11, r7
        const float rr = P.eps / pa;
        logpa = pa > 0.f ? logpa + log1pf(rr) : logf(P.eps);
        pge = pge / (1.f + rr);
      }
      // a11: dz_j = e_j / S (alpha + c_e z_j) (j != a), dz_a; dV = c_v (V - v)
      const float alpha = fmaf(-ce, cshift, pge);
      const float2 k1 = f2(ce * inv_S), k0 = f2(alpha * inv_S);
      float d[32];
      float2 sq2 = f2(0.f);
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const float2 d2 = __fmul2_rn(R.e[k], __ffma2_rn(k1, R.z[k], k0));
        d[2 * k] = d2.x;
        if (2 * k + 1 < A_CT) {
          d[2 * k + 1] = d2.y;
          sq2 = __ffma2_rn(d2, d2, sq2);
        } else {
          sq2.x = fmaf(d2.x, d2.x, sq2.x);
        }
      }
      const float d_wrong = ea_raw * fmaf(k1.x, zap, k0.x);
      const float d_a = fmaf(-pge, rest, ce * (1.f - rest) * (zap - cshift));
#pragma unroll
      for (int k = 0; k < A_CT; ++k) d[k] = (k == a) ? d_a : d[k];
      const float sq = fmaf(d_a, d_a, fmaf(-d_wrong, d_wrong, sq2.x + sq2.y));
      d[A_CT] = (float)(-(double)cv * A_t);
#pragma unroll
      for (int k = A_CT + 1; k < 32; ++k) d[k] = 0.f;
      if (!row_ok) {
#pragma unroll
        for (int k = 0; k < 32; ++k) d[k] = 0.f;
      } else {
        acc.rho += sw.rho;
        if (P.correction == VT_CORRECTION_VTRACE && ratio > P.rho_bar) ++acc.clip;
        acc.H += (double)(lse - cshift);
        acc.pg = fma(-pgd, (double)logpa, acc.pg);
        acc.v2 = fma(A_t, A_t, acc.v2);
        acc.dz += (double)sq;
        const bool bad = (a_raw != a) || !finite || !isfinite(rt) || !isfinite(Vt) ||
                         !(gm >= 0.f && gm <= 1.f);
        if (bad && P.ws) {
          const long long row = (long long)t * B + b;
          if (a_raw != a) record_bad(P.ws, row, VT_DATA_ACTION);
          if (!finite) record_bad(P.ws, row, VT_DATA_LOGITS);
          if (!isfinite(rt)) record_bad(P.ws, row, VT_DATA_REWARD);
          if (!isfinite(Vt)) record_bad(P.ws, row, VT_DATA_VALUE);
          if (!(gm >= 0.f && gm <= 1.f)) record_bad(P.ws, row, VT_DATA_DISCOUNT);
        }
      }
      // dZ as bf16 hi + lo (K-major rows of 64 B, 64-byte swizzle: 16-byte chunk q of row
      // r at q ^ ((r >> 1) & 3)); the previous tile's backward MMAs must be done with it
      if (j >= 1) hf_wait(&dzempty, (uint32_t)(j - 1) & 1u);
      {
        uint8_t* hi = smem + G.o_dz + r * 64;
        uint8_t* lo2 = hi + BM * 64;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t wh[4], wl[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x0 = d[q * 8 + 2 * e], x1 = d[q * 8 + 2 * e + 1];
            const uint32_t ph = pack_bf16(x0, x1);
            const float r0 = x0 - __uint_as_float(ph << 16);
            const float r1 = x1 - __uint_as_float(ph & 0xffff0000u);
            wh[e] = ph;
            wl[e] = pack_bf16(r0, r1);
          }
          const int pq = (q ^ ((r >> 1) & 3)) << 4;
          *reinterpret_cast<uint4*>(hi + pq) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
          *reinterpret_cast<uint4*>(lo2 + pq) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dzfull);
      // db: this lane's running column sums (fp32 over the ~50 tiles of a lane)
#pragma unroll
      for (int k = 0; k <= A_CT; ++k) dsum[k] += d[k];
    }
    // db: butterfly over the lanes, lane n ends with column n's sum of the warp's rows
    {
      float d[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) d[k] = k <= A_CT ? dsum[k] : 0.f;
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) {
        const bool up = (lane & w) != 0;
#pragma unroll
        for (int k = 0; k < w; ++k) {
          const float send = up ? d[k] : d[k + w];
          const float keep = up ? d[k + w] : d[k];
          d[k] = keep + __shfl_xor_sync(0xffffffffu, send, w);
        }
      }
      db_acc = (double)d[0];
    }
    // a12: per-lane sums -> warp
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
    wdb[warp][lane] = db_acc;
  }
  __syncwarp();  // (the single-lane roles reconverge before the CTA barrier)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < NPART) {
    double x = 0.0;
    for (int w = 0; w < 4; ++w) x += wpart[w][threadIdx.x];
    G.l_part[(size_t)blockIdx.x * NPART + threadIdx.x] = x;
  } else if (threadIdx.x >= 32 && threadIdx.x < 64) {
    const int n = threadIdx.x - 32;
    double x = 0.0;
    for (int w = 0; w < 4; ++w) x += wdb[w][n];
    G.db_part[(size_t)blockIdx.x * 32 + n] = x;
  }
  if (warp == W_FWD)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TM_COLS));

  // ---- the sum of the CTAs' partials: a grid barrier (cooperative launch: every CTA is
  // resident), then each CTA adds a slice of the outputs over all CTAs in a fixed order ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire_u32(&G.gbar[1]);
    if (atomicAdd(&G.gbar[0], 1u) == gridDim.x - 1) {
      G.gbar[0] = 0u;
      __threadfence();
      st_release_u32(&G.gbar[1], gen + 1u);
    } else {
      while (ld_acquire_u32(&G.gbar[1]) == gen) __nanosleep(32);
    }
  }
  __syncthreads();
  // (the group sums reuse the behaviour-statistics buffer, idle by now)
  static_assert(sizeof(double) * 8 * RSLOT <= sizeof(double2) * MAX_NS * BM, "racc fits in mus");
  double (*racc)[RSLOT] = reinterpret_cast<double (*)[RSLOT]>(&mus[0][0]);
  const int ncta = gridDim.x, A1 = A + 1, nw = A1 * G.H, nwb = nw + A1;
  const int chunk = (nwb + ncta - 1) / ncta;
  const int o_end = min((int)blockIdx.x * chunk + chunk, nwb);
  const int grp = threadIdx.x / RSLOT, slot = threadIdx.x - grp * RSLOT;
  auto csum = [&](auto load) {  // CTAs grp, grp + 8, ... (four loads in flight), in order
    double x = 0.0;
    for (int c = grp; c < ncta; c += 32) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (c + 8 * u < ncta) ? load(c + 8 * u) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) x += v[u];
    }
    return x;
  };
  for (int base = (int)blockIdx.x * chunk; base < o_end; base += RSLOT) {
    const int n = min(RSLOT, o_end - base), i = base + slot;
    double x = 0.0;
    if (grp < 8 && slot < n) {
      if (i < nw) x = csum([&](int c) { return (double)__ldcg(G.w_part + (size_t)c * nw + i); });
      else x = csum([&](int c) { return __ldcg(G.db_part + (size_t)c * 32 + (i - nw)); });
    }
    if (grp < 8) racc[grp][slot] = x;
    __syncthreads();
    if (threadIdx.x < n) {
      double y = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) y += racc[q][threadIdx.x];
      const int o = base + threadIdx.x;
      if (o < nw) G.grad_w_t[o] = (float)y;
      else G.grad_b[o - nw] = (float)y;
    }
    __syncthreads();
  }
  if (blockIdx.x == gridDim.x - 1) {  // the 8 loss partials (and their total)
    double x = 0.0;
    if (grp < 8 && slot < NPART)
      x = csum([&](int c) { return __ldcg(G.l_part + (size_t)c * NPART + slot); });
    if (grp < 8) racc[grp][slot] = x;
    __syncthreads();
    if (warp == 0) {
      double y = 0.0;
      if (lane < NPART)
        for (int q = 0; q < 8; ++q) y += racc[q][lane];
      const double pg = __shfl_sync(0xffffffffu, y, VT_P_PG_LOSS);
      const double bl = __shfl_sync(0xffffffffu, y, VT_P_BASELINE_LOSS);
      const double en = __shfl_sync(0xffffffffu, y, VT_P_ENTROPY_SUM);
      if (lane == VT_P_TOTAL_LOSS) y = pg + G.P.c_v * bl - G.P.c_e * en;
      if (lane < NPART) G.partials[lane] = y;
    }
  }
}

// ---------------------------------------------------------------------------
// host side

std::mutex g_mu;
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
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

struct Layout {
  uint32_t o_w, o_h, h_stage, o_sm, sm_stage, o_mu, o_a, o_r, o_g, o_dz, o_st, tx, smem;
};

Layout layout(int H, int A, int NS) {
  Layout L{};
  const int KB = H / 64;
  auto up = [](uint32_t x, uint32_t a) { return (x + a - 1) / a * a; };
  L.o_w = 0;
  L.o_h = up(L.o_w + KB * 4096, 1024);
  L.h_stage = KB * 16384;
  L.o_sm = L.o_h + NS * L.h_stage;
  L.o_mu = 0;
  L.o_a = up(L.o_mu + TT * TB * A * 4, 128);
  L.o_r = L.o_a + TT * TB * 4;
  L.o_g = L.o_r + TT * TB * 4;
  L.sm_stage = up(L.o_g + TT * TB * 4, 1024);
  L.o_dz = L.o_sm + NS * L.sm_stage;  // 1024-aligned (the 64-byte swizzle needs 512)
  L.o_st = L.o_dz + 2 * BM * 64;
  L.smem = L.o_st + 2 * 16384 + 1024;  // + alignment slack
  L.tx = KB * 16384 + TT * TB * A * 4 + 3 * TT * TB * 4;
  return L;
}

template <int A_CT>
vt_status launch(const HfArgs& G, const HfMaps& M, int grid, size_t smem, cudaStream_t st) {
  auto kern = head_fused_kernel<A_CT>;
  static std::atomic<unsigned long long> attr_set{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_set.load() & bit)) {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return VT_ERR_CUDA;
    const int dyn_max = 232448 - (int)fa.sharedSizeBytes;  // 227 KB per CTA, static included
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max) !=
        cudaSuccess)
      return VT_ERR_CUDA;
    attr_set.fetch_or(bit);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // the final sum's grid barrier
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, G, M) == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}

bool encode(CUtensorMap* m, CUtensorMapDataType dt, int rank, void* base, const cuuint64_t* dims,
            const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle sw) {
  cuuint32_t es[3] = {1, 1, 1};
  return encoder()(m, dt, rank, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

}  // namespace vthf

extern "C" size_t vtrace_head_workspace_bytes(int64_t T, int64_t B, int32_t H, int32_t A) {
  if (T <= 0 || B <= 0 || H <= 0 || A < 1 || A + 1 > 32) return 0;
  const size_t grid = 256;  // upper bound on the persistent grid (SMs per device)
  return 256 + grid * ((size_t)(A + 1) * H * 4 + 32 * 8 + vthf::NPART * 8) + 256;
}

extern "C" vt_status vtrace_head_loss_and_grad(
    int64_t T, int64_t B, int32_t H, int32_t A, const void* hidden, const void* w_t,
    const float* bias, const float* behaviour_logits, const int32_t* actions,
    const float* discounts, const float* rewards, const float* bootstrap_value,
    const vt_vtrace_params* params, const vt_loss_weights* weights, void* grad_hidden,
    float* grad_w_t, float* grad_bias, double* partials, void* workspace,
    size_t workspace_bytes, vt_stream_t stream) {
  using namespace vthf;
  if (!hidden || !w_t || !behaviour_logits || !actions || !discounts || !rewards ||
      !bootstrap_value || !weights || !grad_hidden || !grad_w_t || !grad_bias || !partials)
    return VT_ERR_INVALID_ARG;
  if (T <= 0 || B <= 0 || T > (1 << 24) || B > (1 << 24) || T * B > (1LL << 31)) return VT_ERR_SHAPE;
  if (!(H == 128 || H == 256)) return VT_ERR_SHAPE;
  if (!(A == 3 || A == 4 || A == 6 || A == 9 || A == 18)) return VT_ERR_SHAPE;
  if (B % 4 != 0) return VT_ERR_SHAPE;  // behaviour-logit boxes of 4 trajectories (16-byte rows)
  vt_status s = check_params(params);
  if (s) return s;
  if (params->behaviour_log_probs) return VT_ERR_PARAM;
  if (!std::isfinite(weights->baseline_cost) || !std::isfinite(weights->entropy_cost))
    return VT_ERR_PARAM;
  auto al = [](const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; };
  if (!al(hidden, 16) || !al(w_t, 16) || !al(grad_hidden, 16) || !al(behaviour_logits, 16) ||
      !al(actions, 16) || !al(discounts, 16) || !al(rewards, 16) || !al(bootstrap_value, 4) ||
      !al(grad_w_t, 4) || !al(grad_bias, 4) || !al(partials, 8) || (bias && !al(bias, 4)))
    return VT_ERR_ALIGNMENT;
  if (!workspace || !al(workspace, 256) ||
      workspace_bytes < vtrace_head_workspace_bytes(T, B, H, A))
    return VT_ERR_WORKSPACE;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return VT_ERR_CUDA;
  sms = cb_num_sms(dev);
  if (sms <= 0) return VT_ERR_CUDA;
  {
    int maj = 0, mnr = 0;
    if (cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
      return VT_ERR_CUDA;
    if (maj != 10 || mnr != 0) return VT_ERR_DEVICE;
  }
  if (!encoder()) return VT_ERR_CUDA;

  // as many h stages as the 227 KB of shared memory hold (the ring depth is what hides the
  // load latency behind the epilogue: H = 128 runs 3 stages, H = 256 2)
  constexpr uint32_t kDynMax = 232448 - 12 * 1024;  // 227 KB per CTA minus the static arrays
  int ns = MAX_NS;
  while (ns > 2 && layout(H, A, ns).smem > kDynMax) --ns;
  const Layout L = layout(H, A, ns);
  if (L.smem > kDynMax) return VT_ERR_SHAPE;
  HfArgs G;
  std::memset(&G, 0, sizeof(G));
  G.T = (int)T;
  G.B = (int)B;
  G.H = H;
  G.A = A;
  G.KB = H / 64;
  G.nblk = (int)((B + TB - 1) / TB);
  G.nch = (int)((T + TT - 1) / TT);
  G.ns = ns;
  const int grid = std::min(std::min(sms, 256), G.nblk);
  G.bias = bias;
  G.boot = bootstrap_value;
  uint8_t* wsb = static_cast<uint8_t*>(workspace);
  G.gbar = reinterpret_cast<unsigned*>(wsb);
  G.w_part = reinterpret_cast<float*>(wsb + 256);
  G.db_part = reinterpret_cast<double*>(wsb + 256 + (size_t)256 * (A + 1) * H * 4);
  G.l_part = G.db_part + (size_t)256 * 32;
  G.grad_w_t = grad_w_t;
  G.grad_b = grad_bias;
  G.partials = partials;
  Params& P = G.P;
  P.T = T; P.B = B; P.A = A; P.T32 = (int)T; P.B32 = (int)B;
  P.rho_bar = (double)params->clip_rho_threshold;
  P.c_bar = (double)params->clip_c_threshold;
  P.pg_rho_bar = (double)params->clip_pg_rho_threshold;
  P.lambda = (double)params->lambda_;
  P.reward_mode = params->reward_mode;
  P.correction = params->correction;
  P.q_values = params->q_from_values;
  P.eps = params->epsilon;
  P.c_v = (double)weights->baseline_cost;
  P.c_e = (double)weights->entropy_cost;
  P.ws = nullptr;
  G.o_w = L.o_w; G.o_h = L.o_h; G.h_stage = L.h_stage; G.o_sm = L.o_sm; G.sm_stage = L.sm_stage;
  G.o_mu = L.o_mu; G.o_a = L.o_a; G.o_r = L.o_r; G.o_g = L.o_g; G.o_dz = L.o_dz; G.o_st = L.o_st;
  G.tx_bytes = L.tx;

  HfMaps M;
  std::memset(&M, 0, sizeof(M));
  void* hp = const_cast<void*>(hidden);
  {  // h [T][B][H] bf16 as (h, t, b): box 64 x 16 x 8 -> rows r = 16 b + t, 128-byte swizzle
    cuuint64_t d[3] = {(cuuint64_t)H, (cuuint64_t)T, (cuuint64_t)B};
    cuuint64_t st[2] = {(cuuint64_t)B * H * 2, (cuuint64_t)H * 2};
    cuuint32_t bx[3] = {64, TT, TB};
    if (!encode(&M.h, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, hp, d, st, bx, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode(&M.dh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, grad_hidden, d, st, bx,
                CU_TENSOR_MAP_SWIZZLE_128B))
      return VT_ERR_CUDA;
  }
  {  // W^T [A+1][H] bf16: box 64 x 32 (rows past A+1 zero-filled)
    cuuint64_t d[2] = {(cuuint64_t)H, (cuuint64_t)(A + 1)};
    cuuint64_t st[1] = {(cuuint64_t)H * 2};
    cuuint32_t bx[2] = {64, 32};
    if (!encode(&M.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w_t), d, st, bx,
                CU_TENSOR_MAP_SWIZZLE_128B))
      return VT_ERR_CUDA;
  }
  {  // behaviour logits [T][B][A] fp32 as (4A within a 4-trajectory group, t, group)
    cuuint64_t d[3] = {(cuuint64_t)4 * A, (cuuint64_t)T, (cuuint64_t)(B / 4)};
    cuuint64_t st[2] = {(cuuint64_t)B * A * 4, (cuuint64_t)4 * A * 4};
    cuuint32_t bx[3] = {(cuuint32_t)(4 * A), TT, TB / 4};
    if (!encode(&M.mu, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(behaviour_logits), d,
                st, bx, CU_TENSOR_MAP_SWIZZLE_NONE))
      return VT_ERR_CUDA;
  }
  {  // a, r, gamma [T][B]: box 8 x 16
    cuuint64_t d[2] = {(cuuint64_t)B, (cuuint64_t)T};
    cuuint64_t st[1] = {(cuuint64_t)B * 4};
    cuuint32_t bx[2] = {TB, TT};
    if (!encode(&M.a, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<int32_t*>(actions), d, st, bx,
                CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode(&M.r, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(rewards), d, st, bx,
                CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode(&M.g, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(discounts), d, st, bx,
                CU_TENSOR_MAP_SWIZZLE_NONE))
      return VT_ERR_CUDA;
  }
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  switch (A) {
    case 3: s = launch<3>(G, M, grid, L.smem, cs); break;
    case 4: s = launch<4>(G, M, grid, L.smem, cs); break;
    case 6: s = launch<6>(G, M, grid, L.smem, cs); break;
    case 9: s = launch<9>(G, M, grid, L.smem, cs); break;
    default: s = launch<18>(G, M, grid, L.smem, cs); break;
  }
  return s;
}
