// NEXT #3, first half: the learner's output layer over all T*B folded
// steps (Fig. 3), [z^pi | V] = h W + b, on the 5th-generation tensor cores.
// See include/vtrace.h (vtrace_output_layer) and DESIGN.md §9b / reading r12.
//
// Persistent kernel, one CTA (8 warps) per SM.  A tile is 128 rows of h: H/64 TMA boxes of
// 64 k x 128 rows land in shared memory in the 128-byte-swizzled K-major layout, in an
// NBUF-deep ring filled by one thread (mbarrier transaction counts).  The same thread
// issues H/16 tcgen05.mma (M = 128, N = 32, K = 16, bf16 in, fp32 accumulate) into 32
// TMEM columns and commits to an mbarrier; warps 0-3 read the accumulator back
// (tcgen05.ld 32x32b: lane = row), add the bias and stage the rows in shared memory, and
// all 8 warps write the [128, A] logits block and the 128 values with coalesced stores.
// The GEMM is HBM-bound (K = 256, N = 19: ~19 flop per byte of h), so the ring keeps the
// loads of the next NBUF-1 tiles in flight while one tile is multiplied and stored.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "../../include/vtrace.h"

namespace vtol {

constexpr int BM = 128;        // rows per tile (MMA M)
constexpr int BN = 32;         // output columns per MMA (A + 1 <= 32)
constexpr int THREADS = 256;
constexpr int SMEM_LIMIT = 232448;
constexpr int SO_LD = BN + 1;   // row stride (floats) of the epilogue staging tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// tcgen05 shared-memory descriptor, K-major, SWIZZLE_128B: start address, SBO = 1024 B
// (8 rows x 128 B), LBO unused (1), version 1 (bit 46), layout type 2 (bits 61-63).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
               "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                      uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}

// KB = H / 64 swizzle atoms per row; NBUF ring depth
template <int KB, int NBUF>
#ifdef OL_NO_MINBLOCKS  // A/B only
__global__ void __launch_bounds__(THREADS)
#else
__global__ void __launch_bounds__(THREADS, 1)
#endif
output_layer_kernel(const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap wmap,
                    const float* __restrict__ bias, float* __restrict__ z_out,
                    float* __restrict__ v_out, int M, int A) {
  constexpr uint32_t STAGE = KB * 16384;  // 128 rows x 64 k x 2 B per atom
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the swizzled atoms, derived from smem_raw so the compiler
  // keeps the shared state space (STS/LDS, not generic stores) for the staging below
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sw = smem_u32(smem);               // W^T: KB atoms of 32 rows x 128 B
  const uint32_t sa0 = sw + KB * 4096;              // NBUF stages
  float* so = reinterpret_cast<float*>(smem + KB * 4096 + NBUF * STAGE);  // [128][SO_LD]
  __shared__ uint64_t full[NBUF], wbar, mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tiles = (M + BM - 1) / BM;

  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&wbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&tmem_base)), "n"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  auto issue = [&](int j) {  // TMA of this CTA's j-th tile into stage j % NBUF
    const int tile = blockIdx.x + j * gridDim.x;
    if (tile >= tiles) return;
    uint64_t* bar = &full[j % NBUF];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(STAGE));
#pragma unroll
    for (int kb = 0; kb < KB; ++kb)
      tma2d(sa0 + (j % NBUF) * STAGE + kb * 16384, &hmap, kb * 64, tile * BM, bar);
  };
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(&wbar)), "r"(KB * 4096));
#pragma unroll
    for (int kb = 0; kb < KB; ++kb) tma2d(sw + kb * 4096, &wmap, kb * 64, 0, &wbar);
    for (int j = 0; j < NBUF - 1; ++j) issue(j);
    mbar_wait(&wbar, 0);
  }
  // idesc: D fp32, A and B bf16, both K-major, N >> 3 at bit 17, M >> 4 at bit 24
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)(BM >> 4) << 24);
  const float b_lane = (lane <= A && bias != nullptr) ? bias[lane] : 0.f;
  // ceil(2^32 / A): floor(i * a_magic / 2^32) = floor(i / A) while i * (a_magic - 2^32/A)
  // < 2^32 / A, i.e. for every i < 128 * 31 (error < 4e3 / 2^32 < 1 / A); A = 1 wraps to 0
  // and takes r = i (checked exhaustively on the host for A = 2..31)
  const uint32_t a_magic = (uint32_t)((0x100000000ull + (uint32_t)A - 1) / (uint32_t)A);

  for (int j = 0;; ++j) {
    const int tile = blockIdx.x + j * gridDim.x;
    if (tile >= tiles) break;
    if (tid == 0) {
      issue(j + NBUF - 1);  // its stage held tile j-1, whose MMAs completed (mbar below)
      mbar_wait(&full[j % NBUF], (j / NBUF) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_base = sa0 + (j % NBUF) * STAGE;
#pragma unroll
      for (int k = 0; k < KB * 4; ++k) {  // K = 16 per MMA: +32 B inside a 128-byte atom
        const uint64_t da = desc_sw128(a_base + (k >> 2) * 16384 + (k & 3) * 32);
        const uint64_t db = desc_sw128(sw + (k >> 2) * 4096 + (k & 3) * 32);
        const uint32_t acc = k > 0;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(smem_u32(&mbar)));
    }
    mbar_wait(&mbar, j & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {  // TMEM lanes 32w..32w+31 = rows of warp w
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
          "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      // all 32 accumulator columns, unconditionally (no per-column branches); the row
      // stride SO_LD = 33 keeps the 32 lanes' stores on distinct banks
      const int r = warp * 32 + lane;
#pragma unroll
      for (int n = 0; n < BN; ++n)
        so[r * SO_LD + n] = __uint_as_float(v[n]) + __shfl_sync(0xffffffffu, b_lane, n);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    const int row0 = tile * BM, rows = min(BM, M - row0);
    float* zdst = z_out + (size_t)row0 * A;
    for (int i = tid; i < rows * A; i += THREADS) {
      const int r = A == 1 ? i : (int)__umulhi((uint32_t)i, a_magic);  // == i / A
      zdst[i] = so[r * SO_LD + (i - r * A)];
    }
    for (int i = tid; i < rows; i += THREADS) v_out[row0 + i] = so[i * SO_LD + A];
    __syncthreads();
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(32));
}

std::mutex g_mu;
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
int g_dev_state[64] = {0};  // 0 unknown, 1 sm_100, 2 other
int g_sms[64] = {0};

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return g_encode;
}

vt_status device_sms(int* sms) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return VT_ERR_CUDA;
  if (dev < 0 || dev >= 64) return VT_ERR_DEVICE;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_dev_state[dev] == 0) {
    int maj = 0, mnr = 0, n = 0;
    if (cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return VT_ERR_CUDA;
    g_dev_state[dev] = (maj == 10 && mnr == 0) ? 1 : 2;
    g_sms[dev] = n;
  }
  *sms = g_sms[dev];
  return g_dev_state[dev] == 1 ? VT_OK : VT_ERR_DEVICE;
}

template <int KB>
vt_status launch(const CUtensorMap& hm, const CUtensorMap& wm, const float* bias, float* z,
                 float* v, int M, int A, int sms, cudaStream_t st) {
  constexpr int NBUF = std::min(4, (SMEM_LIMIT - 1024 - KB * 4096 - BM * SO_LD * 4) / (KB * 16384));
  static_assert(NBUF >= 2, "ring too shallow");
  constexpr int SMEM = 1024 + KB * 4096 + NBUF * KB * 16384 + BM * SO_LD * 4;
  auto kern = output_layer_kernel<KB, NBUF>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
    return VT_ERR_CUDA;
  const int tiles = (M + BM - 1) / BM;
  kern<<<std::min(sms, tiles), THREADS, SMEM, st>>>(hm, wm, bias, z, v, M, A);
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}

}  // namespace vtol

extern "C" vt_status vtrace_output_layer(int64_t M, int32_t H, int32_t A, const void* hidden,
                                         const void* w_t, const float* bias, float* logits_out,
                                         float* values_out, vt_stream_t stream) {
  using namespace vtol;
  if (M < 0 || M > INT32_MAX - BM || H <= 0 || H > 256 || H % 64 != 0 || A < 1 || A + 1 > BN)
    return VT_ERR_SHAPE;
  if (M == 0) return VT_OK;
  if (!hidden || !w_t || !logits_out || !values_out) return VT_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(hidden) & 15) || (reinterpret_cast<uintptr_t>(w_t) & 15) ||
      (reinterpret_cast<uintptr_t>(logits_out) & 3) || (reinterpret_cast<uintptr_t>(values_out) & 3) ||
      (reinterpret_cast<uintptr_t>(bias) & 3))
    return VT_ERR_ALIGNMENT;
  int sms = 0;
  vt_status s = device_sms(&sms);
  if (s != VT_OK) return s;
  auto enc = encoder();
  if (!enc) return VT_ERR_CUDA;
  CUtensorMap hm, wm;
  cuuint64_t hd[2] = {(cuuint64_t)H, (cuuint64_t)M}, hs[1] = {(cuuint64_t)H * 2};
  cuuint64_t wd[2] = {(cuuint64_t)H, (cuuint64_t)(A + 1)}, ws[1] = {(cuuint64_t)H * 2};
  cuuint32_t hb[2] = {64, (cuuint32_t)BM}, wb[2] = {64, (cuuint32_t)BN}, es[2] = {1, 1};
  // rows past M (h) and past A+1 (W^T) are zero-filled by the TMA unit
  if (enc(&hm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(hidden), hd, hs, hb, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      enc(&wm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w_t), wd, ws, wb, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return VT_ERR_CUDA;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int m = (int)M;
  switch (H / 64) {
    case 1: return launch<1>(hm, wm, bias, logits_out, values_out, m, A, sms, st);
    case 2: return launch<2>(hm, wm, bias, logits_out, values_out, m, A, sms, st);
    case 3: return launch<3>(hm, wm, bias, logits_out, values_out, m, A, sms, st);
    default: return launch<4>(hm, wm, bias, logits_out, values_out, m, A, sms, st);
  }
}
