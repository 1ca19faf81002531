// TMA streaming probe: one CTA of W warps per SM; each warp walks its column
// group of a [T][B*A] bf16 matrix (two of them, like z^pi and z^mu) backwards in
// time with a per-warp NSTAGE ring of {cols*A, steps} boxes, optionally storing
// one box per step back to a third matrix (like dlogits).  Reports GB/s.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Cfg { int T, B, A, cols, steps, nstage, store, W, map, promo; };

__global__ void __launch_bounds__(1024, 1) probe(const __grid_constant__ CUtensorMap mpi,
                                                const __grid_constant__ CUtensorMap mmu,
                                                const __grid_constant__ CUtensorMap mdz, Cfg c,
                                                unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[32][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ntask = c.B / c.cols;
  const int tile = c.cols * c.A * 2 * c.steps;
  const int tile_a = (tile + 127) & ~127;
  unsigned char* base = smem + (size_t)w * c.nstage * 2 * tile_a;
  const int K = (c.T + c.steps - 1) / c.steps;
  unsigned long long acc = 0;
  // map 0: SM s, warp w -> task s + S w (tasks spread over SMs); map 1: task s W + w
  // (an SM's warps take adjacent column groups); map 2: contiguous 1D blocks (ceiling)
  for (int task = c.map == 1 ? blockIdx.x * c.W + w : blockIdx.x + gridDim.x * w; task < ntask;
       task += gridDim.x * c.W) {
    const int x = task * c.cols * c.A;
    auto load = [&](int it) {
      if (it >= K) return;
      const int st = it % c.nstage;
      int t0 = (K - 1 - it) * c.steps;
      int xx = x;
      if (c.map == 2) {  // contiguous: this task's it-th block of the flattened rows
        const long long blk = (long long)task * K + it;  // blocks of cols*A*steps elements
        const long long row_elems = (long long)c.B * c.A;
        const long long e0 = blk * (long long)(c.cols * c.A);  // column block within a row band
        xx = (int)(e0 % row_elems);
        t0 = (int)((e0 / row_elems) * c.steps) % c.T;
      }
      unsigned char* sb = base + (size_t)st * 2 * tile_a;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[w][st])), "r"(2 * tile) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sb)), "l"(&mpi), "r"(xx), "r"(t0), "r"(su32(&bar[w][st])) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sb + tile_a)), "l"(&mmu), "r"(xx), "r"(t0), "r"(su32(&bar[w][st])) : "memory");
    };
    if (lane == 0) {
      for (int s = 0; s < c.nstage; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[w][s])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int s = 0; s < c.nstage; ++s) load(s);
    }
    __syncwarp();
    uint32_t ph = 0;
    for (int it = 0; it < K; ++it) {
      const int st = it % c.nstage;
      unsigned char* sb = base + (size_t)st * 2 * tile_a;
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                   ::"r"(su32(&bar[w][st])), "r"((ph >> st) & 1) : "memory");
      ph ^= 1u << st;
      acc += reinterpret_cast<const uint32_t*>(sb)[lane] + reinterpret_cast<const uint32_t*>(sb + tile_a)[lane];
      __syncwarp();
      if (lane == 0) {
        if (c.store) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                       ::"l"(&mdz), "r"(x), "r"((K - 1 - it) * c.steps), "r"(su32(sb)) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (it >= 1) {
          if (c.store) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          load(it + c.nstage - 1);
        }
      }
      __syncwarp();
    }
    if (lane == 0 && c.store) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
    // barriers are re-initialised for the next task of this warp (phases reset)
    if (lane == 0)
      for (int s = 0; s < c.nstage; ++s)
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(su32(&bar[w][s])) : "memory");
    __syncwarp();
  }
  if (acc == 0x1234567) sink[0] = acc;
}

__global__ void raw_read(const float4* a, const float4* b, size_t n4, float4* out, int store,
                         unsigned long long* sink) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    const float4 x = __ldcs(a + i), y = __ldcs(b + i);
    acc += x.x + y.y;
    if (store) __stcs(out + i, x);
  }
  if (acc == 1234.5f) sink[0] = 1;
}

int main(int argc, char** argv) {
  Cfg c;
  c.T = 100; c.B = 8192; c.A = 18;
  c.cols = argc > 1 ? atoi(argv[1]) : 4;
  c.steps = argc > 2 ? atoi(argv[2]) : 8;
  c.nstage = argc > 3 ? atoi(argv[3]) : 4;
  c.store = argc > 4 ? atoi(argv[4]) : 1;
  c.W = argc > 5 ? atoi(argv[5]) : 16;
  c.map = argc > 6 ? atoi(argv[6]) : 0;
  c.promo = argc > 7 ? atoi(argv[7]) : 2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = (size_t)c.T * c.B * c.A;
  const int R = 6;  // rotate over copies (> L2)
  void *pi[R], *mu[R], *dz[R];
  for (int r = 0; r < R; ++r) {
    cudaMalloc(&pi[r], n * 2); cudaMalloc(&mu[r], n * 2); cudaMalloc(&dz[r], n * 2);
    cudaMemset(pi[r], 0, n * 2); cudaMemset(mu[r], 0, n * 2);
  }
  unsigned long long* sink; cudaMalloc(&sink, 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap mp[R], mm[R], md[R];
  for (int r = 0; r < R; ++r) {
    cuuint64_t dims[2] = {(cuuint64_t)c.B * c.A, (cuuint64_t)c.T};
    cuuint64_t str[1] = {(cuuint64_t)c.B * c.A * 2};
    cuuint32_t box[2] = {(cuuint32_t)(c.cols * c.A), (cuuint32_t)c.steps};
    cuuint32_t es[2] = {1, 1};
    void* bases[3] = {pi[r], mu[r], dz[r]};
    CUtensorMap* ms[3] = {&mp[r], &mm[r], &md[r]};
    for (int k = 0; k < 3; ++k)
      if (enc(ms[k], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, bases[k], dims, str, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              (CUtensorMapL2promotion)c.promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n"); return 1;
      }
  }
  const int tile = c.cols * c.A * 2 * c.steps, tile_a = (tile + 127) & ~127;
  const size_t smem = (size_t)c.W * c.nstage * 2 * tile_a;
  if (smem > 227 * 1024) { printf("smem %zu too big\n", smem); return 1; }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (c.map == 9) {  // plain vectorised streaming ceiling
    const size_t n4 = n * 2 / 16;
    for (int i = 0; i < 10; ++i)
      raw_read<<<sms * 8, 512>>>((const float4*)pi[i % R], (const float4*)mu[i % R], n4, (float4*)dz[i % R], c.store, sink);
    cudaEvent_t a0, a1; cudaEventCreate(&a0); cudaEventCreate(&a1);
    cudaEventRecord(a0);
    for (int i = 0; i < 200; ++i)
      raw_read<<<sms * 8, 512>>>((const float4*)pi[i % R], (const float4*)mu[i % R], n4, (float4*)dz[i % R], c.store, sink);
    cudaEventRecord(a1); cudaEventSynchronize(a1);
    float m2; cudaEventElapsedTime(&m2, a0, a1);
    const double us2 = m2 * 1000.0 / 200;
    printf("raw streaming store %d: %.2f us, %.0f GB/s\n", c.store, us2, (double)n * 2 * (c.store ? 3 : 2) / us2 / 1e3);
    return 0;
  }
  for (int i = 0; i < 10; ++i) probe<<<sms, c.W * 32, smem>>>(mp[i % R], mm[i % R], md[i % R], c, sink);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 200;
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) probe<<<sms, c.W * 32, smem>>>(mp[i % R], mm[i % R], md[i % R], c, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms_; cudaEventElapsedTime(&ms_, e0, e1);
  const double us = ms_ * 1000.0 / iters;
  const double bytes = (double)n * 2 * (c.store ? 3 : 2);
  printf("promo %d map %d cols %d steps %d nstage %d store %d W %d: %.2f us, %.0f GB/s (%s)\n", c.promo, c.map, c.cols, c.steps,
         c.nstage, c.store, c.W, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
