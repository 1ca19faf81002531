// pipe_probe.cu -- per-SM throughput of a few instruction classes on sm_100a
// (dev tool): F2F.F64.F32, DADD, DFMA, MUFU.EX2, FADD, FFMA.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 0.5f, d = 0.25f;
  double x = a, y = 1.0, z = 0.5, w = 0.25;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) { x += (double)a; y += (double)b; z += (double)c; w += (double)d; a += 1e-7f; b += 1e-7f; c += 1e-7f; d += 1e-7f; }
      if (OP == 1) { x = x + y; y = y + z; z = z + w; w = w + x; }
      if (OP == 2) { x = fma(x, y, z); y = fma(y, z, w); z = fma(z, w, x); w = fma(w, x, y); }
      if (OP == 3) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a)); a = r * 0.5f; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b)); b = r * 0.5f; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(c)); c = r*0.5f; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d)); d = r*0.5f; }
      if (OP == 4) { a = a + b; b = b + c; c = c + d; d = d + a; }
      if (OP == 5) { a = fmaf(a, b, c); b = fmaf(b, c, d); c = fmaf(c, d, a); d = fmaf(d, a, b); }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[2 + (threadIdx.x & 7)] = a + b + c + d + (float)(x + y + z + w);
}

int main() {
  float* o; cudaMalloc(&o, 64);
  const char* names[] = {"F2F.F64.F32 (+FADD)", "DADD", "DFMA", "MUFU.EX2 (+FMUL)", "FADD", "FFMA"};
  const int per[] = {4, 4, 4, 4, 4, 4};  // ops of the class per inner step
  for (int op = 0; op < 6; ++op) {
    int iters = 2000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto launch = [&](int blocks, int threads) {
      switch (op) {
        case 0: k<0><<<blocks, threads>>>(o, iters); break;
        case 1: k<1><<<blocks, threads>>>(o, iters); break;
        case 2: k<2><<<blocks, threads>>>(o, iters); break;
        case 3: k<3><<<blocks, threads>>>(o, iters); break;
        case 4: k<4><<<blocks, threads>>>(o, iters); break;
        case 5: k<5><<<blocks, threads>>>(o, iters); break;
      }
    };
    launch(148 * 4, 512);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch(148 * 4, 512);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    float h[2]; cudaMemcpy(h, o, 8, cudaMemcpyDeviceToHost);
    double ops = 148.0 * 4 * 512 * iters * 8 * per[op];
    double cyc = h[1];  // cycles of block 0 (all blocks co-resident, 4 per SM)
    printf("%-22s %8.1f ops/clk/SM (block0 cycles %.0f, %.3f ms)\n", names[op],
           ops / 148.0 / cyc, cyc, ms);
  }
  return 0;
}
