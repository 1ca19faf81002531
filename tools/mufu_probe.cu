// mufu_probe.cu -- measures the relative error of ex2.approx.ftz.f32 (MUFU.EX2)
// on sm_100a against exp2 in fp64, over a dense sweep of fp32 arguments in
// [-24, 0] (the range of (z - max z) * log2 e for logits).  Dev tool: the
// numbers decide the EXP_MUFU vs EXP_F64 precision mode.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long n, float lo, float hi) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double se = 0, sa = 0, mx = 0, sb = 0;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) {
    float x = lo + (hi - lo) * (float)((double)i / (double)n);
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    double ref = exp2((double)x);
    double rel = ((double)y - ref) / ref;
    se += rel * rel; sa += fabs(rel); sb += rel;
    if (fabs(rel) > mx) mx = fabs(rel);
  }
  atomicAdd(out + 0, se); atomicAdd(out + 1, sa); atomicAdd(out + 3, sb);
  unsigned long long* m = (unsigned long long*)(out + 2);
  atomicMax(m, __double_as_longlong(mx));
}

int main() {
  double* d; cudaMalloc(&d, 32);
  const long long n = 1LL << 28;
  float ranges[3][2] = {{-24.f, 0.f}, {-1.f, 0.f}, {-0.25f, 0.f}};
  for (auto& r : ranges) {
    cudaMemset(d, 0, 32);
    probe<<<148 * 8, 256>>>(d, n, r[0], r[1]);
    double h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("ex2.approx.ftz.f32 on [%g,%g]: rms rel %.3e  mean|rel| %.3e  max|rel| %.3e  bias %.3e  (ulp 2^-23 = %.3e)\n",
           r[0], r[1], sqrt(h[0] / n), h[1] / n, *(double*)&h[2], h[3] / n, ldexp(1.0, -23));
  }
  return 0;
}
