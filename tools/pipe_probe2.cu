// pipe_probe2.cu -- per-SM throughput and single-warp latency of the instruction
// classes on the V-trace row path (dev tool, B200 sm_100a).
// Throughput: 4 x 512-thread CTAs per SM, 8 independent chains per thread.
// Latency: one warp, one dependent chain.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

enum { F2F64, F2F32, DADD_, DFMA_, DMUL_, EX2, LG2, RCP64, FADD2_, FFMA2_, FFMA_, FMNMX_, SHFL32,
       SHFL64, LDS32, IMAD_, NOPS };
static const char* kName[NOPS] = {"F2F.F64.F32", "F2F.F32.F64", "DADD", "DFMA", "DMUL",
                                  "MUFU.EX2", "MUFU.LG2", "MUFU.RCP64H", "FADD2", "FFMA2",
                                  "FFMA", "FMNMX", "SHFL.32", "SHFL.64(2)", "LDS.32", "IMAD"};

template <int OP, int NCH>
__global__ void k(float* out, int iters, int lat) {
  __shared__ float sh[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = i * 1e-3f;
  __syncthreads();
  float f[NCH];
  double d[NCH];
  float2 g[NCH];
  int ii[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    f[c] = threadIdx.x * 1e-3f + c;
    d[c] = f[c];
    g[c] = make_float2(f[c], f[c] + 1.f);
    ii[c] = threadIdx.x + c;
  }
  const float2 m2 = make_float2(0.999f, 1.001f), a2 = make_float2(1e-3f, 2e-3f);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (OP == F2F64) { d[c] = (double)f[c]; f[c] = __int_as_float(__double2loint(d[c]) | 0x3f800000); }
        if (OP == F2F32) { f[c] = (float)d[c]; d[c] = __longlong_as_double(((long long)__float_as_int(f[c]) << 20) | 0x3ff0000000000000ll); }
        if (OP == DADD_) d[c] = d[c] + 1.0000001;
        if (OP == DFMA_) d[c] = fma(d[c], 0.999999, 1e-3);
        if (OP == DMUL_) d[c] = d[c] * 0.9999999;
        if (OP == EX2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[c]));
        if (OP == LG2) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(f[c]));
        if (OP == RCP64) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(d[c]));
        if (OP == FADD2_) g[c] = __fadd2_rn(g[c], a2);
        if (OP == FFMA2_) g[c] = __ffma2_rn(g[c], m2, a2);
        if (OP == FFMA_) f[c] = fmaf(f[c], 0.9999f, 1e-3f);
        if (OP == FMNMX_) f[c] = fmaxf(f[c], f[(c + 1) % NCH] * 0.5f);
        if (OP == SHFL32) f[c] = __shfl_down_sync(0xffffffffu, f[c], 4);
        if (OP == SHFL64) d[c] = __shfl_down_sync(0xffffffffu, d[c], 4);
        if (OP == LDS32) ii[c] = __float_as_int(sh[(ii[c] & 1023)]) & 1023;
        if (OP == IMAD_) ii[c] = ii[c] * 3 + 7;
      }
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) acc += f[c] + (float)d[c] + g[c].x + g[c].y + ii[c];
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[2 + (threadIdx.x & 7)] = acc;
}

template <int OP>
void run(float* o) {
  const int iters = 256;
  float h[2];
  // throughput: 4 CTAs x 512 threads per SM, 8 chains
  k<OP, 8><<<148 * 4, 512>>>(o, iters, 0);
  k<OP, 8><<<148 * 4, 512>>>(o, iters, 0);
  cudaDeviceSynchronize();
  cudaMemcpy(h, o, 8, cudaMemcpyDeviceToHost);
  const double ops_sm = 4.0 * 512 * iters * 4 * 8;
  const double tput = ops_sm / h[1];
  // latency: 1 warp, 1 chain
  k<OP, 1><<<1, 32>>>(o, iters, 1);
  k<OP, 1><<<1, 32>>>(o, iters, 1);
  cudaDeviceSynchronize();
  cudaMemcpy(h, o, 8, cudaMemcpyDeviceToHost);
  const double lat = h[1] / (iters * 4.0);
  printf("%-14s %7.1f lane-ops/clk/SM  (%5.2f warp-instr/clk/SM)  latency %5.1f clk/op\n",
         kName[OP], tput, tput / 32.0, lat);
}

int main() {
  float* o;
  cudaMalloc(&o, 64);
  run<F2F64>(o); run<F2F32>(o); run<DADD_>(o); run<DFMA_>(o); run<DMUL_>(o); run<EX2>(o);
  run<LG2>(o); run<RCP64>(o); run<FADD2_>(o); run<FFMA2_>(o); run<FFMA_>(o); run<FMNMX_>(o);
  run<SHFL32>(o); run<SHFL64>(o); run<LDS32>(o); run<IMAD_>(o);
  printf("(F2F rows include one integer op per conversion; FMNMX includes an FMUL; FADD2/FFMA2 count one op per float2)\n");
  return 0;
}
