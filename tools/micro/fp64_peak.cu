// FP64 issue-rate microbenchmark (DFMA / DADD / DMUL) on the B200: one grid
// of 148 x k CTAs, 8 independent chains per thread; prints TFLOP/s and
// warp-instructions per SMSP per clock.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = fma(x[i], a, b);
      else if (OP == 1) x[i] = x[i] + b;
      else x[i] = x[i] * a;
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[3] = {"DFMA", "DADD", "DMUL"};
  for (int op = 0; op < 3; ++op)
    for (int wps : {4, 8, 16, 32}) {  // warps per SM
      const int iters = 20000, nt = 256, ctas = sms * wps * 32 / nt;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (op == 0) k<0><<<ctas, nt>>>(o, iters, 0.999, 1e-3);
        else if (op == 1) k<1><<<ctas, nt>>>(o, iters, 0.999, 1e-3);
        else k<2><<<ctas, nt>>>(o, iters, 0.999, 1e-3);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double inst = (double)ctas * nt * iters * 8;  // thread instructions
      const double flops = inst * (op == 0 ? 2 : 1);
      const double warp_inst_per_smsp_clk = inst / 32 / (sms * 4) / (ms * 1e-3 * clk * 1e3);
      printf("%s warps/SM %2d: %.2f ms  %.1f TFLOP/s  %.3f warp-inst/SMSP/clk (at %d MHz nominal)\n", names[op], wps, ms,
             flops / ms / 1e9, warp_inst_per_smsp_clk, clk / 1000);
    }
  return 0;
}
