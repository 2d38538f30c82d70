// microbenchmark: FP32 pipe throughput of the instruction forms used by the
// bit-exact stencils (not part of the product)
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2503_10855_b200/csrc/common.cuh"
using namespace jb;
__constant__ float cc[64];
template <int MODE>
__global__ void k(float *out, int iters) {
  float a[8], b[8];
  unsigned long long p[8], q[8];
  for (int i = 0; i < 8; i++) { a[i] = threadIdx.x * 0.001f + i; b[i] = 0.f; p[i] = f22u(make_float2(a[i], a[i] + 1)); q[i] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
#pragma unroll
      for (int i = 0; i < 8; i++) {
        if (MODE == 0) a[i] = __fadd_rn(a[i], __fmul_rn(a[i], cc[j]));            // FMUL + FADD
        if (MODE == 1) p[i] = f2_add_ftz(p[i], f2_mul(p[i], cc[j]));               // FMUL2 + FADD2.FTZ
        if (MODE == 2) a[i] = fmaf(a[i], cc[j], a[i]);                            // FFMA (const)
        if (MODE == 3) a[i] = fmaf(a[i], a[(i + 1) & 7], a[i]);                   // FFMA 3-reg
      }
    }
  }
  float s = 0;
  for (int i = 0; i < 8; i++) { s += a[i] + b[i]; float2 f = u2f2(p[i]); s += f.x + f.y + u2f2(q[i]).x; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float h[64]; for (int i = 0; i < 64; i++) h[i] = 1e-7f * (i + 1);
  cudaMemcpyToSymbol(cc, h, sizeof(h));
  float *out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000, blocks = 148 * 8, threads = 256;
  const char *names[] = {"FMUL+FADD (2 instr / fma-equiv)", "FMUL2+FADD2.FTZ (2 instr / 2 fma-equiv)", "FFMA c[]", "FFMA 3-reg"};
  for (int mode = 0; mode < 4; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(out, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(out, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(out, iters);
      if (mode == 3) k<3><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 64;           // multiply-adds (per lane-element)
      double lanes = (mode == 1) ? 2.0 : 1.0;
      double instrs = ops * ((mode <= 1) ? 2.0 : 1.0) / 32.0;          // warp instructions
      if (rep) printf("%-42s %8.3f ms  %7.2f T mul-add/s  %6.1f G warp-instr/s  (%.2f warp-instr/clk/SM @1.965GHz)\n",
                      names[mode], ms, ops * lanes / ms / 1e9, instrs / ms / 1e6, instrs / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
