// microbenchmark (not product): per-SM issue rates of the instruction forms the
// bit-exact stencils use, in warp-instructions per clock per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates tools/pipe_rates.cu
#include <cstdio>
#include <cuda_runtime.h>
__constant__ float cc[64];
#define N 8
template <int M>
__global__ void k(float *out, int iters, float s) {
  float a[N], b[N];
  unsigned long long p[N];
  unsigned u[N];
  for (int i = 0; i < N; i++) {
    a[i] = threadIdx.x * 1e-3f + i; b[i] = a[i] * 0.5f + 1.f; u[i] = threadIdx.x + i;
    asm("mov.b64 %0, {%1, %2};" : "=l"(p[i]) : "f"(a[i]), "f"(b[i]));
  }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 16; j++) {
#pragma unroll
      for (int i = 0; i < N; i++) {
        if (M == 0) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
        if (M == 1) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
        if (M == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b[i]), "f"(b[(i + 1) % N]));
        if (M == 3) asm volatile("fma.rn.f32 %0, %0, %1, 0f3F000000;" : "+f"(a[i]) : "f"(b[i]));
        if (M == 4) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(p[(i + 1) % N]), "l"(p[(i + 2) % N]));
        if (M == 5) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(p[(i + 1) % N]));
        if (M == 6) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(p[(i + 1) % N]));
        if (M == 7) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        if (M == 8) { asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b[i]), "f"(b[(i + 1) % N]));
                      asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 1) % N])); }
        if (M == 9) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
        if (M == 10) { asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
                       asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(b[i]) : "f"(a[(i + 1) % N])); }
        if (M == 11) a[i] = __fdiv_rn(a[i], b[i]);
        if (M == 12) asm volatile("sqrt.rn.f32 %0, %0;" : "+f"(a[i]));
        if (M == 13) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(s));
      }
    }
  }
  float r = 0;
  for (int i = 0; i < N; i++) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(p[i])); r += a[i] + b[i] + x + y + (float)u[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
typedef void (*KF)(float *, int, float);
int main() {
  float *out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  KF ks[] = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>, k<10>, k<11>, k<12>, k<13>};
  const char *names[] = {"FADD r,r", "FMUL r,r", "FFMA r,r,r", "FFMA r,r,imm", "FFMA2 (f32x2)", "FMUL2", "FADD2",
                         "MUFU.RCP", "FFMA + IADD (2 instr)", "FMNMX", "FADD + FMUL (2 instr)", "div.rn (per div)",
                         "sqrt.rn (per sqrt)", "FADD r,c (uniform)"};
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 400, threads = 256;
  for (int blocksPerSM = 4; blocksPerSM <= 8; blocksPerSM += 4) {
    const int blocks = sms * blocksPerSM;
    for (int m = 0; m < 14; m++) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        ks[m]<<<blocks, threads>>>(out, iters, 1.0f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double winstr = (double)blocks * (threads / 32) * iters * 16 * N * ((m == 8 || m == 10) ? 2 : 1);
      printf("%2d warps/SMSP  %-24s %8.3f ms  %6.3f warp-instr/clk/SM (at %d MHz)\n", blocksPerSM * 2, names[m], best,
             winstr / (best * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
