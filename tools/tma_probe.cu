// probe: 2-D TMA box loads with unaligned starts / odd box widths (debug tool)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2503_10855_b200/csrc/common.cuh"
#include "../paper_2503_10855_b200/csrc/tcgen05.cuh"
using namespace jb;
struct P { CUtensorMap tm; int x, y, bw, bh; };
__global__ void k(const __grid_constant__ P p, float *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    tc::mbar_arrive_expect_tx(&bar, p.bw * p.bh * 4);
    tc::tma_load_2d(sm, &p.tm, &bar, p.x, p.y);
  }
  tc::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < p.bw * p.bh; i += blockDim.x) out[i] = ((float *)sm)[i];
}

int main(int argc, char **argv) {
  const int W = 200, H = 128;
  float *g, *o; cudaMalloc(&g, W * H * 4); cudaMalloc(&o, 256 * 256 * 4);
  float *h = new float[W * H]; for (int i = 0; i < W * H; i++) h[i] = i;
  cudaMemcpy(g, h, W * H * 4, cudaMemcpyHostToDevice);
  int cases[][4] = {{atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), atoi(argv[4])}};
  for (auto &c : cases) {
    P p; p.bw = c[0]; p.bh = c[1]; p.x = c[2]; p.y = c[3];
    uint64_t dims[2] = {W, H}, str[1] = {W * 4}; uint32_t box[2] = {(uint32_t)p.bw, (uint32_t)p.bh};
    bool ok = make_tmap_f32(&p.tm, g, 2, dims, str, box, 0);
    k<<<1, 128, p.bw * p.bh * 4 + 128>>>(p, o);
    cudaError_t e = cudaDeviceSynchronize();
    float r[4]; cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    printf("box %dx%d at (%d,%d): encode=%d err=%s first=%g expect=%g\n", p.bw, p.bh, p.x, p.y, ok, cudaGetErrorString(e), r[0], (float)(p.y * W + p.x));
    if (e != cudaSuccess) { cudaDeviceReset(); cudaMalloc(&g, W * H * 4); cudaMalloc(&o, 256 * 256 * 4); cudaMemcpy(g, h, W * H * 4, cudaMemcpyHostToDevice); }
  }
}
