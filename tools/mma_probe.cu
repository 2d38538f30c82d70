// Debug probe for tcgen05 kind::tf32 layouts (not part of the product).
#include <cuda_runtime.h>
#include <stdio.h>
#include "../paper_2503_10855_b200/csrc/tcgen05.cuh"
using namespace jb;

// mode bit0: B K-major (else MN-major); bit1: use 4 k-steps (K=32) else 1 (K=8)
// bit2: swap LBO/SBO for MN-major; bit3: MN-major with SWIZZLE_128B_BASE32B
// (layout type 1: 32-byte chunks XOR (row & 3), 4-row K groups)
__global__ void probe(const float* A, const float* B, float* C, float* dbg, int mode) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[64 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool bk = mode & 1;
  // A: 128 rows x 32 k, K-major SW128
  for (int i = tid; i < 128 * 32; i += blockDim.x) {
    int r = i / 32, k = i % 32;
    int off = r * 128 + (((k >> 2) ^ (r & 7)) << 4) + (k & 3) * 4;
    *(float*)(sa + off) = A[r * 32 + k];
  }
  // B logical [K=32][N=64]
  for (int i = tid; i < 32 * 64; i += blockDim.x) {
    int k = i / 64, nn = i % 64;
    int off;
    if (bk) {  // K-major: row = n (64 rows of 128B), chunk by k
      off = nn * 128 + (((k >> 2) ^ (nn & 7)) << 4) + (k & 3) * 4;
    } else if (mode & 8) {  // MN-major BASE32B: 32B chunk (c>>3) ^ (k&3)
      int a = nn >> 5, c = nn & 31;
      off = a * 4096 + k * 128 + (((c >> 3) ^ (k & 3)) << 5) + (c & 7) * 4;
    } else {   // MN-major: atom = nn/32 at 4096*atom, row = k
      int a = nn >> 5, c = nn & 31;
      off = a * 4096 + k * 128 + (((c >> 2) ^ (k & 7)) << 4) + (c & 3) * 4;
    }
    *(float*)(sb + off) = B[k * 64 + nn];
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<64>(&tbase);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  uint32_t td = tbase;
  if (tid == 0) {
    uint32_t idesc = tc::idesc_tf32(128, 64, 0, bk ? 0 : 1);
    int ksteps = (mode & 2) ? 4 : 1;
    for (int k = 0; k < ksteps; k++) {
      uint64_t da = tc::smem_desc_sw128(tc::smem_u32(sa) + k * 32, 16, 1024);
      uint64_t db = bk ? tc::smem_desc_sw128(tc::smem_u32(sb) + k * 32, 16, 1024)
                       : ((mode & 4) ? tc::smem_desc_sw128(tc::smem_u32(sb) + k * 1024, 1024, 4096)
                                     : tc::smem_desc_sw128(tc::smem_u32(sb) + k * 1024, 4096, 1024));
      if (!bk && (mode & 8)) {
        db = (mode & 4) ? tc::smem_desc_sw128(tc::smem_u32(sb) + k * 1024, 512, 4096)
                        : tc::smem_desc_sw128(tc::smem_u32(sb) + k * 1024, 4096, 512);
        db = (db & ~(7ull << 61)) | (1ull << 61);  // layout type 1 = SWIZZLE_128B_BASE32B
      }
      if (k == 0) { dbg[0] = __uint_as_float((uint32_t)da); dbg[1] = __uint_as_float((uint32_t)(da >> 32));
                    dbg[2] = __uint_as_float((uint32_t)db); dbg[3] = __uint_as_float((uint32_t)(db >> 32));
                    dbg[4] = __uint_as_float(idesc); dbg[5] = __uint_as_float(td); }
      tc::mma_tf32(td, da, db, idesc, k > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  int q = warp & 3;
  for (int cb = 0; cb < 64; cb += 16) {
    uint32_t r[16];
    tc::tmem_ld_32x32b_x16(td + ((uint32_t)(q * 32) << 16) + cb, r);
    tc::tmem_ld_wait();
    for (int v = 0; v < 16; v++) C[(q * 32 + lane) * 64 + cb + v] = __uint_as_float(r[v]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc::tc_fence_after(); tc::tmem_dealloc<64>(td); }
}

extern "C" int run_probe(const float* hA, const float* hB, float* hC, float* hdbg, int mode) {
  float *A, *B, *C, *D;
  cudaMalloc(&A, 128 * 32 * 4); cudaMalloc(&B, 32 * 64 * 4); cudaMalloc(&C, 128 * 64 * 4); cudaMalloc(&D, 64);
  cudaMemcpy(A, hA, 128 * 32 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, 32 * 64 * 4, cudaMemcpyHostToDevice);
  cudaMemset(C, 0xff, 128 * 64 * 4);
  probe<<<1, 128>>>(A, B, C, D, mode);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hC, C, 128 * 64 * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hdbg, D, 24, cudaMemcpyDeviceToHost);
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(D);
  return (int)e;
}
