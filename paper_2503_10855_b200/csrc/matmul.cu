// matmul.cu -- matmul<n,m,l>(a: f32[n,m], b: f32[m,l]) -> f32[n,l] on sm_100a.
//
// Juno program: Fig. 1 of the paper, restated in
// oracle/juno_oracle.c:jo_matmul_f32 (res[i,j] += a[i,k]*b[k,j], k ascending).
// The k-reduce is a monoid add that the paper's schedules re-associate
// (monoid-reassociate), so the contract is fp32 tolerance:
//     |C - C_ref| <= (2*gamma_m + 8u) * (|A| |B|)   elementwise, u = 2^-24.
//
// B200 design: 3xTF32 on the 5th-gen tensor cores.
//   split kernels  : A -> (A_hi, A_lo), B -> (Bt_hi, Bt_lo) with x_hi =
//                    rna_tf32(x), x_lo = rna_tf32(x - x_hi); B is transposed
//                    on the way (tiled through shared memory) so both MMA
//                    operands are K-major (an MN-major tf32 B descriptor
//                    produced no result on this part, tools/mma_probe.cu).
//   gemm kernel    : one 128x64 output tile per CTA; warp 0 = TMA producer
//                    (4 operand tiles per 32-wide k-block, 128B swizzle,
//                    4-stage mbarrier ring), warp 1 = TMEM allocator + single
//                    thread tcgen05.mma issuer (D += Ahi*Bhi + Ahi*Blo +
//                    Alo*Bhi, f32 accumulators in 64 TMEM columns), warps 2-5
//                    = epilogue (tcgen05.ld -> registers -> global).
// Shapes the TMA path cannot take (row pitch not a multiple of 16 bytes) run
// an exact SIMT kernel that follows the oracle's k order bit for bit.
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "tcgen05.cuh"

namespace jb {
namespace mm {

constexpr int BM = 128, BN = 64, BK = 32;  // BK fp32 = one 128-byte swizzle row
constexpr int STAGES = 4;
constexpr int A_TILE = BM * BK * 4;        // 16 KiB
constexpr int B_TILE = BK * BN * 4;        // 8 KiB (64 K-major rows of 128 B)
constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;
constexpr int THREADS = 192;
constexpr uint32_t TMEM_COLS = 64;

struct Smem {
  uint8_t a_hi[STAGES][A_TILE];
  uint8_t a_lo[STAGES][A_TILE];
  uint8_t b_hi[STAGES][B_TILE];
  uint8_t b_lo[STAGES][B_TILE];
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tmem_full;
  uint32_t tmem_base;
};
constexpr size_t SMEM_BYTES = sizeof(Smem) + 1024;  // + manual 1 KiB alignment

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void split_tf32_kernel(const float4 *__restrict__ x, float4 *__restrict__ hi, float4 *__restrict__ lo,
                                  long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = __ldg(x + i);
    float4 h, l;
    h.x = tf32_rna(v.x); l.x = tf32_rna(v.x - h.x);
    h.y = tf32_rna(v.y); l.y = tf32_rna(v.y - h.y);
    h.z = tf32_rna(v.z); l.z = tf32_rna(v.z - h.z);
    h.w = tf32_rna(v.w); l.w = tf32_rna(v.w - h.w);
    hi[i] = h;
    lo[i] = l;
  }
}

// B [K][N] -> Bt_hi, Bt_lo [N][K] (32x32 tiles through shared memory)
__global__ void split_tf32_transpose_kernel(const float *__restrict__ b, float *__restrict__ bt_hi,
                                            float *__restrict__ bt_lo, int K, int N) {
  __shared__ float t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  for (int r = ty; r < 32; r += 8) {
    const int k = k0 + r, nn = n0 + tx;
    t[r][tx] = (k < K && nn < N) ? __ldg(b + (size_t)k * N + nn) : 0.f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int nn = n0 + r, k = k0 + tx;
    if (nn < N && k < K) {
      const float v = t[tx][r];
      const float h = tf32_rna(v);
      bt_hi[(size_t)nn * K + k] = h;
      bt_lo[(size_t)nn * K + k] = tf32_rna(v - h);
    }
  }
}

__global__ void __launch_bounds__(THREADS, 1)
gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
                   const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_blo,
                   float *__restrict__ c, int M, int N, int K) {
  extern __shared__ uint8_t smem_raw[];
  Smem &S = *reinterpret_cast<Smem *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kblocks = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; s++) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.empty[s], 1);
    }
    tc::mbar_init(&S.tmem_full, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tm_ahi); tc::tma_prefetch(&tm_alo);
    tc::tma_prefetch(&tm_bhi); tc::tma_prefetch(&tm_blo);
  }
  if (warp == 1) tc::tmem_alloc<TMEM_COLS>(&S.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_d = S.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int kb = 0; kb < kblocks; kb++) {
        const int s = kb % STAGES;
        if (kb >= STAGES) tc::mbar_wait(&S.empty[s], ((kb / STAGES) - 1) & 1);
        tc::mbar_arrive_expect_tx(&S.full[s], STAGE_BYTES);
        const int k0 = kb * BK;
        tc::tma_load_2d(S.a_hi[s], &tm_ahi, &S.full[s], k0, m0);
        tc::tma_load_2d(S.a_lo[s], &tm_alo, &S.full[s], k0, m0);
        tc::tma_load_2d(S.b_hi[s], &tm_bhi, &S.full[s], k0, n0);
        tc::tma_load_2d(S.b_lo[s], &tm_blo, &S.full[s], k0, n0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = tc::idesc_tf32(BM, BN, /*a MN-major*/ 0, /*b MN-major*/ 0);
    for (int kb = 0; kb < kblocks; kb++) {
      const int s = kb % STAGES;
      tc::mbar_wait(&S.full[s], (kb / STAGES) & 1);
      tc::tc_fence_after();
      if (lane == 0) {
        const uint32_t ahi = tc::smem_u32(S.a_hi[s]), alo = tc::smem_u32(S.a_lo[s]);
        const uint32_t bhi = tc::smem_u32(S.b_hi[s]), blo = tc::smem_u32(S.b_lo[s]);
#pragma unroll
        for (int k = 0; k < BK / 8; k++) {
          // A and Bt: K-major, 128B rows, 8-row atoms of 1 KiB -> SBO = 1024;
          // one MMA consumes 8 fp32 of K = 32 bytes of each row.
          const uint64_t da_hi = tc::smem_desc_sw128(ahi + k * 32, 16, 1024);
          const uint64_t da_lo = tc::smem_desc_sw128(alo + k * 32, 16, 1024);
          const uint64_t db_hi = tc::smem_desc_sw128(bhi + k * 32, 16, 1024);
          const uint64_t db_lo = tc::smem_desc_sw128(blo + k * 32, 16, 1024);
          const uint32_t acc0 = (kb | k) != 0;
          tc::mma_tf32(tmem_d, da_hi, db_hi, idesc, acc0);
          tc::mma_tf32(tmem_d, da_hi, db_lo, idesc, 1);
          tc::mma_tf32(tmem_d, da_lo, db_hi, idesc, 1);
        }
        tc::mma_commit(&S.empty[s]);               // smem stage may be refilled
        if (kb == kblocks - 1) tc::mma_commit(&S.tmem_full);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------ epilogue
    tc::mbar_wait(&S.tmem_full, 0);
    tc::tc_fence_after();
    const int q = warp & 3;                 // TMEM lane quarter this warp may read
    const int row = m0 + q * 32 + lane;
#pragma unroll
    for (int cb = 0; cb < BN; cb += 16) {
      uint32_t r[16];
      tc::tmem_ld_32x32b_x16(tmem_d + ((uint32_t)(q * 32) << 16) + cb, r);
      tc::tmem_ld_wait();
      if (row < M) {
        float *dst = c + (size_t)row * N + n0 + cb;
        if (n0 + cb + 16 <= N && (N & 3) == 0) {
#pragma unroll
          for (int v = 0; v < 4; v++)
            reinterpret_cast<float4 *>(dst)[v] =
                make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                            __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
        } else {
          for (int v = 0; v < 16; v++)
            if (n0 + cb + v < N) dst[v] = __uint_as_float(r[v]);
        }
      }
    }
    tc::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<TMEM_COLS>(tmem_d);
  }
}

// exact SIMT path: the oracle's sequential k order with single roundings
__global__ void matmul_exact_kernel(const float *__restrict__ a, const float *__restrict__ b, float *__restrict__ c,
                                    int M, int N, int K) {
  __shared__ float As[32][33];
  __shared__ float Bs[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  const int col = blockIdx.x * 32 + tx;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      const int ar = blockIdx.y * 32 + r, ak = k0 + tx;
      As[r][tx] = (ar < M && ak < K) ? a[(size_t)ar * K + ak] : 0.f;
      const int bk = k0 + r;
      Bs[r][tx] = (bk < K && col < N) ? b[(size_t)bk * N + col] : 0.f;
    }
    __syncthreads();
    const int kmax = min(32, K - k0);
    for (int kk = 0; kk < kmax; kk++)
#pragma unroll
      for (int i = 0; i < 4; i++) acc[i] = add_rn(acc[i], mul_rn(As[ty + 8 * i][kk], Bs[kk][tx]));
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int row = blockIdx.y * 32 + ty + 8 * i;
    if (row < M && col < N) c[(size_t)row * N + col] = acc[i];
  }
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D fp32 tensor [rows][cols] (row pitch = cols), box {32 cols, box_rows}
static bool make_map(CUtensorMap *map, const void *base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace mm
}  // namespace jb

using namespace jb;
using namespace jb::mm;

extern "C" jb_status jb_matmul_f32(uint64_t n, uint64_t m, uint64_t l, const float *a, const float *b,
                                   float *res, void *stream) {
  JB_REQUIRE(n < (1ull << 31) && m < (1ull << 31) && l < (1ull << 31), "matmul: extents too large");
  if (n == 0 || l == 0) return JB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  JB_REQUIRE(res, "matmul: null result pointer");
  if (m == 0) {  // empty k-reduce: every element is the zero initialiser
    JB_CHECK_CUDA(cudaMemsetAsync(res, 0, n * l * 4, s));
    return JB_OK;
  }
  JB_REQUIRE(a && b, "matmul: null pointer");
  const bool tma_ok = (m % 4 == 0) && (l % 4 == 0) && ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0) &&
                      n >= 1 && mm::encode_fn() != nullptr;
  if (!tma_ok) {
    dim3 grid((unsigned)((l + 31) / 32), (unsigned)((n + 31) / 32));
    matmul_exact_kernel<<<grid, 256, 0, s>>>(a, b, res, (int)n, (int)l, (int)m);
    JB_LAUNCHED("matmul_exact");
    return JB_OK;
  }
  const size_t asz = n * m, bsz = m * l;
  char *ws = (char *)workspace((2 * asz + 2 * bsz) * 4 + 1024, s);
  if (!ws) return JB_ECUDA;
  float *a_hi = (float *)ws, *a_lo = a_hi + asz, *b_hi = a_lo + asz, *b_lo = b_hi + bsz;
  split_tf32_kernel<<<sm_count() * 4, 256, 0, s>>>((const float4 *)a, (float4 *)a_hi, (float4 *)a_lo,
                                                   (long long)(asz / 4));
  JB_LAUNCHED("matmul_split_a");
  split_tf32_transpose_kernel<<<dim3((unsigned)((l + 31) / 32), (unsigned)((m + 31) / 32)), 256, 0, s>>>(
      b, b_hi, b_lo, (int)m, (int)l);
  JB_LAUNCHED("matmul_split_b");

  CUtensorMap m_ahi, m_alo, m_bhi, m_blo;
  if (!make_map(&m_ahi, a_hi, n, m, BM) || !make_map(&m_alo, a_lo, n, m, BM) ||
      !make_map(&m_bhi, b_hi, l, m, BN) || !make_map(&m_blo, b_lo, l, m, BN)) {
    set_error("matmul: cuTensorMapEncodeTiled failed");
    return JB_ECUDA;
  }
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    JB_CHECK_CUDA(cudaFuncSetAttribute(gemm_3xtf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMEM_BYTES));
    attr_set[dev] = true;
  }
  dim3 grid((unsigned)((l + BN - 1) / BN), (unsigned)((n + BM - 1) / BM));
  void *tok = prof_begin("matmul_tcgen05", s);
  gemm_3xtf32_kernel<<<grid, THREADS, SMEM_BYTES, s>>>(m_ahi, m_alo, m_bhi, m_blo, res, (int)n, (int)l, (int)m);
  prof_end(tok, s);
  JB_LAUNCHED("matmul_tcgen05");
  return JB_OK;
}

// exact path exposed for tests and the bit-exact mode of the host API
extern "C" JB_API jb_status jb_matmul_exact_f32(uint64_t n, uint64_t m, uint64_t l, const float *a,
                                                const float *b, float *res, void *stream) {
  JB_REQUIRE(n < (1ull << 31) && m < (1ull << 31) && l < (1ull << 31), "matmul: extents too large");
  if (n == 0 || l == 0) return JB_OK;
  dim3 grid((unsigned)((l + 31) / 32), (unsigned)((n + 31) / 32));
  matmul_exact_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a, b, res, (int)n, (int)l, (int)m);
  JB_LAUNCHED("matmul_exact");
  return JB_OK;
}
