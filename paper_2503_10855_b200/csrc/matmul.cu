// matmul.cu -- matmul<n,m,l>(a: f32[n,m], b: f32[m,l]) -> f32[n,l] on sm_100a.
//
// Juno program: Fig. 1 of the paper, restated in
// oracle/juno_oracle.c:jo_matmul_f32 (res[i,j] += a[i,k]*b[k,j], k ascending).
// The k-reduce is a monoid add that the paper's schedules re-associate
// (monoid-reassociate), so the contract is fp32 tolerance:
//     |C - C_ref| <= (2*gamma_m + 8u) * (|A| |B|)   elementwise, u = 2^-24.
//
// B200 design: 3xTF32 on the 5th-gen tensor cores,
//   x_hi = trunc_tf32(x) (what kind::tf32 reads from an f32 container),
//   x_lo = x - x_hi (exact in f32),
//   D += A_hi*B_hi + A_hi*B_lo + A_lo*B_hi   (f32 accumulators in TMEM).
// One kernel, one 128x128 output tile per CTA, 320 threads:
//   warp 0     TMA producer: raw fp32 A tile (K-major, 128B swizzle) and raw
//              B tile (MN-major, 128B swizzle with 32-byte atoms = UMMA
//              layout SWIZZLE_128B_BASE32B) per 32-wide k-block into a
//              4-stage mbarrier ring.  Only raw operands cross L2 -> SMEM;
//              the raw tiles ARE the hi operands (the tensor core truncates
//              the 13 low bits, verified by tools/mma_probe.cu).
//   warps 2-9  converters: lo = x - trunc(x).  B_lo goes to a 2-slot smem
//              ring in B's swizzled layout; A_lo goes to TMEM (tcgen05.st,
//              thread = row of its lane quarter) and the lo*hi MMA reads A
//              from there (kind::tf32 with A in TMEM).  Shared memory, not
//              the tensor core, bounds this loop (per k-block 32 KiB TMA in,
//              converter reads and B_lo writes, three MMA operand reads at
//              ~128 B/clk): keeping A_lo out of it saves 32 KiB per k-block,
//              0.0293 -> 0.0276 ms per 1024^3 call.  Warps 2-5 then run the
//              epilogue (tcgen05.ld -> global).
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer.
// Split-K 2 when the tile count is below one wave: the two partials meet in
// C through f32 vector reductions onto zero (0 + p0 + p1 rounds the same in
// either order: deterministic).  Two designs that drop the memset were
// measured and lost: a CTA-pair kernel (cta_group::2,
// 256x256 pair tiles, split-K 4 through an L2 scratch; its main loop ran at
// the measured tensor peak but the 12 MB partial exchange cost more,
// 0.0303 ms per call) and store-then-add split-K ordered by a per-tile flag
// (the second split waits: 0.0309 ms).
// Shapes the TMA path cannot take (row pitch not a multiple of 16 bytes) run
// an exact SIMT kernel that follows the oracle's k order bit for bit.
#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "tcgen05.cuh"

#ifdef MM_TRACE
// per-CTA phase timestamps (globaltimer ns) for tools/mm_trace.py
__device__ unsigned long long g_mm_trace[512][12];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MM_CTA (blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z))
#define MM_T(slot) g_mm_trace[MM_CTA][slot] = gtimer()
#define MM_ACC_BEGIN unsigned long long _mm_t = gtimer()
#define MM_ACC(slot) g_mm_trace[MM_CTA][slot] += gtimer() - _mm_t
#else
#define MM_T(slot) do {} while (0)
#define MM_ACC_BEGIN do {} while (0)
#define MM_ACC(slot) do {} while (0)
#endif

namespace jb {
namespace mm {

#ifndef MM_BN
#define MM_BN 128
#endif
constexpr int BM = 128, BN = MM_BN, BK = 32;  // BK fp32 = one 128-byte swizzle row
constexpr int B_ATOM = BK * 32 * 4;           // one 32-column MN atom of B: 4 KiB
constexpr int STAGES = 4;                   // raw tiles (TMA ring, also the hi operands)
constexpr int LO_STAGES = 2;                // converted lo operands
constexpr int A_TILE = BM * BK * 4;         // 16 KiB
template <int BNT> constexpr int b_tile() { return BK * BNT * 4; }  // BNT/32 atoms
constexpr int THREADS = 320;
constexpr int CONVERTERS = 256;             // warps 2..9 (warps 2..5 also run the epilogue)
#ifndef MM1_A_SMEM
// A's residual lives in TMEM (columns 128 + 32*stage; written by tcgen05.st,
// read by the lo*hi MMA): 32 KiB less shared-memory traffic per k-block
#define MM1_A_TMEM 1
constexpr uint32_t TMEM_COLS = 256;
#else
#define MM1_A_TMEM 0
constexpr uint32_t TMEM_COLS = 128;
#endif
constexpr uint32_t ALO_COL1 = 128;

template <int BNT>
struct SmemT {
  // raw fp32 tiles straight from TMA; the tensor core reads them as the tf32
  // "hi" operands (it ignores the 13 low mantissa bits, tools/mma_probe.cu)
  uint8_t a_raw[STAGES][A_TILE];  // [128 m][32 k] K-major, 128B swizzle
  uint8_t b_raw[STAGES][b_tile<BNT>()];  // BNT/32 MN atoms x [32 k][32 n], 128B swizzle / 32B atoms
  uint8_t a_lo[LO_STAGES][A_TILE];  // x - trunc_tf32(x), same layouts
  uint8_t b_lo[LO_STAGES][b_tile<BNT>()];
  uint64_t full[STAGES];            // TMA -> converters
  uint64_t empty[STAGES];           // MMA -> TMA (raw slot free)
  uint64_t conv[LO_STAGES];         // converters -> MMA
  uint64_t lo_empty[LO_STAGES];     // MMA -> converters (lo slot free)
  uint64_t tmem_full;
  uint32_t tmem_base;
};
template <int BNT> constexpr size_t smem_bytes() { return sizeof(SmemT<BNT>) + 1024; }  // + manual 1 KiB alignment
static_assert(smem_bytes<128>() <= 232448, "shared memory budget");

// residual of the tensor core's tf32 truncation: exact in f32
__device__ __forceinline__ float tf32_residual(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ void red_add_v4(float *p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// MN-major B descriptor: 128B swizzle with 32-byte atoms (layout type 1),
// 32-column MN atoms B_ATOM apart (LBO), 4-row K groups 512 B apart (SBO)
__device__ __forceinline__ uint64_t desc_b_mn(uint32_t saddr) {
  const uint64_t d = tc::smem_desc_sw128(saddr, B_ATOM, 512);
  return (d & ~(7ull << 61)) | (1ull << 61);
}

// grid (N/BNT, M/128, splitk); blockIdx.z takes k-blocks [kb0, kb1).
// partials == nullptr: the z slices meet in c (plain stores for one slice,
// f32 reductions onto a zeroed c for two); otherwise slice z stores its
// partial tile to partials + z*M*N and a fixed-order fold sums them
// (mm_fold_kernel: the schedule's reduction tree, any slice count).
template <int BNT>
__global__ void __launch_bounds__(THREADS, 1)
gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                   float *__restrict__ c, int M, int N, int K, float *__restrict__ partials) {
  constexpr int BN = BNT, B_TILE = b_tile<BNT>();
  using Smem = SmemT<BNT>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1 KiB alignment by offsetting within the __shared__ array, so the compiler
  // keeps the shared address space (LDS/STS, not generic LD/ST)
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  Smem &S = *reinterpret_cast<Smem *>(smem_raw + pad);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kblocks = (K + BK - 1) / BK;
  const int splitk = gridDim.z;
  const int kb0 = (int)((long long)kblocks * blockIdx.z / splitk);
  const int kb1 = (int)((long long)kblocks * (blockIdx.z + 1) / splitk);
  const int nkb = kb1 - kb0;
  if (partials) c = partials + (size_t)blockIdx.z * M * N;
  const bool reduce_c = splitk > 1 && !partials;
  if (threadIdx.x == 0) MM_T(0);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; s++) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.empty[s], 1);
    }
    for (int s = 0; s < LO_STAGES; s++) {
      tc::mbar_init(&S.conv[s], CONVERTERS);
      tc::mbar_init(&S.lo_empty[s], 1);
    }
    tc::mbar_init(&S.tmem_full, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tm_a);
    tc::tma_prefetch(&tm_b);
  }
  if (warp == 1) tc::tmem_alloc<TMEM_COLS>(&S.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_d = S.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int j = 0; j < nkb; j++) {
        const int s = j % STAGES;
        {
          MM_ACC_BEGIN;
          if (j >= STAGES) tc::mbar_wait(&S.empty[s], ((j / STAGES) - 1) & 1);
          MM_ACC(10);
        }
        tc::mbar_arrive_expect_tx(&S.full[s], A_TILE + B_TILE);
        const int k0 = (kb0 + j) * BK;
        tc::tma_load_2d(S.a_raw[s], &tm_a, &S.full[s], k0, m0);
#pragma unroll
        for (int at = 0; at < BN / 32; at++)
          tc::tma_load_2d(S.b_raw[s] + at * B_ATOM, &tm_b, &S.full[s], n0 + 32 * at, k0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = tc::idesc_tf32(BM, BN, /*a MN-major*/ 0, /*b MN-major*/ 1);
    for (int j = 0; j < nkb; j++) {
      const int s = j % STAGES, ls = j % LO_STAGES;
      {
        MM_ACC_BEGIN;
        tc::mbar_wait(&S.conv[ls], (j / LO_STAGES) & 1);
        if (lane == 0 && j > 0) MM_ACC(6);
      }
      tc::tc_fence_after();
      if (lane == 0 && j == 0) MM_T(2);
      if (lane == 0) {
        const uint32_t ahi = tc::smem_u32(S.a_raw[s]), alo = tc::smem_u32(S.a_lo[ls]);
        const uint32_t bhi = tc::smem_u32(S.b_raw[s]), blo = tc::smem_u32(S.b_lo[ls]);
#pragma unroll
        for (int k = 0; k < BK / 8; k++) {
          // A: K-major, 128B rows in 1 KiB 8-row atoms (SBO 1024), one MMA
          //    consumes 32 bytes of each row.  B: MN-major, one MMA consumes
          //    8 K-rows = 1 KiB of every MN atom.
          const uint64_t da_hi = tc::smem_desc_sw128(ahi + k * 32, 16, 1024);
          const uint64_t da_lo = tc::smem_desc_sw128(alo + k * 32, 16, 1024);
          const uint64_t db_hi = desc_b_mn(bhi + k * 1024);
          const uint64_t db_lo = desc_b_mn(blo + k * 1024);
          const uint32_t acc0 = (j | k) != 0;
          tc::mma_tf32(tmem_d, da_hi, db_hi, idesc, acc0);
          tc::mma_tf32(tmem_d, da_hi, db_lo, idesc, 1);
#if MM1_A_TMEM
          (void)da_lo;
          tc::mma_tf32_ts(tmem_d, tmem_d + ALO_COL1 + ls * BK + k * 8, db_hi, idesc, 1);
#else
          tc::mma_tf32(tmem_d, da_lo, db_hi, idesc, 1);
#endif
        }
        tc::mma_commit(&S.empty[s]);      // raw slot may be refilled by TMA
        tc::mma_commit(&S.lo_empty[ls]);  // lo slot may be rewritten
        if (j == nkb - 1) {
          tc::mma_commit(&S.tmem_full);
          MM_T(3);
        }
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------ converters
    const int ct = threadIdx.x - 64;  // 0..255
    for (int j = 0; j < nkb; j++) {
      const int s = j % STAGES, ls = j % LO_STAGES;
      {
        MM_ACC_BEGIN;
        tc::mbar_wait(&S.full[s], (j / STAGES) & 1);
        if (ct == 0 && j > 0) MM_ACC(7);
      }
      if (j == 0 && ct == 0) MM_T(1);
      {
        MM_ACC_BEGIN;
        if (j >= LO_STAGES) tc::mbar_wait(&S.lo_empty[ls], ((j / LO_STAGES) - 1) & 1);
        if (ct == 0) MM_ACC(8);
      }
      MM_ACC_BEGIN;
      // elementwise, layout preserving: lo = x - trunc_tf32(x) for A and B
      const float4 *ar = reinterpret_cast<const float4 *>(S.a_raw[s]);
      const float4 *br = reinterpret_cast<const float4 *>(S.b_raw[s]);
      float4 *al = reinterpret_cast<float4 *>(S.a_lo[ls]);
      float4 *bl = reinterpret_cast<float4 *>(S.b_lo[ls]);
      float4 vb[B_TILE / 16 / CONVERTERS];
#if MM1_A_TMEM
      // A: thread = row 32q + lane of its TMEM lane quarter (warps 2..9:
      // q = warp & 3, two warps per quarter take k chunks 4h..4h+3 of the
      // 128B-swizzled row; chunk c sits at c ^ (row & 7))
      const int rq = warp & 3, hh = (warp - 2) >> 2, ra = rq * 32 + lane;
      float4 va[4];
#pragma unroll
      for (int i = 0; i < 4; i++)
        va[i] = *reinterpret_cast<const float4 *>(S.a_raw[s] + ra * 128 + (((4 * hh + i) ^ (ra & 7)) << 4));
      (void)ar;
      (void)al;
#else
      float4 va[A_TILE / 16 / CONVERTERS];
#pragma unroll
      for (int i = 0; i < A_TILE / 16 / CONVERTERS; i++) va[i] = ar[ct + i * CONVERTERS];
#endif
#pragma unroll
      for (int i = 0; i < B_TILE / 16 / CONVERTERS; i++) vb[i] = br[ct + i * CONVERTERS];
#if MM1_A_TMEM
      {
        uint32_t lo[16];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          lo[4 * i] = __float_as_uint(tf32_residual(va[i].x));
          lo[4 * i + 1] = __float_as_uint(tf32_residual(va[i].y));
          lo[4 * i + 2] = __float_as_uint(tf32_residual(va[i].z));
          lo[4 * i + 3] = __float_as_uint(tf32_residual(va[i].w));
        }
        tc::tmem_st_32x32b_x16(tmem_d + ((uint32_t)(rq * 32) << 16) + ALO_COL1 + ls * BK + 16 * hh, lo);
      }
#else
#pragma unroll
      for (int i = 0; i < A_TILE / 16 / CONVERTERS; i++)
        al[ct + i * CONVERTERS] = make_float4(tf32_residual(va[i].x), tf32_residual(va[i].y),
                                              tf32_residual(va[i].z), tf32_residual(va[i].w));
#endif
#pragma unroll
      for (int i = 0; i < B_TILE / 16 / CONVERTERS; i++)
        bl[ct + i * CONVERTERS] = make_float4(tf32_residual(vb[i].x), tf32_residual(vb[i].y),
                                              tf32_residual(vb[i].z), tf32_residual(vb[i].w));
      tc::fence_proxy_async_smem();  // generic-proxy writes -> tensor core
#if MM1_A_TMEM
      tc::tmem_st_wait();
      tc::tc_fence_before();
#endif
      tc::mbar_arrive(&S.conv[ls]);
      if (ct == 0) MM_ACC(9);
    }
    // ------------------------------------------------------ epilogue
    if (warp >= 6 || nkb == 0) goto done;  // four warps cover the 128 TMEM lanes
    tc::mbar_wait(&S.tmem_full, 0);
    tc::tc_fence_after();
    if (ct == 0) MM_T(4);
    {
      const int q = warp & 3;  // TMEM lane quarter this warp may read
      const int row = m0 + q * 32 + lane;
      const bool vec = (N & 3) == 0;
#pragma unroll 1
      for (int cb = 0; cb < BN; cb += 16) {
        uint32_t r[16];
        tc::tmem_ld_32x32b_x16(tmem_d + ((uint32_t)(q * 32) << 16) + cb, r);
        tc::tmem_ld_wait();
        if (row < M) {
          float *dst = c + (size_t)row * N + n0 + cb;
          if (n0 + cb + 16 <= N && vec) {
#pragma unroll
            for (int v = 0; v < 4; v++) {
              const float a0 = __uint_as_float(r[4 * v]), a1 = __uint_as_float(r[4 * v + 1]);
              const float a2 = __uint_as_float(r[4 * v + 2]), a3 = __uint_as_float(r[4 * v + 3]);
              if (reduce_c)
                red_add_v4(dst + 4 * v, a0, a1, a2, a3);
              else
                reinterpret_cast<float4 *>(dst)[v] = make_float4(a0, a1, a2, a3);
            }
          } else {
            for (int v = 0; v < 16; v++)
              if (n0 + cb + v < N) {
                if (reduce_c)
                  atomicAdd(dst + v, __uint_as_float(r[v]));
                else
                  dst[v] = __uint_as_float(r[v]);
              }
          }
        }
      }
    }
    tc::tc_fence_before();
    if (ct == 0) MM_T(5);
  }
done:
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<TMEM_COLS>(tmem_d);
  }
}


// res = fold of the partial tiles in the reduction tree's order: counts
// (n1, n2) = partials per level, outermost first (n2 = 1 for one fission):
//   res = 0 + sum_{p1 < n1} (0 + sum_{p2 < n2} part[p1 * n2 + p2])
// (fork-fission's bottom fold over the partials array, passes/fissfuse.py
// :134-145; the second level is reduction_tree! applied to that fold)
__global__ void mm_fold_kernel(const float *__restrict__ part, float *__restrict__ res, long long mn, int n1,
                               int n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < mn;
       i += (long long)gridDim.x * blockDim.x) {
    float r = 0.0f;
    for (int p1 = 0; p1 < n1; p1++) {
      float t = 0.0f;
      for (int p2 = 0; p2 < n2; p2++) t = add_rn(t, __ldcs(part + (size_t)(p1 * n2 + p2) * mn + i));
      r = add_rn(r, t);
    }
    res[i] = r;
  }
}

// exact SIMT path: the oracle's sequential k order with single roundings,
// over k in [k_lo, k_lo + K) of the K_stride-wide operands (a partial sum of
// a reduction tree, or the whole product)
__global__ void matmul_exact_range_kernel(const float *__restrict__ a, const float *__restrict__ b,
                                          float *__restrict__ c, int M, int N, int K, int K_stride, int k_lo) {
  a += k_lo;
  b += (size_t)k_lo * N;
  __shared__ float As[32][33];
  __shared__ float Bs[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  const int col = blockIdx.x * 32 + tx;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      const int ar = blockIdx.y * 32 + r, ak = k0 + tx;
      As[r][tx] = (ar < M && ak < K) ? a[(size_t)ar * K_stride + ak] : 0.f;
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
// 2-D fp32 tensor [rows][cols] (row pitch = cols), box {box_cols, box_rows}
static bool make_map(CUtensorMap *map, const void *base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                     uint32_t box_rows, CUtensorMapSwizzle swz) {
  const uint64_t dims[2] = {cols, rows};
  const uint64_t strides[1] = {cols * 4};
  const uint32_t box[2] = {box_cols, box_rows};
  return make_tmap_f32(map, base, 2, dims, strides, box, (int)swz);
}

}  // namespace mm
}  // namespace jb

using namespace jb;
using namespace jb::mm;

#ifdef MM_TRACE
extern "C" JB_API void jb_mm_trace(unsigned long long *out) {
  cudaMemcpyFromSymbol(out, g_mm_trace, sizeof(g_mm_trace));
}
#endif

extern "C" jb_status jb_matmul_exact_f32(uint64_t n, uint64_t m, uint64_t l, const float *a, const float *b,
                                         float *res, void *stream) {
  JB_REQUIRE(n < (1ull << 31) && m < (1ull << 31) && l < (1ull << 31), "matmul: extents too large");
  if (n == 0 || l == 0) return JB_OK;
  JB_REQUIRE(res && (m == 0 || (a && b)), "matmul: null pointer");
  dim3 grid((unsigned)((l + 31) / 32), (unsigned)((n + 31) / 32));
  matmul_exact_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a, b, res, (int)n, (int)l, (int)m);
  JB_LAUNCHED("matmul_exact");
  return JB_OK;
}

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
  // the epilogue stores res with 16-byte vector stores / reductions
  const bool tma_ok = (m % 4 == 0) && (l % 4 == 0) && ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0) &&
                      ((uintptr_t)res % 16 == 0) && tmap_encode_fn() != nullptr;
  if (!tma_ok) return jb_matmul_exact_f32(n, m, l, a, b, res, stream);

  // tensor maps are encoded on the host (~microseconds each): keep the last
  // pair per device, keyed by operand pointers and extents
  struct MapCache {
    const void *a, *b;
    uint64_t n, m, l;
    CUtensorMap ma, mb;
    bool valid;
  };
  static MapCache cache[64] = {};
  // the caches below are per device and shared by host threads: one lock
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  int cdev = 0;
  cudaGetDevice(&cdev);
  JB_REQUIRE(cdev >= 0 && cdev < 64, "matmul: device index out of range");
  MapCache &mc = cache[cdev];
  if (!(mc.valid && mc.a == a && mc.b == b && mc.n == n && mc.m == m && mc.l == l)) {
    mc.valid = false;
    if (!make_map(&mc.ma, a, n, m, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_map(&mc.mb, b, m, l, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
      set_error("matmul: cuTensorMapEncodeTiled failed");
      return JB_ECUDA;
    }
    mc.a = a; mc.b = b; mc.n = n; mc.m = m; mc.l = l;
    mc.valid = true;
  }
  const CUtensorMap &m_a = mc.ma, &m_b = mc.mb;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    JB_CHECK_CUDA(cudaFuncSetAttribute(gemm_3xtf32_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_bytes<BN>()));
    attr_set[dev] = true;
  }
  const long long tiles = (long long)((l + BN - 1) / BN) * (long long)((n + BM - 1) / BM);
  const int kblocks = (int)((m + BK - 1) / BK);
  // split K in two when that still fits one CTA per SM; the partial tiles
  // meet in C through f32 vector reductions onto zero.  Two addends only:
  // 0 + p0 + p1 rounds the same in either order, so the result is
  // deterministic run to run (more slices would make it depend on the order
  // the reductions land)
  int splitk = 1;
  if (tiles * 2 <= sm_count() && kblocks >= 8) splitk = 2;
  dim3 grid((unsigned)((l + BN - 1) / BN), (unsigned)((n + BM - 1) / BM), (unsigned)splitk);

  // A call that repeats the previous call's operands and extents on this
  // device (a runner, a benchmark loop, the caching allocator handing back
  // the same result block) replays a CUDA graph of memset + GEMM captured on
  // the repeat: one launch, and the memset -> GEMM dependency resolved on the
  // device (0.025 instead of 0.035 ms per 1024^3 call).  New operands take
  // the plain launches; the graph is rebuilt when they repeat.
  struct GraphCache {
    const void *a, *b, *c;
    uint64_t n, m, l;
    cudaGraphExec_t exec;
    bool failed;  // capture/instantiate failed for this key: plain launches
  };
  static GraphCache gcache[64] = {};
  static cudaStream_t cap_stream[64] = {};
  GraphCache &gc = gcache[cdev];
  const bool repeat = gc.a == a && gc.b == b && gc.c == res && gc.n == n && gc.m == m && gc.l == l;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  JB_CHECK_CUDA(cudaStreamIsCapturing(s, &cap));
  // never consume an error the caller has not seen yet: only capture with a
  // clean error state, and clear only what the capture itself raised
  if (repeat && !gc.exec && !gc.failed && cap == cudaStreamCaptureStatusNone &&
      cudaPeekAtLastError() == cudaSuccess) {
    if (!cap_stream[cdev]) JB_CHECK_CUDA(cudaStreamCreateWithFlags(&cap_stream[cdev], cudaStreamNonBlocking));
    cudaStream_t cs = cap_stream[cdev];
    cudaGraph_t graph = nullptr;
    JB_CHECK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    if (splitk > 1) cudaMemsetAsync(res, 0, n * l * 4, cs);
    gemm_3xtf32_kernel<BN><<<grid, THREADS, smem_bytes<BN>(), cs>>>(m_a, m_b, res, (int)n, (int)l, (int)m, nullptr);
    const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
    if (ce == cudaSuccess && graph) {
      if (cudaGraphInstantiate(&gc.exec, graph, 0) != cudaSuccess) gc.exec = nullptr;
      cudaGraphDestroy(graph);
    }
    if (!gc.exec) {
      gc.failed = true;    // a failed capture falls back to plain launches, once
      cudaGetLastError();
    }
  }
  if (repeat && gc.exec && cap == cudaStreamCaptureStatusNone) {  // (a caller's capture records plain launches)
    void *tok = prof_begin("matmul_tcgen05", s);
    JB_CHECK_CUDA(cudaGraphLaunch(gc.exec, s));
    prof_end(tok, s);
    JB_LAUNCHED("matmul_tcgen05");
    return JB_OK;
  }
  if (!repeat) {
    if (gc.exec) cudaGraphExecDestroy(gc.exec);
    gc = GraphCache{a, b, res, n, m, l, nullptr, false};
  }
  if (splitk > 1) JB_CHECK_CUDA(cudaMemsetAsync(res, 0, n * l * 4, s));
  void *tok = prof_begin("matmul_tcgen05", s);
  gemm_3xtf32_kernel<BN><<<grid, THREADS, smem_bytes<BN>(), s>>>(m_a, m_b, res, (int)n, (int)l, (int)m, nullptr);
  prof_end(tok, s);
  JB_LAUNCHED("matmul_tcgen05");
  return JB_OK;
}

// ------------------------------------------------- schedule-parametrised entry
// The launch a scheduled matmul asks for (planner.select_kernel):
//   tile_n   the CTA's output tile width from the J fork's fork-tile factor
//            (64 or 128 columns; the tcgen05 tile is 128 rows: M = 128 is
//            the single-CTA MMA atom);
//   n1, n2   the reduction tree of fork-fission (reduction_tree!): n1 * n2
//            contiguous K chunks, each a partial product (3xTF32 on the
//            tensor cores when the chunk is a whole number of 32-wide
//            k-blocks and the operands suit TMA, else the exact SIMT kernel),
//            folded in the tree's order by mm_fold_kernel.
// n1 * n2 == 1 is the plain entry (its own split heuristics).
namespace jb {
namespace mm {
template <int BNT>
static jb_status launch_partials(const CUtensorMap &ma, const CUtensorMap &mb, float *part, uint64_t n,
                                 uint64_t m, uint64_t l, int parts, cudaStream_t s) {
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    JB_CHECK_CUDA(cudaFuncSetAttribute(gemm_3xtf32_kernel<BNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_bytes<BNT>()));
    attr_set[dev] = true;
  }
  dim3 grid((unsigned)((l + BNT - 1) / BNT), (unsigned)((n + BM - 1) / BM), (unsigned)parts);
  void *tok = prof_begin("matmul_tcgen05", s);
  gemm_3xtf32_kernel<BNT><<<grid, THREADS, smem_bytes<BNT>(), s>>>(ma, mb, part, (int)n, (int)l, (int)m, part);
  prof_end(tok, s);
  JB_LAUNCHED("matmul_tcgen05");
  return JB_OK;
}
}  // namespace mm
}  // namespace jb

extern "C" jb_status jb_matmul_sched_f32(uint64_t n, uint64_t m, uint64_t l, const float *a, const float *b,
                                         float *res, uint32_t tile_n, uint32_t n1, uint32_t n2, void *stream) {
  JB_REQUIRE(n < (1ull << 31) && m < (1ull << 31) && l < (1ull << 31), "matmul: extents too large");
  JB_REQUIRE(tile_n == 64 || tile_n == 128, "matmul: tile_n must be 64 or 128 (got %u)", tile_n);
  JB_REQUIRE(n1 >= 1 && n2 >= 1 && (uint64_t)n1 * n2 <= 4096, "matmul: bad reduction tree %u x %u", n1, n2);
  const uint64_t parts = (uint64_t)n1 * n2;
  JB_REQUIRE(m % parts == 0, "matmul: %llu partials do not divide m = %llu (the schedule's constraint)",
             (unsigned long long)parts, (unsigned long long)m);
  if (parts == 1 && tile_n == 128) return jb_matmul_f32(n, m, l, a, b, res, stream);
  if (n == 0 || l == 0) return JB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  JB_REQUIRE(res, "matmul: null result pointer");
  if (m == 0) {
    JB_CHECK_CUDA(cudaMemsetAsync(res, 0, n * l * 4, s));
    return JB_OK;
  }
  JB_REQUIRE(a && b, "matmul: null pointer");
  const uint64_t chunk = m / parts;
  const uint64_t mn = n * l;
  float *part = (float *)workspace(parts * mn * 4, s);
  if (!part) return JB_ECUDA;
  const bool tma_ok = (m % 4 == 0) && (l % 4 == 0) && chunk % BK == 0 && ((uintptr_t)a % 16 == 0) &&
                      ((uintptr_t)b % 16 == 0) && tmap_encode_fn() != nullptr;
  CUtensorMap ma, mb;
  if (tma_ok && make_map(&ma, a, n, m, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B) &&
      make_map(&mb, b, m, l, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
    jb_status st = tile_n == 64 ? launch_partials<64>(ma, mb, part, n, m, l, (int)parts, s)
                                : launch_partials<128>(ma, mb, part, n, m, l, (int)parts, s);
    if (st != JB_OK) return st;
  } else {
    dim3 grid((unsigned)((l + 31) / 32), (unsigned)((n + 31) / 32));
    for (uint64_t p = 0; p < parts; p++) {
      matmul_exact_range_kernel<<<grid, 256, 0, s>>>(a, b, part + p * mn, (int)n, (int)l, (int)chunk, (int)m,
                                                     (int)(p * chunk));
      JB_LAUNCHED("matmul_exact_range");
    }
  }
  const long long blocks = std::min<long long>((long long)(mn + 255) / 256, (long long)sm_count() * 8);
  mm_fold_kernel<<<(unsigned)blocks, 256, 0, s>>>(part, res, (long long)mn, (int)n1, (int)n2);
  JB_LAUNCHED("matmul_fold");
  return JB_OK;
}
