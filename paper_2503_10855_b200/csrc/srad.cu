// srad.cu -- srad<rows,cols>(niter, lambda, image) on sm_100a (Rodinia srad_v1).
//
// Restated in oracle/juno_oracle.c:jo_srad_f32 / jo_srad_iter / jo_srad_q0sqr:
//   J = exp(I/255)
//   per iteration: q0^2 = var/mean^2 from f64 sums of J and J^2
//                  c    = clamp01(1 / (1 + (qsqr - q0^2)/(q0^2 (1 + q0^2))))
//                         from the 4 clamped neighbour differences
//                  J   += (lambda/4) * (c dN + c_S dS + c dW + c_E dE)
//   out = log(J) * 255
// The per-iteration statistics are the one associative reduction (a Fig. 10
// reduction tree in the paper's schedule); the two passes
// over the image are the loops `fork-fuse` merges (fissfuse.py:232-348).
//
// B200 design: one persistent kernel per iteration.
//  * A CTA owns a 32x128 tile: it stages the clamped J tile + halo
//    (35x131) in shared memory, computes c on the 33x129 region the update
//    needs (halo-1 recompute instead of a second pass over HBM), updates J
//    into the ping-pong buffer and folds sum(J'), sum(J'^2) in f64.
//  * The last CTA to finish (atomic ticket) reduces the per-CTA partials in a
//    fixed order and writes q0^2 for the next iteration: no host round trip,
//    deterministic for a given grid.
//  * HBM traffic: ~8.3 B/px per iteration (read J + halo, write J').
//  * extract is fused with the first statistics; compress is fused into the
//    last iteration's update.
// Arithmetic follows the oracle operation by operation with single-rounding
// ops (-fmad=false, IEEE division), so results are bit-identical whenever
// the f64 statistics round to the same f32 q0^2 (always observed) and the
// double-precision exp/log round to the same f32.
#include "common.cuh"

namespace jb {
namespace srad {

constexpr int TH = 32, TW = 128;
constexpr int JR = TH + 3, JC = TW + 3;     // J region rows/cols (halo N1 S2, W1 E2)
constexpr int JP = 132;                     // J row pitch
constexpr int CR = TH + 1;                  // c region rows (own + south row; cols: own + east)
constexpr int THREADS = 256;

struct Stats {
  double s, s2;
};

struct Args {
  const float *src;   // J (or the raw image when extracting)
  float *dst;         // J' (or the final log-compressed output)
  const float *q0;    // q0sqr[it] (device), null when extracting
  float *q0_next;     // where the last CTA writes q0sqr[it+1] (null: none)
  Stats *partials;    // [gridDim.x]
  unsigned *ticket;
  int rows, cols, tiles_x, tiles;
  int row_lo, row_hi; // output rows [row_lo, row_hi) of src (slab mode: the rest is halo)
  float ql;           // 0.25f * lambda
  int compress;       // write log(J')*255 instead of J'
  double *sums_out;   // slab mode: the last CTA writes (sum, sum2) here instead of q0
};

__device__ __forceinline__ void block_stats(double s, double s2, Stats *out) {
  __shared__ double sh[2][THREADS / 32];
  s = warp_sum(s);
  s2 = warp_sum(s2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sh[0][warp] = s; sh[1][warp] = s2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < THREADS / 32; w++) { a += sh[0][w]; b += sh[1][w]; }
    out->s = a;
    out->s2 = b;
  }
}

// last CTA of the grid: fixed-order f64 reduction of the partials -> q0^2
__device__ void finish_stats(const Args &a, long long npx) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    double s = 0.0, s2 = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) {
      const volatile Stats *p = a.partials + i;
      s += p->s;
      s2 += p->s2;
    }
    s = warp_sum(s);
    s2 = warp_sum(s2);
    if (threadIdx.x == 0) {
      if (a.sums_out) {  // multi-GPU slab: the q0 comes after the allreduce
        a.sums_out[0] = s;
        a.sums_out[1] = s2;
      } else {
        const double mean = s / (double)npx;
        const double var = s2 / (double)npx - mean * mean;
        *a.q0_next = (float)(var / (mean * mean));
      }
      *a.ticket = 0;  // ready for the next launch (stream order)
    }
  }
}

__global__ void __launch_bounds__(THREADS) srad_extract_kernel(Args a) {
  double s = 0.0, s2 = 0.0;
  const long long n = (long long)a.rows * a.cols;
  for (long long i = blockIdx.x * (long long)THREADS + threadIdx.x; i < n; i += (long long)gridDim.x * THREADS) {
    const float j = exp_ref(div_rn(__ldg(a.src + i), 255.0f));
    if (a.compress) {
      a.dst[i] = mul_rn(log_ref(j), 255.0f);  // niter == 0
    } else {
      a.dst[i] = j;
      s += (double)j;
      s2 += (double)j * (double)j;
    }
  }
  if (a.compress) return;
  block_stats(s, s2, a.partials + blockIdx.x);
  finish_stats(a, n);
}

struct Smem {
  float J[JR][JP];
  float c[CR][JP];
};

// c at image position (gy, gx) from the replicated J tile (tile origin y0,x0).
// The replicated halo reproduces the oracle's clamped neighbour indices
// (iN[0] = 0, iS[rows-1] = rows-1, ...): a clamped neighbour equals the centre.
__device__ __forceinline__ float coef(const Smem &S, int jr, int jc, float q0, float q0den) {
  const float Jc = S.J[jr][jc];
  const float n_ = sub_rn(S.J[jr - 1][jc], Jc);
  const float s_ = sub_rn(S.J[jr + 1][jc], Jc);
  const float w_ = sub_rn(S.J[jr][jc - 1], Jc);
  const float e_ = sub_rn(S.J[jr][jc + 1], Jc);
  const float G2 =
      div_rn(add_rn(add_rn(add_rn(mul_rn(n_, n_), mul_rn(s_, s_)), mul_rn(w_, w_)), mul_rn(e_, e_)), mul_rn(Jc, Jc));
  const float L = div_rn(add_rn(add_rn(add_rn(n_, s_), w_), e_), Jc);
  const float num = sub_rn(mul_rn(0.5f, G2), mul_rn(0.0625f, mul_rn(L, L)));
  const float den = add_rn(1.0f, mul_rn(0.25f, L));
  const float qsqr = div_rn(num, mul_rn(den, den));
  const float den2 = div_rn(sub_rn(qsqr, q0), q0den);
  const float cv = div_rn(1.0f, add_rn(1.0f, den2));
  return cv < 0.0f ? 0.0f : (cv > 1.0f ? 1.0f : cv);
}

__global__ void __launch_bounds__(THREADS) srad_iter_kernel(Args a) {
  __shared__ Smem S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = a.rows, cols = a.cols;
  const float q0 = *a.q0;
  const float q0den = mul_rn(q0, add_rn(1.0f, q0));
  double s = 0.0, s2 = 0.0;

  for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
    const int ty = t / a.tiles_x, tx = t - ty * a.tiles_x;
    const int y0 = a.row_lo + ty * TH, x0 = tx * TW;
    // ---- J tile with replicated halo: rows y0-1..y0+TH+1, cols x0-1..x0+TW+1.
    // warp w loads rows w, w+8, ...; lane l loads cols l, l+32, ... (loads first)
    {
      constexpr int RPW = (JR + 7) / 8;  // 5
      float v[RPW][5];
#pragma unroll
      for (int i = 0; i < RPW; i++) {
        const int r = min(warp + 8 * i, JR - 1);
        const float *row = a.src + (size_t)min(max(y0 - 1 + r, 0), rows - 1) * cols;
#pragma unroll
        for (int q = 0; q < 5; q++) {
          const int cc = min(32 * q + lane, JC - 1);
          v[i][q] = __ldg(row + min(max(x0 - 1 + cc, 0), cols - 1));
        }
      }
#pragma unroll
      for (int i = 0; i < RPW; i++) {
        const int r = warp + 8 * i;
#pragma unroll
        for (int q = 0; q < 5; q++) {
          const int cc = 32 * q + lane;
          if (r < JR && cc < JC) S.J[r][cc] = v[i][q];
        }
      }
    }
    __syncthreads();
    // ---- diffusion coefficient on rows y0..y0+TH, cols x0..x0+TW.  A
    // position past the image edge gets the coefficient of the clamped
    // position, which is exactly what the oracle's c[iS[i]] / c[jE[j]] read.
#pragma unroll 1
    for (int r = warp; r < CR; r += 8) {
      const int jr = min(y0 + r, rows - 1) - y0 + 1;
#pragma unroll
      for (int q = 0; q < TW / 32; q++) {  // the tile's own 128 columns
        const int cc = 32 * q + lane;
        const int jc = min(x0 + cc, cols - 1) - x0 + 1;
        S.c[r][cc] = coef(S, jr, jc, q0, q0den);
      }
    }
    if (tid < CR) {  // the east halo column (cc = TW), one row per thread
      const int r = tid;
      const int jr = min(y0 + r, rows - 1) - y0 + 1;
      const int jc = min(x0 + TW, cols - 1) - x0 + 1;
      S.c[r][TW] = coef(S, jr, jc, q0, q0den);
    }
    __syncthreads();
    // ---- update J' = J + ql * D on the tile: warp w rows 4w..4w+3, lane
    // columns l, l+32, l+64, l+96
#pragma unroll
    for (int k = 0; k < TH / 8; k++) {
      const int r = warp * (TH / 8) + k, gy = y0 + r;
      if (gy >= a.row_hi) break;
      const int jr = r + 1;
#pragma unroll
      for (int q = 0; q < TW / 32; q++) {
        const int cc = 32 * q + lane, gx = x0 + cc;
        if (gx < cols) {
          const int jc = cc + 1;
          const float Jc = S.J[jr][jc];
          const float n_ = sub_rn(S.J[jr - 1][jc], Jc);
          const float s_ = sub_rn(S.J[jr + 1][jc], Jc);
          const float w_ = sub_rn(S.J[jr][jc - 1], Jc);
          const float e_ = sub_rn(S.J[jr][jc + 1], Jc);
          const float cN = S.c[r][cc], cS = S.c[r + 1][cc], cE = S.c[r][cc + 1];
          const float D = add_rn(add_rn(add_rn(mul_rn(cN, n_), mul_rn(cS, s_)), mul_rn(cN, w_)), mul_rn(cE, e_));
          const float jn = add_rn(Jc, mul_rn(a.ql, D));
          const size_t o = (size_t)(gy - a.row_lo) * cols + gx;
          if (a.compress) {
            a.dst[o] = mul_rn(log_ref(jn), 255.0f);
          } else {
            a.dst[o] = jn;
            s += (double)jn;
            s2 += (double)jn * (double)jn;
          }
        }
      }
    }
    __syncthreads();  // S.J / S.c are rewritten by the next tile
  }
  if (a.compress) return;
  block_stats(s, s2, a.partials + blockIdx.x);
  finish_stats(a, (long long)(a.row_hi - a.row_lo) * cols);
}

__global__ void copy_q0_kernel(const float *q0, float *out, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = q0[i];
}

}  // namespace srad
}  // namespace jb

using namespace jb;
using namespace jb::srad;

extern "C" jb_status jb_srad_f32(uint64_t rows, uint64_t cols, uint64_t niter, float lambda, const float *image,
                                 float *out, float *q0sqr, void *stream) {
  JB_REQUIRE(rows >= 1 && cols >= 1, "srad: rows and cols must be >= 1");
  JB_REQUIRE(rows * cols < (1ull << 40) && rows < (1u << 30) && cols < (1u << 30), "srad: image too large");
  JB_REQUIRE(niter < (1u << 30), "srad: niter too large");
  JB_REQUIRE(image && out, "srad: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t npx = rows * cols;
  const int tiles_x = (int)((cols + TW - 1) / TW), tiles_y = (int)((rows + TH - 1) / TH);
  const int tiles = tiles_x * tiles_y;
  int per_sm = 0;
  JB_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, srad_iter_kernel, THREADS, 0));
  if (per_sm < 1) per_sm = 1;
  const int grid = tiles < sm_count() * per_sm ? tiles : sm_count() * per_sm;
  const int grid_x = sm_count() * 8;
  const int gmax = grid > grid_x ? grid : grid_x;
  // scratch: J ping-pong (2 images), q0 per iteration, partials, ticket
  const size_t img_bytes = ((npx * 4 + 255) / 256) * 256;
  const size_t q0_bytes = (((niter + 1) * 4 + 255) / 256) * 256;
  const size_t part_bytes = ((gmax * sizeof(Stats) + 255) / 256) * 256;
  char *ws = (char *)workspace(2 * img_bytes + q0_bytes + part_bytes + 256, s);
  if (!ws) return JB_ECUDA;
  float *J[2] = {(float *)ws, (float *)(ws + img_bytes)};
  float *q0 = (float *)(ws + 2 * img_bytes);
  Stats *parts = (Stats *)(ws + 2 * img_bytes + q0_bytes);
  unsigned *ticket = (unsigned *)(ws + 2 * img_bytes + q0_bytes + part_bytes);
  JB_CHECK_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));

  Args a{};
  a.rows = (int)rows; a.cols = (int)cols; a.tiles_x = tiles_x; a.tiles = tiles;
  a.row_lo = 0; a.row_hi = (int)rows; a.sums_out = nullptr;
  a.ql = 0.25f * lambda;  // one IEEE multiply, as in the oracle
  a.partials = parts; a.ticket = ticket;
  // extract (+ stats of J0), or extract+compress when niter == 0
  a.src = image;
  a.dst = niter ? J[0] : out;
  a.q0 = nullptr;
  a.q0_next = q0;
  a.compress = niter == 0;
  srad_extract_kernel<<<grid_x, THREADS, 0, s>>>(a);
  JB_LAUNCHED("srad_extract");
  for (uint64_t it = 0; it < niter; it++) {
    const bool last = it + 1 == niter;
    a.src = J[it & 1];
    a.dst = last ? out : J[(it + 1) & 1];
    a.q0 = q0 + it;
    a.q0_next = q0 + it + 1;
    a.compress = last;
    void *tok = prof_begin("srad_iter", s);
    srad_iter_kernel<<<grid, THREADS, 0, s>>>(a);
    prof_end(tok, s);
    JB_LAUNCHED("srad_iter");
  }
  if (q0sqr && niter) {
    copy_q0_kernel<<<1, 256, 0, s>>>(q0, q0sqr, (int)niter);
    JB_LAUNCHED("srad_q0_copy");
  }
  return JB_OK;
}

// ------------------------------------------------------------ slab entries
// Multi-GPU row slabs (paper_2503_10855_b200/dist.py): each rank owns rows
// [own_lo, own_hi) of an extended slab that carries 1 halo row above and 2
// below (fewer at the image edges); the host exchanges halos and allreduces
// the f64 sums between iterations, then jb_srad_q0_f32 turns them into q0^2.

__global__ void srad_q0_kernel(const double *sums, double npx, float *q0) {
  const double mean = sums[0] / npx;
  const double var = sums[1] / npx - mean * mean;
  *q0 = (float)(var / (mean * mean));
}

extern "C" jb_status jb_srad_extract_f32(uint64_t n, const float *image, float *J, double *sums,
                                         int compress, void *stream) {
  JB_REQUIRE(n >= 1 && n < (1ull << 40), "srad_extract: bad size");
  JB_REQUIRE(image && J, "srad_extract: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = sm_count() * 8;
  char *ws = (char *)workspace(((grid * sizeof(Stats) + 255) / 256) * 256 + 256, s);
  if (!ws) return JB_ECUDA;
  Args a{};
  a.src = image; a.dst = J; a.rows = 1; a.cols = (int)n;
  a.partials = (Stats *)ws;
  a.ticket = (unsigned *)(ws + ((grid * sizeof(Stats) + 255) / 256) * 256);
  a.compress = compress;
  a.sums_out = sums;
  a.q0_next = nullptr;
  JB_CHECK_CUDA(cudaMemsetAsync(a.ticket, 0, sizeof(unsigned), s));
  // extract kernel indexes rows*cols elements as a flat array
  a.rows = 1;
  srad_extract_kernel<<<grid, THREADS, 0, s>>>(a);
  JB_LAUNCHED("srad_extract");
  return JB_OK;
}

extern "C" jb_status jb_srad_slab_step_f32(uint64_t rows_ext, uint64_t cols, uint64_t own_lo, uint64_t own_hi,
                                           const float *J_ext, float *out_own, const float *q0, float lambda,
                                           double *sums, int compress, void *stream) {
  JB_REQUIRE(rows_ext >= 1 && cols >= 1 && own_lo < own_hi && own_hi <= rows_ext, "srad_slab: bad slab");
  JB_REQUIRE(J_ext && out_own && q0, "srad_slab: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int tiles_x = (int)((cols + TW - 1) / TW), tiles_y = (int)((own_hi - own_lo + TH - 1) / TH);
  const int tiles = tiles_x * tiles_y;
  int per_sm = 0;
  JB_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, srad_iter_kernel, THREADS, 0));
  if (per_sm < 1) per_sm = 1;
  const int grid = tiles < sm_count() * per_sm ? tiles : sm_count() * per_sm;
  const size_t pb = ((grid * sizeof(Stats) + 255) / 256) * 256;
  char *ws = (char *)workspace(pb + 256, s);
  if (!ws) return JB_ECUDA;
  Args a{};
  a.src = J_ext; a.dst = out_own; a.q0 = q0; a.q0_next = nullptr;
  a.partials = (Stats *)ws; a.ticket = (unsigned *)(ws + pb);
  a.rows = (int)rows_ext; a.cols = (int)cols; a.tiles_x = tiles_x; a.tiles = tiles;
  a.row_lo = (int)own_lo; a.row_hi = (int)own_hi;
  a.ql = 0.25f * lambda;
  a.compress = compress;
  a.sums_out = sums;
  JB_CHECK_CUDA(cudaMemsetAsync(a.ticket, 0, sizeof(unsigned), s));
  void *tok = prof_begin("srad_iter", s);
  srad_iter_kernel<<<grid, THREADS, 0, s>>>(a);
  prof_end(tok, s);
  JB_LAUNCHED("srad_slab_step");
  return JB_OK;
}

extern "C" jb_status jb_srad_q0_f32(const double *sums, uint64_t npx_global, float *q0, void *stream) {
  JB_REQUIRE(sums && q0 && npx_global >= 1, "srad_q0: bad arguments");
  srad_q0_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(sums, (double)npx_global, q0);
  JB_LAUNCHED("srad_q0");
  return JB_OK;
}
