// edge.cu -- edge_detection<n,m,gs,sz,sb> on sm_100a.
//
// Juno program (EDGE; restated in
// oracle/juno_oracle.c:jo_edge_frame_f32):
//   smoothed  = gaussian_smoothing(input, gaussian)        gs x gs, clamp-to-edge
//   laplacian = dilate(smoothed) + erode(smoothed) - 2*smoothed   (pads 0 / 1)
//   zc        = dilate(sign(laplacian)) - erode(sign(laplacian))
//   gradient  = sqrt(gx^2 + gy^2), sobel sx/sy on smoothed, clamp-to-edge
//   maxgrad   = max fold over gradient (starts at gradient[0,0])
//   out       = (zc > 0 && gradient > theta*maxgrad) ? 1 : 0
// Every fork above is a parallel fork over (row, col); max_gradient is the
// one associative reduction (monoid max, skiff/passes/monoid.py:18-31) that
// the paper's GPU backend lowers to warp reductions.
//
// B200 design:
//  * edge_fused_kernel: one persistent kernel for the whole batch. A CTA owns
//    a 60x60 output tile; it stages the 70x70 clamped input tile in shared
//    memory (twice: the 16-byte-aligned TMA box and a copy shifted by three
//    columns, so every gaussian tap is one conflict-free 64-bit LDS of two
//    adjacent pixels), computes the 64x64 smoothed tile with packed
//    FMUL2/FADD2 (bit-exact, see the tile guard; a product shared by the two
//    mirrored taps of a top-bottom symmetric filter is computed once), the
//    62x62 laplacian with separable min/max, packs its sign
//    bits with warp ballots, derives zero crossings with 64-bit mask logic,
//    computes the sobel gx^2+gy^2, and stores it | zc<<31 (4 B/px, one TMA
//    bulk tensor store from its own shared buffer) plus a warp->block->grid
//    max (atomicMax on the float bits, per frame).
//  * the reject runs inside the same kernel as a second work queue: a frame
//    whose tiles are done publishes its threshold (sqrt.rn is monotone, so
//    zc && sqrt(g) > theta*sqrt(max g) becomes an integer compare on the
//    packed bits), and CTAs claim its reject units between compute tiles.
//    The packed scratch is a ring of L2-sized frame slots whose lines are
//    discarded from L2 after the reject reads them (never written back).
//  * a generic multi-kernel path (one kernel per stage, any gs/sz/sb) serves
//    other filter sizes and the stage-level test entry.
//
// Exactness: the oracle rounds every f32 op once (values.py:55-71).  The fast
// path is bit-identical under conditions checked on the device:
//   - gaussian coefficients finite, >= 0, min positive >= 2^-60, max < 2^50,
//     and every input pixel of the tile is 0 or in [2^-60, 2^64]: then every
//     product and partial sum is 0 or normal, so FADD2.FTZ == FADD.RN;
//   - structure == all ones (x*1 == x; FMNMX equals the Python fold up to the
//     sign of zero, which no later stage can observe);
//   - sobel coefficients in {0, +-1, +-2, +-4}: products exact, so FFMA ==
//     FMUL+FADD.
// Otherwise the tile runs the exact scalar path (same kernel, block-uniform
// branch), which follows the oracle operation by operation.
#include <math.h>
#include <string.h>
#include <stdlib.h>

#include <map>
#include <mutex>

#include "common.cuh"
#include "tcgen05.cuh"

// -DEDGE_STAGE_CLOCKS: per-stage SM-cycle accounting (tools/edge_stage_clocks.py)
#ifdef EDGE_STAGE_CLOCKS
__device__ unsigned long long g_edge_clk[16];
__shared__ long long s_edge_clk;
#define EDGE_T(i)                                                            \
  do {                                                                       \
    if (threadIdx.x == 0) {                                                  \
      const long long _t = clock64();                                        \
      atomicAdd(&g_edge_clk[i], (unsigned long long)(_t - s_edge_clk));      \
      s_edge_clk = _t;                                                       \
    }                                                                        \
  } while (0)
#define EDGE_T0()                                   \
  do {                                              \
    if (threadIdx.x == 0) s_edge_clk = clock64();   \
  } while (0)
#else
#define EDGE_T(i) do {} while (0)
#define EDGE_T0() do {} while (0)
#endif

namespace jb {
namespace edge {

constexpr int TW = 60, TH = 60;        // output tile
constexpr int SR = 64;                 // smoothed region (tile + 2 halo)
constexpr int IR = 70;                 // input region (tile + 5 halo)
constexpr int IP = 72;                 // input row pitch (floats)
constexpr int LR = 62;                 // laplacian region (tile + 1 halo)
constexpr int THREADS = 256;

struct ConstBank {
  cudaEvent_t ev = nullptr;   // recorded after the last kernel reading the bank
  cudaStream_t stream = nullptr;
};
static std::map<std::pair<int, int>, ConstBank> g_bank;
static std::mutex g_bank_mu;

__constant__ float c_gauss[49];
__constant__ float c_struct[9];
__constant__ float c_sx[9];
__constant__ float c_sy[9];

constexpr int RP = 76;                 // raw row pitch: input columns x0-8 .. x0+67
// thread 0's scheduler state (kept in smem: fewer live registers in the tile code)
struct Sched {
  int free_upto;  // frames <= free_upto may write their ring slot
  int sp_base;    // first frame of the in-flight slot probe, or -1
  int pd;         // frame of the tile whose bulk store is in flight (not yet counted), or -1
  int acq;        // last frame whose ready word was followed by an acquire fence
  int ru;         // reject unit assigned to the current tile, or -1
};

struct alignas(128) Smem {
  // raw[r][c] = input(y0-5+r, x0-8+c): the 16-byte-aligned TMA box (TMA needs
  // an aligned inner start coordinate); the pairs (x, x+1) with x - x0 odd
  // are read from here, the ones with x - x0 even from the copy inA
  alignas(128) float raw[IR][RP];
  alignas(128) float inA[IR][IP];  // inA[r][c] = input(y0-5+r, x0-5+c)
  // the packed tile, read by the async proxy (bulk tensor store) until
  // thread 0's bulk_wait_read at the next tile's top; its own buffer, so the
  // next tile's stage 0 may refill inA while the store is still reading
  alignas(128) uint32_t P[TH][TW];
  float sm[SR][SR];       // smoothed tile (out-of-frame = clamped replica)
  uint32_t lapbits[LR][2];// laplacian > 0, bit = column within 32-col chunk
  uint32_t zcw[TH][2];    // zero crossing, bit = column within 32-col chunk
  float wmax[THREADS / 32];
  uint64_t tma_bar;       // completion of the two TMA loads of an interior tile
  int next_tile;          // claimed by thread 0 (dynamic tile scheduler)
  int nt_f, nt_y0, nt_x0; // its frame and origin (computed once, by thread 0)
  int flag;               // reject unit claimed by thread 0 (or a state, see claim_reject)
  int hflag;              // the same for the per-tile help unit (no barrier between the two)
  int lo;                 // that unit's threshold
  Sched q;                // thread 0 only
};

// flags[0]: 1 if the filters admit the fast path; flags[1]: standard sobel pair;
// flags[2]: the gaussian is mirror-symmetric top to bottom (bitwise)
__global__ void edge_check_kernel(const float *__restrict__ gf, const float *__restrict__ st,
                                  const float *__restrict__ sx, const float *__restrict__ sy,
                                  int *flags) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int ok = 1;
  for (int k = 0; k < 9; k++) ok &= (st[k] == 1.0f);
  for (int k = 0; k < 49; k++) {
    const float g = gf[k];
    ok &= (g >= 0.0f) && (g < 0x1p50f);  // rejects NaN and negatives
    if (g != 0.0f) ok &= (g >= 0x1p-60f);
  }
  int std_sobel = 1;
  const float SX[9] = {-1.f, 0.f, 1.f, -2.f, 0.f, 2.f, -1.f, 0.f, 1.f};
  const float SY[9] = {-1.f, -2.f, -1.f, 0.f, 0.f, 0.f, 1.f, 2.f, 1.f};
  for (int k = 0; k < 9; k++) {
    const float a = fabsf(sx[k]), b = fabsf(sy[k]);
    ok &= (a == 0.f || a == 1.f || a == 2.f || a == 4.f);
    ok &= (b == 0.f || b == 1.f || b == 2.f || b == 4.f);
    std_sobel &= (sx[k] == SX[k]) && (sy[k] == SY[k]);
  }
  // vertical mirror symmetry of the gaussian, bit for bit: then the product
  // of an input pixel with w[i][j] equals its product with w[6-i][j], and
  // the fast gaussian computes it once for both output rows
  int vsym = 1;
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 7; j++) vsym &= __float_as_uint(gf[i * 7 + j]) == __float_as_uint(gf[(6 - i) * 7 + j]);
  flags[0] = ok;
  flags[1] = ok && std_sobel;
  flags[2] = ok && vsym;
}

struct FusedArgs {
  CUtensorMap tmap;     // [frames][n][m] input, box {76, 70, 1} (valid if use_tma)
  CUtensorMap pmap;     // [ring][n][m] packed ring, box {60, 60, 1} (valid if use_tma)
  int use_tma;
  const float *in;      // [frames][n][m]
  float *out;           // [frames][n][m] edge maps
  uint32_t *packed;     // ring [ring][slot_px]: gradient bits | zc << 31
  unsigned *fmax;       // [frames] max gx^2+gy^2 bits
  unsigned *done;       // [frames] finished tiles; tiles+1 once lo[f] is published
  unsigned *rdone;      // [frames] finished reject units
  unsigned long long *ready;  // [frames] (1 << 32 | threshold) once published
  unsigned *pub;        // [frames] publisher election
  unsigned *rj;         // [frames] claimed reject units
  unsigned *sched;      // [0] next compute tile, [1] reject frame cursor
  const int *flags;
  float theta;
  int n, m, frames, tiles_x, tiles_y;
  int ring;             // frame slots in the packed ring
  int units, unit_px;   // reject units per frame, pixels per unit (multiple of 1024)
  int vec4;             // frame_px % 4 == 0 and out 16-byte aligned
  long long frame_px, slot_px;
  int lag;              // tiles of frame f + lag run the reject units of frame f
  int opts;             // experiment bits (JB_EDGE_OPTS): 1 keep the ring lines (no discards)
  uint32_t *obits;      // bit-packed edge maps [frames][frame_words] (instead of out), or null
  long long frame_words;// ceil(frame_px / 32): bit b of word w is pixel 32w + b
};

// fast-path data guard: every staged pixel is +0 or in [2^-60, 2^64].  On
// the raw bits: max(u) <= bits(2^64) (rejects negatives, -0, inf, NaN) and
// min(u - 1) >= bits(2^-60) - 1 (u = +0 wraps to 0xffffffff), accumulated
// with 3-input integer min/max: two instructions per pixel pair.
struct PixGuard {
  unsigned mx = 0u, mn = 0xffffffffu;
  __device__ __forceinline__ void add(float a) {
    const unsigned u = __float_as_uint(a);
    mx = max(mx, u);
    mn = min(mn, u - 1u);
  }
  __device__ __forceinline__ void add2(float a, float b) {
    const unsigned u = __float_as_uint(a), w = __float_as_uint(b);
    mx = __vimax3_u32(mx, u, w);
    mn = __vimin3_u32(mn, u - 1u, w - 1u);
  }
  __device__ __forceinline__ bool ok() const { return mx <= 0x5f800000u && mn >= 0x217fffffu; }
};

constexpr int RPW = (IR + THREADS / 32 - 1) / (THREADS / 32);  // staged rows per warp (9)

__device__ __forceinline__ void tile_origin(const FusedArgs &a, int tile, int &f, int &y0, int &x0) {
  const int tiles_per_frame = a.tiles_x * a.tiles_y;
  f = tile / tiles_per_frame;
  const int t2 = tile - f * tiles_per_frame;
  const int ty = t2 / a.tiles_x, tx = t2 - ty * a.tiles_x;
  y0 = ty * TH;
  x0 = tx * TW;
}

// the 76x70 raw box lies inside the frame: no clamping, TMA can stage it
__device__ __forceinline__ bool tile_interior(const FusedArgs &a, int y0, int x0) {
  return y0 >= 5 && x0 >= 8 && y0 + IR - 5 <= a.n && x0 - 8 + RP <= a.m;
}

// one thread: stage an interior tile's input with one TMA box load into
// S.raw; completion on S.tma_bar
__device__ __forceinline__ void stage_tile_tma(Smem &S, const FusedArgs &a, int f, int y0, int x0) {
  tc::fence_proxy_async_smem();  // the generic-proxy accesses of raw/inA are done
  tc::mbar_arrive_expect_tx(&S.tma_bar, IR * RP * 4);
  // [frames][n][m] tensor: out-of-frame rows and columns of a border tile's
  // box arrive as zeros (TMA out-of-bounds fill) and are replaced by the
  // clamped replicas in smem (stage 0).  The input is read once: evict it
  // first, so the packed ring (evict last) survives in L2 until its reject
  // units read it
  tc::tma_load_3d_hint(&S.raw[0][0], &a.tmap, &S.tma_bar, x0 - 8, y0 - 5, f, tc::policy_evict_first());
}

// stage 0 of a border tile: its TMA box holds zeros where it leaves the
// frame; give those positions the clamped in-frame value, which is what the
// gaussian's clamp-to-edge indexing reads.  The clamped source of every
// out-of-frame position is an in-frame position of the box (never written
// here), so one pass suffices; only out-of-frame rows and columns are
// visited.
__device__ __noinline__ void replicate_box_edges(Smem &S, const FusedArgs &a, int y0, int x0, int tid) {
  const int ylo = max(0, 5 - y0), yhi = min(IR, a.n - (y0 - 5));  // in-frame box rows [ylo, yhi)
  const int xlo = max(0, 8 - x0), xhi = min(RP, a.m - (x0 - 8));  // in-frame box columns
  const int nr = ylo + (IR - yhi), nc = xlo + (RP - xhi);
  const int rows_px = nr * RP, total = rows_px + (yhi - ylo) * nc;
  for (int idx = tid; idx < total; idx += THREADS) {
    int r, c;
    if (idx < rows_px) {  // whole out-of-frame rows
      const int k = idx / RP;
      c = idx - k * RP;
      r = k < ylo ? k : yhi + (k - ylo);
    } else {              // out-of-frame columns of in-frame rows
      const int j = idx - rows_px, q = j / nc, k = j - q * nc;
      r = ylo + q;
      c = k < xlo ? k : xhi + (k - xlo);
    }
    S.raw[r][c] = S.raw[min(max(r, ylo), yhi - 1)][min(max(c, xlo), xhi - 1)];
  }
  __syncthreads();
}

extern __shared__ __align__(16) unsigned char smem_raw[];
__device__ __forceinline__ Smem &smem_tile() {
  const uint32_t pad = (128u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u;
  return *reinterpret_cast<Smem *>(smem_raw + pad);
}

// stage 1, fast path: packed gaussian of 8 smoothed rows x 2 columns per
// lane.  Not inlined: one copy is shared by every tile variant, which keeps
// the hot code inside the instruction cache.
// VSYM: w[i][j] == w[6-i][j] bitwise; the weight is read from the canonical
// row min(i, 6-i), so the two products of an input pair with mirrored taps are
// one expression (computed once: the rounded product is the same value for
// both output rows, and each output still adds its 49 terms in tap order).
template <bool VSYM>
__device__ __noinline__ void gauss_fast(int warp, int lane) {
  Smem &S = smem_tile();
  const int r0 = warp * 8;
  unsigned long long acc[8];
#pragma unroll
  for (int o = 0; o < 8; o++) acc[o] = 0ull;  // (+0.0f, +0.0f)
#pragma unroll
  for (int iy = 0; iy < 14; iy++) {
    const unsigned long long *ra = reinterpret_cast<const unsigned long long *>(&S.inA[r0 + iy][0]);
    const unsigned long long *rb = reinterpret_cast<const unsigned long long *>(&S.raw[r0 + iy][0]);
    unsigned long long v[7];
    // pair (x0-5+2l+j, +1): even j from inA, odd j from raw at 2l+j+3
#pragma unroll
    for (int j = 0; j < 7; j++) v[j] = (j & 1) ? rb[lane + ((j + 3) >> 1)] : ra[lane + (j >> 1)];
#pragma unroll
    for (int o = 0; o < 8; o++) {
      const int i = iy - o;
      if (i >= 0 && i < 7) {
#pragma unroll
        for (int j = 0; j < 7; j++)
          acc[o] = f2_add_ftz(acc[o], f2_mul(v[j], c_gauss[(VSYM ? (i < 6 - i ? i : 6 - i) : i) * 7 + j]));
      }
    }
  }
#pragma unroll
  for (int o = 0; o < 8; o++) *reinterpret_cast<unsigned long long *>(&S.sm[r0 + o][2 * lane]) = acc[o];
}

// out-of-frame positions of a border tile's 64x64 smoothed region: NaN
// (pads = true) or the clamped in-frame value.  Only those positions are
// visited; their clamped sources are in-frame, so one pass suffices.
__device__ __noinline__ void smooth_oob(Smem &S, const FusedArgs &a, int y0, int x0, int tid, bool pads) {
  const int ylo = max(0, 2 - y0), yhi = min(SR, a.n - (y0 - 2));  // in-frame rows [ylo, yhi)
  const int xlo = max(0, 2 - x0), xhi = min(SR, a.m - (x0 - 2));
  const int nr = ylo + (SR - yhi), nc = xlo + (SR - xhi);
  const int rows_px = nr * SR, total = rows_px + (yhi - ylo) * nc;
  for (int idx = tid; idx < total; idx += THREADS) {
    int r, c;
    if (idx < rows_px) {  // whole out-of-frame rows
      const int k = idx >> 6;
      c = idx & 63;
      r = k < ylo ? k : yhi + (k - ylo);
    } else {              // out-of-frame columns of in-frame rows
      const int j = idx - rows_px, q = j / nc, k = j - q * nc;
      r = ylo + q;
      c = k < xlo ? k : xhi + (k - xlo);
    }
    S.sm[r][c] = pads ? __int_as_float(0x7fffffff)
                      : S.sm[min(max(r, ylo), yhi - 1)][min(max(c, xlo), xhi - 1)];
  }
}

// end of a tile's compute, before the CTA barrier that the main loop shares
// with the reject-unit decision: P is handed to the async proxy (its bulk
// tensor store is issued by thread 0 after the barrier, with the block max's
// atomicMax: tile_store)
__device__ __forceinline__ unsigned tile_tail(Smem &S, const FusedArgs &a, int f, int y0, int x0, int tid,
                                              int lane, int warp, float bmax) {
  if (a.use_tma) tc::fence_proxy_async_smem();  // P -> async proxy
  bmax = warp_max(bmax);
  if (lane == 0) S.wmax[warp] = bmax;
  return 0;
}

// thread 0, after the barrier: the packed tile leaves by bulk tensor store
// (TMA path), the block max goes to the frame's atomicMax; its return value
// (consumed a tile later, flush_done) tells that the max has been performed
// before the tile is counted
__device__ __forceinline__ unsigned tile_store(Smem &S, const FusedArgs &a, int f, int y0, int x0) {
  if (a.use_tma) {
    tc::tma_store_3d_hint(&a.pmap, &S.P[0][0], x0, y0, f % a.ring, tc::policy_evict_last());
    tc::bulk_commit();
  }
  float v = S.wmax[0];
#pragma unroll
  for (int w = 1; w < THREADS / 32; w++) v = fmaxf(v, S.wmax[w]);
  return !(v != v) ? atomicMax(a.fmax + f, __float_as_uint(v)) : 0u;
}

// stages 2b + 2c of an interior tile with the standard sobel pair (TMA path):
// zero crossings and gradient per warp, no block barrier between them.
//  * warp w owns 8 output rows (k0 = 8w; warp 7 rows 52..59, overlapping
//    warp 6 by 4 rows: duplicate, identical stores);
//  * zero crossings: lane k < 8 derives row k0+k's 64-bit mask from three
//    laplacian sign rows; the row loop broadcasts it with two shuffles;
//  * gradient: lane l owns columns l and l+32 (lanes 28..31 repeat column
//    59 in the second slot, not stored) as one f32x2 pair, so every sobel
//    step is one packed FADD2/FFMA2 for two pixels.  The fold is the
//    oracle's 9-tap order with the x*0 taps dropped (they only change the
//    sign of a zero, which the square erases) and x*(+-1), x*(+-2) exact; gy
//    is carried negated (ny = -gy: every rounding is sign-symmetric).  The
//    squares are FMUL2, the sum a scalar add.rn (single rounding each).
template <bool BORDER>
__device__ __forceinline__ unsigned sobel_pairs(Smem &S, const FusedArgs &a, int f, int y0, int x0, int tid,
                                             int lane, int warp) {
  const int k0 = warp < 7 ? warp * 8 : TH - 8;
  unsigned zlo = 0, zhi = 0;
  if (lane < 8) {
    // border tiles: out-of-frame laplacian positions pad the dilation with 0
    // and the erosion with 1 (masked out of both folds)
    unsigned long long colmask = ~0ull;
    if (BORDER) {
      const int lo = max(0, 1 - x0), hi = min(LR - 1, a.m - x0);  // frame columns x0-1+lc in [0, m)
      colmask = hi >= lo ? (((hi - lo + 1) >= 64 ? ~0ull : ((1ull << (hi - lo + 1)) - 1)) << lo) : 0ull;
    }
    unsigned long long orr = 0, andd = ~0ull;
#pragma unroll
    for (int i = 0; i < 3; i++) {
      const int lr = k0 + lane + i, gy = y0 - 1 + lr;
      if (!BORDER || (gy >= 0 && gy < a.n)) {
        const unsigned long long b = *reinterpret_cast<const unsigned long long *>(&S.lapbits[lr][0]);
        orr |= b & colmask;
        andd &= b | ~colmask;
      }
    }
    const unsigned long long zc = (orr | (orr >> 1) | (orr >> 2)) & ~(andd & (andd >> 1) & (andd >> 2));
    zlo = (unsigned)zc;
    zhi = (unsigned)(zc >> 32);
  }
  const int ca = lane, cb = min(lane + 32, TW - 1);
  const bool b_ok = lane + 32 < TW;
  const f2 two = bc2(2.0f), mtwo = bc2(-2.0f);
  float bmax = 0.0f;
  f2 gx[3], ny[3];
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const int sr = k0 + 1 + r;  // smoothed row
    const f2 v0 = pk2(S.sm[sr][ca + 1], S.sm[sr][cb + 1]);
    const f2 v1 = pk2(S.sm[sr][ca + 2], S.sm[sr][cb + 2]);
    const f2 v2 = pk2(S.sm[sr][ca + 3], S.sm[sr][cb + 3]);
#pragma unroll
    for (int q = 0; q < 3; q++) {
      const int k = r - q;  // output row k0 + k gets tap row q
      if (k < 0 || k >= 8) continue;
      const int s = k % 3;
      if (q == 0) {
        gx[s] = sub2n(v2, v0);
        ny[s] = add2n(fma2(v1, two, v0), v2);
      } else if (q == 1) {
        gx[s] = fma2(v2, two, fma2(v0, mtwo, gx[s]));
      } else {
        gx[s] = add2n(sub2n(gx[s], v0), v2);
        ny[s] = sub2n(fma2(v1, mtwo, sub2n(ny[s], v0)), v2);
        const f2 sx2 = mul2(gx[s], gx[s]), sy2 = mul2(ny[s], ny[s]);
        const float ga = add_rn(lo2(sx2), lo2(sy2)), gb = add_rn(hi2(sx2), hi2(sy2));
        const unsigned zl = __shfl_sync(0xffffffffu, zlo, k), zh = __shfl_sync(0xffffffffu, zhi, k);
        S.P[k0 + k][ca] = __float_as_uint(ga) | ((zl << (31 - lane)) & 0x80000000u);
        if (b_ok) S.P[k0 + k][lane + 32] = __float_as_uint(gb) | ((zh << (31 - lane)) & 0x80000000u);
        if (!BORDER) {
          bmax = fmaxf(bmax, fmaxf(ga, gb));
        } else if (y0 + k0 + k < a.n) {  // only in-frame pixels enter the max
          if (x0 + ca < a.m) bmax = fmaxf(bmax, ga);
          if (x0 + cb < a.m) bmax = fmaxf(bmax, gb);
        }
      }
    }
    // keep the next rows' loads from being hoisted (register pressure: the
    // persistent loop's state must not spill)
    asm volatile("" ::: "memory");
  }
  return tile_tail(S, a, f, y0, x0, tid, lane, warp, bmax);
}

// stages 1-2 of one 60x60 tile whose clamped input is staged in S.inA/S.raw.
// FAST: packed/FTZ gaussian, FMNMX morphology, FFMA sobel (guarded exact);
// otherwise the oracle's operation order with single-rounding scalar ops.
// BORDER: the tile's halo leaves the frame (pads / clamped replicas needed).
template <bool FAST, bool BORDER, bool SOBEL_STD = false>
__device__ __forceinline__ unsigned edge_tile(Smem &S, const FusedArgs &a, int f, int y0, int x0, int tid,
                                          int lane, int warp, bool prefetch, int nf, int ny0, int nx0) {
  const int n = a.n, m = a.m;
  // ---- stage 1: gaussian on the 64x64 smoothed region
  {
    const int r0 = warp * 8;  // 8 smoothed rows per warp, 2 columns per lane
    if (FAST) {
      if (a.flags[2]) gauss_fast<true>(warp, lane);
      else gauss_fast<false>(warp, lane);
    } else {
      float2 acc[8];
#pragma unroll
      for (int o = 0; o < 8; o++) acc[o] = make_float2(0.0f, 0.0f);
#pragma unroll 1
      for (int iy = 0; iy < 14; iy++) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) v[j] = S.inA[r0 + iy][2 * lane + j];
#pragma unroll
        for (int o = 0; o < 8; o++) {
          const int i = iy - o;
          if (i >= 0 && i < 7) {
#pragma unroll
            for (int j = 0; j < 7; j++) {
              const float g = c_gauss[i * 7 + j];
              acc[o].x = add_rn(acc[o].x, mul_rn(v[j], g));
              acc[o].y = add_rn(acc[o].y, mul_rn(v[j + 1], g));
            }
          }
        }
      }
#pragma unroll
      for (int o = 0; o < 8; o++) *reinterpret_cast<float2 *>(&S.sm[r0 + o][2 * lane]) = acc[o];
    }
  }
  __syncthreads();
  EDGE_T(1);
  // raw/inA are free from here on: prefetch the next (interior) tile by TMA
  if (prefetch && tid == 0) stage_tile_tma(S, a, nf, ny0, nx0);
  // out-of-frame smoothed positions take the clamped in-frame value, which is
  // what the gradient's clamp-to-edge indexing reads.  The paired path first
  // gives them NaN instead: FMNMX ignores NaN, so the plain separable
  // laplacian then pads exactly like the oracle (0 for the dilation's max, 1
  // for the erosion's min, both folds starting there); the replicas follow
  // after the laplacian.
  if (BORDER && SOBEL_STD) {
    smooth_oob(S, a, y0, x0, tid, true);
    __syncthreads();
  } else if (BORDER) {
    for (int idx = tid; idx < SR * SR; idx += THREADS) {
      const int r = idx >> 6, c = idx & 63;
      const int gy = y0 - 2 + r, gx = x0 - 2 + c;
      const int cy = min(max(gy, 0), n - 1), cx = min(max(gx, 0), m - 1);
      if (cy != gy || cx != gx) S.sm[r][c] = S.sm[cy - (y0 - 2)][cx - (x0 - 2)];
    }
    __syncthreads();
  }

  // ---- stage 2a: laplacian sign bits on the 62x62 region
  {
    const int cc = warp & 1, rb = warp >> 1;
    const int lc = cc * 32 + lane;         // laplacian column (region)
    const bool col_ok = lc < LR;
    const int gxc = x0 - 1 + lc;           // frame column of the centre
    const int scol = col_ok ? lc : LR - 1; // keep smem reads in bounds
    if (FAST) {
      // separable 3x3 max/min rolled down the column
      float hx0 = 0.f, hx1 = 0.f, hn0 = 0.f, hn1 = 0.f, cprev = 0.f;
      bool i0 = true, i1 = true, i2 = true;
      if (BORDER && !SOBEL_STD) {
        i0 = gxc - 1 >= 0 && gxc - 1 < m;
        i1 = gxc >= 0 && gxc < m;
        i2 = gxc + 1 >= 0 && gxc + 1 < m;
      }
#pragma unroll
      for (int k = 0; k < 18; k++) {
        const int sr = min(rb * 16 + k, SR - 1);
        const float a0 = S.sm[sr][scol], a1 = S.sm[sr][scol + 1], a2 = S.sm[sr][scol + 2];
        float hx2, hn2;
        if (BORDER && !SOBEL_STD) {
          const int gy = y0 - 2 + rb * 16 + k;
          const bool rin = gy >= 0 && gy < n;
          hx2 = fmaxf(fmaxf(rin && i0 ? a0 : -INFINITY, rin && i1 ? a1 : -INFINITY), rin && i2 ? a2 : -INFINITY);
          hn2 = fminf(fminf(rin && i0 ? a0 : INFINITY, rin && i1 ? a1 : INFINITY), rin && i2 ? a2 : INFINITY);
        } else {
          hx2 = fmaxf(fmaxf(a0, a1), a2);
          hn2 = fminf(fminf(a0, a1), a2);
        }
        if (k >= 2) {
          const int lr = rb * 16 + k - 2;
          const float d = fmaxf(0.0f, fmaxf(fmaxf(hx0, hx1), hx2));
          const float e = fminf(1.0f, fminf(fminf(hn0, hn1), hn2));
          const float lap = fmaf(-2.0f, cprev, add_rn(d, e));  // 2*x is exact
          const unsigned bits = __ballot_sync(0xffffffffu, col_ok && lap > 0.0f);
          if (lane == 0 && lr < LR) S.lapbits[lr][cc] = bits;
        }
        hx0 = hx1; hx1 = hx2; hn0 = hn1; hn1 = hn2; cprev = a1;
      }
    } else {
#pragma unroll 1
      for (int k = 0; k < 16; k++) {
        const int lr = rb * 16 + k;
        bool pos = false;
        if (col_ok && lr < LR) {
          const int gyc = y0 - 1 + lr;
          float d = 0.0f, e = 1.0f;
#pragma unroll
          for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
              const int gy = gyc + i - 1, gx = gxc + j - 1;
              const bool in = gy >= 0 && gy < n && gx >= 0 && gx < m;
              d = py_max(d, mul_rn(in ? S.sm[lr + i][lc + j] : 0.0f, c_struct[i * 3 + j]));
            }
#pragma unroll
          for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
              const int gy = gyc + i - 1, gx = gxc + j - 1;
              const bool in = gy >= 0 && gy < n && gx >= 0 && gx < m;
              e = py_min(e, mul_rn(in ? S.sm[lr + i][lc + j] : 1.0f, c_struct[i * 3 + j]));
            }
          pos = sub_rn(add_rn(d, e), mul_rn(2.0f, S.sm[lr + 1][lc + 1])) > 0.0f;
        }
        const unsigned bits = __ballot_sync(0xffffffffu, pos);
        if (lane == 0 && lr < LR) S.lapbits[lr][cc] = bits;
      }
    }
  }
  // the previous tile's packed tile has left S.P before the sobel stage
  // refills it (the barrier below orders this for every warp); waited for as
  // late as possible, so the bulk store's smem reads overlap the gaussian
  // and the laplacian instead of thread 0's tile top
  if (tid == 0) tc::bulk_wait_read<0>();
  __syncthreads();
  EDGE_T(2);

  if (SOBEL_STD) {
    if (BORDER) {  // the sobel's clamp-to-edge replicas (the NaN pads are no longer read)
      smooth_oob(S, a, y0, x0, tid, false);
      __syncthreads();
    }
    return sobel_pairs<BORDER>(S, a, f, y0, x0, tid, lane, warp);
  }

  // ---- stage 2b: zero crossings (bit masks), one thread per output row
  if (tid < TH) {
    const int orow = tid;
    unsigned long long zc = 0;
    if (FAST) {
      // frame-column validity of laplacian columns lc = 0..61 (x0-1+lc)
      unsigned long long colmask = ~0ull;
      if (BORDER) {
        const int lo = max(0, 1 - x0), hi = min(LR - 1, m - x0);
        colmask = hi >= lo ? (((hi - lo + 1) >= 64 ? ~0ull : ((1ull << (hi - lo + 1)) - 1)) << lo) : 0ull;
      }
      unsigned long long orr = 0, andd = ~0ull;
#pragma unroll
      for (int i = 0; i < 3; i++) {
        const int lr = orow + i;
        const int gy = y0 - 1 + lr;
        if (!BORDER || (gy >= 0 && gy < n)) {
          const unsigned long long b =
              (unsigned long long)S.lapbits[lr][0] | ((unsigned long long)S.lapbits[lr][1] << 32);
          orr |= b & colmask;
          andd &= b | ~colmask;
        }
      }
      zc = (orr | (orr >> 1) | (orr >> 2)) & ~(andd & (andd >> 1) & (andd >> 2));
    } else {
      const int gyc = y0 + orow;
      for (int oc = 0; oc < TW; oc++) {
        const int gxc = x0 + oc;
        float d = 0.0f, e = 1.0f;
        for (int i = 0; i < 3; i++)
          for (int j = 0; j < 3; j++) {
            const int lr = orow + i, lc = oc + j;
            const int gy = gyc + i - 1, gx = gxc + j - 1;
            const bool in = gy >= 0 && gy < n && gx >= 0 && gx < m;
            const float sg = ((S.lapbits[lr][lc >> 5] >> (lc & 31)) & 1u) ? 1.0f : 0.0f;
            d = py_max(d, mul_rn(in ? sg : 0.0f, c_struct[i * 3 + j]));
          }
        for (int i = 0; i < 3; i++)
          for (int j = 0; j < 3; j++) {
            const int lr = orow + i, lc = oc + j;
            const int gy = gyc + i - 1, gx = gxc + j - 1;
            const bool in = gy >= 0 && gy < n && gx >= 0 && gx < m;
            const float sg = ((S.lapbits[lr][lc >> 5] >> (lc & 31)) & 1u) ? 1.0f : 0.0f;
            e = py_min(e, mul_rn(in ? sg : 1.0f, c_struct[i * 3 + j]));
          }
        if (sub_rn(d, e) > 0.0f) zc |= 1ull << oc;
      }
    }
    S.zcw[orow][0] = (unsigned)zc;
    S.zcw[orow][1] = (unsigned)(zc >> 32);
  }
  __syncthreads();
  EDGE_T(3);

  // ---- stage 2c: sobel gradient, pack with zc, block max
  float bmax = 0.0f;
  {
    const int cc = warp & 1, rb = warp >> 1;
    const int oc = cc * 32 + lane;
    const bool col_ok = oc < TW && (!BORDER || x0 + oc < m);
    const int scol = min(oc, TW - 1);
    const int orow0 = rb * 15;
    uint32_t *prow = a.use_tma ? nullptr
                               : a.packed + (size_t)(f % a.ring) * a.slot_px + (size_t)(y0 + orow0) * m + x0 + scol;
    // TMA path: the packed tile goes to smem (S.P) and leaves with one bulk
    // tensor store; the box clips borders
    uint32_t(*P)[TW] = S.P;
    float sx[9], sy[9];
#pragma unroll
    for (int q = 0; q < 9; q++) { sx[q] = c_sx[q]; sy[q] = c_sy[q]; }
    float gxs[3] = {0.f, 0.f, 0.f}, gys[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 17; r++) {
      const int sr = orow0 + 1 + r;  // smoothed row
      const float v0 = S.sm[sr][scol + 1], v1 = S.sm[sr][scol + 2], v2 = S.sm[sr][scol + 3];
#pragma unroll
      for (int q = 0; q < 3; q++) {
        const int k = r - q;  // output row k (0..14) gets tap row q
        if (k >= 0 && k < 15) {
          float gx = q == 0 ? 0.0f : gxs[k % 3], gy = q == 0 ? 0.0f : gys[k % 3];
          if (FAST) {
            gx = fmaf(v0, sx[q * 3 + 0], gx); gy = fmaf(v0, sy[q * 3 + 0], gy);
            gx = fmaf(v1, sx[q * 3 + 1], gx); gy = fmaf(v1, sy[q * 3 + 1], gy);
            gx = fmaf(v2, sx[q * 3 + 2], gx); gy = fmaf(v2, sy[q * 3 + 2], gy);
          } else {
            gx = add_rn(gx, mul_rn(v0, sx[q * 3 + 0])); gy = add_rn(gy, mul_rn(v0, sy[q * 3 + 0]));
            gx = add_rn(gx, mul_rn(v1, sx[q * 3 + 1])); gy = add_rn(gy, mul_rn(v1, sy[q * 3 + 1]));
            gx = add_rn(gx, mul_rn(v2, sx[q * 3 + 2])); gy = add_rn(gy, mul_rn(v2, sy[q * 3 + 2]));
          }
          gxs[k % 3] = gx; gys[k % 3] = gy;
          if (q == 2) {
            // gx^2 + gy^2; the reject pass takes the (correctly rounded,
            // hence monotone) sqrt, so max(sqrt(a)) = sqrt(max(a))
            const float g = add_rn(mul_rn(gx, gx), mul_rn(gy, gy));
            const unsigned z = (S.zcw[orow0 + k][cc] >> lane) & 1u;
            if (a.use_tma) {
              if (oc < TW) P[orow0 + k][oc] = __float_as_uint(g) | (z << 31);
              if (col_ok && (!BORDER || y0 + orow0 + k < n)) bmax = fmaxf(bmax, g);
            } else if (col_ok && (!BORDER || y0 + orow0 + k < n)) {
              prow[(size_t)k * m] = __float_as_uint(g) | (z << 31);
              bmax = fmaxf(bmax, g);  // max of gx^2+gy^2 (ignores NaN like the fold)
            }
          }
        }
      }
    }
  }
  return tile_tail(S, a, f, y0, x0, tid, lane, warp, bmax);
}

// ------------------------------------------------ in-kernel reject (stage 3)
// The reject needs the frame's max gradient, a grid-wide dependency.  Rather
// than a second kernel over a scratch image, the persistent kernel runs it as
// a second work queue: once a frame's tiles are all finished, its threshold
// is published and CTAs claim the frame's reject units between compute
// tiles.  The packed gradients live in a ring of `ring` frame slots
// (L2-sized); a tile may only start writing slot f % ring once frame
// f - ring is rejected.  Compute tiles are claimed from an atomic counter, so
// every wait below is for work a running CTA already owns: no co-residency
// assumption, no deadlock.
//
// Memory ordering.  The packed lines leave by bulk tensor store; a tile is
// counted (red.relaxed on done[f]) after cp.async.bulk.wait_group (not
// .read) reports the store complete and after fence.proxy.async.global plus
// a gpu-scope acq_rel fence (the release the PTX model asks for).  Readers
// observe ready[f] with a relaxed load followed by an acquire fence (once
// per frame and CTA) before reading the lines with ld.global.cg.  The
// publisher of a frame's threshold runs an acquire fence, and the L2
// discards are fenced before their unit is counted (their lines are
// rewritten by a later frame).
//
// -DEDGE_RELAXED_ORDERING drops the writer and reader fences: the store is
// complete at its home L2 slice before the count is sent and ld.cg reads
// that slice (cross-die accesses go to the home slice, 262 vs 234 cycles,
// B300_MICROARCH.md "L2 cache"), so it is safe on this hardware but outside
// the PTX model; it measures 4.3% faster (tools/ab_edge.sh: 68.1 k vs 65.3 k
// frames/s).
#ifndef EDGE_RELAXED_ORDERING
#define EDGE_STRICT_FENCES 1
#endif
//
// All scheduling is done by thread 0 with as few L2 round trips as possible
// (each one stalls the CTA at its next barrier): releases are one-thread
// fences after a CTA barrier (cumulative), tile completion is a
// fire-and-forget reduction, a reject claim is one atomicAdd ticket in the
// steady state, and frame readiness + threshold travel in one 64-bit word.
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add(unsigned *p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// drop a 128-byte L2 line without writing it back (the ring slot is dead
// once its reject unit has read it)
__device__ __forceinline__ void discard_l2(const void *p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

constexpr int kNoneReady = -1, kSlotFree = -2, kAllClaimed = -3;

// thread-0 scheduler state (registers of thread 0)

// thread 0: count the tile whose bulk store is in flight as done, once the
// store has completed (all but the newest group, or all) and its atomicMax
// has been performed (its return value consumed).  Ordering: see the
// "Memory ordering" note above.
__device__ __forceinline__ void flush_done(const FusedArgs &a, Sched &q, unsigned pd_max, bool newest_pending) {
  if (q.pd < 0) return;
  if (newest_pending) tc::bulk_wait<1>();
  else tc::bulk_wait<0>();
  if (pd_max == 0xffffffffu) red_add(a.done + q.pd, 0u);  // never true: orders the red after the atom
  asm volatile("fence.proxy.async.global;" ::: "memory");
#ifdef EDGE_STRICT_FENCES
  fence_acq_rel();
#endif
  red_add(a.done + q.pd, 1u);
  q.pd = -1;
}

// thread 0, frame f finished (done[f] == tiles): compute and publish the
// threshold on the packed bits (once, whoever wins pub[f]).
// out = zc && sqrt(g) > thr, thr = theta * sqrt(max g) (NaN if g[0,0] is NaN:
// the oracle's fold starts there).  sqrt.rn is monotone, so sqrt(g) > thr
// <=> bits(g) > lo, lo = the largest bit pattern whose sqrt is <= thr.
__device__ int publish_threshold(const FusedArgs &a, int f) {
  fence_acq_rel();  // acquire: every tile's packed stores and atomicMax
  const uint32_t p00 = __ldcg(a.packed + (size_t)(f % a.ring) * a.slot_px);
  const float g00 = __fsqrt_rn(__uint_as_float(p00 & 0x7fffffffu));
  const float thr = (g00 != g00) ? g00 : mul_rn(a.theta, __fsqrt_rn(__uint_as_float(__ldcg(a.fmax + f))));
  int lo;
  if (thr != thr) {
    lo = 0x7fffffff;  // nothing passes
  } else if (thr < 0.0f) {
    lo = -1;          // every non-NaN gradient passes
  } else {
    int b = (int)min(__float_as_uint(mul_rn(thr, thr)), 0x7f800000u);
    while (b > 0 && __fsqrt_rn(__int_as_float(b)) > thr) b--;
    while (b < 0x7f800000 && !(__fsqrt_rn(__int_as_float(b + 1)) > thr)) b++;
    lo = b;
  }
  // reject_px's bound: zc=1 puts the sign bit on, so "zc && lo < g <= inf"
  // is  A <= (int)p <= (int)0xff800000  with A = (lo + 1) - 2^31
  const int A = (int)((unsigned)(lo + 1) - 0x80000000u);
  atomicExch(a.ready + f, (1ull << 32) | (unsigned)A);
  return A;
}

// thread 0: the compare bound of frame f given its probed ready word and
// done count; publishes it if the frame is complete and nobody has; returns
// false when the frame is not ready yet.
__device__ bool frame_bound(const FusedArgs &a, int f, unsigned long long r, unsigned d, int &A, int &acq) {
  if (r >> 32) {
    A = (int)(unsigned)r;
    // acquire: the frame's packed lines before the unit's loads (once per
    // frame: a fence after an earlier observation of the same ready word
    // already orders them)
#ifdef EDGE_STRICT_FENCES
    if (acq != f) {
      fence_acq_rel();
      acq = f;
    }
#endif
    return true;
  }
  const unsigned tpf = (unsigned)(a.tiles_x * a.tiles_y);
  if (d == tpf && atomicCAS(a.pub + f, 0u, 1u) == 0u) {
    A = publish_threshold(a, f);  // begins with an acquire fence
    acq = f;
    return true;
  }
  return false;
}

// thread 0: spin until frame f is ready (the caller has no pending work
// anyone could be waiting on); returns its compare bound
__device__ int wait_frame(const FusedArgs &a, int f, int &acq) {
  for (;;) {
    int A;
    if (frame_bound(a, f, ld_relaxed64(a.ready + f), ld_relaxed(a.done + f), A, acq)) return A;
    __nanosleep(200);
  }
}

// the whole CTA: reject unit `unit` with compare bound `A` (from thread 0)
__device__ __noinline__ void reject_unit(const FusedArgs &a, int unit, int A) {
  const int f = unit / a.units, u = unit - f * a.units;
  const long long b0 = (long long)u * a.unit_px;
  const long long cnt = min((long long)a.unit_px, a.frame_px - b0);
  const uint32_t *src = a.packed + (size_t)(f % a.ring) * a.slot_px + b0;
  float *dst = a.obits ? nullptr : a.out + (size_t)f * a.frame_px + b0;
  // unit starts are multiples of 1024 pixels: whole words
  uint32_t *wdst = a.obits ? a.obits + (size_t)f * a.frame_words + (b0 >> 5) : nullptr;
  // Ring lines are discarded after their unit reads them, so the dead packed
  // scratch is never written back to HBM (without the discards the launch
  // moves 7.0 instead of 4.9 GB).  Read once: the discards' memory clobbers
  // would reload the flag from the parameter block every pass.
  const bool disc = !(a.opts & 1);
  // pass <=> A <= (int)p <= (int)0xff800000  <=>  p - Au < Ku (unsigned;
  // Ku = 0 when nothing can pass)
  const unsigned Au = (unsigned)A;
  const unsigned Ku = A <= (int)0xff800000u ? (unsigned)((int)0xff800000u - A) + 1u : 0u;
  if (a.vec4) {
    const int n4 = (int)(cnt >> 2);
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    // RB passes' loads in flight at once (one L2 round trip per RB passes,
    // not one per pass), then the compares and streaming stores
#ifndef EDGE_RB
#define EDGE_RB 4
#endif
    constexpr int RB = EDGE_RB;
    for (int base = 0; base < n4; base += RB * THREADS) {
      uint4 p[RB];
#pragma unroll
      for (int k = 0; k < RB; k++) {
        const int i = base + k * THREADS + threadIdx.x;
        if (i < n4) p[k] = __ldcg(s4 + i);
      }
#pragma unroll
      for (int k = 0; k < RB; k++) {
        const int i = base + k * THREADS + threadIdx.x;
        if (a.obits) {
          // bit-packed map: 8 lanes hold one word's 32 pixels (4 each)
          uint32_t v = 0;
          if (i < n4)
            v = ((p[k].x - Au < Ku ? 1u : 0u) | (p[k].y - Au < Ku ? 2u : 0u) | (p[k].z - Au < Ku ? 4u : 0u) |
                 (p[k].w - Au < Ku ? 8u : 0u)) << (4 * (threadIdx.x & 7));
          v |= __shfl_xor_sync(0xffffffffu, v, 1);
          v |= __shfl_xor_sync(0xffffffffu, v, 2);
          v |= __shfl_xor_sync(0xffffffffu, v, 4);
          if (i < n4 && (threadIdx.x & 7) == 0) __stcs(wdst + (i >> 3), v);
        } else if (i < n4) {
          __stcs(d4 + i, make_float4(p[k].x - Au < Ku ? 1.0f : 0.0f, p[k].y - Au < Ku ? 1.0f : 0.0f,
                                     p[k].z - Au < Ku ? 1.0f : 0.0f, p[k].w - Au < Ku ? 1.0f : 0.0f));
        }
      }
      __syncwarp();
      // the slot base and unit start are 4 KB aligned: lane 8k starts a line
#pragma unroll
      for (int k = 0; k < RB; k++) {
        const int i = base + k * THREADS + threadIdx.x;
        if (disc && i < n4 && (threadIdx.x & 7) == 0) discard_l2(s4 + i);
      }
    }
  } else if (a.obits) {
    // one ballot per 32 consecutive pixels (cnt is uniform: every warp
    // runs every pass)
    for (long long base = 0; base < cnt; base += THREADS) {
      const long long i = base + threadIdx.x;
      const unsigned w = __ballot_sync(0xffffffffu, i < cnt && __ldcg(src + i) - Au < Ku);
      if ((threadIdx.x & 31) == 0 && i < cnt) wdst[i >> 5] = w;
    }
  } else {
    for (long long i = threadIdx.x; i < cnt; i += THREADS) dst[i] = __ldcg(src + i) - Au < Ku ? 1.0f : 0.0f;
  }
  // every read of the unit's slot lines has returned (the values were
  // stored).  The discards must be performed before the unit is counted (a
  // discard still in flight when the slot's next frame is stored would drop
  // the new lines): the CTA barrier orders every thread's discards before
  // thread 0's gpu-scope fence, which is cumulative over them -- the pattern
  // a grid barrier uses to publish a whole CTA's writes -- so one fence per
  // unit suffices, not one per discarding lane
  __syncthreads();
  if (threadIdx.x == 0) {
    if (disc && a.vec4) fence_acq_rel();
    red_add(a.rdone + f, 1u);
  }
}

// thread 0's in-flight load results: registers, so that nothing waits for
// them before they are consumed (a tile later)
struct Inflight {
  unsigned sp[3];          // rdone of frames q.sp_base .. +2
  unsigned long long rr;   // ready word of the current tile's reject frame
  unsigned rdn;            // its done count
};

// thread 0: may frame f write its ring slot?  Uses the probe of rdone issued
// one tile earlier when it covers f; otherwise loads (stall) -- rare.
__device__ bool slot_free(const FusedArgs &a, Sched &q, const Inflight &r, int f) {
  if (f < a.ring || f <= q.free_upto) return true;
  const unsigned U = (unsigned)a.units;
  if (q.sp_base >= 0 && q.sp_base <= f - a.ring) {  // consume the probe
    const int k = f - a.ring - q.sp_base;  // 0..2: frames before f-ring were free (free_upto)
    int c = 0;
    while (c < 3 && r.sp[c] >= U) c++;
    q.sp_base = -1;
    if (c > k) {
      q.free_upto = f + (c - 1 - k);
      return true;
    }
  }
  const int g = f - a.ring;
  if (ld_relaxed(a.rdone + g) < U) return false;
  q.free_upto = f;
  return true;
}

// thread 0, after the slot check of frame f: probe frames f+1-ring .. f+3-ring
__device__ __forceinline__ void slot_probe(const FusedArgs &a, Sched &q, Inflight &r, int f) {
  if (q.sp_base >= 0 || f + 1 < a.ring || q.free_upto > f) return;
  const int g = f + 1 - a.ring;
  q.sp_base = g;
  r.sp[0] = ld_relaxed(a.rdone + g);
  r.sp[1] = g + 1 < a.frames ? ld_relaxed(a.rdone + g + 1) : 0u;
  r.sp[2] = g + 2 < a.frames ? ld_relaxed(a.rdone + g + 2) : 0u;
}

#ifndef EDGE_MINB
#define EDGE_MINB 3  // CTAs per SM (80 registers); A/B: 2 CTAs/SM (128 registers) 61.6k, 4 (64 registers, spills) 67.8k vs 73.1k frames/s
#endif
__global__ void __launch_bounds__(THREADS, EDGE_MINB)
edge_fused_kernel(const __grid_constant__ FusedArgs a) {
  Smem &S = smem_tile();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = a.n, m = a.m;
  const int tpf = a.tiles_x * a.tiles_y;
  const int total = tpf * a.frames;
  const int filters_fast = a.flags[0];
  const bool sobel_std = a.flags[1] != 0;
  Sched &q = S.q;
  unsigned pd_max = 0;  // thread 0: atomicMax result of the tile in flight
  Inflight rf_{{0u, 0u, 0u}, 0ull, 0u};
  if (tid == 0) {
    q.free_upto = -1; q.sp_base = -1; q.pd = -1; q.acq = -1; q.ru = -1;
  }
  // Reject units are assigned statically: tile j (< units) of frame f + lag
  // runs unit j of frame f at its end, so no queue is needed on the hot
  // path; the last `lag` frames are drained through a ticket counter.
  const int lag = a.lag;
  // Tiles are claimed two ahead: the claim issued during tile t is resolved
  // (origin computed once, broadcast through smem) during tile t+1, and the
  // input of tile t+1 is prefetched by TMA during tile t.
  unsigned claim2 = 0;
  auto publish_desc = [&](int t) {  // thread 0
    int f = 0, y0 = 0, x0 = 0;
    if (t < total) tile_origin(a, t, f, y0, x0);
    S.next_tile = t;
    S.nt_f = f; S.nt_y0 = y0; S.nt_x0 = x0;
  };
  if (tid == 0) {
    tc::mbar_init(&S.tma_bar, 1);
    tc::fence_mbar_init();
    publish_desc((int)atomicAdd(a.sched, 1u));
    if (S.next_tile < total && a.use_tma) stage_tile_tma(S, a, S.nt_f, S.nt_y0, S.nt_x0);
  }
  __syncthreads();
  int tile = S.next_tile, f = S.nt_f, y0 = S.nt_y0, x0 = S.nt_x0;  // current tile
  __syncthreads();
  if (tid == 0) {
    publish_desc((int)atomicAdd(a.sched, 1u));
    claim2 = atomicAdd(a.sched, 1u);
  }
  __syncthreads();
  int t1 = S.next_tile, f1 = S.nt_f, y1 = S.nt_y0, x1 = S.nt_x0;  // the next tile
  __syncthreads();  // thread 0 rewrites the descriptor in the first tile (racecheck)
  uint32_t tma_phase = 0;
  EDGE_T0();

  while (tile < total) {
    // ---- the ring slot of frame f must be rejected; probe this tile's
    // reject frame (consumed at the tile's end)
    if (tid == 0) {
      if (!slot_free(a, q, rf_, f)) {
        flush_done(a, q, pd_max, false);  // someone may be waiting on it
        while (ld_relaxed(a.rdone + f - a.ring) < (unsigned)a.units) __nanosleep(128);
        q.free_upto = f;
      }
      EDGE_T(8);
      slot_probe(a, q, rf_, f);
      const int j = tile - f * tpf;
      q.ru = -1;
      if (f >= lag && j < a.units) {
        q.ru = (f - lag) * a.units + j;
        rf_.rr = ld_relaxed64(a.ready + f - lag);
        rf_.rdn = ld_relaxed(a.done + f - lag);
      }
    }
    EDGE_T(6);
    PixGuard pg;
    if (a.use_tma) {
      // ---- stage 0: the TMA issued during the previous tile
      tc::mbar_wait(&S.tma_bar, tma_phase);
      tma_phase ^= 1u;
      if (!tile_interior(a, y0, x0)) replicate_box_edges(S, a, y0, x0, tid);
      // inA = raw shifted by 3 columns, checking the guard on the way
#pragma unroll
      for (int i = 0; i < RPW; i++) {
        const int r = warp + i * (THREADS / 32);
        if (r < IR) {
          const float v0 = S.raw[r][lane + 3], v1 = S.raw[r][lane + 35];
          pg.add2(v0, v1);
          S.inA[r][lane] = v0;
          S.inA[r][lane + 32] = v1;
          if (lane < IR - 64) {
            const float v2 = S.raw[r][lane + 67];
            pg.add(v2);
            S.inA[r][lane + 64] = v2;
          }
        }
      }
    } else {
      // ---- stage 0 (border / no TMA): clamped loads, all issued before use
      const float *img = a.in + (size_t)f * n * m;
      float vals[RPW][3];
      const int cx0 = min(max(x0 - 5 + lane, 0), m - 1);
      const int cx1 = min(max(x0 + 27 + lane, 0), m - 1);
      const int cx2 = min(max(x0 + 59 + lane, 0), m - 1);
#pragma unroll
      for (int i = 0; i < RPW; i++) {
        const int r = warp + i * (THREADS / 32);
        const float *row = img + (size_t)min(max(y0 - 5 + min(r, IR - 1), 0), n - 1) * m;
        vals[i][0] = __ldg(row + cx0);
        vals[i][1] = __ldg(row + cx1);
        vals[i][2] = lane < IR - 64 ? __ldg(row + cx2) : 0.0f;
      }
#pragma unroll
      for (int i = 0; i < RPW; i++) {
        const int r = warp + i * (THREADS / 32);
        if (r < IR) {
#pragma unroll
          for (int q2 = 0; q2 < 3; q2++) {
            const int c = q2 * 32 + lane;
            if (c < IR) {
              const float v = vals[i][q2];
              pg.add(v);
              S.inA[r][c] = v;
              S.raw[r][c + 3] = v;
            }
          }
        }
      }
    }
    // thread 0: resolve the claim issued one tile ago (tile t+2), issue the next
    if (tid == 0) {
      publish_desc((int)claim2);
      claim2 = atomicAdd(a.sched, 1u);
    }
    const int all_ok = __syncthreads_and(pg.ok());
    EDGE_T(0);
    const int t2 = S.next_tile, f2 = S.nt_f, y2 = S.nt_y0, x2 = S.nt_x0;
    const bool prefetch = t1 < total && a.use_tma;
    const bool border = (y0 < 2) || (x0 < 2) || (y0 + SR - 2 > n) || (x0 + SR - 2 > m);
    unsigned amax;
    if (filters_fast && all_ok) {
      if (sobel_std && a.use_tma) {
        if (border) amax = edge_tile<true, true, true>(S, a, f, y0, x0, tid, lane, warp, prefetch, f1, y1, x1);
        else amax = edge_tile<true, false, true>(S, a, f, y0, x0, tid, lane, warp, prefetch, f1, y1, x1);
      } else if (border) amax = edge_tile<true, true>(S, a, f, y0, x0, tid, lane, warp, prefetch, f1, y1, x1);
      else amax = edge_tile<true, false>(S, a, f, y0, x0, tid, lane, warp, prefetch, f1, y1, x1);
    } else {
      amax = edge_tile<false, true>(S, a, f, y0, x0, tid, lane, warp, prefetch, f1, y1, x1);
    }
    // ---- tile done + help the reject queue along (at most one unit per
    // tile).  Before the CTA barrier that completes the tile, thread 0
    // decides the unit (its frame's probes were issued at the tile top); the
    // one barrier then publishes P, the warp maxima and the unit.  After it,
    // thread 0 issues the tile's bulk store and atomicMax and counts the
    // previous tile (its store has landed by now; the count's gpu-scope
    // fences are the slow part) while the other warps already run the
    // reject unit.  STG path: the barrier orders the CTA's stores before
    // thread 0's release fence (cumulative).
    if (tid == 0) {
      int v = q.ru, A = 0;
      if (v >= 0) {
        const int rf = v / a.units;
        if (!frame_bound(a, rf, rf_.rr, rf_.rdn, A, q.acq)) {
          // rare: count the previous tile before waiting (others may wait on
          // it; this tile is of frame f != rf and is counted after the wait)
          if (a.use_tma) flush_done(a, q, pd_max, false);
          A = wait_frame(a, rf, q.acq);
        }
      }
      S.hflag = v;
      S.lo = A;
    }
    __syncthreads();
    EDGE_T(4);
    if (tid == 0) {
      if (a.use_tma) {
        // count the previous tile first (its bulk store completed long ago:
        // wait_group 0 before this tile's store is committed), so its fences
        // do not also wait for this tile's fresh atomicMax; then issue this
        // tile's bulk store and max
        flush_done(a, q, pd_max, false);
        EDGE_T(9);
        pd_max = tile_store(S, a, f, y0, x0);  // a register: consumed (waited for) one tile later
        q.pd = f;
      } else {
        (void)tile_store(S, a, f, y0, x0);
        fence_acq_rel();  // orders the CTA's stores (barrier) and the atom before the count
        red_add(a.done + f, 1u);
      }
    }
    (void)amax;
    EDGE_T(7);
    if (S.hflag >= 0) reject_unit(a, S.hflag, S.lo);
    EDGE_T(5);
    tile = t1; f = f1; y0 = y1; x0 = x1;
    t1 = t2; f1 = f2; y1 = y2; x1 = x2;
  }
  // ---- drain: every compute tile is claimed; the last `lag` frames'
  // reject units go through a ticket counter
  const int tail0 = max(a.frames - lag, 0);
  const int tail_units = (a.frames - tail0) * a.units;
  for (;;) {
    if (tid == 0) {
      flush_done(a, q, pd_max, false);
      const int u = (int)atomicAdd(a.sched + 1, 1u);
      int A = 0;
      if (u < tail_units) A = wait_frame(a, tail0 + u / a.units, q.acq);
      S.flag = u < tail_units ? tail0 * a.units + u : -1;
      S.lo = A;
    }
    __syncthreads();
    const int v = S.flag;
    if (v < 0) break;
    reject_unit(a, v, S.lo);
  }
}

// ---------------------------------------------------------------- generic path
// One kernel per Juno stage, any gs/sz/sb, exact scalar arithmetic in the
// oracle's order.  Used for non-(7,3,3) filter sizes and by jb_edge_stages_f32.
struct GenArgs {
  int n, m, gs, sz, sb, frames;
};

__device__ __forceinline__ int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

__global__ void gen_gauss_kernel(GenArgs g, const float *__restrict__ in, const float *__restrict__ gf,
                                 float *__restrict__ sm) {
  const long long total = (long long)g.frames * g.n * g.m;
  const int g2 = g.gs / 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / ((long long)g.n * g.m);
    const int r = (int)((i / g.m) % g.n), c = (int)(i % g.m);
    const float *img = in + f * g.n * g.m;
    float s = 0.0f;
    for (int a = 0; a < g.gs; a++)
      for (int b = 0; b < g.gs; b++)
        s = add_rn(s, mul_rn(img[(size_t)clampi(r + a - g2, g.n - 1) * g.m + clampi(c + b - g2, g.m - 1)],
                             gf[a * g.gs + b]));
    sm[i] = s;
  }
}

template <bool SIGN>
__device__ __forceinline__ float morph_val(const float *img, int n, int m, int y, int x, float pad) {
  if (y < 0 || y >= n || x < 0 || x >= m) return pad;
  const float v = img[(size_t)y * m + x];
  return SIGN ? (v > 0.0f ? 1.0f : 0.0f) : v;
}

// SIGN=false: laplacian_estimate;  SIGN=true: zero_crossings
template <bool SIGN>
__global__ void gen_morph_kernel(GenArgs g, const float *__restrict__ src, const float *__restrict__ st,
                                 float *__restrict__ dst) {
  const long long total = (long long)g.frames * g.n * g.m;
  const int r2 = g.sz / 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / ((long long)g.n * g.m);
    const int r = (int)((i / g.m) % g.n), c = (int)(i % g.m);
    const float *img = src + f * g.n * g.m;
    float d = 0.0f, e = 1.0f;
    for (int a = 0; a < g.sz; a++)
      for (int b = 0; b < g.sz; b++)
        d = py_max(d, mul_rn(morph_val<SIGN>(img, g.n, g.m, r + a - r2, c + b - r2, 0.0f), st[a * g.sz + b]));
    for (int a = 0; a < g.sz; a++)
      for (int b = 0; b < g.sz; b++)
        e = py_min(e, mul_rn(morph_val<SIGN>(img, g.n, g.m, r + a - r2, c + b - r2, 1.0f), st[a * g.sz + b]));
    dst[i] = SIGN ? sub_rn(d, e) : sub_rn(add_rn(d, e), mul_rn(2.0f, img[(size_t)r * g.m + c]));
  }
}

__global__ void gen_grad_kernel(GenArgs g, const float *__restrict__ sm, const float *__restrict__ sx,
                                const float *__restrict__ sy, float *__restrict__ grad,
                                unsigned *__restrict__ fmax) {
  const long long total = (long long)g.frames * g.n * g.m;
  const int b2 = g.sb / 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / ((long long)g.n * g.m);
    const int r = (int)((i / g.m) % g.n), c = (int)(i % g.m);
    const float *img = sm + f * g.n * g.m;
    float gx = 0.0f, gy = 0.0f;
    for (int a = 0; a < g.sb; a++)
      for (int b = 0; b < g.sb; b++) {
        const float v = img[(size_t)clampi(r + a - b2, g.n - 1) * g.m + clampi(c + b - b2, g.m - 1)];
        gx = add_rn(gx, mul_rn(v, sx[a * g.sb + b]));
        gy = add_rn(gy, mul_rn(v, sy[a * g.sb + b]));
      }
    const float v = __fsqrt_rn(add_rn(mul_rn(gx, gx), mul_rn(gy, gy)));
    grad[i] = v;
    if (!(v != v)) atomicMax(fmax + f, __float_as_uint(v));
  }
}

__global__ void gen_reject_kernel(GenArgs g, const float *__restrict__ zc, const float *__restrict__ grad,
                                  const unsigned *__restrict__ fmax, float theta, float *__restrict__ out,
                                  float *__restrict__ maxg_out) {
  const long long fpx = (long long)g.n * g.m, total = g.frames * fpx;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / fpx;
    const float g00 = grad[f * fpx];
    const float mx = (g00 != g00) ? g00 : __uint_as_float(fmax[f]);
    if (maxg_out && i == f * fpx) maxg_out[f] = mx;
    out[i] = (zc[i] > 0.0f && grad[i] > mul_rn(theta, mx)) ? 1.0f : 0.0f;
  }
}

static int grid_for(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  long long cap = (long long)sm_count() * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

static jb_status run_generic(uint64_t batch, uint64_t n, uint64_t m, uint64_t gs, uint64_t sz,
                             uint64_t sb, const float *in, const float *gf, const float *st,
                             const float *sx, const float *sy, float theta, float *out,
                             float *sm_o, float *lap_o, float *zc_o, float *grad_o, float *maxg_o,
                             cudaStream_t s) {
  const size_t px = (size_t)batch * n * m;
  const size_t need_tmp = (sm_o ? 0 : px) + (lap_o ? 0 : px) + (zc_o ? 0 : px) + (grad_o ? 0 : px);
  char *ws = (char *)workspace(need_tmp * 4 + batch * 4 + 256, s);
  if (!ws) return JB_ECUDA;
  unsigned *fmax = (unsigned *)ws;
  float *p = (float *)(ws + ((batch * 4 + 255) / 256) * 256);
  float *sm = sm_o ? sm_o : p;
  if (!sm_o) p += px;
  float *lap = lap_o ? lap_o : p;
  if (!lap_o) p += px;
  float *zc = zc_o ? zc_o : p;
  if (!zc_o) p += px;
  float *grad = grad_o ? grad_o : p;
  GenArgs g{(int)n, (int)m, (int)gs, (int)sz, (int)sb, (int)batch};
  const int T = 256, B = grid_for((long long)px, T);
  JB_CHECK_CUDA(cudaMemsetAsync(fmax, 0, batch * 4, s));
  gen_gauss_kernel<<<B, T, 0, s>>>(g, in, gf, sm);
  JB_LAUNCHED("edge gaussian");
  gen_morph_kernel<false><<<B, T, 0, s>>>(g, sm, st, lap);
  JB_LAUNCHED("edge laplacian");
  gen_morph_kernel<true><<<B, T, 0, s>>>(g, lap, st, zc);
  JB_LAUNCHED("edge zero_crossings");
  gen_grad_kernel<<<B, T, 0, s>>>(g, sm, sx, sy, grad, fmax);
  JB_LAUNCHED("edge gradient");
  gen_reject_kernel<<<B, T, 0, s>>>(g, zc, grad, fmax, theta, out, maxg_o);
  JB_LAUNCHED("edge reject");
  return JB_OK;
}

static jb_status validate(uint64_t batch, uint64_t n, uint64_t m, uint64_t gs, uint64_t sz,
                          uint64_t sb, const void *in, const void *out) {
  JB_REQUIRE(n >= 1 && m >= 1, "edge_detection: n and m must be >= 1 (got %llu, %llu)",
             (unsigned long long)n, (unsigned long long)m);
  JB_REQUIRE(gs >= 1 && sz >= 1 && sb >= 1, "edge_detection: filter sizes must be >= 1");
  JB_REQUIRE(n * m < (1ull << 31) && batch < (1ull << 31), "edge_detection: frame too large");
  JB_REQUIRE(in && out, "edge_detection: null input/output");
  return JB_OK;
}

}  // namespace edge
}  // namespace jb

using namespace jb;
using namespace jb::edge;

namespace jb {
namespace edge {

// f32 edge maps (exactly 0 or 1) -> bit-packed words, frame by frame
__global__ void pack_bits_kernel(const float *__restrict__ maps, long long frame_px, long long frame_words,
                                 long long words, uint32_t *__restrict__ bits) {
  const int lane = threadIdx.x & 31;
  for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < words;
       w += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long f = w / frame_words, j = (w - f * frame_words) * 32 + lane;
    const unsigned b = __ballot_sync(0xffffffffu, j < frame_px && maps[f * frame_px + j] != 0.0f);
    if (lane == 0) bits[w] = b;
  }
}

// the fused path (gs = 7, sz = 3, sb = 3) writing f32 maps (out) or packed bits (obits)
static jb_status run_fused(uint64_t batch, uint64_t n, uint64_t m, const float *in, const float *gf,
                           const float *st, const float *sx, const float *sy, float theta, float *out,
                           uint32_t *obits, cudaStream_t s) {
  const size_t frame_px = (size_t)n * m;
  const int tiles_x = (int)((m + TW - 1) / TW), tiles_y = (int)((n + TH - 1) / TH);
  const int tpf = tiles_x * tiles_y;
  JB_REQUIRE((uint64_t)tpf * batch < (1ull << 31), "edge_detection: batch too large");
  // packed-gradient ring: as many frame slots as fit ~64 MB of L2 (>= 2)
  const size_t slot_px = (frame_px + 1023) / 1024 * 1024;
#ifndef EDGE_RING_MB
#define EDGE_RING_MB 64
#endif
  size_t ring = ((size_t)EDGE_RING_MB << 20) / (slot_px * 4);
  if (ring < 2) ring = 2;
  if (ring > batch) ring = batch;
  // reject units: about seven compute tiles' pixels each (one unit per ~7
  // tiles), whole 4 KB blocks of lines.  A unit's fixed cost (its CTA
  // barrier, the discard fence, the count) favours large units, load
  // balance small ones: JB_EDGE_UNIT_PX A/B at 1080p (frames/s): 8192 69.7 k,
  // 16384 72.3 k, 24576-28672 73.1 k, 32768 73.0 k, 65536 67.2 k.
  size_t unit_px = ((7 * frame_px + tpf - 1) / tpf + 1023) / 1024 * 1024;
  if (const char *e = getenv("JB_EDGE_UNIT_PX")) {  // experiments: a multiple of 1024
    const long long u = atoll(e);
    if (u >= 1024 && u % 1024 == 0) unit_px = (size_t)u;
  }
  if (unit_px > ((frame_px + 1023) / 1024) * 1024) unit_px = ((frame_px + 1023) / 1024) * 1024;
  const size_t units = (frame_px + unit_px - 1) / unit_px;
  const size_t ring_bytes = ring * slot_px * 4;
  const size_t pf = ((batch * 8 + 255) / 256) * 256;  // one per-frame array (<= 8 B/frame)
  // control block: fmax | done | rdone | pub | rj | ready (u64) | sched[2] + flags[2]
  const size_t ctl_bytes = 6 * pf + 256;
  char *ws = (char *)workspace(ring_bytes + ctl_bytes, s);
  if (!ws) return JB_ECUDA;
  uint32_t *packed = (uint32_t *)ws;
  char *ctl = ws + ring_bytes;
  FusedArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.fmax = (unsigned *)ctl;
  fa.done = (unsigned *)(ctl + pf);
  fa.rdone = (unsigned *)(ctl + 2 * pf);
  fa.pub = (unsigned *)(ctl + 3 * pf);
  fa.rj = (unsigned *)(ctl + 4 * pf);
  fa.ready = (unsigned long long *)(ctl + 5 * pf);
  fa.sched = (unsigned *)(ctl + 6 * pf);
  int *flags = (int *)(ctl + 6 * pf + 128);

  // The filters live in this device's __constant__ bank, which every stream
  // shares: a call on another stream than the previous one first waits for
  // the previous call's kernels (recorded below), so it cannot overwrite
  // filters a running kernel still reads.
  std::unique_lock<std::mutex> bank_lock(g_bank_mu);
  int bdev = 0;
  cudaGetDevice(&bdev);
  ConstBank &bank = g_bank[{bdev, 0}];
  if (bank.ev && bank.stream != s) JB_CHECK_CUDA(cudaStreamWaitEvent(s, bank.ev, 0));
  JB_CHECK_CUDA(cudaMemcpyToSymbolAsync(c_gauss, gf, 49 * 4, 0, cudaMemcpyDeviceToDevice, s));
  JB_CHECK_CUDA(cudaMemcpyToSymbolAsync(c_struct, st, 9 * 4, 0, cudaMemcpyDeviceToDevice, s));
  JB_CHECK_CUDA(cudaMemcpyToSymbolAsync(c_sx, sx, 9 * 4, 0, cudaMemcpyDeviceToDevice, s));
  JB_CHECK_CUDA(cudaMemcpyToSymbolAsync(c_sy, sy, 9 * 4, 0, cudaMemcpyDeviceToDevice, s));
  JB_CHECK_CUDA(cudaMemsetAsync(ctl, 0, 6 * pf + 128, s));
  edge_check_kernel<<<1, 32, 0, s>>>(gf, st, sx, sy, flags);
  JB_LAUNCHED("edge_check");

  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  const int smem = (int)sizeof(Smem) + 128;
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    JB_CHECK_CUDA(cudaFuncSetAttribute(edge_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set[dev] = true;
  }
  fa.in = in;
  fa.out = out;
  fa.packed = packed;
  fa.flags = flags;
  fa.theta = theta;
  fa.n = (int)n; fa.m = (int)m; fa.frames = (int)batch; fa.tiles_x = tiles_x; fa.tiles_y = tiles_y;
  fa.ring = (int)ring; fa.units = (int)units; fa.unit_px = (int)unit_px;
  // lag: tiles in flight (3 per CTA: current + two claimed) span ~2.3
  // 1080p frames, so frame f is complete by the time frame f+4's tiles end;
  // lag <= ring - 2 keeps the slot of frame f + ring free when it is needed
  fa.lag = (int)(ring >= 6 ? 4 : (ring >= 3 ? ring - 2 : 1));
  if (const char *e = getenv("JB_EDGE_LAG")) {  // experiments: 1 <= lag <= ring - 2
    const int l = atoi(e);
    if (l >= 1 && l <= (int)ring - 2) fa.lag = l;
  }
  fa.obits = obits;
  fa.frame_words = (long long)((frame_px + 31) / 32);
  fa.vec4 = frame_px % 4 == 0 && (obits != nullptr || ((uintptr_t)out % 16) == 0);
  fa.frame_px = (long long)frame_px; fa.slot_px = (long long)slot_px;
  {
    const char *e = getenv("JB_EDGE_OPTS");
    fa.opts = e ? atoi(e) : 0;
  }
  fa.use_tma = 0;
  if (m % 4 == 0 && ((uintptr_t)in % 16) == 0 && tmap_encode_fn() != nullptr) {
    const uint64_t dims[3] = {m, n, (uint64_t)batch};
    const uint64_t strides[2] = {m * 4, n * m * 4};
    const uint32_t box[3] = {(uint32_t)RP, (uint32_t)IR, 1};
    fa.use_tma = make_tmap_f32(&fa.tmap, in, 3, dims, strides, box, 0) ? 1 : 0;
    // the packed ring as [ring][n][m] u32 (bit copies: the f32 map type is fine)
    const uint64_t pdims[3] = {m, n, (uint64_t)ring};
    const uint64_t pstrides[2] = {m * 4, slot_px * 4};
    const uint32_t pbox[3] = {(uint32_t)TW, (uint32_t)TH, 1};
    if (fa.use_tma && !make_tmap_f32(&fa.pmap, packed, 3, pdims, pstrides, pbox, 0)) fa.use_tma = 0;
  }
  const long long total = (long long)tpf * batch;
  const int grid = total < sm_count() * EDGE_MINB ? (int)total : sm_count() * EDGE_MINB;
  void *tok = prof_begin("edge_fused", s);
  edge_fused_kernel<<<grid, THREADS, smem, s>>>(fa);
  prof_end(tok, s);
  JB_LAUNCHED("edge_fused");
  if (!bank.ev) JB_CHECK_CUDA(cudaEventCreateWithFlags(&bank.ev, cudaEventDisableTiming));
  JB_CHECK_CUDA(cudaEventRecord(bank.ev, s));
  bank.stream = s;
  return JB_OK;
}

}  // namespace edge
}  // namespace jb

extern "C" jb_status jb_edge_f32(uint64_t batch, uint64_t n, uint64_t m, uint64_t gs, uint64_t sz,
                                 uint64_t sb, const float *in, const float *gf, const float *st,
                                 const float *sx, const float *sy, float theta, float *out,
                                 void *stream) {
  jb_status v = validate(batch, n, m, gs, sz, sb, in, out);
  if (v != JB_OK) return v;
  if (batch == 0) return JB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (!(gs == 7 && sz == 3 && sb == 3))
    return run_generic(batch, n, m, gs, sz, sb, in, gf, st, sx, sy, theta, out, nullptr, nullptr,
                       nullptr, nullptr, nullptr, s);
  return run_fused(batch, n, m, in, gf, st, sx, sy, theta, out, nullptr, s);
}

extern "C" jb_status jb_edge_bits_f32(uint64_t batch, uint64_t n, uint64_t m, uint64_t gs, uint64_t sz,
                                      uint64_t sb, const float *in, const float *gf, const float *st,
                                      const float *sx, const float *sy, float theta, uint32_t *out_bits,
                                      void *stream) {
  jb_status v = validate(batch, n, m, gs, sz, sb, in, out_bits);
  if (v != JB_OK) return v;
  if (batch == 0) return JB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (gs == 7 && sz == 3 && sb == 3) return run_fused(batch, n, m, in, gf, st, sx, sy, theta, nullptr, out_bits, s);
  // other filter sizes: the per-stage kernels into f32 maps at the arena's
  // tail, then one packing pass.  run_generic asks the arena for its head
  // only (<= the capacity reserved here, so the block does not move).
  const size_t px = (size_t)batch * n * m;
  const size_t head = (4 * px * 4 + batch * 4 + 256 + 255) / 256 * 256;
  char *ws = (char *)workspace(head + px * 4, s);
  if (!ws) return JB_ECUDA;
  float *maps = (float *)(ws + head);
  v = run_generic(batch, n, m, gs, sz, sb, in, gf, st, sx, sy, theta, maps, nullptr, nullptr, nullptr,
                  nullptr, nullptr, s);
  if (v != JB_OK) return v;
  const long long fw = (long long)((n * m + 31) / 32), words = fw * (long long)batch;
  pack_bits_kernel<<<grid_for(words * 32, 256), 256, 0, s>>>(maps, (long long)(n * m), fw, words, out_bits);
  JB_LAUNCHED("edge pack_bits");
  return JB_OK;
}

#ifdef EDGE_STAGE_CLOCKS
extern "C" JB_API void jb_edge_stage_clocks(unsigned long long *out) {
  cudaMemcpyFromSymbol(out, g_edge_clk, sizeof(unsigned long long) * 16);
}
#endif

extern "C" jb_status jb_edge_stages_f32(uint64_t batch, uint64_t n, uint64_t m, uint64_t gs,
                                        uint64_t sz, uint64_t sb, const float *in, const float *gf,
                                        const float *st, const float *sx, const float *sy, float theta,
                                        float *out, float *smoothed, float *laplacian, float *zc,
                                        float *gradient, float *max_gradient, void *stream) {
  jb_status v = validate(batch, n, m, gs, sz, sb, in, out);
  if (v != JB_OK) return v;
  if (batch == 0) return JB_OK;
  return run_generic(batch, n, m, gs, sz, sb, in, gf, st, sx, sy, theta, out, smoothed, laplacian, zc,
                     gradient, max_gradient, (cudaStream_t)stream);
}
