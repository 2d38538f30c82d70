// backprop.cu -- one Rodinia bpnn_train step on sm_100a
// (oracle/juno_oracle.c:jo_bp_train, BP):
//   hidden = squash(W_ih^T x)      layerforward, W_ih (n_in+1) x (n_hid+1)
//   output = squash(W_ho^T hidden) layerforward
//   delta_o, delta_h, errors       output_error / hidden_error
//   W_ho, W_ih += eta*delta*y + momentum*oldW ; oldW = that step
//
// B200 design: the two passes over the 1.07 GiB input
// weight matrix are HBM streams; everything on the hidden/output side is a
// few hundred values and runs in one small CTA.
//  * bp_forward_kernel: grid-stride over input rows k, f32 products
//    w[k][j]*x[k] accumulated in f64 per thread, warp -> block -> grid
//    (last-CTA ticket, fixed order) reduction -> 16 hidden sums.
//  * bp_small_kernel: squash, hidden->output layer, errors, deltas and the
//    hidden->output weight update (1 CTA).
//  * bp_adjust_kernel: float4 stream over the flat W_ih / oldW arrays
//    (read 8 B, write 8 B per weight).
// The layer sums are the associative reduction the paper's schedule
// parallelises; both sides accumulate them in f64, the rest is
// op-for-op the oracle's single-rounding f32 arithmetic.
#include <stdlib.h>

#include "common.cuh"
#include "tcgen05.cuh"

namespace jb {
namespace bp {

constexpr float ETA = 0.3f, MOMENTUM = 0.3f;
constexpr int MAXH = 32;  // hidden units supported by the fused kernels
constexpr int THREADS = 256;

__device__ __forceinline__ float squash(float x) { return div_rn(1.0f, add_rn(1.0f, exp_ref(-x))); }

struct FwdArgs {
  const float *x;   // input units (x[0] treated as the bias 1.0)
  const float *w;   // (n_in+1) x (n_hid+1)
  double *partials; // [grid][MAXH]
  unsigned *ticket;
  double *sums;     // [n_hid+1] f64 sums (index 1..n_hid)
  long long rows;   // n_in + 1
  int nh1;          // n_hid + 1
};

template <int NH>
__global__ void __launch_bounds__(THREADS) bp_forward_kernel(FwdArgs a) {
  double acc[NH];
#pragma unroll
  for (int j = 0; j < NH; j++) acc[j] = 0.0;
  for (long long k = blockIdx.x * (long long)THREADS + threadIdx.x; k < a.rows;
       k += (long long)gridDim.x * THREADS) {
    const float xk = k == 0 ? 1.0f : __ldg(a.x + k);
    const float *row = a.w + k * (NH + 1);
#pragma unroll
    for (int j = 0; j < NH; j++) acc[j] += (double)mul_rn(__ldg(row + 1 + j), xk);
  }
  __shared__ double sh[THREADS / 32][NH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NH; j++) {
    const double v = warp_sum(acc[j]);
    if (lane == 0) sh[warp][j] = v;
  }
  __syncthreads();
  if (threadIdx.x < NH) {
    double v = 0.0;
    for (int w = 0; w < THREADS / 32; w++) v += sh[w][threadIdx.x];
    a.partials[(size_t)blockIdx.x * MAXH + threadIdx.x] = v;
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < NH) {
    double v = 0.0;
    for (unsigned b = 0; b < gridDim.x; b++) v += ((volatile double *)a.partials)[(size_t)b * MAXH + threadIdx.x];
    a.sums[1 + threadIdx.x] = v;
  }
  if (threadIdx.x == 0) *a.ticket = 0;
}

// The same layer sum with the weight rows streamed into shared memory by
// 1-D bulk copies (TMA), two chunks of THREADS rows in flight per CTA: HBM
// sees whole 16-byte-aligned chunks instead of every thread's 68-byte rows
// through scalar loads.  Thread t takes row t of a chunk (odd row pitch NH+1
// words: conflict-free LDS).  Rows after the last whole chunk take the
// direct loads.  Same per-thread f64 accumulation and reduction order per
// thread as bp_forward_kernel, so the f64 sums round to the same f32 values.
template <int NH>
__global__ void __launch_bounds__(THREADS) bp_forward_tma_kernel(FwdArgs a) {
  constexpr int RW = NH + 1;                        // row pitch (words)
  constexpr uint32_t CB = THREADS * RW * 4;         // chunk bytes (a multiple of 16)
  extern __shared__ __align__(128) float fbuf[];    // [2][THREADS * RW]
  __shared__ __align__(8) uint64_t bar[2];
  double acc[NH];
#pragma unroll
  for (int j = 0; j < NH; j++) acc[j] = 0.0;
  const long long chunks = a.rows / THREADS;
  const long long mine = chunks > blockIdx.x ? (chunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint64_t pol = tc::policy_evict_first();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
    for (int b = 0; b < 2 && b < mine; b++) {
      const long long c = blockIdx.x + (long long)b * gridDim.x;
      tc::mbar_arrive_expect_tx(&bar[b], CB);
      tc::bulk_load_1d(fbuf + b * THREADS * RW, a.w + c * THREADS * RW, CB, &bar[b], pol);
    }
  }
  __syncthreads();
  for (long long i = 0; i < mine; i++) {
    const int b = (int)(i & 1);
    const long long c = blockIdx.x + i * gridDim.x;
    const long long k = c * THREADS + threadIdx.x;
    const float xk = k == 0 ? 1.0f : __ldg(a.x + k);
    tc::mbar_wait(&bar[b], (uint32_t)((i >> 1) & 1));
    const float *row = fbuf + b * THREADS * RW + threadIdx.x * RW;
#pragma unroll
    for (int j = 0; j < NH; j++) acc[j] += (double)mul_rn(row[1 + j], xk);
    __syncthreads();  // every thread is done with buffer b
    if (threadIdx.x == 0 && i + 2 < mine) {
      const long long c2 = c + 2 * (long long)gridDim.x;
      tc::fence_proxy_async_smem();
      tc::mbar_arrive_expect_tx(&bar[b], CB);
      tc::bulk_load_1d(fbuf + b * THREADS * RW, a.w + c2 * THREADS * RW, CB, &bar[b], pol);
    }
  }
  // the rows after the last whole chunk: the CTA and thread the direct
  // kernel's grid-stride gives them, so every thread folds the same rows in
  // the same order as bp_forward_kernel
  if (blockIdx.x == (unsigned)(chunks % gridDim.x)) {
    const long long k = chunks * THREADS + threadIdx.x;
    if (k < a.rows) {
      const float xk = k == 0 ? 1.0f : __ldg(a.x + k);
      const float *row = a.w + k * RW;
#pragma unroll
      for (int j = 0; j < NH; j++) acc[j] += (double)mul_rn(__ldg(row + 1 + j), xk);
    }
  }
  __shared__ double sh[THREADS / 32][NH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NH; j++) {
    const double v = warp_sum(acc[j]);
    if (lane == 0) sh[warp][j] = v;
  }
  __syncthreads();
  if (threadIdx.x < NH) {
    double v = 0.0;
    for (int w = 0; w < THREADS / 32; w++) v += sh[w][threadIdx.x];
    a.partials[(size_t)blockIdx.x * MAXH + threadIdx.x] = v;
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < NH) {
    double v = 0.0;
    for (unsigned b = 0; b < gridDim.x; b++) v += ((volatile double *)a.partials)[(size_t)b * MAXH + threadIdx.x];
    a.sums[1 + threadIdx.x] = v;
  }
  if (threadIdx.x == 0) *a.ticket = 0;
}

template <int NH>
static jb_status launch_forward(const FwdArgs &fa, int grid, cudaStream_t s, bool tma) {
  if (!tma) {
    bp_forward_kernel<NH><<<grid, THREADS, 0, s>>>(fa);
    return JB_OK;
  }
  const int smem = 2 * THREADS * (NH + 1) * 4;
  static bool attr[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr[dev]) {
    JB_CHECK_CUDA(cudaFuncSetAttribute(bp_forward_tma_kernel<NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr[dev] = true;
  }
  bp_forward_tma_kernel<NH><<<grid, THREADS, smem, s>>>(fa);
  return JB_OK;
}

// hidden side of the step, one CTA (n_hid, n_out <= MAXH)
__global__ void bp_small_kernel(const double *sums, float *x, float *hw, float *hpw, const float *target,
                                float *hidden, float *output, float *delta_h, float *errs, int nh, int no) {
  __shared__ float sh_hidden[MAXH + 1], sh_out[MAXH + 1], sh_do[MAXH + 1];
  const int t = threadIdx.x;
  if (t == 0) {
    x[0] = 1.0f;  // bpnn_layerforward sets l1[0] = 1.0 (in place, like Rodinia)
    sh_hidden[0] = 1.0f;
  }
  if (t >= 1 && t <= nh) sh_hidden[t] = squash((float)sums[t]);
  __syncthreads();
  // hidden -> output layerforward (sequential f32 fold over k, as the oracle)
  if (t >= 1 && t <= no) {
    float s = 0.0f;
    for (int k = 0; k <= nh; k++) s = add_rn(s, mul_rn(hw[k * (no + 1) + t], sh_hidden[k]));
    sh_out[t] = squash(s);
  }
  __syncthreads();
  if (t == 0) {
    sh_out[0] = 0.0f;
    float eo = 0.0f;
    for (int j = 1; j <= no; j++) {
      const float o = sh_out[j], tg = target[j];
      sh_do[j] = mul_rn(mul_rn(o, sub_rn(1.0f, o)), sub_rn(tg, o));
      eo = add_rn(eo, fabsf(sh_do[j]));
    }
    float eh = 0.0f;
    for (int j = 1; j <= nh; j++) {
      const float h = sh_hidden[j];
      float s = 0.0f;
      for (int k = 1; k <= no; k++) s = add_rn(s, mul_rn(sh_do[k], hw[j * (no + 1) + k]));
      const float dh = mul_rn(mul_rn(h, sub_rn(1.0f, h)), s);
      delta_h[j] = dh;
      eh = add_rn(eh, fabsf(dh));
    }
    errs[0] = eo;
    errs[1] = eh;
    delta_h[0] = 0.0f;
  }
  __syncthreads();
  if (t <= nh) hidden[t] = sh_hidden[t];
  if (t <= no) output[t] = t == 0 ? 0.0f : sh_out[t];
  // adjust_weights(delta_o, no, hidden, nh, hw, hpw): k over hidden units
  for (int idx = t; idx < (nh + 1) * no; idx += blockDim.x) {
    const int k = idx / no, j = 1 + idx % no;
    const int x2 = k * (no + 1) + j;
    const float ly = sh_hidden[k];
    const float nd = add_rn(mul_rn(mul_rn(ETA, sh_do[j]), ly), mul_rn(MOMENTUM, hpw[x2]));
    hw[x2] = add_rn(hw[x2], nd);
    hpw[x2] = nd;
  }
}

// W_ih/oldW stream: element e of the flat (n_in+1) x (n_hid+1) arrays
__global__ void __launch_bounds__(THREADS) bp_adjust_kernel(const float *__restrict__ delta_h,
                                                            const float *__restrict__ x, float *__restrict__ w,
                                                            float *__restrict__ oldw, long long total, int nh1) {
  __shared__ float sd[MAXH + 1];
  if (threadIdx.x < nh1) sd[threadIdx.x] = delta_h[threadIdx.x];
  __syncthreads();
  const float ly0 = 1.0f;  // input[0] is the bias after layerforward
  const long long total4 = total / 4;
  float4 *w4 = reinterpret_cast<float4 *>(w);
  float4 *o4 = reinterpret_cast<float4 *>(oldw);
  for (long long i = blockIdx.x * (long long)THREADS + threadIdx.x; i < total4; i += (long long)gridDim.x * THREADS) {
    float4 wv = w4[i], ov = o4[i];
    float *wp = &wv.x, *op = &ov.x;
    long long e = i * 4;
    long long k = e / nh1;
    int j = (int)(e - k * nh1);
#pragma unroll
    for (int q = 0; q < 4; q++) {
      if (j != 0) {
        const float ly = k == 0 ? ly0 : __ldg(x + k);
        const float nd = add_rn(mul_rn(mul_rn(ETA, sd[j]), ly), mul_rn(MOMENTUM, op[q]));
        wp[q] = add_rn(wp[q], nd);
        op[q] = nd;
      }
      if (++j == nh1) { j = 0; k++; }
    }
    w4[i] = wv;
    o4[i] = ov;
  }
  // tail
  for (long long e = total4 * 4 + blockIdx.x * (long long)THREADS + threadIdx.x; e < total;
       e += (long long)gridDim.x * THREADS) {
    const long long k = e / nh1;
    const int j = (int)(e - k * nh1);
    if (j == 0) continue;
    const float ly = k == 0 ? ly0 : __ldg(x + k);
    const float nd = add_rn(mul_rn(mul_rn(ETA, sd[j]), ly), mul_rn(MOMENTUM, oldw[e]));
    w[e] = add_rn(w[e], nd);
    oldw[e] = nd;
  }
}

}  // namespace bp
}  // namespace jb

using namespace jb;
using namespace jb::bp;

extern "C" jb_status jb_bp_train_f32(uint64_t n_in, uint64_t n_hid, uint64_t n_out, float *input, float *in_w,
                                     float *hid_w, const float *target, float *in_prev_w, float *hid_prev_w,
                                     float *hidden, float *output, float *errs, void *stream) {
  JB_REQUIRE(n_in >= 1 && n_hid >= 1 && n_out >= 1, "backprop: layer sizes must be >= 1");
  JB_REQUIRE(n_hid == 16 || n_hid == 8 || n_hid == 4 || n_hid == 32,
             "backprop: hidden layer of %llu units (kernels are built for 4/8/16/32)", (unsigned long long)n_hid);
  JB_REQUIRE(n_out <= (uint64_t)MAXH, "backprop: at most %d output units", MAXH);
  JB_REQUIRE(input && in_w && hid_w && target && in_prev_w && hid_prev_w && hidden && output && errs,
             "backprop: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = sm_count() * 4;
  const size_t part_bytes = (size_t)grid * MAXH * sizeof(double);
  char *ws = (char *)workspace(part_bytes + 1024 + 512, s);
  if (!ws) return JB_ECUDA;
  double *partials = (double *)ws;
  double *sums = (double *)(ws + part_bytes);
  float *delta_h = (float *)(ws + part_bytes + 512);
  unsigned *ticket = (unsigned *)(ws + part_bytes + 1024);
  JB_CHECK_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
  FwdArgs fa{input, in_w, partials, ticket, sums, (long long)n_in + 1, (int)n_hid + 1};
  void *tok = prof_begin("bp_forward", s);
  // the weight rows stream through shared memory by bulk copy when the
  // matrix is 16-byte aligned (JB_BP_DIRECT=1: the direct-load kernel)
  static const bool direct = [] {
    const char *e = getenv("JB_BP_DIRECT");
    return e && atoi(e) == 1;
  }();
  const bool tma = !direct && ((uintptr_t)in_w % 16) == 0;
  jb_status fs;
  switch (n_hid) {
    case 4: fs = launch_forward<4>(fa, grid, s, tma); break;
    case 8: fs = launch_forward<8>(fa, grid, s, tma); break;
    case 16: fs = launch_forward<16>(fa, grid, s, tma); break;
    default: fs = launch_forward<32>(fa, grid, s, tma); break;
  }
  if (fs != JB_OK) return fs;
  prof_end(tok, s);
  JB_LAUNCHED("bp_forward");
  bp_small_kernel<<<1, 64, 0, s>>>(sums, input, hid_w, hid_prev_w, target, hidden, output, delta_h, errs,
                                   (int)n_hid, (int)n_out);
  JB_LAUNCHED("bp_small");
  const long long total = (long long)(n_in + 1) * (long long)(n_hid + 1);
  const bool aligned = ((uintptr_t)in_w % 16 == 0) && ((uintptr_t)in_prev_w % 16 == 0);
  JB_REQUIRE(aligned, "backprop: weight arrays must be 16-byte aligned");
  tok = prof_begin("bp_adjust", s);
  bp_adjust_kernel<<<grid, THREADS, 0, s>>>(delta_h, input, in_w, in_prev_w, total, (int)n_hid + 1);
  prof_end(tok, s);
  JB_LAUNCHED("bp_adjust");
  return JB_OK;
}
