// bfs.cu -- bfs<n,m>(starting u32[n], no_of_edges u32[n], edges u32[m], source)
//           -> cost i32[n]    (Rodinia BFS; oracle/juno_oracle.c:jo_bfs)
//
// Levels of a breadth-first search are order independent, so the result is
// bit-identical to the oracle for any traversal order.
//
// B200 design: one persistent cooperative kernel runs every
// level (no host round trip per level):
//  * top-down frontier-queue expansion, two frontier vertices per thread
//    per round; a warp lays its vertices' adjacency ranges back to back in a
//    shared edge-id buffer (warp scan) and all 32 lanes walk it together,
//    8 edges per lane per batch whose edge-id loads, visited probes and
//    claiming atomics are each issued back to back (balanced lanes whatever
//    the degrees; memory-level parallelism instead of three dependent round
//    trips per edge);
//  * a visited bitmap (n/8 bytes: 2 MiB at n = 2^24, L2-resident) filters
//    the random neighbour probes before the claiming atomicOr;
//  * levels go to a byte array (n bytes, L2-resident) instead of random
//    4-byte writes into the HBM cost array; one coalesced pass at the end
//    expands it to i32 costs (levels >= 254 are rare and written directly);
//  * newly claimed vertices go to a block-local queue in shared memory
//    (shared-memory atomics), then one global atomicAdd per block reserves
//    space in the next frontier (block-aggregated atomics);
//  * large levels skip the queue altogether ("dense output"): a claim is a
//    level-byte check in L2 + a plain byte store (every writer of a vertex
//    in one level writes the same level, so the race is benign), no
//    claiming atomics, no bitmap probe or update, no block barriers; the
//    next level finds its frontier in the level bytes: by scanning all n
//    of them when it is large, else by compacting them into a queue first;
//    a queue-output level after it first rebuilds the bitmap from them
//    (32 vertices per word);
//  * one grid-wide barrier (cooperative groups) per level: the frontier
//    sizes rotate through three counters, so the one two levels ahead is
//    cleared while the current one is read.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace jb {
namespace bfs {

constexpr int THREADS = 512;
constexpr int LQ = 4096;  // block-local queue capacity
#ifndef BFS_EB
#define BFS_EB 8
#endif
#ifndef BFS_VPT
#define BFS_VPT 2
#endif
#ifndef BFS_SCAN_SHIFT
#define BFS_SCAN_SHIFT 1  // frontiers > n / 2^shift are read by scanning the level bytes, smaller ones compacted into a queue (A/B: 0 83.7, 1 83.4, 2 80.8, 3 80.6 GTEPS)
#endif
#ifndef BFS_DENSE_SHIFT
#define BFS_DENSE_SHIFT 4  // queue-less output for frontiers >= n / 2^shift (A/B: 3 79.1, 4 80.5, 5 80.0 GTEPS)
#endif
constexpr int EB = BFS_EB;       // edges per lane per batch
constexpr int CAP = 32 * EB;     // per-warp edge-id buffer (one batch)
constexpr int VPT = BFS_VPT;  // frontier vertices per thread per round
constexpr uint8_t kUnseen = 0xFF, kDeep = 0xFE;  // level byte codes

#ifndef BFS_PACK
#define BFS_PACK 0  // 1: (starting, no_of_edges) packed into one 8-byte record per vertex by a prologue
#endif

struct Args {
  const uint32_t *starting, *nedges, *edges;
  const uint2 *rec;   // BFS_PACK: [n] (starting, no_of_edges)
  int32_t *cost;
  uint8_t *level;     // [n] level byte (kUnseen / level / kDeep: see cost[])
  uint32_t *visited;  // bitmap
  uint32_t *q[2];     // frontier queues
  uint32_t *qsize;    // [8]: frontier sizes, slot level % 3; compaction counts at 4 + level % 2
  uint32_t n;
};

// the CSR arrays are streamed (each edge id read once per traversal):
// evict-first loads keep the L2-resident level bytes and visited bitmap in L2
#ifdef BFS_LDG
#define CSR_LD(p) __ldg(p)
#else
#define CSR_LD(p) __ldcs(p)
#endif

// bit i set where byte i of x is not kUnseen (0xFF)
__device__ __forceinline__ uint32_t seen4(uint32_t x) {
  const uint32_t r = __vcmpne4(x, 0xFFFFFFFFu) & 0x80808080u;
  return (r * 0x00204081u) >> 28;
}

__device__ __forceinline__ void red_or(uint32_t *p, uint32_t v) {
  asm volatile("red.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void enqueue(uint32_t *nsize, uint32_t v, uint32_t *lq, uint32_t &lcount,
                                        uint32_t *nq) {
  const uint32_t slot = atomicAdd(&lcount, 1u);
  if (slot < LQ) {
    lq[slot] = v;
  } else {  // overflow: warp-aggregated direct append
    const uint32_t mask = __activemask();
    const int leader = __ffs(mask) - 1;
    uint32_t base = 0;
    if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(nsize, __popc(mask));
    base = __shfl_sync(mask, base, leader);
    nq[base + __popc(mask & ((1u << (threadIdx.x & 31)) - 1))] = v;
  }
}

#ifdef BFS_TRACE
// per-level globaltimer stamps of block 0 (tools/bfs_trace.py)
__device__ unsigned long long g_bfs_trace[64];
#define BFS_T(level)                                                               \
  do {                                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (level) < 64) {                     \
      unsigned long long t;                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                        \
      g_bfs_trace[level] = t;                                                      \
    }                                                                              \
  } while (0)
#else
#define BFS_T(level) do {} while (0)
#endif

#ifndef BFS_MINB
#define BFS_MINB 2  // 2 CTAs/SM at <= 64 registers; A/B: 1 CTA/SM (80 registers) 72.5, 2 82.5, 3 (40 registers) 75.5 GTEPS
#endif
__global__ void __launch_bounds__(THREADS, BFS_MINB) bfs_kernel(Args a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t lq[LQ];
  __shared__ uint32_t lcount, lbase;
  __shared__ uint32_t ebuf[THREADS / 32][CAP];
  const uint32_t gtid = blockIdx.x * THREADS + threadIdx.x;
  const uint32_t gsize = gridDim.x * THREADS;
  const uint32_t gwarp = gtid >> 5, nwarps = gsize >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t *eb = ebuf[threadIdx.x >> 5];
  bool scan_in = false;  // this level's frontier is "level byte == level" (the previous level wrote no queue)
  for (int level = 0;; level++) {
    BFS_T(level);
    const int qc = level & 1, qn = qc ^ 1;                        // queue buffers
    const int sc = level % 3, sn = (level + 1) % 3, sf = (level + 2) % 3;  // size slots
    const uint32_t fsize = *((volatile uint32_t *)&a.qsize[sc]);
    if (fsize == 0) break;
    if (gtid == 0) {
      a.qsize[sf] = 0;                     // last read as the previous level's "current" (before the barrier)
      a.qsize[4 + ((level + 1) & 1)] = 0;  // the next level's compaction count, last read a level ago
    }
    const uint32_t *fq = a.q[qc];
    uint32_t *nq = a.q[qn];
    uint32_t *nsize = a.qsize + sn;
    const int32_t nl = level + 1;
    const uint8_t nb = nl < kDeep ? (uint8_t)nl : kDeep;
    const uint8_t lb = (uint8_t)level;
    // scan-in: the frontier is "level byte == level" (read in vertex order:
    // node records and edge lists stream nearly sequentially)
    bool scan = scan_in || (level < kDeep && fsize > (a.n >> BFS_SCAN_SHIFT));
    uint32_t work = scan ? a.n : fsize;
    // dense output: a large frontier writes only level bytes, the next level scans
    const bool dense = nl < kDeep - 1 && fsize >= (a.n >> BFS_DENSE_SHIFT);
    if (scan_in) {
      // the previous level claimed through level bytes only (no atomics):
      // rebuild the visited bitmap from them, 32 vertices per word, for a
      // queue-output level's claiming atomicOrs (the compaction's grid
      // barrier below orders the rebuild first).  Queue-less levels do not
      // read the bitmap (their level-byte probe decides alone), but the pass
      // still pays before them: 83.6 vs 82.0 GTEPS without it (A/B), the
      // level bytes it streams are the ones their probes hit next.
      const uint32_t nw = (a.n + 31) >> 5;
      for (uint32_t w = gtid; w < nw; w += gsize) {
        const uint4 *p = reinterpret_cast<const uint4 *>(a.level) + 2 * w;
        const uint4 b0 = __ldcg(p), b1 = __ldcg(p + 1);
        a.visited[w] = seen4(b0.x) | seen4(b0.y) << 4 | seen4(b0.z) << 8 | seen4(b0.w) << 12 |
                       seen4(b1.x) << 16 | seen4(b1.y) << 20 | seen4(b1.z) << 24 | seen4(b1.w) << 28;
      }
    }
    if (scan_in && fsize <= (a.n >> BFS_SCAN_SHIFT)) {
      // a small frontier after a queue-less level: compact its level bytes
      // into the queue first (16 bytes per lane per load), then run it as a
      // queue -- walking all n vertices would pay one dependent chain of
      // loads per 64 vertices per warp
      uint32_t *cnt = a.qsize + 4 + (level & 1);
      uint32_t *cq = a.q[qc];
      const uint32_t n16 = a.n >> 4;
      for (uint32_t i0 = 0; i0 < n16 + 1; i0 += gsize) {  // uniform trip count: whole warps shuffle
        const uint32_t i = i0 + gtid;
        uint32_t hits[16];
        int nh = 0;
        if (i < n16) {
          const uint4 b = __ldcg(reinterpret_cast<const uint4 *>(a.level) + i);
          const uint32_t wds[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
          for (int q = 0; q < 4; q++)
#pragma unroll
            for (int y = 0; y < 4; y++)
              if (((wds[q] >> (8 * y)) & 0xffu) == lb) hits[nh++] = 16 * i + 4 * q + y;
        } else if (i == n16) {  // the tail bytes
          for (uint32_t v = 16 * n16; v < a.n; v++)
            if (__ldcg(a.level + v) == lb) hits[nh++] = v;
        }
        // warp-aggregated append
        uint32_t inc = nh;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
          if (lane >= d) inc += t;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
        uint32_t base = 0;
        if (lane == 31 && total) base = atomicAdd(cnt, total);
        base = __shfl_sync(0xffffffffu, base, 31) + inc - nh;
        for (int h = 0; h < nh; h++) cq[base + h] = hits[h];
      }
      grid.sync();
      work = *((volatile uint32_t *)cnt);
      fq = cq;
      scan = false;
    }
    if (dense) {
      // ---------------- warps independent: no queue, no block barrier
      uint32_t claimed = 0;
      for (uint32_t base = gwarp * (32u * VPT); base < work; base += nwarps * (32u * VPT)) {
        uint32_t e0[VPT], ne[VPT];
#pragma unroll
        for (int k = 0; k < VPT; k++) {
          const uint32_t i = base + k * 32 + lane;
          ne[k] = 0;
          e0[k] = 0;
          if (i < work) {
            bool live = true;
            uint32_t u = i;
            if (scan) live = __ldcg(a.level + i) == lb;
            else u = __ldcg(fq + i);
            if (live) {
#if BFS_PACK
              const uint2 r = __ldcg(a.rec + u);
              e0[k] = r.x;
              ne[k] = r.y;
#else
              e0[k] = CSR_LD(a.starting + u);
              ne[k] = CSR_LD(a.nedges + u);
#endif
            }
          }
        }
#pragma unroll
        for (int k = 0; k < VPT; k++) {
          uint32_t cur = e0[k];
          const uint32_t end = e0[k] + ne[k];
#pragma unroll 1
          for (;;) {
            const uint32_t rem = min(end - cur, (uint32_t)CAP);
            uint32_t inc = rem;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
              if (lane >= d) inc += t;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
            if (total == 0) break;
            const uint32_t off = inc - rem;
            const uint32_t take = off >= (uint32_t)CAP ? 0u : min(rem, (uint32_t)CAP - off);
            for (uint32_t j = 0; j < take; j++) eb[off + j] = cur + j;
            cur += take;
            __syncwarp();
            const uint32_t cnt = min(total, (uint32_t)CAP);
#pragma unroll 1
            for (uint32_t b = 0; b < cnt; b += 32 * EB) {
              uint32_t v[EB];
#pragma unroll
              for (int j = 0; j < EB; j++) {
                const uint32_t i = b + j * 32 + lane;
                v[j] = i < cnt ? CSR_LD(a.edges + eb[i]) : 0xffffffffu;
              }
              // the level byte in L2 decides (no bitmap probe: a second
              // dependent round trip per edge costs more than it filters);
              // claims are plain stores
              uint8_t lv[EB];
#pragma unroll
              for (int j = 0; j < EB; j++) lv[j] = v[j] != 0xffffffffu ? __ldcg(a.level + v[j]) : (uint8_t)0;
#pragma unroll
              for (int j = 0; j < EB; j++) {
                if (lv[j] != kUnseen) continue;
                a.level[v[j]] = nb;  // (a queue level rebuilds the bitmap from the level bytes)
                claimed++;
              }
            }
            __syncwarp();
          }
        }
      }
      // the count may include a vertex claimed twice in this level: it only
      // steers the next level's mode
      const uint32_t wc = warp_sum(claimed);
      if (lane == 0 && wc) atomicAdd(nsize, wc);
    } else {
      // ---------------- queue output (claiming atomics, block-local queues)
      const uint32_t per_round = gsize * VPT;
      const uint32_t rounds = (work + per_round - 1) / per_round;
      for (uint32_t r = 0; r < rounds; r++) {
        if (threadIdx.x == 0) lcount = 0;
        __syncthreads();
        uint32_t e0[VPT], ne[VPT];
#pragma unroll
        for (int k = 0; k < VPT; k++) {
          const uint32_t i = r * per_round + k * gsize + gtid;
          ne[k] = 0;
          e0[k] = 0;
          if (i < work) {
            bool live = true;
            uint32_t u = i;
            if (scan) live = __ldcg(a.level + i) == lb;
            else u = __ldcg(fq + i);
            if (live) {
#if BFS_PACK
              const uint2 r = __ldcg(a.rec + u);
              e0[k] = r.x;
              ne[k] = r.y;
#else
              e0[k] = CSR_LD(a.starting + u);
              ne[k] = CSR_LD(a.nedges + u);
#endif
            }
          }
        }
        // warp-cooperative expansion: the warp's adjacency ranges are laid out
        // back to back in a per-warp buffer of edge ids (a warp scan gives each
        // range its offset), then all 32 lanes walk the buffer together --
        // balanced across lanes whatever the degrees, and consecutive lanes
        // read consecutive edges.  Ranges longer than the buffer continue in
        // the next pass.
#pragma unroll
        for (int k = 0; k < VPT; k++) {
          uint32_t cur = e0[k];
          const uint32_t end = e0[k] + ne[k];
#pragma unroll 1
          for (;;) {
            const uint32_t rem = min(end - cur, (uint32_t)CAP);
            uint32_t inc = rem;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
              if (lane >= d) inc += t;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
            if (total == 0) break;
            const uint32_t off = inc - rem;
            const uint32_t take = off >= (uint32_t)CAP ? 0u : min(rem, (uint32_t)CAP - off);
            for (uint32_t j = 0; j < take; j++) eb[off + j] = cur + j;
            cur += take;
            __syncwarp();
            const uint32_t cnt = min(total, (uint32_t)CAP);
#pragma unroll 1
            for (uint32_t b = 0; b < cnt; b += 32 * EB) {
              uint32_t v[EB], w[EB];
#pragma unroll
              for (int j = 0; j < EB; j++) {
                const uint32_t i = b + j * 32 + lane;
                v[j] = i < cnt ? CSR_LD(a.edges + eb[i]) : 0xffffffffu;
              }
              // probes may come from L1 (stale only towards "unseen": the
              // atomicOr below re-checks)
#pragma unroll
              for (int j = 0; j < EB; j++) w[j] = v[j] != 0xffffffffu ? a.visited[v[j] >> 5] : 0xffffffffu;
#pragma unroll
              for (int j = 0; j < EB; j++) {
                if (v[j] == 0xffffffffu) continue;
                const uint32_t bit = 1u << (v[j] & 31);
                if (w[j] & bit) continue;
                const uint32_t old = atomicOr(a.visited + (v[j] >> 5), bit);
                if (old & bit) continue;  // someone else claimed v
                a.level[v[j]] = nb;
                if (nb == kDeep) a.cost[v[j]] = nl;
                enqueue(nsize, v[j], lq, lcount, nq);
              }
            }
            __syncwarp();
          }
        }
        __syncthreads();
        const uint32_t cnt = min(lcount, (uint32_t)LQ);
        if (threadIdx.x == 0 && cnt) lbase = atomicAdd(nsize, cnt);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < cnt; k += THREADS) nq[lbase + k] = lq[k];
      }
    }
    scan_in = dense;
    grid.sync();
  }
}

__global__ void bfs_init_kernel(uint8_t *level, uint32_t *visited, uint32_t n, uint32_t words, uint32_t source,
                                uint32_t *q0, uint32_t *qsize) {
  const uint32_t n4 = 8 * ((n + 31) / 32);  // padded to whole 32-vertex groups (the bitmap rebuild reads them)
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x)
    reinterpret_cast<uint32_t *>(level)[i] = 0xFFFFFFFFu;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += gridDim.x * blockDim.x) visited[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    qsize[0] = 1;
    qsize[1] = 0;
    qsize[2] = 0;
    qsize[4] = 0;
    qsize[5] = 0;
    q0[0] = source;
  }
}

__global__ void bfs_seed_kernel(uint8_t *level, uint32_t *visited, uint32_t source) {
  level[source] = 0;
  visited[source >> 5] |= 1u << (source & 31);
}

// level bytes -> i32 costs (4 vertices per thread, coalesced)
__global__ void bfs_expand_kernel(const uint8_t *level, int32_t *cost, uint32_t n, int vec) {
  const uint32_t n4 = n / 4;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (vec ? n4 : n); i += gridDim.x * blockDim.x) {
    if (vec) {
      const uint32_t b = __ldcs(reinterpret_cast<const unsigned int *>(level) + i);
      int4 c;
      const int32_t *old = cost + 4 * (size_t)i;
      const uint32_t b0 = b & 0xff, b1 = (b >> 8) & 0xff, b2 = (b >> 16) & 0xff, b3 = b >> 24;
      c.x = b0 == kUnseen ? -1 : (b0 == kDeep ? old[0] : (int)b0);
      c.y = b1 == kUnseen ? -1 : (b1 == kDeep ? old[1] : (int)b1);
      c.z = b2 == kUnseen ? -1 : (b2 == kDeep ? old[2] : (int)b2);
      c.w = b3 == kUnseen ? -1 : (b3 == kDeep ? old[3] : (int)b3);
      __stcs(reinterpret_cast<int4 *>(cost) + i, c);
    } else {
      const uint32_t b = level[i];
      cost[i] = b == kUnseen ? -1 : (b == kDeep ? cost[i] : (int)b);
    }
  }
  if (vec) {  // the tail
    for (uint32_t i = 4 * n4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const uint32_t b = level[i];
      cost[i] = b == kUnseen ? -1 : (b == kDeep ? cost[i] : (int)b);
    }
  }
}

}  // namespace bfs
}  // namespace jb

using namespace jb;
using namespace jb::bfs;

#ifdef BFS_TRACE
extern "C" JB_API void jb_bfs_trace(unsigned long long *out) {
  cudaMemcpyFromSymbol(out, jb::bfs::g_bfs_trace, sizeof(jb::bfs::g_bfs_trace));
}
#endif

#if BFS_PACK
__global__ void bfs_pack_kernel(const uint32_t *__restrict__ starting, const uint32_t *__restrict__ nedges,
                                uint2 *__restrict__ rec, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    rec[i] = make_uint2(__ldcs(starting + i), __ldcs(nedges + i));
}
#endif

extern "C" jb_status jb_bfs(uint64_t n, uint64_t m, const uint32_t *starting, const uint32_t *nedges,
                            const uint32_t *edges, uint32_t source, int32_t *cost, void *stream) {
  JB_REQUIRE(n < (1ull << 32) - 64 && m < (1ull << 32), "bfs: graph too large for u32 indices");
  if (n == 0) return JB_OK;
  JB_REQUIRE(source < n, "bfs: source %u out of bounds for n=%llu", source, (unsigned long long)n);
  JB_REQUIRE(starting && nedges && cost && (edges || m == 0), "bfs: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t words = (uint32_t)((n + 31) / 32);
  const size_t qbytes = ((n * 4 + 255) / 256) * 256;
  const size_t vbytes = ((words * 4 + 255) / 256) * 256;
  const size_t lbytes = ((n + 255) / 256) * 256;
  const size_t rbytes = BFS_PACK ? ((n * 8 + 255) / 256) * 256 : 0;
  char *ws = (char *)workspace(2 * qbytes + vbytes + lbytes + 256 + rbytes, s);
  if (!ws) return JB_ECUDA;
  Args a;
  a.starting = starting; a.nedges = nedges; a.edges = edges; a.cost = cost;
  a.q[0] = (uint32_t *)ws;
  a.q[1] = (uint32_t *)(ws + qbytes);
  a.visited = (uint32_t *)(ws + 2 * qbytes);
  a.level = (uint8_t *)(ws + 2 * qbytes + vbytes);
  a.qsize = (uint32_t *)(ws + 2 * qbytes + vbytes + lbytes);
  a.n = (uint32_t)n;
  a.rec = (const uint2 *)(ws + 2 * qbytes + vbytes + lbytes + 256);
#if BFS_PACK
  bfs_pack_kernel<<<sm_count() * 8, 256, 0, s>>>(starting, nedges, (uint2 *)a.rec, (uint32_t)n);
  JB_LAUNCHED("bfs_pack");
#endif
  bfs_init_kernel<<<sm_count() * 4, 256, 0, s>>>(a.level, a.visited, (uint32_t)n, words, source, a.q[0], a.qsize);
  JB_LAUNCHED("bfs_init");
  bfs_seed_kernel<<<1, 1, 0, s>>>(a.level, a.visited, source);
  JB_LAUNCHED("bfs_seed");
  static int carve = [] {
    // experiments: the shared-memory carveout (percent); the rest of the
    // 256 KB is L1, which caches the visited-bitmap probes
    const char *e = getenv("JB_BFS_CARVE");
    const int c = e ? atoi(e) : -1;
    if (c >= 0) cudaFuncSetAttribute(bfs_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, c);
    return c;
  }();
  (void)carve;
  int per_sm = 0;
  JB_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_kernel, THREADS, 0));
  if (const char *e = getenv("JB_BFS_CTAS")) {  // experiments: fewer CTAs per SM than fit
    const int k = atoi(e);
    if (k >= 1 && k < per_sm) per_sm = k;
  }
  if (getenv("JB_BFS_VERBOSE")) fprintf(stderr, "bfs: %d CTAs/SM of %d threads\n", per_sm, THREADS);
  if (per_sm < 1) per_sm = 1;
  const int grid = sm_count() * per_sm;
  void *args[] = {&a};
  void *tok = prof_begin("bfs_levels", s);
  JB_CHECK_CUDA(cudaLaunchCooperativeKernel((void *)bfs_kernel, dim3(grid), dim3(THREADS), args, 0, s));
  prof_end(tok, s);
  JB_LAUNCHED("bfs_levels");
  const int vec = ((uintptr_t)cost % 16) == 0;
  bfs_expand_kernel<<<sm_count() * 8, 256, 0, s>>>(a.level, cost, (uint32_t)n, vec);
  JB_LAUNCHED("bfs_expand");
  return JB_OK;
}
