// runtime.cu -- host runtime of libjunob200.so: status/error reporting, the
// per-device scratch arena and launch accounting.
//
// The arena is the stand-in for the reference runner's allocation model
// ("one allocation per device"): every entry
// point asks for the scratch it needs, the arena grows to the largest request
// seen on that device and is reused by later calls.
#include <stdarg.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "common.cuh"

namespace jb {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
void *tmap_encode_fn() {
  static void *fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = p;
  });
  return fn;
}

bool make_tmap_f32(CUtensorMap *map, const void *base, int rank, const uint64_t *dims, const uint64_t *strides_bytes,
                   const uint32_t *box, int swizzle) {
  return make_tmap(map, (int)CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, rank, dims, strides_bytes, box, swizzle);
}

bool make_tmap(CUtensorMap *map, int dtype, const void *base, int rank, const uint64_t *dims,
               const uint64_t *strides_bytes, const uint32_t *box, int swizzle) {
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tmap_encode_fn());
  if (!fn) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; i++) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) st[i] = strides_bytes[i];
  }
  CUresult r = fn(map, (CUtensorMapDataType)dtype, rank, const_cast<void *>(base), d, st, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static thread_local char g_err[1024] = "";
static std::atomic<uint64_t> g_launches{0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// One scratch arena per (device, stream): two streams of one device never
// share scratch, so concurrent calls on different streams cannot corrupt
// each other.  Growing waits for the stream's own earlier users only; it is
// refused while the stream is being captured into a graph (free/alloc are
// not capturable): run the call once outside the capture to size it.
struct Arena {
  void *ptr = nullptr;
  size_t cap = 0;
};
static std::map<std::pair<int, cudaStream_t>, Arena> g_arenas;
static std::mutex g_arena_mu;

// A caller-owned region bound as a stream's scratch (jb_bind_workspace: the
// runner's single arena).  Requests it cannot hold take the
// library's own arena below; the high-water mark tells the caller how much
// to reserve next time.
struct Bound {
  void *ptr = nullptr;
  size_t cap = 0;
  size_t high = 0;      // largest request since binding
  uint64_t spills = 0;  // requests larger than cap (served by the library arena)
};
static std::map<std::pair<int, cudaStream_t>, Bound> g_bound;

void *workspace(size_t bytes, cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return nullptr;
  std::lock_guard<std::mutex> lk(g_arena_mu);
  {
    auto it = g_bound.find({dev, s});
    if (it != g_bound.end()) {
      Bound &b = it->second;
      if (bytes > b.high) b.high = bytes;
      if (bytes <= b.cap) return b.ptr;
      b.spills++;
    }
  }
  Arena &a = g_arenas[{dev, s}];
  if (bytes <= a.cap) return a.ptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    set_error("scratch arena must grow to %zu bytes while the stream is capturing; "
              "run the call once outside the capture first", bytes);
    return nullptr;
  }
  if (a.ptr) {
    cudaStreamSynchronize(s);  // the old block's users are on this stream
    cudaFree(a.ptr);
    a.ptr = nullptr;
    a.cap = 0;
  }
  size_t want = bytes + (bytes >> 3);  // 12.5% headroom against regrowth
  want = (want + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
  if (cudaMalloc(&a.ptr, want) != cudaSuccess) {
    cudaGetLastError();
    a.ptr = nullptr;
    set_error("scratch arena: cudaMalloc(%zu) failed", want);
    return nullptr;
  }
  a.cap = want;
  return a.ptr;
}

jb_status after_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return JB_ECUDA;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return JB_OK;
}

// ---------------------------------------------------------------- profiler
// When enabled, prof_begin/prof_end record a CUDA event pair around a kernel
// launch on the launching stream; jb_prof_read synchronises the events and
// returns the summed device time per kernel name.  Used by bench.py to time
// the dominant kernel inside the timed region.
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
static std::atomic<int> g_prof_on{0};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof_pending;
static std::map<std::string, std::pair<double, uint64_t>> g_prof_acc;
static std::vector<cudaEvent_t> g_prof_free;

static cudaEvent_t prof_event() {
  if (!g_prof_free.empty()) {
    cudaEvent_t e = g_prof_free.back();
    g_prof_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void *prof_begin(const char *name, cudaStream_t s) {
  if (!g_prof_on.load(std::memory_order_relaxed)) return nullptr;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_pending.push_back(ProfRec{name, prof_event(), prof_event()});
  cudaEventRecord(g_prof_pending.back().a, s);
  return (void *)(uintptr_t)g_prof_pending.size();
}

void prof_end(void *tok, cudaStream_t s) {
  if (!tok) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  size_t i = (size_t)(uintptr_t)tok - 1;
  if (i < g_prof_pending.size()) cudaEventRecord(g_prof_pending[i].b, s);
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return kNumSMs;
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = kNumSMs;
    cached[dev] = v;
  }
  return cached[dev];
}

}  // namespace jb

extern "C" {

const char *jb_last_error(void) { return jb::g_err; }
int jb_abi_version(void) { return JB_ABI_VERSION; }
uint64_t jb_launch_count(void) { return jb::g_launches.load(); }

void jb_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(jb::g_prof_mu);
  jb::g_prof_on.store(on ? 1 : 0);
}

void jb_prof_reset(void) {
  std::lock_guard<std::mutex> lk(jb::g_prof_mu);
  for (auto &r : jb::g_prof_pending) {
    cudaEventSynchronize(r.b);
    jb::g_prof_free.push_back(r.a);
    jb::g_prof_free.push_back(r.b);
  }
  jb::g_prof_pending.clear();
  jb::g_prof_acc.clear();
}

jb_status jb_prof_read(const char *name, double *ms, uint64_t *count) {
  std::lock_guard<std::mutex> lk(jb::g_prof_mu);
  for (auto &r : jb::g_prof_pending) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) {
      jb::set_error("jb_prof_read: event sync failed");
      return JB_ECUDA;
    }
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    auto &acc = jb::g_prof_acc[r.name];
    acc.first += t;
    acc.second += 1;
    jb::g_prof_free.push_back(r.a);
    jb::g_prof_free.push_back(r.b);
  }
  jb::g_prof_pending.clear();
  auto it = jb::g_prof_acc.find(name ? name : "");
  *ms = it == jb::g_prof_acc.end() ? 0.0 : it->second.first;
  *count = it == jb::g_prof_acc.end() ? 0 : it->second.second;
  return JB_OK;
}

jb_status jb_bind_workspace(void *ptr, uint64_t bytes, void *stream) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) {
    jb::set_error("jb_bind_workspace: no current device");
    return JB_ECUDA;
  }
  JB_REQUIRE(((uintptr_t)ptr & 255) == 0, "jb_bind_workspace: region must be 256-byte aligned");
  std::lock_guard<std::mutex> lk(jb::g_arena_mu);
  const auto key = std::make_pair(dev, (cudaStream_t)stream);
  if (!ptr) {
    jb::g_bound.erase(key);
    return JB_OK;
  }
  jb::Bound &b = jb::g_bound[key];
  b.ptr = ptr;
  b.cap = bytes;
  b.high = 0;
  b.spills = 0;
  return JB_OK;
}

jb_status jb_workspace_stats(void *stream, uint64_t *high, uint64_t *spills) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) {
    jb::set_error("jb_workspace_stats: no current device");
    return JB_ECUDA;
  }
  std::lock_guard<std::mutex> lk(jb::g_arena_mu);
  auto it = jb::g_bound.find({dev, (cudaStream_t)stream});
  *high = it == jb::g_bound.end() ? 0 : it->second.high;
  *spills = it == jb::g_bound.end() ? 0 : it->second.spills;
  return JB_OK;
}

jb_status jb_release_workspace(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) {
    jb::set_error("jb_release_workspace: no current device");
    return JB_ECUDA;
  }
  std::lock_guard<std::mutex> lk(jb::g_arena_mu);
  cudaDeviceSynchronize();
  for (auto it = jb::g_arenas.begin(); it != jb::g_arenas.end();) {
    if (it->first.first == dev) {
      if (it->second.ptr) cudaFree(it->second.ptr);
      it = jb::g_arenas.erase(it);
    } else {
      ++it;
    }
  }
  return JB_OK;
}

// Page-lock caller-owned host memory in place (the numpy path of the
// Python mirror uses it so host<->device copies are DMA at full PCIe rate
// without a staging copy).  Registration errors are reported, not sticky.
jb_status jb_host_register(void *ptr, uint64_t bytes) {
  if (!ptr || !bytes) {
    jb::set_error("jb_host_register: null range");
    return JB_EINVAL;
  }
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    jb::set_error("cudaHostRegister(%zu bytes): %s", (size_t)bytes, cudaGetErrorString(e));
    return e == cudaErrorHostMemoryAlreadyRegistered ? JB_EINVAL : JB_ECUDA;
  }
  return JB_OK;
}

jb_status jb_host_unregister(void *ptr) {
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    jb::set_error("cudaHostUnregister: %s", cudaGetErrorString(e));
    return JB_ECUDA;
  }
  return JB_OK;
}

}  // extern "C"

// ---------------------------------------------------------- peer memory (IPC)
extern "C" jb_status jb_p2p_alloc(uint64_t bytes, void **ptr) {
  JB_REQUIRE(ptr && bytes > 0, "p2p_alloc: bad arguments");
  JB_CHECK_CUDA(cudaMalloc(ptr, bytes));
  JB_CHECK_CUDA(cudaMemset(*ptr, 0, bytes));
  return JB_OK;
}
extern "C" jb_status jb_p2p_free(void *ptr) {
  if (ptr) JB_CHECK_CUDA(cudaFree(ptr));
  return JB_OK;
}
extern "C" jb_status jb_ipc_handle(const void *ptr, void *handle64) {
  JB_REQUIRE(ptr && handle64, "ipc_handle: null pointer");
  cudaIpcMemHandle_t h;
  JB_CHECK_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(ptr)));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(handle64, &h, sizeof(h));
  return JB_OK;
}
extern "C" jb_status jb_ipc_open(const void *handle64, void **ptr) {
  JB_REQUIRE(ptr && handle64, "ipc_open: null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  JB_CHECK_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return JB_OK;
}
extern "C" jb_status jb_ipc_close(void *ptr) {
  if (ptr) JB_CHECK_CUDA(cudaIpcCloseMemHandle(ptr));
  return JB_OK;
}
