// Error reporting and device checks for the C ABI.
#include <stdarg.h>
#include <string.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace antkv {

const void *previous_cache_on_stream(cudaStream_t st, const void *key) {
  static std::mutex mu;
  static std::unordered_map<cudaStream_t, const void *> last;
  std::lock_guard<std::mutex> lock(mu);
  const void *prev = nullptr;
  auto it = last.find(st);
  if (it != last.end()) prev = it->second;
  last[st] = key;
  return prev;
}


// Streams whose caller declared that only this library's launches run on
// them (antkv_stream_exclusive): only there may a fused decode launch read
// its inputs before griddepcontrol.wait.  A foreign kernel (a torch copy, a
// cuBLAS GEMM writing q) can be the PDL primary of our launch, and the host
// cannot see it, so the default is to read everything after the wait.
namespace {
std::mutex g_ex_mu;
std::unordered_map<cudaStream_t, int> g_exclusive;
}  // namespace

bool stream_exclusive(cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_ex_mu);
  auto it = g_exclusive.find(st);
  return it != g_exclusive.end() && it->second;
}

namespace {
struct FastOutputs {
  const char *out = nullptr, *lse = nullptr;
  int64_t out_bytes = 0, lse_bytes = 0;
};
std::mutex g_fo_mu;
std::unordered_map<cudaStream_t, FastOutputs> g_fo;
bool overlap(const char *a, int64_t na, const char *b, int64_t nb) {
  return a && b && na > 0 && nb > 0 && a < b + nb && b < a + na;
}
}  // namespace

// The fused decode kernel lets its successor on the stream start early
// (programmatic dependent launch): these record what the last fused launch
// on a stream writes besides its own cache, so the next one knows whether
// its q / qpos may be read before griddepcontrol.wait.
void record_fast_outputs(cudaStream_t st, const void *out, int64_t out_bytes, const void *lse,
                         int64_t lse_bytes) {
  std::lock_guard<std::mutex> lock(g_fo_mu);
  FastOutputs &f = g_fo[st];
  f.out = static_cast<const char *>(out);
  f.out_bytes = out_bytes;
  f.lse = static_cast<const char *>(lse);
  f.lse_bytes = lse_bytes;
}

bool overlaps_previous_fast_outputs(cudaStream_t st, const void *p, int64_t bytes) {
  std::lock_guard<std::mutex> lock(g_fo_mu);
  auto it = g_fo.find(st);
  if (it == g_fo.end()) return false;
  const char *c = static_cast<const char *>(p);
  return overlap(c, bytes, it->second.out, it->second.out_bytes) ||
         overlap(c, bytes, it->second.lse, it->second.lse_bytes);
}

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char *where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return ANTKV_ECUDA;
}

__global__ void probe_kernel(int *out) { *out = 100; }

}  // namespace antkv

using namespace antkv;

extern "C" const char *antkv_last_error(void) { return g_err; }

extern "C" int antkv_version(void) { return 1; }

extern "C" int antkv_stream_exclusive(void *stream, int exclusive) {
  std::lock_guard<std::mutex> lock(g_ex_mu);
  g_exclusive[static_cast<cudaStream_t>(stream)] = exclusive ? 1 : 0;
  return ANTKV_OK;
}

namespace antkv { int decode_fast_smem_base_ok(); }

namespace antkv {
cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64) {
    std::lock_guard<std::mutex> lk(mu);
    if (!done[dev]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      done[dev] = true;
    }
  }
  return cudaMallocAsync(p, bytes, st);
}
}  // namespace antkv

extern "C" int antkv_device_check(int device) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDeviceProperties") ? 0 : 0;
  if (p.major != 10 || p.minor != 0) {
    set_error("device %d is sm_%d%d; this library is built for sm_100a", device, p.major, p.minor);
    return 0;
  }
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, probe_kernel);
  if (e != cudaSuccess) {
    cuda_status(e, "kernel image");
    return 0;
  }
  antkv::decode_fast_smem_base_ok();   // one-time probe, outside any stream capture
  return 1;
}

// ---------------------------------------------------------------- peer memory
// Receive buffers for the sequence-shard exchange are plain cudaMalloc
// allocations (an IPC handle maps a whole allocation), zero-filled.
extern "C" int antkv_p2p_alloc(int64_t bytes, void **ptr) {
  ANTKV_REQUIRE(bytes > 0 && ptr != nullptr, "bad p2p allocation");
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, (size_t)bytes);
  return e == cudaSuccess ? ANTKV_OK : cuda_status(e, "p2p buffer");
}

extern "C" int antkv_p2p_free(void *ptr) {
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? ANTKV_OK : cuda_status(e, "p2p buffer free");
}

extern "C" int antkv_ipc_get_handle(const void *ptr, void *handle) {
  ANTKV_REQUIRE(ptr != nullptr && handle != nullptr, "null argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(ptr));
  if (e != cudaSuccess) return cuda_status(e, "cudaIpcGetMemHandle");
  memcpy(handle, &h, sizeof(h));
  return ANTKV_OK;
}

extern "C" int antkv_ipc_open_handle(const void *handle, void **ptr) {
  ANTKV_REQUIRE(ptr != nullptr && handle != nullptr, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? ANTKV_OK : cuda_status(e, "cudaIpcOpenMemHandle");
}

extern "C" int antkv_ipc_close_handle(void *ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? ANTKV_OK : cuda_status(e, "cudaIpcCloseMemHandle");
}
