// api.cu -- status strings and the launch counter of the C ABI (include/jsvd.h)
#include <cstdlib>
#include <mutex>

#include "jsvd_host.h"

namespace jsvd {
std::atomic<int64_t> g_launches{0};
}

extern "C" const char* jsvd_status_string(jsvd_status s) {
  switch (s) {
    case JSVD_OK: return "JSVD_OK";
    case JSVD_ENOCONV: return "JSVD_ENOCONV: not converged within max_sweeps";
    case JSVD_EINVAL: return "JSVD_EINVAL: invalid argument";
    case JSVD_ENONFINITE: return "JSVD_ENONFINITE: input holds Inf or NaN";
    case JSVD_ERANK: return "JSVD_ERANK: all-zero matrix";
    case JSVD_ECUDA: return "JSVD_ECUDA: CUDA error";
    case JSVD_ENCCL: return "JSVD_ENCCL: NCCL error";
    case JSVD_ENOMEM: return "JSVD_ENOMEM: workspace too small";
  }
  return "JSVD_?: unknown status";
}

extern "C" int64_t jsvd_launch_count(void) { return jsvd::g_launches.load(); }

// ---- JSVD_DEBUG=1: non-finite EVD inputs -> JSVD_ENONFINITE --
// The paper's EVD assumes finite entries and the library does not
// check them on the hot path.  With JSVD_DEBUG=1 in the environment, the EVD
// entry points first run this scan and a synchronous 4-byte readback, and
// return JSVD_ENONFINITE (nothing else launched) if any entry is Inf or NaN.
namespace jsvd {
namespace {
template <typename T>
__global__ void nonfinite_scan(int64_t r, const T* a, const T* b, const T* c, const T* d,
                               int* flag) {
  bool bad = false;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < r;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    bad |= !isfinite(a[i]) || !isfinite(b[i]) || !isfinite(c[i]) || (d && !isfinite(d[i]));
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}
std::mutex g_dbg_mu;
int* g_dbg_flag[64] = {};
}  // namespace

int sm_count() {
  static std::atomic<int> cache[64];  // 0: not queried yet
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0 && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
    cache[dev].store(v, std::memory_order_relaxed);
  return v;
}

bool debug_enabled() {
  const char* v = getenv("JSVD_DEBUG");
  return v && v[0] && v[0] != '0';
}

template <typename T>
jsvd_status debug_check_finite(int64_t r, const T* a, const T* b, const T* c, const T* d,
                               cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return JSVD_ECUDA;
  int* flag;
  {
    std::lock_guard<std::mutex> g(g_dbg_mu);
    if (!g_dbg_flag[dev] && cudaMalloc(&g_dbg_flag[dev], sizeof(int)) != cudaSuccess)
      return JSVD_ECUDA;
    flag = g_dbg_flag[dev];
  }
  int h = 0;
  if (cudaMemsetAsync(flag, 0, sizeof(int), st) != cudaSuccess) return JSVD_ECUDA;
  nonfinite_scan<T><<<592, 256, 0, st>>>(r, a, b, c, d, flag);
  note_launch();
  if (cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return JSVD_ECUDA;
  return h ? JSVD_ENONFINITE : JSVD_OK;
}
template jsvd_status debug_check_finite<double>(int64_t, const double*, const double*,
                                                const double*, const double*, cudaStream_t);
template jsvd_status debug_check_finite<float>(int64_t, const float*, const float*, const float*,
                                               const float*, cudaStream_t);
}  // namespace jsvd
