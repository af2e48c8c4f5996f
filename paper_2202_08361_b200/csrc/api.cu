// api.cu -- status strings and the launch counter of the C ABI (include/jsvd.h)
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
