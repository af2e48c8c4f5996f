// svd_stub.cu -- placeholder entry points (replaced by the step/driver kernels)
#include "jsvd_host.h"
extern "C" {
jsvd_status jsvd_sweep_step(jsvd_dtype, int64_t, int64_t, double*, int64_t, double*, int64_t,
                            const int32_t*, int64_t, double, double*, double*, int64_t*, double*,
                            void*) { return JSVD_EINVAL; }
jsvd_status jsvd_step_rspec(jsvd_dtype, int64_t, int32_t*, int32_t*, int32_t*, int32_t*) {
  return JSVD_EINVAL;
}
jsvd_status jsvd_strategy_pairs(int64_t, int32_t, int64_t, int32_t*, void*) { return JSVD_EINVAL; }
jsvd_status jsvd_gesvj_workspace(jsvd_dtype, int64_t, int64_t, size_t*) { return JSVD_EINVAL; }
jsvd_status jsvd_gesvj(jsvd_dtype, int64_t, int64_t, double*, int64_t, double*, int64_t, double*,
                       double*, double*, int32_t, int32_t, int32_t*, int64_t*, void*, size_t,
                       void*) { return JSVD_EINVAL; }
jsvd_status jsvd_gesvj_batched(jsvd_dtype, int64_t, int64_t, int64_t, double*, int64_t, int64_t,
                               double*, int64_t, int64_t, double*, int32_t, int32_t*, int32_t*,
                               void*) { return JSVD_EINVAL; }
}
