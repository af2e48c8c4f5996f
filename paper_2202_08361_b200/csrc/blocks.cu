// blocks.cu -- column-block building blocks of Alg 4.1 for drivers that hold
// only some columns of G (the column-block-sharded SVD, dist.py):
//   jsvd_maxnorm      line 1: max |component| (NaN -> inf), max-reduced
//   jsvd_scale        lines 1/6: G <- 2^s G (scalef, one rounding)
//   jsvd_colnorms     line 42: (e,f) of columns with the step kernel's lane order (R#23)
//   jsvd_normalize    line 42: u_j = 2^-e_j g_j / f_j
#include "jsvd_host.h"
#include "step_dev.cuh"

namespace jsvd {
cudaError_t launch_colnorm(bool cplx, int64_t m, int64_t n, const double* G, int64_t ldg,
                           double* ce, double* cf, cudaStream_t st);
bool step_supported(bool cplx, int64_t m);

__global__ void maxnorm_cols_kernel(int64_t rows, int64_t n, const double* G, int64_t ld,
                                    unsigned long long* out) {
  __shared__ unsigned long long sm[32];
  unsigned long long mx = 0;
  const int64_t total = rows * n;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = k / rows, i = k % rows;
    const double y = fmin(fabs(G[j * ld + i]), static_cast<double>(INFINITY));
    mx = max(mx, static_cast<unsigned long long>(__double_as_longlong(y)));
  }
#pragma unroll
  for (int o = 16; o >= 1; o /= 2) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) mx = max(mx, sm[w]);
    atomicMax(out, mx);
  }
}

__global__ void scale_cols_kernel(int64_t rows, int64_t n, double* G, int64_t ld, int s) {
  const int64_t total = rows * n;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = k / rows, i = k % rows;
    G[j * ld + i] = scalbn_rn(G[j * ld + i], s);
  }
}

__global__ void normalize_cols_kernel(int64_t rows, double* G, int64_t ld, const double* ce,
                                      const double* cf) {
  const int64_t j = blockIdx.y;
  const double e = ce[j];
  if (isinf(e)) return;  // zero column stays zero (R#19)
  const Pow2 sc(-static_cast<int>(e));
  const Divisor d = make_divisor(cf[j]);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    G[j * ld + i] = divide(sc(G[j * ld + i]), d);
}
}  // namespace jsvd

using namespace jsvd;

static bool dt_ok(jsvd_dtype dt) { return dt == JSVD_R64 || dt == JSVD_C64; }

extern "C" jsvd_status jsvd_maxnorm(jsvd_dtype dt, int64_t m, int64_t n, const double* G,
                                    int64_t ldg, double* mmax_dev, void* stream) {
  if (!dt_ok(dt) || m < 0 || n < 0 || ldg < m || !mmax_dev || (m * n > 0 && !G)) return JSVD_EINVAL;
  if (m * n == 0) return JSVD_OK;
  const int64_t w = dt == JSVD_C64 ? 2 : 1;
  maxnorm_cols_kernel<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w * m, n, G, w * ldg, reinterpret_cast<unsigned long long*>(mmax_dev));
  note_launch();
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}

extern "C" jsvd_status jsvd_scale(jsvd_dtype dt, int64_t m, int64_t n, double* G, int64_t ldg,
                                  int32_t s, void* stream) {
  if (!dt_ok(dt) || m < 0 || n < 0 || ldg < m || (m * n > 0 && !G)) return JSVD_EINVAL;
  if (m * n == 0 || s == 0) return JSVD_OK;
  const int64_t w = dt == JSVD_C64 ? 2 : 1;
  scale_cols_kernel<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(w * m, n, G, w * ldg, s);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}

extern "C" jsvd_status jsvd_colnorms(jsvd_dtype dt, int64_t m, int64_t n, const double* G,
                                     int64_t ldg, double* col_e, double* col_f, void* stream) {
  const bool cplx = dt == JSVD_C64;
  if (!dt_ok(dt) || m < 1 || n < 0 || ldg < m || !step_supported(cplx, m) || (n > 0 && (!G || !col_e || !col_f)))
    return JSVD_EINVAL;
  if (cplx && (reinterpret_cast<uintptr_t>(G) & 15)) return JSVD_EINVAL;
  if (n == 0) return JSVD_OK;
  return launch_colnorm(cplx, m, n, G, ldg, col_e, col_f, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? JSVD_OK
             : JSVD_ECUDA;
}

extern "C" jsvd_status jsvd_normalize(jsvd_dtype dt, int64_t m, int64_t n, double* G, int64_t ldg,
                                      const double* col_e, const double* col_f, void* stream) {
  if (!dt_ok(dt) || m < 0 || n < 0 || ldg < m || (m * n > 0 && (!G || !col_e || !col_f)))
    return JSVD_EINVAL;
  if (m * n == 0) return JSVD_OK;
  const int64_t w = dt == JSVD_C64 ? 2 : 1;
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((w * m + 255) / 256, 64)),
            static_cast<unsigned>(n));
  normalize_cols_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(w * m, G, w * ldg,
                                                                            col_e, col_f);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}
