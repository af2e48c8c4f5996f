// dgsscl.cu -- jsvd_dgsscl: the real Gram-Schmidt orthogonalization of Alg
// SM8.1 / Eq. (DGS) (NEXT-4; reading R#39) for a
// batch of disjoint pivot pairs: g_q <- (g_q 2^-e_q - psi g_p 2^-e_p) 2^e_q,
// psi = a21' (f_q / f_p), g_p unchanged.  Elementwise and HBM-bound (3 m w
// bytes per pair); one CTA per (pair, 1024-row slice), coalesced along the
// column.  Every operation is the paper's (scalef = one correctly rounded
// scaling, one fma), so the results are bit-identical to the oracle.
#include "jsvd_host.h"
#include "jsvd_dev.cuh"

namespace jsvd {
namespace {

constexpr int kGsThreads = 256, kGsRows = 4;  // rows per thread

__global__ void __launch_bounds__(kGsThreads) dgsscl_kernel(
    int64_t m, double* __restrict__ G, int64_t ldg, const int32_t* __restrict__ pairs,
    int64_t npairs, const double* __restrict__ ce, const double* __restrict__ cf,
    const double* __restrict__ a21) {
  for (int64_t l = blockIdx.y; l < npairs; l += gridDim.y) {
    const int p = pairs[2 * l], q = pairs[2 * l + 1];
    const double ep = ce[p], eq = ce[q];
    if (isinf(ep) || isinf(eq)) continue;  // a zero column (R#19)
    const double mpsi = -(a21[l] * __ddiv_rn(cf[q], cf[p]));  // line 1
    const int iep = static_cast<int>(ep), ieq = static_cast<int>(eq);
    const double* __restrict__ gp = G + static_cast<int64_t>(p) * ldg;
    double* __restrict__ gq = G + static_cast<int64_t>(q) * ldg;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * (kGsThreads * kGsRows) + threadIdx.x;
    double x[kGsRows], y[kGsRows];
#pragma unroll
    for (int k = 0; k < kGsRows; ++k) {  // all loads first
      const int64_t i = base + k * kGsThreads;
      x[k] = i < m ? __ldcs(gp + i) : 0.0;
      y[k] = i < m ? __ldcs(gq + i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kGsRows; ++k) {
      const int64_t i = base + k * kGsThreads;
      if (i < m) {  // lines 4-5
        const double xs = scalbn_rn(x[k], -iep), ys = scalbn_rn(y[k], -ieq);
        __stcs(gq + i, scalbn_rn(fma(mpsi, xs, ys), ieq));
      }
    }
  }
}

}  // namespace
}  // namespace jsvd

using namespace jsvd;

extern "C" jsvd_status jsvd_dgsscl(int64_t m, int64_t n, double* G, int64_t ldg,
                                   const int32_t* pairs, int64_t npairs, const double* col_e,
                                   const double* col_f, const double* a21, void* stream) {
  if (m < 0 || n < 0 || npairs < 0 || ldg < m || 2 * npairs > n) return JSVD_EINVAL;
  if (m == 0 || npairs == 0) return JSVD_OK;
  if (!G || !pairs || !col_e || !col_f || !a21) return JSVD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t slices = (m + kGsThreads * kGsRows - 1) / (kGsThreads * kGsRows);
  if (slices > (int64_t(1) << 31) - 1) return JSVD_EINVAL;
  const dim3 grid(static_cast<unsigned>(slices),
                  static_cast<unsigned>(npairs < 65535 ? npairs : 65535));
  dgsscl_kernel<<<grid, kGsThreads, 0, st>>>(m, G, ldg, pairs, npairs, col_e, col_f, a21);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}
