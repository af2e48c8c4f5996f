// diag.cu -- jsvd_fp64_peak: a DFMA-throughput microbenchmark, the measured
// FP64 denominator of the batched SVD's roofline ("the builder
// must measure it").  Every thread runs 8 independent dependent-DFMA chains
// (enough to cover the pipe latency at 8 warps per SM sub-partition); the
// values converge to a fixed point in [1, 2), so no special operands occur.
#include "jsvd_host.h"

namespace jsvd {

__global__ void __launch_bounds__(256) fp64_peak_kernel(int64_t iters, double a, double b,
                                                        double* out) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = 1.0 + 0.125 * k + 1e-9 * threadIdx.x;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x] = s;
}

}  // namespace jsvd

extern "C" jsvd_status jsvd_fp64_peak(int32_t blocks, int64_t iters, double* out,
                                      int64_t* dfma_count, void* stream) {
  if (blocks < 1 || iters < 1 || !out || !dfma_count) return JSVD_EINVAL;
  jsvd::fp64_peak_kernel<<<static_cast<unsigned>(blocks), 256, 0,
                           static_cast<cudaStream_t>(stream)>>>(iters, 0.5, 0.75, out);
  jsvd::note_launch();
  *dfma_count = static_cast<int64_t>(blocks) * 256 * iters * 16 * 8;
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}
