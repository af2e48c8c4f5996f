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

// a plain streaming copy with the EVD kernel's access pattern (16-byte
// streaming loads and stores, one CTA of 256 threads per 8 KB, programmatic
// dependent launch): the context line for the EVD's HBM fraction
__global__ void __launch_bounds__(256) copy16_kernel(int64_t n16, const double2* __restrict__ src,
                                                     double2* __restrict__ dst) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int64_t i = static_cast<int64_t>(blockIdx.x) * 512 + threadIdx.x;
  if (i < n16) __stcs(dst + i, __ldcs(src + i));
  if (i + 256 < n16) __stcs(dst + i + 256, __ldcs(src + i + 256));
}

}  // namespace jsvd

extern "C" jsvd_status jsvd_copy16(int64_t n16, const double* src, double* dst, void* stream) {
  if (n16 < 0 || (n16 && (!src || !dst))) return JSVD_EINVAL;
  if (n16 == 0) return JSVD_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>((n16 + 511) / 512));
  cfg.blockDim = dim3(256);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, jsvd::copy16_kernel, n16, reinterpret_cast<const double2*>(src),
                     reinterpret_cast<double2*>(dst));
  jsvd::note_launch();
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}

extern "C" jsvd_status jsvd_fp64_peak(int32_t blocks, int64_t iters, double* out,
                                      int64_t* dfma_count, void* stream) {
  if (blocks < 1 || iters < 1 || !out || !dfma_count) return JSVD_EINVAL;
  jsvd::fp64_peak_kernel<<<static_cast<unsigned>(blocks), 256, 0,
                           static_cast<cudaStream_t>(stream)>>>(iters, 0.5, 0.75, out);
  jsvd::note_launch();
  *dfma_count = static_cast<int64_t>(blocks) * 256 * iters * 16 * 8;
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}
