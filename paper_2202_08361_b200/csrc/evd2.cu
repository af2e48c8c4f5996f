// evd2.cu -- jsvd_evd2_batched: the batched 2x2 Hermitian / symmetric EVD
// (Alg 2.2/2.3, SM2.1/SM2.2) on sm_100a.
//
// HBM-streaming kernel: each thread owns K = 2 consecutive matrices, loads
// every SoA input stream with one 16-byte LDG.128 (coalesced, 512 B per warp
// per stream), runs the EVD in registers, and stores every output stream with
// one 16-byte STG.128; the permutation words are assembled from two
// shuffles and two warp ballots.  No shared memory, no synchronisation.
// Grid: one 256-thread CTA per 512 matrices (r = 2^26: 131072 CTAs, ~ 110
// waves at 8 CTAs/SM).
#include <cstdlib>

#include "jsvd_dev.cuh"

#include "jsvd_host.h"

namespace jsvd {

// streaming loads of one chunk (512 matrices per CTA, 2 per thread); lanes
// past r read zeros (every lane runs the EVD so the rare-case votes can use
// the full warp mask)
template <bool CPLX>
struct Chunk2 {
  double2 a11, a22, re, im;
  template <typename I>
  __device__ __forceinline__ void load(I r, I tid, const double* __restrict__ p11,
                                       const double* __restrict__ p22,
                                       const double* __restrict__ pre,
                                       const double* __restrict__ pim) {
    const I l0 = 2 * tid;
    a11 = a22 = re = im = make_double2(0.0, 0.0);
    if (l0 + 1 < r) {
      a11 = __ldcs(reinterpret_cast<const double2*>(p11) + tid);
      a22 = __ldcs(reinterpret_cast<const double2*>(p22) + tid);
      re = __ldcs(reinterpret_cast<const double2*>(pre) + tid);
      if (CPLX) im = __ldcs(reinterpret_cast<const double2*>(pim) + tid);
    } else if (l0 < r) {  // ragged tail: one matrix
      a11.x = p11[l0];
      a22.x = p22[l0];
      re.x = pre[l0];
      if (CPLX) im.x = pim[l0];
    }
  }
};

// one chunk: 512 consecutive matrices, 2 per thread (LDG.128 / STG.128 of
// every SoA stream); the permutation words from two shuffles + two ballots
// I: the index type -- uint32_t when 2 r < 2^32 (one IMAD.WIDE.U32 per
// stream address instead of 64-bit shift-and-add pairs), else int64_t
template <bool CPLX, bool TAN, bool NOBACK, typename I>
__device__ __forceinline__ void evd2_chunk(
    I c, I r, const double* __restrict__ a11, const double* __restrict__ a22,
    const double* __restrict__ are, const double* __restrict__ aim, double* __restrict__ l1,
    double* __restrict__ l2, double* __restrict__ cs, double* __restrict__ sr,
    double* __restrict__ si, int32_t* __restrict__ zeta, uint32_t* __restrict__ perm) {
  const I tid = c * 256 + threadIdx.x;
  const I l0 = 2 * tid;
  Chunk2<CPLX> x;
  x.load(r, tid, a11, a22, are, aim);
  const Evd2Out e0 = evd2<CPLX, TAN, NOBACK>(x.a11.x, x.a22.x, x.re.x, x.im.x, kFull);
  const Evd2Out e1 = evd2<CPLX, TAN, NOBACK>(x.a11.y, x.a22.y, x.re.y, x.im.y, kFull);
  const bool p0 = l0 < r && e0.perm, p1 = l0 + 1 < r && e1.perm;
  if (l0 + 1 < r) {
    __stcs(reinterpret_cast<double2*>(l1) + tid, make_double2(e0.l1, e1.l1));
    __stcs(reinterpret_cast<double2*>(l2) + tid, make_double2(e0.l2, e1.l2));
    __stcs(reinterpret_cast<double2*>(cs) + tid, make_double2(e0.c, e1.c));
    __stcs(reinterpret_cast<double2*>(sr) + tid, make_double2(e0.sr, e1.sr));
    if (CPLX) __stcs(reinterpret_cast<double2*>(si) + tid, make_double2(e0.si, e1.si));
    if (zeta) __stcs(reinterpret_cast<int2*>(zeta) + tid, make_int2(e0.zeta, e1.zeta));
  } else if (l0 < r) {
    l1[l0] = e0.l1;
    l2[l0] = e0.l2;
    cs[l0] = e0.c;
    sr[l0] = e0.sr;
    if (CPLX) si[l0] = e0.si;
    if (zeta) zeta[l0] = e0.zeta;
  }
  if (perm) {  // warp covers matrices [64w, 64w+64): words 2w, 2w+1
    // bit j of word 2w + h is matrix 64w + 32h + j, held by lane 16h + j/2 as
    // its EVD j&1: fetch that lane's two bits, then one ballot per word
    const int lane = threadIdx.x & 31;
    const uint32_t v = (p0 ? 1u : 0u) | (p1 ? 2u : 0u);
    const uint32_t v0 = __shfl_sync(0xffffffffu, v, lane >> 1);
    const uint32_t v1 = __shfl_sync(0xffffffffu, v, 16 + (lane >> 1));
    const uint32_t w0 = __ballot_sync(0xffffffffu, (v0 >> (lane & 1)) & 1u);
    const uint32_t w1 = __ballot_sync(0xffffffffu, (v1 >> (lane & 1)) & 1u);
    const I w = c * 16 + 2 * (threadIdx.x >> 5) + lane;  // word 2w + lane (lanes 0, 1)
    if (lane < 2 && 32 * w < r) perm[w] = lane ? w1 : w0;
  }
}

// CPT consecutive chunks per CTA (r/512/CPT CTAs) at <= 64 registers: 4 CTAs
// per SM (a 5-CTA bound spills and measured no better for configs[0], worse
// for configs[1])
template <bool CPLX, bool TAN, bool NOBACK, typename I, int CPT = 1>
__global__ void __launch_bounds__(256, 4) evd2_vec2_kernel(
    int64_t r, const double* __restrict__ a11, const double* __restrict__ a22,
    const double* __restrict__ are, const double* __restrict__ aim, double* __restrict__ l1,
    double* __restrict__ l2, double* __restrict__ cs, double* __restrict__ sr,
    double* __restrict__ si, int32_t* __restrict__ zeta, uint32_t* __restrict__ perm, int pf) {
  // programmatic dependent launch: the next grid in the stream may be scheduled
  // into the SMs this grid's last wave leaves free; every grid waits for its
  // predecessor's completion (and memory) before touching data
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (pf > 0 && threadIdx.x == 0) {
    // L2 prefetch of the input chunk pf CTAs ahead (one bulk request per
    // stream, issued by one thread through the TMA unit): HBM keeps streaming
    // while the resident CTAs compute, and that chunk's loads hit L2
    const int64_t cn = (static_cast<int64_t>(blockIdx.x) + pf) * CPT;
    if ((cn + CPT) * 512 <= r) {
      const double* ps[4] = {a11, a22, are, aim};
#pragma unroll
      for (int k = 0; k < (CPLX ? 4 : 3); ++k)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(ps[k] + cn * 512),
                     "n"(4096 * CPT)
                     : "memory");
    }
  }
#pragma unroll 1
  for (int i = 0; i < CPT; ++i)
    evd2_chunk<CPLX, TAN, NOBACK, I>(static_cast<I>(blockIdx.x) * CPT + i, static_cast<I>(r), a11,
                                     a22, are, aim, l1, l2, cs, sr, si, zeta, perm);
}

// scalar path for pointers that are only 8-byte aligned (I as evd2_chunk)
template <bool CPLX, bool TAN, bool NOBACK, int MINB = 1, typename I = int64_t>
__global__ void __launch_bounds__(256, MINB) evd2_scalar_kernel(
    int64_t r, const double* __restrict__ a11, const double* __restrict__ a22,
    const double* __restrict__ are, const double* __restrict__ aim, double* __restrict__ l1,
    double* __restrict__ l2, double* __restrict__ cs, double* __restrict__ sr,
    double* __restrict__ si, int32_t* __restrict__ zeta, uint32_t* __restrict__ perm, int pf) {
  if (MINB > 1) {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
  }
  if (pf > 0 && threadIdx.x == 0) {  // L2 prefetch pf CTAs ahead (as the vector kernel)
    const int64_t cn = static_cast<int64_t>(blockIdx.x) + pf;
    if ((cn + 1) * 256 <= r) {
      const double* ps[4] = {a11, a22, are, aim};
#pragma unroll
      for (int k = 0; k < (CPLX ? 4 : 3); ++k)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], 2048;\n" ::"l"(ps[k] + cn * 256)
                     : "memory");
    }
  }
  const I l = static_cast<I>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool in = l < static_cast<I>(r);
  const Evd2Out e = evd2<CPLX, TAN, NOBACK>(in ? a11[l] : 0.0, in ? a22[l] : 0.0,
                                            in ? are[l] : 0.0, (CPLX && in) ? aim[l] : 0.0, kFull);
  const bool p = in && e.perm;
  if (in) {
    l1[l] = e.l1;
    l2[l] = e.l2;
    cs[l] = e.c;
    sr[l] = e.sr;
    if (CPLX) si[l] = e.si;
    if (zeta) zeta[l] = e.zeta;
  }
  if (perm) {
    const uint32_t b = __ballot_sync(0xffffffffu, p);
    if ((threadIdx.x & 31) == 0 && in) perm[l / 32] = b;
  }
}

// L2 prefetch distance in CTAs: one wave of resident CTAs ahead (per_sm CTAs
// per SM).  Measured, configs[1] (vector kernel, 4 per SM), 20 launches:
// 0.942 -> 0.905 ms (two waves 0.906, four slower); configs[0] (scalar
// kernel, 8 per SM): 12.8 -> 12.5 us (two or four waves: no gain).
// JSVD_EVD_PF overrides (0: off).
// 32-bit indices for r < 2^31; JSVD_EVD_IDX64=1 forces the 64-bit kernels
// (the form every r beyond 2^31 takes; the GPU tests compare both)
static bool evd_idx32(int64_t r) {
  const char* e = getenv("JSVD_EVD_IDX64");
  return r < (int64_t(1) << 31) && !(e && atoi(e));
}

static int evd_prefetch_distance(int per_sm) {
  const char* e = getenv("JSVD_EVD_PF");
  return e ? atoi(e) : per_sm * sm_count();
}

template <bool CPLX, bool TAN, bool NOBACK>
static cudaError_t launch_evd2(bool vec, int64_t r, const double* a11, const double* a22,
                               const double* re, const double* im, double* l1, double* l2,
                               double* c, double* sr, double* si, int32_t* zeta, uint32_t* perm,
                               cudaStream_t st) {
  const int threads = 256;
  if (!CPLX) {
    // real (configs[0]): one matrix per thread at 32 registers, 8 CTAs per
    // SM (64 warps, the maximum) -- the short (~15 us) launch is latency- and
    // tail-bound: 59% of the HBM peak with the 2-per-thread vector kernel, 63%
    // at 6 CTAs/SM, 67% at 8 (despite 96 bytes of L1-resident spills);
    // 8-byte-aligned pointers suffice
    const int64_t blocks = (r + threads - 1) / threads;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(blocks));
    cfg.blockDim = dim3(threads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (evd_idx32(r))
      cudaLaunchKernelEx(&cfg, evd2_scalar_kernel<CPLX, TAN, NOBACK, 8, uint32_t>, r, a11, a22, re, im,
                         l1, l2, c, sr, si, zeta, perm, evd_prefetch_distance(8));
    else
      cudaLaunchKernelEx(&cfg, evd2_scalar_kernel<CPLX, TAN, NOBACK, 8, int64_t>, r, a11, a22, re, im,
                         l1, l2, c, sr, si, zeta, perm, evd_prefetch_distance(8));
    note_launch();
    return cudaGetLastError();
  }
  if (vec) {
    // 512-matrix chunks, two consecutive ones per CTA (a persistent
    // grid-stride variant was slower for configs[0] and [1], before the L2
    // prefetch)
    const int64_t chunks = (r + 2 * threads - 1) / (2 * threads);
    // two chunks per CTA, one after the other (the per-CTA fixed costs
    // shared): configs[1] 0.893 -> 0.886 ms (20 launches), 0.994 -> 0.988 ms
    // (200); four per CTA: 0.896 / 0.994 ms.  JSVD_EVD_CPT=1: one chunk per CTA.
    const char* ce = getenv("JSVD_EVD_CPT");
    const bool two = !(ce && atoi(ce) == 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(two ? (chunks + 1) / 2 : chunks));
    cfg.blockDim = dim3(threads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool i32 = evd_idx32(r);
    const int pf = evd_prefetch_distance(4) / (two ? 2 : 1);  // the same distance in chunks
    if (two && i32)
      cudaLaunchKernelEx(&cfg, evd2_vec2_kernel<CPLX, TAN, NOBACK, uint32_t, 2>, r, a11, a22, re, im,
                         l1, l2, c, sr, si, zeta, perm, pf);
    else if (two)
      cudaLaunchKernelEx(&cfg, evd2_vec2_kernel<CPLX, TAN, NOBACK, int64_t, 2>, r, a11, a22, re, im,
                         l1, l2, c, sr, si, zeta, perm, pf);
    else if (i32)
      cudaLaunchKernelEx(&cfg, evd2_vec2_kernel<CPLX, TAN, NOBACK, uint32_t>, r, a11, a22, re, im, l1,
                         l2, c, sr, si, zeta, perm, pf);
    else
      cudaLaunchKernelEx(&cfg, evd2_vec2_kernel<CPLX, TAN, NOBACK, int64_t>, r, a11, a22, re, im, l1,
                         l2, c, sr, si, zeta, perm, pf);
  } else {
    const int64_t blocks = (r + threads - 1) / threads;
    evd2_scalar_kernel<CPLX, TAN, NOBACK><<<static_cast<unsigned>(blocks), threads, 0, st>>>(
        r, a11, a22, re, im, l1, l2, c, sr, si, zeta, perm, 0);
  }
  note_launch();
  return cudaGetLastError();
}

template <bool CPLX>
static cudaError_t dispatch_flags(uint32_t flags, bool vec, int64_t r, const double* a11,
                                  const double* a22, const double* re, const double* im,
                                  double* l1, double* l2, double* c, double* sr, double* si,
                                  int32_t* zeta, uint32_t* perm, cudaStream_t st) {
  const bool tan = flags & JSVD_EVD_TAN, nob = flags & JSVD_EVD_NOBACKSCALE;
  if (tan && nob)
    return launch_evd2<CPLX, true, true>(vec, r, a11, a22, re, im, l1, l2, c, sr, si, zeta, perm, st);
  if (tan)
    return launch_evd2<CPLX, true, false>(vec, r, a11, a22, re, im, l1, l2, c, sr, si, zeta, perm, st);
  if (nob)
    return launch_evd2<CPLX, false, true>(vec, r, a11, a22, re, im, l1, l2, c, sr, si, zeta, perm, st);
  return launch_evd2<CPLX, false, false>(vec, r, a11, a22, re, im, l1, l2, c, sr, si, zeta, perm, st);
}

}  // namespace jsvd

static bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

extern "C" jsvd_status jsvd_evd2_batched(jsvd_dtype dt, int64_t r, const double* a11,
                                         const double* a22, const double* a21_re,
                                         const double* a21_im, double* lam1, double* lam2,
                                         double* cos_phi, double* sin_re, double* sin_im,
                                         int32_t* zeta, uint32_t* perm, uint32_t flags,
                                         void* stream) {
  using namespace jsvd;
  if (r < 0 || (dt != JSVD_R64 && dt != JSVD_C64)) return JSVD_EINVAL;
  if (flags & ~(JSVD_EVD_TAN | JSVD_EVD_NOBACKSCALE)) return JSVD_EINVAL;
  if (r == 0) return JSVD_OK;
  if (r > (int64_t(1) << 40)) return JSVD_EINVAL;
  const bool cplx = (dt == JSVD_C64);
  if (!a11 || !a22 || !a21_re || !lam1 || !lam2 || !cos_phi || !sin_re) return JSVD_EINVAL;
  if (cplx != (a21_im != nullptr) || cplx != (sin_im != nullptr)) return JSVD_EINVAL;
  const void* ptrs[] = {a11, a22, a21_re, a21_im, lam1, lam2, cos_phi, sin_re, sin_im};
  bool vec = true;
  for (const void* p : ptrs) {
    if (p && !aligned(p, 8)) return JSVD_EINVAL;
    if (p && !aligned(p, 16)) vec = false;
  }
  if (zeta && !aligned(zeta, 4)) return JSVD_EINVAL;
  if (zeta && !aligned(zeta, 8)) vec = false;
  if (perm && !aligned(perm, 4)) return JSVD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (debug_enabled()) {
    const jsvd_status ds = debug_check_finite<double>(r, a11, a22, a21_re, a21_im, st);
    if (ds != JSVD_OK) return ds;
  }
  cudaError_t e = cplx ? dispatch_flags<true>(flags, vec, r, a11, a22, a21_re, a21_im, lam1, lam2,
                                              cos_phi, sin_re, sin_im, zeta, perm, st)
                       : dispatch_flags<false>(flags, vec, r, a11, a22, a21_re, nullptr, lam1,
                                               lam2, cos_phi, sin_re, nullptr, zeta, perm, st);
  return e == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}

// diagnostic entry point: q[i] = a[i] / b[i] with the library's division
namespace jsvd {
__global__ void debug_div_kernel(int64_t n, const double* a, const double* b, double* q, int mode) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    const double x = a[i], y = b[i];
    switch (mode) {
      case 0: q[i] = div_rn(x, y); break;
      case 1: q[i] = __ddiv_rn(x, y); break;
      case 2: q[i] = scalbn_rn(x, static_cast<int>(y)); break;
      case 3: q[i] = divide_sf<true, true>(x, make_divisor(y), __activemask()); break;
      case 4: q[i] = divide_checked(x, make_divisor(y), __activemask()); break;
      case 5: q[i] = hypot_naive(fabs(x), fabs(y)); break;
      case 7: q[i] = sqrt_plain(x); break;
      case 8: q[i] = div_plain(x, rcp_plain(y)); break;
      case 9: q[i] = divide_small(x, rcp_plain(y), __activemask()); break;
      case 10: q[i] = divide_gen(x, make_ndiv(y), __activemask()); break;
      default: q[i] = divide_sf<false, true>(x, make_divisor(y), __activemask()); break;
    }
  }
}
}  // namespace jsvd

extern "C" jsvd_status jsvd_debug_primitive(int32_t mode, int64_t n, const double* a,
                                            const double* b, double* q, void* stream) {
  if (n < 0 || mode < 0 || mode > 10) return JSVD_EINVAL;
  if (n == 0) return JSVD_OK;
  jsvd::debug_div_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0,
                           static_cast<cudaStream_t>(stream)>>>(n, a, b, q, mode);
  jsvd::note_launch();
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}
