// norm_ef.cu -- jsvd_norm_ef: column norms by the paper's one-pass "(e, f)"
// method (NEXT-3: Alg SM6.3; readings R#35-R#38), one warp per
// column with s = 32 lanes.  Lane l keeps the partial sum of the squares of
// elements l, l+32, ... as (e, f), r = 2^e f, f in [1, 2), updated by the
// fma step of SM6.2 (complex: the real part, then the imaginary part); the 32
// partial sums are then sorted by Eq. (vsort) with a bitonic network of warp
// shuffles and reduced pairwise by Eq. (redj); the root is SM6.1's.
//
// Exponents are int32 with kNegInf for -inf; every exponent operation of the
// paper is exact integer arithmetic there, and every -inf / NaN case of the
// paper's floating-point exponents is mapped explicitly (see ef_update).
// The significand arithmetic (scalef with one rounding, fma, getmant) is the
// paper's, so the results are bit-identical to the oracle.  HBM-bound: m n w
// bytes read once (w = 8 real, 16 complex), 16 bytes written per column.
#include "jsvd_host.h"
#include "step_dev.cuh"

namespace jsvd {
namespace {

constexpr int kNegInf = -(1 << 30);  // exponent -inf (below every finite exponent)

// E(x), F(x) of a finite x (R#35): (kNegInf, 1) for zero
__device__ __forceinline__ void ef_EF(double x, int& e, double& f) {
  const uint64_t b = abs_bits(x);
  if (b >> 52) {  // normal
    e = static_cast<int>(b >> 52) - 1023;
    f = __longlong_as_double(static_cast<long long>((b & 0x000fffffffffffffull) |
                                                    0x3ff0000000000000ull));
  } else if (b == 0) {
    e = kNegInf;
    f = 1.0;
  } else {  // subnormal: exact
    e = ilogb_bits(b);
    f = scalbn_rn(__longlong_as_double(static_cast<long long>(b)), -e);
  }
}

// E, F of a value in [1, 8) (the normalisations of SM6.2 / Eq. redj)
__device__ __forceinline__ void ef_norm(double v, int& de, double& f) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  de = static_cast<int>(b >> 52) - 1023;
  f = __longlong_as_double(static_cast<long long>((b & 0x000fffffffffffffull) |
                                                  0x3ff0000000000000ull));
}

// r <- fma(|x|, |x|, r) (Alg SM6.3 lines 5-13) for one lane: every case
__device__ __forceinline__ void ef_update_general(int& e, double& f, double x) {
  const bool einf = e == kNegInf;
  const int lsb = einf ? 0 : (e & 1);           // cvtpd_epi64(e) & 1, -inf -> 0 (R#37)
  const int ep = einf ? kNegInf : e - lsb;      // e' (even or -inf)
  const double fp = lsb ? f * 2.0 : f;          // f' = scalef(f, lsb), exact
  int ei;
  double fi;
  ef_EF(x, ei, fi);
  const int eh = ei == kNegInf ? kNegInf : 2 * ei;  // scalef(e_i, 1)
  const int emax = max(eh, ep);
  // max(sub(., e_max), -inf): -inf stays -inf (the NaN of -inf - -inf too)
  const int eh2 = eh == kNegInf ? kNegInf : (eh - emax) / 2;  // scalef(., -1): even, exact
  const int epp = ep == kNegInf ? kNegInf : ep - emax;
  const double fh = eh2 == kNegInf ? 0.0 : scalbn_rn(fi, eh2);
  const double fhp = epp == kNegInf ? 0.0 : scalbn_rn(fp, epp);
  const double fpn = fma(fh, fh, fhp);  // >= 1 unless both are 0 (e_max = -inf)
  if (emax == kNegInf) {
    e = kNegInf;
    f = 1.0;  // F(0) = 1
  } else {
    int de;
    ef_norm(fpn, de, f);
    e = emax + de;
  }
}

// The same update with the common case on the integer pipe: r != 0 and x
// normal, and both scalings 2^{e-hat''}, 2^{e''} >= 2^-1022.  Then f' = f or 2f
// is an exponent-field add, E(x) and F(x) are bit fields, and the two scalef
// are exact multiplies by normal powers of two (f_i in [1,2), f' in [1,4)):
// only the fma rounds, exactly as in the general form.  Lanes outside that
// case take ef_update_general in a warp-uniform branch (the first element of
// every lane, zeros, subnormals, and sums 2^2044 apart).
__device__ __forceinline__ void ef_update(int& e, double& f, double x) {
  const uint32_t hx = hi32(x) & 0x7fffffffu;
  const int lsb = e & 1;
  const int ep = e - lsb;
  const double fp = mkd(hi32(f) + (static_cast<uint32_t>(lsb) << 20), lo32(f));
  const int eh = 2 * (static_cast<int>(hx >> 20) - 1023);
  const double fi = mkd((hx & 0x000fffffu) | 0x3ff00000u, lo32(x));
  const int emax = max(eh, ep);
  const int h2 = (eh - emax) >> 1;  // even and <= 0: exact halving
  const int d2 = ep - emax;
  const bool fast = (e != kNegInf) & (hx >= 0x00100000u) & (h2 >= -1022) & (d2 >= -1022);
  const double fh = fi * pow2i(max(h2, -1022));
  const double fhp = fp * pow2i(max(d2, -1022));
  const double fpn = fma(fh, fh, fhp);
  int de;
  double fn;
  ef_norm(fpn, de, fn);
  int en = emax + de;
  if (__any_sync(0xffffffffu, !fast)) {
    int eg = e;
    double fg = f;
    ef_update_general(eg, fg, x);
    if (!fast) {
      en = eg;
      fn = fg;
    }
  }
  e = en;
  f = fn;
}

// a + b for a <= b by Eq. (vsort): Eq. (redj), normalised
__device__ __forceinline__ void ef_add_sorted(int ea, double fa, int& eb, double& fb) {
  const double sc = ea == kNegInf ? 0.0 : scalbn_rn(1.0, ea - eb);  // scalef(1, max(ea-eb, -inf))
  const double fpr = fma(sc, fa, fb);  // >= 1 (fb >= 1)
  int de;
  ef_norm(fpr, de, fb);
  if (eb != kNegInf) eb += de;
}

__device__ __forceinline__ bool ef_le(int ea, double fa, int eb, double fb) {
  return (ea < eb) || (ea == eb && fa <= fb);
}

template <bool CPLX>
__global__ void __launch_bounds__(256) norm_ef_kernel(int64_t m, int64_t n, const double* __restrict__ G,
                                                      int64_t ldg, double* __restrict__ ce,
                                                      double* __restrict__ cf, double* __restrict__ ce2,
                                                      double* __restrict__ cf2) {
  const int lane = threadIdx.x & 31;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (j >= n) return;  // warp-uniform
  int e = kNegInf;
  double f = 1.0;
  constexpr int U = 4;  // elements in flight per lane
  if constexpr (CPLX) {
    const double2* x = reinterpret_cast<const double2*>(G) + j * ldg;
    int64_t i0 = 0;
    for (; i0 + 32 * U <= m; i0 += 32 * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(x + i0 + 32 * u + lane);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ef_update(e, f, v[u].x);
        ef_update(e, f, v[u].y);
      }
    }
    for (int64_t i = i0 + lane; i0 < m; i0 += 32, i += 32) {  // tail (zero padding, Eq. pad0)
      const double2 v = i < m ? x[i] : make_double2(0.0, 0.0);
      ef_update(e, f, v.x);
      ef_update(e, f, v.y);
    }
  } else {
    const double* x = G + j * ldg;
    int64_t i0 = 0;
    for (; i0 + 32 * U <= m; i0 += 32 * U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(x + i0 + 32 * u + lane);
#pragma unroll
      for (int u = 0; u < U; ++u) ef_update(e, f, v[u]);
    }
    for (int64_t i = i0 + lane; i0 < m; i0 += 32, i += 32) {
      const double v = i < m ? x[i] : 0.0;
      ef_update(e, f, v);
    }
  }
  // sort the 32 partial sums by Eq. (vsort): bitonic network (R#38)
#pragma unroll
  for (int k = 2; k <= 32; k *= 2) {
#pragma unroll
    for (int s = k / 2; s >= 1; s /= 2) {
      const int eo = __shfl_xor_sync(0xffffffffu, e, s);
      const double fo = __shfl_xor_sync(0xffffffffu, f, s);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & s) == 0;
      // the lower lane of an ascending pair keeps the smaller element (equal
      // keys are equal pairs, so ties need no rule)
      const bool mine_le = ef_le(e, f, eo, fo);
      if ((lower == up) != mine_le) {
        e = eo;
        f = fo;
      }
    }
  }
  // pairwise reduction, Eq. (redj): element i of level t sits on lane i 2^t
#pragma unroll
  for (int s = 1; s < 32; s *= 2) {
    const int eb = __shfl_down_sync(0xffffffffu, e, s);
    const double fb = __shfl_down_sync(0xffffffffu, f, s);
    if ((lane & (2 * s - 1)) == 0) {  // a = this lane (position 2i), b = partner (2i+1)
      int eb2 = eb;
      double fb2 = fb;
      ef_add_sorted(e, f, eb2, fb2);
      e = eb2;
      f = fb2;
    }
  }
  if (lane == 0) {
    if (ce2) ce2[j] = e == kNegInf ? -INFINITY : static_cast<double>(e);
    if (cf2) cf2[j] = f;
    // the root, SM6.1: odd e -> (e-1, 2f)
    int er = e;
    double fr = f;
    if (e != kNegInf && (e & 1)) {
      er = e - 1;
      fr = 2.0 * f;
    }
    ce[j] = e == kNegInf ? -INFINITY : static_cast<double>(er / 2);
    cf[j] = __dsqrt_rn(fr);
  }
}

}  // namespace
}  // namespace jsvd

using namespace jsvd;

extern "C" jsvd_status jsvd_norm_ef(jsvd_dtype dt, int64_t m, int64_t n, const double* G,
                                    int64_t ldg, double* col_e, double* col_f, double* col_e2,
                                    double* col_f2, void* stream) {
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < 0 || n < 0 || ldg < m || !col_e || !col_f)
    return JSVD_EINVAL;
  if (n == 0) return JSVD_OK;
  if (!G && m > 0) return JSVD_EINVAL;
  if (dt == JSVD_C64 && (reinterpret_cast<uintptr_t>(G) & 15)) return JSVD_EINVAL;
  if (n > (int64_t(1) << 34)) return JSVD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (n + 7) / 8;
  if (dt == JSVD_C64)
    norm_ef_kernel<true><<<static_cast<unsigned>(blocks), 256, 0, st>>>(m, n, G, ldg, col_e, col_f,
                                                                        col_e2, col_f2);
  else
    norm_ef_kernel<false><<<static_cast<unsigned>(blocks), 256, 0, st>>>(m, n, G, ldg, col_e, col_f,
                                                                         col_e2, col_f2);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}
