// batched.cu -- jsvd_gesvj_batched: many independent small one-sided Jacobi
// SVDs (BASELINE configs[3]: 65536 complex 64 x 32), one CTA per matrix, the
// whole iteration (G and V) resident in shared memory: HBM is touched once to
// load A and once to store U, V, sigma.  Same arithmetic as jsvd_gesvj with
// nblocks = n (flat round-robin) and the reduction spec R = (32, 1,
// [16,8,4,2,1]): lane L of a warp owns rows L, L+32, ... of a pair.
//
// Per step (n/2 pairs):
//   A  every warp: norms, scaled dot, convergence test of its pairs (Alg 3.1,
//      3.2; R#14), results to shared memory
//   B  warp 0: the Grammians and 2x2 EVDs of all transformed pairs of the step,
//      ONE LANE PER PAIR -- the batch of EVDs of Alg 4.1 line 26 vectorised
//      across lanes as the paper vectorises it across SIMD lanes
//   C  every warp: rotation of its pairs' G and V columns (Alg 3.4), M-tilde.
// The Eq. (skr) rescale check runs at every step (flat round-robin, R#21).
#include <cmath>

#include "jsvd_host.h"
#include "step_dev.cuh"

namespace jsvd {

constexpr int kBT = 256;  // threads per CTA (8 warps)
constexpr int kBNW = kBT / 32;

struct PairSlot {
  double zr, zi, ep, fp, eq, fq;
  double c, C, S;
  int transform;
  int pad;
};

template <bool CPLX>
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o /= 2) v = v + __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// x 2^-e for a whole column slice, the two-multiply case taken warp-uniformly
template <int NR, typename E, typename F>
__device__ __forceinline__ void scaled_loop(const Pow2& f, F&& body) {
  if (f.two) {
#pragma unroll
    for (int j = 0; j < NR; ++j) body(j, true);
  } else {
#pragma unroll
    for (int j = 0; j < NR; ++j) body(j, false);
  }
}

template <bool CPLX, int NR>
__global__ void __launch_bounds__(kBT) batched_svd_kernel(
    int64_t m, int64_t n, double* A, int64_t lda, int64_t strideA, double* Vg, int64_t ldv,
    int64_t strideV, double* sigma, int max_sweeps, int32_t* sweeps_out, int32_t* status_out,
    int Fm, int Kr, double tol) {
  using E = typename Elem<CPLX>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  E* sG = reinterpret_cast<E*>(smem_raw);
  E* sV = sG + m * n;
  PairSlot* slots = reinterpret_cast<PairSlot*>(sV + n * n);
  double* ce = reinterpret_cast<double*>(slots + n / 2);
  double* cf = ce + n;
  uint8_t* sPairs = reinterpret_cast<uint8_t*>(cf + n);  // (n-1) x n/2 pivot pairs (n <= 64)
  __shared__ unsigned long long sMt, sM0;
  __shared__ int sT;
  __shared__ uint64_t wred[kBNW];

  const int64_t b = blockIdx.x;
  E* Ag = reinterpret_cast<E*>(A) + b * strideA;
  E* Vb = reinterpret_cast<E*>(Vg) + b * strideV;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int np = static_cast<int>(n / 2);
  const int mi = static_cast<int>(m), ni = static_cast<int>(n);
  // the flat round-robin ordering (R#20), once per CTA
  for (int k = threadIdx.x; k < (ni - 1) * np; k += kBT) {
    int p, q;
    strategy_pair(ni, ni, k / np, k % np, p, q);
    sPairs[2 * k] = static_cast<uint8_t>(p);
    sPairs[2 * k + 1] = static_cast<uint8_t>(q);
  }

  // ---- load A, M0 = max |component| (NaN -> inf), V = I
  uint64_t mx = 0;
  for (int64_t k = threadIdx.x; k < m * n; k += kBT) {
    const int64_t j = k / m, i = k % m;
    const E x = Ag[j * lda + i];
    sG[k] = x;
    if constexpr (CPLX) {
      mx = max(mx, abs_bits(fmin(fabs(x.x), static_cast<double>(INFINITY))));
      mx = max(mx, abs_bits(fmin(fabs(x.y), static_cast<double>(INFINITY))));
    } else {
      mx = max(mx, abs_bits(fmin(fabs(x), static_cast<double>(INFINITY))));
    }
  }
  for (int64_t k = threadIdx.x; k < n * n; k += kBT) {
    const int64_t j = k / n, i = k % n;
    if constexpr (CPLX) sV[k] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    else sV[k] = i == j ? 1.0 : 0.0;
  }
  {
    const uint64_t M0 = cta_max_u64<kBT>(mx, wred);
    if (threadIdx.x == 0) sM0 = M0;
    __syncthreads();
  }
  const double M0 = __longlong_as_double(static_cast<long long>(sM0));
  if (isinf(M0) || M0 == 0.0) {
    if (threadIdx.x == 0) {
      if (status_out) status_out[b] = isinf(M0) ? JSVD_ENONFINITE : JSVD_ERANK;
      if (sweeps_out) sweeps_out[b] = 0;
    }
    return;
  }
  // ---- line 1: s0 = F(m) - floor(lg M0) - 1; G1 = 2^s0 G
  int s = Fm - ilogb_bits(sM0) - 1;
  for (int64_t k = threadIdx.x; k < m * n; k += kBT) {
    if constexpr (CPLX) sG[k] = make_double2(scalbn_rn(sG[k].x, s), scalbn_rn(sG[k].y, s));
    else sG[k] = scalbn_rn(sG[k], s);
  }
  if (threadIdx.x == 0) sMt = static_cast<unsigned long long>(__double_as_longlong(scalbn_rn(M0, s)));
  __syncthreads();

  int C = 0;
  bool converged = false;
  for (C = 0; C < max_sweeps; ++C) {
    if (threadIdx.x == 0) sT = 0;
    for (int k = 0; k < ni - 1; ++k) {
      // ---- line 6: rescale check (every step for flat round-robin)
      {
        const int lm = ilogb_bits(sMt);
        const int sn = (Kr - lm < 0) ? Fm - lm - 1 : 0;
        if (sn != 0) {  // uniform
          __syncthreads();
          for (int64_t kk = threadIdx.x; kk < m * n; kk += kBT) {
            if constexpr (CPLX) sG[kk] = make_double2(scalbn_rn(sG[kk].x, sn), scalbn_rn(sG[kk].y, sn));
            else sG[kk] = scalbn_rn(sG[kk], sn);
          }
          if (threadIdx.x == 0) {
            sMt = static_cast<unsigned long long>(__double_as_longlong(
                scalbn_rn(__longlong_as_double(static_cast<long long>(sMt)), sn)));
          }
          s += sn;
          __syncthreads();
        }
      }
      // ---- phase A: norms, dot, convergence test (one warp per pair)
      for (int l = warp; l < np; l += kBNW) {
        const int p = sPairs[2 * (k * np + l)], q = sPairs[2 * (k * np + l) + 1];
        const E* gp = sG + p * mi;
        const E* gq = sG + q * mi;
        E xp[NR], xq[NR];
        uint64_t mp = 0, mq = 0;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          const int i = j * 32 + lane;
          xp[j] = i < mi ? gp[i] : Elem<CPLX>::zero();
          xq[j] = i < mi ? gq[i] : Elem<CPLX>::zero();
          mp = absmax_bits(xp[j], mp);
          mq = absmax_bits(xq[j], mq);
        }
        const int Ep = __reduce_max_sync(0xffffffffu, ilogb_or_min(mp));
        const int Eq = __reduce_max_sync(0xffffffffu, ilogb_or_min(mq));
        double sp = 0.0, sq = 0.0;
        if (Ep != kIntMin) {
          const Pow2 f(-Ep);
          scaled_loop<NR, E>(f, [&](int j, bool) {
            if (j * 32 + lane < mi) sp = ssq_acc(f(xp[j]), sp);
          });
        }
        if (Eq != kIntMin) {
          const Pow2 f(-Eq);
          scaled_loop<NR, E>(f, [&](int j, bool) {
            if (j * 32 + lane < mi) sq = ssq_acc(f(xq[j]), sq);
          });
        }
        sp = warp_sum<CPLX>(sp);
        sq = warp_sum<CPLX>(sq);
        double ep = -INFINITY, fp = 1.0, eq = -INFINITY, fq = 1.0;
        if (Ep != kIntMin) ef_from_ssq(Ep, sp, ep, fp);
        if (Eq != kIntMin) ef_from_ssq(Eq, sq, eq, fq);
        double zr = 0.0, zi = 0.0;
        if (Ep != kIntMin && Eq != kIntMin) {
          const Pow2 fP(-static_cast<int>(ep)), fQ(-static_cast<int>(eq));
          double ar = 0.0, ai = 0.0;
#pragma unroll
          for (int j = 0; j < NR; ++j)
            if (j * 32 + lane < mi) dot_acc(fQ(xq[j]), fP(xp[j]), ar, ai);
          ar = warp_sum<CPLX>(ar);
          if (CPLX) ai = warp_sum<CPLX>(ai);
          const Divisor d = make_divisor(fq * fp);
          zr = divide(ar, d);
          zi = CPLX ? divide(ai, d) : 0.0;
        }
        const double az = CPLX ? hypot_naive(fabs(zr), fabs(zi)) : fabs(zr);
        if (lane == 0) {
          PairSlot& sl = slots[l];
          sl.zr = zr;
          sl.zi = zi;
          sl.ep = ep;
          sl.fp = fp;
          sl.eq = eq;
          sl.fq = fq;
          sl.transform = tol <= az;
        }
      }
      __syncthreads();
      // ---- phase B: Grammians + EVDs of the step, one lane per pair
      if (warp == 0) {
        int tcount = 0;
        for (int l = lane; l < np + (32 - (np % 32)) % 32; l += 32) {
          // every lane runs (dummy pair past np / for converged pairs) so the
          // EVD's rare-case votes use the full warp mask
          const bool tr = l < np && slots[l].transform;
          if (__any_sync(kFull, tr)) {
            const PairSlot& s0 = slots[l < np ? l : 0];
            double b11, b22, br, bi;
            gram(tr ? s0.zr : 0.0, tr ? s0.zi : 0.0, tr ? s0.ep : 0.0, tr ? s0.fp : 1.0,
                 tr ? s0.eq : 0.0, tr ? s0.fq : 1.0, b11, b22, br, bi);
            const Evd2Out o = evd2<CPLX, true, true>(b11, b22, br, bi, kFull);
            if (tr) {
              slots[l].c = o.c;
              slots[l].C = o.sr;
              slots[l].S = o.si;
            }
          }
          tcount += __popc(__ballot_sync(0xffffffffu, tr));
        }
        if (lane == 0) sT += tcount;
      }
      __syncthreads();
      // ---- phase C: rotations of G and V (Alg 3.4), M-tilde
      uint64_t Mw = 0;
      for (int l = warp; l < np; l += kBNW) {
        const PairSlot& sl = slots[l];
        if (!sl.transform) continue;
        const int p = sPairs[2 * (k * np + l)], q = sPairs[2 * (k * np + l) + 1];
        const double c = sl.c, Cc = sl.C, S = sl.S;
        E* gp = sG + p * mi;
        E* gq = sG + q * mi;
        for (int i = lane; i < mi; i += 32) {
          E a = gp[i], bq = gq[i];
          rot_elem(a, bq, c, Cc, S);
          gp[i] = a;
          gq[i] = bq;
          Mw = absmax_bits(a, Mw);
          Mw = absmax_bits(bq, Mw);
        }
        E* vp = sV + p * ni;
        E* vq = sV + q * ni;
        for (int i = lane; i < ni; i += 32) {
          E a = vp[i], bq = vq[i];
          rot_elem(a, bq, c, Cc, S);
          vp[i] = a;
          vq[i] = bq;
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o /= 2) Mw = max(Mw, __shfl_xor_sync(0xffffffffu, Mw, o));
      if (lane == 0 && Mw) atomicMax(&sMt, static_cast<unsigned long long>(Mw));
      __syncthreads();
    }
    if (sT == 0) {
      converged = true;
      ++C;
      break;
    }
    __syncthreads();
  }
  // ---- finalize: norms, U = G diag(2^-e / f), sigma, sort
  for (int64_t j = warp; j < n; j += kBNW) {
    const E* g = sG + j * m;
    uint64_t mj = 0;
    for (int64_t i = lane; i < m; i += 32) mj = absmax_bits(g[i], mj);
    const int Ej = __reduce_max_sync(0xffffffffu, ilogb_or_min(mj));
    double sj = 0.0;
    if (Ej != kIntMin) {
      const Pow2 f(-Ej);
#pragma unroll
      for (int jj = 0; jj < NR; ++jj) {
        const int i = jj * 32 + lane;
        if (i < mi) sj = ssq_acc(f(g[i]), sj);
      }
    }
    sj = warp_sum<CPLX>(sj);
    double e = -INFINITY, f = 1.0;
    if (Ej != kIntMin) ef_from_ssq(Ej, sj, e, f);
    if (lane == 0) {
      ce[j] = e;
      cf[j] = f;
    }
  }
  __syncthreads();
  for (int64_t r0 = warp; r0 < n; r0 += kBNW) {
    // output column r0 <- input column j with rank r0
    int64_t jsel = 0;
    for (int64_t j = lane; j < n; j += 32) {
      const double ej = ce[j], fj = cf[j];
      int64_t rank = 0;
      for (int64_t kk = 0; kk < n; ++kk) {
        const double ek = ce[kk], fk = cf[kk];
        rank += ((ek > ej) || (ek == ej && (fk > fj || (fk == fj && kk < j)))) ? 1 : 0;
      }
      if (rank == r0) jsel = j + 1;
    }
#pragma unroll
    for (int o = 16; o >= 1; o /= 2) jsel = max(jsel, __shfl_xor_sync(0xffffffffu, jsel, o));
    const int64_t j = jsel - 1;
    const double e = ce[j], f = cf[j];
    const bool fin = !isinf(e);
    const Pow2 sc(fin ? -static_cast<int>(e) : 0);
    const Divisor d = make_divisor(f);
    E* ucol = Ag + r0 * lda;
    const E* g = sG + j * m;
    for (int64_t i = lane; i < m; i += 32) {
      E x = g[i];
      if (fin) {
        if constexpr (CPLX) x = make_double2(divide(sc(x.x), d), divide(sc(x.y), d));
        else x = divide(sc(x), d);
      }
      ucol[i] = x;
    }
    E* vcol = Vb + r0 * ldv;
    for (int64_t i = lane; i < n; i += 32) vcol[i] = sV[j * n + i];
    if (lane == 0) {
      const double es = fin ? e - s : e;
      sigma[b * n + r0] = fin ? scalbn_rn(f, static_cast<int>(fmax(fmin(es, 1e5), -1e5))) : 0.0;
    }
  }
  if (threadIdx.x == 0) {
    if (status_out) status_out[b] = converged ? JSVD_OK : JSVD_ENOCONV;
    if (sweeps_out) sweeps_out[b] = C;
  }
}

static size_t batched_smem(bool cplx, int64_t m, int64_t n) {
  const size_t w = cplx ? 16 : 8;
  return w * (m * n + n * n) + sizeof(PairSlot) * (n / 2) + 2 * sizeof(double) * n +
         2 * (n - 1) * (n / 2);
}

static int Fm_host(bool cplx, int64_t m) {
  int k = 0;
  while ((m >> (k + 1)) > 0) ++k;
  if (!cplx) return 1022 - k;
  const unsigned __int128 mm = static_cast<unsigned __int128>(m) * static_cast<unsigned __int128>(m);
  return 1021 - k - (mm >= (static_cast<unsigned __int128>(1) << (2 * k + 1)) ? 1 : 0);
}

}  // namespace jsvd

using namespace jsvd;

extern "C" jsvd_status jsvd_gesvj_batched(jsvd_dtype dt, int64_t batch, int64_t m, int64_t n,
                                          double* A, int64_t lda, int64_t strideA, double* V,
                                          int64_t ldv, int64_t strideV, double* sigma,
                                          int32_t max_sweeps, int32_t* sweeps_done,
                                          int32_t* status, void* stream) {
  const bool cplx = dt == JSVD_C64;
  if ((dt != JSVD_R64 && dt != JSVD_C64) || batch < 0 || m < n || n < 2 || (n & 1) || m > 128 ||
      n > 64 || lda < m || ldv < n || strideA < lda * n || strideV < ldv * n || max_sweeps < 0 ||
      !A || !V || !sigma)
    return JSVD_EINVAL;
  if (cplx && ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(V) & 15)))
    return JSVD_EINVAL;
  if (batch == 0) return JSVD_OK;
  const size_t smem = batched_smem(cplx, m, n);
  if (smem > 220 * 1024) return JSVD_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int Fm = Fm_host(cplx, m), Kr = cplx ? 1020 : 1022;
  const double tol = std::ldexp(std::sqrt(static_cast<double>(m)), -53);
  cudaError_t e;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<static_cast<unsigned>(batch), kBT, smem, st>>>(m, n, A, lda, strideA, V, ldv, strideV,
                                                           sigma, max_sweeps, sweeps_done, status,
                                                           Fm, Kr, tol);
  };
  if (cplx) {
    if (m <= 32) go(batched_svd_kernel<true, 1>);
    else if (m <= 64) go(batched_svd_kernel<true, 2>);
    else go(batched_svd_kernel<true, 4>);
  } else {
    if (m <= 32) go(batched_svd_kernel<false, 1>);
    else if (m <= 64) go(batched_svd_kernel<false, 2>);
    else go(batched_svd_kernel<false, 4>);
  }
  note_launch();
  e = cudaGetLastError();
  return e == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}

extern "C" jsvd_status jsvd_batched_rspec(jsvd_dtype dt, int64_t m, int32_t* W, int32_t* c,
                                          int32_t* offs, int32_t* noffs) {
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < 1 || m > 128 || !W || !c || !offs || !noffs)
    return JSVD_EINVAL;
  *W = 32;
  *c = 1;
  int k = 0;
  for (int o = 16; o >= 1; o /= 2) offs[k++] = o;
  *noffs = k;
  return JSVD_OK;
}
