// batched.cu -- jsvd_gesvj_batched: many independent small one-sided Jacobi
// SVDs (BASELINE configs[3]: 65536 complex 64 x 32), one CTA per matrix, the
// whole iteration (G and V) resident in shared memory: HBM is touched once to
// load A and once to store U, V, sigma.  Same arithmetic as jsvd_gesvj with
// nblocks = n (flat round-robin) and the reduction spec R = (W, 1, [W/2..1]),
// W = 8 for m <= 64 (16 above): lane L of a W-lane group owns rows L, L+W, ...
// of a pair, so one warp serves 32/W pairs at once and every shuffle of a
// reduction serves all of them.  W = 8 (128 threads, 8 rows per lane for
// configs[3]) issues ~30% fewer instructions per step than W = 16: the
// shuffle trees are one level shorter and the per-group overhead is spread
// over twice the rows.
//
// Per step (n/2 pairs; 16 W threads = 16 lane groups):
//   A  every lane group, one pair: exponent max, SSQ of x 2^-E (R#14) and the
//      dot of the columns prescaled by 2^-e (Alg 3.1) -- only the vector work
//      and the sums; the per-pair scalar tail goes to B
//   B  warp 0, ONE LANE PER PAIR: f = sqrt(g), the division of the dot, the
//      convergence test (Alg 3.2), the Grammian (Alg 3.3) and the 2x2 EVD of
//      every transformed pair -- the batch of EVDs of Alg 4.1 line 26
//      vectorised across lanes as the paper vectorises it across SIMD lanes
//
//   C  every lane group, one pair: rotation of its G and V columns (Alg 3.4);
//      M-tilde tracked by its high word (only floor(lg M-tilde) enters Eq. skr)
// The Eq. (skr) rescale check runs at every step (flat round-robin, R#21).
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "jsvd_host.h"
#include "step_dev.cuh"

namespace jsvd {

// Fast mode: every value of G~ is 0 or has |x| >= 2^-400,
// i.e. a high word (sign masked) of at least kFastLo (step_dev.cuh; nonzero
// values below 2^-1022 cannot occur in fast mode: their rotation inputs are
// >= 2^-400, so every nonzero output is >= 2^-905).
// sigma[b n] of a matrix batched_fast.cu's kernel hands over to this one
constexpr unsigned long long kFastMarker = 0x7ff8badc0ffee123ull;
size_t batched_fast_smem(bool cplx, int64_t n);
bool batched_fast_ok(int64_t m, int64_t n);
cudaError_t launch_batched_fast(bool cplx, int64_t batch, int64_t n, double* A, int64_t lda,
                            int64_t strideA, double* V, int64_t ldv, int64_t strideV,
                            double* sigma, int max_sweeps, int32_t* sweeps, int32_t* status,
                            int64_t* transforms, int32_t* scale, int Fm, int Kr, double tol,
                            int adj, unsigned long long* prof, cudaStream_t st);

// W lanes per pair (R.W = 8 for m <= 64, 16 above) and 16 lane groups per CTA
// (16 W threads): one pass of phases A and C covers the 16 pairs of n = 32
constexpr int kBNH = 16;

struct PairSlot {
  double ar, ai;  // sums of the prescaled dot (Alg 3.1 lines 5-6)
  double gp, gq;  // SSQ significands in [1, 4): f = sqrt(g) (R#14)
  int ep, eq;     // norm exponents (kIntMin: zero column, R#19)
  double c, C, S; // rotation (Alg 3.4)
  int transform;
  int pad;
};

// sum over the W lanes of each lane group, xor offsets W/2, ..., 1 (R)
template <int W>
__device__ __forceinline__ double hsum(double v) {
#pragma unroll
  for (int o = W / 2; o >= 1; o /= 2) v = v + __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int W>
__device__ __forceinline__ uint32_t hmax_u32(uint32_t v) {
#pragma unroll
  for (int o = W / 2; o >= 1; o /= 2) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int W>
__device__ __forceinline__ uint64_t hmax_u64(uint64_t v) {
#pragma unroll
  for (int o = W / 2; o >= 1; o /= 2) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}


// floor(lg max|component|) over the lane group's column slice x[0..NR):
// from the high words; a column whose largest component is subnormal (or zero)
// takes the exact 64-bit path (warp-uniform branch).  kIntMin: zero column.
template <int NR, int W, typename E>
__device__ __forceinline__ void col_exponents(const E* xp, const E* xq, int& Ep, int& Eq) {
  uint32_t hp = 0, hq = 0;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    hp = hi_max(xp[j], hp);
    hq = hi_max(xq[j], hq);
  }
  hp = hmax_u32<W>(hp);
  hq = hmax_u32<W>(hq);
  Ep = static_cast<int>(hp >> 20) - 1023;
  Eq = static_cast<int>(hq >> 20) - 1023;
  if (__any_sync(0xffffffffu, hp < 0x00100000u || hq < 0x00100000u)) {
    uint64_t mp = 0, mq = 0;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      mp = absmax_bits(xp[j], mp);
      mq = absmax_bits(xq[j], mq);
    }
    mp = hmax_u64<W>(mp);
    mq = hmax_u64<W>(mq);
    if (hp < 0x00100000u) Ep = ilogb_or_min(mp);
    if (hq < 0x00100000u) Eq = ilogb_or_min(mq);
  }
}

// e = E + k/2 and g = SSQ 2^-k (k even) from the SSQ of x 2^-E (R#14)
__device__ __forceinline__ void eg_from_ssq(int E, double ssq, int& e, double& g) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(ssq));
  int k = static_cast<int>(b >> 52) - 1023;
  g = __longlong_as_double(static_cast<long long>((b & 0x000fffffffffffffull) |
                                                  0x3ff0000000000000ull));
  if (k & 1) {
    g = g * 2.0;
    k -= 1;
  }
  e = E + k / 2;
}

// FULL: m == W NR (configs[3]: 64 = 8 x 8), so no row needs a bounds check
// PROF (diagnostic, jsvd_batched_phase_profile): every warp accumulates the
// clock64 cycles it spends in each phase of a step and in each barrier wait,
// added into prof[(warp == 0 ? 0 : 1) * 8 + k] at exit -- the paper's
// breakdown of Fig 5.4 for this kernel.
template <bool CPLX, int NR, bool FULL, int W, int VH = 0, bool PROF = false, bool FAST = true>
__global__ void __launch_bounds__(16 * W, W == 8 ? 5 : 2) batched_svd_kernel(
    int64_t m, int64_t n, double* A, int64_t lda, int64_t strideA, double* Vg, int64_t ldv,
    int64_t strideV, double* sigma, int max_sweeps, int32_t* sweeps_out, int32_t* status_out,
    int64_t* transforms_out, int32_t* scale_out, int Fm, int Kr, double tol, int s0_adjust,
    unsigned long long* prof = nullptr, int marked_only = 0) {
  using E = typename Elem<CPLX>::T;
  constexpr int kBT = kBNH * W, kBNW = kBT / 32, kBW = W, kGPW = 32 / W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  E* sG = reinterpret_cast<E*>(smem_raw);
  // V lives in global memory, in the matrix's own A storage (free once A is in
  // shared memory; V(i, j) at Ag[j lda + i], n <= m <= lda): shared memory then
  // holds only G, so 5 CTAs fit per SM.  V is touched only by the rotations in
  // phase B's shadow, where its L1/L2 latency is hidden.
  PairSlot* slots2 = reinterpret_cast<PairSlot*>(sG + m * n);  // [2][n/2]: steps alternate
  double* ce = reinterpret_cast<double*>(slots2 + n);
  double* cf = ce + n;
  // rows 0..VH-1 of the working V in shared memory (column-major, VH x n): the
  // fast half of every V rotation; rows VH.. live in A's storage
  E* sVh = reinterpret_cast<E*>(cf + n);
  uint8_t* sPairs = reinterpret_cast<uint8_t*>(sVh + VH * n);  // (n-1) x n/2 pivot pairs (n <= 64)
  __shared__ unsigned long long sM0;
  __shared__ uint32_t sMt;  // high word of M-tilde (its floor(lg) is all Eq. skr uses)
  __shared__ int sT;
  __shared__ int sBad;  // fast mode: the invariant of DESIGN.md 4.6 failed this step
  __shared__ uint64_t wred[kBNW];
  __shared__ int sSel[64];  // finalize: input column of each output rank

  const int64_t b = blockIdx.x;
  // after batched_fast.cu's kernel: only the matrices it handed over
  if (marked_only &&
      reinterpret_cast<const unsigned long long*>(sigma)[b * n] != kFastMarker)
    return;
  E* Ag = reinterpret_cast<E*>(A) + b * strideA;
  E* Vb = reinterpret_cast<E*>(Vg) + b * strideV;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hl = threadIdx.x & (W - 1), hw = threadIdx.x / W;
  const int np = static_cast<int>(n / 2);
  const int mi = static_cast<int>(m), ni = static_cast<int>(n);
  // the flat round-robin ordering (R#20), once per CTA
  for (int k = threadIdx.x; k < (ni - 1) * np; k += kBT) {
    int p, q;
    strategy_pair(ni, ni, k / np, k % np, p, q);
    sPairs[2 * k] = static_cast<uint8_t>(p);
    sPairs[2 * k + 1] = static_cast<uint8_t>(q);
  }

  // ---- load A, M0 = max |component| (NaN -> inf), V = I; mn = the smallest
  // nonzero |component| (bits; zero -> all ones), for the fast mode's check
  uint64_t mx = 0, mn = ~0ull;
  for (int k = threadIdx.x; k < mi * ni; k += kBT) {
    const int j = k / mi, i = k - j * mi;
    const E x = Ag[static_cast<int64_t>(j) * lda + i];
    sG[k] = x;
    if constexpr (CPLX) {
      mx = max(mx, abs_bits(fmin(fabs(x.x), static_cast<double>(INFINITY))));
      mx = max(mx, abs_bits(fmin(fabs(x.y), static_cast<double>(INFINITY))));
      if (FAST) mn = min(mn, min(abs_bits(x.x) - 1, abs_bits(x.y) - 1));
    } else {
      mx = max(mx, abs_bits(fmin(fabs(x), static_cast<double>(INFINITY))));
      if (FAST) mn = min(mn, abs_bits(x) - 1);
    }
  }
  {
    const uint64_t M0 = cta_max_u64<kBT>(mx, wred);
    if (threadIdx.x == 0) sM0 = M0;
    __syncthreads();
  }
  uint64_t mn_all = 0;
  if constexpr (FAST) {
    mn_all = ~cta_max_u64<kBT>(~mn, wred);  // min over the CTA
    __syncthreads();
  }
  const double M0 = __longlong_as_double(static_cast<long long>(sM0));
  if (isinf(M0) || M0 == 0.0) {
    if (threadIdx.x == 0) {
      if (status_out) status_out[b] = isinf(M0) ? JSVD_ENONFINITE : JSVD_ERANK;
      if (sweeps_out) sweeps_out[b] = 0;
      if (transforms_out) transforms_out[b] = 0;
      if (scale_out) scale_out[b] = 0;
    }
    return;
  }
  // ---- line 1: s0 = F(m) - floor(lg M0) - 1 (+ s0_adjust, R#40); G1 = 2^s0 G.
  // Fast mode: shared memory holds G~ = G 2^-cs with cs =
  // floor(lg M~1), i.e. G~ = A 2^-floor(lg M0), when every nonzero |a_ij| is
  // at least 2^-400 M0 (then every value of G~ is 0 or in [2^-400, 2^16]).
  int s = Fm - ilogb_bits(sM0) - 1 + s0_adjust;
  bool fast = false;
  int cs = 0;
  if constexpr (FAST) {
    const int lm0 = ilogb_bits(sM0);
    cs = lm0 + s;
    // G = G~ 2^cs must stay normal (G~ >= 2^-905 needs cs >= 0), and the
    // squares of G~ <= 2^(1024 - cs) must not overflow (cs >= 600)
    fast = (mn_all == ~0ull || ilogb_bits(mn_all + 1) >= lm0 - 400) && cs >= 600;
  }
  {
    const int sh = fast ? s - cs : s;
    for (int k = threadIdx.x; k < mi * ni; k += kBT) {
      if constexpr (CPLX) sG[k] = make_double2(scalbn_rn(sG[k].x, sh), scalbn_rn(sG[k].y, sh));
      else sG[k] = scalbn_rn(sG[k], sh);
    }
  }
  if (threadIdx.x == 0) {
    sMt = hi32(scalbn_rn(M0, s));
    sBad = 0;
  }
  // leave the fast mode (CTA-uniform, after a barrier): G = G~ 2^cs exactly,
  // every value of G~ being 0 or normal
  const auto leave_fast = [&]() {
    for (int kk = threadIdx.x; kk < mi * ni; kk += kBT) {
      if constexpr (CPLX) sG[kk] = make_double2(scalbn_rn(sG[kk].x, cs), scalbn_rn(sG[kk].y, cs));
      else sG[kk] = scalbn_rn(sG[kk], cs);
    }
    fast = false;
    __syncthreads();
  };
  // V = I over A's storage (every read of A above precedes the barrier in
  // cta_max_u64)
  for (int k = threadIdx.x; k < ni * ni; k += kBT) {
    const int j = k / ni, i = k - j * ni;
    E v;
    if constexpr (CPLX) v = make_double2(i == j ? 1.0 : 0.0, 0.0);
    else v = i == j ? 1.0 : 0.0;
    if (i < VH) sVh[j * VH + i] = v;
    else Ag[static_cast<int64_t>(j) * lda + i] = v;
  }
  __syncthreads();

  // V of step k is rotated by warps 1.. while warp 0 runs phase B of step
  // k+1 (V never enters a decision, Alg 3.4 applies the same (c, C, S) to it);
  // the slots of consecutive steps alternate between two buffers
  const auto rotate_v = [&](const PairSlot* sl_, int kstep, int l_begin, int l_step, int lane0,
                            int lanes) {
    for (int l = l_begin; l < np; l += l_step) {
      const PairSlot& sl = sl_[l];
      if (!sl.transform) continue;
      const int p = sPairs[2 * (kstep * np + l)], q = sPairs[2 * (kstep * np + l) + 1];
      E* vp = Ag + static_cast<int64_t>(p) * lda;
      E* vq = Ag + static_cast<int64_t>(q) * lda;
      // one row at a time: prefetching rows costs registers, and at the
      // 96-register cap of 5 CTAs per SM any spill costs more than it hides;
      // the shared-memory rows first (short latency), then the global ones
      int i = lane0;
      for (; i < VH && i < ni; i += lanes) {
        E* sp = sVh + p * VH;
        E* sq = sVh + q * VH;
        E a = sp[i], bq = sq[i];
        rot_elem(a, bq, sl.c, sl.C, sl.S);
        sp[i] = a;
        sq[i] = bq;
      }
      for (; i < ni; i += lanes) {
        E a = vp[i], bq = vq[i];
        rot_elem(a, bq, sl.c, sl.C, sl.S);
        vp[i] = a;
        vq[i] = bq;
      }
    }
  };
  int pend_k = -1, pend_buf = 0;  // step whose V rotation is pending
  int gstep = 0;
  int C = 0;
  int64_t Ttot = 0;  // transformed pair-steps (thread 0)
  bool converged = false;
  // PROF: cycles per warp in [0] phase A, [1] wait after A, [2] phase B
  // (warp 0) / V rotation (warps 1..), [3] wait after B, [4] phase C, [5] wait
  // after C, [6] rescale check, [7] whole sweep loop
  unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = 0, tloop = 0;
  const auto mark = [&](int k) {
    if constexpr (PROF) {
      const long long t = clock64();
      pc[k] += static_cast<unsigned long long>(t - tprev);
      tprev = t;
    }
  };
  if constexpr (PROF) tloop = tprev = clock64();
  for (C = 0; C < max_sweeps; ++C) {
    if (threadIdx.x == 0) sT = 0;
    for (int k = 0; k < ni - 1; ++k, ++gstep) {
      PairSlot* slots = slots2 + (gstep & 1) * np;
      if constexpr (PROF) tprev = clock64();
      // ---- line 6: rescale check (every step for flat round-robin); M-tilde
      // is normal here (G is scaled to ~ omega / m), so its high word's
      // exponent field is floor(lg M-tilde)
      {
        const int lm = static_cast<int>(sMt >> 20) - 1023;
        const int sn = (Kr - lm < 0) ? Fm - lm - 1 : 0;
        if (sn != 0 && fast) {  // G = G~ 2^cs: the scaling moves into cs
          __syncthreads();
          if (threadIdx.x == 0) sMt = hi32(scalbn_rn(mkd(sMt, 0u), sn));
          cs += sn;
          s += sn;
          __syncthreads();
        } else if (sn != 0) {  // uniform
          __syncthreads();
          for (int kk = threadIdx.x; kk < mi * ni; kk += kBT) {
            if constexpr (CPLX) sG[kk] = make_double2(scalbn_rn(sG[kk].x, sn), scalbn_rn(sG[kk].y, sn));
            else sG[kk] = scalbn_rn(sG[kk], sn);
          }
          if (threadIdx.x == 0) sMt = hi32(scalbn_rn(mkd(sMt, 0u), sn));
          s += sn;
          __syncthreads();
        }
      }
      mark(6);
      // ---- phase A: lane group per pair: exponent max, SSQ, prescaled dot.
      // Fast mode: G~ needs no prescaling -- the SSQ and the dot of the raw
      // values are exact power-of-two multiples of the oracle's (DESIGN.md
      // 4.6), accumulated in one pass in the same lane order R; B rescales.
      if (fast) {
        for (int l0 = 0; l0 < np; l0 += kBNH) {
          const int l = l0 + hw;
          const bool act = l < np;
          const int p = act ? sPairs[2 * (k * np + l)] : 0;
          const int q = act ? sPairs[2 * (k * np + l) + 1] : 1;
          const E* gp = sG + p * mi;
          const E* gq = sG + q * mi;
          double sp = 0.0, sq = 0.0, ar = 0.0, ai = 0.0;
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            const int i = j * kBW + hl;
            const E xpj = (FULL || i < mi) ? gp[i] : Elem<CPLX>::zero();
            const E xqj = (FULL || i < mi) ? gq[i] : Elem<CPLX>::zero();
            sp = ssq_acc(xpj, sp);
            sq = ssq_acc(xqj, sq);
            dot_acc(xqj, xpj, ar, ai);
          }
          sp = hsum<W>(sp);
          sq = hsum<W>(sq);
          ar = hsum<W>(ar);
          if (CPLX) ai = hsum<W>(ai);
          if (act && hl == 0) {
            PairSlot& sl = slots[l];
            sl.ar = ar;
            sl.ai = ai;
            sl.gp = sp;  // the raw SSQ of G~ (B derives (e, f))
            sl.gq = sq;
          }
        }
      } else
      for (int l0 = 0; l0 < np; l0 += kBNH) {  // uniform trip count: both halves shuffle
        const int l = l0 + hw;
        const bool act = l < np;
        const int p = act ? sPairs[2 * (k * np + l)] : 0;
        const int q = act ? sPairs[2 * (k * np + l) + 1] : 1;
        const E* gp = sG + p * mi;
        const E* gq = sG + q * mi;
        E xp[NR], xq[NR];
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          const int i = j * kBW + hl;
          xp[j] = (FULL || i < mi) ? gp[i] : Elem<CPLX>::zero();
          xq[j] = (FULL || i < mi) ? gq[i] : Elem<CPLX>::zero();
        }
        int Ep, Eq;
        col_exponents<NR, W>(xp, xq, Ep, Eq);
        double sp = Ep != kIntMin ? ssq_lane<NR>(xp, Ep) : 0.0;
        double sq = Eq != kIntMin ? ssq_lane<NR>(xq, Eq) : 0.0;
        sp = hsum<W>(sp);
        sq = hsum<W>(sq);
        int ep = kIntMin, eq = kIntMin;
        double gpv = 1.0, gqv = 1.0;
        if (Ep != kIntMin) eg_from_ssq(Ep, sp, ep, gpv);
        if (Eq != kIntMin) eg_from_ssq(Eq, sq, eq, gqv);
        const bool zero_col = (Ep == kIntMin) || (Eq == kIntMin);  // R#19
        double ar = 0.0, ai = 0.0;
        if (!zero_col) dot_lane<NR>(xq, xp, eq, ep, ar, ai);
        ar = hsum<W>(ar);
        if (CPLX) ai = hsum<W>(ai);
        if (act && hl == 0) {
          PairSlot& sl = slots[l];
          sl.ar = zero_col ? 0.0 : ar;
          sl.ai = zero_col ? 0.0 : ai;
          sl.gp = gpv;
          sl.gq = gqv;
          sl.ep = ep;
          sl.eq = eq;
        }
      }
      mark(0);
      __syncthreads();
      mark(1);
      // ---- phase B: norms' f, the dot's division, convergence test,
      // Grammian and EVD of the step, one lane per pair
      if (warp == 0) {
        int tcount = 0;
        for (int l0 = 0; l0 < np; l0 += 32) {
          const int l = l0 + lane;
          const bool act = l < np;
          const PairSlot& s0 = slots[act ? l : 0];
          bool zp, zq;
          int iep, ieq;
          double gpv, gqv, arv = s0.ar, aiv = s0.ai;
          if (fast) {
            // the raw SSQ of G~ = G 2^-cs is 2^(2E - 2cs) times the oracle's
            // SSQ of x 2^-E (exactly), so R#14's (e, f) follow with E := cs;
            // the dot of G~ is 2^(e_q + e_p - 2cs) times the prescaled one
            zp = !(s0.gp > 0.0);
            zq = !(s0.gq > 0.0);
            iep = ieq = kIntMin;
            gpv = gqv = 1.0;
            if (!zp) eg_from_ssq(cs, s0.gp, iep, gpv);
            if (!zq) eg_from_ssq(cs, s0.gq, ieq, gqv);
            if (!(zp || zq)) {
              const double f2 = pow2i(2 * cs - iep - ieq);
              arv *= f2;
              aiv *= f2;
            }
            if (act) {
              slots[l].ep = iep;
              slots[l].eq = ieq;
            }
          } else {
            zp = s0.ep == kIntMin;
            zq = s0.eq == kIntMin;
            iep = s0.ep;
            ieq = s0.eq;
            gpv = s0.gp;
            gqv = s0.gq;
          }
          const double fp = zp ? 1.0 : sqrt_plain(gpv), fq = zq ? 1.0 : sqrt_plain(gqv);
          const double ep = zp ? -INFINITY : static_cast<double>(iep);
          const double eq = zq ? -INFINITY : static_cast<double>(ieq);
          // z = (ar, ai) / fl(fq fp), fl(fq fp) in [1, 4) (Alg 3.1 line 8)
          const Rcp d = rcp_plain(fq * fp);
          const double zr = dot_div(arv, d, kFull);
          const double zi = CPLX ? dot_div(aiv, d, kFull) : 0.0;
          const double az = CPLX ? hypot_naive(fabs(zr), fabs(zi)) : fabs(zr);
          const bool tr = act && !(zp || zq) && tol <= az;  // Alg 3.2
          if (__any_sync(kFull, tr)) {
            double b11, b22, br, bi;
            gram_fast(tr ? zr : 0.0, tr ? zi : 0.0, tr ? ep : 0.0, tr ? fp : 1.0, tr ? eq : 0.0,
                      tr ? fq : 1.0, b11, b22, br, bi, kFull);
            const Evd2Out o = evd2<CPLX, true, true, false>(b11, b22, br, bi, kFull);
            if (tr) {
              slots[l].c = o.c;
              slots[l].C = o.sr;
              slots[l].S = o.si;
            }
            // fast mode needs C, S in {0} u [2^-400, 1]
            const bool bad = fast && tr &&
                             (abs_hi(o.sr) - 1u < kFastLo - 1u || abs_hi(o.si) - 1u < kFastLo - 1u);
            if (__any_sync(kFull, bad) && lane == 0) sBad = 1;
          }
          if (act) slots[l].transform = tr;
          tcount += __popc(__ballot_sync(0xffffffffu, tr));
        }
        if (lane == 0) sT += tcount;
      } else if (pend_k >= 0) {  // the lane groups of warps 1..: V of the previous step
        rotate_v(slots2 + pend_buf * np, pend_k, hw - kGPW, kBNH - kGPW, hl, kBW);
      }
      mark(2);
      __syncthreads();
      mark(3);
      if (fast && sBad) leave_fast();  // a C or S below 2^-400: rotate in G's scale
      // ---- phase C: rotations of G (Alg 3.4), M-tilde
      uint32_t Mw = 0, lmin = ~0u;
      for (int l = hw; l < np; l += kBNH) {
        const PairSlot& sl = slots[l];
        if (!sl.transform) continue;
        const int p = sPairs[2 * (k * np + l)], q = sPairs[2 * (k * np + l) + 1];
        const double c = sl.c, Cc = sl.C, S = sl.S;
        E* gp = sG + p * mi;
        E* gq = sG + q * mi;
        // M-tilde only matters once it reaches 2^(K+1) (Eq. skr): every
        // component after the rotation is below 2^(max(e_p,e_q) + 1.5), so a
        // pair with max(e) <= K - 1 is not tracked (same checks and rescales
        // as the exact M; see step.cu)
        const bool track = max(sl.ep, sl.eq) > Kr - 1;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          const int i = j * kBW + hl;
          if (FULL || i < mi) {
            E a = gp[i], bq = gq[i];
            rot_elem(a, bq, c, Cc, S);
            gp[i] = a;
            gq[i] = bq;
            if (track) {
              Mw = hi_max(a, Mw);
              Mw = hi_max(bq, Mw);
            }
            if (fast) lmin = lo_hi_min(a, lo_hi_min(bq, lmin));
          }
        }
      }
      pend_k = k;
      pend_buf = gstep & 1;
      Mw = __reduce_max_sync(0xffffffffu, Mw);
      if (fast && Mw) Mw += static_cast<uint32_t>(cs) << 20;  // G = G~ 2^cs (normal values)
      if (lane == 0 && Mw > sMt) atomicMax(&sMt, Mw);
      // fast mode keeps every value of G~ in {0} u [2^-400, 2^16]
      if (fast && lmin < kFastLo - 1u) sBad = 1;
      mark(4);
      __syncthreads();
      mark(5);
      if (fast && sBad) leave_fast();
    }
    if (threadIdx.x == 0) Ttot += sT;
    if (sT == 0) {
      converged = true;
      ++C;
      break;
    }
    __syncthreads();
  }
  if constexpr (PROF) {
    pc[7] = static_cast<unsigned long long>(clock64() - tloop);
    if (lane == 0)
      for (int k = 0; k < 8; ++k) atomicAdd(&prof[(warp == 0 ? 0 : 1) * 8 + k], pc[k]);
  }
  if (pend_k >= 0) {  // the last step's V rotation
    rotate_v(slots2 + pend_buf * np, pend_k, hw, kBNH, hl, kBW);
    __syncthreads();
  }
  if (fast) leave_fast();
  // ---- finalize: norms with the step's R (R#23),
  // U = G diag(2^-e / f), sigma, sort
  for (int j0 = 0; j0 < ni; j0 += kBNH) {  // lane group per column, uniform trip count
    const int j = j0 + hw;
    const bool act = j < ni;
    const E* g = sG + (act ? j : 0) * mi;
    E x[NR];
    uint64_t mj = 0;
#pragma unroll
    for (int jj = 0; jj < NR; ++jj) {
      const int i = jj * kBW + hl;
      x[jj] = (FULL || i < mi) ? g[i] : Elem<CPLX>::zero();
      mj = absmax_bits(x[jj], mj);
    }
    mj = hmax_u64<W>(mj);
    const int Ej = ilogb_or_min(mj);
    double sj = 0.0;
    if (Ej != kIntMin) {
      const Pow2 f(-Ej);
#pragma unroll
      for (int jj = 0; jj < NR; ++jj)
        if (FULL || jj * kBW + hl < mi) sj = ssq_acc(f(x[jj]), sj);
    }
    sj = hsum<W>(sj);
    double e = -INFINITY, f = 1.0;
    if (Ej != kIntMin) ef_from_ssq(Ej, sj, e, f);
    if (act && hl == 0) {
      ce[j] = e;
      cf[j] = f;
    }
  }
  __syncthreads();
  // converged: sigma sorted (R#24), U normalised; not converged (C = S):
  // Alg 4.1 line 41 does not finalize -- U = G, V and Sigma' (not backscaled)
  // in column order (R#25)
  for (int r0 = warp; r0 < ni; r0 += kBNW) {
    // output column r0 <- input column j with rank r0
    int jsel = converged ? 0 : r0 + 1;
    for (int j = lane; converged && j < ni; j += 32) {
      const double ej = ce[j], fj = cf[j];
      int rank = 0;
      for (int kk = 0; kk < ni; ++kk) {
        const double ek = ce[kk], fk = cf[kk];
        rank += ((ek > ej) || (ek == ej && (fk > fj || (fk == fj && kk < j)))) ? 1 : 0;
      }
      if (rank == r0) jsel = j + 1;
    }
    jsel = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(jsel));
    const int j = jsel - 1;
    if (lane == 0) sSel[r0] = j;
    // V's output column r0 from the working V in A's storage
    E* vcol = Vb + static_cast<int64_t>(r0) * ldv;
    const E* vw = Ag + static_cast<int64_t>(j) * lda;
    for (int i = lane; i < ni; i += 32) vcol[i] = i < VH ? sVh[j * VH + i] : vw[i];
    if (lane == 0) {
      const double e = ce[j], f = cf[j];
      const bool fin = !isinf(e);
      const double es = (fin && converged) ? e - s : e;
      sigma[b * n + r0] = fin ? scalbn_rn(f, static_cast<int>(fmax(fmin(es, 1e5), -1e5))) : 0.0;
    }
  }
  __syncthreads();  // every read of the working V precedes the writes of U over it
  for (int r0 = warp; r0 < ni; r0 += kBNW) {
    const int j = sSel[r0];
    const double e = ce[j], f = cf[j];
    const bool fin = !isinf(e) && converged;
    const Pow2 sc(fin ? -static_cast<int>(e) : 0);
    const Divisor d = make_divisor(f);
    E* ucol = Ag + static_cast<int64_t>(r0) * lda;
    const E* g = sG + j * mi;
    for (int i = lane; i < mi; i += 32) {
      E x = g[i];
      if (fin) {
        if constexpr (CPLX) x = make_double2(divide(sc(x.x), d), divide(sc(x.y), d));
        else x = divide(sc(x), d);
      }
      ucol[i] = x;
    }
  }
  if (threadIdx.x == 0) {
    if (status_out) status_out[b] = converged ? JSVD_OK : JSVD_ENOCONV;
    if (sweeps_out) sweeps_out[b] = C;
    if (transforms_out) transforms_out[b] = Ttot;
    if (scale_out) scale_out[b] = s;
  }
}

// lanes per pair of the kernel jsvd_gesvj_batched launches for m (R.W)
static int batched_w(int64_t m) { return m <= 64 ? 8 : 16; }

static size_t batched_smem(bool cplx, int64_t m, int64_t n, int vh = 0) {
  const size_t w = cplx ? 16 : 8;
  return w * (m * n) + sizeof(PairSlot) * n + 2 * sizeof(double) * n + w * vh * n +
         2 * (n - 1) * (n / 2);
}

static int Fm_host(bool cplx, int64_t m) {
  int k = 0;
  while ((m >> (k + 1)) > 0) ++k;
  if (!cplx) return 1022 - k;
  const unsigned __int128 mm = static_cast<unsigned __int128>(m) * static_cast<unsigned __int128>(m);
  return 1021 - k - (mm >= (static_cast<unsigned __int128>(1) << (2 * k + 1)) ? 1 : 0);
}

// the shape / dtype conditions of jsvd_gesvj_batched (also checked by the
// host-buffer entry point before it queues anything)
bool gesvj_batched_args_ok(jsvd_dtype dt, int64_t m, int64_t n) {
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < n || n < 2 || (n & 1) || m > 128 || n > 64)
    return false;
  return batched_smem(dt == JSVD_C64, m, n) <= 220 * 1024;
}

}  // namespace jsvd

using namespace jsvd;

static jsvd_status batched_impl(jsvd_dtype dt, int64_t batch, int64_t m, int64_t n, double* A,
                                int64_t lda, int64_t strideA, double* V, int64_t ldv,
                                int64_t strideV, double* sigma, int32_t max_sweeps,
                                int32_t* sweeps_done, int32_t* status, int64_t* transforms,
                                int32_t* scale, const jsvd_gesvj_opts* opts, void* stream,
                                unsigned long long* prof) {
  const bool cplx = dt == JSVD_C64;
  if (!gesvj_batched_args_ok(dt, m, n) || batch < 0 || lda < m || ldv < n || strideA < lda * n || strideV < ldv * n || max_sweeps < 0 ||
      !A || !V || !sigma)
    return JSVD_EINVAL;
  if (cplx && ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(V) & 15)))
    return JSVD_EINVAL;
  if (batch == 0) return JSVD_OK;
  const size_t smem = batched_smem(cplx, m, n);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int Fm = Fm_host(cplx, m), Kr = cplx ? 1020 : 1022;
  const int adj = opts ? opts->s0_adjust : 0;
  if ((opts && opts->max_steps) || adj < -2200 || adj > 1024 - Fm) return JSVD_EINVAL;
  const double tol = std::ldexp(std::sqrt(static_cast<double>(m)), -53);
  cudaError_t e;
  int marked = 0;  // 1: only the matrices batched_fast.cu's kernel handed over
  auto go = [&](auto kern, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<static_cast<unsigned>(batch), threads, smem, st>>>(m, n, A, lda, strideA, V, ldv, strideV,
                                                              sigma, max_sweeps, sweeps_done, status,
                                                              transforms, scale, Fm, Kr, tol, adj,
                                                              prof, marked);
  };
  // W = batched_w(m) lanes per pair; NR = rows per lane
  // 16 rows of V in shared memory when 5 CTAs per SM still fit (64 x 32 complex)
  const size_t smem16 = batched_smem(cplx, m, n, 16);
  auto go16 = [&](auto kern, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem16));
    kern<<<static_cast<unsigned>(batch), threads, smem16, st>>>(m, n, A, lda, strideA, V, ldv,
                                                                strideV, sigma, max_sweeps,
                                                                sweeps_done, status, transforms, scale,
                                                                Fm, Kr, tol, adj, prof, marked);
  };
  // JSVD_BATCHED_VH=0 keeps all of V in A's storage (same results, bit for
  // bit: only where V lives changes; the GPU tests compare both)
  const char* vh_s = getenv("JSVD_BATCHED_VH");
  const int vh_env = vh_s ? atoi(vh_s) : 1;
  bool vh16 = false;
  if (vh_env && n <= 32) {
    int dev = 0, per_sm = 0, reserved = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    vh16 = 5 * (smem16 + 320 + static_cast<size_t>(reserved)) <= static_cast<size_t>(per_sm);
  }
  // JSVD_BATCHED_FAST=0: never use the scaled fast kernels (
  // same results bit for bit -- the GPU tests compare both)
  const char* fast_s = getenv("JSVD_BATCHED_FAST");
  const bool fast_env = !fast_s || atoi(fast_s) != 0;
  const char* b2_s = getenv("JSVD_BATCHED_KERNEL");  // 0: batched.cu's kernel for configs[3] too (A/B runs)
  const bool b2_env = !b2_s || atoi(b2_s) != 0;
  if (fast_env && b2_env && batched_fast_ok(m, n)) {
    // configs[3]'s shape: the persistent two-slot kernel (batched_fast.cu), then
    // this kernel, in G's own scale, on the matrices it handed over
    e = launch_batched_fast(cplx, batch, n, A, lda, strideA, V, ldv, strideV, sigma, max_sweeps,
                        sweeps_done, status, transforms, scale, Fm, Kr, tol, adj, prof, st);
    if (e != cudaSuccess) return JSVD_ECUDA;
    marked = 1;
    prof = nullptr;
  } else if (prof && !(m == 64 && vh16)) {
    return JSVD_EINVAL;  // the profile covers configs[3]'s kernels
  }
  auto pick = [&](auto cplx_t) {
    constexpr bool C = decltype(cplx_t)::value;
    if (prof && fast_env) go16(batched_svd_kernel<C, 8, true, 8, 16, true, true>, 128);
    else if (prof) go16(batched_svd_kernel<C, 8, true, 8, 16, true, false>, 128);
    else if (m == 32) go(batched_svd_kernel<C, 4, true, 8>, 128);
    else if (m == 64 && vh16 && fast_env && !marked) go16(batched_svd_kernel<C, 8, true, 8, 16>, 128);
    else if (m == 64 && vh16) go16(batched_svd_kernel<C, 8, true, 8, 16, false, false>, 128);
    else if (m == 64) go(batched_svd_kernel<C, 8, true, 8>, 128);
    else if (m < 32) go(batched_svd_kernel<C, 4, false, 8>, 128);
    else if (m < 64) go(batched_svd_kernel<C, 8, false, 8>, 128);
    else if (m == 128) go(batched_svd_kernel<C, 8, true, 16>, 256);
    else go(batched_svd_kernel<C, 8, false, 16>, 256);
  };
  if (cplx) pick(std::true_type{});
  else pick(std::false_type{});
  note_launch();
  e = cudaGetLastError();
  return e == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}

extern "C" jsvd_status jsvd_gesvj_batched(jsvd_dtype dt, int64_t batch, int64_t m, int64_t n,
                                          double* A, int64_t lda, int64_t strideA, double* V,
                                          int64_t ldv, int64_t strideV, double* sigma,
                                          int32_t max_sweeps, int32_t* sweeps_done,
                                          int32_t* status, int64_t* transforms, int32_t* scale,
                                          const jsvd_gesvj_opts* opts, void* stream) {
  return batched_impl(dt, batch, m, n, A, lda, strideA, V, ldv, strideV, sigma, max_sweeps,
                      sweeps_done, status, transforms, scale, opts, stream, nullptr);
}

extern "C" jsvd_status jsvd_batched_phase_profile(jsvd_dtype dt, int64_t batch, int64_t m,
                                                  int64_t n, double* A, int64_t lda,
                                                  int64_t strideA, double* V, int64_t ldv,
                                                  int64_t strideV, double* sigma,
                                                  int32_t max_sweeps, unsigned long long* prof,
                                                  void* stream) {
  if (!prof) return JSVD_EINVAL;
  if (cudaMemsetAsync(prof, 0, 16 * sizeof(unsigned long long), static_cast<cudaStream_t>(stream)) !=
      cudaSuccess)
    return JSVD_ECUDA;
  return batched_impl(dt, batch, m, n, A, lda, strideA, V, ldv, strideV, sigma, max_sweeps,
                      nullptr, nullptr, nullptr, nullptr, nullptr, stream, prof);
}

extern "C" jsvd_status jsvd_batched_rspec(jsvd_dtype dt, int64_t m, int32_t* W, int32_t* c,
                                          int32_t* offs, int32_t* noffs) {
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < 1 || m > 128 || !W || !c || !offs || !noffs)
    return JSVD_EINVAL;
  *W = batched_w(m);
  *c = 1;
  int k = 0;
  for (int o = *W / 2; o >= 1; o /= 2) offs[k++] = o;
  *noffs = k;
  return JSVD_OK;
}
