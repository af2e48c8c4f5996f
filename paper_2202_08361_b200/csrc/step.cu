// step.cu -- jsvd_sweep_step and the per-step kernel of jsvd_gesvj:
// one parallel step of the one-sided Jacobi SVD (Alg 4.1 lines 7-38,
// P:1530-1583) with s = 1 (R#13) and P = I (R#20).
//
// One pivot pair per CTA, or per thread-block cluster of CL CTAs when the
// columns are long (DSMEM carries the cross-CTA reductions).  The pair's two
// columns are loaded ONCE into registers (lane L = i mod W holds rows L, L+W,
// ...: coalesced 8/16-byte loads), and every phase of the step runs on them:
//   spade  column norms: exponent max, then SSQ of x 2^-E        (R#14)
//   club   scaled dot a21' = g_q^* g_p (Alg 3.1)
//   heart  convergence test (Alg 3.2), Grammian (Alg 3.3)     -- warp 0
//   diam.  2x2 EVD (Alg 2.2, TAN|NOBACKSCALE)                 -- warp 0
//   star   rotation of g_p, g_q in registers + store, then v_p, v_q (Alg 3.4)
// so G is read once and written once per transformed pair, V read+written
// once per transformed pair, nothing for a converged pair (R#26: no max on V).
#include <cstdlib>
#include <mutex>
#include <vector>
#include <utility>

#include "jsvd_host.h"
#include "step_dev.cuh"
#include "step_params.h"

#ifndef JSVD_STEP_NV_REAL
#define JSVD_STEP_NV_REAL 4
#endif
#ifndef JSVD_STEP_NV_CPLX
#define JSVD_STEP_NV_CPLX 4
#endif

namespace jsvd {

// 16-byte / 8-byte asynchronous global -> shared copies (LDGSTS), zero-filled
// past the end of the column (src_size 0)
__device__ __forceinline__ void cp_async_el(double2* dst, const double2* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src),
               "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void cp_async_el(double* dst, const double* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
               "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
// a hint: [ptr, ptr + bytes) into L2 (16-byte aligned interior, 1 MB requests)
__device__ __forceinline__ void prefetch_l2(const void* ptr, int64_t bytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(ptr);
  const uintptr_t e = (a + static_cast<uintptr_t>(bytes > 0 ? bytes : 0)) & ~uintptr_t(15);
  a = (a + 15) & ~uintptr_t(15);
  for (; a < e; a += (1u << 20)) {
    const uint32_t sz = static_cast<uint32_t>(e - a < (1u << 20) ? e - a : (1u << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"(sz) : "memory");
  }
}

__device__ __forceinline__ double scalbn_el(double x, int n) { return scalbn_rn(x, n); }
__device__ __forceinline__ double2 scalbn_el(double2 x, int n) {
  return make_double2(scalbn_rn(x.x, n), scalbn_rn(x.y, n));
}

// Lane L of the W = T*CL lanes holds rows j*W + L of both columns: j < NR in
// registers, NR <= j < NR+NS in shared memory (NS > 0 for the longest columns:
// twice the rows per lane at the same register count, so a pair needs half the
// CTAs and twice as many pairs are resident).  Every pass walks j upwards, so
// the per-lane accumulation order of R is unchanged.
template <bool CPLX, int T, int CL, int NR, int NS>
__global__ void __launch_bounds__(T, 2) step_kernel(const StepParams P) {
  using E = typename Elem<CPLX>::T;
  constexpr int W = T * CL;
  constexpr int NW = T / 32;
  __shared__ RedSlot<NW, int> rs_e;
  __shared__ RedSlot<NW, double> rs_ssq;
  __shared__ RedSlot<NW, double> rs_dot;
  __shared__ uint32_t rs_m[NW];
  __shared__ double rot[3];
  __shared__ TxSlot<CL, int> tx_e;
  __shared__ TxSlot<CL, double> tx_ssq, tx_dot, tx_f1, tx_f2;
  __shared__ RedSlot<NW, double> rs_f1, rs_f2;
  extern __shared__ __align__(16) unsigned char step_smem[];
  E* sx = reinterpret_cast<E*>(step_smem);  // [NS][2][T]
  const auto sP = [&](int j) -> E& { return sx[(2 * j) * T + threadIdx.x]; };
  const auto sQ = [&](int j) -> E& { return sx[(2 * j + 1) * T + threadIdx.x]; };

  // programmatic dependent launch: the next step's CTAs may be scheduled into
  // the SMs this step's last wave frees; no global data is touched before the
  // previous step has completed and its memory is visible
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int crank = CL > 1 ? static_cast<int>(blockIdx.x % CL) : 0;
  const int64_t pair = blockIdx.x / CL;
  if constexpr (CL > 1) {  // the DSMEM rounds' mbarriers (published before any push)
    if (threadIdx.x == 0) {
      txslot_init(tx_e);
      txslot_init(tx_ssq);
      txslot_init(tx_dot);
      txslot_init(tx_f1);
      txslot_init(tx_f2);
    }
    txred_publish();
  }
  int p, q;
  if (P.pairs) {
    p = P.pairs[2 * pair];
    q = P.pairs[2 * pair + 1];
  } else if (P.dist_nr > 0) {
    dist_pair(static_cast<int>(P.n), static_cast<int>(P.B), P.dist_nr, P.dist_rank,
              static_cast<int>(P.step), static_cast<int>(pair), p, q);
  } else {
    strategy_pair(P.n, P.B, P.step, pair, p, q);
  }
  if (P.pf > 0 && threadIdx.x == 0) {
    // L2 prefetch of the pair P.pf pairs ahead (one resident wave): this
    // CTA's 1/CL of both columns, as bulk requests through the TMA unit
    const int64_t pair2 = pair + P.pf;
    if (pair2 < static_cast<int64_t>(gridDim.x / CL)) {
      int p2, q2;
      if (P.pairs) {
        p2 = P.pairs[2 * pair2];
        q2 = P.pairs[2 * pair2 + 1];
      } else if (P.dist_nr > 0) {
        dist_pair(static_cast<int>(P.n), static_cast<int>(P.B), P.dist_nr, P.dist_rank,
                  static_cast<int>(P.step), static_cast<int>(pair2), p2, q2);
      } else {
        strategy_pair(P.n, P.B, P.step, pair2, p2, q2);
      }
      const int64_t rows = (P.m + CL - 1) / CL, r0 = crank * rows;
      const int64_t nr = min(rows, P.m - r0);
      const E* G0 = reinterpret_cast<const E*>(P.G);
      prefetch_l2(G0 + static_cast<int64_t>(p2) * P.ldg + r0, nr * static_cast<int64_t>(sizeof(E)));
      prefetch_l2(G0 + static_cast<int64_t>(q2) * P.ldg + r0, nr * static_cast<int64_t>(sizeof(E)));
      if (P.V && P.pfv) {  // and its V columns (used if the pair transforms)
        const int64_t vr = (P.n + CL - 1) / CL, v0 = crank * vr, vn = min(vr, P.n - v0);
        const E* V0 = reinterpret_cast<const E*>(P.V);
        prefetch_l2(V0 + static_cast<int64_t>(p2) * P.ldv + v0, vn * static_cast<int64_t>(sizeof(E)));
        prefetch_l2(V0 + static_cast<int64_t>(q2) * P.ldv + v0, vn * static_cast<int64_t>(sizeof(E)));
      }
    }
  }
  const int L = crank * T + static_cast<int>(threadIdx.x);
  E* gp = reinterpret_cast<E*>(P.G) + static_cast<int64_t>(p) * P.ldg;
  E* gq = reinterpret_cast<E*>(P.G) + static_cast<int64_t>(q) * P.ldg;
  const bool lead = (crank == 0) && (threadIdx.x == 0);

  // @phase load+rescale
  // the shared-memory rows first (asynchronous), then the register rows
#pragma unroll 2
  for (int j = 0; j < NS; ++j) {
    const int64_t i = static_cast<int64_t>(NR + j) * W + L;
    const bool ok = i < P.m;
    cp_async_el(&sP(j), gp + (ok ? i : 0), ok);
    cp_async_el(&sQ(j), gq + (ok ? i : 0), ok);
  }
  if constexpr (NS > 0) asm volatile("cp.async.commit_group;\n" ::);

  // rescale check (Alg 4.1 line 6; Eqs. skn/skr; R#21): every step touches all
  // n columns, so each pair scales its own two columns on load.
  int sn = 0;
  uint64_t mt_cur = 0;
  if (P.Mt) {
    mt_cur = P.Mt[P.slot];
    if (P.checkpoint) {
      const int lm = ilogb_bits(mt_cur);
      if (P.Kr - lm < 0) sn = P.Fm - lm - 1;
    }
  }

  E xp[NR], xq[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int64_t i = static_cast<int64_t>(j) * W + L;
    if (i < P.m) {
      xp[j] = gp[i];
      xq[j] = gq[i];
    } else {
      xp[j] = Elem<CPLX>::zero();
      xq[j] = Elem<CPLX>::zero();
    }
  }
  if constexpr (NS > 0) cp_async_wait_all();  // each thread reads only its own slots
  if (sn != 0) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      xp[j] = scalbn_el(xp[j], sn);
      xq[j] = scalbn_el(xq[j], sn);
    }
#pragma unroll 2
    for (int j = 0; j < NS; ++j) {
      sP(j) = scalbn_el(sP(j), sn);
      sQ(j) = scalbn_el(sQ(j), sn);
    }
  }

  // ---- the norms (spade) and the dot (club) of the pair, two ways with the
  // same bits.  Fast (DESIGN.md 4.6 applied to the step): every component
  // scaled by one 2^-c (c: floor(lg M-tilde) in the driver, F(m) - 1 for the
  // public step), the sums of squares and the dot accumulated in ONE pass and
  // reduced in one round of two pairs; valid while every nonzero value is in
  // [2^(c-400), 2^(c+16)) (checked per lane on the unscaled values; a failing
  // lane turns its SSQ into NaN, so the whole pair sees it and takes the
  // exact path).  Exact: the
  // per-column exponent max, then the SSQ of x 2^-E, then the prescaled dot
  // (three rounds).
  double ep = -INFINITY, fp = 1.0, eq = -INFINITY, fq = 1.0, zr = 0.0, zi = 0.0;
  bool zero_col = false, fastp = false;
  // @phase spade+club:fast
  if (P.fast) {
    const int c = P.Mt ? ilogb_bits(mt_cur) + sn : P.Fm - 1;
    if (c >= 600 && c <= 1022) {  // cluster-uniform (2^-c normal)
      const double a = pow2i(-c);
      double sp = 0.0, sq = 0.0, ar = 0.0, ai = 0.0;
      // the domain check on the UNscaled values (a scaled value could have
      // underflowed): nonzero |x| in [2^(c-400), 2^(c+16))
      uint32_t lmin = ~0u, lmax = 0;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const E yp = scale1(xp[j], a), yq = scale1(xq[j], a);
        sp = ssq_acc(yp, sp);
        sq = ssq_acc(yq, sq);
        dot_acc(yq, yp, ar, ai);
        lmin = lo_hi_min(xp[j], lo_hi_min(xq[j], lmin));
        lmax = hi_max(xp[j], hi_max(xq[j], lmax));
      }
#pragma unroll 2
      for (int j = 0; j < NS; ++j) {
        const E xpj = sP(j), xqj = sQ(j);
        const E yp = scale1(xpj, a), yq = scale1(xqj, a);
        sp = ssq_acc(yp, sp);
        sq = ssq_acc(yq, sq);
        dot_acc(yq, yp, ar, ai);
        lmin = lo_hi_min(xpj, lo_hi_min(xqj, lmin));
        lmax = hi_max(xpj, hi_max(xqj, lmax));
      }
      const uint32_t lo = static_cast<uint32_t>(c - 400 + 1023) << 20;
      const uint32_t hi = static_cast<uint32_t>(min(c + 16 + 1023, 2047)) << 20;
      if (lmin < lo - 1u || lmax >= hi) sp = __longlong_as_double(0x7ff8000000000000ll);
      if constexpr (CL > 1) {
        tree_sum2_tx<T, CL>(sp, sq, rs_f1, tx_f1);
        tree_sum2_tx<T, CL>(ar, ai, rs_f2, tx_f2);
      } else {
        tree_sum2<T, 1>(sp, sq, rs_f1);
        tree_sum2<T, 1>(ar, ai, rs_f2);
      }
      if (!isnan(sp)) {  // uniform: every lane holds the totals
        fastp = true;
        // R#14 with E := c (the SSQ of x 2^-c carries 2^(2E - 2c) exactly)
        int iep = kIntMin, ieq = kIntMin;
        double gp = 1.0, gq = 1.0;
        if (sp > 0.0) {
          eg_from_ssq_c(c, sp, iep, gp);
          ep = static_cast<double>(iep);
          fp = sqrt_plain(gp);
        }
        if (sq > 0.0) {
          eg_from_ssq_c(c, sq, ieq, gq);
          eq = static_cast<double>(ieq);
          fq = sqrt_plain(gq);
        }
        zero_col = !(sp > 0.0) || !(sq > 0.0);  // R#19
        if (!zero_col) {  // the dot of x 2^-c carries 2^(2c - e_q - e_p) exactly
          const double f2 = pow2i(2 * c - iep - ieq);
          const Rcp d = rcp_plain(fq * fp);  // fl(f_q f_p) in [1, 4)
          zr = dot_div(ar * f2, d, kFull);
          zi = CPLX ? dot_div(ai * f2, d, kFull) : 0.0;
        }
        if (lead) {
          P.col_e[p] = ep;
          P.col_f[p] = fp;
          P.col_e[q] = eq;
          P.col_f[q] = fq;
        }
      }
    }
  }
  if (!fastp) {
    // @phase spade:norms
    // ---- spade: E = floor(lg max |component|) per column (high words)
    uint32_t hp = 0, hq = 0;
  #pragma unroll
    for (int j = 0; j < NR; ++j) {
      hp = hi_max(xp[j], hp);
      hq = hi_max(xq[j], hq);
    }
  #pragma unroll 2
    for (int j = 0; j < NS; ++j) {
      hp = hi_max(sP(j), hp);
      hq = hi_max(sQ(j), hq);
    }
    int Ep, Eq;
    if (hp >= 0x00100000u) {
      Ep = static_cast<int>(hp >> 20) - 1023;
    } else {  // largest component subnormal or zero: exact from the bit patterns
      uint64_t mb = 0;
  #pragma unroll
      for (int j = 0; j < NR; ++j) mb = absmax_bits(xp[j], mb);
  #pragma unroll 2
      for (int j = 0; j < NS; ++j) mb = absmax_bits(sP(j), mb);
      Ep = ilogb_or_min(mb);
    }
    if (hq >= 0x00100000u) {
      Eq = static_cast<int>(hq >> 20) - 1023;
    } else {
      uint64_t mb = 0;
  #pragma unroll
      for (int j = 0; j < NR; ++j) mb = absmax_bits(xq[j], mb);
  #pragma unroll 2
      for (int j = 0; j < NS; ++j) mb = absmax_bits(sQ(j), mb);
      Eq = ilogb_or_min(mb);
    }
    if constexpr (CL > 1) tree_max2i_tx<T, CL>(Ep, Eq, rs_e, tx_e);
    else tree_max2i<T, 1>(Ep, Eq, rs_e);
    // ---- spade: SSQ of x 2^-E in the lane order of R (E is CTA-uniform; the
    // two-multiply case 2^-E < 2^-1074 is a uniform branch).  Zero padding adds
    // exact zeros to a non-negative sum.
    double sp = 0.0, sq = 0.0;
    if (Ep != kIntMin) {
      if (-Ep > 1023) {
        const double a = 0x1p1023, b = pow2i(-Ep - 1023);
  #pragma unroll
        for (int j = 0; j < NR; ++j) sp = ssq_acc(scale2(xp[j], a, b), sp);
  #pragma unroll 2
        for (int j = 0; j < NS; ++j) sp = ssq_acc(scale2(sP(j), a, b), sp);
      } else {
        // 2^-E normal (the step's precondition keeps max|x| < 2^1022): exponent
        // field only; a subnormal 2^-E (outside it) the general construction
        const double a = -Ep >= -1022 ? pow2i(-Ep) : pow2_any(-Ep);
  #pragma unroll
        for (int j = 0; j < NR; ++j) sp = ssq_acc(scale1(xp[j], a), sp);
  #pragma unroll 2
        for (int j = 0; j < NS; ++j) sp = ssq_acc(scale1(sP(j), a), sp);
      }
    }
    if (Eq != kIntMin) {
      if (-Eq > 1023) {
        const double a = 0x1p1023, b = pow2i(-Eq - 1023);
  #pragma unroll
        for (int j = 0; j < NR; ++j) sq = ssq_acc(scale2(xq[j], a, b), sq);
  #pragma unroll 2
        for (int j = 0; j < NS; ++j) sq = ssq_acc(scale2(sQ(j), a, b), sq);
      } else {
        // 2^-E normal (the step's precondition keeps max|x| < 2^1022): exponent
        // field only; a subnormal 2^-E (outside it) the general construction
        const double a = -Eq >= -1022 ? pow2i(-Eq) : pow2_any(-Eq);
  #pragma unroll
        for (int j = 0; j < NR; ++j) sq = ssq_acc(scale1(xq[j], a), sq);
  #pragma unroll 2
        for (int j = 0; j < NS; ++j) sq = ssq_acc(scale1(sQ(j), a), sq);
      }
    }
    if constexpr (CL > 1) tree_sum2_tx<T, CL>(sp, sq, rs_ssq, tx_ssq);
    else tree_sum2<T, 1>(sp, sq, rs_ssq);
    if (Ep != kIntMin) ef_from_ssq(Ep, sp, ep, fp);
    if (Eq != kIntMin) ef_from_ssq(Eq, sq, eq, fq);
    if (lead) {
      P.col_e[p] = ep;
      P.col_f[p] = fp;
      P.col_e[q] = eq;
      P.col_f[q] = fq;
    }

    // @phase club:dot
    // ---- club: a21' = (g_q 2^-e_q)^* (g_p 2^-e_p) / fl(f_q f_p)  (Alg 3.1)
    zero_col = (Ep == kIntMin) || (Eq == kIntMin);  // R#19 (cluster-uniform)
    if (!zero_col) {
      const int iq = static_cast<int>(eq), ip = static_cast<int>(ep);
      double ar = 0.0, ai = 0.0;
      if (-iq > 1023 || -ip > 1023) {
        const Pow2 fQ(-iq), fP(-ip);
  #pragma unroll
        for (int j = 0; j < NR; ++j)
          dot_acc(scale2(xq[j], fQ.a, fQ.b), scale2(xp[j], fP.a, fP.b), ar, ai);
  #pragma unroll 2
        for (int j = 0; j < NS; ++j)
          dot_acc(scale2(sQ(j), fQ.a, fQ.b), scale2(sP(j), fP.a, fP.b), ar, ai);
      } else {
        const double aq = pow2_any(-iq), ap = pow2_any(-ip);
  #pragma unroll
        for (int j = 0; j < NR; ++j) dot_acc(scale1(xq[j], aq), scale1(xp[j], ap), ar, ai);
  #pragma unroll 2
        for (int j = 0; j < NS; ++j) dot_acc(scale1(sQ(j), aq), scale1(sP(j), ap), ar, ai);
      }
      if constexpr (CL > 1) tree_sum2_tx<T, CL>(ar, ai, rs_dot, tx_dot);
      else tree_sum2<T, 1>(ar, ai, rs_dot);
      const Rcp d = rcp_plain(fq * fp);  // fl(f_q f_p) in [1, 4)
      zr = dot_div(ar, d, kFull);
      zi = CPLX ? dot_div(ai, d, kFull) : 0.0;
    }
  }
  // the last cross-CTA round is done: arrive now, wait at exit (no CTA leaves
  // while a peer's push into its shared memory could still be in flight)
  if constexpr (CL > 1) {
    if (fastp || !zero_col) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  }
  // @phase heart:test+V-prefetch
  // ---- heart: transform iff upsilon <= |a21'| (Alg 3.2)
  const double az = CPLX ? hypot_naive(fabs(zr), fabs(zi)) : fabs(zr);
  const bool transform = P.tol <= az;

  // V columns of a transformed pair: the first NV rows per lane are loaded
  // now, so their latency overlaps the Grammian + EVD of warp 0 (real single
  // CTAs: 4 rows -- all of configs[2]'s V with W = 256 lanes)
  constexpr int NV = (!CPLX && CL == 1 && NS == 0) ? (JSVD_STEP_NV_REAL)
                     : (CPLX && NS > 0) ? (JSVD_STEP_NV_CPLX) : 2;
  E va[NV], vb[NV];
  E* vp = reinterpret_cast<E*>(P.V) + static_cast<int64_t>(p) * P.ldv;
  E* vq = reinterpret_cast<E*>(P.V) + static_cast<int64_t>(q) * P.ldv;
  if (transform && P.V) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int64_t i = static_cast<int64_t>(j) * W + L;
      if (i < P.n) {
        va[j] = vp[i];
        vb[j] = vq[i];
      }
    }
  }

  // @phase heart+diamond:Gram+EVD
  if (transform) {
    if (threadIdx.x < 32) {  // heart + diamond, computed by one warp per CTA
      double b11, b22, br, bi;
      gram_fast(zr, zi, ep, fp, eq, fq, b11, b22, br, bi, kFull);
      const Evd2Out o = evd2<CPLX, true, true, false>(b11, b22, br, bi, kFull);  // warp 0, all lanes
      if (threadIdx.x == 0) {
        rot[0] = o.c;
        rot[1] = o.sr;
        rot[2] = o.si;
      }
    }
    __syncthreads();
    const double c = rot[0], C = rot[1], S = rot[2];
    // @phase star:rotate-G
    // ---- star: rotate the pair (registers; shared rows back in place)
#pragma unroll
    for (int j = 0; j < NR; ++j) rot_elem(xp[j], xq[j], c, C, S);
#pragma unroll 2
    for (int j = 0; j < NS; ++j) {
      E a = sP(j), b = sQ(j);
      rot_elem(a, b, c, C, S);
      sP(j) = a;
      sQ(j) = b;
    }
  }
  if (transform || sn != 0) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int64_t i = static_cast<int64_t>(j) * W + L;
      if (i < P.m) {
        gp[i] = xp[j];
        gq[i] = xq[j];
      }
    }
#pragma unroll 2
    for (int j = 0; j < NS; ++j) {
      const int64_t i = static_cast<int64_t>(NR + j) * W + L;
      if (i < P.m) {
        gp[i] = sP(j);
        gq[i] = sQ(j);
      }
    }
  }
  // @phase star:rotate-V
  if (transform) {
    if (P.V) {
      const double c = rot[0], C = rot[1], S = rot[2];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int64_t i = static_cast<int64_t>(j) * W + L;
        if (i < P.n) {
          rot_elem(va[j], vb[j], c, C, S);
          vp[i] = va[j];
          vq[i] = vb[j];
        }
      }
      for (int64_t i = NV * W + L; i < P.n; i += W) {
        E a = vp[i], b = vq[i];
        rot_elem(a, b, c, C, S);
        vp[i] = a;
        vq[i] = b;
      }
    }
    // @phase M+bookkeeping
    // ---- M: max |component| of the transformed pair.  In the driver
    // (Mt) only floor(lg M-tilde) >= K + 1 matters (Eq. skr): every component
    // is below sqrt(|g_p|^2 + |g_q|^2) <= 2^(max(e_p,e_q) + 1.5), so a pair
    // with max(e) <= K - 1 cannot reach 2^(K+1) and is not tracked; an
    // untracked M only lowers M-tilde while it stays below 2^(K+1), so every
    // check and every rescale is the same as with the exact M.  Otherwise the
    // exact max: high words first (one CTA reduction), then the low words of
    // the lanes holding the largest high word, straight to the atomic.
    const bool track = !P.Mt || fmax(ep, eq) > static_cast<double>(P.Kr - 1);
    if (track) {
      uint32_t hm = 0;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        hm = hi_max(xp[j], hm);
        hm = hi_max(xq[j], hm);
      }
#pragma unroll 2
      for (int j = 0; j < NS; ++j) {
        hm = hi_max(sP(j), hm);
        hm = hi_max(sQ(j), hm);
      }
      const uint32_t H = cta_max_u32<T>(hm, rs_m);
      if (hm == H && H != 0u) {
        uint32_t lmax = 0;
#pragma unroll
        for (int j = 0; j < NR; ++j) lmax = lo_max_at(xp[j], H, lo_max_at(xq[j], H, lmax));
#pragma unroll 2
        for (int j = 0; j < NS; ++j) lmax = lo_max_at(sP(j), H, lo_max_at(sQ(j), H, lmax));
        const unsigned long long Mx = (static_cast<unsigned long long>(H) << 32) | lmax;
        atomicMax(P.Mt ? &P.Mt[(P.slot + 1) % 3] : P.mmax, Mx);
      }
    }
    if (threadIdx.x == 0 && crank == 0) atomicAdd(P.t_dev, 1ull);
  }
  if (P.Mt && pair == 0 && lead) {  // M-tilde / s bookkeeping for the next step
    const double cur = __longlong_as_double(static_cast<long long>(mt_cur));
    const double scaled = sn ? scalbn_rn(cur, sn) : cur;
    atomicMax(&P.Mt[(P.slot + 1) % 3],
              static_cast<unsigned long long>(__double_as_longlong(scaled)));
    P.Mt[(P.slot + 2) % 3] = 0ull;
    P.s_slots[(P.slot + 1) % 3] = P.s_slots[P.slot] + sn;
  }
  if constexpr (CL > 1) {
    if (!fastp && zero_col) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
}

// @phase finalize
// ---- finalize helpers ---------------------------------------
// norms of all columns with the same code and lane order as the step (R#23)
template <bool CPLX, int T, int CL, int NR>
__global__ void __launch_bounds__(T) colnorm_kernel(int64_t m, const double* G, int64_t ldg,
                                                    double* col_e, double* col_f) {
  using E = typename Elem<CPLX>::T;
  constexpr int W = T * CL;
  constexpr int NW = T / 32;
  __shared__ RedSlot<NW, int> rs_e;
  __shared__ RedSlot<NW, double> rs_ssq;
  const int crank = CL > 1 ? static_cast<int>(blockIdx.x % CL) : 0;
  const int64_t col = blockIdx.x / CL;
  const int L = crank * T + static_cast<int>(threadIdx.x);
  const E* g = reinterpret_cast<const E*>(G) + col * ldg;
  E x[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int64_t i = static_cast<int64_t>(j) * W + L;
    x[j] = i < m ? g[i] : Elem<CPLX>::zero();
  }
  uint64_t mx = 0;
#pragma unroll
  for (int j = 0; j < NR; ++j) mx = absmax_bits(x[j], mx);
  int Ex = ilogb_or_min(mx), dummy = kIntMin;
  tree_max2i<T, CL>(Ex, dummy, rs_e);
  double s = 0.0, s2 = 0.0;
  if (Ex != kIntMin) {
    const Pow2 f(-Ex);
#pragma unroll
    for (int j = 0; j < NR; ++j)
      if (static_cast<int64_t>(j) * W + L < m) s = ssq_acc(f(x[j]), s);
  }
  tree_sum2<T, CL>(s, s2, rs_ssq);
  double e = -INFINITY, f = 1.0;
  if (Ex != kIntMin) ef_from_ssq(Ex, s, e, f);
  if (crank == 0 && threadIdx.x == 0) {
    col_e[col] = e;
    col_f[col] = f;
  }
  if constexpr (CL > 1) cg::this_cluster().sync();
}

// ---- geometry --------------------------------------------------------------
struct Geo {
  int T, CL, NR, NS;
};

// W = 256 * CL lanes (CL = 1 ... 16 CTAs of 256 threads), the smallest W with
// W * NR >= m (NR register rows per lane and column).  256-thread CTAs at
// <= 128 registers leave room for two CTAs (of different pairs) per SM, so
// one pair's loads overlap another's reductions and EVD.  Columns that would
// need W > 2048 hold 2 NR rows per lane instead, NR/2 in registers and 3NR/2
// in shared memory (96 KB per CTA): W halves, a pair needs half the CTAs,
// twice as many pairs are in flight.  CL = 16 is a non-portable cluster size (opted in at launch).
static Geo pick_geo(bool cplx, int64_t m) {
  const int NR = cplx ? 8 : 16;
  int64_t need = (m + NR - 1) / NR, W = 256;
  while (W < need) W *= 2;
  int NS = 0;
  if (W > 2048) {
    NS = NR;
    need = (m + 2 * NR - 1) / (2 * NR);
    W = 256;
    while (W < need) W *= 2;
  }
  if (W > 4096) return Geo{0, 0, 0, 0};
  return Geo{256, static_cast<int>(W / 256), NR, NS};
}

// kernel attributes (cluster size > 8, > 48 KB dynamic shared memory) are
// per device: remember (kernel, device) pairs already configured
static std::mutex g_attr_mu;
static std::vector<std::pair<const void*, int>> g_attr_done;
static bool attrs_done(const void* k, int dev) {
  std::lock_guard<std::mutex> g(g_attr_mu);
  for (const auto& p : g_attr_done)
    if (p.first == k && p.second == dev) return true;
  return false;
}
static void mark_attrs_done(const void* k, int dev) {
  std::lock_guard<std::mutex> g(g_attr_mu);
  g_attr_done.emplace_back(k, dev);
}

template <typename Kern, typename... Args>
static cudaError_t launch_cl(Kern k, int64_t grid, int T, int CL, size_t smem, cudaStream_t st,
                             bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CL > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CL;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  // kernel attributes are set once per (kernel, device) (not inside a CUDA-graph
  // capture of later launches)
  int dev = 0;
  if (CL > 8 || smem > 48 * 1024) {
    cudaError_t a = cudaGetDevice(&dev);
    if (a != cudaSuccess) return a;
  }
  if ((CL > 8 || smem > 48 * 1024) && !attrs_done(reinterpret_cast<const void*>(k), dev)) {
    if (CL > 8) {
      cudaError_t a = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (a != cudaSuccess) return a;
    }
    if (smem > 48 * 1024) {
      cudaError_t a = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (a != cudaSuccess) return a;
    }
    mark_attrs_done(reinterpret_cast<const void*>(k), dev);
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, args...);
  note_launch();
  return e;
}

// L2 prefetch distance of the long-column step (shared-memory rows: G far
// beyond L2): a quarter of the resident pairs (2 CTAs per SM, CL per pair).
// Measured, configs[4] step: 2.145 ms without, 2.07 at 4 or 9 pairs ahead,
// 2.09 at 13, 2.20 at 24, 2.35 at a full wave (37).  JSVD_STEP_PF overrides
// (0: off).
static int step_prefetch_distance(int CL) {
  const char* e = getenv("JSVD_STEP_PF");
  if (e) return atoi(e);
  const int sms = sm_count();
  return sms ? max(1, sms / (2 * CL)) : 0;
}

template <bool CPLX>
static cudaError_t launch_step_t(const Geo& g, int64_t npairs, const StepParams& P0,
                                 cudaStream_t st) {
  StepParams P = P0;
  P.pf = g.NS ? step_prefetch_distance(g.CL) : 0;
  {  // V too (2.065 -> 2.003 ms per configs[4] step when every pair
     // transforms; a pair that then does not transform wastes its V bytes)
    const char* e = getenv("JSVD_STEP_PFV");
    P.pfv = P.pf > 0 && (e ? atoi(e) : 1);
  }
  constexpr int NR = CPLX ? 8 : 16;
  using E = typename Elem<CPLX>::T;
  const int64_t grid = npairs * g.CL;
  // shared-row geometry: NR/2 rows in registers, 3NR/2 in shared memory
  // (96 KB per CTA, two CTAs per SM) -- 2 NR rows per lane in all
  constexpr int NRr = NR / 2, NSs = 3 * NR / 2;
  const size_t sm = static_cast<size_t>(NSs) * 2 * 256 * sizeof(E);
  if (g.NS) {
    switch (g.CL) {
      case 8: return launch_cl(step_kernel<CPLX, 256, 8, NRr, NSs>, grid, 256, 8, sm, st, true, P);
      case 16: return launch_cl(step_kernel<CPLX, 256, 16, NRr, NSs>, grid, 256, 16, sm, st, true, P);
    }
    return cudaErrorInvalidValue;
  }
  switch (g.CL) {
    case 1: return launch_cl(step_kernel<CPLX, 256, 1, NR, 0>, grid, 256, 1, 0, st, true, P);
    case 2: return launch_cl(step_kernel<CPLX, 256, 2, NR, 0>, grid, 256, 2, 0, st, true, P);
    case 4: return launch_cl(step_kernel<CPLX, 256, 4, NR, 0>, grid, 256, 4, 0, st, true, P);
    case 8: return launch_cl(step_kernel<CPLX, 256, 8, NR, 0>, grid, 256, 8, 0, st, true, P);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_step(bool cplx, int64_t npairs, const StepParams& P, cudaStream_t st) {
  const Geo g = pick_geo(cplx, P.m);
  return cplx ? launch_step_t<true>(g, npairs, P, st) : launch_step_t<false>(g, npairs, P, st);
}

// the finalize norms: one column per CTA / cluster, NR + NS rows per lane in
// registers -- the same W and lane order as the step (R#23)
template <bool CPLX>
static cudaError_t launch_colnorm_t(const Geo& g, int64_t m, int64_t n, const double* G,
                                    int64_t ldg, double* ce, double* cf, cudaStream_t st) {
  constexpr int NR = CPLX ? 8 : 16;
  const int64_t grid = n * g.CL;
  if (g.NS) {
    switch (g.CL) {
      case 8: return launch_cl(colnorm_kernel<CPLX, 256, 8, 2 * NR>, grid, 256, 8, 0, st, false, m, G, ldg, ce, cf);
      case 16: return launch_cl(colnorm_kernel<CPLX, 256, 16, 2 * NR>, grid, 256, 16, 0, st, false, m, G, ldg, ce, cf);
    }
    return cudaErrorInvalidValue;
  }
  switch (g.CL) {
    case 1: return launch_cl(colnorm_kernel<CPLX, 256, 1, NR>, grid, 256, 1, 0, st, false, m, G, ldg, ce, cf);
    case 2: return launch_cl(colnorm_kernel<CPLX, 256, 2, NR>, grid, 256, 2, 0, st, false, m, G, ldg, ce, cf);
    case 4: return launch_cl(colnorm_kernel<CPLX, 256, 4, NR>, grid, 256, 4, 0, st, false, m, G, ldg, ce, cf);
    case 8: return launch_cl(colnorm_kernel<CPLX, 256, 8, NR>, grid, 256, 8, 0, st, false, m, G, ldg, ce, cf);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_colnorm(bool cplx, int64_t m, int64_t n, const double* G, int64_t ldg,
                           double* ce, double* cf, cudaStream_t st) {
  const Geo g = pick_geo(cplx, m);
  return cplx ? launch_colnorm_t<true>(g, m, n, G, ldg, ce, cf, st)
              : launch_colnorm_t<false>(g, m, n, G, ldg, ce, cf, st);
}

bool step_supported(bool cplx, int64_t m) { return pick_geo(cplx, m).T != 0; }

// JSVD_STEP_FAST=0: the step kernel's exact norms + dot only (A/B runs; the
// same bits either way -- the GPU tests compare both)
bool step_fast_enabled() {
  const char* e = getenv("JSVD_STEP_FAST");
  return !e || atoi(e) != 0;
}

// floor(lg(omega/(2m))) (real) / floor(lg(omega/(4 m sqrt2))) (complex) (R#28):
// the public step's scale 2^(F(m)-1) bounds a matrix pre-scaled as jsvd_gesvj does
static int Fm_step(bool cplx, int64_t m) {
  int k = 0;
  while ((m >> (k + 1)) > 0) ++k;
  if (!cplx) return 1022 - k;
  const unsigned __int128 mm = static_cast<unsigned __int128>(m) * static_cast<unsigned __int128>(m);
  return 1021 - k - (mm >= (static_cast<unsigned __int128>(1) << (2 * k + 1)) ? 1 : 0);
}

__global__ void strategy_kernel(int64_t n, int64_t B, int64_t step, int32_t* pairs) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l < n / 2) {
    int p, q;
    strategy_pair(n, B, step, l, p, q);
    pairs[2 * l] = p;
    pairs[2 * l + 1] = q;
  }
}

bool strategy_ok(int64_t n, int64_t B) {
  if (n < 2 || (n & 1) || B < 2 || n % B) return false;
  const int64_t b = n / B;
  return b == 1 || (b % 2) == 0;
}

}  // namespace jsvd

using namespace jsvd;

extern "C" jsvd_status jsvd_step_rspec(jsvd_dtype dt, int64_t m, int32_t* W, int32_t* c,
                                       int32_t* offs, int32_t* noffs) {
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < 1 || !W || !c || !offs || !noffs)
    return JSVD_EINVAL;
  const Geo g = pick_geo(dt == JSVD_C64, m);
  if (!g.T) return JSVD_EINVAL;
  *W = g.T * g.CL;
  *c = 1;
  int k = 0;
  for (int o = 16; o >= 1; o /= 2) offs[k++] = o;
  for (int o = g.T / 2; o >= 32; o /= 2) offs[k++] = o;
  for (int o = g.T * g.CL / 2; o >= g.T; o /= 2) offs[k++] = o;
  *noffs = k;
  return JSVD_OK;
}

extern "C" jsvd_status jsvd_strategy_pairs(int64_t n, int32_t nblocks, int64_t step,
                                           int32_t* pairs, void* stream) {
  if (!strategy_ok(n, nblocks) || step < 0 || step >= n - 1 || !pairs) return JSVD_EINVAL;
  const int64_t np = n / 2;
  strategy_kernel<<<static_cast<unsigned>((np + 255) / 256), 256, 0,
                    static_cast<cudaStream_t>(stream)>>>(n, nblocks, step, pairs);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}

static double upsilon_host(int64_t m) { return std::ldexp(std::sqrt(static_cast<double>(m)), -53); }

extern "C" jsvd_status jsvd_sweep_step(jsvd_dtype dt, int64_t m, int64_t n, double* G, int64_t ldg,
                                       double* V, int64_t ldv, const int32_t* pairs,
                                       int64_t npairs, double tol, double* col_e, double* col_f,
                                       int64_t* t_dev, double* mmax_dev, void* stream) {
  const bool cplx = dt == JSVD_C64;
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < 1 || n < 2 || ldg < m || !G || !pairs ||
      npairs < 0 || npairs > n / 2 || !col_e || !col_f || !t_dev || !mmax_dev)
    return JSVD_EINVAL;
  if (V && ldv < n) return JSVD_EINVAL;
  if (!step_supported(cplx, m)) return JSVD_EINVAL;
  if (cplx && ((reinterpret_cast<uintptr_t>(G) & 15) || (V && (reinterpret_cast<uintptr_t>(V) & 15))))
    return JSVD_EINVAL;
  if (npairs == 0) return JSVD_OK;
  StepParams P{};
  P.m = m;
  P.n = n;
  P.G = G;
  P.ldg = ldg;
  P.V = V;
  P.ldv = ldv;
  P.pairs = pairs;
  P.tol = tol > 0.0 ? tol : upsilon_host(m);
  P.col_e = col_e;
  P.col_f = col_f;
  P.t_dev = reinterpret_cast<unsigned long long*>(t_dev);
  P.mmax = reinterpret_cast<unsigned long long*>(mmax_dev);
  P.fast = step_fast_enabled() ? 1 : 0;
  P.Fm = Fm_step(cplx, m);
  cudaError_t e = launch_step(cplx, npairs, P, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}
