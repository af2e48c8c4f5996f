// batched_fast.cu -- jsvd_gesvj_batched's kernel for BASELINE configs[3]'s
// shape (m = 64, n <= 32) in the scaled domain of DESIGN.md 4.6: one matrix
// per CTA of 128 threads (16 lane groups of 8), G~ = G 2^-cs in shared memory
// (32 KB), the working V in the V output (L2-resident), six CTAs per SM.
//
// Arithmetic: Alg 4.1 exactly as batched.cu's kernel (flat round-robin, the
// reduction spec R = (8, 1, [4, 2, 1]), the Eq. (skr) check at every step,
// line 41), computed on G~: while every value of G~ is 0 or in [2^-400,
// 2^(1024-cs)] and every transformed pair's C, S is 0 or at least 2^-400, the
// norms' sums of squares, the dots and the rotations of G~ are exact
// power-of-two multiples of the oracle's, so the scaling multiplies of R#14 /
// Alg 3.1 and the exponent reductions are not needed.  A matrix that leaves
// that domain (checked at its load, on every transformed pair's C, S in
// phase B, on every rotated value in phase C) is handed over: its A is still
// intact (V lives in the V output, G only in shared memory), a NaN marker
// goes into sigma, and batched.cu's kernel runs it from the start in G's
// own scale.
//
// Per step:
//   A  lane group g, pair g: the SSQ of both columns and the dot of the raw
//      G~ values (8 rows per lane, four independent accumulations)
//   B  warp 0, lane l, pair l: (e, f) of the norms, the dot's rescale and
//      division, the convergence test (Alg 3.2), Grammian (Alg 3.3), 2x2 EVD
//      (Alg 2.2) | warps 1-3: the V rotations of the previous step
//   C  lane group g: the rotation of G~'s pair (Alg 3.4) and the domain check
#include <cmath>

#include "jsvd_host.h"
#include "step_dev.cuh"

namespace jsvd {

namespace bf {

constexpr int kT = 128, kW = 8, kNR = 8, kM = 64, kG = 16;
// sigma[b n] of a matrix handed to batched.cu's kernel (a NaN payload)
constexpr unsigned long long kMarker = 0x7ff8badc0ffee123ull;

struct Pair {
  double ar, ai, sp, sq;  // A: raw sums of G~ (dot, SSQ of p and q)
  double c, C, S;         // B: rotation
  int ep, eq;             // B: norm exponents (kIntMin: zero column)
  int transform, pad;
};


template <int W>
__device__ __forceinline__ double hsum(double v) {
#pragma unroll
  for (int o = W / 2; o >= 1; o /= 2) v = v + __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// e = E + k/2, g = SSQ 2^-k (k even) from a sum of squares (R#14), E the
// scale exponent the squared values carry
__device__ __forceinline__ void eg_of(int E, double ssq, int& e, double& g) {
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(ssq));
  int k = static_cast<int>(bits >> 52) - 1023;
  g = __longlong_as_double(static_cast<long long>((bits & 0x000fffffffffffffull) |
                                                  0x3ff0000000000000ull));
  if (k & 1) {
    g = g * 2.0;
    k -= 1;
  }
  e = E + k / 2;
}

}  // namespace bf

using namespace bf;

template <bool CPLX, bool PROF>
__global__ void __launch_bounds__(kT, 6) batched_fast_kernel(
    int n, double* A, int64_t lda, int64_t strideA, double* Vg, int64_t ldv, int64_t strideV,
    double* sigma, int max_sweeps, int32_t* sweeps_out, int32_t* status_out,
    int64_t* transforms_out, int32_t* scale_out, int Fm, int Kr, double tol, int s0_adjust,
    unsigned long long* prof) {
  using E = typename Elem<CPLX>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int np = n / 2;
  E* sG = reinterpret_cast<E*>(smem_raw);                         // 64 x n
  Pair* sP = reinterpret_cast<Pair*>(sG + kM * n);                // [2 buf][16]
  double* ce = reinterpret_cast<double*>(sP + 2 * kG);             // [32] line 41
  double* cf = ce + 32;                                            // [32]
  uint8_t* sPairs = reinterpret_cast<uint8_t*>(cf + 32);          // (n-1) x np pivot pairs
  __shared__ uint64_t wred[kT / 32];
  __shared__ int sSel[32];
  __shared__ int sT, sBad;
  __shared__ uint32_t sMt;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hl = threadIdx.x & (kW - 1), g = threadIdx.x / kW;  // lane in group, group
  const int64_t b = blockIdx.x;
  const E* Ag = reinterpret_cast<const E*>(A) + b * strideA;
  E* Vb = reinterpret_cast<E*>(Vg) + b * strideV;  // the working V: the V output

  unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = 0;
  const auto mark = [&](int k) {
    if constexpr (PROF) {
      const long long t = clock64();
      pc[k] += static_cast<unsigned long long>(t - tprev);
      tprev = t;
    }
  };
  if constexpr (PROF) tprev = clock64();

  for (int k = threadIdx.x; k < (n - 1) * np; k += kT) {
    int p, q;
    strategy_pair(n, n, k / np, k % np, p, q);
    sPairs[2 * k] = static_cast<uint8_t>(p);
    sPairs[2 * k + 1] = static_cast<uint8_t>(q);
  }

  // @phase load
  // ---- load A; M0 = max |component| (NaN -> inf), mn = the smallest nonzero
  uint64_t mx = 0, mn = ~0ull;
  {
    constexpr int kPer = 8;  // elements per thread and round (loads issued together)
    for (int k0 = 0; k0 < kM * n; k0 += kT * kPer) {
      E x[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int k = k0 + u * kT + threadIdx.x;
        const int kc = k < kM * n ? k : 0;
        const int j = kc / kM, i = kc - j * kM;
        x[u] = Ag[static_cast<int64_t>(j) * lda + i];
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int k = k0 + u * kT + threadIdx.x;
        if (k < kM * n) {
          sG[k] = x[u];
          if constexpr (CPLX) {
            mx = max(mx, abs_bits(fmin(fabs(x[u].x), static_cast<double>(INFINITY))));
            mx = max(mx, abs_bits(fmin(fabs(x[u].y), static_cast<double>(INFINITY))));
            mn = min(mn, min(abs_bits(x[u].x) - 1, abs_bits(x[u].y) - 1));
          } else {
            mx = max(mx, abs_bits(fmin(fabs(x[u]), static_cast<double>(INFINITY))));
            mn = min(mn, abs_bits(x[u]) - 1);
          }
        }
      }
    }
  }
  const uint64_t M0b = cta_max_u64<kT>(mx, wred);
  __syncthreads();
  const uint64_t mnb = ~cta_max_u64<kT>(~mn, wred);
  const double M0 = __longlong_as_double(static_cast<long long>(M0b));
  if (isinf(M0) || M0 == 0.0) {  // the matrix is left as it was
    if (threadIdx.x == 0) {
      if (status_out) status_out[b] = isinf(M0) ? JSVD_ENONFINITE : JSVD_ERANK;
      if (sweeps_out) sweeps_out[b] = 0;
      if (transforms_out) transforms_out[b] = 0;
      if (scale_out) scale_out[b] = 0;
    }
    return;
  }
  const int lm0 = ilogb_bits(M0b);
  int s = Fm - lm0 - 1 + s0_adjust;  // Eq. (skn) (+ s0_adjust, R#40)
  int cs = lm0 + s;                  // floor(lg M-tilde_1): G~ = A 2^-lm0
  if (!((mnb == ~0ull || ilogb_bits(mnb + 1) >= lm0 - 400) && cs >= 600)) {
    // outside the fast domain from the start: batched.cu's kernel
    if (threadIdx.x == 0) reinterpret_cast<unsigned long long*>(sigma)[b * n] = kMarker;
    return;
  }
  {
    const double sc = pow2i(-lm0 >= -1022 ? -lm0 : -1022);
    const double sc2 = -lm0 >= -1022 ? 1.0 : pow2i(-lm0 + 1022);
    for (int k = threadIdx.x; k < kM * n; k += kT) {
      if constexpr (CPLX) sG[k] = make_double2((sG[k].x * sc) * sc2, (sG[k].y * sc) * sc2);
      else sG[k] = (sG[k] * sc) * sc2;
    }
    for (int k = threadIdx.x; k < n * n; k += kT) {  // V = I
      const int j = k / n, i = k - j * n;
      E v;
      if constexpr (CPLX) v = make_double2(i == j ? 1.0 : 0.0, 0.0);
      else v = i == j ? 1.0 : 0.0;
      Vb[static_cast<int64_t>(j) * ldv + i] = v;
    }
  }
  if (threadIdx.x == 0) {
    sMt = hi32(scalbn_rn(M0, s));
    sT = 0;
    sBad = 0;
  }
  __syncthreads();

  // @phase star:V
  // V rotation of pair l of step kk (parameters in buffer buf), by the 8
  // lanes of the caller's group: 4 rows per lane, two at a time
  const auto rotate_v = [&](int kk, int buf, int l) {
    const Pair& pr = sP[buf * kG + l];
    if (!pr.transform) return;
    const int p = sPairs[2 * (kk * np + l)], q = sPairs[2 * (kk * np + l) + 1];
    E* vp = Vb + static_cast<int64_t>(p) * ldv;
    E* vq = Vb + static_cast<int64_t>(q) * ldv;
    const double c = pr.c, C = pr.C, S = pr.S;
#pragma unroll
    for (int h = 0; h < 4; h += 2) {
      E a[2], bq[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {  // (rows past n reread row hl; not stored)
        const int i = (h + r) * kW + hl < n ? (h + r) * kW + hl : hl;
        a[r] = vp[i];
        bq[r] = vq[i];
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int i = (h + r) * kW + hl;
        rot_elem(a[r], bq[r], c, C, S);
        if (i < n) {
          vp[i] = a[r];
          vq[i] = bq[r];
        }
      }
    }
  };
  mark(6);

  int k = 0, C = 0, pend = -1, pend_buf = 0, T0 = 0, fin = max_sweeps == 0 ? 2 : 0;
  for (int tick = 0; !fin; ++tick) {
    const int buf = tick & 1;
    // @phase rescale-check
    // line 6, the Eq. (skr) check (every step of the flat ordering): in G~'s
    // scale a rescale only moves cs
    {
      const uint32_t mt = sMt;
      const int lm = static_cast<int>(mt >> 20) - 1023;
      if (Kr - lm < 0) {  // uniform
        const int sn = Fm - lm - 1;
        cs += sn;
        s += sn;
        __syncthreads();  // every thread has read sMt
        if (threadIdx.x == 0) sMt = hi32(scalbn_rn(mkd(mt, 0u), sn));
      }
    }
    // @phase A:spade+club
    // ---- phase A (a group without a pair, n < 32, computes pair 0 and
    // stores nothing, so every lane takes part in the shuffles)
    {
      const int la = g < np ? g : 0;
      const int p = sPairs[2 * (k * np + la)], q = sPairs[2 * (k * np + la) + 1];
      const E* gp = sG + p * kM;
      const E* gq = sG + q * kM;
      double sp = 0.0, sq = 0.0, ar = 0.0, ai = 0.0;
#pragma unroll
      for (int r = 0; r < kNR; ++r) {
        const int i = r * kW + hl;
        const E xp = gp[i], xq = gq[i];
        sp = ssq_acc(xp, sp);
        sq = ssq_acc(xq, sq);
        dot_acc(xq, xp, ar, ai);
      }
      sp = hsum<kW>(sp);
      sq = hsum<kW>(sq);
      ar = hsum<kW>(ar);
      if (CPLX) ai = hsum<kW>(ai);
      if (hl == 0 && g < np) {
        Pair& P = sP[buf * kG + g];
        P.sp = sp;
        P.sq = sq;
        P.ar = ar;
        P.ai = ai;
      }
    }
    mark(0);
    __syncthreads();
    mark(1);
    // @phase B:heart+diamond
    // ---- phase B (warp 0, lane l: pair l) | V of the previous step (warps 1-3)
    if (warp == 0) {
      const int l = lane;
      const bool on = l < np;
      Pair& P = sP[buf * kG + (on ? l : 0)];
      const double spv = on ? P.sp : 1.0, sqv = on ? P.sq : 1.0;
      // R#14 with E := cs (the SSQ of G~ carries 2^(2E - 2cs) exactly)
      const bool zp = !(spv > 0.0), zq = !(sqv > 0.0);
      int iep = kIntMin, ieq = kIntMin;
      double gp = 1.0, gq = 1.0;
      if (!zp) eg_of(cs, spv, iep, gp);
      if (!zq) eg_of(cs, sqv, ieq, gq);
      // lanes without a pair divide a dummy 1 (a zero would send the whole
      // warp into dot_div's tiny-dividend branch at every step)
      double arv = on ? P.ar : 1.0, aiv = on ? P.ai : 1.0;
      if (!(zp || zq)) {  // the dot of G~ carries 2^(2cs - e_q - e_p) exactly
        const double f2 = pow2i(2 * cs - iep - ieq);
        arv *= f2;
        aiv *= f2;
      }
      const double fp = zp ? 1.0 : sqrt_plain(gp), fq = zq ? 1.0 : sqrt_plain(gq);
      const Rcp d = rcp_plain(fq * fp);  // Alg 3.1 line 8
      const double zr = dot_div(arv, d, kFull);
      const double zi = CPLX ? dot_div(aiv, d, kFull) : 0.0;
      const double az = CPLX ? hypot_naive(fabs(zr), fabs(zi)) : fabs(zr);
      const bool tr = on && !(zp || zq) && tol <= az;  // Alg 3.2
      bool bad = false;
      if (__any_sync(kFull, tr)) {
        double b11, b22, br, bi;
        const bool gf = gram_fast_i(tr ? zr : 0.0, tr ? zi : 0.0, tr ? iep : 0, tr ? fp : 1.0,
                                    tr ? ieq : 0, tr ? fq : 1.0, b11, b22, br, bi, kFull);
        // |a21| = the test's |z| (a non-transformed lane's zero Grammian: 0)
        const Evd2Out o = evd2<CPLX, true, true, false>(b11, b22, br, bi, kFull,
                                                        !gf ? -1.0 : tr ? az : 0.0);
        if (tr) {
          P.c = o.c;
          P.C = o.sr;
          P.S = o.si;
          bad = (abs_hi(o.sr) - 1u < kFastLo - 1u) || (abs_hi(o.si) - 1u < kFastLo - 1u);
        }
      }
      if (on) {
        P.transform = tr;
        P.ep = iep;
        P.eq = ieq;
      }
      const unsigned tb = __ballot_sync(kFull, tr), bb = __ballot_sync(kFull, bad);
      if (lane == 0) {
        sT += __popc(tb);
        if (bb) sBad = 1;
      }
    // @phase star:V
    } else if (pend >= 0) {  // groups 4..15: V of the previous step
      for (int l = g - 4; l < np; l += kG - 4) rotate_v(pend, buf ^ 1, l);
    }
    mark(2);
    __syncthreads();
    mark(3);
    // @phase C:star-G
    if (sBad) break;  // a C or S below 2^-400: hand the matrix over (uniform)
    // ---- phase C: the rotation of G~'s pair g (Alg 3.4), the domain check
    {
      uint32_t Mw = 0, lmin = ~0u;
      const Pair& P = sP[buf * kG + g];
      if (g < np && P.transform) {
        const int p = sPairs[2 * (k * np + g)], q = sPairs[2 * (k * np + g) + 1];
        E* gp = sG + p * kM;
        E* gq = sG + q * kM;
        const double c = P.c, Cc = P.C, S = P.S;
        // M-tilde: only pairs with max(e) > K - 1 can reach 2^(K+1) (see step.cu)
        const bool track = max(P.ep, P.eq) > Kr - 1;
        constexpr int kH = kNR / 2;  // half of the lane's rows at a time (registers)
#pragma unroll
        for (int h = 0; h < kNR / kH; ++h) {
          E a[kH], bq[kH];
#pragma unroll
          for (int r = 0; r < kH; ++r) {
            a[r] = gp[(h * kH + r) * kW + hl];
            bq[r] = gq[(h * kH + r) * kW + hl];
          }
#pragma unroll
          for (int r = 0; r < kH; ++r) {
            rot_elem(a[r], bq[r], c, Cc, S);
            gp[(h * kH + r) * kW + hl] = a[r];
            gq[(h * kH + r) * kW + hl] = bq[r];
            lmin = lo_hi_min(a[r], lo_hi_min(bq[r], lmin));
            if (track) Mw = hi_max(a[r], hi_max(bq[r], Mw));
          }
        }
      }
      Mw = __reduce_max_sync(0xffffffffu, Mw);  // G = G~ 2^cs (normal values)
      if (lane == 0 && Mw) atomicMax(&sMt, Mw + (static_cast<uint32_t>(cs) << 20));
      if (lmin < kFastLo - 1u) sBad = 1;
    }
    mark(4);
    __syncthreads();
    mark(5);
    if (sBad) break;  // a rotated value below 2^-400 (uniform)
    // @phase bookkeeping
    // ---- step / sweep counters (every thread), line 40
    pend = k;
    pend_buf = buf;
    if (++k == n - 1) {
      k = 0;
      ++C;
      const int tc = sT;
      if (tc == T0) fin = 1;
      else if (C == max_sweeps) fin = 2;
      T0 = tc;
    }
    mark(6);
  }
  if constexpr (PROF) {  // [6]: load, bookkeeping, line 41; [7]: the whole kernel
    pc[7] = pc[0] + pc[1] + pc[2] + pc[3] + pc[4] + pc[5] + pc[6];
    if (lane == 0)
      for (int q = 0; q < 8; ++q) atomicAdd(&prof[(warp == 0 ? 0 : 1) * 8 + q], pc[q]);
  }
  if (!fin) {  // left the fast domain: batched.cu's kernel redoes the matrix
    if (threadIdx.x == 0) reinterpret_cast<unsigned long long*>(sigma)[b * n] = kMarker;
    return;
  }
  // @phase line41
  if (pend >= 0) {  // the last step's V rotation
    if (g < np) rotate_v(pend, pend_buf, g);
    __syncthreads();
  }
  // ---- line 41: converged -> norms (R#23), U = G diag(2^-e/f), sigma sorted
  // (R#24), V permuted; capped -> G = U Sigma', Sigma' (R#25)
  const bool conv = fin == 1;
  for (int j0 = 0; j0 < n; j0 += kG) {  // lane group per column, the step's R
    const int j = j0 + g;
    const E* x = sG + (j < n ? j : 0) * kM;
    double ssq = 0.0;
#pragma unroll
    for (int r = 0; r < kNR; ++r) ssq = ssq_acc(x[r * kW + hl], ssq);
    ssq = hsum<kW>(ssq);
    if (j < n && hl == 0) {
      int e;
      double gg;
      if (ssq > 0.0) {  // R#14 with E := cs
        eg_of(cs, ssq, e, gg);
        ce[j] = static_cast<double>(e);
        cf[j] = sqrt_plain(gg);
      } else {
        ce[j] = -INFINITY;
        cf[j] = 1.0;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < n) {  // the rank of column j: sSel[rank] = j
    const int j = threadIdx.x;
    int rank = j;
    if (conv) {
      const double ej = ce[j], fj = cf[j];
      rank = 0;
      for (int kk = 0; kk < n; ++kk) {
        const double ek = ce[kk], fk = cf[kk];
        rank += ((ek > ej) || (ek == ej && (fk > fj || (fk == fj && kk < j)))) ? 1 : 0;
      }
    }
    sSel[rank] = j;
  }
  __syncthreads();
  if (threadIdx.x < n) {
    const int r0 = threadIdx.x, j = sSel[r0];
    const double e = ce[j], f = cf[j];
    const bool fin_ = !isinf(e);
    const double es = (fin_ && conv) ? e - s : e;
    sigma[b * n + r0] = fin_ ? scalbn_rn(f, static_cast<int>(fmax(fmin(es, 1e5), -1e5))) : 0.0;
  }
  E* Aw = reinterpret_cast<E*>(A) + b * strideA;
  for (int r0 = warp; r0 < n; r0 += kT / 32) {  // U (or G) into A's storage
    const int j = sSel[r0];
    const double e = ce[j], f = cf[j];
    const bool fin_ = !isinf(e);
    // converged: 2^-e g / f = 2^(cs - e) g~ / f; capped: g = 2^cs g~
    const Pow2 sc(conv ? (fin_ ? cs - static_cast<int>(e) : 0) : cs);
    const Divisor d = make_divisor(f);
    const E* x = sG + j * kM;
    E* ucol = Aw + static_cast<int64_t>(r0) * lda;
    for (int i = lane; i < kM; i += 32) {
      E y = x[i];
      if (conv && fin_) {
        if constexpr (CPLX) y = make_double2(divide(sc(y.x), d), divide(sc(y.y), d));
        else y = divide(sc(y), d);
      } else if (!conv) {
        y = sc(y);
      }
      ucol[i] = y;
    }
  }
  __syncthreads();
  if (conv) {  // V's columns into sigma's order, staged through shared memory
    E* st = sG;  // G is no longer needed
    for (int q = threadIdx.x; q < n * n; q += kT) {
      const int j = q / n, i = q - j * n;
      st[q] = Vb[static_cast<int64_t>(j) * ldv + i];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < n * n; q += kT) {
      const int r0 = q / n, i = q - r0 * n;
      Vb[static_cast<int64_t>(r0) * ldv + i] = st[sSel[r0] * n + i];
    }
  }
  if (threadIdx.x == 0) {
    if (status_out) status_out[b] = conv ? JSVD_OK : JSVD_ENOCONV;
    if (sweeps_out) sweeps_out[b] = C;
    if (transforms_out) transforms_out[b] = sT;
    if (scale_out) scale_out[b] = s;
  }
}

size_t batched_fast_smem(bool cplx, int64_t n) {
  const size_t w = cplx ? 16 : 8;
  return w * kM * n + sizeof(Pair) * 2 * kG + sizeof(double) * 64 + 2 * (n - 1) * (n / 2);
}

bool batched_fast_ok(int64_t m, int64_t n) { return m == kM && n >= 2 && n <= 32 && (n & 1) == 0; }

// one CTA per matrix; `prof` (16 uint64, zeroed by the caller) selects the
// clock64-instrumented build
cudaError_t launch_batched_fast(bool cplx, int64_t batch, int64_t n, double* A, int64_t lda,
                            int64_t strideA, double* V, int64_t ldv, int64_t strideV,
                            double* sigma, int max_sweeps, int32_t* sweeps, int32_t* status,
                            int64_t* transforms, int32_t* scale, int Fm, int Kr, double tol,
                            int adj, unsigned long long* prof, cudaStream_t st) {
  const size_t smem = batched_fast_smem(cplx, n);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(batch), kT, smem, st>>>(static_cast<int>(n), A, lda, strideA, V,
                                                        ldv, strideV, sigma, max_sweeps, sweeps,
                                                        status, transforms, scale, Fm, Kr, tol,
                                                        adj, prof);
    note_launch();
    return cudaGetLastError();
  };
  if (cplx) return prof ? go(batched_fast_kernel<true, true>) : go(batched_fast_kernel<true, false>);
  return prof ? go(batched_fast_kernel<false, true>) : go(batched_fast_kernel<false, false>);
}

}  // namespace jsvd
