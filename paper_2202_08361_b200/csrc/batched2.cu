// batched2.cu -- the persistent two-slot kernel of jsvd_gesvj_batched for
// BASELINE configs[3]'s shape (m = 64, n <= 32): each CTA of 128 threads keeps
// TWO independent matrices ("slots") in shared memory and steps them together,
// so every lane group has two independent pairs in flight (twice the FP64
// instruction-level parallelism of batched.cu's kernel) and the scalar phase B
// fills all 32 lanes of its warp (the 16 pairs of each slot).  Each slot
// walks its own sequence of matrices (slot s of CTA i: matrices 2i + s,
// 2i + s + 2G, ...), loading the next one when its matrix is finished.
//
// Arithmetic: Alg 4.1 exactly as batched.cu (flat round-robin, the reduction
// spec R = (8, 1, [4, 2, 1]), the Eq. (skr) check at every step, line 41),
// computed on G~ = G 2^-cs: while every value of G~ is 0 or
// in [2^-400, 2^(1024-cs)] and every transformed pair's C, S is 0 or at least
// 2^-400, the norms' sums of squares, the dots and the rotations of G~ are
// exact power-of-two multiples of the oracle's, so the scaling multiplies of
// R#14 / Alg 3.1 and the exponent reductions are not needed.  A matrix that
// leaves that domain (checked at its load, on every transformed pair's C, S
// in phase B and on every rotated value in phase C) is abandoned -- its A is
// still intact (the working V lives in the V output, G only in shared
// memory) -- and marked in sigma; batched.cu's kernel then runs it from the
// start in G's own scale.
//
// Per tick (one step of each slot):
//   A  lane group g: pair g of slot 0 and pair g of slot 1 interleaved: the
//      SSQ of both columns and the dot of the raw G~ values (8 rows per lane)
//   B  warp 0, lane L: pair L mod 16 of slot L / 16: (e, f) of the norms, the
//      dot's rescale and division, the convergence test (Alg 3.2), Grammian
//      (Alg 3.3), 2x2 EVD (Alg 2.2); warps 1-3: the V rotations of the
//      previous tick (both slots; V in global memory, L2-resident)
//   C  lane group g: the rotations of G~ (Alg 3.4) for both slots
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "jsvd_host.h"
#include "step_dev.cuh"

namespace jsvd {

namespace b2 {

constexpr int kT = 256, kW = 8, kNR = 8, kM = 64, kGroups = 32, kPS = 16;  // kPS: pairs per slot
constexpr uint32_t kFastLo = static_cast<uint32_t>(1023 - 400) << 20;  // hi word of 2^-400
// sigma[b n] of a matrix abandoned to batched.cu's kernel (a NaN payload)
constexpr unsigned long long kMarker = 0x7ff8badc0ffee123ull;

struct Pair {
  double ar, ai, sp, sq;  // A: raw sums of G~ (dot, SSQ of p and q)
  double c, C, S;         // B: rotation
  int ep, eq;             // B: norm exponents (kIntMin: zero column)
  int transform, pad;
};

__device__ __forceinline__ uint32_t lo_hi_min(double2 x, uint32_t m) {
  return min(m, min(abs_hi(x.x) - 1u, abs_hi(x.y) - 1u));
}
__device__ __forceinline__ uint32_t lo_hi_min(double x, uint32_t m) { return min(m, abs_hi(x) - 1u); }

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

}  // namespace b2

using namespace b2;

template <bool CPLX, bool PROF>
__global__ void __launch_bounds__(kT, 3) batched2_kernel(
    int64_t batch, int n, double* A, int64_t lda, int64_t strideA, double* Vg, int64_t ldv,
    int64_t strideV, double* sigma, int max_sweeps, int32_t* sweeps_out, int32_t* status_out,
    int64_t* transforms_out, int32_t* scale_out, int Fm, int Kr, double tol, int s0_adjust,
    unsigned long long* prof) {
  using E = typename Elem<CPLX>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int np = n / 2;
  E* sG0 = reinterpret_cast<E*>(smem_raw);                   // [2][64 n]
  Pair* sP = reinterpret_cast<Pair*>(sG0 + 2 * kM * n);      // [2 slot][2 buf][16]
  double* sE = reinterpret_cast<double*>(sP + 2 * 2 * kPS);  // [2][2][32] finalize (e, f)
  uint8_t* sPairs = reinterpret_cast<uint8_t*>(sE + 2 * 2 * 32);  // (n-1) x np pivot pairs
  __shared__ uint64_t wred[kT / 32];
  __shared__ int sSel[32];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hl = threadIdx.x & (kW - 1), g = threadIdx.x / kW;  // lane in group, group
  const int64_t nslots_total = 2 * static_cast<int64_t>(gridDim.x);
  const auto G_of = [&](int s) { return sG0 + s * kM * n; };

  for (int k = threadIdx.x; k < (n - 1) * np; k += kT) {
    int p, q;
    strategy_pair(n, n, k / np, k % np, p, q);
    sPairs[2 * k] = static_cast<uint8_t>(p);
    sPairs[2 * k + 1] = static_cast<uint8_t>(q);
  }

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

  // Per-slot state in shared memory, written by thread 0 (then a barrier) and
  // read by every thread at the start of the phase that needs it, so nothing
  // of it stays live in registers across the phases.  sTc: the cumulative
  // transformation count (added by phase B); sBad: the domain flag (B, C);
  // sMt: M-tilde's high word (max-reduced by C).
  struct SlotSt {
    long long b;  // matrix (-1: no more work)
    int s, cs;    // scaling exponents of G and of G~ = G 2^-cs
  };
  __shared__ SlotSt st[2];
  // the step counters, uniform over the CTA, in every thread's registers:
  // step, sweep, pending V step, line-40 state (1 converged, 2 capped, 3
  // handed over) and the transformation count at the sweep's start
  int rk[2] = {0, 0}, rC[2] = {0, 0}, rpend[2] = {-1, -1}, rfin[2] = {0, 0}, rT0[2] = {0, 0};
  __shared__ int sTc[2], sBad[2];
  __shared__ uint32_t sMt[2];

  // ---- load matrix b into slot s (all threads); true: the slot runs it (fast
  // domain); false: ERANK / ENONFINITE written, or handed to batched.cu's kernel
  const auto load = [&](int s, long long b) -> bool {
    const E* Ag = reinterpret_cast<const E*>(A) + b * strideA;
    E* sG = G_of(s);
    uint64_t mx = 0, mn = ~0ull;
    constexpr int kPer = 8;  // elements per thread and round (loads issued together)
    for (int k0 = 0; k0 < kM * n; k0 += kT * kPer) {
      E x[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int k = k0 + u * kT + threadIdx.x;
        if (k < kM * n) {
          const int j = k / kM, i = k - j * kM;
          x[u] = Ag[static_cast<int64_t>(j) * lda + i];
        }
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
    const uint64_t M0b = cta_max_u64<kT>(mx, wred);
    __syncthreads();
    const uint64_t mnb = ~cta_max_u64<kT>(~mn, wred);
    __syncthreads();
    const double M0 = __longlong_as_double(static_cast<long long>(M0b));
    if (isinf(M0) || M0 == 0.0) {  // the matrix is left as it was
      if (threadIdx.x == 0) {
        if (status_out) status_out[b] = isinf(M0) ? JSVD_ENONFINITE : JSVD_ERANK;
        if (sweeps_out) sweeps_out[b] = 0;
        if (transforms_out) transforms_out[b] = 0;
        if (scale_out) scale_out[b] = 0;
      }
      return false;
    }
    const int lm0 = ilogb_bits(M0b);
    const int s0 = Fm - lm0 - 1 + s0_adjust;  // Eq. (skn) (+ s0_adjust, R#40)
    const int cs = lm0 + s0;                  // floor(lg M-tilde_1)
    const bool fast = (mnb == ~0ull || ilogb_bits(mnb + 1) >= lm0 - 400) && cs >= 600;
    if (!fast) {  // outside the fast domain from the start: batched.cu's kernel
      if (threadIdx.x == 0) reinterpret_cast<unsigned long long*>(sigma)[b * n] = kMarker;
      return false;
    }
    const double sc = pow2i(-lm0 >= -1022 ? -lm0 : -1022);  // G~ = A 2^-lm0 (lm0 <= 1023)
    const double sc2 = -lm0 >= -1022 ? 1.0 : pow2i(-lm0 + 1022);
    for (int k = threadIdx.x; k < kM * n; k += kT) {
      if constexpr (CPLX) sG[k] = make_double2((sG[k].x * sc) * sc2, (sG[k].y * sc) * sc2);
      else sG[k] = (sG[k] * sc) * sc2;
    }
    E* Vb = reinterpret_cast<E*>(Vg) + b * strideV;  // the working V: the V output
    for (int k = threadIdx.x; k < n * n; k += kT) {
      const int j = k / n, i = k - j * n;
      E v;
      if constexpr (CPLX) v = make_double2(i == j ? 1.0 : 0.0, 0.0);
      else v = i == j ? 1.0 : 0.0;
      Vb[static_cast<int64_t>(j) * ldv + i] = v;
    }
    rk[s] = rC[s] = rT0[s] = 0;
    rpend[s] = -1;
    rfin[s] = max_sweeps == 0 ? 2 : 0;
    if (threadIdx.x == 0) {
      st[s].b = b;
      st[s].s = s0;
      st[s].cs = cs;
      sMt[s] = hi32(scalbn_rn(M0, s0));
      sBad[s] = 0;
      sTc[s] = 0;
    }
    __syncthreads();
    return true;
  };

  // load matrices into slot s until one runs or the slot's sequence ends
  const auto next = [&](int s, long long b) {
    while (b < batch) {
      if (load(s, b)) return;
      b += nslots_total;
    }
    if (threadIdx.x == 0) st[s].b = -1;
    __syncthreads();
  };

  // V rotation of pair l of slot s's step kk (pair parameters in buffer buf),
  // by the 8 lanes of the caller's group: 4 rows per lane, loads first
  const auto rotate_v = [&](int s, int kk, int buf, int l) {
    const Pair& pr = sP[(s * 2 + buf) * kPS + l];
    if (!pr.transform) return;
    E* Vb = reinterpret_cast<E*>(Vg) + st[s].b * strideV;
    const int p = sPairs[2 * (kk * np + l)], q = sPairs[2 * (kk * np + l) + 1];
    E* vp = Vb + static_cast<int64_t>(p) * ldv;
    E* vq = Vb + static_cast<int64_t>(q) * ldv;
    constexpr int kRV = 4;  // rows per lane for n <= 32, two at a time (registers)
    const double c = pr.c, C = pr.C, S = pr.S;
#pragma unroll
    for (int h = 0; h < kRV; h += 2) {
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

  // ---- line 41 for slot s: converged -> norms (R#23), U = G diag(2^-e/f),
  // sigma sorted (R#24), V permuted; capped -> G = U Sigma', Sigma' (R#25)
  const auto finalize = [&](int s) {
    const bool conv = rfin[s] == 1;
    const int cs_ = st[s].cs, s_ = st[s].s;
    const long long b = st[s].b;
    E* sG = G_of(s);
    double* ce = sE + s * 64;
    double* cf = ce + 32;
    for (int j0 = 0; j0 < n; j0 += kGroups) {  // lane group per column, the step's R
      const int j = j0 + g;
      const E* x = sG + (j < n ? j : 0) * kM;
      double ssq = 0.0;
#pragma unroll
      for (int r = 0; r < kNR; ++r) ssq = ssq_acc(x[r * kW + hl], ssq);
      ssq = hsum<kW>(ssq);
      if (j < n && hl == 0) {
        int e;
        double gg;
        if (ssq > 0.0) {
          eg_of(cs_, ssq, e, gg);
          ce[j] = static_cast<double>(e);
          cf[j] = sqrt_plain(gg);
        } else {
          ce[j] = -INFINITY;
          cf[j] = 1.0;
        }
      }
    }
    __syncthreads();
    // rank of every column (stable by (e desc, f desc, index asc); R#24):
    // sSel[rank] = column
    if (threadIdx.x < n) {
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
      const bool fin = !isinf(e);
      const double es = (fin && conv) ? e - s_ : e;
      sigma[b * n + r0] = fin ? scalbn_rn(f, static_cast<int>(fmax(fmin(es, 1e5), -1e5))) : 0.0;
    }
    E* Ag = reinterpret_cast<E*>(A) + b * strideA;
    E* Vb = reinterpret_cast<E*>(Vg) + b * strideV;
    // U (or G) from shared memory into A's storage
    for (int r0 = warp; r0 < n; r0 += kT / 32) {
      const int j = sSel[r0];
      const double e = ce[j], f = cf[j];
      const bool fin = !isinf(e);
      // converged: 2^-e g / f = 2^(cs - e) g~ / f; capped: g = 2^cs g~
      const Pow2 sc(conv ? (fin ? cs_ - static_cast<int>(e) : 0) : cs_);
      const Divisor d = make_divisor(f);
      const E* x = sG + j * kM;
      E* ucol = Ag + static_cast<int64_t>(r0) * lda;
      for (int i = lane; i < kM; i += 32) {
        E y = x[i];
        if (conv && fin) {
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
      for (int k = threadIdx.x; k < n * n; k += kT) {
        const int j = k / n, i = k - j * n;
        st[k] = Vb[static_cast<int64_t>(j) * ldv + i];
      }
      __syncthreads();
      for (int k = threadIdx.x; k < n * n; k += kT) {
        const int r0 = k / n, i = k - r0 * n;
        Vb[static_cast<int64_t>(r0) * ldv + i] = st[sSel[r0] * n + i];
      }
    }
    if (threadIdx.x == 0) {
      if (status_out) status_out[b] = conv ? JSVD_OK : JSVD_ENOCONV;
      if (sweeps_out) sweeps_out[b] = rC[s];
      if (transforms_out) transforms_out[b] = sTc[s];
      if (scale_out) scale_out[b] = s_;
    }
    __syncthreads();
  };

  // ---- the slots' first matrices
  next(0, 2 * static_cast<long long>(blockIdx.x));
  next(1, 2 * static_cast<long long>(blockIdx.x) + 1);
  mark(6);

  int tick = 0;
  for (;;) {
    // finished slots: the pending V rotation, line 41, the next matrix
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const long long b = st[s].b;
      const int fin = rfin[s], pend = rpend[s];
      if (b < 0 || !fin) continue;
      if (fin != 3) {  // (3: handed over -- nothing to finish)
        if (pend >= 0) {
          if (g < np) rotate_v(s, pend, (tick - 1) & 1, g);
          __syncthreads();
        }
        finalize(s);
      }
      next(s, b + nslots_total);
    }
    if (st[0].b < 0 && st[1].b < 0) break;
    mark(6);
    const int buf = tick & 1;
    const bool act[2] = {st[0].b >= 0, st[1].b >= 0};
    // line 6, the Eq. (skr) check (every step of the flat ordering): in G~'s
    // scale a rescale only moves cs
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (!act[s]) continue;
      const uint32_t mt = sMt[s];
      const int lm = static_cast<int>(mt >> 20) - 1023;
      if (Kr - lm < 0) {  // uniform
        const int sn = Fm - lm - 1;
        __syncthreads();  // every thread has read sMt[s]
        if (threadIdx.x == 0) {
          sMt[s] = hi32(scalbn_rn(mkd(mt, 0u), sn));
          st[s].cs += sn;
          st[s].s += sn;
        }
      }
    }
    const int kk[2] = {rk[0], rk[1]};
    // ---- phase A: group g takes pair g mod 16 of slot g / 16 (raw sums of
    // G~); a group without a pair (n < 32) computes pair 0 and stores
    // nothing, so every lane takes part in the shuffles
    {
      const int sa = g >> 4, l = g & 15, la = l < np ? l : 0;
      const int p = sPairs[2 * (kk[sa] * np + la)], q = sPairs[2 * (kk[sa] * np + la) + 1];
      const E* gp = G_of(sa) + p * kM;
      const E* gq = G_of(sa) + q * kM;
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
      if (hl == 0 && l < np) {
        Pair& P = sP[(sa * 2 + buf) * kPS + l];
        P.sp = sp;
        P.sq = sq;
        P.ar = ar;
        P.ai = ai;
      }
    }
    mark(0);
    __syncthreads();
    mark(1);
    // ---- phase B (warp 0, lane L: slot L/16, pair L mod 16) | V (warps 1-3)
    if (warp == 0) {
      const int s = lane >> 4, l = lane & 15;
      const bool on = act[s] && l < np;
      Pair& P = sP[(s * 2 + buf) * kPS + l];
      const double spv = on ? P.sp : 1.0, sqv = on ? P.sq : 1.0;
      const int c_s = st[s].cs;
      // R#14 with E := cs (the SSQ of G~ carries 2^(2E - 2cs) exactly)
      const bool zp = !(spv > 0.0), zq = !(sqv > 0.0);
      int iep = kIntMin, ieq = kIntMin;
      double gp = 1.0, gq = 1.0;
      if (!zp) eg_of(c_s, spv, iep, gp);
      if (!zq) eg_of(c_s, sqv, ieq, gq);
      double arv = on ? P.ar : 0.0, aiv = on ? P.ai : 0.0;
      if (!(zp || zq)) {  // the dot of G~ carries 2^(2cs - e_q - e_p) exactly
        const double f2 = pow2i(2 * c_s - iep - ieq);
        arv *= f2;
        aiv *= f2;
      }
      const double fp = zp ? 1.0 : sqrt_plain(gp), fq = zq ? 1.0 : sqrt_plain(gq);
      const double ep = zp ? -INFINITY : static_cast<double>(iep);
      const double eq = zq ? -INFINITY : static_cast<double>(ieq);
      const Rcp d = rcp_plain(fq * fp);  // Alg 3.1 line 8
      const double zr = dot_div(arv, d, kFull);
      const double zi = CPLX ? dot_div(aiv, d, kFull) : 0.0;
      const double az = CPLX ? hypot_naive(fabs(zr), fabs(zi)) : fabs(zr);
      const bool tr = on && !(zp || zq) && tol <= az;  // Alg 3.2
      bool bad = false;
      if (__any_sync(kFull, tr)) {
        double b11, b22, br, bi;
        gram_fast(tr ? zr : 0.0, tr ? zi : 0.0, tr ? ep : 0.0, tr ? fp : 1.0, tr ? eq : 0.0,
                  tr ? fq : 1.0, b11, b22, br, bi, kFull);
        const Evd2Out o = evd2<CPLX, true, true, false>(b11, b22, br, bi, kFull);
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
        sTc[0] += __popc(tb & 0xffffu);
        sTc[1] += __popc(tb >> 16);
        if (bb & 0xffffu) sBad[0] = 1;
        if (bb >> 16) sBad[1] = 1;
      }
    } else {  // groups 4..31: the V rotations of the previous tick (both slots)
      for (int lv = g - 4; lv < 2 * kPS; lv += kGroups - 4) {
        const int s = lv >> 4, l = lv & 15;
        if (l < np && act[s] && rpend[s] >= 0) rotate_v(s, rpend[s], buf ^ 1, l);
      }
    }
    mark(2);
    __syncthreads();
    mark(3);
    const bool bad_b[2] = {sBad[0] != 0, sBad[1] != 0};
    // ---- phase C: rotations of G~ (Alg 3.4) and the fast-domain check;
    // warps 0-3 hold slot 0's groups, warps 4-7 slot 1's
    {
      const int sc_ = g >> 4, l = g & 15;
      uint32_t Mw = 0, lmin = ~0u;
      const Pair& P = sP[(sc_ * 2 + buf) * kPS + l];
      if (l < np && act[sc_] && !bad_b[sc_] && P.transform) {
        const int p = sPairs[2 * (kk[sc_] * np + l)], q = sPairs[2 * (kk[sc_] * np + l) + 1];
        E* gp = G_of(sc_) + p * kM;
        E* gq = G_of(sc_) + q * kM;
        const double c = P.c, Cc = P.C, S = P.S;
        // M-tilde: only pairs with max(e) > K - 1 can reach 2^(K+1) (see step.cu)
        const bool track = max(P.ep, P.eq) > Kr - 1;
        constexpr int kH = kNR / 4;  // a quarter of the lane's rows at a time (registers)
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
      Mw = __reduce_max_sync(0xffffffffu, Mw);
      if (lane == 0 && Mw) atomicMax(&sMt[sc_], Mw + (static_cast<uint32_t>(st[sc_].cs) << 20));
      if (lmin < kFastLo - 1u) sBad[sc_] = 1;  // G = G~ 2^cs above (normal values)
    }
    mark(4);
    __syncthreads();
    mark(5);
    // ---- bookkeeping, in every thread (registers): step / sweep counters,
    // line 40; the next barrier (after phase A) orders the shared state
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (!act[s]) continue;
      if (sBad[s]) {  // left the fast domain: batched.cu's kernel redoes it
        if (threadIdx.x == 0) reinterpret_cast<unsigned long long*>(sigma)[st[s].b * n] = kMarker;
        rfin[s] = 3;
        continue;
      }
      rpend[s] = rk[s];
      if (++rk[s] == n - 1) {  // end of a sweep (line 40)
        rk[s] = 0;
        ++rC[s];
        const int tc = sTc[s];
        if (tc == rT0[s]) rfin[s] = 1;
        else if (rC[s] == max_sweeps) rfin[s] = 2;
        rT0[s] = tc;
      }
    }
    ++tick;
    mark(6);
  }
  if constexpr (PROF) {  // [6]: loads, line 41 and bookkeeping; [7]: the whole kernel
    pc[7] = pc[0] + pc[1] + pc[2] + pc[3] + pc[4] + pc[5] + pc[6];
    if (lane == 0)
      for (int k = 0; k < 8; ++k) atomicAdd(&prof[(warp == 0 ? 0 : 1) * 8 + k], pc[k]);
  }
}

size_t batched2_smem(bool cplx, int64_t n) {
  const size_t w = cplx ? 16 : 8;
  return w * 2 * kM * n + sizeof(Pair) * 2 * 2 * kPS + sizeof(double) * 2 * 2 * 32 +
         2 * (n - 1) * (n / 2);
}

bool batched2_ok(int64_t m, int64_t n) { return m == kM && n >= 2 && n <= 32 && (n & 1) == 0; }

// launch the persistent kernel over the batch; `prof` (16 uint64, zeroed by
// the caller) selects the clock64-instrumented build
cudaError_t launch_batched2(bool cplx, int64_t batch, int64_t n, double* A, int64_t lda,
                            int64_t strideA, double* V, int64_t ldv, int64_t strideV,
                            double* sigma, int max_sweeps, int32_t* sweeps, int32_t* status,
                            int64_t* transforms, int32_t* scale, int Fm, int Kr, double tol,
                            int adj, unsigned long long* prof, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = batched2_smem(cplx, n);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kT, smem);
    const int64_t want = (batch + 1) / 2;
    const int64_t grid = std::min<int64_t>(want, static_cast<int64_t>(std::max(per_sm, 1)) * sms);
    kern<<<static_cast<unsigned>(grid), kT, smem, st>>>(batch, static_cast<int>(n), A, lda,
                                                       strideA, V, ldv, strideV, sigma,
                                                       max_sweeps, sweeps, status, transforms,
                                                       scale, Fm, Kr, tol, adj, prof);
    note_launch();
    return cudaGetLastError();
  };
  if (cplx) return prof ? go(batched2_kernel<true, true>) : go(batched2_kernel<true, false>);
  return prof ? go(batched2_kernel<false, true>) : go(batched2_kernel<false, false>);
}

}  // namespace jsvd
