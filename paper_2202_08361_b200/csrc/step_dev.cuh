// step_dev.cuh -- device building blocks of one Jacobi step (Alg 4.1 lines
// 7-38) for a pivot pair held in registers by a CTA or a
// thread-block cluster of CL CTAs x T threads (W = CL*T lanes).
//
// Reduction spec R (R#15): element i of a column lives in lane L = i mod W
// (CTA rank L / T, thread L % T) and is accumulated in increasing i; lanes
// combine by xor-butterfly over offsets [16,8,4,2,1] (warp shuffles), then the
// warp-index bits high->low (shared memory), then the CTA-rank bits high->low
// (distributed shared memory).  Addition is commutative, so every lane ends
// with the identical total: the result depends only on (W, m), never on launch
// geometry, scheduling or GPU count.
#pragma once
#include <cooperative_groups.h>

#include "jsvd_dev.cuh"

namespace jsvd {
namespace cg = cooperative_groups;

constexpr int kIntMin = -2147483647 - 1;

// ---------------------------------------------------------------- elements
template <bool CPLX> struct Elem;
template <> struct Elem<false> {
  using T = double;
  static __device__ __forceinline__ T zero() { return 0.0; }
};
template <> struct Elem<true> {
  using T = double2;
  static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
};

__device__ __forceinline__ uint64_t absmax_bits(double x, uint64_t m) { return max(m, abs_bits(x)); }
__device__ __forceinline__ uint64_t absmax_bits(double2 x, uint64_t m) {
  return max(m, max(abs_bits(x.x), abs_bits(x.y)));
}

// 2^n for any n in [-1074, 1023]: normal or subnormal power of two, exact
__device__ __forceinline__ double pow2_any(int n) {
  return n >= -1022 ? pow2i(n) : __longlong_as_double(1ll << (n + 1074));
}

__device__ __forceinline__ double scale1(double x, double a) { return x * a; }
__device__ __forceinline__ double2 scale1(double2 x, double a) { return make_double2(x.x * a, x.y * a); }
__device__ __forceinline__ double scale2(double x, double a, double b) { return (x * a) * b; }
__device__ __forceinline__ double2 scale2(double2 x, double a, double b) {
  return make_double2((x.x * a) * b, (x.y * a) * b);
}

// x * 2^n with one rounding for n in [-1074, 2046] (R#3): one multiply, or two
// when n > 1023 (the first, an upscaling, is exact).
struct Pow2 {
  double a, b;
  bool two;
  __device__ __forceinline__ explicit Pow2(int n) {
    two = n > 1023;
    a = two ? 0x1p1023 : pow2_any(n);
    b = two ? pow2i(n - 1023) : 1.0;
  }
  __device__ __forceinline__ double operator()(double x) const { return two ? (x * a) * b : x * a; }
  __device__ __forceinline__ double2 operator()(double2 x) const {
    return make_double2((*this)(x.x), (*this)(x.y));
  }
};

// ---------------------------------------------------------------- reductions
// Fold s[0..N) by offsets N/2, ..., 1 keeping lane 0's view of the butterfly.
template <int N, typename V, typename Op>
__device__ __forceinline__ V fold(const V* s, Op op) {
  V t[N];
#pragma unroll
  for (int k = 0; k < N; ++k) t[k] = s[k];
#pragma unroll
  for (int h = N / 2; h >= 1; h /= 2) {
#pragma unroll
    for (int k = 0; k < h; ++k) t[k] = op(t[k], t[k + h]);
  }
  return t[0];
}

struct AddOp {
  __device__ __forceinline__ double operator()(double a, double b) const { return a + b; }
};
struct MaxIOp {
  __device__ __forceinline__ int operator()(int a, int b) const { return max(a, b); }
};
struct MaxU64Op {
  __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const { return max(a, b); }
};

// Shared-memory slots of one 2-value reduction.
template <int NW, typename V> struct RedSlot {
  V warp[2][NW];
  V cta[2];
};

// Sum of (a, b) over all W lanes in the order of R; every thread gets the result.
template <int T, int CL>
__device__ __forceinline__ void tree_sum2(double& a, double& b, RedSlot<T / 32, double>& s) {
  constexpr int NW = T / 32;
#pragma unroll
  for (int o = 16; o >= 1; o /= 2) {
    a = a + __shfl_xor_sync(0xffffffffu, a, o);
    b = b + __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s.warp[0][w] = a;
    s.warp[1][w] = b;
  }
  __syncthreads();
  a = fold<NW>(s.warp[0], AddOp());
  b = fold<NW>(s.warp[1], AddOp());
  if constexpr (CL > 1) {
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0) {
      s.cta[0] = a;
      s.cta[1] = b;
    }
    cl.sync();
    double ra[CL], rb[CL];
#pragma unroll
    for (int r = 0; r < CL; ++r) {
      const double* rs = cl.map_shared_rank(s.cta, r);
      ra[r] = rs[0];
      rb[r] = rs[1];
    }
    a = fold<CL>(ra, AddOp());
    b = fold<CL>(rb, AddOp());
  }
}

// Max of two ints over all W lanes (exact, order-free).
template <int T, int CL>
__device__ __forceinline__ void tree_max2i(int& a, int& b, RedSlot<T / 32, int>& s) {
  constexpr int NW = T / 32;
  a = __reduce_max_sync(0xffffffffu, a);
  b = __reduce_max_sync(0xffffffffu, b);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s.warp[0][w] = a;
    s.warp[1][w] = b;
  }
  __syncthreads();
  a = fold<NW>(s.warp[0], MaxIOp());
  b = fold<NW>(s.warp[1], MaxIOp());
  if constexpr (CL > 1) {
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0) {
      s.cta[0] = a;
      s.cta[1] = b;
    }
    cl.sync();
    int ra[CL], rb[CL];
#pragma unroll
    for (int r = 0; r < CL; ++r) {
      const int* rs = cl.map_shared_rank(s.cta, r);
      ra[r] = rs[0];
      rb[r] = rs[1];
    }
    a = fold<CL>(ra, MaxIOp());
    b = fold<CL>(rb, MaxIOp());
  }
}

// ---- cross-CTA rounds through distributed shared memory without cluster
// barriers: thread 0 of every CTA pushes the CTA's partial pair into slot
// [own rank] of every CTA of the cluster with st.async, whose completion
// (complete_tx) lands on the receiver's mbarrier; each CTA waits on its own
// mbarrier for all CL partials and folds them in rank order (the CTA bits of R,
// high to low).  One mbarrier per round (each used once per launch: phase 0).
// The barriers are initialised and published once per launch (txred_init).
template <int CL, typename V>
struct alignas(16) TxSlot {
  alignas(16) V part[CL][2];  // st.async.v2 targets: 16-byte (f64) / 8-byte (s32) aligned
  unsigned long long bar;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
template <int CL, typename V>
__device__ __forceinline__ void txslot_init(TxSlot<CL, V>& t) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&t.bar)), "r"(1) : "memory");
}
// after every txslot_init of the launch: make the barriers visible to the peers
__device__ __forceinline__ void txred_publish() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void st_async_pair(uint32_t dst, double a, double b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n"
               ::"r"(dst), "d"(a), "d"(b), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_pair(uint32_t dst, int a, int b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.s32 [%0], {%1, %2}, [%3];\n"
               ::"r"(dst), "r"(a), "r"(b), "r"(bar) : "memory");
}
// the CTA's partial (a, b), known to thread 0 -> every CTA gets all CL partials
template <int CL, typename V, typename Op>
__device__ __forceinline__ void tx_exchange(V& a, V& b, TxSlot<CL, V>& t, Op op) {
  const uint32_t bar = smem_u32(&t.bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                 ::"r"(bar), "r"(static_cast<int>(CL * 2 * sizeof(V))) : "memory");
    const uint32_t me = cg::this_cluster().block_rank();
    const uint32_t slot = smem_u32(&t.part[me][0]);
#pragma unroll
    for (int r = 0; r < CL; ++r) st_async_pair(mapa_u32(slot, r), a, b, mapa_u32(bar, r));
  }
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(bar), "r"(0) : "memory");
  } while (!done);
  V ra[CL], rb[CL];
#pragma unroll
  for (int r = 0; r < CL; ++r) {
    ra[r] = t.part[r][0];
    rb[r] = t.part[r][1];
  }
  a = fold<CL>(ra, op);
  b = fold<CL>(rb, op);
}

// tree_sum2 / tree_max2i with the cross-CTA level through tx_exchange
template <int T, int CL>
__device__ __forceinline__ void tree_sum2_tx(double& a, double& b, RedSlot<T / 32, double>& s,
                                             TxSlot<CL, double>& t) {
  constexpr int NW = T / 32;
#pragma unroll
  for (int o = 16; o >= 1; o /= 2) {
    a = a + __shfl_xor_sync(0xffffffffu, a, o);
    b = b + __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s.warp[0][w] = a;
    s.warp[1][w] = b;
  }
  __syncthreads();
  a = fold<NW>(s.warp[0], AddOp());
  b = fold<NW>(s.warp[1], AddOp());
  tx_exchange<CL>(a, b, t, AddOp());
}
template <int T, int CL>
__device__ __forceinline__ void tree_max2i_tx(int& a, int& b, RedSlot<T / 32, int>& s,
                                              TxSlot<CL, int>& t) {
  constexpr int NW = T / 32;
  a = __reduce_max_sync(0xffffffffu, a);
  b = __reduce_max_sync(0xffffffffu, b);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s.warp[0][w] = a;
    s.warp[1][w] = b;
  }
  __syncthreads();
  a = fold<NW>(s.warp[0], MaxIOp());
  b = fold<NW>(s.warp[1], MaxIOp());
  tx_exchange<CL>(a, b, t, MaxIOp());
}

// CTA-wide max of a u64 (result valid in thread 0 only).
template <int T>
__device__ __forceinline__ uint64_t cta_max_u64(uint64_t v, uint64_t* warp_slots) {
#pragma unroll
  for (int o = 16; o >= 1; o /= 2) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) warp_slots[threadIdx.x >> 5] = v;
  __syncthreads();
  return fold<T / 32>(warp_slots, MaxU64Op());
}

// CTA-wide max of a u32, every thread gets it
template <int T>
__device__ __forceinline__ uint32_t cta_max_u32(uint32_t v, uint32_t* warp_slots) {
  v = __reduce_max_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) warp_slots[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t r = warp_slots[0];
#pragma unroll
  for (int w = 1; w < T / 32; ++w) r = max(r, warp_slots[w]);
  return r;
}
// max of m and the low words of the components whose |high word| is H
__device__ __forceinline__ uint32_t lo_max_at(double x, uint32_t H, uint32_t m) {
  return (hi32(x) & 0x7fffffffu) == H ? max(m, lo32(x)) : m;
}
__device__ __forceinline__ uint32_t lo_max_at(double2 x, uint32_t H, uint32_t m) {
  return lo_max_at(x.y, H, lo_max_at(x.x, H, m));
}

// floor(lg max|x|) of the lane's elements as an int (kIntMin if all zero)
__device__ __forceinline__ int ilogb_or_min(uint64_t b) { return b ? ilogb_bits(b) : kIntMin; }

// |x| high words: their max carries floor(lg max|x|) unless it is subnormal
__device__ __forceinline__ uint32_t abs_hi(double x) { return hi32(x) & 0x7fffffffu; }
__device__ __forceinline__ uint32_t hi_max(double x, uint32_t m) { return max(m, abs_hi(x)); }
__device__ __forceinline__ uint32_t hi_max(double2 x, uint32_t m) {
  return max(m, max(abs_hi(x.x), abs_hi(x.y)));
}
// floor(lg max|component|) of a lane's NR elements from their high-word max h;
// a lane whose largest component is subnormal (or zero) takes the exact path
template <int NR, typename E>
__device__ __forceinline__ int lane_exponent(uint32_t h, const E* x) {
  if (h >= 0x00100000u) return static_cast<int>(h >> 20) - 1023;
  uint64_t m = 0;
#pragma unroll
  for (int j = 0; j < NR; ++j) m = absmax_bits(x[j], m);
  return ilogb_or_min(m);
}


// (e, f) of a column from E = floor(lg max) and the total SSQ of x 2^-E
// (R#14): k = logb(SSQ), g = SSQ 2^-k, odd k -> (2g, k-1),
// f = sqrt(g), e = E + k/2.  SSQ >= 1 here (the max element scales to [1,2)).
__device__ __forceinline__ void ef_from_ssq(int E, double ssq, double& e, double& f) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(ssq));
  int k = static_cast<int>(b >> 52) - 1023;
  double g = __longlong_as_double(static_cast<long long>((b & 0x000fffffffffffffull) |
                                                         0x3ff0000000000000ull));
  if (k & 1) {
    g = g * 2.0;
    k -= 1;
  }
  f = sqrt_plain(g);  // g in [1, 4)
  e = static_cast<double>(E + k / 2);
}

// ---- the scaled domain of DESIGN.md 4.6 (batched kernels, step kernel):
// every nonzero scaled value in [2^-400, 2^16], i.e. a high word (sign
// masked) of at least kFastLo and below kFastHi.  lo_hi_min folds hi(|x|) - 1
// into a running minimum (0 maps to 0xffffffff and passes).
constexpr uint32_t kFastLo = static_cast<uint32_t>(1023 - 400) << 20;
constexpr uint32_t kFastHi = static_cast<uint32_t>(1023 + 16) << 20;
__device__ __forceinline__ uint32_t lo_hi_min(double x, uint32_t m) {
  return min(m, (hi32(x) & 0x7fffffffu) - 1u);
}
__device__ __forceinline__ uint32_t lo_hi_min(double2 x, uint32_t m) {
  return min(m, min((hi32(x.x) & 0x7fffffffu) - 1u, (hi32(x.y) & 0x7fffffffu) - 1u));
}
// e = E + k/2 and g = SSQ 2^-k (k even) from a positive normal sum of squares
// (R#14), E the scale exponent the squared values carry
__device__ __forceinline__ void eg_from_ssq_c(int E, double ssq, int& e, double& g) {
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

// fold one element into the SSQ accumulator (fma(y,y,.) re then im)
__device__ __forceinline__ double ssq_acc(double y, double acc) { return fma(y, y, acc); }
__device__ __forceinline__ double ssq_acc(double2 y, double acc) {
  acc = fma(y.x, y.x, acc);
  return fma(y.y, y.y, acc);
}

// Alg 3.1 lines 5-6: accumulate conj(q) p of prescaled elements
__device__ __forceinline__ void dot_acc(double q, double p, double& ar, double&) {
  ar = fma(q, p, ar);
}
__device__ __forceinline__ void dot_acc(double2 q, double2 p, double& ar, double& ai) {
  ar = fma(q.x, p.x, ar);
  ai = fma(q.x, p.y, ai);
  ar = fma(q.y, p.y, ar);
  ai = fma(-q.y, p.x, ai);
}

// SSQ of x 2^-E over a lane's NR elements in increasing index (R#14); E is
// uniform over the caller's group, so the two-multiply case (2^-E not
// representable: E < -1023) is a uniform branch.  Zero-filled padding adds
// exact zeros to a non-negative sum.
template <int NR, typename E>
__device__ __forceinline__ double ssq_lane(const E* x, int Ex) {
  double s = 0.0;
  if (-Ex > 1023) {
    const double a = 0x1p1023, b = pow2i(-Ex - 1023);
#pragma unroll
    for (int j = 0; j < NR; ++j) s = ssq_acc(scale2(x[j], a, b), s);
  } else if (-Ex < -1022) {  // 2^-E subnormal (max |x| >= 2^1023: outside the step's precondition)
    const double a = pow2_any(-Ex);
#pragma unroll
    for (int j = 0; j < NR; ++j) s = ssq_acc(scale1(x[j], a), s);
  } else {  // the common case: 2^-E normal, built from its exponent field alone
    const double a = pow2i(-Ex);
#pragma unroll
    for (int j = 0; j < NR; ++j) s = ssq_acc(scale1(x[j], a), s);
  }
  return s;
}

// Alg 3.1 lines 5-6 over a lane's NR elements with the prescale 2^-e (e
// uniform over the caller's group; two multiplies only when 2^-e is not
// representable).  Zero padding adds exact zeros (at most the sign of a zero
// partial sum changes, which no output depends on: z = 0 is never transformed).
template <int NR, typename E>
__device__ __forceinline__ void dot_lane(const E* xq, const E* xp, int eq, int ep, double& ar,
                                         double& ai) {
  ar = ai = 0.0;
  if (-eq > 1023 || -ep > 1023) {
    const Pow2 fQ(-eq), fP(-ep);
#pragma unroll
    for (int j = 0; j < NR; ++j)
      dot_acc(scale2(xq[j], fQ.a, fQ.b), scale2(xp[j], fP.a, fP.b), ar, ai);
  } else if (-eq < -1022 || -ep < -1022) {
    const double aq = pow2_any(-eq), ap = pow2_any(-ep);
#pragma unroll
    for (int j = 0; j < NR; ++j) dot_acc(scale1(xq[j], aq), scale1(xp[j], ap), ar, ai);
  } else {  // the common case: both factors normal powers of two
    const double aq = pow2i(-eq), ap = pow2i(-ep);
#pragma unroll
    for (int j = 0; j < NR; ++j) dot_acc(scale1(xq[j], aq), scale1(xp[j], ap), ar, ai);
  }
}

// Alg 3.4 with P = I: x_p' = fma(x_q, e', x_p) c, x_q' = fma(x_p, -conj(e'), x_q) c
__device__ __forceinline__ void rot_elem(double& xp, double& xq, double c, double C, double) {
  const double p = xp, q = xq;
  xp = fma(q, C, p) * c;
  xq = fma(p, -C, q) * c;
}
__device__ __forceinline__ void rot_elem(double2& xp, double2& xq, double c, double C, double S) {
  const double rp = xp.x, ip = xp.y, rq = xq.x, iq = xq.y;
  xp.x = fma(rq, C, fma(-iq, S, rp)) * c;
  xp.y = fma(rq, S, fma(iq, C, ip)) * c;
  xq.x = fma(rp, -C, fma(-ip, S, rq)) * c;
  xq.y = fma(rp, S, fma(ip, -C, iq)) * c;
}

// getmant(x, [1,2), sign zero) and logb for a positive finite normal x
__device__ __forceinline__ int ilogb_pos(double x) { return ilogb_bits(abs_bits(x)); }
__device__ __forceinline__ double mant12(double x) {
  const uint64_t b = abs_bits(x);
  if (b >> 52) return __longlong_as_double(static_cast<long long>((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
  return scalbn_rn(__longlong_as_double(static_cast<long long>(b)), -ilogb_bits(b));
}

// Alg 3.3: the non-overflowing scaled Grammian of the pair
__device__ __forceinline__ void gram(double zr, double zi, double e1, double f1, double e2,
                                     double f2, double& a11, double& a22, double& br, double& bi) {
  double f12 = f1 / f2, e12 = e1 - e2;
  double f21 = f2 / f1, e21 = e2 - e1;
  e12 = e12 + static_cast<double>(ilogb_pos(f12));
  f12 = mant12(f12);
  e21 = e21 + static_cast<double>(ilogb_pos(f21));
  f21 = mant12(f21);
  const double sA = fmin(static_cast<double>(kEtaHat) - fmax(e12, e21), 0.0);
  e12 = e12 + sA;
  e21 = e21 + sA;
  a11 = scalbn_rn(f12, static_cast<int>(e12));
  a22 = scalbn_rn(f21, static_cast<int>(e21));
  br = scalbn_rn(zr, static_cast<int>(sA));
  bi = scalbn_rn(zi, static_cast<int>(sA));
}

// Alg 3.3 for the norm significands the step produces (f1, f2 in [1, 2), e
// integral): f12 = f1/f2 and f21 = f2/f1 lie in (1/2, 2), so both quotients
// are plain divisions, logb is -1 or 0 and getmant a doubling.  The common
// case -- s_A = 0 and both exponents >= -1022 -- then needs one exact multiply
// per diagonal entry and leaves z unscaled; any lane outside it (exponents of
// the two norms more than ~1022 apart) takes gram() in a uniform branch.
// Same bits as gram() for every input it accepts (tested against the oracle).
// returns true when this lane took the fast path (then br, bi = zr, zi)
__device__ __forceinline__ bool gram_fast(double zr, double zi, double e1, double f1, double e2,
                                          double f2, double& a11, double& a22, double& br,
                                          double& bi, unsigned mask) {
  double f12 = div_plain(f1, rcp_plain(f2));
  double f21 = div_plain(f2, rcp_plain(f1));
  int e12 = static_cast<int>(e1 - e2), e21 = -e12;
  const bool l12 = f12 < 1.0, l21 = f21 < 1.0;
  e12 -= l12 ? 1 : 0;
  e21 -= l21 ? 1 : 0;
  f12 = l12 ? f12 * 2.0 : f12;
  f21 = l21 ? f21 * 2.0 : f21;
  const bool fast = max(e12, e21) <= kEtaHat && min(e12, e21) >= -1022;
  a11 = f12 * pow2i(fast ? e12 : 0);
  a22 = f21 * pow2i(fast ? e21 : 0);
  br = zr;
  bi = zi;
  if (__any_sync(mask, !fast)) {
    double g11, g22, gr, gi;
    gram(zr, zi, e1, f1, e2, f2, g11, g22, gr, gi);
    if (!fast) {
      a11 = g11;
      a22 = g22;
      br = gr;
      bi = gi;
    }
  }
  return fast;
}

// gram_fast with integral exponents passed as ints (no int <-> double
// conversions on the caller's dependency chain; the same bits)
__device__ __forceinline__ bool gram_fast_i(double zr, double zi, int e1, double f1, int e2,
                                            double f2, double& a11, double& a22, double& br,
                                            double& bi, unsigned mask) {
  double f12 = div_plain(f1, rcp_plain(f2));
  double f21 = div_plain(f2, rcp_plain(f1));
  int e12 = e1 - e2, e21 = -e12;
  const bool l12 = f12 < 1.0, l21 = f21 < 1.0;
  e12 -= l12 ? 1 : 0;
  e21 -= l21 ? 1 : 0;
  f12 = l12 ? f12 * 2.0 : f12;
  f21 = l21 ? f21 * 2.0 : f21;
  const bool fast = max(e12, e21) <= kEtaHat && min(e12, e21) >= -1022;
  a11 = f12 * pow2i(fast ? e12 : 0);
  a22 = f21 * pow2i(fast ? e21 : 0);
  br = zr;
  bi = zi;
  if (__any_sync(mask, !fast)) {
    double g11, g22, gr, gi;
    gram(zr, zi, static_cast<double>(e1), f1, static_cast<double>(e2), f2, g11, g22, gr, gi);
    if (!fast) {
      a11 = g11;
      a22 = g22;
      br = gr;
      bi = gi;
    }
  }
  return fast;
}

// z = a / d for the dot's sums over d = fl(f_q f_p) in [1, 4) (Alg 3.1 line
// 8): the plain division when |a| >= 2^-968 (then the quotient is normal),
// the general one in a uniform branch for tiny or zero sums
__device__ __forceinline__ double dot_div(double a, const Rcp& r, unsigned mask) {
  double z = div_plain(a, r);
  const bool tiny = !(fabs(a) >= 0x1p-968);
  if (__any_sync(mask, tiny)) {
    const double g = divide_sf<true, false>(a, make_divisor_normal(r.d), mask);
    z = tiny ? g : z;
  }
  return z;
}

// ---------------------------------------------------------------- strategy
// R#20: circle method on P players, round r: position 0 = player 0, position
// k >= 1 = player ((k-1+r) mod (P-1)) + 1; pair i = positions (i, P-1-i).
// 0 <= pos, r < P - 1 (or pos = 0), so (pos - 1 + r) mod (P - 1) is one
// conditional subtraction (n < 2^31: 32-bit arithmetic).
__device__ __host__ __forceinline__ int circle_player(int P, int r, int pos) {
  int x = pos - 1 + r;
  x = x >= P - 1 ? x - (P - 1) : x;
  return pos == 0 ? 0 : x + 1;
}

// pair l of step `step` of the block round-robin with B blocks of b = n/B
__device__ __host__ __forceinline__ void strategy_pair(int64_t n64, int64_t B64, int64_t step64,
                                                       int64_t l64, int& p, int& q) {
  const int n = static_cast<int>(n64), B = static_cast<int>(B64);
  const int step = static_cast<int>(step64), l = static_cast<int>(l64);
  const int b = n / B;
  int x, y;
  if (step < b - 1) {  // phase I: flat RR inside every block
    const int beta = l / (b / 2), i = l - beta * (b / 2);
    x = beta * b + circle_player(b, step, i);
    y = beta * b + circle_player(b, step, b - 1 - i);
  } else {  // phase II: rounds of flat RR over blocks, b steps per round
    const int s2 = step - (b - 1), rr = s2 / b, tt = s2 - rr * b;
    const int i = l / b, j = l - i * b;
    const int u = circle_player(B, rr, i), v = circle_player(B, rr, B - 1 - i);
    const int be = u < v ? u : v, bf = u < v ? v : u;  // block pair (beta < beta')
    const int jt = j + tt;
    x = be * b + j;
    y = bf * b + (jt >= b ? jt - b : jt);
  }
  p = x < y ? x : y;
  q = x < y ? y : x;
}

// ---- the block round-robin sharded over nr ranks ----------
// Rank g owns the per = B/2/nr position pairs (i, B-1-i), i in [g per,
// (g+1) per): local slot 2k holds position g per + k, slot 2k+1 position
// B-1-(g per + k); slot s is local columns [s b, (s+1) b).  In round r
// position k holds block circle_player(B, r, k) (round 0: block k).
__device__ __host__ __forceinline__ int dist_slot_position(int B, int nr, int rank, int slot) {
  const int i = rank * (B / 2 / nr) + slot / 2;
  return (slot & 1) ? B - 1 - i : i;
}

// (rank, slot) holding circle position pos
__device__ __host__ __forceinline__ void dist_owner(int B, int nr, int pos, int& rank, int& slot) {
  const int per = B / 2 / nr;
  const bool low = pos < B / 2;
  const int i = low ? pos : B - 1 - pos;
  rank = i / per;
  slot = 2 * (i - rank * per) + (low ? 0 : 1);
}

// global column of local column l at round 0 (every sweep starts and ends
// there: B - 1 rounds move every block once around the circle)
__device__ __host__ __forceinline__ int dist_gcol(int n, int B, int nr, int rank, int l) {
  const int b = n / B;
  return dist_slot_position(B, nr, rank, l / b) * b + l % b;
}

// pair l (of n/(2 nr)) of step `step` on rank `rank`, as LOCAL columns (p, q)
// ordered as the global pair of strategy_pair (p the lower global column):
// phase I is flat RR inside every local block; in phase II the block pair of
// slots (2k, 2k+1) is (circle_player(B, r, i), circle_player(B, r, B-1-i)),
// i = rank per + k, and step t of the round pairs column j of the lower
// block with column (j + t) mod b of the higher.
__device__ __host__ __forceinline__ void dist_pair(int n, int B, int nr, int rank, int step, int l,
                                                   int& p, int& q) {
  const int b = n / B;
  if (step < b - 1) {
    const int slot = l / (b / 2), i = l - slot * (b / 2);
    const int x = circle_player(b, step, i), y = circle_player(b, step, b - 1 - i);
    p = slot * b + (x < y ? x : y);
    q = slot * b + (x < y ? y : x);
    return;
  }
  const int s2 = step - (b - 1), rr = s2 / b, tt = s2 - rr * b;
  const int k = l / b, j = l - k * b;
  const int i = rank * (B / 2 / nr) + k;
  const int u = circle_player(B, rr, i), v = circle_player(B, rr, B - 1 - i);
  const int lo = u < v ? 2 * k : 2 * k + 1, hi = u < v ? 2 * k + 1 : 2 * k;
  const int jt = j + tt;
  p = lo * b + j;
  q = hi * b + (jt >= b ? jt - b : jt);
}

}  // namespace jsvd
