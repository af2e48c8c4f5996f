// gesvj.cu -- jsvd_gesvj: the one-sided Jacobi SVD driver (Alg 4.1,
// P:1518-1596) over the step kernel of step.cu.
//
//   line 1   max-norm (NaN -> inf) -> s0 (Eq. skn) -> G1 = 2^s0 G
//   line 2   V = I
//   lines 3-41  sweeps x (n-1) steps, one kernel launch per step; the rescale
//            check (Eq. skr) and the M-tilde / s bookkeeping run on the device
//            (3 rotating slots), so the host synchronises once per sweep to
//            read the transformation count T (8 bytes).
//   line 42  finalize: norms recomputed with the step's lane order (R#23),
//            U = G diag(2^-e_j / f_j), sigma_j = (e_j - s, f_j), sorted
//            non-increasingly (R#24), U and V permuted alike.
#include <cmath>
#include <cstring>

#include "jsvd_host.h"
#include "step_dev.cuh"
#include "step_params.h"

namespace jsvd {

cudaError_t launch_step(bool cplx, int64_t npairs, const StepParams& P, cudaStream_t st);
cudaError_t launch_colnorm(bool cplx, int64_t m, int64_t n, const double* G, int64_t ldg,
                           double* ce, double* cf, cudaStream_t st);
bool step_supported(bool cplx, int64_t m);
bool strategy_ok(int64_t n, int64_t B);

struct WsHeader {
  unsigned long long Mt[3];
  unsigned long long M0;
  unsigned long long t;
  int s[3];
  int pad;
};

// M0 = max |component| with NaN -> inf (order-independent max of the bits)
__global__ void maxnorm_kernel(int64_t rows, int64_t n, const double* G, int64_t ld,
                               unsigned long long* out) {
  __shared__ unsigned long long sm[32];
  unsigned long long mx = 0;
  const int64_t total = rows * n;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = k / rows, i = k % rows;
    const double y = fmin(fabs(G[j * ld + i]), static_cast<double>(INFINITY));  // NaN -> inf
    mx = max(mx, static_cast<unsigned long long>(__double_as_longlong(y)));
  }
#pragma unroll
  for (int o = 16; o >= 1; o /= 2) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) mx = max(mx, sm[w]);
    atomicMax(out, mx);
  }
}

// G <- 2^s0 G, V <- I, slot initialisation
__global__ void init_kernel(int64_t rows, int64_t n, double* G, int64_t ld, double* V,
                            int64_t vrows, int64_t ldv, int cplx, int s0, WsHeader* h) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t k = t0; k < rows * n; k += stride) {
    const int64_t j = k / rows, i = k % rows;
    G[j * ld + i] = scalbn_rn(G[j * ld + i], s0);
  }
  for (int64_t k = t0; k < vrows * n; k += stride) {
    const int64_t j = k / vrows, i = k % vrows;
    V[j * ldv + i] = (i == (cplx ? 2 * j : j)) ? 1.0 : 0.0;
  }
  if (t0 == 0) {
    const double m0 = __longlong_as_double(static_cast<long long>(h->M0));
    h->Mt[0] = static_cast<unsigned long long>(__double_as_longlong(scalbn_rn(m0, s0)));
    h->Mt[1] = 0;
    h->Mt[2] = 0;
    h->s[0] = s0;
  }
}

// sigma_j = (e_j - s, f_j); stable rank by (e desc, f desc, j asc) (R#24)
__global__ void sort_kernel(int64_t n, const double* ce, const double* cf, const int* s_slot,
                            int32_t* perm, double* sig, double* sig_e, double* sig_f) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int s = *s_slot;
  const double ej = isinf(ce[j]) ? ce[j] : ce[j] - s, fj = cf[j];
  int64_t rank = 0;
  for (int64_t k = 0; k < n; ++k) {
    const double ek = isinf(ce[k]) ? ce[k] : ce[k] - s, fk = cf[k];
    const bool before = (ek > ej) || (ek == ej && (fk > fj || (fk == fj && k < j)));
    rank += before ? 1 : 0;
  }
  perm[rank] = static_cast<int32_t>(j);
  if (sig_e) sig_e[rank] = ej;
  if (sig_f) sig_f[rank] = fj;
  if (sig) sig[rank] = isinf(ej) ? 0.0 : scalbn_rn(fj, static_cast<int>(fmax(fmin(ej, 1e5), -1e5)));
}

// U[:, r] = scalbn(G[:, perm r], -e) / f ; V[:, r] = V[:, perm r]  (into buffers)
__global__ void gather_kernel(int64_t rows, int64_t n, const double* G, int64_t ld,
                              const double* V, int64_t vrows, int64_t ldv, const int32_t* perm,
                              const double* ce, const double* cf, double* Ub, double* Vb) {
  const int64_t r = blockIdx.y;
  const int64_t j = perm[r];
  const double e = ce[j];
  const bool fin = !isinf(e);
  const Pow2 sc(fin ? -static_cast<int>(e) : 0);
  const Divisor d = make_divisor(cf[j]);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double g = G[j * ld + i];
    Ub[r * rows + i] = fin ? divide(sc(g), d) : g;
  }
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < vrows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    Vb[r * vrows + i] = V[j * ldv + i];
}

static int ilog2_floor(int64_t m) {
  int k = 0;
  while ((m >> (k + 1)) > 0) ++k;
  return k;
}

// floor(lg(omega/(2m))) (real) / floor(lg(omega/(4 m sqrt2))) (complex), exact (R#28)
static int Fm_of(bool cplx, int64_t m) {
  const int k = ilog2_floor(m);
  if (!cplx) return 1022 - k;
  const unsigned __int128 mm = static_cast<unsigned __int128>(m) * static_cast<unsigned __int128>(m);
  const unsigned __int128 th = static_cast<unsigned __int128>(1) << (2 * k + 1);
  return 1021 - k - (mm >= th ? 1 : 0);
}

static bool is_checkpoint(int64_t n, int64_t B, int64_t step) {
  const int64_t b = n / B;
  if (step == 0) return true;
  if (step < b - 1) return false;
  return ((step - (b - 1)) % b) == 0;
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct WsLayout {
  size_t hdr, ce, cf, perm, ub, vb, total;
};

static WsLayout layout(bool cplx, int64_t m, int64_t n) {
  const size_t w = cplx ? 2 : 1;
  WsLayout L;
  size_t o = 0;
  L.hdr = o;
  o = align_up(o + sizeof(WsHeader));
  L.ce = o;
  o = align_up(o + sizeof(double) * n);
  L.cf = o;
  o = align_up(o + sizeof(double) * n);
  L.perm = o;
  o = align_up(o + sizeof(int32_t) * n);
  L.ub = o;
  o = align_up(o + sizeof(double) * w * m * n);
  L.vb = o;
  o = align_up(o + sizeof(double) * w * n * n);
  L.total = o;
  return L;
}

}  // namespace jsvd

using namespace jsvd;

extern "C" jsvd_status jsvd_gesvj_workspace(jsvd_dtype dt, int64_t m, int64_t n, size_t* bytes) {
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < 1 || n < 1 || !bytes) return JSVD_EINVAL;
  *bytes = layout(dt == JSVD_C64, m, n).total;
  return JSVD_OK;
}

#define CK(x)                                  \
  do {                                         \
    if ((x) != cudaSuccess) return JSVD_ECUDA; \
  } while (0)

extern "C" jsvd_status jsvd_gesvj(jsvd_dtype dt, int64_t m, int64_t n, double* A, int64_t lda,
                                  double* V, int64_t ldv, double* sigma, double* sigma_e,
                                  double* sigma_f, int32_t nblocks, int32_t max_sweeps,
                                  int32_t* sweeps_done, int64_t* tps, void* work,
                                  size_t work_bytes, void* stream) {
  const bool cplx = dt == JSVD_C64;
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < n || n < 2 || (n & 1) || lda < m || ldv < n ||
      !A || !V || !work || max_sweeps < 0 || !strategy_ok(n, nblocks) ||
      !step_supported(cplx, m))
    return JSVD_EINVAL;
  if (cplx && ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(V) & 15)))
    return JSVD_EINVAL;
  const WsLayout WL = layout(cplx, m, n);
  if (work_bytes < WL.total) return JSVD_ENOMEM;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(work);
  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws + WL.hdr);
  double* ce = reinterpret_cast<double*>(ws + WL.ce);
  double* cf = reinterpret_cast<double*>(ws + WL.cf);
  int32_t* perm = reinterpret_cast<int32_t*>(ws + WL.perm);
  double* Ub = reinterpret_cast<double*>(ws + WL.ub);
  double* Vb = reinterpret_cast<double*>(ws + WL.vb);
  const int64_t w = cplx ? 2 : 1;
  const int64_t rows = w * m, vrows = w * n;

  CK(cudaMemsetAsync(hdr, 0, sizeof(WsHeader), st));
  // line 1: M-tilde_0
  maxnorm_kernel<<<592, 256, 0, st>>>(rows, n, A, w * lda, &hdr->M0);
  note_launch();
  CK(cudaGetLastError());
  unsigned long long m0b = 0;
  CK(cudaMemcpyAsync(&m0b, &hdr->M0, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double M0;
  std::memcpy(&M0, &m0b, 8);
  if (std::isinf(M0)) return JSVD_ENONFINITE;
  if (M0 == 0.0) return JSVD_ERANK;
  const int Fm = Fm_of(cplx, m);
  const int s0 = Fm - std::ilogb(M0) - 1;
  init_kernel<<<592, 256, 0, st>>>(rows, n, A, w * lda, V, vrows, w * ldv, cplx, s0, hdr);
  note_launch();
  CK(cudaGetLastError());

  StepParams P{};
  P.m = m;
  P.n = n;
  P.G = A;
  P.ldg = lda;
  P.V = V;
  P.ldv = ldv;
  P.pairs = nullptr;
  P.B = nblocks;
  P.tol = std::ldexp(std::sqrt(static_cast<double>(m)), -53);  // upsilon (Eq. tol)
  P.col_e = ce;
  P.col_f = cf;
  P.t_dev = &hdr->t;
  P.mmax = nullptr;
  P.Mt = hdr->Mt;
  P.s_slots = hdr->s;
  P.Fm = Fm;
  P.Kr = cplx ? 1020 : 1022;

  int64_t gstep = 0;
  int32_t C = 0;
  bool converged = false;
  for (C = 0; C < max_sweeps; ++C) {
    CK(cudaMemsetAsync(&hdr->t, 0, 8, st));
    for (int64_t k = 0; k < n - 1; ++k, ++gstep) {
      P.step = k;
      P.slot = static_cast<int>(gstep % 3);
      P.checkpoint = is_checkpoint(n, nblocks, k) ? 1 : 0;
      CK(launch_step(cplx, n / 2, P, st));
    }
    unsigned long long T = 0;
    CK(cudaMemcpyAsync(&T, &hdr->t, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (tps) tps[C] = static_cast<int64_t>(T);
    if (T == 0) {
      converged = true;
      ++C;
      break;
    }
  }
  if (sweeps_done) *sweeps_done = C;
  // finalize
  CK(launch_colnorm(cplx, m, n, A, lda, ce, cf, st));
  sort_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(
      n, ce, cf, &hdr->s[gstep % 3], perm, sigma, sigma_e, sigma_f);
  note_launch();
  CK(cudaGetLastError());
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((rows + 255) / 256, 64)),
            static_cast<unsigned>(n));
  gather_kernel<<<grid, 256, 0, st>>>(rows, n, A, w * lda, V, vrows, w * ldv, perm, ce, cf, Ub, Vb);
  note_launch();
  CK(cudaGetLastError());
  CK(cudaMemcpy2DAsync(A, sizeof(double) * w * lda, Ub, sizeof(double) * rows,
                       sizeof(double) * rows, n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpy2DAsync(V, sizeof(double) * w * ldv, Vb, sizeof(double) * vrows,
                       sizeof(double) * vrows, n, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  return converged ? JSVD_OK : JSVD_ENOCONV;
}
