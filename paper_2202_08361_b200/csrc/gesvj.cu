// gesvj.cu -- jsvd_gesvj: the one-sided Jacobi SVD driver (Alg 4.1,
// P:1518-1596) over the step kernel of step.cu, on one GPU or sharded by
// column blocks over several.
//
//   line 1   max-norm (NaN -> inf) -> s0 (Eq. skn) -> G1 = 2^s0 G
//            (sharded: all-reduce max of the local max-norms)
//   line 2   V = I
//   lines 3-41  sweeps x (n-1) steps, one kernel launch per step; the rescale
//            check (Eq. skr) and the M-tilde / s bookkeeping run on the device
//            (3 rotating slots), so the host synchronises once per sweep to
//            read the transformation count T (8 bytes).  Sharded: the pairs
//            of a step are this rank's (dist_pair), M-tilde is all-reduced
//            (max) before every check point, blocks move between ranks after
//            every phase-II round (send/recv), T is all-reduced (sum).
//   line 41  converged: norms recomputed with the step's lane order (R#23),
//            U = G diag(2^-e_j / f_j), sigma_j = (e_j - s, f_j), sorted
//            non-increasingly (R#24); not converged (C = S): G = U Sigma' and
//            Sigma' are returned as they are (R#25).
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <utility>
#include <vector>

#include "jsvd_host.h"
#include "step_dev.cuh"
#include "step_params.h"

namespace jsvd {

cudaError_t launch_step(bool cplx, int64_t npairs, const StepParams& P, cudaStream_t st);
cudaError_t launch_colnorm(bool cplx, int64_t m, int64_t n, const double* G, int64_t ldg,
                           double* ce, double* cf, cudaStream_t st);
bool step_supported(bool cplx, int64_t m);
bool strategy_ok(int64_t n, int64_t B);
bool step_fast_enabled();

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

// G <- 2^s0 G, V <- I (local column l is global column gcol(l): the sharded
// ordering's slots, or l itself), slot initialisation
struct ColMap {
  int n, B, nr, rank;  // nr == 0: identity
  __device__ int operator()(int l) const { return nr ? dist_gcol(n, B, nr, rank, l) : l; }
};

__global__ void init_kernel(int64_t rows, int64_t ncols, double* G, int64_t ld, double* V,
                            int64_t vrows, int64_t ldv, int cplx, int s0, ColMap cm,
                            WsHeader* h) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t k = t0; k < rows * ncols; k += stride) {
    const int64_t j = k / rows, i = k % rows;
    G[j * ld + i] = scalbn_rn(G[j * ld + i], s0);
  }
  for (int64_t k = t0; k < vrows * ncols; k += stride) {
    const int64_t j = k / vrows, i = k % vrows;
    const int64_t g = cm(static_cast<int>(j));
    V[j * ldv + i] = (i == (cplx ? 2 * g : g)) ? 1.0 : 0.0;
  }
  if (t0 == 0) {
    const double m0 = __longlong_as_double(static_cast<long long>(h->M0));
    h->Mt[0] = static_cast<unsigned long long>(__double_as_longlong(scalbn_rn(m0, s0)));
    h->Mt[1] = 0;
    h->Mt[2] = 0;
    h->s[0] = s0;
  }
}

// keys of the final sort: (e_j - s, f_j, global column) of every local column
// (converged), or (e_j, f_j, column) for Sigma' (not converged)
__global__ void keys_kernel(int64_t nl, const double* ce, const double* cf, const int* s_slot,
                            int backscale, ColMap cm, double* keys) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nl) return;
  const double e = ce[l];
  keys[3 * l] = (backscale && !isinf(e)) ? e - *s_slot : e;
  keys[3 * l + 1] = cf[l];
  keys[3 * l + 2] = static_cast<double>(cm(static_cast<int>(l)));
}

__device__ __forceinline__ double sigma_of(double e, double f) {
  return isinf(e) ? 0.0 : scalbn_rn(f, static_cast<int>(fmax(fmin(e, 1e5), -1e5)));
}

// sorted = 1: stable rank by (e desc, f desc, column asc) (R#24) -> sigma,
// sigma_e, sigma_f, perm (global column of each rank) and, for the
// single-GPU path, the local column of each rank (loc).  sorted = 0: Sigma'
// in column order (ENOCONV), perm = identity.
__global__ void sigma_kernel(int64_t n, const double* keys, int sorted, double* sig,
                             double* sig_e, double* sig_f, int32_t* perm, int32_t* loc) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double ej = keys[3 * j], fj = keys[3 * j + 1], cj = keys[3 * j + 2];
  int64_t rank;
  if (sorted) {
    rank = 0;
    for (int64_t k = 0; k < n; ++k) {
      const double ek = keys[3 * k], fk = keys[3 * k + 1], ck = keys[3 * k + 2];
      const bool before = (ek > ej) || (ek == ej && (fk > fj || (fk == fj && ck < cj)));
      rank += before ? 1 : 0;
    }
  } else {
    rank = static_cast<int64_t>(cj);
  }
  if (perm) perm[rank] = sorted ? static_cast<int32_t>(cj) : static_cast<int32_t>(rank);
  if (loc) loc[rank] = static_cast<int32_t>(j);
  if (sig_e) sig_e[rank] = ej;
  if (sig_f) sig_f[rank] = fj;
  if (sig) sig[rank] = sigma_of(ej, fj);
}

// U[:, r] = scalbn(G[:, loc r], -e) / f ; V[:, r] = V[:, loc r]  (into buffers)
__global__ void gather_kernel(int64_t rows, int64_t n, const double* G, int64_t ld,
                              const double* V, int64_t vrows, int64_t ldv, const int32_t* loc,
                              const double* ce, const double* cf, double* Ub, double* Vb) {
  const int64_t r = blockIdx.y;
  const int64_t j = loc[r];
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

// u_j = 2^-e_j g_j / f_j in place (the sharded finalize: U stays distributed)
__global__ void normalize_kernel(int64_t rows, double* G, int64_t ld, const double* ce,
                                 const double* cf) {
  const int64_t j = blockIdx.y;
  const double e = ce[j];
  if (isinf(e)) return;  // zero column stays zero (R#19)
  const Pow2 sc(-static_cast<int>(e));
  const Divisor d = make_divisor(cf[j]);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    G[j * ld + i] = divide(sc(G[j * ld + i]), d);
}

// a rank's own block moves of one exchange in one launch: block k of the
// table goes from slot src[k] to slot dst[k] of G and of V (16-byte words)
struct LocalMoves {
  int n;
  int src[32], dst[32];
};
__global__ void local_moves_kernel(const double2* __restrict__ G, double2* __restrict__ G2,
                                   int64_t gw, const double2* __restrict__ V,
                                   double2* __restrict__ V2, int64_t vw, LocalMoves mv) {
  const int k = blockIdx.y;
  const int64_t s = mv.src[k], d = mv.dst[k];
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < gw + vw;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i < gw) G2[d * gw + i] = G[s * gw + i];
    else V2[d * vw + (i - gw)] = V[s * vw + (i - gw)];
  }
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

// the last step of a phase-II round: the blocks move after it
static bool is_round_end(int64_t n, int64_t B, int64_t step) {
  const int64_t b = n / B;
  return step >= b - 1 && ((step - (b - 1)) % b) == b - 1;
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct WsLayout {
  size_t hdr, ce, cf, keys, loc, ub, vb, g2, v2, total;
};

// single GPU: U/V staging of the final permutation; sharded: the second
// buffers of the block exchange (packed m x nl and n x nl)
static WsLayout layout(bool cplx, int64_t m, int64_t n, int64_t nl, bool dist) {
  const size_t w = cplx ? 2 : 1;
  WsLayout L{};
  size_t o = 0;
  L.hdr = o;
  o = align_up(o + sizeof(WsHeader));
  L.ce = o;
  o = align_up(o + sizeof(double) * nl);
  L.cf = o;
  o = align_up(o + sizeof(double) * nl);
  L.keys = o;
  o = align_up(o + 3 * sizeof(double) * n);
  L.loc = o;
  o = align_up(o + sizeof(int32_t) * n);
  if (!dist) {
    L.ub = o;
    o = align_up(o + sizeof(double) * w * m * n);
    L.vb = o;
    o = align_up(o + sizeof(double) * w * n * n);
  } else {
    L.g2 = o;
    o = align_up(o + sizeof(double) * w * m * nl);
    L.v2 = o;
    o = align_up(o + sizeof(double) * w * n * nl);
  }
  L.total = o;
  return L;
}

// ---------------------------------------------------------------- transport
// The collectives and block moves of the sharded driver: NCCL on `stream`
// (device buffers), or the host-staged callbacks of jsvd_transport.
class Comm {
 public:
  Comm(const jsvd_dist* d, cudaStream_t st) : d_(d), st_(st) {}
  ~Comm() {
    for (void* p : host_) cudaFreeHost(p);
  }
  bool nccl() const { return d_->nccl_comm != nullptr; }
  int rank() const { return d_->rank; }

  // in place over one 64-bit word on the device: op 0 max (u64), 1 sum (i64)
  jsvd_status allreduce(void* dev, int op) {
    // one rank: the local value is the global one (JSVD_DIST_SELF_P2P still
    // runs the NCCL collective, to exercise it on one GPU)
    if (d_->nranks == 1 && !(d_->flags & JSVD_DIST_SELF_P2P)) return JSVD_OK;
    if (nccl()) {
      ncclResult_t r = ncclAllReduce(dev, dev, 1, op == 0 ? ncclUint64 : ncclInt64,
                                     op == 0 ? ncclMax : ncclSum,
                                     static_cast<ncclComm_t>(d_->nccl_comm), st_);
      return r == ncclSuccess ? JSVD_OK : JSVD_ENCCL;
    }
    uint64_t v = 0;
    if (cudaMemcpyAsync(&v, dev, 8, cudaMemcpyDeviceToHost, st_) != cudaSuccess ||
        cudaStreamSynchronize(st_) != cudaSuccess)
      return JSVD_ECUDA;
    if (d_->xport->allreduce(d_->xport->ctx, &v, 1, op) != 0) return JSVD_ENCCL;
    if (cudaMemcpyAsync(dev, &v, 8, cudaMemcpyHostToDevice, st_) != cudaSuccess ||
        cudaStreamSynchronize(st_) != cudaSuccess)
      return JSVD_ECUDA;
    return JSVD_OK;
  }

  // recv (device, nranks * bytes) = every rank's send (device, bytes)
  jsvd_status allgather(const void* send, void* recv, size_t bytes, int nranks) {
    if (nranks == 1 && !(d_->flags & JSVD_DIST_SELF_P2P) && send == recv) return JSVD_OK;
    if (nccl()) {
      ncclResult_t r = ncclAllGather(send, recv, bytes, ncclUint8,
                                     static_cast<ncclComm_t>(d_->nccl_comm), st_);
      return r == ncclSuccess ? JSVD_OK : JSVD_ENCCL;
    }
    char* hs = static_cast<char*>(host(bytes * (nranks + 1)));
    if (!hs) return JSVD_ECUDA;
    char* hr = hs + bytes;
    if (cudaMemcpyAsync(hs, send, bytes, cudaMemcpyDeviceToHost, st_) != cudaSuccess ||
        cudaStreamSynchronize(st_) != cudaSuccess)
      return JSVD_ECUDA;
    if (d_->xport->allgather(d_->xport->ctx, hs, hr, static_cast<int64_t>(bytes)) != 0)
      return JSVD_ENCCL;
    if (cudaMemcpyAsync(recv, hr, bytes * nranks, cudaMemcpyHostToDevice, st_) != cudaSuccess ||
        cudaStreamSynchronize(st_) != cudaSuccess)
      return JSVD_ECUDA;
    return JSVD_OK;
  }

  struct Op {
    int peer, dir;  // dir 0 send, 1 receive
    char* buf;      // device
    size_t bytes;
  };
  // one group of point-to-point operations
  jsvd_status p2p(const std::vector<Op>& ops) {
    if (ops.empty()) return JSVD_OK;
    if (nccl()) {
      ncclComm_t c = static_cast<ncclComm_t>(d_->nccl_comm);
      if (ncclGroupStart() != ncclSuccess) return JSVD_ENCCL;
      ncclResult_t r = ncclSuccess;
      for (const Op& o : ops) {
        if (r != ncclSuccess) break;
        r = o.dir == 0 ? ncclSend(o.buf, o.bytes, ncclUint8, o.peer, c, st_)
                       : ncclRecv(o.buf, o.bytes, ncclUint8, o.peer, c, st_);
      }
      const ncclResult_t r2 = ncclGroupEnd();
      return (r == ncclSuccess && r2 == ncclSuccess) ? JSVD_OK : JSVD_ENCCL;
    }
    size_t tot = 0;
    for (const Op& o : ops) tot += align_up(o.bytes);
    char* h = static_cast<char*>(host(tot));
    if (!h) return JSVD_ECUDA;
    std::vector<int32_t> peer, dir;
    std::vector<void*> buf;
    std::vector<int64_t> nb;
    size_t off = 0;
    for (const Op& o : ops) {
      if (o.dir == 0 &&
          cudaMemcpyAsync(h + off, o.buf, o.bytes, cudaMemcpyDeviceToHost, st_) != cudaSuccess)
        return JSVD_ECUDA;
      peer.push_back(o.peer);
      dir.push_back(o.dir);
      buf.push_back(h + off);
      nb.push_back(static_cast<int64_t>(o.bytes));
      off += align_up(o.bytes);
    }
    if (cudaStreamSynchronize(st_) != cudaSuccess) return JSVD_ECUDA;
    if (d_->xport->sendrecv(d_->xport->ctx, static_cast<int32_t>(ops.size()), peer.data(),
                            dir.data(), buf.data(), nb.data()) != 0)
      return JSVD_ENCCL;
    off = 0;
    for (const Op& o : ops) {
      if (o.dir == 1 &&
          cudaMemcpyAsync(o.buf, h + off, o.bytes, cudaMemcpyHostToDevice, st_) != cudaSuccess)
        return JSVD_ECUDA;
      off += align_up(o.bytes);
    }
    return cudaStreamSynchronize(st_) == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
  }

 private:
  // pinned staging, grown on demand, freed with the call
  void* host(size_t bytes) {
    if (bytes <= host_cap_ && !host_.empty()) return host_.back();
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
    host_.push_back(p);
    host_cap_ = bytes;
    return p;
  }
  const jsvd_dist* d_;
  cudaStream_t st_;
  std::vector<void*> host_;
  size_t host_cap_ = 0;
};

static bool dist_ok(const jsvd_dist* d, int64_t n, int32_t B) {
  if (!d) return true;
  if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks) return false;
  if (!d->nccl_comm &&
      !(d->xport && d->xport->sendrecv && d->xport->allreduce && d->xport->allgather))
    return false;
  if (d->flags & ~JSVD_DIST_SELF_P2P) return false;
  if (!strategy_ok(n, B) || B >= n || B % 2 || (B / 2) % d->nranks) return false;
  if (d->nccl_comm) {
    int cnt = 0, me = 0;
    if (ncclCommCount(static_cast<ncclComm_t>(d->nccl_comm), &cnt) != ncclSuccess ||
        ncclCommUserRank(static_cast<ncclComm_t>(d->nccl_comm), &me) != ncclSuccess)
      return false;
    if (cnt != d->nranks || me != d->rank) return false;
  }
  return true;
}

}  // namespace jsvd

using namespace jsvd;

#define CK(x)                                  \
  do {                                         \
    if ((x) != cudaSuccess) return JSVD_ECUDA; \
  } while (0)
#define CS(x)                          \
  do {                                 \
    const jsvd_status s_ = (x);        \
    if (s_ != JSVD_OK) return s_;      \
  } while (0)

extern "C" jsvd_status jsvd_gesvj_workspace(jsvd_dtype dt, int64_t m, int64_t n, int32_t nblocks,
                                            const jsvd_dist* dist, size_t* bytes) {
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < 1 || n < 1 || !bytes) return JSVD_EINVAL;
  if (dist && (n < 2 || (n & 1) || !dist_ok(dist, n, nblocks))) return JSVD_EINVAL;
  const int64_t nl = dist ? n / dist->nranks : n;
  *bytes = layout(dt == JSVD_C64, m, n, nl, dist != nullptr).total;
  return JSVD_OK;
}

extern "C" jsvd_status jsvd_dist_columns(int64_t n, int32_t nblocks, int32_t rank,
                                         int32_t nranks, int32_t* cols) {
  jsvd_dist d{};
  d.nccl_comm = nullptr;
  d.rank = rank;
  d.nranks = nranks;
  static const jsvd_transport dummy{nullptr, [](void*, int32_t, const int32_t*, const int32_t*,
                                                void* const*, const int64_t*) { return 0; },
                                    [](void*, void*, int32_t, int32_t) { return 0; },
                                    [](void*, const void*, void*, int64_t) { return 0; }};
  d.xport = &dummy;
  if (!cols || !dist_ok(&d, n, nblocks)) return JSVD_EINVAL;
  for (int64_t l = 0; l < n / nranks; ++l)
    cols[l] = dist_gcol(static_cast<int>(n), nblocks, nranks, rank, static_cast<int>(l));
  return JSVD_OK;
}

extern "C" jsvd_status jsvd_dist_local_pairs(int64_t n, int32_t nblocks, int32_t rank,
                                             int32_t nranks, int64_t step, int32_t* pairs) {
  int32_t dummy = 0;
  if (!pairs || step < 0 || step >= n - 1 ||
      jsvd_dist_columns(n, nblocks, rank, nranks, n > 0 && nranks > 0 ? pairs : &dummy) !=
          JSVD_OK)
    return JSVD_EINVAL;
  for (int64_t l = 0; l < n / (2 * nranks); ++l) {
    int p, q;
    dist_pair(static_cast<int>(n), nblocks, nranks, rank, static_cast<int>(step),
              static_cast<int>(l), p, q);
    pairs[2 * l] = p;
    pairs[2 * l + 1] = q;
  }
  return JSVD_OK;
}

extern "C" jsvd_status jsvd_gesvj(jsvd_dtype dt, int64_t m, int64_t n, double* A, int64_t lda,
                                  double* V, int64_t ldv, double* sigma, double* sigma_e,
                                  double* sigma_f, int32_t* perm, int32_t nblocks,
                                  int32_t max_sweeps, int32_t* sweeps_done, int64_t* tps,
                                  int32_t* scale, const jsvd_gesvj_opts* opts, void* work,
                                  size_t work_bytes, const jsvd_dist* dist, void* stream) {
  const bool cplx = dt == JSVD_C64;
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < n || n < 2 || (n & 1) || lda < m || ldv < n ||
      !A || !V || !work || max_sweeps < 0 || !strategy_ok(n, nblocks) ||
      !step_supported(cplx, m) || !dist_ok(dist, n, nblocks))
    return JSVD_EINVAL;
  if (cplx && ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(V) & 15)))
    return JSVD_EINVAL;
  if (dist && (lda != m || ldv != n)) return JSVD_EINVAL;  // packed local blocks
  const int Fm = Fm_of(cplx, m);
  const int adj = opts ? opts->s0_adjust : 0;
  const int64_t max_steps = opts ? opts->max_steps : 0;
  if (max_steps < 0 || adj < -2200 || adj > 1024 - Fm) return JSVD_EINVAL;
  const int nr = dist ? dist->nranks : 1;
  const int64_t nl = n / nr;  // local columns
  const WsLayout WL = layout(cplx, m, n, nl, dist != nullptr);
  if (work_bytes < WL.total) return JSVD_ENOMEM;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(work);
  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws + WL.hdr);
  double* ce = reinterpret_cast<double*>(ws + WL.ce);
  double* cf = reinterpret_cast<double*>(ws + WL.cf);
  double* keys = reinterpret_cast<double*>(ws + WL.keys);
  int32_t* loc = reinterpret_cast<int32_t*>(ws + WL.loc);
  const int64_t w = cplx ? 2 : 1;
  const int64_t rows = w * m, vrows = w * n;
  Comm comm(dist, st);
  const ColMap cm{static_cast<int>(n), nblocks, dist ? nr : 0, dist ? dist->rank : 0};

  CK(cudaMemsetAsync(hdr, 0, sizeof(WsHeader), st));
  // line 1: M-tilde_0 (global)
  maxnorm_kernel<<<592, 256, 0, st>>>(rows, nl, A, w * lda, &hdr->M0);
  note_launch();
  CK(cudaGetLastError());
  if (dist) CS(comm.allreduce(&hdr->M0, 0));
  unsigned long long m0b = 0;
  CK(cudaMemcpyAsync(&m0b, &hdr->M0, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double M0;
  std::memcpy(&M0, &m0b, 8);
  if (std::isinf(M0)) return JSVD_ENONFINITE;
  if (M0 == 0.0) return JSVD_ERANK;
  const int s0 = Fm - std::ilogb(M0) - 1 + adj;
  init_kernel<<<592, 256, 0, st>>>(rows, nl, A, w * lda, V, vrows, w * ldv, cplx, s0, cm, hdr);
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
  P.dist_nr = dist ? nr : 0;
  P.dist_rank = dist ? dist->rank : 0;
  P.tol = std::ldexp(std::sqrt(static_cast<double>(m)), -53);  // upsilon (Eq. tol)
  P.col_e = ce;
  P.col_f = cf;
  P.t_dev = &hdr->t;
  P.mmax = nullptr;
  P.Mt = hdr->Mt;
  P.s_slots = hdr->s;
  P.Fm = Fm;
  P.Kr = cplx ? 1020 : 1022;
  P.fast = step_fast_enabled() ? 1 : 0;
  // col_e/col_f of the step are indexed by local column: sized nl

  // the block moves after a phase-II round (position k -> k-1, 1 -> B-1, 0
  // stays): this rank's outgoing (slot -> rank', slot') and incoming moves
  const int64_t b = n / nblocks;
  const size_t gblk = sizeof(double) * w * m * b, vblk = sizeof(double) * w * n * b;
  double* Gcur = A;
  double* Vcur = V;
  double* Galt = dist ? reinterpret_cast<double*>(ws + WL.g2) : nullptr;
  double* Valt = dist ? reinterpret_cast<double*>(ws + WL.v2) : nullptr;
  const bool self_p2p = dist && dist->nccl_comm && (dist->flags & JSVD_DIST_SELF_P2P);
  // Point-to-point operations between two ranks match in the order they are
  // posted, so both sides list them by the SOURCE circle position (G then V
  // per block): a rank sending several blocks to one peer -- only itself,
  // with JSVD_DIST_SELF_P2P -- then pairs every send with its receive.
  auto exchange = [&]() -> jsvd_status {
    const int nslots = static_cast<int>(nl / b);
    std::vector<std::pair<int, Comm::Op>> sends, recvs;
    LocalMoves mv{};
    for (int sl = 0; sl < nslots; ++sl) {  // outgoing
      const int pos = dist_slot_position(nblocks, nr, dist->rank, sl);
      const int dpos = pos == 0 ? 0 : (pos >= 2 ? pos - 1 : nblocks - 1);
      int dr, ds;
      dist_owner(nblocks, nr, dpos, dr, ds);
      char* gs = reinterpret_cast<char*>(Gcur) + sl * gblk;
      char* vs = reinterpret_cast<char*>(Vcur) + sl * vblk;
      if (dr == dist->rank && !self_p2p) {  // one kernel for all of them (below)
        mv.src[mv.n] = sl;
        mv.dst[mv.n] = ds;
        ++mv.n;
      } else {
        sends.push_back({2 * pos, {dr, 0, gs, gblk}});
        sends.push_back({2 * pos + 1, {dr, 0, vs, vblk}});
      }
    }
    for (int ds = 0; ds < nslots; ++ds) {  // incoming
      const int dpos = dist_slot_position(nblocks, nr, dist->rank, ds);
      const int spos = dpos == 0 ? 0 : (dpos == nblocks - 1 ? 1 : dpos + 1);
      int sr, ss;
      dist_owner(nblocks, nr, spos, sr, ss);
      if (sr == dist->rank && !self_p2p) continue;
      recvs.push_back({2 * spos, {sr, 1, reinterpret_cast<char*>(Galt) + ds * gblk, gblk}});
      recvs.push_back({2 * spos + 1, {sr, 1, reinterpret_cast<char*>(Valt) + ds * vblk, vblk}});
    }
    const auto by_pos = [](const std::pair<int, Comm::Op>& a, const std::pair<int, Comm::Op>& b) {
      return a.first < b.first;
    };
    std::sort(sends.begin(), sends.end(), by_pos);
    std::sort(recvs.begin(), recvs.end(), by_pos);
    std::vector<Comm::Op> ops;
    for (const auto& o : sends) ops.push_back(o.second);
    for (const auto& o : recvs) ops.push_back(o.second);
    if (mv.n) {
      const int64_t gw = static_cast<int64_t>(gblk / 16), vw = static_cast<int64_t>(vblk / 16);
      const unsigned bx = static_cast<unsigned>(std::min<int64_t>((gw + vw + 255) / 256, 512));
      local_moves_kernel<<<dim3(bx, mv.n), 256, 0, st>>>(
          reinterpret_cast<const double2*>(Gcur), reinterpret_cast<double2*>(Galt), gw,
          reinterpret_cast<const double2*>(Vcur), reinterpret_cast<double2*>(Valt), vw, mv);
      note_launch();
      CK(cudaGetLastError());
    }
    CS(comm.p2p(ops));
    std::swap(Gcur, Galt);
    std::swap(Vcur, Valt);
    P.G = Gcur;
    P.V = Vcur;
    return JSVD_OK;
  };

  int64_t gstep = 0;
  int32_t C = 0;
  bool converged = false, cut = false;
  for (C = 0; C < max_sweeps && !cut; ++C) {
    CK(cudaMemsetAsync(&hdr->t, 0, 8, st));
    for (int64_t k = 0; k < n - 1; ++k, ++gstep) {
      if (max_steps && gstep == max_steps) {  // opts.max_steps: stop here
        cut = true;
        break;
      }
      P.step = k;
      P.slot = static_cast<int>(gstep % 3);
      P.checkpoint = is_checkpoint(n, nblocks, k) ? 1 : 0;
      if (dist && P.checkpoint) CS(comm.allreduce(&hdr->Mt[P.slot], 0));  // global M-tilde
      CK(launch_step(cplx, nl / 2, P, st));
      if (dist && is_round_end(n, nblocks, k)) CS(exchange());
    }
    if (dist) CS(comm.allreduce(&hdr->t, 1));
    unsigned long long T = 0;
    CK(cudaMemcpyAsync(&T, &hdr->t, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (tps) tps[C] = static_cast<int64_t>(T);
    if (T == 0 && !cut) {
      converged = true;
      ++C;
      break;
    }
  }
  if (sweeps_done) *sweeps_done = C;
  if (cut) {  // a bounded run: no finalize, the iterate stays where it is
    if (scale) CK(cudaMemcpyAsync(scale, &hdr->s[gstep % 3], 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return JSVD_ENOCONV;
  }
  // every sweep returns each block to its round-0 slot; after an odd number
  // of exchanges the data sits in the second buffers
  if (dist && Gcur != A) {
    CK(cudaMemcpyAsync(A, Gcur, sizeof(double) * w * m * nl, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(V, Vcur, sizeof(double) * w * n * nl, cudaMemcpyDeviceToDevice, st));
  }
  const int* s_slot = &hdr->s[gstep % 3];
  if (scale) {
    CK(cudaMemcpyAsync(scale, s_slot, 4, cudaMemcpyDeviceToHost, st));
  }
  // line 41: the norms of the final iterate (R#23), then finalize if converged
  CK(launch_colnorm(cplx, m, nl, A, lda, ce, cf, st));
  const unsigned kb = static_cast<unsigned>((nl + 127) / 128);
  keys_kernel<<<kb, 128, 0, st>>>(nl, ce, cf, s_slot, converged ? 1 : 0, cm,
                                  keys + 3 * nl * (dist ? dist->rank : 0));
  note_launch();
  CK(cudaGetLastError());
  if (dist) CS(comm.allgather(keys + 3 * nl * dist->rank, keys, 3 * sizeof(double) * nl, nr));
  sigma_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(
      n, keys, converged ? 1 : 0, sigma, sigma_e, sigma_f, perm, dist ? nullptr : loc);
  note_launch();
  CK(cudaGetLastError());
  if (converged) {
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>((rows + 255) / 256, 64)),
                    static_cast<unsigned>(nl));
    if (dist) {  // U stays distributed: normalise in place
      normalize_kernel<<<grid, 256, 0, st>>>(rows, A, w * lda, ce, cf);
      note_launch();
      CK(cudaGetLastError());
    } else {  // U and V permuted into sigma's order
      double* Ub = reinterpret_cast<double*>(ws + WL.ub);
      double* Vb = reinterpret_cast<double*>(ws + WL.vb);
      gather_kernel<<<grid, 256, 0, st>>>(rows, n, A, w * lda, V, vrows, w * ldv, loc, ce, cf,
                                          Ub, Vb);
      note_launch();
      CK(cudaGetLastError());
      CK(cudaMemcpy2DAsync(A, sizeof(double) * w * lda, Ub, sizeof(double) * rows,
                           sizeof(double) * rows, n, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpy2DAsync(V, sizeof(double) * w * ldv, Vb, sizeof(double) * vrows,
                           sizeof(double) * vrows, n, cudaMemcpyDeviceToDevice, st));
    }
  }
  CK(cudaStreamSynchronize(st));
  return converged ? JSVD_OK : JSVD_ENOCONV;
}

extern "C" jsvd_status jsvd_nccl_unique_id(void* id128) {
  if (!id128) return JSVD_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return JSVD_ENCCL;
  std::memcpy(id128, &id, sizeof(id));
  return JSVD_OK;
}

extern "C" jsvd_status jsvd_nccl_comm_init(void** comm, int32_t nranks, const void* id128,
                                           int32_t rank) {
  if (!comm || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return JSVD_EINVAL;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  if (ncclCommInitRank(&c, nranks, id, rank) != ncclSuccess) return JSVD_ENCCL;
  *comm = c;
  return JSVD_OK;
}

extern "C" jsvd_status jsvd_nccl_comm_destroy(void* comm) {
  if (!comm) return JSVD_EINVAL;
  return ncclCommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? JSVD_OK : JSVD_ENCCL;
}
