// host_pipe.cu -- the C-ABI entry points on HOST buffers: the batched EVD and
// the batched SVD streamed through the GPU in chunks.  Chunk i uploads,
// computes and downloads on internal stream i mod 3, so the upload of chunk
// i+1 and the download of chunk i-1 overlap the kernel of chunk i (separate
// copy engines for each direction).  The device buffers of the three slots
// live in a caller-provided workspace (no allocation on the path); the
// internal streams and events are created once per device.  Results are the
// device entry points' (the same kernels on the same data), bit for bit.
#include <mutex>

#include "jsvd_host.h"

namespace jsvd {
namespace {

constexpr int kSlots = 3;

struct PipeStreams {
  int dev = -1;
  cudaStream_t s[kSlots] = {};
  cudaEvent_t e[kSlots + 1] = {};
};

constexpr int kMaxDevices = 64;
std::mutex g_pipe_mu;
PipeStreams g_pipes[kMaxDevices];  // per device, created once, never moved

// the internal streams / events of the current device (created once).  Calls
// from several host threads on one device share them: every cross-stream edge
// is captured when it is enqueued, so interleaved calls can only over-order.
cudaError_t pipe_streams(PipeStreams** out) {
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> g(g_pipe_mu);
  PipeStreams& p = g_pipes[dev];
  if (p.dev != dev) {
    for (int k = 0; k < kSlots; ++k) {
      if ((err = cudaStreamCreateWithFlags(&p.s[k], cudaStreamNonBlocking)) != cudaSuccess) return err;
    }
    for (int k = 0; k <= kSlots; ++k) {
      if ((err = cudaEventCreateWithFlags(&p.e[k], cudaEventDisableTiming)) != cudaSuccess) return err;
    }
    p.dev = dev;
  }
  *out = &p;
  return cudaSuccess;
}

// internal streams wait for the caller's stream; at the end the caller's
// stream waits for them.  The shared fork event is recorded and waited on
// under the lock, so a second host thread cannot re-record it between this
// call's record and its waits (which would order this call's uploads after
// the other caller's stream instead of its own).  join's per-stream events
// are recorded and waited under the lock too; interleaving there could only
// over-order, but the lock keeps each edge exactly the call's own.
cudaError_t fork(PipeStreams* p, cudaStream_t caller) {
  std::lock_guard<std::mutex> g(g_pipe_mu);
  cudaError_t e = cudaEventRecord(p->e[kSlots], caller);
  for (int k = 0; k < kSlots && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(p->s[k], p->e[kSlots], 0);
  return e;
}
cudaError_t join(PipeStreams* p, cudaStream_t caller) {
  std::lock_guard<std::mutex> g(g_pipe_mu);
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < kSlots && e == cudaSuccess; ++k) {
    e = cudaEventRecord(p->e[k], p->s[k]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(caller, p->e[k], 0);
  }
  return e;
}

// an error after fork(): the caller's stream still waits for everything the
// call already queued on the internal streams (e.g. an upload reading the
// caller's host buffer), so synchronising `stream` stays a sufficient fence
jsvd_status fail_joined(PipeStreams* p, cudaStream_t caller, jsvd_status st) {
  join(p, caller);
  return st;
}

inline size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

size_t evd_slot_bytes(bool cplx, size_t w, int64_t chunk) {
  const size_t v = align256(w * static_cast<size_t>(chunk));
  return (cplx ? 9 : 7) * v + align256(4 * static_cast<size_t>(chunk)) +
         align256(4 * static_cast<size_t>((chunk + 31) / 32));
}

size_t svd_slot_bytes(bool cplx, int64_t m, int64_t n, int64_t chunk) {
  const size_t w = cplx ? 16 : 8;
  return align256(w * m * n * chunk) + align256(w * n * n * chunk) + align256(8 * n * chunk) +
         3 * align256(8 * chunk);
}

}  // namespace
}  // namespace jsvd

using namespace jsvd;

extern "C" jsvd_status jsvd_evd2_host_workspace(jsvd_dtype dt, int64_t chunk, size_t* bytes) {
  if (!bytes || chunk < 32 || (chunk % 32) || dt < JSVD_R64 || dt > JSVD_C32) return JSVD_EINVAL;
  const bool cplx = dt == JSVD_C64 || dt == JSVD_C32;
  const size_t w = (dt == JSVD_R64 || dt == JSVD_C64) ? 8 : 4;
  *bytes = kSlots * evd_slot_bytes(cplx, w, chunk);
  return JSVD_OK;
}

extern "C" jsvd_status jsvd_evd2_batched_host(jsvd_dtype dt, int64_t r, const void* a11,
                                              const void* a22, const void* a21_re,
                                              const void* a21_im, void* lam1, void* lam2,
                                              void* cos_phi, void* sin_re, void* sin_im,
                                              int32_t* zeta, uint32_t* perm, uint32_t flags,
                                              int64_t chunk, void* work, size_t work_bytes,
                                              void* stream) {
  if (r < 0 || chunk < 32 || (chunk % 32) || dt < JSVD_R64 || dt > JSVD_C32) return JSVD_EINVAL;
  const bool cplx = dt == JSVD_C64 || dt == JSVD_C32;
  const bool f64 = dt == JSVD_R64 || dt == JSVD_C64;
  const size_t w = f64 ? 8 : 4;
  if (!a11 || !a22 || !a21_re || !lam1 || !lam2 || !cos_phi || !sin_re) return JSVD_EINVAL;
  if (cplx != (a21_im != nullptr) || cplx != (sin_im != nullptr)) return JSVD_EINVAL;
  if (flags & ~(JSVD_EVD_TAN | JSVD_EVD_NOBACKSCALE)) return JSVD_EINVAL;
  if (r == 0) return JSVD_OK;
  const size_t slot = evd_slot_bytes(cplx, w, chunk);
  if (!work || work_bytes < kSlots * slot) return JSVD_ENOMEM;
  PipeStreams* p = nullptr;
  if (pipe_streams(&p) != cudaSuccess) return JSVD_ECUDA;
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  if (fork(p, caller) != cudaSuccess) return JSVD_ECUDA;
  const void* in[4] = {a11, a22, a21_re, a21_im};
  void* out[5] = {lam1, lam2, cos_phi, sin_re, sin_im};
  const int nin = cplx ? 4 : 3, nout = cplx ? 5 : 4;
  const size_t v = align256(w * static_cast<size_t>(chunk));
  const int64_t nchunks = (r + chunk - 1) / chunk;
  for (int64_t i = 0; i < nchunks; ++i) {
    const int k = static_cast<int>(i % kSlots);
    cudaStream_t s = p->s[k];
    char* base = static_cast<char*>(work) + k * slot;
    const int64_t off = i * chunk, n = (r - off < chunk) ? r - off : chunk;
    const size_t nb = w * static_cast<size_t>(n);
    char* din[4];
    char* dout[5];
    for (int j = 0; j < 4; ++j) din[j] = base + j * v;
    for (int j = 0; j < 5; ++j) dout[j] = base + (nin + j) * v;
    int32_t* dz = reinterpret_cast<int32_t*>(base + (nin + nout) * v);
    uint32_t* dp = reinterpret_cast<uint32_t*>(base + (nin + nout) * v + align256(4 * chunk));
    for (int j = 0; j < nin; ++j)
      if (cudaMemcpyAsync(din[j], static_cast<const char*>(in[j]) + w * off, nb,
                          cudaMemcpyHostToDevice, s) != cudaSuccess)
        return fail_joined(p, caller, JSVD_ECUDA);
    jsvd_status st;
    if (f64)
      st = jsvd_evd2_batched(dt, n, reinterpret_cast<const double*>(din[0]),
                             reinterpret_cast<const double*>(din[1]),
                             reinterpret_cast<const double*>(din[2]),
                             cplx ? reinterpret_cast<const double*>(din[3]) : nullptr,
                             reinterpret_cast<double*>(dout[0]), reinterpret_cast<double*>(dout[1]),
                             reinterpret_cast<double*>(dout[2]), reinterpret_cast<double*>(dout[3]),
                             cplx ? reinterpret_cast<double*>(dout[4]) : nullptr,
                             zeta ? dz : nullptr, perm ? dp : nullptr, flags, s);
    else
      st = jsvd_evd2_batched_f32(dt, n, reinterpret_cast<const float*>(din[0]),
                                 reinterpret_cast<const float*>(din[1]),
                                 reinterpret_cast<const float*>(din[2]),
                                 cplx ? reinterpret_cast<const float*>(din[3]) : nullptr,
                                 reinterpret_cast<float*>(dout[0]), reinterpret_cast<float*>(dout[1]),
                                 reinterpret_cast<float*>(dout[2]), reinterpret_cast<float*>(dout[3]),
                                 cplx ? reinterpret_cast<float*>(dout[4]) : nullptr,
                                 zeta ? dz : nullptr, perm ? dp : nullptr, flags, s);
    if (st != JSVD_OK) return fail_joined(p, caller, st);
    for (int j = 0; j < nout; ++j)
      if (cudaMemcpyAsync(static_cast<char*>(out[j]) + w * off, dout[j], nb,
                          cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return fail_joined(p, caller, JSVD_ECUDA);
    if (zeta && cudaMemcpyAsync(zeta + off, dz, 4 * n, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return fail_joined(p, caller, JSVD_ECUDA);
    if (perm && cudaMemcpyAsync(perm + off / 32, dp, 4 * ((n + 31) / 32), cudaMemcpyDeviceToHost,
                                s) != cudaSuccess)
      return fail_joined(p, caller, JSVD_ECUDA);
  }
  return join(p, caller) == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}

extern "C" jsvd_status jsvd_gesvj_batched_host_workspace(jsvd_dtype dt, int64_t m, int64_t n,
                                                         int64_t chunk, size_t* bytes) {
  if (!bytes || chunk < 1 || !gesvj_batched_args_ok(dt, m, n)) return JSVD_EINVAL;
  *bytes = kSlots * svd_slot_bytes(dt == JSVD_C64, m, n, chunk);
  return JSVD_OK;
}

extern "C" jsvd_status jsvd_gesvj_batched_host(jsvd_dtype dt, int64_t batch, int64_t m, int64_t n,
                                               const double* A, double* U, double* V,
                                               double* sigma, int32_t max_sweeps,
                                               int32_t* sweeps_done, int32_t* status,
                                               int64_t* transforms, int64_t chunk, void* work,
                                               size_t work_bytes, void* stream) {
  if (batch < 0 || chunk < 1 || !A || !U || !V || !sigma || max_sweeps < 0 ||
      !gesvj_batched_args_ok(dt, m, n))
    return JSVD_EINVAL;  // everything jsvd_gesvj_batched checks, before fork()
  if (batch == 0) return JSVD_OK;
  const bool cplx = dt == JSVD_C64;
  const size_t w = cplx ? 16 : 8;
  const size_t slot = svd_slot_bytes(cplx, m, n, chunk);
  if (!work || work_bytes < kSlots * slot) return JSVD_ENOMEM;
  PipeStreams* p = nullptr;
  if (pipe_streams(&p) != cudaSuccess) return JSVD_ECUDA;
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  if (fork(p, caller) != cudaSuccess) return JSVD_ECUDA;
  const int64_t nchunks = (batch + chunk - 1) / chunk;
  for (int64_t i = 0; i < nchunks; ++i) {
    const int k = static_cast<int>(i % kSlots);
    cudaStream_t s = p->s[k];
    char* base = static_cast<char*>(work) + k * slot;
    const int64_t off = i * chunk, nb = (batch - off < chunk) ? batch - off : chunk;
    double* dA = reinterpret_cast<double*>(base);
    double* dV = reinterpret_cast<double*>(base + align256(w * m * n * chunk));
    double* ds = reinterpret_cast<double*>(base + align256(w * m * n * chunk) + align256(w * n * n * chunk));
    char* tail = base + align256(w * m * n * chunk) + align256(w * n * n * chunk) + align256(8 * n * chunk);
    int32_t* dsw = reinterpret_cast<int32_t*>(tail);
    int32_t* dst = reinterpret_cast<int32_t*>(tail + align256(8 * chunk));
    int64_t* dtr = reinterpret_cast<int64_t*>(tail + 2 * align256(8 * chunk));
    if (cudaMemcpyAsync(dA, reinterpret_cast<const char*>(A) + w * m * n * off, w * m * n * nb,
                        cudaMemcpyHostToDevice, s) != cudaSuccess)
      return fail_joined(p, caller, JSVD_ECUDA);
    const jsvd_status st = jsvd_gesvj_batched(dt, nb, m, n, dA, m, m * n, dV, n, n * n, ds,
                                              max_sweeps, dsw, dst, dtr, nullptr, nullptr, s);
    if (st != JSVD_OK) return fail_joined(p, caller, st);
    if (cudaMemcpyAsync(reinterpret_cast<char*>(U) + w * m * n * off, dA, w * m * n * nb,
                        cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(reinterpret_cast<char*>(V) + w * n * n * off, dV, w * n * n * nb,
                        cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(sigma + n * off, ds, 8 * n * nb, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return fail_joined(p, caller, JSVD_ECUDA);
    if (sweeps_done && cudaMemcpyAsync(sweeps_done + off, dsw, 4 * nb, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return fail_joined(p, caller, JSVD_ECUDA);
    if (status && cudaMemcpyAsync(status + off, dst, 4 * nb, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return fail_joined(p, caller, JSVD_ECUDA);
    if (transforms && cudaMemcpyAsync(transforms + off, dtr, 8 * nb, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return fail_joined(p, caller, JSVD_ECUDA);
  }
  return join(p, caller) == cudaSuccess ? JSVD_OK : JSVD_ECUDA;
}

// ---- the full SVD on host buffers: upload, jsvd_gesvj, download ------------
namespace {
jsvd_status gesvj_host_parts(bool cplx, int64_t m, int64_t n, int32_t nblocks, size_t* own,
                             size_t* ws) {
  const size_t w = cplx ? 16 : 8;
  const jsvd_status st = jsvd_gesvj_workspace(cplx ? JSVD_C64 : JSVD_R64, m, n, nblocks, nullptr, ws);
  *own = align256(w * m * n) + align256(w * n * n) + align256(8 * n);
  return st;
}
}  // namespace

extern "C" jsvd_status jsvd_gesvj_host_workspace(jsvd_dtype dt, int64_t m, int64_t n,
                                                 int32_t nblocks, size_t* bytes) {
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < 1 || n < 1 || !bytes) return JSVD_EINVAL;
  size_t ws = 0, own = 0;
  const jsvd_status st = gesvj_host_parts(dt == JSVD_C64, m, n, nblocks, &own, &ws);
  if (st != JSVD_OK) return st;
  *bytes = own + ws;
  return JSVD_OK;
}

extern "C" jsvd_status jsvd_gesvj_host(jsvd_dtype dt, int64_t m, int64_t n, const double* A,
                                       int64_t lda, double* U, double* V, double* sigma,
                                       int32_t nblocks, int32_t max_sweeps, int32_t* sweeps_done,
                                       int64_t* transforms_per_sweep, int32_t* scale, void* work,
                                       size_t work_bytes, void* stream) {
  if ((dt != JSVD_R64 && dt != JSVD_C64) || m < 1 || n < 1 || lda < m || !A || !U || !V ||
      !sigma || !work)
    return JSVD_EINVAL;
  const bool cplx = dt == JSVD_C64;
  const size_t w = cplx ? 16 : 8;
  size_t ws = 0, own = 0;
  const jsvd_status q = gesvj_host_parts(cplx, m, n, nblocks, &own, &ws);
  if (q != JSVD_OK) return q;
  if (work_bytes < own + ws) return JSVD_ENOMEM;
  char* base = static_cast<char*>(work);
  double* dA = reinterpret_cast<double*>(base);
  double* dV = reinterpret_cast<double*>(base + align256(w * m * n));
  double* ds = reinterpret_cast<double*>(base + align256(w * m * n) + align256(w * n * n));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // A (ld = lda on the host) -> packed m x n on the device
  if (cudaMemcpy2DAsync(dA, w * m, A, w * lda, w * m, n, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return JSVD_ECUDA;
  const jsvd_status s = jsvd_gesvj(dt, m, n, dA, m, dV, n, ds, nullptr, nullptr, nullptr, nblocks,
                                   max_sweeps, sweeps_done, transforms_per_sweep, scale, nullptr,
                                   base + own, ws, nullptr, stream);
  if (s != JSVD_OK && s != JSVD_ENOCONV) return s;
  if (cudaMemcpyAsync(U, dA, w * m * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(V, dV, w * n * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(sigma, ds, 8 * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return JSVD_ECUDA;
  return s;
}
