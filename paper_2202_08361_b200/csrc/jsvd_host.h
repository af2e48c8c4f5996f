// jsvd_host.h -- internal host-side declarations of libjsvd.so
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/jsvd.h"

namespace jsvd {
extern std::atomic<int64_t> g_launches;
inline void note_launch(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
// JSVD_DEBUG=1 (api.cu): scan EVD inputs for Inf/NaN, synchronously
bool debug_enabled();
template <typename T>
jsvd_status debug_check_finite(int64_t r, const T* a, const T* b, const T* c, const T* d,
                               cudaStream_t st);
// the current device's SM count, queried once per device (0 on error)
int sm_count();
// batched.cu: the shape / dtype conditions of jsvd_gesvj_batched
bool gesvj_batched_args_ok(jsvd_dtype dt, int64_t m, int64_t n);
}  // namespace jsvd
