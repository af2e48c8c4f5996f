// jsvd_host.h -- internal host-side declarations of libjsvd.so
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/jsvd.h"

namespace jsvd {
extern std::atomic<int64_t> g_launches;
inline void note_launch(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
}  // namespace jsvd
