// Shared host/device plumbing for the bt200 library: error state, launch
// accounting, dtype helpers.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/bt200.h"

namespace bt {

// thread-local last error message (bt_last_error)
void set_error(const char* fmt, ...);
const char* last_error();

// process-wide count of kernels launched by this library (bt_launch_count)
extern std::atomic<long long> g_launches;
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms();

inline cudaStream_t as_stream(bt_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch (PDL) is on unless BT_PDL=0: every kernel is
// launched with programmatic stream serialisation, runs its prologue
// (barrier init, TMEM alloc, descriptor / weight prefetch) while the previous
// kernel drains, and waits on griddepcontrol.wait before touching activations.
bool pdl_enabled();

// cudaLaunchKernelEx with the PDL attribute (and an optional cluster size).
template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster_x,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// bt_plan_sched buffer: int2 sched[bs] (sequences, longest first), then at
// sched_units_offset(bs) int nunits, int queue[2] (the MHA tile-list
// claim counter and finished-CTA count, zeroed here, reset by the MHA), pad; then int2 units[bs * ceil(mx/128)]
// (query-tile units {start row, qt << 20 | length}, longest sequences first).
// Then at sched_segs_offset(bs, mx) int nsegs (16 B) and int4 segs[2 *
// bs * ceil(mx/128)]: the MHA segment kernel's work items, two int4 each:
// {first key row, key end row, first query row, query end row}, {first
// sequence, last sequence, -, -} (written for bs <= 256, mx <= 256).
constexpr int SEG_MAX_BS = 256, SEG_MAX_MX = 256;
inline size_t sched_units_offset(int bs) { return (static_cast<size_t>(bs) * 8 + 15) / 16 * 16; }
inline size_t sched_segs_offset(int bs, int mx) {
  return sched_units_offset(bs) + 16 + (static_cast<size_t>(bs) * ((mx + 127) / 128) * 8 + 15) / 16 * 16;
}
inline size_t sched_bytes(int bs, int mx) {
  return sched_segs_offset(bs, mx) + 16 + static_cast<size_t>(bs) * ((mx + 127) / 128) * 32;
}
}  // namespace bt

// Validate a condition on the host before any launch; returns `code`.
#define BT_REQUIRE(cond, code, ...)     \
  do {                                  \
    if (!(cond)) {                      \
      ::bt::set_error(__VA_ARGS__);     \
      return (code);                    \
    }                                   \
  } while (0)

#define BT_CUDA_CHECK(expr)                                                                      \
  do {                                                                                           \
    cudaError_t _e = (expr);                                                                     \
    if (_e != cudaSuccess) {                                                                     \
      ::bt::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
      return BT_ECUDA;                                                                           \
    }                                                                                            \
  } while (0)

// After a <<<>>> launch: record it and surface launch-configuration errors.
#define BT_LAUNCH_CHECK()                                                                          \
  do {                                                                                             \
    ::bt::count_launch();                                                                          \
    cudaError_t _e = cudaGetLastError();                                                           \
    if (_e != cudaSuccess) {                                                                       \
      ::bt::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), __FILE__, __LINE__); \
      return BT_ECUDA;                                                                             \
    }                                                                                              \
  } while (0)

// Launch through bt::launch (PDL attribute), record it, surface errors.
#define BT_LAUNCH(kern, grid, block, smem, stream, cluster, ...)                                        \
  do {                                                                                                 \
    cudaError_t _le = ::bt::launch(kern, grid, block, smem, stream, cluster, __VA_ARGS__);             \
    if (_le != cudaSuccess) {                                                                          \
      ::bt::set_error("launch of %s failed: %s (%s:%d)", #kern, cudaGetErrorString(_le), __FILE__, __LINE__); \
      return BT_ECUDA;                                                                                 \
    }                                                                                                  \
    ::bt::count_launch();                                                                              \
  } while (0)

#define BT_TRY(expr)          \
  do {                        \
    int _rc = (expr);         \
    if (_rc != BT_OK) return _rc; \
  } while (0)
