// Host-side helpers shared by the engine's translation units (engine.cu,
// refresh.cu): error text for mecefo_last_error(), the launch counter, the
// CUDA-event launch profiler, per-device shared-memory opt-in and PDL
// launches. Implemented in engine.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "../../include/mecefo.h"

namespace mecefo_host {

int set_err(int code, const char* fmt, ...);
int check_launch(const char* what);
int64_t prof_begin(const char* tag, double flops, double bytes, cudaStream_t s);
void prof_end(int64_t idx, cudaStream_t s);
bool pdl_enabled();
int ensure_smem(const void* kern, int bytes);

#define CUDA_TRY(expr)                                                                                 \
  do {                                                                                                 \
    cudaError_t _e = (expr);                                                                           \
    if (_e != cudaSuccess)                                                                             \
      return ::mecefo_host::set_err(MECEFO_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                                    __FILE__, __LINE__);                                               \
  } while (0)

#define TRY(expr)                     \
  do {                                \
    int _rc = (expr);                 \
    if (_rc != MECEFO_OK) return _rc; \
  } while (0)

// CUDA events around a kernel (group) while the profiler is on; no-op otherwise.
struct ProfScope {
  int64_t idx;
  cudaStream_t s;
  ProfScope(const char* tag, double flops, double bytes, cudaStream_t st) : idx(prof_begin(tag, flops, bytes, st)), s(st) {}
  ~ProfScope() { prof_end(idx, s); }
};

// Every engine kernel goes out with programmatic stream serialization (PDL):
// it may be scheduled while its predecessor drains, runs its prologue
// (barrier init, TMEM alloc, descriptor prefetch) and blocks in
// griddepcontrol.wait until the predecessor's results are visible. Kept in
// CUDA-graph capture as programmatic edges. MECEFO_NO_PDL=1 disables it.
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace mecefo_host
