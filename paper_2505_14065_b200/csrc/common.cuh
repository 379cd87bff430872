// Shared host/device plumbing for libpcclb200.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pcclb200.h"

namespace pcclb {

// last CUDA error seen on this host thread (exported via pcclb_last_cuda_error)
extern thread_local int g_last_cuda_error;

inline int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return PCCLB_OK;
  g_last_cuda_error = (int)e;
  return PCCLB_ECUDA;
}

#define PCCLB_CUDA(expr)                                   \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return ::pcclb::cuda_status(_e); \
  } while (0)

#define PCCLB_LAUNCH_CHECK() PCCLB_CUDA(cudaGetLastError())

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// number of SMs of the current device (cached per device)
int sm_count();

// grid for a grid-stride elementwise kernel: enough CTAs to cover `work`
// items of `per_cta` each, capped at `ctas_per_sm` waves of the SM count.
inline unsigned grid_for(uint64_t work, uint64_t per_cta, int ctas_per_sm = 8) {
  uint64_t need = (work + per_cta - 1) / per_cta;
  uint64_t cap = (uint64_t)sm_count() * (uint64_t)ctas_per_sm;
  if (need > cap) need = cap;
  if (need < 1) need = 1;
  return (unsigned)need;
}

inline bool valid_dtype(int dt) { return dt == PCCLB_F32 || dt == PCCLB_F64 || dt == PCCLB_BF16; }
inline bool valid_op(int op) { return op >= PCCLB_SUM && op <= PCCLB_PROD; }
inline size_t dtype_size(int dt) { return dt == PCCLB_F64 ? 8 : dt == PCCLB_BF16 ? 2 : 4; }

}  // namespace pcclb
