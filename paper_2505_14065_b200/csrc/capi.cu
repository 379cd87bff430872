// Host-only parts of the C ABI: status strings, chunk partition, device query.
#include <cuda_runtime.h>

#include <mutex>

#include "common.cuh"

namespace pcclb {

thread_local int g_last_cuda_error = 0;

int sm_count() {
  static std::mutex mu;
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

}  // namespace pcclb

extern "C" {

const char *pcclb_strerror(int status) {
  switch (status) {
    case PCCLB_OK:
      return "ok";
    case PCCLB_EINVAL:
      return "invalid argument";
    case PCCLB_ECUDA:
      return "CUDA error";
    case PCCLB_EABORTED:
      return "aborted";
    case PCCLB_ETIMEOUT:
      return "peer timeout";
    case PCCLB_ENONFINITE:
      return "non-finite values cannot be quantized";
    case PCCLB_EIO:
      return "local io failure";
    case PCCLB_ENOMEM:
      return "out of memory";
  }
  return "unknown status";
}

int pcclb_last_cuda_error(void) { return pcclb::g_last_cuda_error; }

const char *pcclb_version(void) { return "pcclb200 0.1 sm_100a"; }

// collective.py:86-101
int pcclb_chunk_bounds(uint64_t n, uint32_t w, uint64_t *out) {
  if (w < 1 || !out) return PCCLB_EINVAL;
  uint64_t base = n / w, extra = n % w, start = 0;
  for (uint32_t r = 0; r < w; ++r) {
    uint64_t size = base + (r < extra ? 1 : 0);
    out[2 * r] = start;
    out[2 * r + 1] = start + size;
    start += size;
  }
  return PCCLB_OK;
}

}  // extern "C"
