// Microbenchmark + self-check of the bitsliced lo-chain scan (phase 1 of the
// two-phase simplehash path) against the serial lo chain, on one big entry.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o loscan loscan.cu
//   ./loscan [MiB]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cudaTypedefs.h>

#include "../../paper_2505_14065_b200/csrc/loscan.cuh"

__global__ void __launch_bounds__(pcclb::kLsThreads, 1)
    loscan_kernel(const __grid_constant__ CUtensorMap map, const uint8_t *ptr, uint64_t rounds, uint64_t *fin) {
  extern __shared__ __align__(1024) uint8_t smem[];
  auto *sh = reinterpret_cast<pcclb::LsShared *>(smem + pcclb::kLsStageBytes * pcclb::kLsStages);
  const uint32_t lane0 = blockIdx.x * pcclb::kLsLanes;
  pcclb::loscan_cta(&map, ptr, rounds, lane0, smem, sh);
  if (threadIdx.x < pcclb::kLsLanes)
    fin[lane0 + threadIdx.x] = ((uint64_t)sh->final_hi[threadIdx.x] << 32) | sh->final_lo[threadIdx.x];
}

static bool encode4d(CUtensorMap *m, const void *p, uint64_t rounds) {
  void *fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q) != cudaSuccess) return false;
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  cuuint64_t dims[4] = {256, 32, 32, rounds >> 10};
  cuuint64_t strides[3] = {32768, 1024, 1u << 20};
  cuuint32_t box[4] = {pcclb::kLsLanes, 32, 32, pcclb::kLsWarps};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<void *>(p), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return r == CUDA_SUCCESS;
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__global__ void fill(uint32_t *p, uint64_t n, uint32_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 15; x *= 0x2c1b3c6du; x ^= x >> 12; x *= 0x297a2d39u; x ^= x >> 15;
    p[i] = x;
  }
}

// serial reference: one thread per lane, the full FNV-1a-64 chain
__global__ void serial_fnv(const uint32_t *p, uint64_t rounds, uint64_t *fin) {
  const uint32_t lane = threadIdx.x + blockIdx.x * blockDim.x;
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t r = 0; r < rounds; ++r) h = (h ^ p[r * 256 + lane]) * 0x100000001b3ull;
  fin[lane] = h;
}

int main(int argc, char **argv) {
  const uint64_t mib = argc > 1 ? strtoull(argv[1], 0, 10) : 1002;
  const uint64_t extra = argc > 2 ? strtoull(argv[2], 0, 10) : 0;  // extra rows past whole MiB
  const uint64_t rounds = mib * 1024 + extra;
  const uint64_t words = rounds * 256;
  uint32_t *d;
  uint64_t *fin0, *fin1;
  CK(cudaMalloc(&d, words * 4 + 4));
  CK(cudaMalloc(&fin0, 256 * 8));
  CK(cudaMalloc(&fin1, 256 * 8));
  fill<<<1184, 512>>>(d, words, 12345u);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  serial_fnv<<<8, 32>>>(d, rounds, fin0);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms0;
  cudaEventElapsedTime(&ms0, a, b);
  CUtensorMap map;
  if ((rounds >> 10) && !encode4d(&map, d, rounds)) return 2;
  CK(cudaFuncSetAttribute(loscan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pcclb::kLsSmem));
  float best = 1e9;
  for (int it = 0; it < 5; ++it) {
    CK(cudaMemset(fin1, 0xff, 256 * 8));
    cudaEventRecord(a);
    loscan_kernel<<<256 / pcclb::kLsLanes, pcclb::kLsThreads, pcclb::kLsSmem>>>(
        map, reinterpret_cast<const uint8_t *>(d), rounds, fin1);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  std::vector<uint64_t> f0(256), f1(256);
  CK(cudaMemcpy(f0.data(), fin0, 2048, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(f1.data(), fin1, 2048, cudaMemcpyDeviceToHost));
  uint64_t bad = 0;
  for (int i = 0; i < 256; ++i) bad += f0[i] != f1[i];
  printf("rows=%llu serial %.3f ms  bitsliced %.3f ms (%.1f GB/s)  mismatches=%llu\n",
         (unsigned long long)rounds, ms0, best, words * 4 / best / 1e6, (unsigned long long)bad);
  return bad ? 1 : 0;
}
