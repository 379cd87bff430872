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
    loscan_kernel(const __grid_constant__ CUtensorMap map, const uint8_t *ptr, uint64_t rounds, uint32_t *ck,
                  uint32_t *lofinal, uint32_t *progress) {
  extern __shared__ __align__(1024) uint8_t smem[];
  auto *sh = reinterpret_cast<pcclb::LsShared *>(smem + pcclb::kLsStageBytes * pcclb::kLsStages);
  const uint32_t lane0 = blockIdx.x * pcclb::kLsLanes;
  pcclb::loscan_cta(&map, ptr, rounds, lane0, ck, 32768u, progress + blockIdx.x, smem, sh);
  if (threadIdx.x < pcclb::kLsLanes) lofinal[lane0 + threadIdx.x] = sh->final_lo[threadIdx.x];
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

// serial reference: one thread per lane
__global__ void serial_lo(const uint32_t *p, uint64_t rounds, uint32_t *ck, uint32_t *fin, uint32_t ckrows) {
  const uint32_t lane = threadIdx.x + blockIdx.x * blockDim.x;
  uint32_t lo = 0x84222325u;
  for (uint64_t r = 0; r < rounds; ++r) {
    if (r % ckrows == 0) ck[(r / ckrows) * 256 + lane] = lo;
    lo = (lo ^ p[r * 256 + lane]) * 435u;
  }
  fin[lane] = lo;
}

int main(int argc, char **argv) {
  const uint64_t mib = argc > 1 ? strtoull(argv[1], 0, 10) : 1002;
  const uint64_t extra = argc > 2 ? strtoull(argv[2], 0, 10) : 0;  // extra rows past whole MiB
  const uint64_t rounds = mib * 1024 + extra;
  const uint64_t words = rounds * 256;
  const uint32_t ckrows = 32768;
  const uint64_t nseg = (rounds + ckrows - 1) / ckrows;
  uint32_t *d, *ck0, *ck1, *fin0, *fin1, *prog;
  CK(cudaMalloc(&d, words * 4));
  CK(cudaMalloc(&ck0, nseg * 256 * 4));
  CK(cudaMalloc(&ck1, nseg * 256 * 4));
  CK(cudaMalloc(&fin0, 256 * 4));
  CK(cudaMalloc(&fin1, 256 * 4));
  CK(cudaMalloc(&prog, 4096));
  fill<<<1184, 512>>>(d, words, 12345u);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  serial_lo<<<8, 32>>>(d, rounds, ck0, fin0, ckrows);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms0;
  cudaEventElapsedTime(&ms0, a, b);
  CUtensorMap map;
  if ((rounds >> 10) && !encode4d(&map, d, rounds)) return 2;
  CK(cudaFuncSetAttribute(loscan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pcclb::kLsSmem));
  float best = 1e9;
  for (int it = 0; it < 5; ++it) {
    CK(cudaMemset(ck1, 0xff, nseg * 256 * 4));
    CK(cudaMemset(prog, 0, 4096));
    cudaEventRecord(a);
    loscan_kernel<<<256 / pcclb::kLsLanes, pcclb::kLsThreads, pcclb::kLsSmem>>>(
        map, reinterpret_cast<const uint8_t *>(d), rounds, ck1, fin1, prog);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  std::vector<uint32_t> h0(nseg * 256), h1(nseg * 256), f0(256), f1(256);
  CK(cudaMemcpy(h0.data(), ck0, nseg * 1024, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h1.data(), ck1, nseg * 1024, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(f0.data(), fin0, 1024, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(f1.data(), fin1, 1024, cudaMemcpyDeviceToHost));
  uint64_t bad = 0;
  for (uint64_t i = 0; i < nseg * 256; ++i) bad += h0[i] != h1[i];
  for (int i = 0; i < 256; ++i) bad += f0[i] != f1[i];
  printf("rows=%llu serial %.3f ms  bitsliced %.3f ms (%.1f GB/s)  mismatches=%llu\n",
         (unsigned long long)rounds, ms0, best, words * 4 / best / 1e6, (unsigned long long)bad);
  return bad ? 1 : 0;
}
