// Microbenchmarks behind the simplehash design (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_micro stream_micro.cu
// 1. per-CTA streaming read throughput: TMA bulk ring vs cp.async (LDGSTS)
//    ring vs LDG.128 into registers, consumer does a trivial xor-reduce;
// 2. FNV-1a-64 chain step latency (cycles) with the split lo/hi form.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c)); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// each CTA streams its own contiguous slice of `bytes_per_cta`
template <int STAGE, int NST>
__global__ void __launch_bounds__(256) tma_stream(const uint8_t *p, uint64_t bytes_per_cta, uint32_t *sink) {
  extern __shared__ __align__(1024) uint8_t st[];
  __shared__ __align__(8) uint64_t bars[NST];
  const uint8_t *base = p + blockIdx.x * bytes_per_cta;
  if (threadIdx.x == 0) { for (int i = 0; i < NST; ++i) mbar_init(&bars[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const uint64_t nst = bytes_per_cta / STAGE;
  if (threadIdx.x == 0) for (int s = 0; s < NST && s < (int)nst; ++s) { mbar_expect_tx(&bars[s], STAGE); bulk(st + s * STAGE, base + (uint64_t)s * STAGE, STAGE, &bars[s]); }
  uint32_t acc = 0, par = 0;
  for (uint64_t s = 0; s < nst; ++s) {
    int slot = s % NST;
    mbar_wait(&bars[slot], (par >> slot) & 1); par ^= 1u << slot;
    const uint32_t *w = reinterpret_cast<const uint32_t *>(st + slot * STAGE);
    for (int i = threadIdx.x; i < STAGE / 4; i += 256) acc ^= w[i];
    __syncthreads();
    if (threadIdx.x == 0 && s + NST < nst) { mbar_expect_tx(&bars[slot], STAGE); bulk(st + slot * STAGE, base + (s + NST) * STAGE, STAGE, &bars[slot]); }
  }
  if (acc == 0x12345678) sink[0] = acc;
}

// 2-D TMA: the buffer viewed as [rows x 256] u32; the CTA streams its column
// slice [x0, x0 + BOXW) through NST stages of BOXH rows
template <int BOXW, int BOXH, int NST>
__global__ void __launch_bounds__(128) tma2d_stream(const __grid_constant__ CUtensorMap map, uint64_t rows_per_cta, uint32_t *sink) {
  extern __shared__ __align__(1024) uint8_t st[];
  __shared__ __align__(8) uint64_t bars[NST];
  constexpr int STAGE = BOXW * BOXH * 4;
  const int x0 = (blockIdx.x % (256 / BOXW)) * BOXW;
  const uint64_t y0 = (blockIdx.x / (256 / BOXW)) * rows_per_cta;
  if (threadIdx.x == 0) { for (int i = 0; i < NST; ++i) mbar_init(&bars[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const uint64_t nst = rows_per_cta / BOXH;
  auto issue = [&](uint64_t s, int slot) {
    mbar_expect_tx(&bars[slot], STAGE);
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(st + slot * STAGE)), "l"(&map), "r"(x0), "r"((int)(y0 + s * BOXH)), "r"(smem_u32(&bars[slot])) : "memory");
  };
  if (threadIdx.x == 0) for (int s = 0; s < NST && s < (int)nst; ++s) issue(s, s);
  uint32_t acc = 0, par = 0;
  for (uint64_t s = 0; s < nst; ++s) {
    int slot = s % NST;
    mbar_wait(&bars[slot], (par >> slot) & 1); par ^= 1u << slot;
    const uint32_t *w = reinterpret_cast<const uint32_t *>(st + slot * STAGE);
    for (int i = threadIdx.x; i < STAGE / 4; i += 128) acc ^= w[i];
    __syncthreads();
    if (threadIdx.x == 0 && s + NST < nst) issue(s + NST, slot);
  }
  if (acc == 0x12345678) sink[0] = acc;
}

// LDG.128: each thread keeps U loads in flight
template <int U>
__global__ void __launch_bounds__(256) ldg_stream(const uint4 *p, uint64_t vec_per_cta, uint32_t *sink) {
  const uint4 *base = p + blockIdx.x * vec_per_cta;
  uint32_t acc = 0;
  for (uint64_t i = threadIdx.x; i < vec_per_cta; i += 256 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(base + i + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678) sink[0] = acc;
}

// FNV chain latency: one warp, steps dependent on the previous
__global__ void fnv_chain(const uint32_t *w, int steps, uint64_t *out, long long *cyc) {
  uint32_t lo = 0x84222325u ^ threadIdx.x, hi = 0xcbf29ce4u;
  uint32_t ww = w[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) {
    const uint32_t x = lo ^ (ww + i);
    const uint64_t p = (uint64_t)x * 435u;
    const uint32_t add = (uint32_t)(p >> 32) + (x << 8);
    lo = (uint32_t)p;
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
  }
  long long t1 = clock64();
  out[threadIdx.x] = ((uint64_t)hi << 32) | lo;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

// 64-bit naive form for comparison
__global__ void fnv_chain64(const uint32_t *w, int steps, uint64_t *out, long long *cyc) {
  uint64_t h = 0xcbf29ce484222325ull ^ threadIdx.x;
  uint32_t ww = w[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) h = (h ^ (uint64_t)(ww + i)) * 0x100000001b3ull;
  long long t1 = clock64();
  out[threadIdx.x] = h;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <class F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const uint64_t total = 8ull << 30;
  uint8_t *buf; uint32_t *sink;
  CK(cudaMalloc(&buf, total)); CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(buf, 1, total));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run_tma = [&](auto kern, int stage, int nst, int ctas, uint64_t per) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, stage * nst));
    float ms = time_ms([&] { kern<<<ctas, 256, stage * nst>>>(buf, per, sink); });
    CK(cudaGetLastError());
    printf("tma stage=%6d nst=%2d ctas=%4d : %8.1f GB/s total, %7.1f GB/s per CTA\n", stage, nst, ctas, ctas * per / ms / 1e6, per / ms / 1e6);
    return 0;
  };
  for (int ctas : {1, 4, sms, 2 * sms}) {
    uint64_t per = (ctas == 1 ? (1ull << 30) : (total / ctas)) & ~((1ull << 16) - 1);
    run_tma(tma_stream<16384, 4>, 16384, 4, ctas, per);
    run_tma(tma_stream<16384, 12>, 16384, 12, ctas, per);
    run_tma(tma_stream<32768, 6>, 32768, 6, ctas, per);
    run_tma(tma_stream<65536, 3>, 65536, 3, ctas, per);
    float ms = time_ms([&] { ldg_stream<8><<<ctas, 256>>>((const uint4 *)buf, per / 16, sink); });
    printf("ldg U=8  ctas=%4d : %8.1f GB/s total, %7.1f GB/s per CTA\n", ctas, ctas * per / ms / 1e6, per / ms / 1e6);
    ms = time_ms([&] { ldg_stream<16><<<ctas, 256>>>((const uint4 *)buf, per / 16, sink); });
    printf("ldg U=16 ctas=%4d : %8.1f GB/s total, %7.1f GB/s per CTA\n", ctas, ctas * per / ms / 1e6, per / ms / 1e6);
  }
  {
    void *fp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    auto run2d = [&](auto kern, int boxw, int boxh, int nst, int ctas) {
      CUtensorMap m;
      cuuint64_t dims[2] = {256, total / 1024};
      cuuint64_t strides[1] = {1024};
      cuuint32_t box[2] = {(cuuint32_t)boxw, (cuuint32_t)boxh};
      cuuint32_t es[2] = {1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      int smem = boxw * boxh * 4 * nst;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int groups = ctas / (256 / boxw); if (groups < 1) groups = 1;
      uint64_t rows = (total / 1024 / groups) / boxh * boxh;
      if (ctas == 1 || ctas == 2) rows = (1ull << 20) / boxh * boxh;  // 1 GiB of rounds
      float ms = time_ms([&] { kern<<<ctas, 128, smem>>>(m, rows, sink); });
      uint64_t bytes = (uint64_t)ctas * rows * boxw * 4;
      printf("tma2d box=%3dx%3d nst=%d ctas=%4d : %8.1f GB/s total, %7.1f GB/s per CTA (%s)\n", boxw, boxh, nst, ctas,
             bytes / ms / 1e6, bytes / ms / 1e6 / ctas, cudaGetErrorString(cudaGetLastError()));
    };
    for (int ctas : {1, 4}) {
      run2d(tma2d_stream<64, 256, 3>, 64, 256, 3, ctas);
      run2d(tma2d_stream<64, 128, 6>, 64, 128, 6, ctas);
      run2d(tma2d_stream<128, 128, 3>, 128, 128, 3, ctas);
      run2d(tma2d_stream<128, 64, 6>, 128, 64, 6, ctas);
      run2d(tma2d_stream<256, 64, 3>, 256, 64, 3, ctas);
      run2d(tma2d_stream<256, 32, 6>, 256, 32, 6, ctas);
      run2d(tma2d_stream<256, 16, 12>, 256, 16, 12, ctas);
    }
  }
  uint64_t *out; long long *cyc; long long h;
  CK(cudaMalloc(&out, 8 * 1024)); CK(cudaMalloc(&cyc, 8));
  for (int warps : {1, 8}) {
    fnv_chain<<<1, 32 * warps>>>((const uint32_t *)buf, 1 << 20, out, cyc);
    CK(cudaDeviceSynchronize()); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("fnv split chain: %d warps: %.2f cycles/step\n", warps, (double)h / (1 << 20));
    fnv_chain64<<<1, 32 * warps>>>((const uint32_t *)buf, 1 << 20, out, cyc);
    CK(cudaDeviceSynchronize()); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("fnv 64-bit chain: %d warps: %.2f cycles/step\n", warps, (double)h / (1 << 20));
  }
  return 0;
}
