// Streaming read-modify-write ceiling on one GPU (what the quantized gather's
// owner step A' -- x <- D(Q(x))/W in place + 1 code byte per element -- could
// reach). nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o rmw rmw.cu
// ./rmw [elements]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

struct alignas(16) F4 {
  float x, y, z, w;
};

__device__ __forceinline__ F4 ld(const float *p) {
  F4 r;
  asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st(float *p, F4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ uint32_t q1(float v) { return (uint32_t)fminf(fmaxf(rintf(v * 0.25f + 100.f), 0.f), 255.f); }
__device__ __forceinline__ float d1(uint32_t q) { return ((float)q - 100.f) * 4.f * 0.5f; }

// MODE 0: y = f(x) out of place; 1: x = f(x) in place; 2: in place + codes; 3: out of place + codes
template <int MODE, int U>
__global__ void __launch_bounds__(256) rmw(float *x, float *y, uint8_t *codes, uint64_t nv16) {
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv16; v += nt * U) {
    F4 in[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v + u * nt < nv16)
#pragma unroll
        for (int g = 0; g < 4; ++g) in[u][g] = ld(x + (v + u * nt) * 16 + 4 * g);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (v + u * nt >= nv16) break;
      uint32_t w[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint32_t q[4] = {q1(in[u][g].x), q1(in[u][g].y), q1(in[u][g].z), q1(in[u][g].w)};
        F4 o{d1(q[0]), d1(q[1]), d1(q[2]), d1(q[3])};
        w[g] = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
        st(((MODE == 0 || MODE == 3) ? y : x) + (v + u * nt) * 16 + 4 * g, o);
      }
      if (MODE >= 2) *reinterpret_cast<uint4 *>(codes + (v + u * nt) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// item-based (like the fused ring kernels): CTAs claim ITEM-element items in
// order from a counter and sweep each with a CTA-stride loop
template <int U>
__global__ void __launch_bounds__(256) rmw_items(float *x, uint8_t *codes, uint64_t n, uint64_t item,
                                                 uint32_t *claim) {
  __shared__ uint32_t s_it;
  const uint64_t nitems = (n + item - 1) / item;
  for (;;) {
    if (threadIdx.x == 0) s_it = atomicAdd(claim, 1u);
    __syncthreads();
    const uint64_t it = s_it;
    __syncthreads();
    if (it >= nitems) break;
    const uint64_t b = it * item, nv = (min(n, b + item) - b) / 16;
    for (uint64_t v = threadIdx.x; v < nv; v += 256 * U) {
      F4 in[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (v + u * 256 < nv)
#pragma unroll
          for (int g = 0; g < 4; ++g) in[u][g] = ld(x + b + (v + u * 256) * 16 + 4 * g);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v + u * 256 >= nv) break;
        uint32_t w[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t q[4] = {q1(in[u][g].x), q1(in[u][g].y), q1(in[u][g].z), q1(in[u][g].w)};
          F4 o{d1(q[0]), d1(q[1]), d1(q[2]), d1(q[3])};
          w[g] = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
          st(x + b + (v + u * 256) * 16 + 4 * g, o);
        }
        *reinterpret_cast<uint4 *>(codes + b + (v + u * 256) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
}

template <int U>
float run_items(float *x, uint8_t *c, uint64_t n, int grid, uint64_t item, uint32_t *claim) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int i = 0; i < 6; ++i) {
    cudaMemset(claim, 0, 4);
    cudaEventRecord(a);
    rmw_items<U><<<grid, 256>>>(x, c, n, item, claim);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i && ms < best) best = ms;
  }
  return best;
}

template <int MODE, int U>
float run(float *x, float *y, uint8_t *c, uint64_t n, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  rmw<MODE, U><<<grid, 256>>>(x, y, c, n / 16);
  float best = 1e9;
  for (int i = 0; i < 5; ++i) {
    cudaEventRecord(a);
    rmw<MODE, U><<<grid, 256>>>(x, y, c, n / 16);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char **argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 600000000ull;
  float *x, *y;
  uint8_t *c;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&y, n * 4);
  cudaMalloc(&c, n);
  cudaMemset(x, 0, n * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes[4] = {8.0 * n, 8.0 * n, 9.0 * n, 9.0 * n};
  const char *names[4] = {"out-of-place", "in-place", "in-place+codes", "out-of-place+codes"};
  for (int per : {1, 2, 3}) {
    const int g = sms * per;
    float t[4][3];
    t[0][0] = run<0, 1>(x, y, c, n, g); t[0][1] = run<0, 2>(x, y, c, n, g); t[0][2] = run<0, 4>(x, y, c, n, g);
    t[1][0] = run<1, 1>(x, y, c, n, g); t[1][1] = run<1, 2>(x, y, c, n, g); t[1][2] = run<1, 4>(x, y, c, n, g);
    t[2][0] = run<2, 1>(x, y, c, n, g); t[2][1] = run<2, 2>(x, y, c, n, g); t[2][2] = run<2, 4>(x, y, c, n, g);
    t[3][0] = run<3, 1>(x, y, c, n, g); t[3][1] = run<3, 2>(x, y, c, n, g); t[3][2] = run<3, 4>(x, y, c, n, g);
    for (int m = 0; m < 4; ++m)
      printf("CTAs/SM %d %-20s U=1 %.3f ms (%.0f GB/s)  U=2 %.3f ms (%.0f)  U=4 %.3f ms (%.0f)\n", per, names[m],
             t[m][0], bytes[m] / t[m][0] / 1e6, t[m][1], bytes[m] / t[m][1] / 1e6, t[m][2], bytes[m] / t[m][2] / 1e6);
  }
  uint32_t *claim;
  cudaMalloc(&claim, 4);
  for (int per : {1, 2, 3, 4})
    for (uint64_t item : {16384ull, 65536ull, 262144ull, 1048576ull}) {
      const int g = sms * per;
      const float u1 = run_items<1>(x, c, n, g, item, claim), u2 = run_items<2>(x, c, n, g, item, claim),
                  u4 = run_items<4>(x, c, n, g, item, claim);
      printf("items CTAs/SM %d item %7llu  U=1 %.3f ms (%.0f GB/s)  U=2 %.3f (%.0f)  U=4 %.3f (%.0f)\n", per,
             (unsigned long long)item, u1, 9.0 * n / u1 / 1e6, u2, 9.0 * n / u2 / 1e6, u4, 9.0 * n / u4 / 1e6);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
