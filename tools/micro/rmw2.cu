// A' of the quantized gather (x <- D(Q(x))/W in place + 1 code byte per
// element) with the library's exact arithmetic: direct loads vs a TMA
// bulk-copy pipeline (producer warp + mbarrier ring).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -prec-div=true -ftz=false \
//   -std=c++17 -I../../include -I../../paper_2505_14065_b200/csrc --expt-relaxed-constexpr -o rmw2 rmw2.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#include "numerics.cuh"
#include "tma.cuh"

using namespace pcclb;

struct alignas(16) F4 {
  float v[4];
};
__device__ __forceinline__ F4 ldg(const float *p) {
  F4 r;
  asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg(float *p, F4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.v[0]), "f"(v.v[1]), "f"(v.v[2]), "f"(v.v[3])
               : "memory");
}

// 16 elements: codes word + adopted values
__device__ __forceinline__ uint4 adopt16(F4 (&in)[4], const QParams &qp) {
  uint32_t w[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      q[k] = quant1_fast(in[g].v[k], qp.mn, qp.scale, qp.inv);
      in[g].v[k] = div_world_x<false>(dequant1x<false>(q[k], qp.mn, qp.scale), 2.0f);
    }
    w[g] = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// V bit 1: claim also reads a volatile status word; bit 2: every other
// position is an empty one (like the gather's B' slots)
template <int U, int V = 0>
__global__ void __launch_bounds__(256) direct(float *x, uint8_t *codes, uint64_t n, uint64_t item, uint32_t *claim,
                                              QParams qp) {
  __shared__ uint32_t s_it, s_ok;
  const uint64_t nitems = (n + item - 1) / item;
  for (;;) {
    if (threadIdx.x == 0) {
      s_it = atomicAdd(claim, 1u);
      if (V & 1) s_ok = *(volatile uint32_t *)(claim + 1) == 0;
    }
    __syncthreads();
    uint64_t it = s_it;
    __syncthreads();
    if (V & 2) {
      if (it & 1) {
        if (it / 2 >= nitems) break;
        continue;
      }
      it /= 2;
    }
    if (it >= nitems) break;
    const uint64_t b = it * item, nv = (min(n, b + item) - b) / 16;
    for (uint64_t v = threadIdx.x; v < nv; v += 256 * U) {
      F4 in[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (v + u * 256 < nv)
#pragma unroll
          for (int g = 0; g < 4; ++g) in[u][g] = ldg(x + b + (v + u * 256) * 16 + 4 * g);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v + u * 256 >= nv) break;
        const uint4 c = adopt16(in[u], qp);
#pragma unroll
        for (int g = 0; g < 4; ++g) stg(x + b + (v + u * 256) * 16 + 4 * g, in[u][g]);
        *reinterpret_cast<uint4 *>(codes + b + (v + u * 256) * 16) = c;
      }
    }
  }
}

// B' of the quantized gather: out <- D(codes) / W
template <int U>
__global__ void __launch_bounds__(256) deq(float *x, const uint8_t *codes, uint64_t n, uint64_t item, uint32_t *claim,
                                           QParams qp) {
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
      uint4 q[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (v + u * 256 < nv) q[u] = __ldcg(reinterpret_cast<const uint4 *>(codes + b + (v + u * 256) * 16));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v + u * 256 >= nv) break;
        const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          F4 o;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            o.v[k] = div_world_x<false>(dequant1x<false>((w[g] >> (8 * k)) & 255u, qp.mn, qp.scale), 2.0f);
          stg(x + b + (v + u * 256) * 16 + 4 * g, o);
        }
      }
    }
  }
}

// coalesced forms: a lane owns 4 consecutive elements per unit (16-byte
// float accesses and 4-byte code accesses contiguous across the warp)
template <int U>
__global__ void __launch_bounds__(256) deqc(float *x, const uint8_t *codes, uint64_t n, uint64_t item, uint32_t *claim,
                                            QParams qp) {
  __shared__ uint32_t s_it;
  const uint64_t nitems = (n + item - 1) / item;
  for (;;) {
    if (threadIdx.x == 0) s_it = atomicAdd(claim, 1u);
    __syncthreads();
    const uint64_t it = s_it;
    __syncthreads();
    if (it >= nitems) break;
    const uint64_t b = it * item, nv = (min(n, b + item) - b) / 4;
    for (uint64_t v = threadIdx.x; v < nv; v += 256 * U) {
      uint32_t q[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (v + u * 256 < nv) q[u] = __ldcg(reinterpret_cast<const uint32_t *>(codes + b + (v + u * 256) * 4));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v + u * 256 >= nv) break;
        F4 o;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          o.v[k] = div_world_x<false>(dequant1x<false>((q[u] >> (8 * k)) & 255u, qp.mn, qp.scale), 2.0f);
        stg(x + b + (v + u * 256) * 4, o);
      }
    }
  }
}

template <int U>
__global__ void __launch_bounds__(256) directc(float *x, uint8_t *codes, uint64_t n, uint64_t item, uint32_t *claim,
                                               QParams qp) {
  __shared__ uint32_t s_it;
  const uint64_t nitems = (n + item - 1) / item;
  for (;;) {
    if (threadIdx.x == 0) s_it = atomicAdd(claim, 1u);
    __syncthreads();
    const uint64_t it = s_it;
    __syncthreads();
    if (it >= nitems) break;
    const uint64_t b = it * item, nv = (min(n, b + item) - b) / 4;
    for (uint64_t v = threadIdx.x; v < nv; v += 256 * U) {
      F4 in[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (v + u * 256 < nv) in[u] = ldg(x + b + (v + u * 256) * 4);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v + u * 256 >= nv) break;
        uint32_t q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          q[k] = quant1_fast(in[u].v[k], qp.mn, qp.scale, qp.inv);
          in[u].v[k] = div_world_x<false>(dequant1x<false>(q[k], qp.mn, qp.scale), 2.0f);
        }
        stg(x + b + (v + u * 256) * 4, in[u]);
        *reinterpret_cast<uint32_t *>(codes + b + (v + u * 256) * 4) = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
      }
    }
  }
}

// TMA pipeline: warp 8 claims items and streams TILE-element tiles into a
// STAGES-deep shared ring; warps 0-7 adopt from shared memory and store.
template <int TILE, int STAGES>
struct Ring {
  float tile[STAGES][TILE];
  uint64_t full[STAGES], empty[STAGES];
  uint64_t off[STAGES];
  uint32_t cnt[STAGES];
};

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int TILE, int STAGES>
__global__ void __launch_bounds__(288) piped(float *x, uint8_t *codes, uint64_t n, uint64_t item, uint32_t *claim,
                                             QParams qp) {
  extern __shared__ __align__(128) unsigned char smraw[];
  auto &R = *reinterpret_cast<Ring<TILE, STAGES> *>(smraw);
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], 8);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const uint64_t nitems = (n + item - 1) / item;
  if (warp == 8) {
    if (lane == 0) {
      uint32_t k = 0;  // tiles issued
      for (;;) {
        const uint64_t it = atomicAdd(claim, 1u);
        const bool done = it >= nitems;
        const uint64_t b = it * item, e = done ? b : (n < b + item ? n : b + item);
        for (uint64_t o = b;; o += TILE) {
          const uint32_t s = k % STAGES;
          if (k >= STAGES) mbar_wait(&R.empty[s], ((k / STAGES) - 1) & 1);
          const uint32_t c = done ? 0u : (uint32_t)(e - o < (uint64_t)TILE ? e - o : (uint64_t)TILE);
          R.off[s] = o;
          R.cnt[s] = c;
          if (c) {
            mbar_expect_tx(&R.full[s], c * 4);
            bulk_g2s(R.tile[s], x + o, c * 4, &R.full[s]);
          } else {
            mbar_arrive(&R.full[s]);
          }
          ++k;
          if (!c || o + TILE >= e) break;
        }
        if (done) break;
      }
    }
    return;
  }
  for (uint32_t k = 0;; ++k) {
    const uint32_t s = k % STAGES;
    mbar_wait(&R.full[s], (k / STAGES) & 1);
    const uint32_t c = R.cnt[s];
    const uint64_t o = R.off[s];
    if (!c) break;
    for (uint32_t v = threadIdx.x; v * 16 < c; v += 256) {
      F4 in[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) in[g] = *reinterpret_cast<const F4 *>(&R.tile[s][v * 16 + 4 * g]);
      const uint4 cw = adopt16(in, qp);
#pragma unroll
      for (int g = 0; g < 4; ++g) stg(x + o + v * 16 + 4 * g, in[g]);
      *reinterpret_cast<uint4 *>(codes + o + v * 16) = cw;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&R.empty[s]);
  }
}

__global__ void fill(float *x, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    x[i] = __sinf((float)(i % 100003)) * 0.9f;
}

template <typename K>
float timeit(K k, uint32_t *claim) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int i = 0; i < 6; ++i) {
    cudaMemset(claim, 0, 4);
    cudaEventRecord(a);
    k();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i && ms < best) best = ms;
  }
  return best;
}

int main(int argc, char **argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 600000000ull;
  float *x;
  uint8_t *c;
  uint32_t *claim;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&c, n);
  cudaMalloc(&claim, 8);
  cudaMemset(claim, 0, 8);
  fill<<<1184, 256>>>(x, n);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  QParams qp;
  qp.mn = -1.0f;
  qp.scale = 2.0f / 255.0f;
  qp.inv = 1.0f / qp.scale;
  const double bytes = 9.0 * n;
  for (int rep = 0; rep < 2; ++rep) {
    const int g = sms * 3;
    float a = timeit([&] { direct<2, 0><<<g, 256>>>(x, c, n, 262144, claim, qp); }, claim);
    float b = timeit([&] { direct<2, 1><<<g, 256>>>(x, c, n, 262144, claim, qp); }, claim);
    float d = timeit([&] { direct<2, 2><<<g, 256>>>(x, c, n, 262144, claim, qp); }, claim);
    float e = timeit([&] { direct<2, 3><<<g, 256>>>(x, c, n, 262144, claim, qp); }, claim);
    printf("claim variants 3 CTAs/SM 256Ki U=2: plain %.3f  +status %.3f  +skips %.3f  +both %.3f ms\n", a, b, d, e);
  }
  if (getenv("ONLY")) {
    timeit([&] { direct<2><<<sms * 3, 256>>>(x, c, n, 262144, claim, qp); }, claim);
    return 0;
  }
  for (int per : {2, 3, 4})
    for (uint64_t item : {65536ull, 262144ull}) {
      const int g = sms * per;
      float t2 = timeit([&] { direct<2><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      float t1 = timeit([&] { direct<1><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      printf("direct CTAs/SM %d item %7llu U=1 %.3f ms (%.0f GB/s) U=2 %.3f ms (%.0f GB/s)\n", per,
             (unsigned long long)item, t1, bytes / t1 / 1e6, t2, bytes / t2 / 1e6);
    }
  for (int per : {2, 3, 4})
    for (uint64_t item : {65536ull, 262144ull}) {
      const int g = sms * per;
      float t2 = timeit([&] { deq<2><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      float t4 = timeit([&] { deq<4><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      float t8 = timeit([&] { deq<8><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      printf("deq CTAs/SM %d item %7llu U=2 %.3f ms (%.0f GB/s) U=4 %.3f ms (%.0f) U=8 %.3f ms (%.0f)\n", per,
             (unsigned long long)item, t2, 5.0 * n / t2 / 1e6, t4, 5.0 * n / t4 / 1e6, t8, 5.0 * n / t8 / 1e6);
    }
  for (int per : {2, 3, 4})
    for (uint64_t item : {65536ull, 262144ull}) {
      const int g = sms * per;
      float t2 = timeit([&] { deqc<4><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      float t4 = timeit([&] { deqc<8><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      float t8 = timeit([&] { deqc<16><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      printf("deqc CTAs/SM %d item %7llu U=4 %.3f ms (%.0f GB/s) U=8 %.3f ms (%.0f) U=16 %.3f ms (%.0f)\n", per,
             (unsigned long long)item, t2, 5.0 * n / t2 / 1e6, t4, 5.0 * n / t4 / 1e6, t8, 5.0 * n / t8 / 1e6);
    }
  for (int per : {2, 3, 4})
    for (uint64_t item : {65536ull, 262144ull}) {
      const int g = sms * per;
      float t2 = timeit([&] { directc<4><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      float t4 = timeit([&] { directc<8><<<g, 256>>>(x, c, n, item, claim, qp); }, claim);
      printf("directc CTAs/SM %d item %7llu U=4 %.3f ms (%.0f GB/s) U=8 %.3f ms (%.0f)\n", per,
             (unsigned long long)item, t2, 9.0 * n / t2 / 1e6, t4, 9.0 * n / t4 / 1e6);
    }
  if (getenv("PIPED") == nullptr) return 0;
#define PIPED(TILE, ST)                                                                                          \
  {                                                                                                              \
    const int sm = sizeof(Ring<TILE, ST>);                                                                       \
    cudaFuncSetAttribute(piped<TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                      \
    for (int per : {1, 2, 3})                                                                                    \
      for (uint64_t item : {65536ull, 262144ull}) {                                                              \
        if (per * (sm + 1024) > 227 * 1024) continue;                                                            \
        const int g = sms * per;                                                                                 \
        float t = timeit([&] { piped<TILE, ST><<<g, 288, sm>>>(x, c, n, item, claim, qp); }, claim);              \
        printf("piped tile %5d stages %d CTAs/SM %d item %7llu %.3f ms (%.0f GB/s) %s\n", TILE, ST, per,        \
               (unsigned long long)item, t, bytes / t / 1e6, cudaGetErrorString(cudaGetLastError()));            \
      }                                                                                                          \
  }
  PIPED(4096, 4)
  PIPED(4096, 8)
  PIPED(2048, 8)
  PIPED(8192, 4)
  PIPED(4096, 3)
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
