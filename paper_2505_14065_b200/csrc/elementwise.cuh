// Grid-stride elementwise loop with 128-bit vector bodies.
//
// A functor F provides
//   __device__ void one(uint64_t i);             // scalar element i
//   using In = ...;                              // loaded operands of one vector
//   __device__ In vload(uint64_t i);             // loads for elements [i, i+VEC)
//   __device__ void vapply(uint64_t i, const In&);  // compute + stores
// `head` scalar elements are peeled so that vec() sees 16-byte aligned
// addresses (the host computes it); VEC == 1 selects a scalar-only loop for
// pointer sets whose misalignments differ.
#pragma once

#include <stdint.h>
#include <string.h>

namespace pcclb {

template <typename T>
struct alignas(16) Pack16 {
  static constexpr int N = 16 / sizeof(T);
  T e[N];
};

template <typename T>
__device__ __forceinline__ Pack16<T> ld16(const T *p) {
  return *reinterpret_cast<const Pack16<T> *>(p);
}
template <typename T>
__device__ __forceinline__ void st16(T *p, const Pack16<T> &v) {
  *reinterpret_cast<Pack16<T> *>(p) = v;
}
// streaming (evict-first) variants for data touched exactly once
__device__ __forceinline__ Pack16<float> ld16_cs(const float *p) {
  float4 v = __ldcs(reinterpret_cast<const float4 *>(p));
  Pack16<float> r;
  r.e[0] = v.x;
  r.e[1] = v.y;
  r.e[2] = v.z;
  r.e[3] = v.w;
  return r;
}
__device__ __forceinline__ Pack16<double> ld16_cs(const double *p) {
  double2 v = __ldcs(reinterpret_cast<const double2 *>(p));
  Pack16<double> r;
  r.e[0] = v.x;
  r.e[1] = v.y;
  return r;
}

template <typename T>
__device__ __forceinline__ Pack16<T> ld16_cs(const T *p) {  // 2-byte types (bf16)
  const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(p));
  Pack16<T> r;
  memcpy(&r, &v, 16);
  return r;
}

template <int VEC, int UNROLL, typename F>
__device__ __forceinline__ void ew_loop(uint64_t n, uint64_t head, F &f) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  if constexpr (VEC == 1) {
    for (uint64_t i = tid; i < n; i += nth) f.one(i);
  } else {
    if (head > n) head = n;
    if (tid < head) f.one(tid);
    const uint64_t nv = (n - head) / VEC;
    uint64_t base = tid;
    // full unrolled rounds: all UNROLL vectors are loaded before any is
    // stored, so each thread keeps UNROLL loads in flight (the compiler
    // cannot hoist loads over stores through possibly aliasing pointers)
    for (; base + (UNROLL - 1) * nth < nv; base += UNROLL * nth) {
      typename F::In in[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) in[u] = f.vload(head + (base + u * nth) * VEC);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) f.vapply(head + (base + u * nth) * VEC, in[u]);
    }
    for (; base < nv; base += nth) {
      typename F::In in = f.vload(head + base * VEC);
      f.vapply(head + base * VEC, in);
    }
    const uint64_t t0 = head + nv * VEC;
    if (tid < n - t0) f.one(t0 + tid);
  }
}

// Elements to peel before `p` is 16-byte aligned (p must be element-aligned).
template <typename T>
inline uint64_t peel16(const void *p) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  return (uint64_t)(((16 - (a & 15)) & 15) / sizeof(T));
}

}  // namespace pcclb
