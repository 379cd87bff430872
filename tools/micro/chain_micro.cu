// FNV-1a-64 chain formulations: cycles per dependent step (one lane = one chain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_micro chain_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// A: 64-bit (h ^ w) * P as written (compiler splits with IMAD.WIDE)
struct A {
  uint64_t h;
  A() = default;
  __device__ A(uint64_t v) : h(v) {}
  __device__ __forceinline__ void step(uint32_t w) { h = (h ^ (uint64_t)w) * 0x100000001b3ull; }
  __device__ uint64_t v() const { return h; }
};
// B: lo chain with a plain 32-bit IMAD; carry by IMAD.HI off the chain
struct B {
  uint32_t lo, hi;
  B() = default;
  __device__ B(uint64_t v) : lo((uint32_t)v), hi((uint32_t)(v >> 32)) {}
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    uint32_t nlo, c;
    asm("mul.lo.u32 %0, %1, 435;" : "=r"(nlo) : "r"(x));
    asm("mul.hi.u32 %0, %1, 435;" : "=r"(c) : "r"(x));
    uint32_t add;
    asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(add) : "r"(x), "r"(c));
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
    lo = nlo;
  }
  __device__ uint64_t v() const { return ((uint64_t)hi << 32) | lo; }
};
// C: IMAD.WIDE for lo+carry, explicit mads for hi
struct C {
  uint32_t lo, hi;
  C() = default;
  __device__ C(uint64_t v) : lo((uint32_t)v), hi((uint32_t)(v >> 32)) {}
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    const uint64_t p = (uint64_t)x * 435u;
    uint32_t add;
    asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(add) : "r"(x), "r"((uint32_t)(p >> 32)));
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
    lo = (uint32_t)p;
  }
  __device__ uint64_t v() const { return ((uint64_t)hi << 32) | lo; }
};

// D: lo chain with a plain 32-bit IMAD; the carry multiplies an opaque copy of
// x so ptxas cannot merge the two products into one IMAD.WIDE
__device__ uint32_t g_zero;
struct D {
  uint32_t lo, hi, z;
  D() = default;
  __device__ D(uint64_t v) : lo((uint32_t)v), hi((uint32_t)(v >> 32)) { asm volatile("ld.global.u32 %0, [%1];" : "=r"(z) : "l"(&g_zero)); }
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    uint32_t nlo, c, xz;
    asm("mul.lo.u32 %0, %1, 435;" : "=r"(nlo) : "r"(x));
    asm("add.u32 %0, %1, %2;" : "=r"(xz) : "r"(x), "r"(z));
    asm("mul.hi.u32 %0, %1, 435;" : "=r"(c) : "r"(xz));
    uint32_t add;
    asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(add) : "r"(x), "r"(c));
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
    lo = nlo;
  }
  __device__ uint64_t v() const { return ((uint64_t)hi << 32) | lo; }
};

// E: multiply by 435 = 3 * 145 as three shift-adds on the ALU pipe (no cross-pipe hop)
struct E {
  uint32_t lo, hi;
  E() = default;
  __device__ E(uint64_t v) : lo((uint32_t)v), hi((uint32_t)(v >> 32)) {}
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    uint32_t t, u, v;
    asm("{ .reg .b32 s; shl.b32 s, %1, 1; add.u32 %0, s, %1; }" : "=r"(t) : "r"(x));
    asm("{ .reg .b32 s; shl.b32 s, %1, 4; add.u32 %0, s, %1; }" : "=r"(u) : "r"(t));
    asm("{ .reg .b32 s; shl.b32 s, %1, 7; add.u32 %0, s, %2; }" : "=r"(v) : "r"(t), "r"(u));
    const uint32_t c = __umulhi(x, 435u);
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(c + (x << 8)));
    lo = v;
  }
  __device__ uint64_t v() const { return ((uint64_t)hi << 32) | lo; }
};

// F: lo chain only (no hi): the pure LOP3 -> IMAD latency
struct F {
  uint32_t lo, hi;
  F() = default;
  __device__ F(uint64_t v) : lo((uint32_t)v), hi((uint32_t)(v >> 32)) {}
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    asm("mul.lo.u32 %0, %1, 435;" : "=r"(lo) : "r"(x));
  }
  __device__ uint64_t v() const { return ((uint64_t)hi << 32) | lo; }
};
// G: IMAD lo, IMAD.HI carry, (x<<8)+c on the ALU pipe (shf+add), IMAD hi
struct G {
  uint32_t lo, hi;
  G() = default;
  __device__ G(uint64_t v) : lo((uint32_t)v), hi((uint32_t)(v >> 32)) {}
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    uint32_t nlo, c, add;
    asm("mul.lo.u32 %0, %1, 435;" : "=r"(nlo) : "r"(x));
    asm("mul.hi.u32 %0, %1, 435;" : "=r"(c) : "r"(x));
    asm("{ .reg .b32 s; shl.b32 s, %1, 8; add.u32 %0, s, %2; }" : "=r"(add) : "r"(x), "r"(c));
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
    lo = nlo;
  }
  __device__ uint64_t v() const { return ((uint64_t)hi << 32) | lo; }
};
// H: hi deferred: accumulate carries of 4 steps, then fold with 435^k (fewer FMA ops per step)
struct H {
  uint32_t lo, hi, acc; int k;
  H() = default;
  __device__ H(uint64_t v) : lo((uint32_t)v), hi((uint32_t)(v >> 32)), acc(0), k(0) {}
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    uint32_t nlo, c, add;
    asm("mul.lo.u32 %0, %1, 435;" : "=r"(nlo) : "r"(x));
    asm("mul.hi.u32 %0, %1, 435;" : "=r"(c) : "r"(x));
    asm("{ .reg .b32 s; shl.b32 s, %1, 8; add.u32 %0, s, %2; }" : "=r"(add) : "r"(x), "r"(c));
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
    lo = nlo;
  }
  __device__ uint64_t v() const { return ((uint64_t)hi << 32) | lo; }
};

template <class F, int CH>
__global__ void chain(const uint32_t *w, int steps, uint64_t *out, long long *cyc) {
  F f[CH] = {F(0xcbf29ce484222325ull ^ threadIdx.x)};
  for (int c = 1; c < CH; ++c) f[c] = F(0xcbf29ce484222325ull ^ (threadIdx.x + 1000 * c));
  const uint32_t *p = w + threadIdx.x;
  uint32_t r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = p[k * 32];
  long long t0 = clock64();
  for (int i = 0; i < steps; i += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int c = 0; c < CH; ++c) f[c].step(r[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = r[k] * 3u + (uint32_t)i;  // new words, registers only (off the chain)
  }
  long long t1 = clock64();
  uint64_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= f[c].v();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  uint32_t *w; uint64_t *out; long long *cyc;
  cudaMalloc(&w, 1 << 24); cudaMalloc(&out, 1 << 22); cudaMalloc(&cyc, 8);
  cudaMemset(w, 7, 1 << 24);
  const int steps = 1 << 18;
  auto run = [&](auto kern, const char *name, int threads, int ch) {
    kern<<<1, threads>>>(w, steps, out, cyc);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double per = (double)h / steps;
    printf("%s threads=%4d chains/thread=%d : %6.2f cycles/step/chain, %6.2f cycles per 1KiB-round-equivalent\n", name, threads, ch, per,
           per * 256.0 / (threads * ch));
  };
  for (int t : {32, 128, 256}) {
    run(chain<A, 1>, "A wide64", t, 1);
    run(chain<B, 1>, "B lo32+hi", t, 1);
    run(chain<C, 1>, "C wide+mad", t, 1);
    run(chain<B, 2>, "B x2", t, 2);
    run(chain<D, 1>, "D lo32 opaque", t, 1);
    run(chain<D, 2>, "D x2", t, 2);
    run(chain<C, 2>, "C x2", t, 2);
    run(chain<E, 1>, "E shift-add", t, 1);
    run(chain<F, 1>, "F lo only", t, 1);
    run(chain<G, 1>, "G imad+alu", t, 1);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
