// FNV-1a-64 lane chain fed from shared memory (as in the hash kernel):
// cycles per dependent step for several instruction mixes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_lds chain_lds.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ uint32_t g_zero;

struct Cur {  // hash.cu Fnv (IMAD.WIDE + mixed IMAD/LEA + IMAD)
  uint32_t lo, hi, z;
  __device__ void init(uint64_t v) { lo = (uint32_t)v; hi = (uint32_t)(v >> 32); }
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    const uint64_t p = (uint64_t)x * 435u;
    const uint32_t add = (uint32_t)(p >> 32) + (x << 8);
    lo = (uint32_t)p;
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
  }
};
struct LoOnly {
  uint32_t lo, hi, z;
  __device__ void init(uint64_t v) { lo = (uint32_t)v; hi = (uint32_t)(v >> 32); }
  __device__ __forceinline__ void step(uint32_t w) { lo = (lo ^ w) * 435u; }
};
struct Sep {  // IMAD lo on the chain; IMAD.HI on an opaque copy (no merge); LEA; IMAD hi
  uint32_t lo, hi, z;
  __device__ void init(uint64_t v) {
    lo = (uint32_t)v; hi = (uint32_t)(v >> 32);
    asm volatile("ld.global.u32 %0, [%1];" : "=r"(z) : "l"(&g_zero));
  }
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    uint32_t nlo, c, xz, add;
    asm("mul.lo.u32 %0, %1, 435;" : "=r"(nlo) : "r"(x));
    asm("add.u32 %0, %1, %2;" : "=r"(xz) : "r"(x), "r"(z));
    asm("mul.hi.u32 %0, %1, 435;" : "=r"(c) : "r"(xz));
    asm("{ .reg .b32 s; shl.b32 s, %1, 8; add.u32 %0, s, %2; }" : "=r"(add) : "r"(x), "r"(c));
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
    lo = nlo;
  }
};
struct SepZ {  // as Sep but the opaque copy is the LOP3 itself: xz = (lo ^ z) ^ w off the chain
  uint32_t lo, hi, z;
  __device__ void init(uint64_t v) {
    lo = (uint32_t)v; hi = (uint32_t)(v >> 32);
    asm volatile("ld.global.u32 %0, [%1];" : "=r"(z) : "l"(&g_zero));
  }
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    uint32_t nlo, c, xz, add;
    asm("mul.lo.u32 %0, %1, 435;" : "=r"(nlo) : "r"(x));
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(xz) : "r"(lo), "r"(w), "r"(z));
    asm("mul.hi.u32 %0, %1, 435;" : "=r"(c) : "r"(xz));
    asm("{ .reg .b32 s; shl.b32 s, %1, 8; add.u32 %0, s, %2; }" : "=r"(add) : "r"(x), "r"(c));
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
    lo = nlo;
  }
};

// Deferred hi: per block of B words, run the lo chain keeping the x values in
// registers, then fold them into hi (the hi work no longer sits between the
// chain's dependent instructions in the in-order issue stream).
template <int ROWS, int B>
__global__ void chain_defer(int stages, uint64_t *out, long long *cyc) {
  extern __shared__ uint32_t sw[];
  for (int i = threadIdx.x; i < ROWS * blockDim.x; i += blockDim.x) sw[i] = i * 2654435761u;
  __syncthreads();
  uint32_t lo = 0x84222325u ^ threadIdx.x, hi = 0xcbf29ce4u;
  const uint32_t *wds = sw + threadIdx.x;
  long long t0 = clock64();
  for (int s = 0; s < stages; ++s) {
#pragma unroll
    for (int b = 0; b < ROWS; b += B) {
      uint32_t x[B];
#pragma unroll
      for (int r = 0; r < B; ++r) {
        x[r] = lo ^ wds[(b + r) * 128];
        lo = x[r] * 435u;
      }
#pragma unroll
      for (int r = 0; r < B; ++r) hi = hi * 435u + (__umulhi(x[r], 435u) + (x[r] << 8));
    }
    __syncwarp();
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = ((uint64_t)hi << 32) | lo;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

// Software-pipelined: the lo chain of block b and the hi fold of block b-1's
// x values interleave; the hi work is independent of the running chain.
template <int ROWS, int B>
__global__ void chain_pipe(int stages, uint64_t *out, long long *cyc) {
  extern __shared__ uint32_t sw[];
  for (int i = threadIdx.x; i < ROWS * blockDim.x; i += blockDim.x) sw[i] = i * 2654435761u;
  __syncthreads();
  uint32_t lo = 0x84222325u ^ threadIdx.x, hi = 0xcbf29ce4u;
  const uint32_t *wds = sw + threadIdx.x;
  uint32_t xp[B];
#pragma unroll
  for (int r = 0; r < B; ++r) xp[r] = 0;
  long long t0 = clock64();
  for (int s = 0; s < stages; ++s) {
#pragma unroll
    for (int b = 0; b < ROWS; b += B) {
      uint32_t x[B];
#pragma unroll
      for (int r = 0; r < B; ++r) {
        x[r] = lo ^ wds[(b + r) * 128];
        lo = x[r] * 435u;
        hi = hi * 435u + (__umulhi(xp[r], 435u) + (xp[r] << 8));
      }
#pragma unroll
      for (int r = 0; r < B; ++r) xp[r] = x[r];
    }
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < B; ++r) hi = hi * 435u + (__umulhi(xp[r], 435u) + (xp[r] << 8));
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = ((uint64_t)hi << 32) | lo;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

// Split warps: warp w+nw runs the lo chain of lanes [32w, 32w+32) and leaves
// x in place; warp w folds x into hi one stage later (double-buffered stages).
template <int ROWS>
__global__ void chain_split(int stages, uint64_t *out, long long *cyc) {
  extern __shared__ uint32_t sw[];  // 2 x [ROWS][lanes]
  const int lanes = blockDim.x / 2;
  for (int i = threadIdx.x; i < 2 * ROWS * lanes; i += blockDim.x) sw[i] = i * 2654435761u;
  __syncthreads();
  const bool lo_side = threadIdx.x >= lanes;
  const int t = threadIdx.x % lanes;
  uint32_t lo = 0x84222325u ^ t, hi = 0xcbf29ce4u;
  long long t0 = clock64();
  for (int s = 0; s <= stages; ++s) {
    uint32_t *buf = sw + (s & 1) * ROWS * lanes + t;
    if (lo_side) {
      if (s < stages) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          const uint32_t x = lo ^ buf[r * lanes];
          buf[r * lanes] = x;
          lo = x * 435u;
        }
      }
    } else if (s > 0) {
      uint32_t *pb = sw + ((s - 1) & 1) * ROWS * lanes + t;
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        const uint32_t x = pb[r * lanes];
        hi = hi * 435u + (__umulhi(x, 435u) + (x << 8));
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (!lo_side) out[threadIdx.x] = hi;
  else out[threadIdx.x] = lo;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <class F, int ROWS>
__global__ void chain(int stages, uint64_t *out, long long *cyc) {
  extern __shared__ uint32_t sw[];  // [ROWS][blockDim]
  for (int i = threadIdx.x; i < ROWS * blockDim.x; i += blockDim.x) sw[i] = i * 2654435761u;
  __syncthreads();
  F f;
  f.init(0xcbf29ce484222325ull ^ threadIdx.x);
  const uint32_t *wds = sw + threadIdx.x;
  long long t0 = clock64();
  for (int s = 0; s < stages; ++s) {
#pragma unroll
    for (int r = 0; r < ROWS; ++r) f.step(wds[r * blockDim.x]);
    __syncwarp();
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = ((uint64_t)f.hi << 32) | f.lo;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  uint64_t *out; long long *cyc;
  cudaMalloc(&out, 1 << 22); cudaMalloc(&cyc, 8);
  const int stages = 4096, ROWS = 64;
  auto run = [&](auto kern, const char *name, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    kern<<<1, threads, ROWS * threads * 4>>>(stages, out, cyc);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-8s threads=%3d : %6.2f cycles/step\n", name, threads, (double)h / (stages * ROWS));
  };
  auto runr = [&](auto kern, const char *name, int threads, int rows) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    kern<<<1, threads, rows * threads * 4>>>(stages / 4, out, cyc);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-8s threads=%3d rows=%3d : %6.2f cycles/step\n", name, threads, rows, (double)h / (stages / 4 * rows));
  };
  // phase-1 shape: 64 lanes, 256 rows unrolled per stage
  runr(chain<LoOnly, 256>, "lo-only", 64, 256);
  runr(chain<LoOnly, 128>, "lo-only", 64, 128);
  runr(chain<LoOnly, 64>, "lo-only", 64, 64);
  runr(chain<LoOnly, 256>, "lo-only", 96, 256);
  for (int t : {128}) {
    run(chain<Cur, 64>, "cur", t);
    run(chain<LoOnly, 64>, "lo-only", t);
    run(chain<Sep, 64>, "sep", t);
    run(chain<SepZ, 64>, "sepz", t);
    run(chain_defer<64, 16>, "defer16", t);
    run(chain_defer<64, 32>, "defer32", t);
    run(chain_defer<64, 64>, "defer64", t);
    run(chain_pipe<64, 8>, "pipe8", t);
    run(chain_pipe<64, 16>, "pipe16", t);
    run(chain_pipe<64, 32>, "pipe32", t);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
