// simplehash on B200 (sharedstate.py:45-128).
//
// Definition: buffer as little-endian u32 words (tail zero-padded); word i
// feeds lane i mod 256, each lane runs FNV-1a-64 h = (h ^ w) * P from the
// offset basis; lanes fold by a depth-8 tree (a ^ rotl(b, 27)) * P over pairs
// (2j, 2j+1); root ^ byte length.
//
// Mapping: one 256-thread CTA per entry, thread t = lane t, so a warp reads
// 128 contiguous bytes per round and every chain stays in one register pair.
// Entries stream HBM -> shared memory through a 4-stage ring of 16 KiB TMA
// bulk copies (cp.async.bulk + mbarrier complete_tx), issued by one thread,
// so the per-word chain reads shared memory instead of waiting on DRAM.
// A single entry is bounded by the chain latency (LOP3 -> IMAD.WIDE per word
// and lane); many entries in flight make the launch HBM-bound,
// hence the multi-entry launch with largest-first static assignment.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <numeric>
#include <vector>

#include "common.cuh"

namespace pcclb {

constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr int kHashThreads = 256;
constexpr int kStageBytes = 16384;  // 16 rounds of 1 KiB
constexpr int kStages = 4;
constexpr int kHashSmem = kStageBytes * kStages;
constexpr int kMaxBatch = 1024;

struct HashEntry {
  const uint8_t *ptr;
  uint64_t nbytes;
  uint64_t *out;
};

struct HashBatch {
  uint32_t count;
  uint32_t pad;
  HashEntry e[kMaxBatch];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// One FNV-1a-64 step h = (h ^ w) * P on the split state (lo, hi).
// P = 2^40 + 435 and w is a zero-extended u32, so with x = lo ^ w:
//   lo' = (x * 435) mod 2^32
//   hi' = hi * 435 + floor(x * 435 / 2^32) + (x << 8)     (mod 2^32)
// The loop-carried paths are LOP3 -> IMAD.WIDE on lo and a single IMAD on hi
// (the x-dependent addend is computed off the hi chain).
struct Fnv {
  uint32_t lo, hi;
  __device__ __forceinline__ explicit Fnv(uint64_t h) : lo((uint32_t)h), hi((uint32_t)(h >> 32)) {}
  __device__ __forceinline__ uint64_t value() const { return ((uint64_t)hi << 32) | lo; }
  __device__ __forceinline__ void step(uint32_t w) {
    const uint32_t x = lo ^ w;
    const uint64_t p = (uint64_t)x * 435u;
    const uint32_t add = (uint32_t)(p >> 32) + (x << 8);
    lo = (uint32_t)p;
    // explicit mad so the compiler cannot re-associate x-terms onto the hi chain
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(add));
  }
};
__device__ __forceinline__ uint64_t fnv_step(uint64_t h, uint32_t w) {
  return (h ^ (uint64_t)w) * kFnvPrime;
}
__device__ __forceinline__ uint64_t rotl27(uint64_t v) { return (v << 27) | (v >> 37); }

// little-endian u32 at an arbitrary byte address (zero beyond `avail` bytes)
__device__ __forceinline__ uint32_t load_word_any(const uint8_t *p, uint32_t avail) {
  if (avail >= 4 && ((uintptr_t)p & 3) == 0) return __ldg(reinterpret_cast<const uint32_t *>(p));
  uint32_t w = 0;
  for (uint32_t b = 0; b < 4 && b < avail; ++b) w |= (uint32_t)__ldg(p + b) << (8 * b);
  return w;
}

// Run every lane of one segment. Lane t = threadIdx.x; h is that lane's state.
// Must be called by all 256 threads of the CTA (uses __syncthreads).
__device__ __forceinline__ uint64_t hash_segment(const uint8_t *p, uint64_t nbytes, uint64_t h,
                                                 uint8_t *stage, uint64_t *bars,
                                                 uint32_t &parity) {
  const int tid = threadIdx.x;
  const uint64_t full_words = nbytes >> 2;
  const uint64_t rounds = full_words >> 8;
  if (rounds > 0 && ((uintptr_t)p & 15) == 0) {
    const uint64_t bulk = rounds << 10;
    const uint64_t nst = (bulk + kStageBytes - 1) / kStageBytes;
    if (tid == 0) {
      for (uint64_t s = 0; s < nst && s < (uint64_t)kStages; ++s) {
        uint32_t bytes = (uint32_t)min((uint64_t)kStageBytes, bulk - s * kStageBytes);
        mbar_expect_tx(&bars[s], bytes);
        bulk_g2s(stage + s * kStageBytes, p + s * kStageBytes, bytes, &bars[s]);
      }
    }
    for (uint64_t st = 0; st < nst; ++st) {
      const int slot = (int)(st % kStages);
      mbar_wait(&bars[slot], (parity >> slot) & 1u);
      parity ^= 1u << slot;
      const uint32_t *wds = reinterpret_cast<const uint32_t *>(stage + slot * kStageBytes) + tid;
      const uint64_t left = bulk - st * kStageBytes;
      Fnv f(h);
      if (left >= (uint64_t)kStageBytes) {
#pragma unroll
        for (int r = 0; r < kStageBytes / 1024; ++r) f.step(wds[r * 256]);
      } else {
        const int nr = (int)(left >> 10);
        for (int r = 0; r < nr; ++r) f.step(wds[r * 256]);
      }
      h = f.value();
      __syncthreads();  // every lane done with this slot before it is refilled
      if (tid == 0 && st + kStages < nst) {
        const uint64_t s = st + kStages;
        uint32_t bytes = (uint32_t)min((uint64_t)kStageBytes, bulk - s * kStageBytes);
        mbar_expect_tx(&bars[slot], bytes);
        bulk_g2s(stage + slot * kStageBytes, p + s * kStageBytes, bytes, &bars[slot]);
      }
    }
  } else {
    for (uint64_t r = 0; r < rounds; ++r) h = fnv_step(h, load_word_any(p + ((r << 8) + tid) * 4, 4));
  }
  const uint64_t done = rounds << 8;
  const uint64_t rem = full_words - done;  // < 256
  const uint8_t *q = p + done * 4;
  if ((uint64_t)tid < rem) h = fnv_step(h, load_word_any(q + 4 * tid, 4));
  const uint32_t tail = (uint32_t)(nbytes & 3);
  if (tail && (uint64_t)tid == rem) h = fnv_step(h, load_word_any(q + 4 * tid, tail));
  return h;
}

// depth-8 tree over lanes in shared memory; returns root (valid in thread 0)
__device__ __forceinline__ uint64_t tree_fold(uint64_t *lane_s, uint64_t h) {
  const int tid = threadIdx.x;
  lane_s[tid] = h;
  __syncthreads();
  for (int width = 128; width >= 1; width >>= 1) {
    uint64_t v = 0;
    if (tid < width) v = (lane_s[2 * tid] ^ rotl27(lane_s[2 * tid + 1])) * kFnvPrime;
    __syncthreads();
    if (tid < width) lane_s[tid] = v;
    __syncthreads();
  }
  return lane_s[0];
}

__global__ void __launch_bounds__(kHashThreads) simplehash_batch_kernel(const __grid_constant__ HashBatch b) {
  extern __shared__ __align__(1024) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ uint64_t lane_s[kHashThreads];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t parity = 0;
  for (uint32_t e = blockIdx.x; e < b.count; e += gridDim.x) {
    const HashEntry E = b.e[e];
    uint64_t h = hash_segment(E.ptr, E.nbytes, kFnvOffset, stage, bars, parity);
    uint64_t root = tree_fold(lane_s, h);
    if (threadIdx.x == 0) *E.out = root ^ E.nbytes;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kHashThreads)
    simplehash_update_kernel(uint64_t *state, const uint8_t *p, uint64_t nbytes) {
  extern __shared__ __align__(1024) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t parity = 0;
  uint64_t h = state[threadIdx.x];
  h = hash_segment(p, nbytes, h, stage, bars, parity);
  state[threadIdx.x] = h;
}

__global__ void simplehash_init_kernel(uint64_t *state) { state[threadIdx.x] = kFnvOffset; }

__global__ void __launch_bounds__(kHashThreads)
    simplehash_final_kernel(const uint64_t *state, uint64_t total, uint64_t *out) {
  __shared__ uint64_t lane_s[kHashThreads];
  uint64_t root = tree_fold(lane_s, state[threadIdx.x]);
  if (threadIdx.x == 0) *out = root ^ total;
}

static int prepare_hash_kernels() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  PCCLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && done[dev]) return PCCLB_OK;
  PCCLB_CUDA(cudaFuncSetAttribute(simplehash_batch_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem));
  PCCLB_CUDA(cudaFuncSetAttribute(simplehash_update_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem));
  if (dev >= 0 && dev < 64) done[dev] = true;
  return PCCLB_OK;
}

}  // namespace pcclb

using namespace pcclb;

extern "C" {

int pcclb_simplehash_multi(const void *const *h_ptrs, const uint64_t *h_nbytes, uint32_t count,
                           uint64_t *d_out, void *stream) {
  if (count == 0) return PCCLB_OK;
  if (!h_ptrs || !h_nbytes || !d_out) return PCCLB_EINVAL;
  for (uint32_t i = 0; i < count; ++i)
    if (h_nbytes[i] && !h_ptrs[i]) return PCCLB_EINVAL;
  int rc = prepare_hash_kernels();
  if (rc) return rc;
  // largest first: the longest chains start first (LPT order)
  std::vector<uint32_t> order(count);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t a, uint32_t b) { return h_nbytes[a] > h_nbytes[b]; });
  cudaStream_t s = as_stream(stream);
  int occ = 0;
  PCCLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, simplehash_batch_kernel,
                                                           kHashThreads, kHashSmem));
  if (occ < 1) occ = 1;
  const uint32_t slots = (uint32_t)(sm_count() * occ);
  static thread_local HashBatch batch;
  for (uint32_t base = 0; base < count; base += kMaxBatch) {
    uint32_t m = std::min<uint32_t>(kMaxBatch, count - base);
    batch.count = m;
    for (uint32_t i = 0; i < m; ++i) {
      uint32_t k = order[base + i];
      batch.e[i].ptr = static_cast<const uint8_t *>(h_ptrs[k]);
      batch.e[i].nbytes = h_nbytes[k];
      batch.e[i].out = d_out + k;
    }
    unsigned grid = std::min<uint32_t>(m, slots);
    simplehash_batch_kernel<<<grid, kHashThreads, kHashSmem, s>>>(batch);
    PCCLB_LAUNCH_CHECK();
  }
  return PCCLB_OK;
}

int pcclb_simplehash(const void *d_data, uint64_t nbytes, uint64_t *d_out, void *stream) {
  return pcclb_simplehash_multi(&d_data, &nbytes, 1, d_out, stream);
}

int pcclb_simplehash_init(uint64_t *d_state, void *stream) {
  if (!d_state) return PCCLB_EINVAL;
  simplehash_init_kernel<<<1, kHashThreads, 0, as_stream(stream)>>>(d_state);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

int pcclb_simplehash_update(uint64_t *d_state, const void *d_data, uint64_t nbytes, void *stream) {
  if (!d_state || (nbytes && !d_data)) return PCCLB_EINVAL;
  if (nbytes == 0) return PCCLB_OK;
  int rc = prepare_hash_kernels();
  if (rc) return rc;
  simplehash_update_kernel<<<1, kHashThreads, kHashSmem, as_stream(stream)>>>(
      d_state, static_cast<const uint8_t *>(d_data), nbytes);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

int pcclb_simplehash_final(const uint64_t *d_state, uint64_t total_nbytes, uint64_t *d_out,
                           void *stream) {
  if (!d_state || !d_out) return PCCLB_EINVAL;
  simplehash_final_kernel<<<1, kHashThreads, 0, as_stream(stream)>>>(d_state, total_nbytes, d_out);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

}  // extern "C"
