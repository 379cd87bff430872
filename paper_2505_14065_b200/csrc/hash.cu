// simplehash on B200 (sharedstate.py:45-128).
//
// Definition: buffer as little-endian u32 words (tail zero-padded); word i
// feeds lane i mod 256, each lane runs FNV-1a-64 h = (h ^ w) * P from the
// offset basis; lanes fold by a depth-8 tree (a ^ rotl(b, 27)) * P over pairs
// (2j, 2j+1); root ^ byte length.
//
// Bounds (measured, tools/micro/chain_micro.cu): one FNV step is a dependent
// LOP3 -> IMAD.WIDE pair of ~14.3 cycles, so one entry (256 chains) cannot go
// faster than 1 KiB per 14.3 cycles (~141 GB/s at 1.97 GHz) however many SMs
// it gets; an SM issues at most ~1 KiB of steps per ~13.4 cycles (~150 GB/s),
// so the whole chip (~22 TB/s) is far above HBM. Many entries in flight are
// therefore HBM-bound, and the largest entry sets a latency floor.
//
// Mapping (default): an entry's 256 lanes are split over kGroups = 2 CTAs of
// 128 threads (thread t = lane 128g + t), each on its own SM, so a lone large
// entry runs at its chain bound. A CTA streams its 512-byte slice of every
// 1 KiB round through a 3-stage shared-memory ring; each stage (64 rounds) is
// ONE 2-D TMA copy (cp.async.bulk.tensor.2d, the entry viewed as a
// [rounds x 256] u32 tensor, box 128 x 64) completing on an mbarrier.
// Entries are dealt largest first, so the longest chains start first; the
// last group of an entry to finish runs the tree fold.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <vector>

#include "common.cuh"

namespace pcclb {

constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr int kMaxBatch = 1000;  // HashBatch must fit the 32 KiB kernel-parameter space
#ifndef HASH_UNROLL
#define HASH_UNROLL 0  // 0: fully unrolled (measured best: 64 > 32 > 16 > 8)
#endif
constexpr int kHashUnroll = HASH_UNROLL;  // unroll of the per-stage chain loop  // HashBatch must fit the 32 KiB kernel-parameter space

struct HashEntry {
  const uint8_t *ptr;
  uint64_t nbytes;
  uint64_t *out;
  const CUtensorMap *map;  // 2-D view [rounds x 256] u32, or null (fallback loads)
};

struct HashBatch {
  uint32_t count;
  uint32_t dynamic;  // 1: items from an atomic counter (list scheduling), 0: grid-stride
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
__device__ __forceinline__ void tma_2d_g2s(void *dst, const CUtensorMap *map, int x, int y,
                                           uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tensormap_acquire(const CUtensorMap *map) {
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(map) : "memory");
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

// Kernel shape: LANES threads per CTA (thread t = lane lane0 + t), a ring of
// STAGES shared-memory stages of ROWS rounds each; a stage holds the CTA's
// LANES*4-byte slice of ROWS consecutive 1 KiB rounds. TMA2D: stages are
// filled by one 2-D tensor copy; otherwise (LANES == 256 only) by one 1-D
// bulk copy of ROWS contiguous KiB.
template <int LANES_, int ROWS_, int STAGES_, bool TMA2D_, bool PROD_ = false>
struct HashCfg {
  static constexpr int LANES = LANES_;
  static constexpr int ROWS = ROWS_;
  static constexpr int STAGES = STAGES_;
  static constexpr bool TMA2D = TMA2D_;
  // PROD: one extra warp issues the TMA stages; the lane warps release slots
  // through per-slot "empty" mbarriers instead of a CTA-wide barrier per stage
  static constexpr bool PROD = PROD_;
  static constexpr int THREADS = LANES + (PROD ? 32 : 0);
  static constexpr int GROUPS = 256 / LANES;
  static constexpr int SLICE = LANES * 4;
  static constexpr int STAGE_BYTES = ROWS * SLICE;
  static constexpr int SMEM = STAGE_BYTES * STAGES;
  static_assert(TMA2D || LANES == 256, "1-D bulk stages need whole rounds");
  static_assert(!PROD || TMA2D, "the producer warp issues 2-D TMA boxes");
};

// Run lanes [lane0, lane0 + LANES) of one segment; h is the lane's state.
// Must be called by all threads of the CTA (uses __syncthreads).
template <class C>
__device__ __forceinline__ uint64_t hash_group(const uint8_t *p, uint64_t nbytes,
                                               const CUtensorMap *map, uint32_t lane0, uint64_t h,
                                               uint8_t *stage, uint64_t *bars, uint32_t &parity) {
  const int tid = threadIdx.x;
  const uint32_t lane = lane0 + tid;
  const uint64_t full_words = nbytes >> 2;
  const uint64_t rounds = full_words >> 8;
  const bool fast = rounds > 0 && (C::TMA2D ? map != nullptr : ((uintptr_t)p & 15) == 0);
  if (fast) {
    const uint64_t nst = (rounds + C::ROWS - 1) / C::ROWS;
    auto issue = [&](uint64_t s, int slot) {  // called by thread 0
      uint8_t *dst = stage + slot * C::STAGE_BYTES;
      if constexpr (C::TMA2D) {
        // out-of-range rows of the last box are zero-filled and still counted
        mbar_expect_tx(&bars[slot], C::STAGE_BYTES);
        tma_2d_g2s(dst, map, (int)lane0, (int)(s * C::ROWS), &bars[slot]);
      } else {
        const uint32_t rows = (uint32_t)min((uint64_t)C::ROWS, rounds - s * C::ROWS);
        mbar_expect_tx(&bars[slot], rows * 1024);
        bulk_g2s(dst, p + s * C::ROWS * 1024, rows * 1024, &bars[slot]);
      }
    };
    if (tid == 0) {
      if constexpr (C::TMA2D) tensormap_acquire(map);
      for (uint64_t s = 0; s < nst && s < (uint64_t)C::STAGES; ++s) issue(s, (int)s);
    }
    for (uint64_t st = 0; st < nst; ++st) {
      const int slot = (int)(st % C::STAGES);
      mbar_wait(&bars[slot], (parity >> slot) & 1u);
      parity ^= 1u << slot;
      const uint32_t *wds = reinterpret_cast<const uint32_t *>(stage + slot * C::STAGE_BYTES) + tid;
      const uint64_t left = rounds - st * C::ROWS;
      Fnv f(h);
      if (left >= (uint64_t)C::ROWS) {
        if constexpr (kHashUnroll == 0) {
          // fully unrolled: the compiler hoists the shared-memory loads well
          // ahead of the chain (config 4: 10.75 ms vs 11.85 ms at unroll 16)
#pragma unroll
          for (int r = 0; r < C::ROWS; ++r) f.step(wds[r * C::LANES]);
        } else {
#pragma unroll kHashUnroll
          for (int r = 0; r < C::ROWS; ++r) f.step(wds[r * C::LANES]);
        }
      } else {
        const int nr = (int)left;
        for (int r = 0; r < nr; ++r) f.step(wds[r * C::LANES]);
      }
      h = f.value();
      __syncthreads();  // every lane done with this slot before it is refilled
      if (tid == 0 && st + C::STAGES < nst) issue(st + C::STAGES, slot);
    }
  } else {
    for (uint64_t r = 0; r < rounds; ++r) h = fnv_step(h, load_word_any(p + ((r << 8) + lane) * 4, 4));
  }
  const uint64_t done = rounds << 8;
  const uint64_t rem = full_words - done;  // < 256
  const uint8_t *q = p + done * 4;
  if ((uint64_t)lane < rem) h = fnv_step(h, load_word_any(q + 4 * lane, 4));
  const uint32_t tail = (uint32_t)(nbytes & 3);
  if (tail && (uint64_t)lane == rem) h = fnv_step(h, load_word_any(q + 4 * lane, tail));
  return h;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// hash_group with a producer warp (C::PROD, blockDim = LANES + 32). Thread
// LANES issues every stage of the lane group into a ring slot once the lane
// warps released it (empty[slot], one arrival per lane warp); lane warps wait
// for full[slot] and never synchronise with each other, so one slow warp no
// longer holds the other three at a per-stage __syncthreads. `g` numbers the
// stages of the whole launch (it carries over from one entry to the next), so
// slot = g % STAGES and the mbarrier phase parity is (g / STAGES) & 1.
template <class C>
__device__ __forceinline__ uint64_t hash_group_prod(const uint8_t *p, uint64_t nbytes,
                                                    const CUtensorMap *map, uint32_t lane0,
                                                    uint64_t h, uint8_t *stage, uint64_t *full,
                                                    uint64_t *empty, uint32_t &g) {
  const int tid = threadIdx.x;
  const bool producer = tid >= C::LANES;
  const uint32_t lane = lane0 + tid;
  const uint64_t full_words = nbytes >> 2;
  const uint64_t rounds = full_words >> 8;
  if (rounds > 0 && map != nullptr) {
    const uint32_t nst = (uint32_t)((rounds + C::ROWS - 1) / C::ROWS);
    if (producer) {
      if (tid == C::LANES) {
        tensormap_acquire(map);
        for (uint32_t s = 0; s < nst; ++s) {
          const uint32_t G = g + s, slot = G % C::STAGES;
          if (G >= (uint32_t)C::STAGES) mbar_wait(&empty[slot], ((G / C::STAGES) - 1) & 1u);
          mbar_expect_tx(&full[slot], C::STAGE_BYTES);
          tma_2d_g2s(stage + slot * C::STAGE_BYTES, map, (int)lane0, (int)(s * C::ROWS), &full[slot]);
        }
      }
    } else {
      for (uint32_t s = 0; s < nst; ++s) {
        const uint32_t G = g + s, slot = G % C::STAGES;
        mbar_wait(&full[slot], (G / C::STAGES) & 1u);
        const uint32_t *wds = reinterpret_cast<const uint32_t *>(stage + slot * C::STAGE_BYTES) + tid;
        const uint64_t left = rounds - (uint64_t)s * C::ROWS;
        Fnv f(h);
        if (left >= (uint64_t)C::ROWS) {
#pragma unroll
          for (int r = 0; r < C::ROWS; ++r) f.step(wds[r * C::LANES]);
        } else {
          const int nr = (int)left;
          for (int r = 0; r < nr; ++r) f.step(wds[r * C::LANES]);
        }
        h = f.value();
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
      }
    }
    g += nst;
  } else if (!producer) {
    for (uint64_t r = 0; r < rounds; ++r) h = fnv_step(h, load_word_any(p + ((r << 8) + lane) * 4, 4));
  }
  if (producer) return 0;
  const uint64_t done = rounds << 8;
  const uint64_t rem = full_words - done;  // < 256
  const uint8_t *q = p + done * 4;
  if ((uint64_t)lane < rem) h = fnv_step(h, load_word_any(q + 4 * lane, 4));
  const uint32_t tail = (uint32_t)(nbytes & 3);
  if (tail && (uint64_t)lane == rem) h = fnv_step(h, load_word_any(q + 4 * lane, tail));
  return h;
}

// depth-8 tree over 256 lanes in shared memory (pairs (2j, 2j+1), lower is a);
// CTA size >= 64; returns the root in every thread
__device__ __forceinline__ uint64_t tree_fold(uint64_t *lane_s) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __syncthreads();
  for (int width = 128; width >= 1; width >>= 1) {
    uint64_t v0 = 0, v1 = 0;
    if (tid < width) v0 = (lane_s[2 * tid] ^ rotl27(lane_s[2 * tid + 1])) * kFnvPrime;
    if (tid + nt < width) v1 = (lane_s[2 * (tid + nt)] ^ rotl27(lane_s[2 * (tid + nt) + 1])) * kFnvPrime;
    __syncthreads();
    if (tid < width) lane_s[tid] = v0;
    if (tid + nt < width) lane_s[tid + nt] = v1;
    __syncthreads();
  }
  return lane_s[0];
}

template <class C>
__device__ __forceinline__ void init_bars(uint64_t *bars) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[s], 1);
    if constexpr (C::PROD)
      for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[C::STAGES + s], C::LANES / 32);
    mbar_fence_init();
  }
  __syncthreads();
}

template <class C>
__device__ __forceinline__ uint64_t hash_any(const uint8_t *p, uint64_t nbytes, const CUtensorMap *map,
                                             uint32_t lane0, uint64_t h, uint8_t *stage, uint64_t *bars,
                                             uint32_t &sync) {
  if constexpr (C::PROD)
    return hash_group_prod<C>(p, nbytes, map, lane0, h, stage, bars, bars + C::STAGES, sync);
  else
    return hash_group<C>(p, nbytes, map, lane0, h, stage, bars, sync);
}

// Work item = (entry, lane group); the last group of an entry folds.
template <class C>
__global__ void __launch_bounds__(C::THREADS)
    simplehash_batch_kernel(const __grid_constant__ HashBatch b, uint64_t *lanes, uint32_t *arrived) {
  extern __shared__ __align__(1024) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[2 * C::STAGES];
  __shared__ uint64_t lane_s[256];
  __shared__ uint32_t s_last;
  init_bars<C>(bars);
  uint32_t parity = 0;
  const uint32_t items = b.count * C::GROUPS;
  // dynamic list scheduling: items are taken in LPT order (largest entries
  // first) by whichever CTA is free, from a counter behind the arrival counts
  uint32_t *next = arrived + b.count;
  __shared__ uint32_t s_item;
  for (uint32_t k = 0;; ++k) {
    if (b.dynamic) {
      if (threadIdx.x == 0) s_item = atomicAdd(next, 1u);
      __syncthreads();
    }
    const uint32_t it = b.dynamic ? s_item : blockIdx.x + k * gridDim.x;
    if (it >= items) break;
    const uint32_t e = it / C::GROUPS, g = it % C::GROUPS;
    const HashEntry E = b.e[e];
    const uint32_t lane0 = g * C::LANES;
    uint64_t h = hash_any<C>(E.ptr, E.nbytes, E.map, lane0, kFnvOffset, stage, bars, parity);
    if constexpr (C::GROUPS == 1) {
      if (threadIdx.x < C::LANES) lane_s[threadIdx.x] = h;
      uint64_t root = tree_fold(lane_s);
      if (threadIdx.x == 0) *E.out = root ^ E.nbytes;
    } else {
      if (threadIdx.x < C::LANES) lanes[(uint64_t)e * 256 + lane0 + threadIdx.x] = h;
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = (atomicAdd(&arrived[e], 1u) == C::GROUPS - 1) ? 1u : 0u;
      __syncthreads();
      if (s_last) {
        __threadfence();
        for (int j = threadIdx.x; j < 256; j += blockDim.x)
          lane_s[j] = __ldcg(&lanes[(uint64_t)e * 256 + j]);
        uint64_t root = tree_fold(lane_s);
        if (threadIdx.x == 0) *E.out = root ^ E.nbytes;
      }
    }
    __syncthreads();
  }
}

// streaming update of one segment: grid = GROUPS CTAs, lane state in/out
template <class C>
__global__ void __launch_bounds__(C::THREADS)
    simplehash_update_kernel(uint64_t *state, const uint8_t *p, uint64_t nbytes,
                             const __grid_constant__ CUtensorMap map, int have_map) {
  extern __shared__ __align__(1024) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[2 * C::STAGES];
  init_bars<C>(bars);
  uint32_t parity = 0;
  const uint32_t lane = blockIdx.x * C::LANES + (threadIdx.x % C::LANES);
  uint64_t h = hash_any<C>(p, nbytes, have_map ? &map : nullptr, blockIdx.x * C::LANES,
                           state[lane], stage, bars, parity);
  if (threadIdx.x < C::LANES) state[lane] = h;
}

__global__ void simplehash_init_kernel(uint64_t *state) { state[threadIdx.x] = kFnvOffset; }

__global__ void __launch_bounds__(256)
    simplehash_final_kernel(const uint64_t *state, uint64_t total, uint64_t *out) {
  __shared__ uint64_t lane_s[256];
  lane_s[threadIdx.x] = state[threadIdx.x];
  uint64_t root = tree_fold(lane_s);
  if (threadIdx.x == 0) *out = root ^ total;
}

// Variants (env PCCLB_HASH_VARIANT, for experiments; 0 is the default),
// measured on B200 with list scheduling (config-4 layout / one 1.05 GB entry /
// 64 x 64 MiB, tools/hash_variants.py, median of 7):
//   <128,128,3,P>  8.5 ms / 131 GB/s / 7.1 TB/s   (default)
//   <64,128,4,P>   8.2 ms / 128 GB/s / 4.0 TB/s   (64 lanes per SM: HBM-starved)
//   <128,64,3>    12.5 ms / 111 GB/s / 6.7 TB/s   (no producer warp; 10.6 ms grid-stride)
//   <128,96,4,P>   9.0 ms / 123 GB/s / 7.1 TB/s
// One entry is bounded by its lane chain (14.5 cycles per LOP3->IMAD.WIDE
// step with the hi side interleaved, tools/micro/chain_lds.cu): 1 KiB per step
// => 139 GB/s, 7.6 ms for the 1.05 GB embedding. Deep stages (128 rows) keep
// ~2 us of TMA lookahead per CTA and amortise the per-stage handshakes.
using HashV0 = HashCfg<128, 128, 3, true, true>;
using HashV1 = HashCfg<64, 128, 4, true, true>;
using HashV2 = HashCfg<128, 64, 3, true>;
using HashV3 = HashCfg<128, 96, 4, true, true>;
static bool hash_dynamic() {
  static bool on = [] {
    const char *e = getenv("PCCLB_HASH_DYN");
    return !(e && e[0] == '0');
  }();
  return on;
}

int hash_variant() {
  static int v = [] {
    const char *e = getenv("PCCLB_HASH_VARIANT");
    int x = e ? atoi(e) : 0;
    return (x < 0 || x > 3) ? 0 : x;
  }();
  return v;
}

// ---------------------------------------------------------------------------
// host: tensor maps
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// [rounds x 256] u32 view of an entry, box LANES x ROWS; false if not encodable
template <class C>
static bool encode_map(CUtensorMap *m, const void *p, uint64_t nbytes) {
  const uint64_t rounds = (nbytes >> 2) >> 8;
  if (!rounds || (reinterpret_cast<uintptr_t>(p) & 15) || rounds >= (1ull << 31)) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {256, rounds};
  cuuint64_t strides[1] = {1024};
  cuuint32_t box[2] = {(cuuint32_t)C::LANES, (cuuint32_t)C::ROWS};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(p), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// pinned staging for tensor maps, reused once the previous upload finished
struct MapStaging {
  CUtensorMap *host = nullptr;
  cudaEvent_t done = nullptr;
  ~MapStaging() {
    if (host) cudaFreeHost(host);
    if (done) cudaEventDestroy(done);
  }
};

template <class C>
static int prepare_variant() {
  PCCLB_CUDA(cudaFuncSetAttribute(simplehash_batch_kernel<C>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  PCCLB_CUDA(cudaFuncSetAttribute(simplehash_update_kernel<C>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  return PCCLB_OK;
}

static int prepare_hash_kernels() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  PCCLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && done[dev]) return PCCLB_OK;
  int rc = prepare_variant<HashV0>();
  if (!rc) rc = prepare_variant<HashV1>();
  if (!rc) rc = prepare_variant<HashV2>();
  if (!rc) rc = prepare_variant<HashV3>();
  if (rc) return rc;
  if (dev >= 0 && dev < 64) done[dev] = true;
  return PCCLB_OK;
}

template <class C>
static int launch_batches(const std::vector<uint32_t> &order, const void *const *h_ptrs,
                          const uint64_t *h_nbytes, uint64_t *d_out, cudaStream_t s) {
  const uint32_t count = (uint32_t)order.size();
  if (count == 0) return PCCLB_OK;
  int occ = 0;
  PCCLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, simplehash_batch_kernel<C>,
                                                           C::THREADS, C::SMEM));
  if (occ < 1) occ = 1;
  const uint32_t slots = (uint32_t)(sm_count() * occ);
  // per-launch device scratch: lane values, arrival counters, tensor maps
  const uint32_t m_max = std::min<uint32_t>(kMaxBatch, count);
  const size_t lanes_bytes = (size_t)m_max * 256 * sizeof(uint64_t);
  const size_t cnt_bytes = ((size_t)(m_max + 1) * sizeof(uint32_t) + 127) & ~size_t(127);
  const size_t map_bytes = C::TMA2D ? (size_t)m_max * sizeof(CUtensorMap) : 0;
  char *scratch = nullptr;
  PCCLB_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&scratch), lanes_bytes + cnt_bytes + map_bytes, s));
  uint64_t *lanes = reinterpret_cast<uint64_t *>(scratch);
  uint32_t *arrived = reinterpret_cast<uint32_t *>(scratch + lanes_bytes);
  CUtensorMap *d_maps = reinterpret_cast<CUtensorMap *>(scratch + lanes_bytes + cnt_bytes);
  static thread_local HashBatch batch;
  static thread_local MapStaging staging;
  int rc = PCCLB_OK;
  for (uint32_t base = 0; base < count && rc == PCCLB_OK; base += kMaxBatch) {
    const uint32_t m = std::min<uint32_t>(kMaxBatch, count - base);
    if (C::TMA2D) {
      if (!staging.host) {
        cudaError_t e = cudaHostAlloc(&staging.host, sizeof(CUtensorMap) * kMaxBatch, cudaHostAllocDefault);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&staging.done, cudaEventDisableTiming);
        if (e != cudaSuccess) {
          rc = cuda_status(e);
          break;
        }
      } else {
        cudaEventSynchronize(staging.done);  // previous upload out of the staging area
      }
    }
    batch.count = m;
    batch.dynamic = hash_dynamic() ? 1u : 0u;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t k = order[base + i];
      HashEntry &E = batch.e[i];
      E.ptr = static_cast<const uint8_t *>(h_ptrs[k]);
      E.nbytes = h_nbytes[k];
      E.out = d_out + k;
      E.map = nullptr;
      if (C::TMA2D && encode_map<C>(&staging.host[i], E.ptr, E.nbytes)) E.map = d_maps + i;
    }
    cudaError_t e = cudaSuccess;
    if (C::TMA2D) {
      e = cudaMemcpyAsync(d_maps, staging.host, sizeof(CUtensorMap) * m, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaEventRecord(staging.done, s);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(arrived, 0, (m + 1) * sizeof(uint32_t), s);
    if (e != cudaSuccess) {
      rc = cuda_status(e);
      break;
    }
    unsigned grid = std::min<uint32_t>(m * C::GROUPS, slots);
    simplehash_batch_kernel<C><<<grid, C::THREADS, C::SMEM, s>>>(batch, lanes, arrived);
    e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_status(e);
  }
  cudaError_t e = cudaFreeAsync(scratch, s);
  if (rc == PCCLB_OK && e != cudaSuccess) rc = cuda_status(e);
  return rc;
}

template <class C>
static int launch_update(uint64_t *state, const void *d, uint64_t nbytes, cudaStream_t s) {
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  int have = (C::TMA2D && encode_map<C>(&map, d, nbytes)) ? 1 : 0;
  simplehash_update_kernel<C><<<C::GROUPS, C::THREADS, C::SMEM, s>>>(
      state, static_cast<const uint8_t *>(d), nbytes, map, have);
  PCCLB_LAUNCH_CHECK();
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
  switch (hash_variant()) {
    case 1:
      return launch_batches<HashV1>(order, h_ptrs, h_nbytes, d_out, s);
    case 2:
      return launch_batches<HashV2>(order, h_ptrs, h_nbytes, d_out, s);
    case 3:
      return launch_batches<HashV3>(order, h_ptrs, h_nbytes, d_out, s);
    default:
      return launch_batches<HashV0>(order, h_ptrs, h_nbytes, d_out, s);
  }
}

int pcclb_simplehash(const void *d_data, uint64_t nbytes, uint64_t *d_out, void *stream) {
  return pcclb_simplehash_multi(&d_data, &nbytes, 1, d_out, stream);
}

int pcclb_simplehash_init(uint64_t *d_state, void *stream) {
  if (!d_state) return PCCLB_EINVAL;
  simplehash_init_kernel<<<1, 256, 0, as_stream(stream)>>>(d_state);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

int pcclb_simplehash_update(uint64_t *d_state, const void *d_data, uint64_t nbytes, void *stream) {
  if (!d_state || (nbytes && !d_data)) return PCCLB_EINVAL;
  if (nbytes == 0) return PCCLB_OK;
  int rc = prepare_hash_kernels();
  if (rc) return rc;
  return launch_update<HashV0>(d_state, d_data, nbytes, as_stream(stream));
}

int pcclb_simplehash_final(const uint64_t *d_state, uint64_t total_nbytes, uint64_t *d_out,
                           void *stream) {
  if (!d_state || !d_out) return PCCLB_EINVAL;
  simplehash_final_kernel<<<1, 256, 0, as_stream(stream)>>>(d_state, total_nbytes, d_out);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

}  // extern "C"
