// simplehash on B200 (sharedstate.py:45-128).
//
// Definition: buffer as little-endian u32 words (tail zero-padded); word i
// feeds lane i mod 256, each lane runs FNV-1a-64 h = (h ^ w) * P from the
// offset basis; lanes fold by a depth-8 tree (a ^ rotl(b, 27)) * P over pairs
// (2j, 2j+1); root ^ byte length.
//
// Bounds (measured on B200, tools/micro/chain_lds.cu): one FNV step fed from
// shared memory costs 14.5 cycles when the lane also carries the hi half, and
// 10.5 cycles for the 32-bit lo chain alone (LOP3 -> IMAD, one cross-pipe hop
// each way). One entry has only 256 chains, so it cannot go faster than 1 KiB
// per step however many SMs it gets (139 GB/s full step, 192 GB/s lo only);
// many entries in flight are HBM-bound, and the largest entry sets a floor.
//
// Mapping: an entry's 256 lanes are split over GROUPS = 2 lane groups of 128;
// a work item is one lane group of one entry (or of one segment, below) and
// runs on one CTA of 4 lane warps + 1 producer warp. The producer streams the
// group's 512-byte slice of 128 consecutive 1 KiB rounds per 2-D TMA box
// (cp.async.bulk.tensor.2d over the entry viewed as [rounds x 256] u32) into a
// 3-stage shared-memory ring; lane warps release slots through per-slot
// mbarriers. Items are handed out by an atomic counter in LPT order (largest
// entries first) -- list scheduling -- and the last group of an entry folds.
//
// Big entries -- those whose 256 chains would outlast the HBM-bound time of
// the whole call, e.g. config 4's 1.05 GB embedding and LM head -- go to a
// second kernel launched concurrently on a side stream: loscan.cuh runs the
// lo half of each chain as 32 bitsliced prefix scans (the lo step is a
// T-function) instead of a serial 10.5-cycle-per-row chain, and derives the
// affine hi half from the x values the scan leaves behind, so the entry is
// read once and finished inside that kernel (lane states, tail words, fold).
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
#include "loscan.cuh"
#include "tma.cuh"

namespace pcclb {

// 12 resident CTAs' worth of registers (32 per thread): with more, ptxas
// schedules the hi half of the full step worse (single 1 GB entry 11.2 vs
// 8.1 ms measured with 48 registers)
constexpr int kHashMinBlocks = 12;
constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr uint32_t kMaxBig = 16;     // big entries per call
constexpr int kMaxBatch = 560;       // HashBatch must fit the 32 KiB kernel-parameter space
constexpr uint32_t kBigCtas = 256 / kLsLanes;  // loscan CTAs per big entry

struct HashEntry {
  const uint8_t *ptr;
  uint64_t nbytes;
  uint64_t *out;
  const CUtensorMap *map;  // 2-D view [rounds x 256] u32, or null (direct loads)
};

// ordinary entries: item = one lane group of one entry, entries in LPT order
struct HashBatch {
  uint32_t count;
  uint32_t pad;
  HashEntry e[kMaxBatch];
};

// big entries: kBigCtas loscan CTAs each
struct BigEntry {
  CUtensorMap map;  // 4-D view [segment][i][t][lane] (loscan.cuh)
  const uint8_t *ptr;
  uint64_t nbytes;
  uint64_t *out;
  uint64_t pad;
};
struct BigBatch {
  BigEntry e[kMaxBig];
};

// One FNV-1a-64 step h = (h ^ w) * P on the split state (lo, hi).
// P = 2^40 + 435 and w is a zero-extended u32, so with x = lo ^ w:
//   lo' = (x * 435) mod 2^32
//   hi' = hi * 435 + floor(x * 435 / 2^32) + (x << 8)     (mod 2^32)
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

// CTA shape: LANES lane threads (thread t = lane lane0 + t) plus one producer
// warp; a ring of STAGES shared-memory stages, each the group's LANES*4-byte
// slice of ROWS consecutive 1 KiB rounds (one 2-D TMA box).
template <int LANES_, int ROWS_, int STAGES_>
struct HashCfg {
  static constexpr int LANES = LANES_;
  static constexpr int ROWS = ROWS_;
  static constexpr int STAGES = STAGES_;
  static constexpr int THREADS = LANES + 32;
  static constexpr int WARPS = LANES / 32;
  static constexpr int GROUPS = 256 / LANES;
  static constexpr int STAGE_BYTES = ROWS * LANES * 4;
  static constexpr int SMEM = STAGE_BYTES * STAGES;
};
// Measured (config-4 layout / one 1.05 GB entry / 64 x 64 MiB, full steps,
// tools/hash_variants.py): <128,128,3> 8.5 ms / 131 GB/s / 7.1 TB/s;
// <64,128,4> 8.2 ms / 128 GB/s / 4.0 TB/s (64 lanes per SM starve HBM);
// <128,96,4> 9.0 ms; <128,64,3> without the producer warp 10.6 ms. Deep
// stages keep ~2 us of TMA lookahead per CTA and amortise the handshakes.
#ifndef PCCLB_HASH_ROWS
#define PCCLB_HASH_ROWS 64
#endif
#ifndef PCCLB_HASH_STAGES
#define PCCLB_HASH_STAGES 3
#endif
#ifndef PCCLB_HASH_LANES
#define PCCLB_HASH_LANES 128
#endif
using HashC = HashCfg<PCCLB_HASH_LANES, PCCLB_HASH_ROWS, PCCLB_HASH_STAGES>;

// Rows [0, nrows) of lanes [lane0, lane0 + C::LANES) through the TMA ring
// (boxes of C::LANES lanes x C::ROWS rows); h is the lane's state (threads <
// C::LANES). The producer thread (thread C::LANES) issues a stage into slot
// g % STAGES once the C::WARPS lane warps released it (empty[slot]); `g`
// numbers the stages of the whole launch, so the mbarrier phase parity is
// (g / STAGES) & 1.
template <class C>
__device__ __forceinline__ uint64_t run_rows(const CUtensorMap *map, uint32_t lane0, uint64_t nrows, uint64_t h,
                                             uint8_t *stage, uint64_t *full, uint64_t *empty, uint32_t &g) {
  constexpr int L = C::LANES, R = C::ROWS;
  const int tid = threadIdx.x;
  const uint32_t nst = (uint32_t)((nrows + R - 1) / R);
  if (tid >= C::LANES) {
    if (tid == C::LANES) {
      tensormap_acquire(map);
      for (uint32_t s = 0; s < nst; ++s) {
        const uint32_t G = g + s, slot = G % C::STAGES;
        if (G >= (uint32_t)C::STAGES) mbar_wait(&empty[slot], ((G / C::STAGES) - 1) & 1u);
        // rows past the end of the tensor are zero-filled and still counted
        mbar_expect_tx(&full[slot], L * R * 4);
        tma_2d_g2s(stage + slot * C::STAGE_BYTES, map, (int)lane0, (int)((uint64_t)s * R), &full[slot]);
      }
    }
  } else {
    const int t = tid;
    for (uint32_t s = 0; s < nst; ++s) {
      const uint32_t G = g + s, slot = G % C::STAGES;
      mbar_wait(&full[slot], (G / C::STAGES) & 1u);
      // the state is unpacked per stage: it keeps the compiler from
      // rescheduling the hi chain across stages (measured 35% slower)
      Fnv f(h);
      const uint32_t *wds = reinterpret_cast<const uint32_t *>(stage + slot * C::STAGE_BYTES) + t;
      const uint64_t left = nrows - (uint64_t)s * R;
      if (left >= (uint64_t)R) {
        // fully unrolled: the shared-memory loads are hoisted ahead of the chain
#pragma unroll
        for (int r = 0; r < R; ++r) f.step(wds[r * L]);
      } else {
        const int nr = (int)left;
        for (int r = 0; r < nr; ++r) f.step(wds[r * L]);
      }
      h = f.value();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
    }
  }
  g += nst;
  return h;
}

// the words after the whole rounds: lane < rem takes one full word, lane ==
// rem the zero-padded tail (sharedstate.py:45-54)
__device__ __forceinline__ uint64_t tail_steps(uint64_t h, const uint8_t *p, uint64_t nbytes,
                                               uint32_t lane) {
  const uint64_t full_words = nbytes >> 2;
  const uint64_t done = (full_words >> 8) << 8;
  const uint64_t rem = full_words - done;  // < 256
  const uint8_t *q = p + done * 4;
  if ((uint64_t)lane < rem) h = fnv_step(h, load_word_any(q + 4 * lane, 4));
  const uint32_t tail = (uint32_t)(nbytes & 3);
  if (tail && (uint64_t)lane == rem) h = fnv_step(h, load_word_any(q + 4 * lane, tail));
  return h;
}

// All rounds of lanes [lane0, lane0 + LANES) plus the tail words, from state h.
template <class C>
__device__ __forceinline__ uint64_t hash_group(const uint8_t *p, uint64_t nbytes,
                                               const CUtensorMap *map, uint32_t lane0, uint64_t h,
                                               uint8_t *stage, uint64_t *bars, uint32_t &g) {
  const uint32_t lane = lane0 + threadIdx.x;
  const uint64_t rounds = nbytes >> 10;
  if (rounds > 0 && map != nullptr) {
    h = run_rows<C>(map, lane0, rounds, h, stage, bars, bars + C::STAGES, g);
  } else if (threadIdx.x < C::LANES) {
    for (uint64_t r = 0; r < rounds; ++r) h = fnv_step(h, load_word_any(p + ((r << 8) + lane) * 4, 4));
  }
  if (threadIdx.x >= C::LANES) return 0;
  return tail_steps(h, p, nbytes, lane);
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
    for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[C::STAGES + s], C::WARPS);
    mbar_fence_init();
  }
  __syncthreads();
}

// Count one finished part; the CTA that completes all `parts` gets true.
__device__ __forceinline__ bool last_part(uint32_t *counter, uint32_t parts, uint32_t *s_flag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *s_flag = (atomicAdd(counter, 1u) == parts - 1) ? 1u : 0u;
  __syncthreads();
  const bool last = *s_flag != 0;
  if (last) __threadfence();
  return last;
}

#ifdef PCCLB_HASH_TRACE
// debug timeline: per CTA {kernel, smid, start, end} (globaltimer ns)
__device__ unsigned long long g_trace[8192][4];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define TRACE_BEGIN() const uint64_t tr_t0 = gtimer()
#define TRACE_END(kind)                                             \
  if (threadIdx.x == 0) {                                           \
    const uint32_t i = atomicAdd(&g_trace_n, 1u);                   \
    if (i < 8192) {                                                 \
      g_trace[i][0] = kind;                                         \
      g_trace[i][1] = smid();                                       \
      g_trace[i][2] = tr_t0;                                        \
      g_trace[i][3] = gtimer();                                     \
    }                                                               \
  }
// per batch item: {3, nbytes of the entry << 16 | smid, start, end}
#define TRACE_ITEM_BEGIN() const uint64_t tri_t0 = gtimer()
#define TRACE_ITEM_END(nb)                                          \
  if (threadIdx.x == 0) {                                           \
    const uint32_t i = atomicAdd(&g_trace_n, 1u);                   \
    if (i < 8192) {                                                 \
      g_trace[i][0] = 3;                                            \
      g_trace[i][1] = ((uint64_t)(nb) << 16) | smid();              \
      g_trace[i][2] = tri_t0;                                       \
      g_trace[i][3] = gtimer();                                     \
    }                                                               \
  }
#else
#define TRACE_BEGIN()
#define TRACE_END(kind)
#define TRACE_ITEM_BEGIN()
#define TRACE_ITEM_END(nb)
#endif

// One launch for a batch of ordinary entries. Scratch: lanes[count x 256]
// (lane values), cnt = [count arrivals | item counter].
template <class C>
__global__ void __launch_bounds__(C::THREADS, kHashMinBlocks)
    simplehash_batch_kernel(const __grid_constant__ HashBatch b, uint64_t *lanes, uint32_t *cnt) {
  TRACE_BEGIN();
  extern __shared__ __align__(1024) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[2 * C::STAGES];
  __shared__ uint64_t lane_s[256];
  __shared__ uint32_t s_flag, s_item;
  init_bars<C>(bars);
  constexpr uint32_t G = C::GROUPS;
  uint32_t *arrived = cnt;
  uint32_t *next = cnt + b.count;
  const uint32_t items = b.count * G;
  uint32_t g = 0;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(next, 1u);
    __syncthreads();
    const uint32_t it = s_item;
    if (it >= items) break;
    // an entry's lane group; the last group of the entry folds
    const uint32_t e = it / G, grp = it % G;
    const HashEntry E = b.e[e];
    const uint32_t lane0 = grp * C::LANES;
    TRACE_ITEM_BEGIN();
    const uint64_t h = hash_group<C>(E.ptr, E.nbytes, E.map, lane0, kFnvOffset, stage, bars, g);
    TRACE_ITEM_END(E.nbytes);
    if (threadIdx.x < C::LANES) lanes[(uint64_t)e * 256 + lane0 + threadIdx.x] = h;
    if (last_part(&arrived[e], G, &s_flag)) {
      for (int j = threadIdx.x; j < 256; j += blockDim.x) lane_s[j] = __ldcg(&lanes[(uint64_t)e * 256 + j]);
      const uint64_t root = tree_fold(lane_s);
      if (threadIdx.x == 0) *E.out = root ^ E.nbytes;
    }
    __syncthreads();
  }
  TRACE_END(1);
}

// Big entries: kBigCtas CTAs per entry, each the whole chains of kLsLanes
// lanes (loscan.cuh), then the tail words; the last CTA of an entry folds.
// Scratch: lanes[kMaxBig x 256], done[kMaxBig].
__global__ void __launch_bounds__(kLsThreads, 1)
    simplehash_big_kernel(const __grid_constant__ BigBatch bb, uint64_t *lanes, uint32_t *done, uint32_t *started) {
  TRACE_BEGIN();
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t s_flag;
  if (threadIdx.x == 0) atomicAdd(started, 1u);
  auto *sh = reinterpret_cast<LsShared *>(smem + kLsStageBytes * kLsStages);
  const uint32_t e = blockIdx.x / kBigCtas, q = blockIdx.x % kBigCtas;
  const BigEntry &E = bb.e[e];
  const uint32_t lane0 = q * kLsLanes;
  loscan_cta(&E.map, E.ptr, E.nbytes >> 10, lane0, smem, sh);
  if (threadIdx.x < kLsLanes) {
    const uint32_t lane = lane0 + threadIdx.x;
    const uint64_t h = ((uint64_t)sh->final_hi[threadIdx.x] << 32) | sh->final_lo[threadIdx.x];
    lanes[(uint64_t)e * 256 + lane] = tail_steps(h, E.ptr, E.nbytes, lane);
  }
  if (last_part(&done[e], kBigCtas, &s_flag)) {
    uint64_t *lane_s = reinterpret_cast<uint64_t *>(smem);  // the stage area is free now
    for (int j = threadIdx.x; j < 256; j += blockDim.x) lane_s[j] = __ldcg(&lanes[(uint64_t)e * 256 + j]);
    const uint64_t root = tree_fold(lane_s);
    if (threadIdx.x == 0) *E.out = root ^ E.nbytes;
  }
  TRACE_END(2);
}

// Holds the stream until `need` big-entry CTAs are resident, so the batch
// kernel queued behind it fills the SMs around them instead of taking the
// shared memory first (the two kernels' launch order across streams is
// otherwise a race: config 4 3.0 ms when the big-entry CTAs land first, 3.7
// when the batch CTAs do).
__global__ void simplehash_gate_kernel(const uint32_t *started, uint32_t need) {
  while (ld_acquire(started) < need) __nanosleep(500);
}

// streaming update of one segment: grid = GROUPS CTAs, lane state in/out
template <class C>
__global__ void __launch_bounds__(C::THREADS)
    simplehash_update_kernel(uint64_t *state, const uint8_t *p, uint64_t nbytes,
                             const __grid_constant__ CUtensorMap map, int have_map) {
  extern __shared__ __align__(1024) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[2 * C::STAGES];
  init_bars<C>(bars);
  uint32_t g = 0;
  const uint32_t lane = blockIdx.x * C::LANES + (threadIdx.x % C::LANES);
  const uint64_t h = hash_group<C>(p, nbytes, have_map ? &map : nullptr, blockIdx.x * C::LANES,
                                   state[lane], stage, bars, g);
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

// PCCLB_HASH_BIG=0 keeps every entry on the batch kernel (measurements, tests)
static bool big_path_enabled() {
  static bool on = [] {
    const char *e = getenv("PCCLB_HASH_BIG");
    return !(e && e[0] == '0');
  }();
  return on;
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

// [rounds x 256] u32 view of an entry, box L lanes x R rows; false if not encodable
template <int L, int R>
static bool encode_map(CUtensorMap *m, const void *p, uint64_t nbytes) {
  const uint64_t rounds = nbytes >> 10;
  if (!rounds || (reinterpret_cast<uintptr_t>(p) & 15) || rounds >= (1ull << 31)) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {256, rounds};
  cuuint64_t strides[1] = {1024};
  cuuint32_t box[2] = {(cuuint32_t)L, (cuuint32_t)R};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(p), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int prepare_hash_kernels() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  PCCLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && done[dev]) return PCCLB_OK;
  PCCLB_CUDA(cudaFuncSetAttribute(simplehash_batch_kernel<HashC>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, HashC::SMEM));
  PCCLB_CUDA(cudaFuncSetAttribute(simplehash_update_kernel<HashC>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, HashC::SMEM));
  PCCLB_CUDA(cudaFuncSetAttribute(simplehash_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLsSmem));
  // the batch and big-entry kernels share SMs: both ask for the full shared
  // memory carveout, so an SM configured for one has room for the other
  PCCLB_CUDA(cudaFuncSetAttribute(simplehash_batch_kernel<HashC>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  PCCLB_CUDA(cudaFuncSetAttribute(simplehash_big_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  if (dev >= 0 && dev < 64) done[dev] = true;
  return PCCLB_OK;
}

// Big entries: those whose full-step chain (~139 GB/s) would outlast the
// HBM-bound time of the whole call (total bytes at ~6 TB/s), at least 64 MiB,
// with a 16-byte aligned base (TMA).
static bool is_big(const void *p, uint64_t nbytes, uint64_t total) {
  return big_path_enabled() && nbytes >= (64ull << 20) && nbytes * 40 > total &&
         (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (nbytes >> 10) < (1ull << 31);
}

// 4-D view of a big entry for loscan.cuh: dims {256 lanes, 32 t, 32 i, whole
// 1024-row segments}, strides {4 B, 32 KiB, 1 KiB, 1 MiB}
static bool encode_big_map(CUtensorMap *m, const void *p, uint64_t nbytes) {
  const uint64_t nseg = nbytes >> 20;
  auto fn = encode_fn();
  if (!fn || nseg == 0) return false;
  cuuint64_t dims[4] = {256, 32, 32, nseg};
  cuuint64_t strides[3] = {32768, 1024, 1ull << 20};
  cuuint32_t box[4] = {(cuuint32_t)kLsLanes, 32, 32, (cuuint32_t)kLsWarps};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<void *>(p), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// side stream + fork/join events of the calling host thread (big entries run
// beside the batch kernel)
struct SideStream {
  int dev = -1;
  cudaStream_t s = nullptr;
  cudaStream_t cap = nullptr;  // graph capture (the caller's stream may be the legacy one)
  cudaEvent_t fork = nullptr, join = nullptr;
  ~SideStream() {
    // process teardown: the context may already be gone, errors are ignored
    if (s) cudaStreamDestroy(s);
    if (cap) cudaStreamDestroy(cap);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
  }
};

static int side_stream(SideStream &ss) {
  int dev = 0;
  PCCLB_CUDA(cudaGetDevice(&dev));
  if (ss.s && ss.dev == dev) return PCCLB_OK;
  ss.dev = dev;
  PCCLB_CUDA(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
  PCCLB_CUDA(cudaStreamCreateWithFlags(&ss.cap, cudaStreamNonBlocking));
  PCCLB_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
  PCCLB_CUDA(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
  return PCCLB_OK;
}

// A call's launch plan: which entries go to the big-entry kernel, the
// ordinary entries' batches in LPT order and their tensor maps (in device
// memory). Encoding ~300 tensor maps costs ~3 ms of host time, as much as the
// GPU work of config 4, so the plan of the previous call (same device,
// pointers and sizes, e.g. a training loop re-hashing its shared state) is
// reused as is.
struct HashPlan {
  int dev = -1;
  std::vector<const void *> ptrs;
  std::vector<uint64_t> sizes;
  uint64_t *d_out = nullptr;
  BigBatch big;
  uint32_t nbig = 0;
  std::vector<HashBatch> batches;
  uint32_t m_max = 0;
  CUtensorMap *d_maps = nullptr;  // batches' maps, stream-ordered allocation
  cudaEvent_t last_use = nullptr; // after the last launch reading d_maps
  bool used = false;
  std::vector<CUtensorMap> host_maps;
  CUtensorMap *pinned = nullptr;
  size_t pinned_cap = 0;
  cudaEvent_t uploaded = nullptr; // the pinned staging area is free again
  cudaGraphExec_t exec = nullptr;  // the call's stream operations, replayed per call
  ~HashPlan() {
    // process teardown: the context may already be gone, errors are ignored
    if (exec) cudaGraphExecDestroy(exec);
    if (pinned) cudaFreeHost(pinned);
    if (last_use) cudaEventDestroy(last_use);
    if (uploaded) cudaEventDestroy(uploaded);
  }
};

static int build_plan(HashPlan &P, const std::vector<uint32_t> &order, const void *const *h_ptrs,
                      const uint64_t *h_nbytes, uint64_t *d_out, cudaStream_t s) {
  using C = HashC;
  const uint32_t count = (uint32_t)order.size();
  if (!P.last_use) PCCLB_CUDA(cudaEventCreateWithFlags(&P.last_use, cudaEventDisableTiming));
  if (!P.uploaded) PCCLB_CUDA(cudaEventCreateWithFlags(&P.uploaded, cudaEventDisableTiming));
  uint64_t total = 0;
  for (uint32_t i = 0; i < count; ++i) total += h_nbytes[i];
  // big entries (largest first) go to the loscan kernel, the rest to batches
  std::vector<uint32_t> rest;
  P.nbig = 0;
  for (uint32_t k : order) {
    BigEntry &B = P.big.e[P.nbig];
    if (P.nbig < kMaxBig && is_big(h_ptrs[k], h_nbytes[k], total) && encode_big_map(&B.map, h_ptrs[k], h_nbytes[k])) {
      B.ptr = static_cast<const uint8_t *>(h_ptrs[k]);
      B.nbytes = h_nbytes[k];
      B.out = d_out + k;
      B.pad = 0;
      ++P.nbig;
    } else {
      rest.push_back(k);
    }
  }
  const uint32_t nrest = (uint32_t)rest.size();
  P.m_max = std::min<uint32_t>(kMaxBatch, nrest);
  if (P.exec) {  // the previous plan's graph (its launches are stream-ordered before any new one)
    cudaGraphExecDestroy(P.exec);
    P.exec = nullptr;
  }
  // the previous maps may still be read by an earlier launch: free them after it
  if (P.d_maps) {
    if (P.used) PCCLB_CUDA(cudaStreamWaitEvent(s, P.last_use, 0));
    PCCLB_CUDA(cudaFreeAsync(P.d_maps, s));
    P.d_maps = nullptr;
  }
  P.used = false;
  P.batches.clear();
  P.host_maps.resize(nrest);
  if (nrest) PCCLB_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&P.d_maps), sizeof(CUtensorMap) * nrest, s));
  for (uint32_t base = 0; base < nrest; base += kMaxBatch) {
    const uint32_t m = std::min<uint32_t>(kMaxBatch, nrest - base);
    P.batches.emplace_back();
    HashBatch &batch = P.batches.back();
    std::memset(&batch, 0, sizeof(batch));
    batch.count = m;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t k = rest[base + i];
      HashEntry &E = batch.e[i];
      E.ptr = static_cast<const uint8_t *>(h_ptrs[k]);
      E.nbytes = h_nbytes[k];
      E.out = d_out + k;
      E.map = encode_map<C::LANES, C::ROWS>(&P.host_maps[base + i], E.ptr, E.nbytes) ? P.d_maps + base + i : nullptr;
    }
  }
  if (nrest) {
    const size_t bytes = sizeof(CUtensorMap) * nrest;
    if (P.pinned_cap < nrest) {
      if (P.pinned) {
        PCCLB_CUDA(cudaEventSynchronize(P.uploaded));
        PCCLB_CUDA(cudaFreeHost(P.pinned));
        P.pinned = nullptr;
      }
      PCCLB_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&P.pinned), bytes, cudaHostAllocDefault));
      P.pinned_cap = nrest;
    } else {
      PCCLB_CUDA(cudaEventSynchronize(P.uploaded));  // previous upload out of the staging area
    }
    std::memcpy(P.pinned, P.host_maps.data(), bytes);
    PCCLB_CUDA(cudaMemcpyAsync(P.d_maps, P.pinned, bytes, cudaMemcpyHostToDevice, s));
    PCCLB_CUDA(cudaEventRecord(P.uploaded, s));
  }
  PCCLB_CUDA(cudaGetDevice(&P.dev));
  P.ptrs.assign(h_ptrs, h_ptrs + count);
  P.sizes.assign(h_nbytes, h_nbytes + count);
  P.d_out = d_out;
  return PCCLB_OK;
}

static bool plan_matches(const HashPlan &P, const void *const *h_ptrs, const uint64_t *h_nbytes, uint32_t count,
                         uint64_t *d_out) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != P.dev || P.d_out != d_out || P.ptrs.size() != count) return false;
  return std::equal(h_ptrs, h_ptrs + count, P.ptrs.begin()) && std::equal(h_nbytes, h_nbytes + count, P.sizes.begin());
}

// order: entry indices, largest first
// The stream operations of one call for `plan` (direct, or recorded into
// the plan's CUDA graph).
static int enqueue_call(HashPlan &plan, SideStream &side, cudaStream_t s) {
  using C = HashC;
  int occ = 0;
  PCCLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, simplehash_batch_kernel<C>, C::THREADS, C::SMEM));
  if (occ < 1) occ = 1;
  const uint32_t slots = (uint32_t)(sm_count() * occ);
  const uint32_t nbig = plan.nbig, m_max = plan.m_max;
  // per-call device scratch: lane values and counters
  const size_t lanes_bytes = ((size_t)m_max + nbig) * 256 * sizeof(uint64_t);
  const size_t cnt_words = (size_t)m_max + 1 + nbig + 1;
  char *scratch = nullptr;
  PCCLB_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&scratch), lanes_bytes + cnt_words * sizeof(uint32_t), s));
  uint64_t *lanes = reinterpret_cast<uint64_t *>(scratch);
  uint64_t *big_lanes = lanes + (size_t)m_max * 256;
  uint32_t *cnt = reinterpret_cast<uint32_t *>(scratch + lanes_bytes);
  uint32_t *big_done = cnt + m_max + 1;
  uint32_t *big_started = big_done + nbig;
  int rc = PCCLB_OK;
  bool forked = false;
  cudaError_t e = cudaMemsetAsync(cnt, 0, cnt_words * sizeof(uint32_t), s);
  if (e != cudaSuccess) rc = cuda_status(e);
  // the big-entry kernel first, on the side stream (launching it after the
  // batch kernel measured slower: 3.85 vs 3.35 ms on config 4)
  if (rc == PCCLB_OK && nbig) {
    e = cudaEventRecord(side.fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side.s, side.fork, 0);
    if (e == cudaSuccess) {
      forked = true;
      simplehash_big_kernel<<<nbig * kBigCtas, kLsThreads, kLsSmem, side.s>>>(plan.big, big_lanes, big_done,
                                                                               big_started);
      e = cudaGetLastError();
      if (e == cudaSuccess && !plan.batches.empty()) {
        const uint32_t need = std::min<uint32_t>(nbig * kBigCtas, (uint32_t)sm_count());
        simplehash_gate_kernel<<<1, 32, 0, s>>>(big_started, need);
        e = cudaGetLastError();
      }
    }
    if (e != cudaSuccess) rc = cuda_status(e);
  }
  for (size_t bi = 0; bi < plan.batches.size() && rc == PCCLB_OK; ++bi) {
    const HashBatch &batch = plan.batches[bi];
    if (bi > 0) {
      e = cudaMemsetAsync(cnt, 0, ((size_t)m_max + 1) * sizeof(uint32_t), s);
      if (e != cudaSuccess) {
        rc = cuda_status(e);
        break;
      }
    }
    const uint64_t items = (uint64_t)batch.count * C::GROUPS;
    // beside the big-entry kernel: one batch CTA shares each SM with a loscan
    // CTA (both ask for the full carveout and fit together), the others wait
    // for SMs the loscan CTAs leave -- one extra CTA per SM for those
    // (config 4: 3.07 ms at occupancy, 3.03 ms with the extra wave)
    const unsigned grid = (unsigned)std::min<uint64_t>(items, nbig ? slots + (uint64_t)sm_count() : slots);
    simplehash_batch_kernel<C><<<grid, C::THREADS, C::SMEM, s>>>(batch, lanes, cnt);
    e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_status(e);
  }
  if (forked) {
    // join even after an error, so the scratch is not freed under the big kernel
    e = cudaEventRecord(side.join, side.s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, side.join, 0);
    if (rc == PCCLB_OK && e != cudaSuccess) rc = cuda_status(e);
  }
  e = cudaFreeAsync(scratch, s);
  if (rc == PCCLB_OK && e != cudaSuccess) rc = cuda_status(e);
  return rc;
}

// PCCLB_HASH_GRAPH=0: enqueue every call directly instead of replaying the plan's graph
static bool hash_graphs_enabled() {
  static bool on = [] {
    const char *e = getenv("PCCLB_HASH_GRAPH");
    return !(e && e[0] == '0');
  }();
  return on;
}

// order: entry indices, largest first
static int launch_batches(const std::vector<uint32_t> &order, const void *const *h_ptrs,
                          const uint64_t *h_nbytes, uint64_t *d_out, cudaStream_t s) {
  const uint32_t count = (uint32_t)order.size();
  if (count == 0) return PCCLB_OK;
  static thread_local HashPlan plan;
  static thread_local SideStream side;
  int rc = side_stream(side);
  if (rc) return rc;
  if (!plan_matches(plan, h_ptrs, h_nbytes, count, d_out)) {
    plan.dev = -1;  // a failed build leaves no stale plan behind
    rc = build_plan(plan, order, h_ptrs, h_nbytes, d_out, s);
    if (rc) {
      plan.ptrs.clear();
      return rc;
    }
  }
  // A repeated call replays one CUDA graph of the plan's stream operations:
  // the two streams' launches then start without per-launch front-end work
  // (measured on config 4: back-to-back direct calls 3.30 ms, with an event
  // between calls 3.08 ms). Not while the caller is capturing `s` itself.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  PCCLB_CUDA(cudaStreamIsCapturing(s, &cap));
  const bool graph = hash_graphs_enabled() && cap == cudaStreamCaptureStatusNone;
  if (graph && !plan.exec) {
    // recorded on a private stream: capture is not allowed on the legacy one
    PCCLB_CUDA(cudaStreamBeginCapture(side.cap, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_call(plan, side, side.cap);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(side.cap, &g);
    if (rc == PCCLB_OK && e != cudaSuccess) rc = cuda_status(e);
    if (rc == PCCLB_OK) {
      const cudaError_t ie = cudaGraphInstantiate(&plan.exec, g, 0);
      if (ie != cudaSuccess) {
        plan.exec = nullptr;
        rc = cuda_status(ie);
      }
    }
    if (g) cudaGraphDestroy(g);
    if (rc) return rc;
  }
  if (graph) PCCLB_CUDA(cudaGraphLaunch(plan.exec, s));
  else rc = enqueue_call(plan, side, s);
  if (rc == PCCLB_OK && !plan.batches.empty()) {
    PCCLB_CUDA(cudaEventRecord(plan.last_use, s));  // the batches' tensor maps were read
    plan.used = true;
  }
  return rc;
}

static int launch_update(uint64_t *state, const void *d, uint64_t nbytes, cudaStream_t s) {
  using C = HashC;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  int have = encode_map<C::LANES, C::ROWS>(&map, d, nbytes) ? 1 : 0;
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
  return launch_batches(order, h_ptrs, h_nbytes, d_out, as_stream(stream));
}

#ifdef PCCLB_HASH_TRACE
__attribute__((visibility("default"))) int pcclb_debug_hash_trace(unsigned long long *host, int max, int reset) {
  unsigned int n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, g_trace_n, sizeof(n));
  if (n > 8192) n = 8192;
  if ((int)n > max) n = (unsigned)max;
  cudaMemcpyFromSymbol(host, g_trace, (size_t)n * 32);
  if (reset) {
    unsigned int z = 0;
    cudaMemcpyToSymbol(g_trace_n, &z, sizeof(z));
  }
  return (int)n;
}
#endif

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
  return launch_update(d_state, d_data, nbytes, as_stream(stream));
}

int pcclb_simplehash_final(const uint64_t *d_state, uint64_t total_nbytes, uint64_t *d_out,
                           void *stream) {
  if (!d_state || !d_out) return PCCLB_EINVAL;
  simplehash_final_kernel<<<1, 256, 0, as_stream(stream)>>>(d_state, total_nbytes, d_out);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

}  // extern "C"
