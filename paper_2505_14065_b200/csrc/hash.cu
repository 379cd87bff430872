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
// Two-phase path for entries whose chain outlasts the rest of the batch
// ("big" entries, e.g. config 4's 1.05 GB embedding and LM head). The FNV step
// splits into lo' = (lo ^ w) * 435 mod 2^32, which depends on lo alone, and
// hi' = 435 hi + umulhi(x, 435) + (x << 8) with x = lo ^ w, which is affine in
// hi. So:
//   phase 1 (one item per kP1Lanes-lane slice, 32 lanes x 512-row stages): run only the lo chain over the
//     whole entry (10.5 instead of 14.5 cycles per step) and publish lo at
//     every kSegRows-row checkpoint;
//   phase 2 (one item per segment and lane group, run by any free CTA as soon
//     as its checkpoint is published): rerun the full step over the segment
//     from (lo = checkpoint, hi = 0), which leaves hi = A_j, the segment's
//     additive term;
//   combine (by the last finisher): hi = 435^m_j * hi + A_j over the segments,
//     h = hi:lo_final, then the tail words and the tree fold.
// Phase 2 reads the entry a second time, in parallel on otherwise idle SMs.
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
#ifndef PCCLB_SEGROWS
#define PCCLB_SEGROWS 32768  // measured (one 1.05 GB entry): 4096 6.38 ms, 16384 6.06 / 5.74, 32768 5.69-5.71, 65536 5.76, 131072 5.91 ms
#endif
constexpr uint32_t kSegRows = PCCLB_SEGROWS;  // checkpoint spacing of the two-phase path (rows of 1 KiB)
constexpr uint32_t kMaxBig = 16;     // big entries per launch
constexpr int kMaxBatch = 560;       // HashBatch must fit the 32 KiB kernel-parameter space
// phase-1 items: 64 lanes per CTA and 256-row boxes, so each lo chain CTA keeps
// ~2.7 us of TMA in flight (the lo chain consumes 512 B per ~10.5 cycles per
// 128 lanes, more than one CTA's stream of 128-lane boxes sustains)
#ifndef PCCLB_P1_LANES
#define PCCLB_P1_LANES 32  // measured (one 1.05 GB entry): 64 lanes x 256 rows 6.06 ms, 32 x 512 5.74 ms
#endif
constexpr int kP1Lanes = PCCLB_P1_LANES;
constexpr int kP1Rows = 256 * 64 / kP1Lanes;  // one 64 KiB stage
constexpr int kP1Groups = 256 / kP1Lanes;
#ifndef PCCLB_P1_UNROLL
#define PCCLB_P1_UNROLL 512
#endif
constexpr int kP1Unroll = PCCLB_P1_UNROLL;  // rows per unrolled block of the phase-1 loop

struct HashEntry {
  const uint8_t *ptr;
  uint64_t nbytes;
  uint64_t *out;
  const CUtensorMap *map;  // 2-D view [rounds x 256] u32, or null (direct loads)
  const CUtensorMap *map1; // big entries: the same view with phase-1 boxes
  uint32_t *aux;           // big entries: [nseg x 256] checkpoints, [256] final lo, [nseg x 256] A
  uint32_t nseg;           // big entries: number of kSegRows segments
  uint32_t pad;
};

// Entries [0, nbig) are big (two-phase); item space:
//   [0, n1 = nbig*P1)                   phase-1 lo chains (P1 = kP1Groups)
//   [n1, n2 = n1 + (count-nbig)*G)      ordinary entries' lane groups
//   [n2, n2 + segmax*nbig*G)            phase-2 segments, segment-major
struct HashBatch {
  uint32_t count;
  uint32_t nbig;
  uint32_t segmax;
  uint32_t pad;
  HashEntry e[kMaxBatch];
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
  // phase 1 of the two-phase path: the lo chain alone
  __device__ __forceinline__ void step_lo(uint32_t w) { lo = (lo ^ w) * 435u; }
};
__device__ __forceinline__ uint64_t fnv_step(uint64_t h, uint32_t w) {
  return (h ^ (uint64_t)w) * kFnvPrime;
}
__device__ __forceinline__ uint64_t rotl27(uint64_t v) { return (v << 27) | (v >> 37); }
// 435^m mod 2^32
__device__ __forceinline__ uint32_t pow435(uint32_t m) {
  uint32_t r = 1, b = 435u;
  while (m) {
    if (m & 1u) r *= b;
    b *= b;
    m >>= 1;
  }
  return r;
}

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
  static_assert(kSegRows % ROWS == 0, "segments are whole stages");
};
// Measured (config-4 layout / one 1.05 GB entry / 64 x 64 MiB, full steps,
// tools/hash_variants.py): <128,128,3> 8.5 ms / 131 GB/s / 7.1 TB/s;
// <64,128,4> 8.2 ms / 128 GB/s / 4.0 TB/s (64 lanes per SM starve HBM);
// <128,96,4> 9.0 ms; <128,64,3> without the producer warp 10.6 ms. Deep
// stages keep ~2 us of TMA lookahead per CTA and amortise the handshakes.
using HashC = HashCfg<128, 128, 3>;

// Rows [row0, row0 + nrows) of lanes [lane0, lane0 + L) through the TMA ring
// (boxes of L lanes x R rows); h is the lane's state (threads < L). The
// producer thread (thread C::LANES) issues a stage into slot g % STAGES once
// the C::WARPS lane warps released it (empty[slot]); `g` numbers the stages of
// the whole launch, so the mbarrier phase parity is (g / STAGES) & 1. Lane
// warps beyond L only keep the ring protocol. LO_ONLY: step the lo chain only
// and, every kSegRows rows (row0 = 0), store the lo value that starts the
// segment to ck[seg * 256 + lane] and count each writing warp in *progress.
template <class C, int L, int R, bool LO_ONLY>
__device__ __forceinline__ uint64_t run_rows(const CUtensorMap *map, uint32_t lane0, uint64_t row0,
                                             uint64_t nrows, uint64_t h, uint8_t *stage,
                                             uint64_t *full, uint64_t *empty, uint32_t &g,
                                             uint32_t *ck, uint32_t *progress) {
  static_assert(L * R * 4 <= C::STAGE_BYTES && kSegRows % R == 0, "box fits a slot");
  static_assert(L == C::LANES || L + 32 <= C::LANES, "narrow boxes start at warp 1");
  const int tid = threadIdx.x;
  const uint32_t nst = (uint32_t)((nrows + R - 1) / R);
  if (tid >= C::LANES) {
    if (tid == C::LANES) {
      tensormap_acquire(map);
      for (uint32_t s = 0; s < nst; ++s) {
        const uint32_t G = g + s, slot = G % C::STAGES;
        if (G >= (uint32_t)C::STAGES) mbar_wait(&empty[slot], ((G / C::STAGES) - 1) & 1u);
        // rows past the end of the tensor are zero-filled and still counted;
        // stages taller than a TMA box (256 rows) take several boxes
        constexpr int BR = R < 256 ? R : 256;
        mbar_expect_tx(&full[slot], L * R * 4);
#pragma unroll
        for (int b = 0; b < R / BR; ++b)
          tma_2d_g2s(stage + slot * C::STAGE_BYTES + b * BR * L * 4, map, (int)lane0,
                     (int)(row0 + (uint64_t)s * R + b * BR), &full[slot]);
      }
    }
  } else {
    // narrower boxes run on warps 1.. (warp 0 shares its SMSP with the producer)
    constexpr int off = (L < C::LANES) ? 32 : 0;
    const int t = tid - off;
    const bool active = t >= 0 && t < L;
    for (uint32_t s = 0; s < nst; ++s) {
      const uint32_t G = g + s, slot = G % C::STAGES;
      if constexpr (LO_ONLY) {
        if (active && (s * R) % kSegRows == 0) {
          ck[(s * R / kSegRows) * 256 + lane0 + t] = (uint32_t)h;
          __syncwarp();
          if ((tid & 31) == 0) {
            __threadfence();  // ~3% of phase 1 (measured against an unordered count)
            atomicAdd(progress, 1u);
          }
        }
      }
      mbar_wait(&full[slot], (G / C::STAGES) & 1u);
      if (active) {
        // the state is unpacked per stage: it keeps the compiler from
        // rescheduling the hi chain across stages (measured 35% slower)
        Fnv f(h);
        const uint32_t *wds = reinterpret_cast<const uint32_t *>(stage + slot * C::STAGE_BYTES) + t;
        const uint64_t left = nrows - (uint64_t)s * R;
        if (LO_ONLY && kP1Unroll < R && left >= (uint64_t)R) {
          // lo chain in kP1Unroll-row unrolled blocks (smaller code body)
          constexpr int UB = kP1Unroll < R ? kP1Unroll : R;
#pragma unroll 1
          for (int r0 = 0; r0 < R; r0 += UB) {
#pragma unroll
            for (int r = 0; r < UB; ++r) f.step_lo(wds[(r0 + r) * L]);
          }
        } else if (left >= (uint64_t)R) {
          // fully unrolled: the shared-memory loads are hoisted ahead of the chain
          // (measured best for both forms, e.g. phase 1: 6.24 ms at 256 vs 6.8 at 32)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if constexpr (LO_ONLY)
              f.step_lo(wds[r * L]);
            else
              f.step(wds[r * L]);
          }
        } else {
          const int nr = (int)left;
          for (int r = 0; r < nr; ++r) {
            if constexpr (LO_ONLY)
              f.step_lo(wds[r * L]);
            else
              f.step(wds[r * L]);
          }
        }
        h = f.value();
      }
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
    h = run_rows<C, C::LANES, C::ROWS, false>(map, lane0, 0, rounds, h, stage, bars, bars + C::STAGES, g,
                                              nullptr, nullptr);
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

// Combine of the two-phase path: hi over the segments, the tail, the fold.
__device__ __forceinline__ void big_combine(const HashEntry &E, uint64_t *lane_s) {
  const uint64_t rounds = E.nbytes >> 10;
  const uint32_t *lofinal = E.aux + (size_t)E.nseg * 256;
  const uint32_t *A = lofinal + 256;
  const uint32_t pw = pow435(kSegRows);
  for (int lane = threadIdx.x; lane < 256; lane += blockDim.x) {
    uint32_t hi = (uint32_t)(kFnvOffset >> 32);
#pragma unroll 8
    for (uint32_t j = 0; j < E.nseg; ++j) {
      const uint64_t m = min((uint64_t)kSegRows, rounds - (uint64_t)j * kSegRows);
      hi = (m == kSegRows ? pw : pow435((uint32_t)m)) * hi + __ldcg(&A[(size_t)j * 256 + lane]);
    }
    const uint64_t h = ((uint64_t)hi << 32) | __ldcg(&lofinal[lane]);
    lane_s[lane] = tail_steps(h, E.ptr, E.nbytes, lane);
  }
  const uint64_t root = tree_fold(lane_s);
  if (threadIdx.x == 0) *E.out = root ^ E.nbytes;
}

// One launch for a batch of entries. Scratch: lanes[count x 256] (ordinary
// entries' lane values), cnt = [count arrivals | item counter | nbig*G phase-1
// progress counters | nbig completion counters].
template <class C>
__global__ void __launch_bounds__(C::THREADS, kHashMinBlocks)
    simplehash_batch_kernel(const __grid_constant__ HashBatch b, uint64_t *lanes, uint32_t *cnt) {
  extern __shared__ __align__(1024) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[2 * C::STAGES];
  __shared__ uint64_t lane_s[256];
  __shared__ uint32_t s_flag, s_item;
  init_bars<C>(bars);
  constexpr uint32_t G = C::GROUPS, P1 = kP1Groups;
  uint32_t *arrived = cnt;
  uint32_t *next = cnt + b.count;
  uint32_t *progress = next + 1;
  uint32_t *bigdone = progress + b.nbig * P1;
  const uint32_t n1 = b.nbig * P1, n2 = n1 + (b.count - b.nbig) * G, nseg_items = b.nbig * G;
  const uint32_t items = n2 + b.segmax * nseg_items;
  uint32_t g = 0;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(next, 1u);
    __syncthreads();
    const uint32_t it = s_item;
    if (it >= items) break;
    if (it < n1) {
      // phase 1: the lo chain of one kP1Lanes-lane slice of a big entry
      const uint32_t e = it / P1, q = it % P1;
      const HashEntry E = b.e[e];
      const uint32_t lane0 = q * kP1Lanes;
      const uint64_t h = run_rows<C, kP1Lanes, kP1Rows, true>(E.map1, lane0, 0, E.nbytes >> 10, kFnvOffset,
                                                              stage, bars, bars + C::STAGES, g, E.aux,
                                                              &progress[it]);
      if (threadIdx.x >= 32 && threadIdx.x < 32 + kP1Lanes)  // run_rows' lane offset
        E.aux[(size_t)E.nseg * 256 + lane0 + threadIdx.x - 32] = (uint32_t)h;
      if (last_part(&bigdone[e], P1 + G * E.nseg, &s_flag)) big_combine(E, lane_s);
    } else if (it < n2) {
      // an ordinary entry's lane group; the last group of the entry folds
      const uint32_t e = b.nbig + (it - n1) / G, grp = (it - n1) % G;
      const HashEntry E = b.e[e];
      const uint32_t lane0 = grp * C::LANES;
      const uint64_t h = hash_group<C>(E.ptr, E.nbytes, E.map, lane0, kFnvOffset, stage, bars, g);
      if (threadIdx.x < C::LANES) lanes[(uint64_t)e * 256 + lane0 + threadIdx.x] = h;
      if (last_part(&arrived[e], G, &s_flag)) {
        for (int j = threadIdx.x; j < 256; j += blockDim.x)
          lane_s[j] = __ldcg(&lanes[(uint64_t)e * 256 + j]);
        const uint64_t root = tree_fold(lane_s);
        if (threadIdx.x == 0) *E.out = root ^ E.nbytes;
      }
    } else {
      // phase 2: segment j of one 128-lane group of a big entry, once phase 1
      // published the lo values that start it (C::LANES / kP1Lanes slices)
      const uint32_t kk = it - n2;
      const uint32_t j = kk / nseg_items, r = kk % nseg_items, e = r / G, grp = r % G;
      const HashEntry E = b.e[e];
      if (j < E.nseg) {
        if (threadIdx.x == 0) {
          constexpr uint32_t per = C::LANES / kP1Lanes, wq = kP1Lanes / 32;
          for (uint32_t q = 0; q < per; ++q)
            while (ld_acquire(&progress[e * P1 + grp * per + q]) < (j + 1) * wq) __nanosleep(256);
        }
        __syncthreads();
        const uint32_t lane0 = grp * C::LANES;
        const uint64_t rounds = E.nbytes >> 10;
        const uint64_t row0 = (uint64_t)j * kSegRows;
        const uint32_t lo0 =
            threadIdx.x < C::LANES ? __ldcg(&E.aux[(size_t)j * 256 + lane0 + threadIdx.x]) : 0u;
        const uint64_t h = run_rows<C, C::LANES, C::ROWS, false>(
            E.map, lane0, row0, min((uint64_t)kSegRows, rounds - row0), (uint64_t)lo0, stage, bars,
            bars + C::STAGES, g, nullptr, nullptr);
        if (threadIdx.x < C::LANES)
          E.aux[(size_t)(E.nseg + 1) * 256 + (size_t)j * 256 + lane0 + threadIdx.x] = (uint32_t)(h >> 32);
        if (last_part(&bigdone[e], P1 + G * E.nseg, &s_flag)) big_combine(E, lane_s);
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

// PCCLB_HASH_TWO_PHASE=0 disables the two-phase path (measurements, tests)
static bool two_phase_enabled() {
  static bool on = [] {
    const char *e = getenv("PCCLB_HASH_TWO_PHASE");
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

// pinned staging for tensor maps, reused once the previous upload finished
struct MapStaging {
  CUtensorMap *host = nullptr;
  cudaEvent_t done = nullptr;
  ~MapStaging() {
    if (host) cudaFreeHost(host);
    if (done) cudaEventDestroy(done);
  }
};

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
  if (dev >= 0 && dev < 64) done[dev] = true;
  return PCCLB_OK;
}

// Big entries: those whose full-step chain (~139 GB/s) would outlast the
// HBM-bound time of the whole call (total bytes at ~6 TB/s), at least 64 MiB.
static bool is_big(uint64_t nbytes, uint64_t total) {
  return two_phase_enabled() && nbytes >= (64ull << 20) && nbytes * 40 > total;
}

// order: entry indices, largest first
static int launch_batches(const std::vector<uint32_t> &order, const void *const *h_ptrs,
                          const uint64_t *h_nbytes, uint64_t *d_out, cudaStream_t s) {
  using C = HashC;
  const uint32_t count = (uint32_t)order.size();
  if (count == 0) return PCCLB_OK;
  int occ = 0;
  PCCLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, simplehash_batch_kernel<C>,
                                                           C::THREADS, C::SMEM));
  if (occ < 1) occ = 1;
  const uint32_t slots = (uint32_t)(sm_count() * occ);
  uint64_t total = 0;
  for (uint32_t i = 0; i < count; ++i) total += h_nbytes[i];
  // per-call device scratch: lane values, counters, tensor maps, big-entry aux
  const uint32_t m_max = std::min<uint32_t>(kMaxBatch, count);
  const size_t lanes_bytes = (size_t)m_max * 256 * sizeof(uint64_t);
  const size_t cnt_words = (size_t)m_max + 1 + kMaxBig * (kP1Groups + 1);
  const size_t cnt_bytes = (cnt_words * sizeof(uint32_t) + 127) & ~size_t(127);
  const size_t map_bytes = ((size_t)kMaxBatch + kMaxBig) * sizeof(CUtensorMap);
  size_t aux_bytes = 0;
  for (uint32_t i = 0, nb = 0; i < count && nb < kMaxBig; ++i) {
    const uint64_t n = h_nbytes[order[i]];
    if (!is_big(n, total)) continue;
    const uint64_t nseg = ((n >> 10) + kSegRows - 1) / kSegRows;
    aux_bytes += (2 * nseg + 1) * 256 * sizeof(uint32_t);
    ++nb;
  }
  char *scratch = nullptr;
  PCCLB_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&scratch),
                             lanes_bytes + cnt_bytes + map_bytes + aux_bytes, s));
  uint64_t *lanes = reinterpret_cast<uint64_t *>(scratch);
  uint32_t *cnt = reinterpret_cast<uint32_t *>(scratch + lanes_bytes);
  CUtensorMap *d_maps = reinterpret_cast<CUtensorMap *>(scratch + lanes_bytes + cnt_bytes);
  uint32_t *aux = reinterpret_cast<uint32_t *>(scratch + lanes_bytes + cnt_bytes + map_bytes);
  static thread_local HashBatch batch;
  static thread_local MapStaging staging;
  int rc = PCCLB_OK;
  bool first = true;  // big entries are only taken in the first launch
  for (uint32_t base = 0; base < count && rc == PCCLB_OK; base += kMaxBatch) {
    const uint32_t m = std::min<uint32_t>(kMaxBatch, count - base);
    if (!staging.host) {
      cudaError_t e = cudaHostAlloc(&staging.host, sizeof(CUtensorMap) * (kMaxBatch + kMaxBig),
                                    cudaHostAllocDefault);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&staging.done, cudaEventDisableTiming);
      if (e != cudaSuccess) {
        rc = cuda_status(e);
        break;
      }
    } else {
      cudaEventSynchronize(staging.done);  // previous upload out of the staging area
    }
    batch.count = m;
    batch.nbig = 0;
    batch.segmax = 0;
    uint32_t *aux_next = aux;
    uint32_t slot = 0;
    auto fill = [&](uint32_t k) {
      HashEntry &E = batch.e[slot];
      E.ptr = static_cast<const uint8_t *>(h_ptrs[k]);
      E.nbytes = h_nbytes[k];
      E.out = d_out + k;
      E.map = encode_map<C::LANES, C::ROWS>(&staging.host[slot], E.ptr, E.nbytes) ? d_maps + slot : nullptr;
      E.map1 = nullptr;
      E.aux = nullptr;
      E.nseg = 0;
      E.pad = 0;
      ++slot;
      return E;
    };
    // big entries first (slots [0, nbig)), then the others in LPT order
    std::vector<uint32_t> rest;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t k = order[base + i];
      if (!(first && batch.nbig < kMaxBig && is_big(h_nbytes[k], total))) {
        rest.push_back(k);
        continue;
      }
      HashEntry &E = batch.e[slot];
      fill(k);
      const uint32_t mi = kMaxBatch + batch.nbig;  // phase-1 map slot
      if (!E.map || !encode_map<kP1Lanes, (kP1Rows < 256 ? kP1Rows : 256)>(&staging.host[mi], E.ptr, E.nbytes)) {
        --slot;  // no tensor map: ordinary entry after all
        rest.push_back(k);
        continue;
      }
      E.map1 = d_maps + mi;
      E.nseg = (uint32_t)(((E.nbytes >> 10) + kSegRows - 1) / kSegRows);
      E.aux = aux_next;
      aux_next += (size_t)(2 * E.nseg + 1) * 256;
      batch.segmax = std::max(batch.segmax, E.nseg);
      ++batch.nbig;
    }
    std::stable_sort(rest.begin(), rest.end(),
                     [&](uint32_t a, uint32_t b) { return h_nbytes[a] > h_nbytes[b]; });
    for (uint32_t k : rest) fill(k);
    first = false;
    cudaError_t e =
        cudaMemcpyAsync(d_maps, staging.host, sizeof(CUtensorMap) * m, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && batch.nbig)
      e = cudaMemcpyAsync(d_maps + kMaxBatch, staging.host + kMaxBatch, sizeof(CUtensorMap) * batch.nbig,
                          cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventRecord(staging.done, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, cnt_words * sizeof(uint32_t), s);
    if (e != cudaSuccess) {
      rc = cuda_status(e);
      break;
    }
    const uint64_t items = (uint64_t)batch.nbig * kP1Groups + (uint64_t)(m - batch.nbig) * C::GROUPS +
                           (uint64_t)batch.segmax * batch.nbig * C::GROUPS;
    const unsigned grid = (unsigned)std::min<uint64_t>(items, slots);
    simplehash_batch_kernel<C><<<grid, C::THREADS, C::SMEM, s>>>(batch, lanes, cnt);
    e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_status(e);
  }
  cudaError_t e = cudaFreeAsync(scratch, s);
  if (rc == PCCLB_OK && e != cudaSuccess) rc = cuda_status(e);
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
