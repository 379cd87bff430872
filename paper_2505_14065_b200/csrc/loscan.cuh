// Bitsliced scan of the simplehash lo chain (phase 1 of the two-phase path in
// hash.cu; sharedstate.py:57-72 is the chain it reproduces).
//
// The lo half of one lane's FNV-1a-64 chain is lo' = (lo ^ w) * 435 mod 2^32.
// XOR and multiplication by an odd constant are T-functions: bit b of lo'
// depends only on bits 0..b of lo and w. With x = lo ^ w,
//   lo'[b] = x[b] ^ F_b(x[0..b-1]) = lo[b] ^ w[b] ^ F_b(x[0..b-1]),
// so once the lower bit planes of every row are known, bit plane b of the
// whole chain is a prefix XOR over rows: lo_r[b] = lo_0[b] ^ XOR_{k<r} t_k,
// t_k = w_k[b] ^ F_b(x_k). A serial chain of 10.5 cycles per row becomes 32
// parallel prefix scans.
//
// Layout: one warp runs one lane; thread t holds 32 consecutive rows of a
// 1024-row segment, one bit per row in each of 32 plane words (a 32x32 bit
// transpose of the 32 words it read). F_b is bit b of (x mod 2^b) * 435,
// computed bitsliced with 435 = 3 * 145 = (1 + 2)(1 + 16 * (1 + 8)):
// y = x + 2x, v = y + 8y, z = y + 16v, three two-term additions with one carry
// plane each. Per plane: an in-word prefix XOR (5 shift/xor pairs), a warp
// ballot of the words' parities and a popcount give the exclusive prefix
// across the 32 threads. K segments are in flight per warp; segment k+1's
// plane b needs only segment k's end bit b, so their dependent chains overlap
// (the code is written phase by phase so the compiler interleaves them: a
// ballot is a scheduling barrier).
//
// A lane is run by kLsWarps warps, each owning one segment of every block of
// kLsWarps consecutive segments: warp m's plane b needs the end bit b of warp
// m-1's segment (warp 0: of the last warp's segment in the previous block),
// which that warp publishes in shared memory with a plane counter as soon as
// its plane b is done. The warps form a pipeline one plane apart, so a lane
// gets kLsWarps warps of issue bandwidth.
//
// Loads: a producer warp streams blocks with one 4-D TMA box each (kLsLanes
// lanes x kLsWarps segments), the tensor viewed as [segment][i][t][lane]
// (strides 1 MiB, 1 KiB, 32 KiB, 4 B): shared memory holds word (s, i, t, l)
// at ((s*32 + i)*32 + t)*4 + l, the column read of thread t is at worst a
// 4-way bank conflict, and every TMA row request moves the 16 bytes of all
// the CTA's lanes.
#pragma once

#include <cstdint>

#include "tma.cuh"

namespace pcclb {

constexpr int kLsLanes = 4;  // lanes per CTA: 16 B of every 1 KiB row
#ifndef PCCLB_LS_WARPS
#define PCCLB_LS_WARPS 5
#endif
constexpr int kLsWarps = PCCLB_LS_WARPS;  // warps (1024-row segments per block) per lane
#ifndef PCCLB_LS_STAGES
#define PCCLB_LS_STAGES 1
#endif
constexpr int kLsStages = PCCLB_LS_STAGES;
constexpr int kLsThreads = (kLsLanes * kLsWarps + 1) * 32;  // + the TMA producer warp
constexpr uint32_t kLsBlockRows = 1024u * kLsWarps;
constexpr uint32_t kLsStageBytes = kLsBlockRows * kLsLanes * 4;
constexpr uint32_t kLoOffset = 0x84222325u;  // lo half of the FNV-1a-64 offset basis

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (a & c) | (b & c);
}

// 32x32 bit transpose: afterwards a[b] bit r = bit b of the input a[r]. The
// halfword and byte exchanges are single byte permutes (PRMT); the nibble, pair
// and bit exchanges are masked shift/xor swaps.
__device__ __forceinline__ void transpose32(uint32_t (&a)[32]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t lo = __byte_perm(a[k], a[k + 16], 0x5410), hi = __byte_perm(a[k], a[k + 16], 0x7632);
    a[k] = lo;
    a[k + 16] = hi;
  }
#pragma unroll
  for (int k = 0; k < 32; k = (k + 9) & ~8) {
    const uint32_t lo = __byte_perm(a[k], a[k + 8], 0x6240), hi = __byte_perm(a[k], a[k + 8], 0x7351);
    a[k] = lo;
    a[k + 8] = hi;
  }
#pragma unroll
  for (int j = 4, m = 0x0F0F0F0F; j != 0; j >>= 1, m ^= m << j) {
#pragma unroll
    for (int k = 0; k < 32; k = (k + j + 1) & ~j) {
      const uint32_t t = ((a[k] >> j) ^ a[k + j]) & (uint32_t)m;
      a[k + j] ^= t;
      a[k] ^= t << j;
    }
  }
}

__device__ __forceinline__ uint32_t prefix_xor32(uint32_t v) {
  v ^= v << 1;
  v ^= v << 2;
  v ^= v << 4;
  v ^= v << 8;
  v ^= v << 16;
  return v;
}

__device__ __forceinline__ uint2 ld_volatile_shared2(const uint2 *p) {
  uint2 v;
  asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_shared2(uint2 *p, uint32_t x, uint32_t y) {
  asm volatile("st.volatile.shared.v2.u32 [%0], {%1, %2};" ::"r"(smem_u32(p)), "r"(x), "r"(y) : "memory");
}
// spins until p->y == tag (warp-uniform address), returns p->x
__device__ __forceinline__ uint32_t ls_await(const uint2 *p, uint32_t tag) {
  uint32_t x;
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 y;\n"
      "LS_WAIT_%=:\n\t"
      "ld.volatile.shared.v2.u32 {%0, y}, [%1];\n\t"
      "setp.ne.u32 p, y, %2;\n\t"
      "@p bra LS_WAIT_%=;\n}"
      : "=r"(x)
      : "r"(smem_u32(p)), "r"(tag)
      : "memory");
  return x;
}
// the end word of a warp's segment from its 32 published plane bits
__device__ __forceinline__ uint32_t ls_gather(const uint2 *slots) {
  uint32_t v = 0;
#pragma unroll
  for (int b = 0; b < 32; ++b) v |= (ld_volatile_shared2(&slots[b]).x & 1u) << b;
  return v;
}
__device__ __forceinline__ uint32_t ballot_all(uint32_t pred_sign) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.lt.s32 p, %1, 0;\n\t"
      "vote.sync.ballot.b32 %0, p, 0xffffffff;\n}"
      : "=r"(r)
      : "r"(pred_sign));
  return r;
}

// The 32 plane scans of one segment. X holds the transposed words and is
// overwritten with the x planes. start_bit(b) returns bit b (in bit 0, higher
// bits ignored) of the lo value starting the segment; publish(b, e) hands on
// bit b of the value ending it (in bit 0) as soon as plane b is done. MASKED: rows whose bit in `valid` is clear
// (past the end of the entry) do not advance the chain.
template <bool MASKED, class StartBit, class Publish>
__device__ __forceinline__ void ls_planes(uint32_t (&X)[32], uint32_t valid, StartBit start_bit, Publish publish) {
  const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;
  // x[b-1], y[b-1..b-3], v[b-1..b-4], carries of y, v and z
  uint32_t xp = 0, y1 = 0, y2 = 0, y3 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0, cy = 0, cv = 0, cz = 0;
#pragma unroll
  for (int b = 0; b < 32; ++b) {
    // z[b] = x[b] ^ (x[b-1] ^ cy) ^ v[b-4] ^ cz, and lo'[b] = z[b]
    uint32_t tk = X[b] ^ xp ^ cy;
    tk ^= v4 ^ cz;
    if (MASKED) tk &= valid;
    const uint32_t incl = prefix_xor32(tk);
    const uint32_t bal = ballot_all(incl);
    const uint32_t sb = start_bit(b);
    publish(b, sb ^ (uint32_t)__popc(bal));
    const uint32_t run = (sb ^ (uint32_t)__popc(bal & lt)) & 1u;
    const uint32_t x = (incl << 1) ^ (0u - run) ^ X[b];  // x[b] = lo[b] ^ w[b]
    X[b] = x;
    const uint32_t y = x ^ xp ^ cy;
    cy = maj3(x, xp, cy);
    const uint32_t v = y ^ y3 ^ cv;
    cv = maj3(y, y3, cv);
    cz = maj3(y, v4, cz);
    xp = x;
    y3 = y2;
    y2 = y1;
    y1 = y;
    v4 = v3;
    v3 = v2;
    v2 = v1;
    v1 = v;
  }
}

// Shared state of one loscan CTA (after the TMA stages in dynamic smem).
struct LsShared {
  uint64_t full[kLsStages], empty[kLsStages];
  // per lane, warp, block parity and plane: {end bit b of the warp's segment
  // (in bit 0), block + 1}, written with one 8-byte store so a reader that
  // sees the block number also sees the bit
  uint2 endw[kLsLanes][kLsWarps][2][32];
  uint32_t hi_part[kLsLanes][kLsWarps];  // each warp's additive share of the final hi
  uint32_t final_lo[kLsLanes], final_hi[kLsLanes];
};

// dynamic shared memory of one loscan CTA: the TMA stages, then LsShared
constexpr uint32_t kLsSmem = kLsStageBytes * kLsStages + (uint32_t)sizeof(LsShared);

// 435^e mod 2^32
__device__ __forceinline__ uint32_t pow435u(uint64_t e) {
  uint32_t r = 1u, b = 435u;
  while (e) {
    if (e & 1u) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}
constexpr uint32_t kInv435 = 0xaff6957bu;  // 435^-1 mod 2^32
constexpr uint32_t kHiOffset = 0xcbf29ce4u;  // hi half of the FNV-1a-64 offset basis

// hi half of one segment's rows. X holds the x planes; turned back into row
// words it gives x_r = lo_r ^ w_r of rows 32t + i, and
//   hi' = 435 hi + c,  c = floor(435 x / 2^32) + (x << 8)  (mod 2^32)
// is affine, so a segment adds sum_r 435^(rows after r) c_r to the chain's
// final hi: Horner over the thread's 32 rows, scaled by 435^(32 (31 - t)),
// summed over the warp. MASKED: only rows with their bit set in `valid`
// count (a suffix of the segment is missing), `after` = valid rows after the
// thread's last valid row.
template <bool MASKED>
__device__ __forceinline__ uint32_t ls_hi_segment(uint32_t (&X)[32], uint32_t scale, uint32_t valid) {
  transpose32(X);
  uint32_t a = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint32_t x = X[i];
    const uint32_t c = __umulhi(x, 435u) + (x << 8);
    if (!MASKED || (valid >> i) & 1u) a = a * 435u + c;
  }
  return __reduce_add_sync(0xFFFFFFFFu, a * scale);
}

// One CTA (kLsThreads threads): the FNV-1a-64 chains of lanes lane0 ..
// lane0 + kLsLanes - 1 of one entry over its `rounds` whole rows of 1 KiB --
// the lo chain by the bitsliced scan, the hi chain from the x values the scan
// leaves behind. map: the 4-D view (box kLsLanes x 32 x 32 x kLsWarps), used
// when the entry has at least one whole 1024-row segment. Leaves lane
// lane0 + j's state after the rounds in sh->final_lo[j], sh->final_hi[j]
// (after a block-wide barrier). smem: kLsSmem bytes, 1024-byte aligned.
__device__ __forceinline__ void loscan_cta(const CUtensorMap *map, const uint8_t *ptr, uint64_t rounds,
                                           uint32_t lane0, uint8_t *smem, LsShared *sh) {
  constexpr int M = kLsWarps;
  const int t = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t nfull = rounds >> 10;                   // whole 1024-row segments
  const uint64_t nblk = (nfull + M - 1) / M;             // blocks of M segments
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLsStages; ++s) {
      mbar_init(&sh->full[s], 1);
      mbar_init(&sh->empty[s], kLsLanes * M);
    }
    mbar_fence_init();
  }
  // the slots warp 0's first segment reads (the last warp, "block -1", tag 0)
  // hold the FNV offset basis; every other slot starts out unpublished
  for (int j = threadIdx.x; j < kLsLanes * M * 64; j += blockDim.x) {
    const int b = j & 31, par = (j >> 5) & 1, ww = (j >> 6) % M;
    (&sh->endw[0][0][0][0])[j] = make_uint2(ww == M - 1 && par == 1 ? (kLoOffset >> b) & 1u : 0u, 0u);
  }
  __syncthreads();
  if (wid == kLsLanes * M) {
    // producer warp
    if (t == 0 && nblk > 0) {
      tensormap_acquire(map);
      for (uint64_t n = 0; n < nblk; ++n) {
        const int s = (int)(n % kLsStages);
        if (n >= (uint64_t)kLsStages) mbar_wait(&sh->empty[s], (uint32_t)((n / kLsStages - 1) & 1));
        mbar_expect_tx(&sh->full[s], kLsStageBytes);
        tma_4d_g2s(smem + s * kLsStageBytes, map, (int)lane0, 0, 0, (int)(n * M), &sh->full[s]);
      }
    }
  } else {
    const int l = wid / M, m = wid % M;
    const uint32_t lane = lane0 + l;
    // the warp whose end bits start this warp's segment
    const int pm = (m + M - 1) % M;
    const uint32_t scale = pow435u(32u * (31u - (uint32_t)t));
    // 435^(rows after the warp's current segment), stepped by 435^-(M * 1024)
    uint32_t mul = (uint64_t)m < nfull ? pow435u(rounds - ((uint64_t)m + 1) * 1024u) : 0u;
    const uint32_t step = [] {
      uint32_t r = 1u, b = kInv435;
      for (uint32_t e = M * 1024u; e; e >>= 1, b *= b)
        if (e & 1u) r *= b;
      return r;
    }();
    uint32_t hi = 0;
    for (uint64_t n = 0; n < nblk; ++n) {
      const int s = (int)(n % kLsStages);
      uint32_t X[32];
      mbar_wait(&sh->full[s], (uint32_t)((n / kLsStages) & 1));
      const uint32_t *sm = reinterpret_cast<const uint32_t *>(smem + s * kLsStageBytes);
#pragma unroll
      for (int i = 0; i < 32; ++i) X[i] = sm[((m * 32 + i) * 32 + t) * kLsLanes + l];
      __syncwarp();
      if (t == 0) mbar_arrive(&sh->empty[s]);
      const uint64_t seg = n * M + m;
      transpose32(X);
      // segment start: from the previous warp of this block (or the last warp
      // of the previous block; for the lane's first segment the preset slots)
      const uint64_t sn = m == 0 ? n - 1 : n;  // the source's block
      const uint2 *pend = sh->endw[l][pm][sn & 1];
      uint2 *myend = sh->endw[l][m][n & 1];
      const uint32_t stag = (uint32_t)sn + 1u, mytag = (uint32_t)n + 1u;
      auto start_bit = [&](int b) -> uint32_t { return ls_await(&pend[b], stag); };
      auto publish = [&](int b, uint32_t bit) {
        if (t == 0) st_volatile_shared2(&myend[b], bit, mytag);
      };
      if (seg < nfull) {
        ls_planes<false>(X, 0u, start_bit, publish);
        hi += mul * ls_hi_segment<false>(X, scale, 0u);
      } else {
        // past the last whole segment (zero-filled by the TMA): the chain stays as it is
        ls_planes<true>(X, 0u, start_bit, publish);
      }
      mul *= step;
    }
    // the last, partial segment (rows past the end masked): the warp that
    // follows the last whole segment runs it
    const uint64_t tail0 = nfull << 10;
    if (tail0 < rounds && m == (int)(nfull % M)) {
      uint32_t X[32];
      const uint64_t r = tail0 + 32u * t;
      const uint32_t *src = reinterpret_cast<const uint32_t *>(ptr) + lane;
#pragma unroll
      for (int i = 0; i < 32; ++i) X[i] = r + i < rounds ? __ldg(src + (r + i) * 256) : 0u;
      transpose32(X);
      const uint32_t valid = r + 32 <= rounds ? 0xFFFFFFFFu : (r >= rounds ? 0u : (1u << (uint32_t)(rounds - r)) - 1u);
      // start: the end bits of segment nfull - 1, published in block nblk - 1
      const uint2 *pend = sh->endw[l][pm][(nblk - 1) & 1];
      const uint32_t stag = (uint32_t)nblk;
      uint32_t endw = 0;
      ls_planes<true>(
          X, valid, [&](int b) -> uint32_t { return ls_await(&pend[b], stag); },
          [&](int b, uint32_t bit) { endw |= (bit & 1u) << b; });
      hi += ls_hi_segment<true>(X, pow435u(rounds > r + 32 ? rounds - (r + 32) : 0u), valid);
      if (t == 0) sh->final_lo[l] = endw;
    } else if (tail0 >= rounds && nfull > 0 && m == (int)((nfull - 1) % M)) {
      if (t == 0) sh->final_lo[l] = ls_gather(sh->endw[l][m][(nblk - 1) & 1]);
    }
    if (t == 0) sh->hi_part[l][m] = hi;
  }
  __syncthreads();
  if (threadIdx.x < kLsLanes) {
    uint32_t hi = pow435u(rounds) * kHiOffset;
#pragma unroll
    for (int m = 0; m < M; ++m) hi += sh->hi_part[threadIdx.x][m];
    sh->final_hi[threadIdx.x] = hi;
  }
  __syncthreads();
}

}  // namespace pcclb
