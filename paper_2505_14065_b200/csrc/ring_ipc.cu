// Intra-box ring all-reduce over NVLink: one process per GPU, one engine per
// process (SURVEY §8(b) engine seam; reference run_all_reduce,
// collective.py:489-576).
//
// Transport. Every rank cudaMalloc's one workspace, exports it with
// cudaIpcGetMemHandle and maps every peer's workspace
// (cudaIpcOpenMemHandle): kernels then load peer memory directly over
// NVLink 5 / NVSwitch. No NCCL collective is used -- ncclAllReduce / NVLS
// reduce in a different order and would not be bit-exact.
//
// Workspace layout (identical offsets on every rank for a given N):
//   [0, 16 KiB)       Signal: barrier arrivals / abort tokens written by peers,
//                     quantization metas, range slots, status word
//   in   [N elems]    copy of the caller's input = the backup (collective.py:501-504)
//   res  [n_c elems]  plain: fold result of the owned chunk
//   codes[s] [n_c B]  quantized: wire codes of reduce step s, written by the
//                     predecessor (one buffer per step: no reuse within an op)
//   codesF   [n_c B]  quantized: owned chunk's final codes for the gather
//   flags[s] [u64 per 64 Ki-element block] quantized: block-ready tokens of
//                     step s, written by the predecessor
//
// Plain schedule (2 barriers). Each chunk's fold chain x_c, x_{c+1}, ..., x_{c-1}
// (SURVEY §0 finding 2) is computed by the chunk's owner (rank c-1, as in the
// reference) in ONE kernel that loads the W inputs of an element -- W-1 of
// them from peers over NVLink -- folds them in ring order, divides (AVG) and
// stores. NVLink ingress per rank is (W-1)*n_c for the fold plus (W-1)*n_c for
// the gather: the ring's 2(W-1)/W*N, in one step instead of W-1.
//   copy-in  buf -> in                 (local)
//   barrier 0
//   fold     owned chunk <- fold(peers' in)  -> res, buf[owned]
//   barrier 1
//   gather   buf[c'] <- owner(c').res   for the W-1 other chunks
// Quantized schedule (W barriers): the fold order includes a quantize/
// dequantize round trip whose range spans the whole partial sum, so hops
// cannot be fused; it runs the reference's ring steps, sending u8 codes:
//   copy-in; range(tx_0)
//   step s: codes[s%2] <- Q(buf[tx_s]); barrier s;
//           buf[rx_s] <- buf[rx_s] (+) D(pred.codes[s%2]) (+ range of result)
//   prologue: codesF <- Q(buf[own]); buf[own] <- D(codesF)/W; barrier W-1
//   gather: buf[c'] <- D(owner(c').codesF)/W
//
// Synchronisation. A barrier is one tiny kernel: thread j stores the token
// (attempt << 8 | index) into peer j's arrival slot with st.release.sys and
// thread 0 polls its own slots with ld.acquire.sys. It aborts instead of
// arriving when the host abort word (set by the control plane, like the
// reference's abort_event, client.py:196-204) is raised, when a fault is
// injected (reference fault_hook, collective.py:268-272), when a quantized
// span was non-finite, when a peer posted an abort token for this attempt,
// or on timeout; it then posts its own abort token to every peer. Later
// kernels of the op see the status word and skip. The host reads the status
// at the end and restores the caller's buffer from `in` (collective.py:568-574).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>

#include "common.cuh"
#include "elementwise.cuh"
#include "ew_ops.cuh"
#include "numerics.cuh"

namespace pcclb {

constexpr int kIpcMaxWorld = 64;
constexpr uint64_t kSignalBytes = 16384;
#ifndef PCCLB_QB
#define PCCLB_QB 65536
#endif
constexpr int kIpcThreads = 512;
constexpr uint64_t kQB = PCCLB_QB;  // elements per ready-flag block of the fused quantized steps
// fused gather blocks: larger (fewer release fences; measured W=2: 64 Ki 1.92 ms, 256 Ki 1.80 ms)
#ifndef PCCLB_QF_MUL
#define PCCLB_QF_MUL 4
#endif
#ifndef PCCLB_QF_U
#define PCCLB_QF_U 2
#endif
constexpr uint64_t kQF = PCCLB_QF_MUL * kQB;
#ifndef PCCLB_QTHREADS
#define PCCLB_QTHREADS 256
#endif
constexpr int kQThreads = PCCLB_QTHREADS;
#ifndef PCCLB_QMINB
#define PCCLB_QMINB (1024 / PCCLB_QTHREADS)
#endif
constexpr int kQMinBlocks = PCCLB_QMINB;  // default 4 x 256 threads: 64 registers per thread

struct Signal {
  uint64_t arrive[kIpcMaxWorld];     // written by peer j: its latest barrier token
  uint64_t abort_tok[kIpcMaxWorld];  // written by peer j: attempt it aborted
  uint64_t desc[kIpcMaxWorld];       // written by peer j: its buffer descriptor (barrier 0)
  pcclb_qmeta meta[2];               // reduce-step metas (by step parity)
  pcclb_qmeta meta_final;            // owned chunk's gather meta
  uint32_t status;                   // this rank's op status (0 = ok)
  uint32_t pad;
  pcclb_range range[kIpcMaxWorld + 1];  // range of the span sent at step s
  pcclb_qmeta qmeta[kIpcMaxWorld];      // written by the predecessor: meta of its step-s codes
  uint32_t claim[kIpcMaxWorld + 1];     // fused quantized steps + gather: work counters
  pcclb_qmeta gmeta[kIpcMaxWorld];      // written by chunk c's owner: meta of its final codes
  uint64_t vote[kIpcMaxWorld];          // coordinator only: peer j's completion vote (attempt << 8 | failed)
  uint64_t decision;                    // written by the coordinator: attempt << 8 | 1 commit / 2 abort
  uint64_t small_copied;                // small path: attempt << 8 | 1 copied in + arrived / 2 failed
  uint64_t small_go;                    // small path: attempt << 8 | 1 every peer arrived / 2 failed
  uint32_t small_ctr[2];                // small path: CTAs done copying / folding (reset by the last CTA)
};
static_assert(sizeof(Signal) <= kSignalBytes, "signal area too small");

struct HostFlags {
  // set by the control plane: every attempt <= abort aborts (attempt-scoped,
  // so queued later attempts are not affected and nothing needs resetting)
  volatile uint64_t abort;
  uint64_t pad[7];
};

__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// polling: relaxed loads (no fence per poll), one acquire fence on success
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct BarrierArgs {
  Signal *mine;
  Signal *peer[kIpcMaxWorld];
  const HostFlags *host;   // device view of host-mapped flags
  const pcclb_range *check_range;  // nullable: abort if non-finite
  uint64_t token;
  uint64_t attempt;
  uint64_t timeout_ns;
  uint64_t desc;   // this rank's buffer descriptor (registration slot/offset)
  uint32_t rank, world;
  uint32_t fault;  // 1: inject a local fault here
  uint32_t check_desc;  // 1: every rank must publish the same descriptor
};

__global__ void __launch_bounds__(64) ipc_barrier_kernel(const __grid_constant__ BarrierArgs a) {
  __shared__ uint32_t s_verdict;
  const uint32_t t = threadIdx.x;
  Signal *me = a.mine;
  if (t == 0) {
    uint32_t v = *(volatile uint32_t *)&me->status;
    if (v == 0) {
      if (a.fault) v = PCCLB_EIO;
      else if (a.host->abort >= a.attempt) v = PCCLB_EABORTED;
      else if (a.check_range && a.check_range->nonfinite) v = PCCLB_ENONFINITE;
    }
    s_verdict = v;
  }
  __syncthreads();
  uint32_t v = s_verdict;
  if (v != 0) {
    // abort instead of arriving (keeps peers from passing this barrier)
    if (t < a.world && t != a.rank) st_release_sys(&a.peer[t]->abort_tok[a.rank], a.attempt);
    if (t == 0) *(volatile uint32_t *)&me->status = v;
    return;
  }
  __threadfence_system();
  if (t < a.world && t != a.rank) {
    if (a.check_desc) *(volatile uint64_t *)&a.peer[t]->desc[a.rank] = a.desc;
    st_release_sys(&a.peer[t]->arrive[a.rank], a.token);  // orders the desc store before it
  }
  if (t != 0) return;
  const uint64_t t0 = globaltimer();
  uint32_t verdict = 0;
  for (;;) {
    bool all = true;
    for (uint32_t j = 0; j < a.world; ++j) {
      if (j == a.rank) continue;
      if (ld_acquire_sys(&me->arrive[j]) < a.token) all = false;
      if (ld_acquire_sys(&me->abort_tok[j]) == a.attempt) verdict = PCCLB_EABORTED;
    }
    if (verdict) break;
    if (all) {
      // SPMD check: zero-copy needs every rank on the same registered buffer
      if (a.check_desc)
        for (uint32_t j = 0; j < a.world; ++j)
          if (j != a.rank && *(volatile uint64_t *)&me->desc[j] != a.desc) verdict = PCCLB_EINVAL;
      break;
    }
    if (a.host->abort >= a.attempt) {
      verdict = PCCLB_EABORTED;
      break;
    }
    if (globaltimer() - t0 > a.timeout_ns) {
      verdict = PCCLB_ETIMEOUT;
      break;
    }
    __nanosleep(64);
  }
  if (verdict) {
    for (uint32_t j = 0; j < a.world; ++j)
      if (j != a.rank) st_release_sys(&a.peer[j]->abort_tok[a.rank], a.attempt);
    *(volatile uint32_t *)&me->status = verdict;
  }
}

// peel16 usable on device too
template <typename T>
__device__ __forceinline__ uint64_t dpeel16(const void *p) {
  uintptr_t x = reinterpret_cast<uintptr_t>(p);
  return (uint64_t)(((16 - (x & 15)) & 15) / sizeof(T));
}

__device__ __forceinline__ bool op_failed(const Signal *me) {
  return *(volatile const uint32_t *)&me->status != 0;
}

// ---------------------------------------------------------------------------
// completion vote (reference COLLECTIVE_COMPLETE_VOTE, client.py:950-983):
// the op commits on every rank or on none
// ---------------------------------------------------------------------------
// Every rank posts its outcome to the coordinator (ring position 0) after all
// of its kernels of the attempt -- including remote stores into peers'
// buffers, so a vote also means "my pushes into you landed"; the coordinator
// waits for every vote and posts one decision to every rank; a rank adopts
// it. Any failure (own, a peer's, a missing vote, the host abort word)
// decides "abort" everywhere and the restore kernel that follows puts the
// caller's bytes back on every rank. Without a coordinator decision (the
// coordinator died), the wait times out and the rank aborts.
struct VoteArgs {
  Signal *mine;
  Signal *peer[kIpcMaxWorld];
  const HostFlags *host;
  uint64_t attempt;
  uint64_t timeout_ns;
  uint32_t rank, world, coord;
  uint32_t fault;  // 1: inject a local failure at the vote
};

__device__ void vote_thread0(const VoteArgs &a);

__global__ void __launch_bounds__(32) ipc_vote_kernel(const __grid_constant__ VoteArgs a) {
  if (threadIdx.x == 0) vote_thread0(a);
}

__device__ void vote_thread0(const VoteArgs &a) {
  Signal *me = a.mine;
  uint32_t st = *(volatile uint32_t *)&me->status;
  if (st == 0 && a.fault) st = PCCLB_EIO;
  if (st == 0 && a.host->abort >= a.attempt) st = PCCLB_EABORTED;
  const uint64_t tag = a.attempt << 8;
  __threadfence_system();  // this rank's earlier remote stores before its vote
  st_release_sys(&a.peer[a.coord]->vote[a.rank], tag | (st ? 1u : 0u));
  uint64_t decision = 0;
  const uint64_t t0 = globaltimer();
  if (a.rank == a.coord) {
    bool commit = st == 0;
    for (uint32_t j = 0; j < a.world; ++j) {
      if (j == a.rank) continue;
      uint64_t v;
      while (((v = ld_acquire_sys(&me->vote[j])) >> 8) != a.attempt) {
        if (globaltimer() - t0 > a.timeout_ns) break;
        __nanosleep(32);
      }
      if ((v >> 8) != a.attempt || (v & 0xff) != 0) commit = false;
    }
    decision = tag | (commit ? 1u : 2u);
    for (uint32_t j = 0; j < a.world; ++j)
      if (j != a.rank) st_release_sys(&a.peer[j]->decision, decision);
  } else {
    while (((decision = ld_acquire_sys(&me->decision)) >> 8) != a.attempt) {
      if (globaltimer() - t0 > a.timeout_ns) {
        decision = tag | 2u;
        break;
      }
      __nanosleep(32);
    }
  }
  if ((decision & 0xff) != 1u && st == 0) st = PCCLB_EABORTED;  // vetoed by a peer's failure
  *(volatile uint32_t *)&me->status = st;
}

// puts the caller's bytes back (collective.py:568-574) when the attempt
// failed -- on the device, in stream order, so a later op queued on the same
// engine copies in (and overwrites the backup) only after the restore
__global__ void __launch_bounds__(kIpcThreads) ipc_restore_kernel(const Signal *me, const uint8_t *bak, uint8_t *buf,
                                                                   uint64_t nbytes) {
  if (!op_failed(me)) return;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  // 16-byte vectors when bak and buf share their offset modulo 16, else
  // words (f32/f64 buffers are 4-byte aligned; the backup starts 16-aligned)
  const uintptr_t pb = reinterpret_cast<uintptr_t>(buf), pk = reinterpret_cast<uintptr_t>(bak);
  const uint32_t g = ((pb ^ pk) & 15) == 0 ? 16u : ((pb ^ pk) & 3) == 0 ? 4u : 1u;
  uint64_t head = (g - (pb & (g - 1))) & (g - 1);
  if (head > nbytes) head = nbytes;
  const uint64_t nv = (nbytes - head) / g;
  if (g == 16)
    for (uint64_t v = tid; v < nv; v += nth)
      reinterpret_cast<uint4 *>(buf + head)[v] = reinterpret_cast<const uint4 *>(bak + head)[v];
  else if (g == 4)
    for (uint64_t v = tid; v < nv; v += nth)
      reinterpret_cast<uint32_t *>(buf + head)[v] = reinterpret_cast<const uint32_t *>(bak + head)[v];
  else
    for (uint64_t v = tid; v < nv; v += nth) buf[head + v] = bak[head + v];
  for (uint64_t i = tid; i < head; i += nth) buf[i] = bak[i];
  for (uint64_t i = head + nv * g + tid; i < nbytes; i += nth) buf[i] = bak[i];
}

// ---------------------------------------------------------------------------
// plain fold: owned chunk from W inputs (W-1 remote), chain order
// ---------------------------------------------------------------------------
template <typename T>
struct FoldArgs {
  const T *src[kIpcMaxWorld];  // src[k] = input of ring position (c + k) at chunk c
  T *dst0;                     // res
  T *dst1;                     // caller buffer at chunk c (null: zero-copy mode)
  const Signal *mine;
  uint64_t n;
  uint32_t w;
  uint32_t avg;
  // zero-copy mode: CTAs [fold_ctas, gridDim.x) copy the caller buffer into
  // the backup meanwhile (the fold is NVLink-bound; local HBM has room)
  uint32_t fold_ctas;
  const void *bak_src;
  void *bak_dst;
  uint64_t bak_skip_lo, bak_skip_hi;  // byte range the fold itself backs up (own chunk)
  uint64_t bak_bytes;
  T *bak_own;  // fold CTAs: save src[w-1] (this rank's own input) here
};

// copy by a subset of CTAs: 16-byte vectors, with byte head/tail peeled
// (src and dst must share their offset modulo 16)
__device__ __forceinline__ void cta_range_copy(const void *src, void *dst, uint64_t bytes,
                                               uint32_t cta, uint32_t nctas) {
  const char *sc = static_cast<const char *>(src);
  char *dc = static_cast<char *>(dst);
  const uint64_t tid = (uint64_t)cta * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)nctas * blockDim.x;
  uint64_t head = (16 - (reinterpret_cast<uintptr_t>(sc) & 15)) & 15;
  if (head > bytes) head = bytes;
  if (tid < head) dc[tid] = sc[tid];
  const uint4 *s4 = reinterpret_cast<const uint4 *>(sc + head);
  uint4 *d4 = reinterpret_cast<uint4 *>(dc + head);
  const uint64_t nv = (bytes - head) / 16;
  uint64_t v = tid;
  for (; v + 3 * nth < nv; v += 4 * nth) {
    uint4 a = __ldcs(s4 + v), b = __ldcs(s4 + v + nth), c = __ldcs(s4 + v + 2 * nth), d = __ldcs(s4 + v + 3 * nth);
    __stcs(d4 + v, a);
    __stcs(d4 + v + nth, b);
    __stcs(d4 + v + 2 * nth, c);
    __stcs(d4 + v + 3 * nth, d);
  }
  for (; v < nv; v += nth) __stcs(d4 + v, __ldcs(s4 + v));
  const uint64_t t0 = head + nv * 16;
  if (tid < bytes - t0) dc[t0 + tid] = sc[t0 + tid];
}

constexpr int kFoldThreads = 256;  // 64 regs/thread: 4 CTAs (3 fold + 1 copy) fit an SM

template <typename T, int OP, int VEC>
__global__ void __launch_bounds__(kFoldThreads) ipc_fold_kernel(const __grid_constant__ FoldArgs<T> a) {
  if (blockIdx.x >= a.fold_ctas) {  // the backup runs even after a failure: restores need it
    const uint32_t c = blockIdx.x - a.fold_ctas, nc = gridDim.x - a.fold_ctas;
    cta_range_copy(a.bak_src, a.bak_dst, a.bak_skip_lo, c, nc);
    cta_range_copy(static_cast<const char *>(a.bak_src) + a.bak_skip_hi,
                   static_cast<char *>(a.bak_dst) + a.bak_skip_hi, a.bak_bytes - a.bak_skip_hi, c, nc);
    return;
  }
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)a.fold_ctas * blockDim.x;
  const uint32_t w = a.w;
  if (op_failed(a.mine)) {
    // no fold: still back up the own chunk the copy CTAs skip
    if (a.bak_own)
      for (uint64_t i = tid; i < a.n; i += nth) a.bak_own[i] = a.src[w - 1][i];
    return;
  }
  auto fin = [&](T v) { return a.avg ? div_world(v, (T)a.avg) : v; };
  auto one = [&](uint64_t i) {
    T acc = a.src[0][i];
    for (uint32_t k = 1; k < w; ++k) acc = reduce_op<OP>(a.src[k][i], acc);
    if (a.bak_own) a.bak_own[i] = a.src[w - 1][i];
    acc = fin(acc);
    a.dst0[i] = acc;
    if (a.dst1) a.dst1[i] = acc;
  };
  if constexpr (VEC == 1) {
    for (uint64_t i = tid; i < a.n; i += nth) one(i);
  } else {
    constexpr int N = Pack16<T>::N;
    uint64_t head = dpeel16<T>(a.dst0);
    if (head > a.n) head = a.n;
    if (tid < head) one(tid);
    const uint64_t nv = (a.n - head) / N;
    // U independent vectors per thread keep U*W loads (U*(W-1) over NVLink)
    // in flight; U shrinks as W grows so the registers stay bounded
    auto body = [&](auto ucount, uint64_t v0) {
      constexpr int U = decltype(ucount)::value;
      Pack16<T> acc[U], x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = ld16(a.src[0] + head + (v0 + u * nth) * N);
#pragma unroll 4
      for (uint32_t k = 1; k < w; ++k) {
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld16(a.src[k] + head + (v0 + u * nth) * N);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int e = 0; e < N; ++e) acc[u].e[e] = reduce_op<OP>(x[u].e[e], acc[u].e[e]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = head + (v0 + u * nth) * N;
        if (a.bak_own) st16(a.bak_own + i, x[u]);  // x = src[w-1], this rank's input
#pragma unroll
        for (int e = 0; e < N; ++e) acc[u].e[e] = fin(acc[u].e[e]);
        st16(a.dst0 + i, acc[u]);
        if (a.dst1) st16(a.dst1 + i, acc[u]);
      }
    };
    uint64_t v = tid;
    if (w <= 2) {
      for (; v + 3 * nth < nv; v += 4 * nth) body(std::integral_constant<int, 4>{}, v);
    } else if (w <= 4) {
      for (; v + nth < nv; v += 2 * nth) body(std::integral_constant<int, 2>{}, v);
    }
    for (; v < nv; v += nth) body(std::integral_constant<int, 1>{}, v);
    const uint64_t t0 = head + nv * N;
    if (tid < a.n - t0) one(t0 + tid);
  }
}


// ---------------------------------------------------------------------------
// small messages (plain ops): the whole attempt in one kernel
// ---------------------------------------------------------------------------
// For short buffers the attempt is latency-bound: every kernel boundary and
// barrier costs microseconds. One kernel of G co-resident CTAs copies the
// caller's buffer into `in`, arrives (the last CTA to finish copying posts
// the arrival token and the parameter descriptor to every peer), waits for
// every peer's arrival, folds EVERY chunk locally from the W inputs (W-1 read
// over NVLink) in its ring order x_c, x_{c+1}, ..., x_{c-1} -- the same values
// as the owner's fold, with (W-1)*N instead of 2(W-1)/W*N ingress, which does
// not matter at these sizes -- and the last CTA to finish folding runs the
// completion vote and, on a failed attempt, the restore. Abort points:
// fault_at 0/1 at the arrival, 2 at the vote.
template <typename T>
struct SmallArgs {
  T *buf;                         // caller buffer (written with the result)
  T *in;                          // this rank's workspace copy (read by peers)
  const T *pin[kIpcMaxWorld];     // input of ring position p (pin[rank] = in)
  uint64_t lo[kIpcMaxWorld + 1];  // chunk bounds
  uint64_t n;
  VoteArgs v;                     // mine, peers, host, attempt, timeout, rank, world, coord, fault (vote)
  uint64_t desc;
  uint32_t fault_arrive;
  uint32_t avg;
  uint32_t *status_out;           // host-mapped: the attempt's final status
};

// copy over CTAs [cta, cta + nctas): 16-byte vectors when both sides share
// their offset modulo 16, else 4-byte words (f32/f64 buffers)
__device__ __forceinline__ void cta_copy_any(const void *src, void *dst, uint64_t bytes, uint32_t cta,
                                             uint32_t nctas) {
  if (((reinterpret_cast<uintptr_t>(src) ^ reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    cta_range_copy(src, dst, bytes, cta, nctas);
    return;
  }
  const uint32_t *s4 = static_cast<const uint32_t *>(src);
  uint32_t *d4 = static_cast<uint32_t *>(dst);
  const uint64_t tid = (uint64_t)cta * blockDim.x + threadIdx.x, nth = (uint64_t)nctas * blockDim.x;
  for (uint64_t i = tid; i < bytes / 4; i += nth) d4[i] = s4[i];
}

template <typename T, int OP>
__global__ void __launch_bounds__(kIpcThreads) ipc_small_kernel(const __grid_constant__ SmallArgs<T> a) {
  __shared__ uint32_t s_flag;
  Signal *me = a.v.mine;
  const uint32_t G = gridDim.x, w = a.v.world, rank = a.v.rank;
  const uint64_t token = a.v.attempt << 8;  // barrier index 0
  if (blockIdx.x == 0 && threadIdx.x == 0) *(volatile uint32_t *)&me->status = 0u;  // read after the copy counter
  // 1. copy-in (every CTA its share)
  cta_copy_any(a.buf, a.in, a.n * sizeof(T), blockIdx.x, G);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_flag = atomicAdd(&me->small_ctr[0], 1u) == G - 1;
  }
  __syncthreads();
  if (s_flag && threadIdx.x == 0) {
    // the last copier arrives for this rank (or aborts instead)
    uint32_t v = *(volatile uint32_t *)&me->status;
    if (v == 0 && a.fault_arrive) v = PCCLB_EIO;
    if (v == 0 && a.v.host->abort >= a.v.attempt) v = PCCLB_EABORTED;
    if (v) {
      *(volatile uint32_t *)&me->status = v;
      for (uint32_t j = 0; j < w; ++j)
        if (j != rank) st_release_sys(&a.v.peer[j]->abort_tok[rank], a.v.attempt);
    } else {
      __threadfence_system();
      for (uint32_t j = 0; j < w; ++j)
        if (j != rank) {
          *(volatile uint64_t *)&a.v.peer[j]->desc[rank] = a.desc;
          st_release_sys(&a.v.peer[j]->arrive[rank], token);
        }
    }
    __threadfence();
    *(volatile uint64_t *)&me->small_copied = token | (v ? 2u : 1u);
  }
  // 2. CTA 0 waits for this rank's own arrival and every peer's (host abort
  // and timeout polled there only), then releases the other CTAs through a
  // local flag
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t verdict = 0;
    uint64_t c;
    while (((c = *(volatile uint64_t *)&me->small_copied) >> 8) != a.v.attempt) {
    }
    if ((c & 0xff) != 1u) verdict = PCCLB_EABORTED;
    const uint64_t t0 = globaltimer();
    for (uint32_t spin = 0; !verdict; ++spin) {
      bool all = true;
      for (uint32_t j = 0; j < w; ++j) {
        if (j == rank) continue;
        if (ld_relaxed_sys(&me->arrive[j]) < token) all = false;
        if (ld_relaxed_sys(&me->abort_tok[j]) == a.v.attempt) verdict = PCCLB_EABORTED;
      }
      if (verdict) break;
      if (all) {
        __threadfence_system();  // acquire: the peers' copies are visible
        for (uint32_t j = 0; j < w; ++j)
          if (j != rank && *(volatile uint64_t *)&me->desc[j] != a.desc) verdict = PCCLB_EINVAL;
        break;
      }
      if ((spin & 63) == 63) {  // host memory and the clock: every 64 polls
        if (a.v.host->abort >= a.v.attempt) verdict = PCCLB_EABORTED;
        else if (globaltimer() - t0 > a.v.timeout_ns) verdict = PCCLB_ETIMEOUT;
      }
    }
    if (verdict) {
      atomicCAS(&me->status, 0u, verdict);
      for (uint32_t j = 0; j < w; ++j)
        if (j != rank) st_release_sys(&a.v.peer[j]->abort_tok[rank], a.v.attempt);
    }
    __threadfence();
    *(volatile uint64_t *)&me->small_go = token | (verdict ? 2u : 1u);
  }
  if (threadIdx.x == 0) {
    uint64_t gv;
    while (((gv = *(volatile uint64_t *)&me->small_go) >> 8) != a.v.attempt) __nanosleep(20);
    s_flag = (gv & 0xff) == 1u;
    __threadfence();
  }
  __syncthreads();
  // 3. fold every chunk in its ring order: 16-byte loads of every input (the
  // workspaces are 16-byte aligned), U vectors per thread in flight
  if (s_flag) {
    constexpr int N = Pack16<T>::N, U = 4;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (uint64_t)G * blockDim.x;
    const bool vst = (reinterpret_cast<uintptr_t>(a.buf) & 15) == 0;
    auto fin = [&](T v) { return a.avg ? div_world(v, (T)a.avg) : v; };
    for (uint32_t c = 0; c < w; ++c) {
      const uint64_t c0 = a.lo[c], c1 = a.lo[c + 1];
      auto src = [&](uint32_t k) { return a.pin[c + k < w ? c + k : c + k - w]; };
      auto one = [&](uint64_t i) {
        T acc = src(0)[i];
        for (uint32_t k = 1; k < w; ++k) acc = reduce_op<OP>(src(k)[i], acc);
        a.buf[i] = fin(acc);
      };
      uint64_t v0 = (c0 + N - 1) / N, v1 = c1 / N;
      if (v1 < v0) v1 = v0;
      for (uint64_t i = c0 + tid; i < c1 && i < v0 * N; i += nth) one(i);  // head
      for (uint64_t i = v1 * N + tid; i < c1; i += nth)                     // tail
        if (i >= v0 * N) one(i);
      for (uint64_t vb = v0 + tid; vb < v1; vb += nth * U) {
        Pack16<T> acc[U], x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (vb + u * nth < v1) acc[u] = ld16(src(0) + (vb + u * nth) * N);
        for (uint32_t k = 1; k < w; ++k) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (vb + u * nth < v1) x[u] = ld16(src(k) + (vb + u * nth) * N);
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < N; ++e) acc[u].e[e] = reduce_op<OP>(x[u].e[e], acc[u].e[e]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (vb + u * nth >= v1) continue;
#pragma unroll
          for (int e = 0; e < N; ++e) acc[u].e[e] = fin(acc[u].e[e]);
          T *d = a.buf + (vb + u * nth) * N;
          if (vst) {
            st16(d, acc[u]);
          } else {
#pragma unroll
            for (int e = 0; e < N; ++e) d[e] = acc[u].e[e];
          }
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    s_flag = atomicAdd(&me->small_ctr[1], 1u) == G - 1;
  }
  __syncthreads();
  if (!s_flag) return;
  // 4. the last CTA: completion vote, then the restore of a failed attempt
  if (threadIdx.x == 0) vote_thread0(a.v);
  __syncthreads();
  if (op_failed(me)) cta_copy_any(a.in, a.buf, a.n * sizeof(T), 0, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    me->small_ctr[0] = 0;
    me->small_ctr[1] = 0;
    __threadfence_system();
    *(volatile uint32_t *)a.status_out = *(volatile uint32_t *)&me->status;
  }
}

// ---------------------------------------------------------------------------
// gather: W-1 chunk copies (grid.y = job), plain (verbatim) or quantized (dequant)
// ---------------------------------------------------------------------------
struct GatherArgs {
  const void *src[kIpcMaxWorld];       // plain: owner's res; quantized: owner's codesF
  const pcclb_qmeta *meta[kIpcMaxWorld];  // quantized: owner's meta_final
  void *dst[kIpcMaxWorld];             // caller buffer at that chunk
  void *bak[kIpcMaxWorld];             // plain, zero-copy: save the old bytes here first
  uint64_t n[kIpcMaxWorld];
  const Signal *mine;
  uint32_t avg;
};

// dst <- src, optionally saving dst's old contents to bak (fused backup:
// the gather is NVLink-bound, so the extra local read+write is free)
template <typename T, bool BAK>
__device__ __forceinline__ void gather_copy(const T *src, T *dst, T *bak, uint64_t n) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  constexpr int N = Pack16<T>::N;
  auto one = [&](uint64_t i) {
    if (BAK) bak[i] = dst[i];
    dst[i] = src[i];
  };
  uint64_t head = dpeel16<T>(dst);
  if (head > n) head = n;
  const bool vec = dpeel16<T>(src) == head && (!BAK || dpeel16<T>(bak) == head);
  if (!vec) {
    for (uint64_t i = tid; i < n; i += nth) one(i);
    return;
  }
  if (tid < head) one(tid);
  const uint64_t nv = (n - head) / N;
  const T *s0 = src + head;
  T *d0 = dst + head;
  T *b0 = BAK ? bak + head : nullptr;
  uint64_t v = tid;
  constexpr int U = 4;
  for (; v + (U - 1) * nth < nv; v += U * nth) {
    Pack16<T> x[U], o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = ld16(s0 + (v + u * nth) * N);
    if (BAK) {
#pragma unroll
      for (int u = 0; u < U; ++u) o[u] = ld16(d0 + (v + u * nth) * N);
#pragma unroll
      for (int u = 0; u < U; ++u) st16(b0 + (v + u * nth) * N, o[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) st16(d0 + (v + u * nth) * N, x[u]);
  }
  for (; v < nv; v += nth) {
    Pack16<T> x = ld16(s0 + v * N);
    if (BAK) st16(b0 + v * N, ld16(d0 + v * N));
    st16(d0 + v * N, x);
  }
  const uint64_t t0 = head + nv * N;
  if (tid < n - t0) one(t0 + tid);
}

// All chunk copies interleaved in one grid: iteration v moves vector v of
// EVERY job (a load from each owner issued before any store), so every peer
// link is busy all the time, like the fold's access pattern. Chunk lengths
// differ by at most one element; the shared alignment is checked on the host.
template <typename T>
__global__ void __launch_bounds__(kIpcThreads, 2)
    ipc_gather_interleaved_kernel(const __grid_constant__ GatherArgs a, uint32_t jobs, uint64_t head) {
  if (op_failed(a.mine)) return;
  constexpr int N = Pack16<T>::N;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  uint64_t nmin = a.n[0];
  for (uint32_t j = 1; j < jobs; ++j) nmin = a.n[j] < nmin ? a.n[j] : nmin;
  if (head > nmin) head = nmin;
  const uint64_t nv = (nmin - head) / N;
  for (uint64_t v = tid; v < nv; v += nth) {
    Pack16<T> x[kIpcMaxWorld > 8 ? 8 : kIpcMaxWorld];
    for (uint32_t j0 = 0; j0 < jobs; j0 += 8) {
      const uint32_t m = jobs - j0 < 8 ? jobs - j0 : 8;
#pragma unroll
      for (uint32_t j = 0; j < 8; ++j)
        if (j < m) x[j] = ld16(static_cast<const T *>(a.src[j0 + j]) + head + v * N);
#pragma unroll
      for (uint32_t j = 0; j < 8; ++j)
        if (j < m) st16(static_cast<T *>(a.dst[j0 + j]) + head + v * N, x[j]);
    }
  }
  // heads and tails (incl. the longer chunks' last element) element-wise
  const uint64_t t0 = head + nv * N;
  for (uint32_t j = 0; j < jobs; ++j) {
    const T *src = static_cast<const T *>(a.src[j]);
    T *dst = static_cast<T *>(a.dst[j]);
    if (tid < head) dst[tid] = src[tid];
    for (uint64_t i = t0 + tid; i < a.n[j]; i += nth) dst[i] = src[i];
  }
}

template <typename T>
__global__ void __launch_bounds__(kIpcThreads, 2) ipc_gather_plain_kernel(const __grid_constant__ GatherArgs a) {
  if (op_failed(a.mine)) return;
  const uint32_t j = blockIdx.y;
  const T *src = static_cast<const T *>(a.src[j]);
  T *dst = static_cast<T *>(a.dst[j]);
  if (a.bak[j])
    gather_copy<T, true>(src, dst, static_cast<T *>(a.bak[j]), a.n[j]);
  else
    gather_copy<T, false>(src, dst, nullptr, a.n[j]);
}

// Push gather (zero-copy buffers only): the owner stores its folded chunk
// straight into every peer's registered buffer (remote stores; a third
// barrier then tells each rank that all pushes into it landed).
template <typename T>
struct PushArgs {
  const T *src;                 // own result (local)
  T *dst[kIpcMaxWorld];         // peers' registered buffers at the owned chunk
  uint32_t ndst;
  uint32_t vec;  // every dst shares src's offset modulo 16
  uint64_t n;
  const Signal *mine;
};

template <typename T>
__global__ void __launch_bounds__(kIpcThreads, 2) ipc_push_kernel(const __grid_constant__ PushArgs<T> a) {
  if (op_failed(a.mine)) return;
  constexpr int N = Pack16<T>::N;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  uint64_t head = a.vec ? dpeel16<T>(a.src) : 0;
  if (head > a.n) head = a.n;
  const uint64_t nv = a.vec ? (a.n - head) / N : 0;
  for (uint64_t v = tid; v < nv; v += nth) {
    const Pack16<T> x = ld16(a.src + head + v * N);
    for (uint32_t j = 0; j < a.ndst; ++j) st16(a.dst[j] + head + v * N, x);
  }
  const uint64_t t0 = head + nv * N;
  for (uint32_t j = 0; j < a.ndst; ++j) {
    if (tid < head) a.dst[j][tid] = a.src[tid];
    for (uint64_t i = t0 + tid; i < a.n; i += nth) a.dst[j][i] = a.src[i];
  }
}

// Quantized gather: every owner's final codes dequantized (+ AVG division)
// into this rank's buffer, all jobs interleaved per thread like the plain
// gather, 16 codes (one 16-byte NVLink load) per job per iteration. Each job
// has its own head (chunk starts differ modulo 16 elements).
__global__ void __launch_bounds__(kIpcThreads, 2)
    ipc_gather_quant_kernel(const __grid_constant__ GatherArgs a, uint32_t jobs, int vec) {
  if (op_failed(a.mine)) return;
  __shared__ float s_mn[kIpcMaxWorld], s_sc[kIpcMaxWorld];
  __shared__ uint64_t s_head[kIpcMaxWorld];
  for (uint32_t j = threadIdx.x; j < jobs; j += blockDim.x) {
    const pcclb_qmeta m = *a.meta[j];  // owner's meta_final (peer memory)
    s_mn[j] = m.min_val;
    s_sc[j] = m.scale;
    uint64_t h = vec ? dpeel64f(static_cast<const float *>(a.dst[j])) : 0;
    s_head[j] = h > a.n[j] ? a.n[j] : h;
  }
  __syncthreads();
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const float avg = (float)a.avg;
  const bool div = a.avg > 1;
  auto val = [&](uint32_t j, uint32_t q) {
    float d = dequant1(q, s_mn[j], s_sc[j]);
    return div ? div_world(d, avg) : d;
  };
  uint64_t nv = ~0ull;
  for (uint32_t j = 0; j < jobs; ++j) {
    const uint64_t v = (a.n[j] - s_head[j]) / 16;
    nv = v < nv ? v : nv;
  }
  if (!vec) nv = 0;  // codes and floats not co-aligned: element-wise below
  for (uint64_t v = tid; v < nv; v += nth) {
    for (uint32_t j0 = 0; j0 < jobs; j0 += 8) {
      const uint32_t m = jobs - j0 < 8 ? jobs - j0 : 8;
      uint4 q[8];
#pragma unroll
      for (uint32_t j = 0; j < 8; ++j)
        if (j < m)
          q[j] = *reinterpret_cast<const uint4 *>(static_cast<const uint8_t *>(a.src[j0 + j]) + s_head[j0 + j] + v * 16);
#pragma unroll
      for (uint32_t j = 0; j < 8; ++j)
        if (j < m) {
          float *dst = static_cast<float *>(a.dst[j0 + j]) + s_head[j0 + j] + v * 16;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            Pack16<float> d;
#pragma unroll
            for (int e = 0; e < 4; ++e) d.e[e] = val(j0 + j, code_byte(q[j], 4 * g + e));
            st16(dst + 4 * g, d);
          }
        }
    }
  }
  // heads and tails element-wise
  for (uint32_t j = 0; j < jobs; ++j) {
    const uint8_t *codes = static_cast<const uint8_t *>(a.src[j]);
    float *dst = static_cast<float *>(a.dst[j]);
    const uint64_t h = s_head[j], t0 = h + nv * 16;
    if (tid < h) dst[tid] = val(j, codes[tid]);
    for (uint64_t i = t0 + tid; i < a.n[j]; i += nth) dst[i] = val(j, codes[i]);
  }
}

// ---------------------------------------------------------------------------
// quantized step kernels (skip after a failure)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kIpcThreads, 2)
    ipc_range_kernel(const float *x, uint64_t n, pcclb_range *out, float *bak, const Signal *mine) {
  // runs before the first barrier: also saves this (never rx) chunk's input
  RangeBakF f{x, bak, RangeAcc()};
  uint64_t head = dpeel16<float>(x);
  if (dpeel16<float>(bak) == head)
    ew_loop<4, 4>(n, head, f);
  else
    ew_loop<1, 1>(n, 0, f);
  range_block_commit(f.acc, out);
}

__global__ void __launch_bounds__(kIpcThreads, 2)
    ipc_quantize_kernel(const float *x, uint64_t n, const pcclb_range *range, uint8_t *codes,
                        pcclb_qmeta *meta, float *adopt, uint32_t avg, const Signal *mine) {
  if (op_failed(mine)) return;
  QParams qp = qparams_from_range(*range);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    meta->min_val = qp.mn;
    meta->scale = qp.scale;
  }
  const uint64_t head = dpeel64f(x);
  if (((reinterpret_cast<uintptr_t>(codes) + head) & 15) == 0 &&
      (!adopt || dpeel64f(adopt) == head)) {
    Quant16F f{x, codes, adopt, qp, (float)avg, avg > 1};
    ew_loop<16, 2>(n, head, f);
  } else {
    QuantF f{x, codes, adopt, qp, (float)avg, avg > 1};
    ew_loop<1, 1>(n, 0, f);
  }
}

template <int OP>
__global__ void __launch_bounds__(kIpcThreads, 2)
    ipc_dequant_acc_kernel(float *acc, const uint8_t *codes, uint64_t n, const pcclb_qmeta *meta,
                           pcclb_range *next, float *bak, const Signal *mine, int mode) {
  const uint64_t head = dpeel64f(acc);
  const bool bak_ok = dpeel16<float>(bak) == dpeel16<float>(acc);
  const bool vec = ((reinterpret_cast<uintptr_t>(codes) + head) & 15) == 0 && bak_ok;
  if (op_failed(mine)) {
    // no accumulate, but the backup of this rx chunk must exist for the restore
    CopyF f{acc, bak};
    if (bak_ok)
      ew_loop<4, 4>(n, dpeel16<float>(acc), f);
    else
      ew_loop<1, 1>(n, 0, f);
    return;
  }
  const pcclb_qmeta m = *meta;  // peer memory
  const uint64_t head4 = dpeel16<float>(acc);
  if (mode == 1 && bak_ok && ((reinterpret_cast<uintptr_t>(codes) + head4) & 3) == 0) {
    DequantAccF<OP> f{acc, codes, m.min_val, m.scale, true, RangeAcc(), bak};
    ew_loop<4, 4>(n, head4, f);
    range_block_commit(f.r, next);
  } else if (vec && mode == 2) {
    DequantAcc16F<OP> f{acc, codes, m.min_val, m.scale, RangeAcc(), bak};
    ew_loop<16, 4>(n, head, f);
    range_block_commit(f.r, next);
  } else if (vec) {
    DequantAcc16F<OP> f{acc, codes, m.min_val, m.scale, RangeAcc(), bak};
    ew_loop<16, 2>(n, head, f);
    range_block_commit(f.r, next);
  } else {
    DequantAccF<OP> f{acc, codes, m.min_val, m.scale, true, RangeAcc(), bak};
    ew_loop<1, 1>(n, 0, f);
    range_block_commit(f.r, next);
  }
}

// ---------------------------------------------------------------------------
// Fused quantized reduce step (one kernel per ring step, no barrier).
//
// Step s of the reference's quantized ring (collective.py:521-536) on rank r:
//   A: codes <- Q(buf[tx_s]) with the range the previous step produced, sent
//      to the successor -- here pushed over NVLink into the successor's
//      codes[s] with remote 16-byte stores, 64 Ki elements per block, each
//      block followed by a ready token (st.release.sys) in its flags[s];
//   B: for each block once the predecessor's token for it is visible
//      (ld.acquire.sys): save buf[rx_s] (first touch of the rx chunk = the
//      backup) and accumulate the range of the partial buf[rx_s] (+) D(pred's
//      codes[s]) for step s+1's quantization. The partial itself is not
//      stored: step s+1's A (or the owner's adoption) recomputes it.
// Work items are claimed in order from a per-step counter, A block j at
// position 2j and B block j at 2j + 2*lag + 1, the same positions on every
// rank. A items never wait, so a claimed B item always has its producer's A
// item claimed or claimable on the predecessor (its position is smaller):
// no cyclic wait, with any number of resident CTAs. The interleaving keeps
// the NVLink pushes (A) and the HBM-bound accumulation (B) running at once.
// Failures (fault injection, non-finite range, host abort, a peer's abort
// token, timeout) set the status word and post abort tokens like the barrier
// kernel; after a failure A items are skipped and B items only save the
// backup, so the host restore finds every chunk's input.
// ---------------------------------------------------------------------------
struct QStepArgs {
  const float *tx;            // this rank's tx chunk (caller buffer)
  uint8_t *tcodes;            // successor's codes[s] at element 0 of the tx chunk
  pcclb_qmeta *tmeta;         // successor's qmeta[s]
  uint64_t *tflags;           // successor's flags[s]
  const pcclb_range *trange;  // range of the tx chunk (previous step)
  const uint8_t *pcodes;      // step >= 1: own codes[s-1] at element 0 of the tx chunk (the
  const pcclb_qmeta *pmeta;   //   tx chunk's partial is buf (+) D(codes[s-1]), never stored)
  float *rx;                  // rx chunk (caller buffer)
  float *rbak;                // backup of the rx chunk
  const uint8_t *rcodes;      // own codes[s] at element 0 of the rx chunk
  const pcclb_qmeta *rmeta;   // own qmeta[s]
  const uint64_t *rflags;     // own flags[s]
  pcclb_range *rrange;        // range of the new partial (next step)
  Signal *mine;
  Signal *peer[kIpcMaxWorld];
  const HostFlags *host;
  uint32_t *claim;
  uint64_t tlo, tn, rlo, rn;
  uint64_t token, attempt, timeout_ns;
  uint32_t rank, world, fault, lag;
  uint32_t tvec, rvec;  // 16-element vector bodies usable on the A / B side
  uint32_t dbg;         // experiments (PCCLB_QDEBUG bits): 1 = B never waits, 2 = A stores locally
};

__device__ __forceinline__ uint64_t qblocks(uint64_t lo, uint64_t n, uint64_t qb = kQB) {
  return n ? (lo + n - 1) / qb - lo / qb + 1 : 0;
}
// chunk-relative element range of block j (blocks follow the global kQB grid,
// so producer and consumer agree whatever their buffers' alignment)
__device__ __forceinline__ void qblock_range(uint64_t lo, uint64_t n, uint64_t j, uint64_t &i0, uint64_t &i1,
                                             uint64_t qb = kQB) {
  const uint64_t k = lo / qb + j;
  uint64_t g0 = k * qb, g1 = g0 + qb;
  if (g0 < lo) g0 = lo;
  if (g1 > lo + n) g1 = lo + n;
  i0 = g0 - lo;
  i1 = g1 - lo;
}

template <class A>
__device__ __forceinline__ void qfail(const A &a, uint32_t v) {
  if (atomicCAS(&a.mine->status, 0u, v) == 0u)
    for (uint32_t j = 0; j < a.world; ++j)
      if (j != a.rank) st_release_sys(&a.peer[j]->abort_tok[a.rank], a.attempt);
}

// thread 0: wait for the predecessor's ready token (0) or a failure (status)
template <class A>
__device__ uint32_t qwait(const A &a, const uint64_t *flag) {
  uint32_t rc = 0;
  if (ld_relaxed_sys(flag) < a.token) {
    const uint64_t t0 = globaltimer();
    uint32_t ns = 64;
    for (uint32_t it = 0;; ++it) {
      __nanosleep(ns);
      if (ns < 1024) ns *= 2;
      if (ld_relaxed_sys(flag) >= a.token) break;
      const uint32_t st = *(volatile uint32_t *)&a.mine->status;
      if (st) return st;
      if ((it & 7) == 0) {
        if (a.host->abort >= a.attempt) return PCCLB_EABORTED;
        for (uint32_t j = 0; j < a.world; ++j)
          if (j != a.rank && ld_relaxed_sys(&a.mine->abort_tok[j]) == a.attempt) return PCCLB_EABORTED;
        if (globaltimer() - t0 > a.timeout_ns) return PCCLB_ETIMEOUT;
      }
    }
  }
  // acquire (an acquire load, not a fence: no MEMBAR behind this CTA's own
  // outstanding stores): the block's codes and meta are visible after this
  (void)ld_acquire_sys(flag);
  return rc;
}

// CTA-wide loop over chunk-relative elements [i0, i1): 16-element vectors
// where the global index is a multiple of 16, scalar head and tail
template <int U, typename F>
__device__ __forceinline__ void cta_loop16(uint64_t lo, uint64_t i0, uint64_t i1, bool vec, F &f) {
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  if (!vec) {
    for (uint64_t i = i0 + t; i < i1; i += nt) f.one(i);
    return;
  }
  uint64_t head = (16 - ((lo + i0) & 15)) & 15;
  if (head > i1 - i0) head = i1 - i0;
  if (t < head) f.one(i0 + t);
  const uint64_t b = i0 + head;
  const uint64_t nv = (i1 - b) / 16;
  uint64_t v = t;
  for (; v + (U - 1) * nt < nv; v += U * nt) {
    typename F::In in[U];
#pragma unroll
    for (int u = 0; u < U; ++u) in[u] = f.vload(b + (v + u * nt) * 16);
#pragma unroll
    for (int u = 0; u < U; ++u) f.vapply(b + (v + u * nt) * 16, in[u]);
  }
  for (; v < nv; v += nt) {
    typename F::In in = f.vload(b + v * 16);
    f.vapply(b + v * 16, in);
  }
  const uint64_t t0 = b + nv * 16;
  if (t0 + t < i1) f.one(t0 + t);
}

// the same with 4-element vectors (lane-contiguous 16-byte accesses)
template <int U, typename F>
__device__ __forceinline__ void cta_loop4(uint64_t lo, uint64_t i0, uint64_t i1, bool vec, F &f) {
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  if (!vec) {
    for (uint64_t i = i0 + t; i < i1; i += nt) f.one(i);
    return;
  }
  uint64_t head = (4 - ((lo + i0) & 3)) & 3;
  if (head > i1 - i0) head = i1 - i0;
  if (t < head) f.one(i0 + t);
  const uint64_t b = i0 + head;
  const uint64_t nv = (i1 - b) / 4;
  uint64_t v = t;
  for (; v + (U - 1) * nt < nv; v += U * nt) {
    typename F::In in[U];
#pragma unroll
    for (int u = 0; u < U; ++u) in[u] = f.vload(b + (v + u * nt) * 4);
#pragma unroll
    for (int u = 0; u < U; ++u) f.vapply(b + (v + u * nt) * 4, in[u]);
  }
  for (; v < nv; v += nt) {
    typename F::In in = f.vload(b + v * 4);
    f.vapply(b + v * 4, in);
  }
  const uint64_t t0 = b + nv * 4;
  if (t0 + t < i1) f.one(t0 + t);
}

#ifndef PCCLB_QB_U
#define PCCLB_QB_U 8
#endif
#ifndef PCCLB_QR_U
#define PCCLB_QR_U 4
#endif

// The running partial of a chunk is never written back to the caller's
// buffer: the consumer of step s only saves the backup and accumulates the
// range of buf[rx] (+) D(codes[s]); whoever needs the partial next (the
// producer of step s+1, or the owner's adoption) recomputes it from the same
// two inputs with the same arithmetic -- 5 bytes read instead of a 4-byte
// write plus a 4-byte read per element and step.
template <int OP>
__device__ __forceinline__ float partial_of(float local, uint32_t q, float mn, float scale) {
  return reduce_op_x<OP, false>(local, dequant1x<false>(q, mn, scale));
}

// consumer of a step: bak <- buf[rx], range of buf[rx] (+) D(codes)
template <int OP>
struct DequantRange4F {
  const float *__restrict__ acc;
  const uint8_t *__restrict__ codes;
  float mn, scale;
  RangeAcc r;
  float *__restrict__ bak;
  __device__ __forceinline__ void one(uint64_t i) {
    const float old = acc[i];
    bak[i] = old;
    r.add(partial_of<OP>(old, __ldcg(codes + i), mn, scale));
  }
  struct In {
    Pack16<float> a;
    uint32_t q;
  };
  __device__ __forceinline__ In vload(uint64_t i) {
    In v;
    v.a = ld16(acc + i);
    v.q = __ldcg(reinterpret_cast<const uint32_t *>(codes + i));
    return v;
  }
  __device__ __forceinline__ void vapply(uint64_t i, const In &v) {
    st16(bak + i, v.a);
#pragma unroll
    for (int k = 0; k < 4; ++k) r.add(partial_of<OP>(v.a.e[k], (v.q >> (8 * k)) & 0xffu, mn, scale));
  }
};

// producer of step s >= 1: codes <- Q(buf[tx] (+) D(codes[s-1]))
template <int OP>
struct QuantPart16F {
  const float *__restrict__ x;
  const uint8_t *__restrict__ pcodes;
  float pmn, pscale;
  uint8_t *__restrict__ codes;
  QParams qp;
  __device__ __forceinline__ void one(uint64_t i) {
    const float v = partial_of<OP>(x[i], __ldcg(pcodes + i), pmn, pscale);
    codes[i] = (uint8_t)quant1_fast(v, qp.mn, qp.scale, qp.inv);
  }
  struct In {
    Pack16<float> a[4];
    uint4 p;
  };
  __device__ __forceinline__ In vload(uint64_t i) {
    In v;
    v.p = __ldcg(reinterpret_cast<const uint4 *>(pcodes + i));
#pragma unroll
    for (int g = 0; g < 4; ++g) v.a[g] = ld16(x + i + 4 * g);
    return v;
  }
  __device__ __forceinline__ void vapply(uint64_t i, const In &v) {
    uint32_t w[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint32_t q[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        q[k] = quant1_fast(partial_of<OP>(v.a[g].e[k], code_byte(v.p, 4 * g + k), pmn, pscale), qp.mn, qp.scale,
                           qp.inv);
      w[g] = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
    }
    *reinterpret_cast<uint4 *>(codes + i) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};

template <int OP>
__global__ void __launch_bounds__(kQThreads, kQMinBlocks) ipc_qstep_kernel(const __grid_constant__ QStepArgs a) {
  __shared__ uint32_t s_item, s_ok;
  const uint64_t nA = qblocks(a.tlo, a.tn), nB = qblocks(a.rlo, a.rn);
  uint64_t npos = 2 * nA;
  if (nB && 2 * (nB + a.lag) > npos) npos = 2 * (nB + a.lag);
  if (threadIdx.x == 0 && *(volatile uint32_t *)&a.mine->status == 0) {
    if (blockIdx.x == 0 && a.fault) qfail(a, PCCLB_EIO);  // reference fault_hook
    else if (a.tn && a.trange->nonfinite) qfail(a, PCCLB_ENONFINITE);
  }
  const QParams qp = qparams_from_range(*a.trange);
  RangeAcc racc;
  for (;;) {
    if (threadIdx.x == 0) {
      const uint32_t it = atomicAdd(a.claim, 1u);
      uint32_t ok = *(volatile uint32_t *)&a.mine->status == 0;
      if ((it & 1) && it < npos) {
        const uint64_t q = (it - 1) / 2;
        if (q >= a.lag && q - a.lag < nB && ok && !(a.dbg & 1)) {
          const uint32_t st = qwait(a, a.rflags + (q - a.lag));
          if (st) {
            qfail(a, st);
            ok = 0;
          }
        }
      }
      s_item = it;
      s_ok = ok;
    }
    __syncthreads();
    const uint32_t it = s_item;
    const bool ok = s_ok != 0;
    __syncthreads();
    if (it >= npos) break;
    uint64_t i0, i1;
    if (!(it & 1)) {
      const uint64_t j = it / 2;
      if (j >= nA || !ok) continue;
      qblock_range(a.tlo, a.tn, j, i0, i1);
      uint8_t *dst = (a.dbg & 2) ? const_cast<uint8_t *>(a.rcodes) : a.tcodes;
      if (a.pcodes) {
        const volatile pcclb_qmeta *pm = a.pmeta;
        QuantPart16F<OP> f{a.tx, a.pcodes, pm->min_val, pm->scale, dst, qp};
        cta_loop16<2>(a.tlo, i0, i1, a.tvec != 0, f);
      } else {
        Quant16F f{a.tx, dst, nullptr, qp, 1.0f, false};
        cta_loop16<2>(a.tlo, i0, i1, a.tvec != 0, f);
      }
      __syncthreads();  // every thread's remote stores precede the token
      if (threadIdx.x == 0) {
        volatile pcclb_qmeta *m = a.tmeta;
        m->min_val = qp.mn;
        m->scale = qp.scale;
        // release (cumulative over the CTA's stores, ordered by the barrier)
        st_release_sys(a.tflags + j, a.token);
      }
    } else {
      const uint64_t q = (it - 1) / 2;
      if (q < a.lag || q - a.lag >= nB) continue;
      const uint64_t j = q - a.lag;
      qblock_range(a.rlo, a.rn, j, i0, i1);
      if (!ok) {  // no accumulate, but the restore needs this block's input
        CopyF f{a.rx, a.rbak};
        for (uint64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) f.one(i);
        continue;
      }
      const volatile pcclb_qmeta *m = a.rmeta;
      // plain arithmetic: a NaN here makes the next range non-finite -> abort + restore
      DequantRange4F<OP> f{a.rx, a.rcodes, m->min_val, m->scale, racc, a.rbak};
      cta_loop4<PCCLB_QR_U>(a.rlo, i0, i1, a.rvec != 0, f);
      racc = f.r;
    }
  }
  range_block_commit(racc, a.rrange);
}

// ---------------------------------------------------------------------------
// Fused gather (quantized): the owner's adoption and the W-1 dequantizing
// copies in one kernel, without the barrier between them.
//   A' (owner of chunk own = rank+1, collective.py:538-551): codes <- Q(own),
//      own = buf[own] (+) D(codes[W-2]) recomputed (see partial_of),
//      with the last step's range, own <- D(codes) / W in place, and the codes
//      pushed into every peer's gcodes[own] (remote 16-byte stores), one
//      ready token per 64 Ki-element block in each peer's gflags[own];
//   B' (collective.py:553-565): for every other chunk c, buf[c] <- D(gcodes[c])
//      (/ W) once its owner's token for the block is visible.
// Positions: round r holds W slots, slot 0 = A' block r, slot k >= 1 = block
// r - lag of chunk (own + k) mod W; the owner's A' block j (position W*j)
// precedes every B' item that waits for it (W*(j+lag)+k) on every rank, so
// claims in position order cannot wait cyclically (see ipc_qstep_kernel).
// ---------------------------------------------------------------------------
struct QFinalArgs {
  float *buf;
  uint64_t lo[kIpcMaxWorld + 1];  // chunk bounds: chunk c = [lo[c], lo[c+1])
  const pcclb_range *orange;      // range of the own chunk's final partial
  const uint8_t *ocodes;          // own codes[W-2] at element 0 of the own chunk: the final
  const pcclb_qmeta *ometa;       //   partial is buf[own] (+) D(ocodes) (never stored)
  uint64_t gcodes_off, codes_stride, gflags_off, flags_stride;  // workspace offsets (same on every rank)
  Signal *mine;
  Signal *peer[kIpcMaxWorld];     // peer workspaces (Signal at offset 0)
  const HostFlags *host;
  uint32_t *claim;
  uint64_t token, attempt, timeout_ns;
  uint32_t rank, world, own, fault, lag, vec;
  float avg;  // 1: no division
  uint32_t do_div;
  uint32_t dbg;  // experiments (PCCLB_QDEBUG bits): 1 B' never waits, 4 A' pushes to its own
                 // workspace, 8 B' items skipped, 16 A' posts no tokens, 32 A' items skipped
};

__device__ __forceinline__ uint8_t *gcodes_of(const QFinalArgs &a, Signal *ws, uint32_t c) {
  return reinterpret_cast<uint8_t *>(ws) + a.gcodes_off + c * a.codes_stride + a.lo[c] % 16;
}
__device__ __forceinline__ uint64_t *gflags_of(const QFinalArgs &a, Signal *ws, uint32_t c) {
  return reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(ws) + a.gflags_off + c * a.flags_stride);
}

// recompute the final partial, quantize + adopt in place + push the codes to
// every peer
template <bool X86, int OP>
struct QuantPushF {
  const QFinalArgs *a;
  float *x;
  QParams qp;
  uint64_t coff;  // chunk's code offset inside a peer's workspace
  const uint8_t *pcodes;
  float pmn, pscale;
  __device__ __forceinline__ float adopt_val(uint32_t q) {
    float d = dequant1x<X86>(q, qp.mn, qp.scale);
    return a->do_div ? div_world_x<X86>(d, a->avg) : d;
  }
  __device__ __forceinline__ void one(uint64_t i) {
    const uint32_t q = quant1_fast(partial_of<OP>(x[i], __ldcg(pcodes + i), pmn, pscale), qp.mn, qp.scale, qp.inv);
    x[i] = adopt_val(q);
    for (uint32_t p = 0; p < a->world; ++p)
      if (p != a->rank) (reinterpret_cast<uint8_t *>(a->peer[p]) + coff)[i] = (uint8_t)q;
  }
  struct In {
    Pack16<float> v[4];
    uint4 p;
  };
  __device__ __forceinline__ In vload(uint64_t i) {
    In r;
    r.p = __ldcg(reinterpret_cast<const uint4 *>(pcodes + i));
#pragma unroll
    for (int g = 0; g < 4; ++g) r.v[g] = ld16(x + i + 4 * g);
    return r;
  }
  __device__ __forceinline__ void vapply(uint64_t i, const In &in) {
    uint32_t w[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint32_t q[4];
      Pack16<float> d;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        q[k] = quant1_fast(partial_of<OP>(in.v[g].e[k], code_byte(in.p, 4 * g + k), pmn, pscale), qp.mn, qp.scale,
                           qp.inv);
        d.e[k] = adopt_val(q[k]);
      }
      w[g] = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
      st16(x + i + 4 * g, d);
    }
    const uint4 c = make_uint4(w[0], w[1], w[2], w[3]);
    for (uint32_t p = 0; p < a->world; ++p)
      if (p != a->rank)
        *reinterpret_cast<uint4 *>(reinterpret_cast<uint8_t *>((a->dbg & 4) ? a->mine : a->peer[p]) + coff + i) = c;
  }
};

template <int OP>
__global__ void __launch_bounds__(kQThreads, kQMinBlocks) ipc_qfinal_kernel(const __grid_constant__ QFinalArgs a) {
  __shared__ uint32_t s_item, s_ok;
  const uint32_t w = a.world, own = a.own;
  const uint64_t olo = a.lo[own], on = a.lo[own + 1] - olo;
  const uint64_t nO = qblocks(olo, on, kQF);
  uint64_t rounds = nO, maxg = 0;
  for (uint32_t k = 1; k < w; ++k) {
    const uint32_t c = (own + k) % w;
    const uint64_t nb = qblocks(a.lo[c], a.lo[c + 1] - a.lo[c], kQF);
    maxg = nb > maxg ? nb : maxg;
  }
  if (maxg && maxg + a.lag > rounds) rounds = maxg + a.lag;
  const uint64_t npos = rounds * w;
  if (threadIdx.x == 0 && *(volatile uint32_t *)&a.mine->status == 0) {
    if (blockIdx.x == 0 && a.fault) qfail(a, PCCLB_EIO);
    else if (a.host->abort >= a.attempt) qfail(a, PCCLB_EABORTED);
    else if (on && a.orange->nonfinite) qfail(a, PCCLB_ENONFINITE);
  }
  const QParams qp = qparams_from_range(*a.orange);
  for (;;) {
    if (threadIdx.x == 0) {
      const uint32_t it = atomicAdd(a.claim, 1u);
      uint32_t ok = *(volatile uint32_t *)&a.mine->status == 0;
      const uint32_t k = it % w;
      const uint64_t r = it / w;
      if (k && it < npos && ok && r >= a.lag && !(a.dbg & 1)) {
        const uint32_t c = (own + k) % w;
        if (r - a.lag < qblocks(a.lo[c], a.lo[c + 1] - a.lo[c], kQF)) {
          const uint32_t st = qwait(a, gflags_of(a, a.mine, c) + (r - a.lag));
          if (st) {
            qfail(a, st);
            ok = 0;
          }
        }
      }
      s_item = it;
      s_ok = ok;
    }
    __syncthreads();
    const uint32_t it = s_item;
    const bool ok = s_ok != 0;
    __syncthreads();
    if (it >= npos) break;
    if (!ok) continue;  // every chunk's input is already in the backup
    const uint32_t k = it % w;
    const uint64_t r = it / w;
    uint64_t i0, i1;
    if (k == 0) {
      if (r >= nO || (a.dbg & 32)) continue;
      qblock_range(olo, on, r, i0, i1, kQF);
      const uint64_t coff = a.gcodes_off + own * a.codes_stride + olo % 16;
      // finite scale and min: no NaN can arise (the x86 NaN rules only matter
      // for an overflowed range, scale = inf)
      const volatile pcclb_qmeta *pm = a.ometa;
      const float pmn = pm->min_val, psc = pm->scale;
      if (finite_f(qp.scale) && finite_f(qp.mn)) {
        QuantPushF<false, OP> f{&a, a.buf + olo, qp, coff, a.ocodes, pmn, psc};
        cta_loop16<PCCLB_QF_U>(olo, i0, i1, a.vec != 0, f);
      } else {
        QuantPushF<true, OP> f{&a, a.buf + olo, qp, coff, a.ocodes, pmn, psc};
        cta_loop16<PCCLB_QF_U>(olo, i0, i1, a.vec != 0, f);
      }
      __syncthreads();
      if (threadIdx.x < w && threadIdx.x != a.rank && !(a.dbg & 16)) {
        Signal *p = a.peer[threadIdx.x];
        volatile pcclb_qmeta *m = &p->gmeta[own];
        m->min_val = qp.mn;
        m->scale = qp.scale;
        st_release_sys(gflags_of(a, p, own) + r, a.token);
      }
    } else {
      if (r < a.lag || (a.dbg & 8)) continue;
      const uint32_t c = (own + k) % w;
      const uint64_t clo = a.lo[c], cn = a.lo[c + 1] - clo;
      if (r - a.lag >= qblocks(clo, cn, kQF)) continue;
      qblock_range(clo, cn, r - a.lag, i0, i1, kQF);
      const volatile pcclb_qmeta *m = &a.mine->gmeta[c];
      const float mn = m->min_val, sc = m->scale;
      if (finite_f(sc) && finite_f(mn)) {
        Dequant4T<false> f{a.buf + clo, gcodes_of(a, a.mine, c), mn, sc, a.avg, a.do_div != 0};
        cta_loop4<PCCLB_QB_U>(clo, i0, i1, a.vec != 0, f);
      } else {
        Dequant16F f{a.buf + clo, gcodes_of(a, a.mine, c), mn, sc, a.avg, a.do_div != 0};
        cta_loop16<PCCLB_QF_U>(clo, i0, i1, a.vec != 0, f);
      }
    }
  }
}

}  // namespace pcclb

using namespace pcclb;

struct PhaseTimer {
  static constexpr int kMax = 48;
  bool on = false;
  int n = 0;
  cudaEvent_t ev[kMax];
  void mark(cudaStream_t s) {
    if (on && n < kMax) cudaEventRecord(ev[n++], s);
  }
};

// A caller buffer registered on every rank (collective; SPMD order): peers'
// kernels read it in place, so the copy-in leaves the critical path.
struct RegSlot {
  bool used = false;
  const char *local = nullptr;
  uint64_t bytes = 0;
  const char *peer[kIpcMaxWorld] = {};
};
constexpr int kMaxReg = 64;

// one enqueued all-reduce (pcclb_ring_enqueue .. pcclb_ring_wait)
constexpr int kMaxOps = 64;
struct OpRec {
  bool pending = false;
  bool quantize = false;
  bool zero_copy = false;
  bool timed = false;
  void *buf = nullptr;
  uint64_t n = 0;
  int dtype = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
};

struct pcclb_ring {
  PhaseTimer timer;
  RegSlot reg[kMaxReg];
  std::map<std::string, char *> opened;  // peer allocations by IPC handle bytes
  bool last_zero_copy = false;           // last op read the caller buffer in place
  int device;
  uint32_t rank, world;
  uint64_t capacity;
  char *ws;                        // own workspace
  char *peer_ws[kIpcMaxWorld];     // mapped (own rank: ws)
  bool imported[kIpcMaxWorld];
  HostFlags *host;                 // host-mapped
  HostFlags *host_dev;             // device alias
  uint32_t *status_host;           // pinned status readback, one slot per op record (host-mapped)
  uint32_t *status_dev;            // device alias of status_host
  uint32_t *cur_status_dev = nullptr;  // the slot of the op being enqueued (small path writes it)
  OpRec ops[kMaxOps];
  cudaEvent_t op_events[kMaxOps];
  uint32_t next_ticket = 0;
  uint32_t slots = 2;  // engines that may run ops concurrently on this GPU (pcclb_ring_set_slots)
  uint64_t small_max = ~0ull;  // plain ops up to this many bytes: one-kernel path (~0: default)
  uint64_t last_n;
  int last_dtype;
  bool have_backup;
};

static Signal *sig_of(char *base) { return reinterpret_cast<Signal *>(base); }

namespace {

struct Layout {
  uint64_t in, res, codes, codes_stride, codesF, flags, flags_stride, gcodes, gflags, end;
  uint64_t codes_step(uint32_t s) const { return codes + s * codes_stride; }
  uint64_t flags_step(uint32_t s) const { return flags + s * flags_stride; }
};

// Chunk-local buffers keep the chunk's sub-16-byte alignment (floats) or
// sub-16-element alignment (codes), so 16-byte vector bodies line up with the
// caller's buffer at the same element offset.
uint64_t res_off(const Layout &L, uint64_t lo, size_t esz) { return L.res + (lo * esz) % 16; }
uint64_t codes_at(uint64_t off, uint64_t lo) { return off + lo % 16; }

Layout layout_for(uint64_t n, uint32_t w, size_t esz, bool quant) {
  Layout L{};
  const uint64_t nc = (n + w - 1) / w;
  auto up = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  L.in = kSignalBytes;
  uint64_t off = up(L.in + n * esz);
  if (!quant) {
    L.res = off;
    off = up(off + nc * esz + 16);
  } else {
    const uint32_t steps = w > 1 ? w - 1 : 1;
    L.codes = off;
    L.codes_stride = up(nc + 16);
    off += steps * L.codes_stride;
    L.codesF = off;
    off = up(off + nc + 16);
    L.flags = off;
    L.flags_stride = up((nc / kQB + 3) * 8);
    off += steps * L.flags_stride;
    // fused gather: every chunk's final codes, pushed by its owner
    L.gcodes = off;
    off += w * L.codes_stride;
    L.gflags = off;
    off += w * L.flags_stride;
  }
  L.end = off;
  return L;
}

int launch_barrier(pcclb_ring *r, uint64_t attempt, uint32_t index, int fault_at,
                   const pcclb_range *check, uint64_t timeout_ns, cudaStream_t s,
                   uint64_t desc = 0, bool check_desc = false) {
  BarrierArgs a{};
  a.desc = desc;
  a.check_desc = check_desc ? 1u : 0u;
  a.mine = sig_of(r->ws);
  for (uint32_t j = 0; j < r->world; ++j) a.peer[j] = sig_of(r->peer_ws[j]);
  a.host = r->host_dev;
  a.check_range = check;
  a.token = (attempt << 8) | index;
  a.attempt = attempt;
  a.timeout_ns = timeout_ns;
  a.rank = r->rank;
  a.world = r->world;
  a.fault = (fault_at >= 0 && (uint32_t)fault_at == index) ? 1u : 0u;
  ipc_barrier_kernel<<<1, 64, 0, s>>>(a);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

unsigned ipc_grid(uint64_t n_vec, int ctas_per_sm = 4) {
  return grid_for(n_vec, kIpcThreads, ctas_per_sm);
}

// Plain ops up to this size take the one-kernel small path (ipc_small_kernel).
// PCCLB_SMALL_MAX (bytes) overrides; 0 disables.
uint64_t small_max_bytes(const pcclb_ring *r) {
  if (r->small_max != ~0ull) return r->small_max;  // pcclb_ring_set_small_max
  static const long long env = [] {
    const char *e = getenv("PCCLB_SMALL_MAX");
    return e ? atoll(e) : -1ll;
  }();
  if (env >= 0) return (uint64_t)env;
  // the small path's NVLink ingress is (W-1)*N against the ring's 2(W-1)/W*N:
  // equal at W=2, W/2 times more beyond. Measured (bench.py --workload sweep,
  // small path vs multi-kernel schedule): W=2 1 MiB 32 vs 57 us, 16 MiB 59 vs
  // 85, 64 MiB 157 vs 167, 256 MiB 542 vs 476; W=4 4 MiB 68 vs 74, 16 MiB
  // 144 vs 110
  const uint32_t w = r->world ? r->world : 1;
  return w == 2 ? (64ull << 20) : (32ull << 20) / w;
}
// co-resident grid (the CTAs wait for each other): one CTA per 8 Ki elements, at most 128
unsigned small_grid(uint64_t n) {
  uint64_t g = (n + 8191) / 8192;
  if (g < 1) g = 1;
  if (g > 128) g = 128;
  return (unsigned)g;
}

// The attempt's last two kernels: completion vote (fault point `index`),
// then the device-side restore of a failed attempt.
int launch_vote_and_restore(pcclb_ring *r, void *buf, uint64_t nbytes, uint64_t attempt, uint32_t index,
                            int fault_at, uint64_t timeout_ns, cudaStream_t s) {
  VoteArgs a{};
  a.mine = sig_of(r->ws);
  for (uint32_t j = 0; j < r->world; ++j) a.peer[j] = sig_of(r->peer_ws[j]);
  a.host = r->host_dev;
  a.attempt = attempt;
  a.timeout_ns = timeout_ns;
  a.rank = r->rank;
  a.world = r->world;
  a.coord = 0;
  a.fault = (fault_at >= 0 && (uint32_t)fault_at == index) ? 1u : 0u;
  ipc_vote_kernel<<<1, 32, 0, s>>>(a);
  PCCLB_LAUNCH_CHECK();
  if (nbytes) {
    ipc_restore_kernel<<<ipc_grid(nbytes / 16 + 1, 2), kIpcThreads, 0, s>>>(
        a.mine, reinterpret_cast<const uint8_t *>(r->ws + kSignalBytes), static_cast<uint8_t *>(buf), nbytes);
    PCCLB_LAUNCH_CHECK();
  }
  return PCCLB_OK;
}

// dequant-accumulate shape (experiments): PCCLB_DQA=0 16 floats x 2 (default),
// 1: 4 floats x 4, 2: 16 floats x 4
int dqa_mode_value() {
  static int m = [] {
    const char *e = getenv("PCCLB_DQA");
    return e ? atoi(e) : 0;
  }();
  return m;
}

// plain gather engine: copy engines (default) or SM loads (PCCLB_GATHER=sm)
// (SM by default: with IPC-mapped peers the copy engines measured slower,
// 1.00 vs 0.82 ms for a 512 MiB chunk each way between two B200s)
bool gather_on_copy_engines() {
  static bool ce = [] {
    const char *e = getenv("PCCLB_GATHER");
    return e && e[0] == 'c';
  }();
  return ce;
}

// gather engine: PCCLB_GATHER = push (default: SM remote stores into the
// registered peer buffers, then a third barrier) | il (SM interleaved pull;
// always used for unregistered buffers) | jobs (SM, one CTA group per chunk)
// | ce (copy engines; PCCLB_CE_SPLIT pieces). Measured W=2/W=4 gather
// phases: push 0.78/1.19 ms, il 0.84/1.23, ce 1.00/2.2 (profiles/).
int gather_mode() {
  static int m = [] {
    const char *e = getenv("PCCLB_GATHER");
    if (!e) return 3;  // push when the buffers are registered, else interleaved pull
    if (e[0] == 'c') return 2;
    if (e[0] == 'p') return 3;
    if (e[0] == 'j') return 1;
    return 0;
  }();
  return m;
}
int ce_split() {
  static int k = [] {
    const char *e = getenv("PCCLB_CE_SPLIT");
    int v = e ? atoi(e) : 1;
    return v < 1 ? 1 : (v > 64 ? 64 : v);
  }();
  return k;
}

// plain SM gather: all chunks interleaved per thread (default) or one CTA
// group per chunk (PCCLB_GATHER=jobs)
bool gather_interleaved() {
  static bool il = [] {
    const char *e = getenv("PCCLB_GATHER");
    return !(e && e[0] == 'j');
  }();
  return il;
}

// 16-bit digest of the op parameters in the descriptor's top bits: barrier 0
// rejects an op whose (count, dtype, op, quantize) differ across ranks, the
// check the reference's master does on init votes (master.py:400-434)
uint64_t param_tag(uint64_t n, int dtype, int op, bool quant) {
  uint64_t h = n * 0x9E3779B97F4A7C15ull ^ ((uint64_t)dtype << 8) ^ ((uint64_t)op << 16) ^ (quant ? 1ull << 24 : 0);
  h ^= h >> 29;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 32;
  return (h & 0xffffull) << 48;
}

// registered slot containing [p, p + bytes), or -1
int find_reg(const pcclb_ring *r, const void *p, uint64_t bytes) {
  const char *c = static_cast<const char *>(p);
  for (int i = 0; i < kMaxReg; ++i) {
    const RegSlot &g = r->reg[i];
    if (g.used && c >= g.local && c + bytes <= g.local + g.bytes) return i;
  }
  return -1;
}

template <typename T>
int plain_allreduce(pcclb_ring *r, T *buf, uint64_t n, int op, uint64_t attempt, int fault_at,
                    uint64_t timeout_ns, cudaStream_t s) {
  const uint32_t w = r->world, rank = r->rank;
  const Layout L = layout_for(n, w, sizeof(T), false);
  uint64_t lo[2 * kIpcMaxWorld];
  pcclb_chunk_bounds(n, w, lo);  // lo[2c], lo[2c+1]
  const uint32_t own = (rank + 1) % w;  // collective.py:538
  const uint64_t own_lo = lo[2 * own], own_n = lo[2 * own + 1] - lo[2 * own];
  Signal *me = sig_of(r->ws);
  uint64_t desc = param_tag(n, sizeof(T) == 8 ? (int)PCCLB_F64 : sizeof(T) == 2 ? (int)PCCLB_BF16 : (int)PCCLB_F32, op, false);
  if (n * sizeof(T) <= small_max_bytes(r)) {
    // latency-bound size: the whole attempt in one kernel (ipc_small_kernel)
    r->last_zero_copy = false;
    SmallArgs<T> a{};
    a.buf = buf;
    a.in = reinterpret_cast<T *>(r->ws + L.in);
    for (uint32_t j = 0; j < w; ++j) a.pin[j] = reinterpret_cast<const T *>(r->peer_ws[j] + L.in);
    for (uint32_t c = 0; c < w; ++c) a.lo[c] = lo[2 * c];
    a.lo[w] = n;
    a.n = n;
    a.v.mine = me;
    for (uint32_t j = 0; j < w; ++j) a.v.peer[j] = sig_of(r->peer_ws[j]);
    a.v.host = r->host_dev;
    a.v.attempt = attempt;
    a.v.timeout_ns = timeout_ns;
    a.v.rank = rank;
    a.v.world = w;
    a.v.coord = 0;
    a.v.fault = (fault_at == 2) ? 1u : 0u;
    a.fault_arrive = (fault_at == 0 || fault_at == 1) ? 1u : 0u;
    a.desc = desc | (1ull << 38);  // bit 38: small path (ranks must agree)
    a.avg = (op == PCCLB_AVG) ? w : 0;
    a.status_out = r->cur_status_dev;
    const unsigned grid = small_grid(n);
    r->timer.mark(s);
    switch (op) {
      case PCCLB_MAX:
        ipc_small_kernel<T, PCCLB_MAX><<<grid, kIpcThreads, 0, s>>>(a);
        break;
      case PCCLB_MIN:
        ipc_small_kernel<T, PCCLB_MIN><<<grid, kIpcThreads, 0, s>>>(a);
        break;
      case PCCLB_PROD:
        ipc_small_kernel<T, PCCLB_PROD><<<grid, kIpcThreads, 0, s>>>(a);
        break;
      default:
        ipc_small_kernel<T, PCCLB_SUM><<<grid, kIpcThreads, 0, s>>>(a);
        break;
    }
    PCCLB_LAUNCH_CHECK();
    r->timer.mark(s);
    return PCCLB_OK;
  }
  const int slot = find_reg(r, buf, n * sizeof(T));
  const bool zero_copy = slot >= 0;
  r->last_zero_copy = zero_copy;
  const T *inputs[kIpcMaxWorld];  // where each ring position's input lives
  r->timer.mark(s);
  if (zero_copy) {
    // peers read the registered buffer in place. Nothing writes the buffer
    // before barrier 1, and no abort point follows it, so engine aborts need
    // no backup; the fold launch copies it into `in` on spare CTAs (local HBM
    // is idle while the fold waits on NVLink), keeping pcclb_ring_restore
    // (completion veto) available.
    const uint64_t off = reinterpret_cast<const char *>(buf) - r->reg[slot].local;
    desc |= ((uint64_t)(slot + 1) << 40) | off;
    for (uint32_t j = 0; j < w; ++j)
      inputs[j] = reinterpret_cast<const T *>(j == rank ? (const char *)buf : r->reg[slot].peer[j] + off);
    if (own_n == 0 || (reinterpret_cast<uintptr_t>(buf) & 15) != 0)  // rare: no fused backup
      PCCLB_CUDA(cudaMemcpyAsync(r->ws + L.in, buf, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
  } else {
    // copy-in: the caller's bytes become the backup and the peers' fold input
    PCCLB_CUDA(cudaMemcpyAsync(r->ws + L.in, buf, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
    for (uint32_t j = 0; j < w; ++j) inputs[j] = reinterpret_cast<const T *>(r->peer_ws[j] + L.in);
  }
  r->timer.mark(s);
  int rc = launch_barrier(r, attempt, 0, fault_at, nullptr, timeout_ns, s, desc, true);
  if (rc) return rc;
  r->timer.mark(s);
  if (own_n) {
    FoldArgs<T> f{};
    for (uint32_t k = 0; k < w; ++k) f.src[k] = inputs[(own + k) % w] + own_lo;
    f.dst0 = reinterpret_cast<T *>(r->ws + res_off(L, own_lo, sizeof(T)));
    f.dst1 = buf + own_lo;  // nobody else reads this rank's own chunk
    f.mine = me;
    f.n = own_n;
    f.w = w;
    f.avg = (op == PCCLB_AVG) ? w : 0;
    unsigned grid = grid_for(own_n / Pack16<T>::N + 1, kFoldThreads, 4);
    f.fold_ctas = grid;
    if (zero_copy && (reinterpret_cast<uintptr_t>(buf) & 15) == 0) {
      // backup: the caller's buffer -> in, on one CTA per SM next to three
      // fold CTAs (all co-resident, so the copy overlaps the NVLink-bound
      // fold). The fold writes the own chunk in place, so it saves that
      // chunk's input itself and the copy CTAs skip it.
      f.fold_ctas = std::min<unsigned>(grid, 3u * (unsigned)sm_count());
      f.bak_src = buf;
      f.bak_dst = r->ws + L.in;
      f.bak_bytes = n * sizeof(T);
      f.bak_skip_lo = own_lo * sizeof(T);
      f.bak_skip_hi = (own_lo + own_n) * sizeof(T);
      f.bak_own = reinterpret_cast<T *>(r->ws + L.in) + own_lo;
      grid = f.fold_ctas + (unsigned)sm_count();
    }
    // every source and destination must share the sub-16-byte offset
    bool vec = f.dst1 == nullptr || peel16<T>(f.dst1) == peel16<T>(f.dst0);
    for (uint32_t k = 0; k < w; ++k) vec = vec && peel16<T>(f.src[k]) == peel16<T>(f.dst0);
#define PCCLB_IPC_FOLD(OPC)                                                             \
  if (vec)                                                                              \
    ipc_fold_kernel<T, OPC, 16 / sizeof(T)><<<grid, kFoldThreads, 0, s>>>(f);           \
  else                                                                                  \
    ipc_fold_kernel<T, OPC, 1><<<grid, kFoldThreads, 0, s>>>(f);
    switch (op) {
      case PCCLB_MAX:
        PCCLB_IPC_FOLD(PCCLB_MAX);
        break;
      case PCCLB_MIN:
        PCCLB_IPC_FOLD(PCCLB_MIN);
        break;
      case PCCLB_PROD:
        PCCLB_IPC_FOLD(PCCLB_PROD);
        break;
      default:
        PCCLB_IPC_FOLD(PCCLB_SUM);
        break;
    }
#undef PCCLB_IPC_FOLD
    PCCLB_LAUNCH_CHECK();
  }
  r->timer.mark(s);
  rc = launch_barrier(r, attempt, 1, fault_at, nullptr, timeout_ns, s);
  if (rc) return rc;
  r->timer.mark(s);
  GatherArgs g{};
  g.mine = me;
  uint32_t jobs = 0;
  uint64_t maxn = 0;
  for (uint32_t c = 0; c < w; ++c) {
    if (c == own) continue;  // written by the fold
    const uint64_t cn = lo[2 * c + 1] - lo[2 * c];
    if (!cn) continue;
    const uint32_t owner = (c + w - 1) % w;
    g.src[jobs] = r->peer_ws[owner] + res_off(L, lo[2 * c], sizeof(T));
    g.dst[jobs] = buf + lo[2 * c];
    g.bak[jobs] = nullptr;
    g.n[jobs] = cn;
    maxn = cn > maxn ? cn : maxn;
    ++jobs;
  }
  if (zero_copy && gather_mode() == 3) {
    if (own_n) {
      PushArgs<T> pa{};
      pa.src = reinterpret_cast<const T *>(r->ws + res_off(L, own_lo, sizeof(T)));
      for (uint32_t j = 0; j < w; ++j)
        if (j != rank) pa.dst[pa.ndst++] = const_cast<T *>(inputs[j]) + own_lo;
      pa.n = own_n;
      pa.mine = me;
      pa.vec = 1;
      for (uint32_t j = 0; j < pa.ndst; ++j) pa.vec &= peel16<T>(pa.dst[j]) == peel16<T>(pa.src) ? 1u : 0u;
      ipc_push_kernel<T><<<ipc_grid(own_n / Pack16<T>::N + 1, 2), kIpcThreads, 0, s>>>(pa);
      PCCLB_LAUNCH_CHECK();
    }
    // the vote that follows also tells every rank that all pushes into it landed
  } else if (jobs && (gather_on_copy_engines() || gather_mode() == 2)) {
    // verbatim chunk copies on the copy engines (759 GB/s per direction for
    // plain peer allocations in tools/micro/p2p_micro.cu). CE copies cannot
    // test the op status, so an aborted op is always restored from `in`.
    const int k = ce_split();
    for (int piece = 0; piece < k; ++piece)
      for (uint32_t j = 0; j < jobs; ++j) {
        const uint64_t a0 = g.n[j] * piece / k, a1 = g.n[j] * (piece + 1) / k;
        if (a1 > a0)
          PCCLB_CUDA(cudaMemcpyAsync(static_cast<T *>(g.dst[j]) + a0, static_cast<const T *>(g.src[j]) + a0,
                                     (a1 - a0) * sizeof(T), cudaMemcpyDeviceToDevice, s));
      }
  } else if (jobs) {
    bool same = true;
    const uint64_t h0 = peel16<T>(g.dst[0]);
    for (uint32_t j = 0; j < jobs; ++j)
      same = same && peel16<T>(g.dst[j]) == h0 && peel16<T>(g.src[j]) == h0;
    if (same && gather_interleaved()) {
      int occ = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ipc_gather_interleaved_kernel<T>, kIpcThreads, 0);
      ipc_gather_interleaved_kernel<T><<<ipc_grid(maxn / Pack16<T>::N + 1, occ < 1 ? 1 : occ), kIpcThreads, 0, s>>>(
          g, jobs, h0);
    } else {
      unsigned per = ipc_grid(maxn / Pack16<T>::N + 1, 4);
      per = (per + jobs - 1) / jobs;
      if (per < 1) per = 1;
      ipc_gather_plain_kernel<T><<<dim3(per, jobs), kIpcThreads, 0, s>>>(g);
    }
    PCCLB_LAUNCH_CHECK();
  }
  r->timer.mark(s);
  rc = launch_vote_and_restore(r, buf, n * sizeof(T), attempt, 2, fault_at, timeout_ns, s);
  if (rc) return rc;
  r->timer.mark(s);
  return PCCLB_OK;
}

// fused quantized steps (default) or the barrier-per-step schedule
// (PCCLB_QSTEP=0, and when too many engines may run at once for the fused
// kernel's spinning CTAs to leave room for the others)
bool qstep_enabled() {
  static bool on = [] {
    const char *e = getenv("PCCLB_QSTEP");
    return !(e && e[0] == '0');
  }();
  return on;
}

int quant_allreduce(pcclb_ring *r, float *buf, uint64_t n, int op, uint64_t attempt, int fault_at,
                    uint64_t timeout_ns, cudaStream_t s) {
  const uint32_t w = r->world, rank = r->rank;
  const Layout L = layout_for(n, w, 4, true);
  uint64_t lo[2 * kIpcMaxWorld];
  pcclb_chunk_bounds(n, w, lo);
  Signal *me = sig_of(r->ws);
  const uint32_t pred = (rank + w - 1) % w, succ = (rank + 1) % w;
  Signal *pred_sig = sig_of(r->peer_ws[pred]);
  r->timer.mark(s);
  // no copy-in: every chunk's input is saved into `in` by the first kernel
  // that reads it (range for chunk `rank`, the step's dequant-accumulate for
  // each rx chunk), which also runs when the op already failed
  float *bak = reinterpret_cast<float *>(r->ws + L.in);
  // range slots and step counters reset; ready flags cleared (peers write
  // them only after barrier 0, which this rank reaches after the memset)
  PCCLB_CUDA(cudaMemsetAsync(me->range, 0, sizeof(pcclb_range) * (w + 1), s));
  static const int occ_q = [] {
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ipc_qstep_kernel<PCCLB_SUM>, kQThreads, 0);
    return o < 1 ? 1 : o;
  }();
  static const int slots_env = [] {
    const char *e = getenv("PCCLB_QSLOTS");
    return e ? atoi(e) : 0;
  }();
  // CTAs per SM for this engine's fused steps: the other slots' engines
  // (spinning the same way) must still find a free CTA slot on every SM,
  // (slots - 1) * per_sm <= occ - 1, so every engine's kernel makes progress
  const int slots = slots_env > 0 ? slots_env : (int)(r->slots ? r->slots : 1);
  const int per_sm = slots <= 1 ? occ_q : (occ_q - 1) / (slots - 1) < occ_q ? (occ_q - 1) / (slots - 1) : occ_q;
  const bool fused = qstep_enabled() && per_sm >= 1;
  static const uint32_t dbg = [] {
    const char *e = getenv("PCCLB_QDEBUG");
    return e ? (uint32_t)atoi(e) : 0u;
  }();
  if (fused) {
    PCCLB_CUDA(cudaMemsetAsync(me->claim, 0, sizeof(uint32_t) * (w + 1), s));
    PCCLB_CUDA(cudaMemsetAsync(r->ws + L.flags, 0, L.flags_stride * (w - 1), s));
    PCCLB_CUDA(cudaMemsetAsync(r->ws + L.gflags, 0, L.flags_stride * w, s));
  }
  auto span = [&](uint32_t c, uint64_t &a, uint64_t &len) {
    a = lo[2 * c];
    len = lo[2 * c + 1] - lo[2 * c];
  };
  uint64_t a0, n0;
  span(rank % w, a0, n0);  // step-0 tx chunk = rank (collective.py:522)
  if (n0) {
    ipc_range_kernel<<<ipc_grid(n0 / 4 + 1), kIpcThreads, 0, s>>>(buf + a0, n0, &me->range[0], bak + a0, me);
    PCCLB_LAUNCH_CHECK();
  }
  r->timer.mark(s);
  int rc;
  if (fused) {
    // descriptor bit 39: this rank runs the fused schedule (a rank on the
    // barrier-per-step schedule publishes it clear -> EINVAL on both sides)
    rc = launch_barrier(r, attempt, 0, fault_at, &me->range[0], timeout_ns, s,
                        param_tag(n, PCCLB_F32, op, true) | (1ull << 39), true);
    if (rc) return rc;
    r->timer.mark(s);
    QStepArgs q{};
    q.mine = me;
    for (uint32_t j = 0; j < w; ++j) q.peer[j] = sig_of(r->peer_ws[j]);
    q.host = r->host_dev;
    q.token = attempt;
    q.attempt = attempt;
    q.timeout_ns = timeout_ns;
    q.rank = rank;
    q.world = w;
    const unsigned grid = (unsigned)(sm_count() * per_sm);
    static const double lag_mul = [] {
      const char *e = getenv("PCCLB_QLAG");
      return e ? atof(e) : 2.0;
    }();
    q.lag = (uint32_t)(grid * lag_mul);
    q.dbg = dbg;
    const bool buf_vec = (reinterpret_cast<uintptr_t>(buf) & 63) == 0;
    for (uint32_t step = 0; step + 1 < w; ++step) {
      const uint32_t tx = (rank + w - step % w) % w;     // (rank - step) mod w
      const uint32_t rx = (rank + 2 * w - step - 1) % w;  // (rank - step - 1) mod w
      span(tx, q.tlo, q.tn);
      span(rx, q.rlo, q.rn);
      q.tx = buf + q.tlo;
      q.tcodes = reinterpret_cast<uint8_t *>(r->peer_ws[succ] + codes_at(L.codes_step(step), q.tlo));
      q.tmeta = &sig_of(r->peer_ws[succ])->qmeta[step];
      q.tflags = reinterpret_cast<uint64_t *>(r->peer_ws[succ] + L.flags_step(step));
      q.trange = &me->range[step];
      q.pcodes = step ? reinterpret_cast<const uint8_t *>(r->ws + codes_at(L.codes_step(step - 1), q.tlo)) : nullptr;
      q.pmeta = step ? &me->qmeta[step - 1] : nullptr;
      q.rx = buf + q.rlo;
      q.rbak = bak + q.rlo;
      q.rcodes = reinterpret_cast<const uint8_t *>(r->ws + codes_at(L.codes_step(step), q.rlo));
      q.rmeta = &me->qmeta[step];
      q.rflags = reinterpret_cast<const uint64_t *>(r->ws + L.flags_step(step));
      q.rrange = &me->range[step + 1];
      q.claim = &me->claim[step];
      q.fault = (step > 0 && fault_at >= 0 && (uint32_t)fault_at == step) ? 1u : 0u;
      q.tvec = q.rvec = buf_vec ? 1u : 0u;
      switch (op) {
        case PCCLB_MAX:
          ipc_qstep_kernel<PCCLB_MAX><<<grid, kQThreads, 0, s>>>(q);
          break;
        case PCCLB_MIN:
          ipc_qstep_kernel<PCCLB_MIN><<<grid, kQThreads, 0, s>>>(q);
          break;
        case PCCLB_PROD:
          ipc_qstep_kernel<PCCLB_PROD><<<grid, kQThreads, 0, s>>>(q);
          break;
        default:
          ipc_qstep_kernel<PCCLB_SUM><<<grid, kQThreads, 0, s>>>(q);
          break;
      }
      PCCLB_LAUNCH_CHECK();
      r->timer.mark(s);
    }
  } else {
  for (uint32_t step = 0; step + 1 < w; ++step) {
    const uint32_t tx = (rank + w - step % w) % w;         // (rank - step) mod w
    const uint32_t rx = (rank + 2 * w - step - 1) % w;      // (rank - step - 1) mod w
    uint64_t ta, tn, ra, rn;
    span(tx, ta, tn);
    span(rx, ra, rn);
    const uint64_t codes_off = L.codes_step(step);
    // quantize what we send (its range was produced by the previous step)
    ipc_quantize_kernel<<<ipc_grid(tn / 4 + 1), kIpcThreads, 0, s>>>(
        buf + ta, tn, &me->range[step], reinterpret_cast<uint8_t *>(r->ws + codes_at(codes_off, ta)),
        &me->meta[step & 1], nullptr, 1, me);
    PCCLB_LAUNCH_CHECK();
    r->timer.mark(s);
    rc = launch_barrier(r, attempt, step, fault_at, &me->range[step], timeout_ns, s,
                        param_tag(n, PCCLB_F32, op, true), step == 0);
    if (rc) return rc;
    r->timer.mark(s);
    if (rn) {
      const uint8_t *codes = reinterpret_cast<const uint8_t *>(r->peer_ws[pred] + codes_at(codes_off, ra));
      const pcclb_qmeta *meta = &pred_sig->meta[step & 1];
      const unsigned grid = ipc_grid(rn / 4 + 1);
      switch (op) {
        case PCCLB_MAX:
          ipc_dequant_acc_kernel<PCCLB_MAX><<<grid, kIpcThreads, 0, s>>>(buf + ra, codes, rn, meta, &me->range[step + 1], bak + ra, me, dqa_mode_value());
          break;
        case PCCLB_MIN:
          ipc_dequant_acc_kernel<PCCLB_MIN><<<grid, kIpcThreads, 0, s>>>(buf + ra, codes, rn, meta, &me->range[step + 1], bak + ra, me, dqa_mode_value());
          break;
        case PCCLB_PROD:
          ipc_dequant_acc_kernel<PCCLB_PROD><<<grid, kIpcThreads, 0, s>>>(buf + ra, codes, rn, meta, &me->range[step + 1], bak + ra, me, dqa_mode_value());
          break;
        default:
          ipc_dequant_acc_kernel<PCCLB_SUM><<<grid, kIpcThreads, 0, s>>>(buf + ra, codes, rn, meta, &me->range[step + 1], bak + ra, me, dqa_mode_value());
          break;
      }
      PCCLB_LAUNCH_CHECK();
    }
  }
  }
  r->timer.mark(s);
  const uint32_t own = (rank + 1) % w;
  if (fused) {
    QFinalArgs g{};
    g.buf = buf;
    for (uint32_t c = 0; c < w; ++c) g.lo[c] = lo[2 * c];
    g.lo[w] = n;
    g.orange = &me->range[w - 1];
    g.ocodes = reinterpret_cast<const uint8_t *>(r->ws + codes_at(L.codes_step(w - 2), lo[2 * own]));
    g.ometa = &me->qmeta[w - 2];
    g.gcodes_off = L.gcodes;
    g.codes_stride = L.codes_stride;
    g.gflags_off = L.gflags;
    g.flags_stride = L.flags_stride;
    g.mine = me;
    for (uint32_t j = 0; j < w; ++j) g.peer[j] = sig_of(r->peer_ws[j]);
    g.host = r->host_dev;
    g.claim = &me->claim[w - 1];
    g.token = attempt;
    g.attempt = attempt;
    g.timeout_ns = timeout_ns;
    g.rank = rank;
    g.world = w;
    g.own = own;
    g.fault = (fault_at >= 0 && (uint32_t)fault_at == w - 1) ? 1u : 0u;
    const unsigned grid = (unsigned)(sm_count() * per_sm);
    static const double glag = [] {
      const char *e = getenv("PCCLB_GLAG");
      return e ? atof(e) : 4.0;  // measured (64 Ki blocks): 2 -> 2.26 ms, 8 -> 1.98 ms (W=2, 1.2 B elements)
    }();
    g.lag = (uint32_t)((glag * grid + w - 1) / w);  // rounds of w positions
    g.dbg = dbg;
    g.vec = (reinterpret_cast<uintptr_t>(buf) & 63) == 0 ? 1u : 0u;
    g.avg = (op == PCCLB_AVG) ? (float)w : 1.0f;
    g.do_div = op == PCCLB_AVG ? 1u : 0u;
    switch (op) {
      case PCCLB_MAX:
        ipc_qfinal_kernel<PCCLB_MAX><<<grid, kQThreads, 0, s>>>(g);
        break;
      case PCCLB_MIN:
        ipc_qfinal_kernel<PCCLB_MIN><<<grid, kQThreads, 0, s>>>(g);
        break;
      case PCCLB_PROD:
        ipc_qfinal_kernel<PCCLB_PROD><<<grid, kQThreads, 0, s>>>(g);
        break;
      default:
        ipc_qfinal_kernel<PCCLB_SUM><<<grid, kQThreads, 0, s>>>(g);
        break;
    }
    PCCLB_LAUNCH_CHECK();
    r->timer.mark(s);
    rc = launch_vote_and_restore(r, buf, n * sizeof(float), attempt, w, fault_at, timeout_ns, s);
    if (rc) return rc;
    r->timer.mark(s);
    return PCCLB_OK;
  }
  // gather prologue: owner adopts D(Q(own)) (collective.py:538-551), fused with AVG
  uint64_t oa, on;
  span(own, oa, on);
  const uint32_t avg = (op == PCCLB_AVG) ? w : 1;
  ipc_quantize_kernel<<<ipc_grid(on / 4 + 1), kIpcThreads, 0, s>>>(
      buf + oa, on, &me->range[w - 1], reinterpret_cast<uint8_t *>(r->ws + codes_at(L.codesF, oa)),
      &me->meta_final, buf + oa, avg, me);
  PCCLB_LAUNCH_CHECK();
  rc = launch_barrier(r, attempt, w - 1, fault_at, &me->range[w - 1], timeout_ns, s);
  if (rc) return rc;
  r->timer.mark(s);
  GatherArgs g{};
  g.mine = me;
  g.avg = avg;
  uint32_t jobs = 0;
  uint64_t maxn = 0;
  for (uint32_t c = 0; c < w; ++c) {
    if (c == own) continue;
    uint64_t ca, cn;
    span(c, ca, cn);
    if (!cn) continue;
    const uint32_t owner = (c + w - 1) % w;
    g.src[jobs] = r->peer_ws[owner] + codes_at(L.codesF, ca);
    g.meta[jobs] = &sig_of(r->peer_ws[owner])->meta_final;
    g.dst[jobs] = buf + ca;
    g.n[jobs] = cn;
    maxn = cn > maxn ? cn : maxn;
    ++jobs;
  }
  if (jobs) {
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ipc_gather_quant_kernel, kIpcThreads, 0);
    int vec = 1;  // 16-byte code loads need codes 16-byte aligned where dst is 64-byte aligned
    for (uint32_t j = 0; j < jobs; ++j) {
      const uintptr_t d = reinterpret_cast<uintptr_t>(g.dst[j]);
      const uint64_t head = ((64 - (d & 63)) & 63) / 4;
      vec &= (d & 3) == 0 && ((reinterpret_cast<uintptr_t>(g.src[j]) + head) & 15) == 0;
    }
    ipc_gather_quant_kernel<<<ipc_grid(maxn / 4 + 1, occ < 1 ? 1 : occ), kIpcThreads, 0, s>>>(g, jobs, vec);
    PCCLB_LAUNCH_CHECK();
  }
  r->timer.mark(s);
  rc = launch_vote_and_restore(r, buf, n * sizeof(float), attempt, w, fault_at, timeout_ns, s);
  if (rc) return rc;
  r->timer.mark(s);
  return PCCLB_OK;
}

}  // namespace

extern "C" {

int pcclb_ring_create(int device, uint32_t rank, uint32_t world, uint64_t capacity_bytes,
                      pcclb_ring **out) {
  if (!out || world < 1 || world > (uint32_t)kIpcMaxWorld || rank >= world) return PCCLB_EINVAL;
  *out = nullptr;
  PCCLB_CUDA(cudaSetDevice(device));
  pcclb_ring *r = new (std::nothrow) pcclb_ring();
  // value-initialised: pointers null, flags false
  if (!r) return PCCLB_ENOMEM;
  r->device = device;
  r->rank = rank;
  r->world = world;
  r->capacity = capacity_bytes < kSignalBytes + 4096 ? kSignalBytes + 4096 : capacity_bytes;
  cudaError_t e = cudaMalloc(&r->ws, r->capacity);
  if (e != cudaSuccess) {
    delete r;
    return cuda_status(e);
  }
  e = cudaMemset(r->ws, 0, kSignalBytes);
  if (e == cudaSuccess) e = cudaHostAlloc(&r->host, sizeof(HostFlags), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&r->host_dev, r->host, 0);
  if (e == cudaSuccess) e = cudaHostAlloc(&r->status_host, sizeof(uint32_t) * kMaxOps, cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&r->status_dev, r->status_host, 0);
  for (int i = 0; i < kMaxOps && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(&r->op_events[i], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    pcclb_ring_destroy(r);
    return cuda_status(e);
  }
  std::memset((void *)r->host, 0, sizeof(HostFlags));
  const char *prof = getenv("PCCLB_RING_PROFILE");
  if (prof && prof[0] == '1') {
    r->timer.on = true;
    for (int i = 0; i < PhaseTimer::kMax; ++i) cudaEventCreate(&r->timer.ev[i]);
  }
  r->peer_ws[rank] = r->ws;
  r->imported[rank] = true;
  *out = r;
  return PCCLB_OK;
}

int pcclb_ring_export(pcclb_ring *r, void *handle64_out) {
  if (!r || !handle64_out) return PCCLB_EINVAL;
  PCCLB_CUDA(cudaSetDevice(r->device));
  cudaIpcMemHandle_t h;
  PCCLB_CUDA(cudaIpcGetMemHandle(&h, r->ws));
  static_assert(sizeof(h) == 64, "ipc handle size");
  std::memcpy(handle64_out, &h, 64);
  return PCCLB_OK;
}

int pcclb_ring_import(pcclb_ring *r, uint32_t peer, const void *handle64) {
  if (!r || !handle64 || peer >= r->world) return PCCLB_EINVAL;
  if (peer == r->rank) return PCCLB_OK;
  PCCLB_CUDA(cudaSetDevice(r->device));
  if (r->imported[peer]) {
    PCCLB_CUDA(cudaIpcCloseMemHandle(r->peer_ws[peer]));
    r->imported[peer] = false;
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  void *p = nullptr;
  PCCLB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  r->peer_ws[peer] = static_cast<char *>(p);
  r->imported[peer] = true;
  return PCCLB_OK;
}

uint64_t pcclb_ring_workspace_bytes(uint64_t n, uint32_t world, int dtype, int quantize) {
  if (world < 1 || world > (uint32_t)kIpcMaxWorld || !valid_dtype(dtype)) return 0;
  return layout_for(n, world, dtype_size(dtype), quantize != 0).end;
}

int pcclb_ring_set_small_max(pcclb_ring *r, uint64_t bytes) {
  if (!r) return PCCLB_EINVAL;
  r->small_max = bytes;
  return PCCLB_OK;
}

int pcclb_ring_set_slots(pcclb_ring *r, uint32_t slots) {
  if (!r || slots < 1) return PCCLB_EINVAL;
  r->slots = slots;
  return PCCLB_OK;
}

volatile uint64_t *pcclb_ring_abort_word(pcclb_ring *r) { return r ? &r->host->abort : nullptr; }

uint64_t pcclb_ring_capacity(pcclb_ring *r, int dtype, int quantize) {
  if (!r || !valid_dtype(dtype)) return 0;
  // largest n whose layout fits (layout is monotone in n)
  const size_t esz = dtype_size(dtype);
  uint64_t lo = 0, hi = r->capacity / esz + 1;
  while (lo + 1 < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (layout_for(mid, r->world, esz, quantize != 0).end <= r->capacity) lo = mid;
    else hi = mid;
  }
  return lo;
}

int pcclb_ring_enqueue(pcclb_ring *r, void *d_buf, uint64_t n, int dtype, int op, int quantize,
                       uint64_t attempt, int fault_at, double timeout_s, void *stream,
                       uint32_t *ticket_out) {
  if (!r || !ticket_out || !valid_dtype(dtype) || !valid_op(op) || (n && !d_buf)) return PCCLB_EINVAL;
  if (quantize && dtype != PCCLB_F32) return PCCLB_EINVAL;  // client.py:818-819
  if (attempt == 0 || attempt >= (1ull << 55)) return PCCLB_EINVAL;
  for (uint32_t j = 0; j < r->world; ++j)
    if (!r->imported[j]) return PCCLB_EINVAL;
  const size_t esz = dtype_size(dtype);
  if (layout_for(n, r->world, esz, quantize != 0).end > r->capacity) return PCCLB_ENOMEM;
  const uint32_t t = r->next_ticket % kMaxOps;
  OpRec &o = r->ops[t];
  if (o.pending) return PCCLB_EINVAL;  // too many outstanding ops
  PCCLB_CUDA(cudaSetDevice(r->device));
  cudaStream_t s = as_stream(stream);
  const uint32_t w = r->world;
  o = OpRec{};
  o.done = r->op_events[t];
  o.buf = d_buf;
  o.n = n;
  o.dtype = dtype;
  o.quantize = quantize != 0;
  o.stream = s;
  o.timed = r->timer.on;
  r->status_host[t] = 0;
  if (w == 1) {  // client.py:896-900
    int rc = pcclb_finalize(d_buf, n, dtype, op, 1, stream);
    if (rc) return rc;
  } else {
    Signal *me = sig_of(r->ws);
    r->timer.n = 0;
    // the one-kernel small path resets the status word and hands its outcome to
    // the host itself (status_dev); the other schedules use a memset and a copy
    const bool small = !quantize && n * esz <= small_max_bytes(r);
    r->cur_status_dev = small ? &r->status_dev[t] : nullptr;
    if (!small) PCCLB_CUDA(cudaMemsetAsync(&me->status, 0, sizeof(uint32_t), s));
    const uint64_t timeout_ns = (uint64_t)((timeout_s > 0 ? timeout_s : 60.0) * 1e9);
    int rc;
    if (quantize)
      rc = quant_allreduce(r, static_cast<float *>(d_buf), n, op, attempt, fault_at, timeout_ns, s);
    else if (dtype == PCCLB_F32)
      rc = plain_allreduce<float>(r, static_cast<float *>(d_buf), n, op, attempt, fault_at, timeout_ns, s);
    else if (dtype == PCCLB_BF16)
      rc = plain_allreduce<Bf16>(r, static_cast<Bf16 *>(d_buf), n, op, attempt, fault_at, timeout_ns, s);
    else
      rc = plain_allreduce<double>(r, static_cast<double *>(d_buf), n, op, attempt, fault_at, timeout_ns, s);
    if (rc) return rc;
    o.zero_copy = !quantize && r->last_zero_copy;
    if (!small)
      PCCLB_CUDA(cudaMemcpyAsync(&r->status_host[t], &me->status, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  }
  PCCLB_CUDA(cudaEventRecord(o.done, s));
  o.pending = true;
  r->next_ticket++;
  *ticket_out = t;
  return PCCLB_OK;
}

int pcclb_ring_wait(pcclb_ring *r, uint32_t ticket, pcclb_stats *out_stats) {
  if (!r || ticket >= (uint32_t)kMaxOps || !r->ops[ticket].pending) return PCCLB_EINVAL;
  OpRec &o = r->ops[ticket];
  o.pending = false;
  PCCLB_CUDA(cudaSetDevice(r->device));
  PCCLB_CUDA(cudaEventSynchronize(o.done));
  const uint32_t w = r->world;
  const size_t esz = dtype_size(o.dtype);
  if (out_stats) {
    // algorithmic payload per peer: 2(W-1)/W * N * elem (test_ring_engine.py:99-108)
    uint64_t lo[2 * kIpcMaxWorld];
    pcclb_chunk_bounds(o.n, w, lo);
    uint64_t tx = 0;
    const uint64_t ebytes = o.quantize ? 1 : esz;
    for (uint32_t step = 0; w > 1 && step + 1 < w; ++step) {
      uint32_t c = (r->rank + w - step % w) % w;
      tx += (lo[2 * c + 1] - lo[2 * c]) * ebytes;
    }
    uint32_t cur = (r->rank + 1) % w;
    for (uint32_t step = 0; w > 1 && step + 1 < w; ++step) {
      tx += (lo[2 * cur + 1] - lo[2 * cur]) * ebytes;
      cur = (cur + w - 1) % w;
    }
    out_stats->tx_payload_bytes = tx;
    out_stats->rx_payload_bytes = tx;
    out_stats->n_phases = 0;
    if (o.timed)
      for (int i = 1; i < r->timer.n && i <= 47; ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, r->timer.ev[i - 1], r->timer.ev[i]);
        out_stats->phase_ms[out_stats->n_phases++] = ms;
      }
  }
  const uint32_t st = r->status_host[ticket];
  r->last_n = o.n;
  r->last_dtype = o.dtype;
  // `in` holds the op's input in both modes (copy-in, or the backup CTAs of
  // a zero-copy fold, which run even when the op failed)
  r->have_backup = w > 1;
  // a failed attempt was restored on the device, in stream order (ipc_restore_kernel)
  return (int)st;
}

int pcclb_ring_allreduce(pcclb_ring *r, void *d_buf, uint64_t n, int dtype, int op, int quantize,
                         uint64_t attempt, int fault_at, double timeout_s, pcclb_stats *out_stats,
                         void *stream) {
  uint32_t t = 0;
  int rc = pcclb_ring_enqueue(r, d_buf, n, dtype, op, quantize, attempt, fault_at, timeout_s, stream, &t);
  if (rc) return rc;
  return pcclb_ring_wait(r, t, out_stats);
}

int pcclb_ring_restore(pcclb_ring *r, void *d_buf, uint64_t n, int dtype, void *stream) {
  if (!r || !d_buf || !r->have_backup || n != r->last_n || dtype != r->last_dtype) return PCCLB_EINVAL;
  PCCLB_CUDA(cudaSetDevice(r->device));
  cudaStream_t s = as_stream(stream);
  PCCLB_CUDA(cudaMemcpyAsync(d_buf, r->ws + kSignalBytes, n * dtype_size(dtype), cudaMemcpyDeviceToDevice, s));
  PCCLB_CUDA(cudaStreamSynchronize(s));
  return PCCLB_OK;
}

int pcclb_ipc_handle(const void *d_ptr, void *handle64_out, uint64_t *offset_out) {
  if (!d_ptr || !handle64_out || !offset_out) return PCCLB_EINVAL;
  static PFN_cuMemGetAddressRange_v3020 range_fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  }();
  if (!range_fn) return PCCLB_ECUDA;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, (CUdeviceptr)d_ptr) != CUDA_SUCCESS) return PCCLB_EINVAL;
  cudaIpcMemHandle_t h;
  PCCLB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
  std::memcpy(handle64_out, &h, 64);
  *offset_out = (uint64_t)((CUdeviceptr)d_ptr - base);
  return PCCLB_OK;
}

int pcclb_ring_register(pcclb_ring *r, uint32_t slot, const void *local_ptr, uint64_t nbytes,
                        const void *handles, const uint64_t *offsets) {
  if (!r || slot >= (uint32_t)kMaxReg || !local_ptr || !handles || !offsets) return PCCLB_EINVAL;
  PCCLB_CUDA(cudaSetDevice(r->device));
  RegSlot g;
  g.local = static_cast<const char *>(local_ptr);
  g.bytes = nbytes;
  for (uint32_t j = 0; j < r->world; ++j) {
    if (j == r->rank) {
      g.peer[j] = g.local;
      continue;
    }
    std::string key(static_cast<const char *>(handles) + 64 * (size_t)j, 64);
    auto it = r->opened.find(key);
    char *base = nullptr;
    if (it != r->opened.end()) {
      base = it->second;
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, key.data(), 64);
      void *p = nullptr;
      PCCLB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      base = static_cast<char *>(p);
      r->opened.emplace(key, base);
    }
    g.peer[j] = base + offsets[j];
  }
  g.used = true;
  r->reg[slot] = g;
  return PCCLB_OK;
}

int pcclb_ring_deregister(pcclb_ring *r, uint32_t slot) {
  if (!r || slot >= (uint32_t)kMaxReg) return PCCLB_EINVAL;
  r->reg[slot] = RegSlot();  // mappings stay cached until destroy
  return PCCLB_OK;
}

namespace {
std::mutex g_ipc_mu;
std::map<std::string, std::pair<char *, int>> g_ipc_open;  // handle -> (ptr, refs)
}  // namespace

int pcclb_ipc_open(const void *handle64, void **ptr_out) {
  if (!handle64 || !ptr_out) return PCCLB_EINVAL;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  std::string key(static_cast<const char *>(handle64), 64);
  auto it = g_ipc_open.find(key);
  if (it != g_ipc_open.end()) {
    it->second.second++;
    *ptr_out = it->second.first;
    return PCCLB_OK;
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  void *p = nullptr;
  PCCLB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  g_ipc_open.emplace(key, std::make_pair(static_cast<char *>(p), 1));
  *ptr_out = p;
  return PCCLB_OK;
}

int pcclb_ipc_close(void *ptr) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (auto it = g_ipc_open.begin(); it != g_ipc_open.end(); ++it) {
    if (it->second.first == ptr) {
      if (--it->second.second == 0) {
        cudaError_t e = cudaIpcCloseMemHandle(ptr);
        g_ipc_open.erase(it);
        if (e != cudaSuccess) return cuda_status(e);
      }
      return PCCLB_OK;
    }
  }
  return PCCLB_EINVAL;
}

int pcclb_copy(void *dst, const void *src, uint64_t bytes, void *stream) {
  if (bytes && (!dst || !src)) return PCCLB_EINVAL;
  if (!bytes) return PCCLB_OK;
  PCCLB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
  return PCCLB_OK;
}

void pcclb_ring_destroy(pcclb_ring *r) {
  if (!r) return;
  cudaSetDevice(r->device);
  cudaDeviceSynchronize();
  for (uint32_t j = 0; j < r->world; ++j)
    if (j != r->rank && r->imported[j] && r->peer_ws[j]) cudaIpcCloseMemHandle(r->peer_ws[j]);
  for (auto &kv : r->opened) cudaIpcCloseMemHandle(kv.second);
  if (r->ws) cudaFree(r->ws);
  if (r->host) cudaFreeHost((void *)r->host);
  if (r->status_host) cudaFreeHost(r->status_host);
  for (int i = 0; i < kMaxOps; ++i)
    if (r->op_events[i]) cudaEventDestroy(r->op_events[i]);
  if (r->timer.on)
    for (int i = 0; i < PhaseTimer::kMax; ++i) cudaEventDestroy(r->timer.ev[i]);
  delete r;
}

}  // extern "C"
