// CRC-32 (zlib / IEEE 802.3: reflected, polynomial 0xEDB88320, init and final
// xor 0xFFFFFFFF) of device buffers -- the north_star's alternative shared-
// state digest. The reference has no CRC32; the checker is
// zlib.crc32 itself (tests/test_extensions_gpu.py).
//
// CRC is linear over GF(2). With raw(D) the register after D from a zero
// start, raw(A || B) = shift(raw(A), |B|) ^ raw(B), where shift multiplies by
// x^(8|B|) mod P (zlib's multmodp / x2nmodp), and
//   crc32(D) = raw(D) ^ shift(0xFFFFFFFF, |D|) ^ 0xFFFFFFFF.
// So a buffer is cut into 256 KiB segments, one per CTA: each thread takes
// 1 KiB (slice-by-8 table lookups from shared memory, 16-byte loads), the CTA
// combines its threads' registers with constant shifts, and a second kernel
// combines the segments of every entry (Horner over each thread's run of
// segments, then one shift per thread). Bound: shared-memory table lookups,
// one per byte.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace pcclb {

constexpr uint32_t kCrcPoly = 0xedb88320u;
constexpr int kCrcThreads = 256;
constexpr uint32_t kCrcPerThread = 1024;                        // bytes per thread of a full segment
constexpr uint64_t kCrcSeg = (uint64_t)kCrcThreads * kCrcPerThread;  // bytes per segment (CTA item)
constexpr int kCrcMaxEntries = 512;

__host__ __device__ inline uint32_t crc_multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
  }
  return p;
}

struct CrcConst {
  uint32_t x2n[32];            // x^(2^k) mod P
  uint32_t thread_mul[kCrcThreads];  // x^(8 * kCrcPerThread * (kCrcThreads - 1 - t)) mod P
  uint32_t seg_mul;            // x^(8 * kCrcSeg) mod P
  uint32_t table[8][256];      // slice-by-8
};
__constant__ CrcConst c_crc;

__host__ inline uint32_t host_x2nmodp(const uint32_t *x2n, uint64_t n, uint32_t k) {
  uint32_t p = 1u << 31;
  while (n) {
    if (n & 1) p = crc_multmodp(x2n[k & 31], p);
    n >>= 1;
    ++k;
  }
  return p;
}

__device__ __forceinline__ uint32_t crc_x2nmodp(uint64_t n, uint32_t k) {
  uint32_t p = 1u << 31;
  while (n) {
    if (n & 1) p = crc_multmodp(c_crc.x2n[k & 31], p);
    n >>= 1;
    ++k;
  }
  return p;
}
// register advanced through `nbytes` zero bytes
__device__ __forceinline__ uint32_t crc_shift(uint32_t crc, uint64_t nbytes) {
  return nbytes ? crc_multmodp(crc_x2nmodp(nbytes, 3), crc) : crc;
}

struct CrcEntry {
  const uint8_t *ptr;
  uint64_t nbytes;
  uint32_t *out;
  uint32_t seg0;  // first segment item of the entry
  uint32_t nseg;
};
struct CrcBatch {
  uint32_t count;
  uint32_t items;
  CrcEntry e[kCrcMaxEntries];
};

__device__ __forceinline__ uint32_t crc_bytes(const uint32_t (*T)[256], uint32_t c, const uint8_t *p, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) c = T[0][(c ^ p[i]) & 0xff] ^ (c >> 8);
  return c;
}

// one 8-byte slice-by-8 step on the replicated tables: entry i of table s,
// copy r sits at word ((s * 256 + i) * kCrcCopies + r); a lane reads copy
// lane % kCrcCopies, so the 32 lanes of a lookup spread over
// (entry * kCrcCopies + copy) mod 32 banks (random entries: ~1.6 instead of
// ~3.5 wavefronts per lookup)
constexpr int kCrcCopies = 8;
__device__ __forceinline__ uint32_t crc_step8r(const uint32_t *T, uint32_t r, uint32_t c, uint32_t lo, uint32_t hi) {
  c ^= lo;
#define CRC_T(s, i) T[(((s) * 256u + (i)) * kCrcCopies) + r]
  return CRC_T(7, c & 0xff) ^ CRC_T(6, (c >> 8) & 0xff) ^ CRC_T(5, (c >> 16) & 0xff) ^ CRC_T(4, c >> 24) ^
         CRC_T(3, hi & 0xff) ^ CRC_T(2, (hi >> 8) & 0xff) ^ CRC_T(1, (hi >> 16) & 0xff) ^ CRC_T(0, hi >> 24);
#undef CRC_T
}

constexpr int kCrcSmem = 8 * 256 * kCrcCopies * 4;

__global__ void __launch_bounds__(kCrcThreads) crc32_seg_kernel(const __grid_constant__ CrcBatch b, uint32_t *seg_raw) {
  extern __shared__ uint32_t TR[];  // 8 tables x 256 entries x kCrcCopies
  __shared__ uint32_t s_red[kCrcThreads / 32];
  for (int i = threadIdx.x; i < 8 * 256 * kCrcCopies; i += blockDim.x) TR[i] = (&c_crc.table[0][0])[i / kCrcCopies];
  __syncthreads();
  const uint32_t t = threadIdx.x, rcopy = t % kCrcCopies;
  const uint32_t(*T)[256] = reinterpret_cast<const uint32_t(*)[256]>(&c_crc.table[0][0]);  // byte tail path
  for (uint32_t item = blockIdx.x; item < b.items; item += gridDim.x) {
    // entry of the item (entries hold consecutive item ranges)
    uint32_t lo = 0, hi = b.count;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) / 2;
      if (b.e[mid].seg0 <= item) lo = mid;
      else hi = mid;
    }
    const CrcEntry &E = b.e[lo];
    const uint64_t s0 = (uint64_t)(item - E.seg0) * kCrcSeg;
    const uint64_t seg_len = E.nbytes - s0 < kCrcSeg ? E.nbytes - s0 : kCrcSeg;
    const uint64_t a0 = (uint64_t)t * kCrcPerThread;
    const uint32_t len = a0 >= seg_len ? 0u : (uint32_t)(seg_len - a0 < kCrcPerThread ? seg_len - a0 : kCrcPerThread);
    const uint8_t *p = E.ptr + s0 + a0;
    uint32_t c = 0;
    if (len == kCrcPerThread && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      const uint4 *q = reinterpret_cast<const uint4 *>(p);
#pragma unroll 4
      for (uint32_t i = 0; i < kCrcPerThread / 16; ++i) {
        const uint4 v = __ldcs(q + i);
        c = crc_step8r(TR, rcopy, c, v.x, v.y);
        c = crc_step8r(TR, rcopy, c, v.z, v.w);
      }
    } else {
      c = crc_bytes(T, c, p, len);
    }
    // this thread's register shifted past the bytes after it in the segment
    if (seg_len == kCrcSeg) c = crc_multmodp(c_crc.thread_mul[t], c);
    else c = crc_shift(c, seg_len - (a0 + len < seg_len ? a0 + len : seg_len));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c ^= __shfl_xor_sync(0xffffffffu, c, o);
    if ((t & 31) == 0) s_red[t >> 5] = c;
    __syncthreads();
    if (t == 0) {
      uint32_t r = 0;
      for (int w = 0; w < kCrcThreads / 32; ++w) r ^= s_red[w];
      seg_raw[item] = r;
    }
    __syncthreads();
  }
}

// one CTA per entry: segments -> entry register -> zlib crc32
__global__ void __launch_bounds__(1024) crc32_combine_kernel(const __grid_constant__ CrcBatch b,
                                                             const uint32_t *seg_raw) {
  __shared__ uint32_t s_red[32];
  const CrcEntry &E = b.e[blockIdx.x];
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  const uint32_t per = (E.nseg + nt - 1) / nt;
  const uint32_t j0 = min(E.nseg, t * per), j1 = min(E.nseg, j0 + per);
  uint32_t acc = 0;
  uint64_t end = (uint64_t)j0 * kCrcSeg;  // bytes covered so far
  for (uint32_t j = j0; j < j1; ++j) {
    const uint64_t rem = E.nbytes - (uint64_t)j * kCrcSeg, len = rem < kCrcSeg ? rem : kCrcSeg;
    acc = (len == kCrcSeg ? crc_multmodp(c_crc.seg_mul, acc) : crc_shift(acc, len)) ^ seg_raw[E.seg0 + j];
    end = (uint64_t)j * kCrcSeg + len;
  }
  if (j1 > j0) acc = crc_shift(acc, E.nbytes - end);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if ((t & 31) == 0) s_red[t >> 5] = acc;
  __syncthreads();
  if (t == 0) {
    uint32_t r = 0;
    for (uint32_t w = 0; w < (nt + 31) / 32; ++w) r ^= s_red[w];
    *E.out = r ^ crc_shift(0xffffffffu, E.nbytes) ^ 0xffffffffu;
  }
}

static int crc_init_constants() {
  static bool done[64] = {false};
  int dev = 0;
  PCCLB_CUDA(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && done[dev]) return PCCLB_OK;
  static CrcConst h = [] {
    CrcConst k{};
    k.x2n[0] = 1u << 30;  // x^1
    for (int i = 1; i < 32; ++i) k.x2n[i] = crc_multmodp(k.x2n[i - 1], k.x2n[i - 1]);
    for (int t = 0; t < kCrcThreads; ++t)
      k.thread_mul[t] = host_x2nmodp(k.x2n, (uint64_t)kCrcPerThread * (kCrcThreads - 1 - t), 3);
    k.seg_mul = host_x2nmodp(k.x2n, kCrcSeg, 3);
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int j = 0; j < 8; ++j) c = (c & 1) ? (c >> 1) ^ kCrcPoly : c >> 1;
      k.table[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
      for (int s = 1; s < 8; ++s) k.table[s][i] = k.table[0][k.table[s - 1][i] & 0xff] ^ (k.table[s - 1][i] >> 8);
    return k;
  }();
  PCCLB_CUDA(cudaMemcpyToSymbol(c_crc, &h, sizeof(h)));
  if (dev >= 0 && dev < 64) done[dev] = true;
  return PCCLB_OK;
}

}  // namespace pcclb

using namespace pcclb;

extern "C" {

int pcclb_crc32_multi(const void *const *h_ptrs, const uint64_t *h_nbytes, uint32_t count, uint32_t *d_out,
                      void *stream) {
  if (count == 0) return PCCLB_OK;
  if (!h_ptrs || !h_nbytes || !d_out) return PCCLB_EINVAL;
  for (uint32_t i = 0; i < count; ++i)
    if (h_nbytes[i] && !h_ptrs[i]) return PCCLB_EINVAL;
  int rc = crc_init_constants();
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  static const cudaError_t attr = cudaFuncSetAttribute(crc32_seg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       kCrcSmem);
  if (attr != cudaSuccess) return cuda_status(attr);
  static thread_local CrcBatch batch;
  for (uint32_t base = 0; base < count; base += kCrcMaxEntries) {
    const uint32_t m = std::min<uint32_t>(kCrcMaxEntries, count - base);
    uint64_t items = 0;
    for (uint32_t i = 0; i < m; ++i) {
      CrcEntry &E = batch.e[i];
      E.ptr = static_cast<const uint8_t *>(h_ptrs[base + i]);
      E.nbytes = h_nbytes[base + i];
      E.out = d_out + base + i;
      E.seg0 = (uint32_t)items;
      E.nseg = (uint32_t)((E.nbytes + kCrcSeg - 1) / kCrcSeg);
      items += E.nseg;
    }
    if (items >= (1ull << 32)) return PCCLB_EINVAL;
    batch.count = m;
    batch.items = (uint32_t)items;
    uint32_t *seg_raw = nullptr;
    if (items) PCCLB_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&seg_raw), items * sizeof(uint32_t), s));
    if (items) {
      const unsigned grid = (unsigned)std::min<uint64_t>(items, (uint64_t)sm_count() * 8);
      crc32_seg_kernel<<<grid, kCrcThreads, kCrcSmem, s>>>(batch, seg_raw);
      PCCLB_LAUNCH_CHECK();
    }
    crc32_combine_kernel<<<m, 1024, 0, s>>>(batch, seg_raw);
    PCCLB_LAUNCH_CHECK();
    if (seg_raw) PCCLB_CUDA(cudaFreeAsync(seg_raw, s));
  }
  return PCCLB_OK;
}

int pcclb_crc32(const void *d_data, uint64_t nbytes, uint32_t *d_out, void *stream) {
  return pcclb_crc32_multi(&d_data, &nbytes, 1, d_out, stream);
}

}  // extern "C"
