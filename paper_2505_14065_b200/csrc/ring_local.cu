// Local ring: W logical peers whose buffers all live on one GPU.
//
// Equivalent of the reference's in-process RingSession
// (tests/ring_harness.py:24-105 driving collective.py:489-567 per rank), and
// the single-GPU emulation of the intra-box ring: instead of 2(W-1) stepped
// kernels that would wait on each other, every chunk's fold chain runs in one
// launch (SURVEY §0 finding 2: chunk c folds x_c, x_{c+1}, ..., x_{c-1} as
// acc <- local (+) incoming; chunks are independent).
//
//   plain:     ONE kernel. Each thread reads the W inputs of one element of
//              chunk c, folds them in ring order, and writes the (AVG-divided)
//              result to all W buffers: W reads + W writes per element, the
//              minimum traffic. Reading all inputs before writing any output
//              at the same index makes the in-place update hazard-free.
//   quantized: W+1 kernels. Hop 0 computes each chunk's range; hop k fuses
//              "quantize acc_{k-1} with its range, dequantize, accumulate into
//              x_{c+k}, range of acc_k" (the wire codes never need to exist on
//              one GPU); the last kernel is the owner's adoption D(Q(acc)),
//              AVG division and the gather to every buffer.
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"
#include "elementwise.cuh"
#include "numerics.cuh"

namespace pcclb {

constexpr int kLocalThreads = 256;
constexpr int kMaxWorld = 64;

template <typename T>
struct LocalBufs {
  T *b[kMaxWorld];
  uint64_t n;
  uint32_t w;
  uint32_t avg;  // W when op is AVG, else 0
};

__device__ __forceinline__ void chunk_range(uint64_t n, uint32_t w, uint32_t c, uint64_t &lo,
                                            uint64_t &len) {
  const uint64_t base = n / w, extra = n % w;
  lo = c * base + min((uint64_t)c, extra);
  len = base + ((uint64_t)c < extra ? 1 : 0);
}

// ---------------------------------------------------------------------------
// plain: fold all chunks, write result everywhere
// ---------------------------------------------------------------------------
template <typename T, int OP>
struct FoldAllF {
  const LocalBufs<T> *P;
  uint32_t c;
  uint64_t lo;
  __device__ __forceinline__ T finish(T acc) const {
    return P->avg ? div_world(acc, (T)P->avg) : acc;
  }
  __device__ __forceinline__ void one(uint64_t i) {
    const uint32_t w = P->w;
    const uint64_t j = lo + i;
    uint32_t r = c;
    T acc = P->b[r][j];
    for (uint32_t k = 1; k < w; ++k) {
      r = (r + 1 == w) ? 0 : r + 1;
      acc = reduce_op<OP>(P->b[r][j], acc);
    }
    acc = finish(acc);
    for (uint32_t d = 0; d < w; ++d) P->b[d][j] = acc;
  }
  __device__ __forceinline__ void vec(uint64_t i) {
    constexpr int N = Pack16<T>::N;
    const uint32_t w = P->w;
    const uint64_t j = lo + i;
    uint32_t r = c;
    Pack16<T> acc = ld16(P->b[r] + j);
#pragma unroll 4
    for (uint32_t k = 1; k < w; ++k) {
      r = (r + 1 == w) ? 0 : r + 1;
      Pack16<T> x = ld16(P->b[r] + j);
#pragma unroll
      for (int e = 0; e < N; ++e) acc.e[e] = reduce_op<OP>(x.e[e], acc.e[e]);
    }
#pragma unroll
    for (int e = 0; e < N; ++e) acc.e[e] = finish(acc.e[e]);
    for (uint32_t d = 0; d < w; ++d) st16(P->b[d] + j, acc);
  }
  // two independent vectors: both fold chains' loads are in flight together
  __device__ __forceinline__ void vec2(uint64_t i0, uint64_t i1) {
    constexpr int N = Pack16<T>::N;
    const uint32_t w = P->w;
    const uint64_t j0 = lo + i0, j1 = lo + i1;
    uint32_t r = c;
    Pack16<T> a0 = ld16(P->b[r] + j0), a1 = ld16(P->b[r] + j1);
#pragma unroll 4
    for (uint32_t k = 1; k < w; ++k) {
      r = (r + 1 == w) ? 0 : r + 1;
      Pack16<T> x0 = ld16(P->b[r] + j0), x1 = ld16(P->b[r] + j1);
#pragma unroll
      for (int e = 0; e < N; ++e) {
        a0.e[e] = reduce_op<OP>(x0.e[e], a0.e[e]);
        a1.e[e] = reduce_op<OP>(x1.e[e], a1.e[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < N; ++e) {
      a0.e[e] = finish(a0.e[e]);
      a1.e[e] = finish(a1.e[e]);
    }
    for (uint32_t d = 0; d < w; ++d) {
      st16(P->b[d] + j0, a0);
      st16(P->b[d] + j1, a1);
    }
  }
};

template <typename T, int OP, int VEC>
__global__ void __launch_bounds__(kLocalThreads, 4) local_fold_all_kernel(const __grid_constant__ LocalBufs<T> P) {
  const uint32_t c = blockIdx.y;
  uint64_t lo, len;
  chunk_range(P.n, P.w, c, lo, len);
  if (len == 0) return;
  FoldAllF<T, OP> f{&P, c, lo};
  uint64_t head = 0;
  if (VEC > 1) {
    uintptr_t a = reinterpret_cast<uintptr_t>(P.b[0] + lo);
    head = ((16 - (a & 15)) & 15) / sizeof(T);
  }
  // this chunk's blocks form a 1-D grid of gridDim.x CTAs
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  if (VEC == 1) {
    for (uint64_t i = tid; i < len; i += nth) f.one(i);
    return;
  }
  if (head > len) head = len;
  if (tid < head) f.one(tid);
  const uint64_t nv = (len - head) / VEC;
  uint64_t v = tid;
  for (; v + nth < nv; v += 2 * nth) f.vec2(head + v * VEC, head + (v + nth) * VEC);
  for (; v < nv; v += nth) f.vec(head + v * VEC);
  const uint64_t t0 = head + nv * VEC;
  if (tid < len - t0) f.one(t0 + tid);
}

// ---------------------------------------------------------------------------
// quantized hops
// ---------------------------------------------------------------------------
// hop 0: range of x_c over chunk c (ranges[c*w + 0])
__global__ void __launch_bounds__(kLocalThreads, 4)
    local_q_range0_kernel(const __grid_constant__ LocalBufs<float> P, pcclb_range *ranges) {
  const uint32_t c = blockIdx.y;
  uint64_t lo, len;
  chunk_range(P.n, P.w, c, lo, len);
  if (len == 0) return;
  const float *x = P.b[c] + lo;
  RangeAcc acc;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  uintptr_t a = reinterpret_cast<uintptr_t>(x);
  uint64_t head = min((uint64_t)(((16 - (a & 15)) & 15) / 4), len);
  if (tid < head) acc.add(x[tid]);
  const uint64_t nv = (len - head) / 4;
  for (uint64_t v = tid; v < nv; v += nth) {
    Pack16<float> p = ld16(x + head + v * 4);
#pragma unroll
    for (int e = 0; e < 4; ++e) acc.add(p.e[e]);
  }
  const uint64_t t0 = head + nv * 4;
  if (tid < len - t0) acc.add(x[t0 + tid]);
  range_block_commit(acc, &ranges[(uint64_t)c * P.w]);
}

// hop k >= 1: x_{c+k} <- x_{c+k} (+) D(Q(acc_{k-1})), range -> ranges[c*w + k]
template <int OP, int QF>
__global__ void __launch_bounds__(kLocalThreads, 4)
    local_q_hop_kernel(const __grid_constant__ LocalBufs<float> P, pcclb_range *ranges, uint32_t k) {
  const uint32_t c = blockIdx.y;
  const uint32_t w = P.w;
  uint64_t lo, len;
  chunk_range(P.n, w, c, lo, len);
  if (len == 0) return;
  const float *prev = P.b[(c + k - 1) % w] + lo;
  float *cur = P.b[(c + k) % w] + lo;
  const QParams qp = qparams_q<QF>(ranges[(uint64_t)c * w + k - 1]);
  RangeAcc acc;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  auto one = [&](uint64_t i) {
    float d = dequantq<QF>(quantq<QF>(prev[i], qp), qp);
    float v = reduce_op<OP>(cur[i], d);
    cur[i] = v;
    acc.add(v);
  };
  uintptr_t a = reinterpret_cast<uintptr_t>(cur);
  uint64_t head = min((uint64_t)(((16 - (a & 15)) & 15) / 4), len);
  if (tid < head) one(tid);
  const uint64_t nv = (len - head) / 4;
  auto apply = [&](uint64_t i, const Pack16<float> &pv, Pack16<float> cv) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float d = dequantq<QF>(quantq<QF>(pv.e[e], qp), qp);
      cv.e[e] = reduce_op<OP>(cv.e[e], d);
      acc.add(cv.e[e]);
    }
    st16(cur + i, cv);
  };
  constexpr int U = 4;  // loads of U vectors issued before any store
  uint64_t v = tid;
  for (; v + (U - 1) * nth < nv; v += U * nth) {
    Pack16<float> pv[U], cv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      pv[u] = ld16(prev + head + (v + u * nth) * 4);
      cv[u] = ld16(cur + head + (v + u * nth) * 4);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) apply(head + (v + u * nth) * 4, pv[u], cv[u]);
  }
  for (; v < nv; v += nth) {
    const uint64_t i = head + v * 4;
    apply(i, ld16(prev + i), ld16(cur + i));
  }
  const uint64_t t0 = head + nv * 4;
  if (tid < len - t0) one(t0 + tid);
  range_block_commit(acc, &ranges[(uint64_t)c * w + k]);
}

// owner adoption + AVG + gather: every buffer's chunk c <- D(Q(acc_{W-1})) [/W]
template <int QF>
__global__ void __launch_bounds__(kLocalThreads, 4)
    local_q_final_kernel(const __grid_constant__ LocalBufs<float> P, const pcclb_range *ranges) {
  const uint32_t c = blockIdx.y;
  const uint32_t w = P.w;
  uint64_t lo, len;
  chunk_range(P.n, w, c, lo, len);
  if (len == 0) return;
  const uint32_t owner = (c + w - 1) % w;
  const float *acc = P.b[owner] + lo;
  const QParams qp = qparams_q<QF>(ranges[(uint64_t)c * w + w - 1]);
  const float avg = (float)P.avg;
  auto val = [&](float x) {
    float d = dequantq<QF>(quantq<QF>(x, qp), qp);
    return P.avg ? div_world(d, avg) : d;
  };
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  uintptr_t a = reinterpret_cast<uintptr_t>(acc);
  uint64_t head = min((uint64_t)(((16 - (a & 15)) & 15) / 4), len);
  auto one = [&](uint64_t i) {
    float v = val(acc[i]);
    for (uint32_t d = 0; d < w; ++d) P.b[d][lo + i] = v;
  };
  if (tid < head) one(tid);
  const uint64_t nv = (len - head) / 4;
  for (uint64_t v = tid; v < nv; v += nth) {
    const uint64_t i = head + v * 4;
    Pack16<float> pv = ld16(acc + i);
#pragma unroll
    for (int e = 0; e < 4; ++e) pv.e[e] = val(pv.e[e]);
    for (uint32_t d = 0; d < w; ++d) st16(P.b[d] + lo + i, pv);
  }
  const uint64_t t0 = head + nv * 4;
  if (tid < len - t0) one(t0 + tid);
}

template <typename T>
static bool same_alignment(void *const *bufs, uint32_t w) {
  uintptr_t a0 = reinterpret_cast<uintptr_t>(bufs[0]) & 15;
  for (uint32_t i = 1; i < w; ++i)
    if ((reinterpret_cast<uintptr_t>(bufs[i]) & 15) != a0) return false;
  return true;
}

template <typename T>
static int local_plain(const LocalBufs<T> &P, int op, bool vec, dim3 grid, cudaStream_t s) {
#define PCCLB_FOLD(OPC)                                                                  \
  if (vec)                                                                               \
    local_fold_all_kernel<T, OPC, 16 / sizeof(T)><<<grid, kLocalThreads, 0, s>>>(P);     \
  else                                                                                   \
    local_fold_all_kernel<T, OPC, 1><<<grid, kLocalThreads, 0, s>>>(P);
  switch (op) {
    case PCCLB_MAX:
      PCCLB_FOLD(PCCLB_MAX);
      break;
    case PCCLB_MIN:
      PCCLB_FOLD(PCCLB_MIN);
      break;
    case PCCLB_PROD:
      PCCLB_FOLD(PCCLB_PROD);
      break;
    default:
      PCCLB_FOLD(PCCLB_SUM);
      break;
  }
#undef PCCLB_FOLD
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}


// hops 1..W-1 and the final adoption+gather for quantization format QF
template <int QF>
int local_q_hops(const LocalBufs<float> &P, pcclb_range *ranges, int op, dim3 grid, cudaStream_t s) {
  for (uint32_t k = 1; k < P.w; ++k) {
    switch (op) {
      case PCCLB_MAX:
        local_q_hop_kernel<PCCLB_MAX, QF><<<grid, kLocalThreads, 0, s>>>(P, ranges, k);
        break;
      case PCCLB_MIN:
        local_q_hop_kernel<PCCLB_MIN, QF><<<grid, kLocalThreads, 0, s>>>(P, ranges, k);
        break;
      case PCCLB_PROD:
        local_q_hop_kernel<PCCLB_PROD, QF><<<grid, kLocalThreads, 0, s>>>(P, ranges, k);
        break;
      default:
        local_q_hop_kernel<PCCLB_SUM, QF><<<grid, kLocalThreads, 0, s>>>(P, ranges, k);
        break;
    }
    PCCLB_LAUNCH_CHECK();
  }
  local_q_final_kernel<QF><<<grid, kLocalThreads, 0, s>>>(P, ranges);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

}  // namespace pcclb

using namespace pcclb;

extern "C" {

uint64_t pcclb_local_scratch_bytes(uint32_t world) {
  return (uint64_t)world * world * sizeof(pcclb_range);
}

int pcclb_local_allreduce(void *const *h_bufs, uint32_t w, uint64_t n, int dtype, int op,
                          int quantize, void *d_scratch, void *d_backup, void *stream) {
  return pcclb_local_allreduce_ex(h_bufs, w, n, dtype, op, quantize ? PCCLB_Q_U8 : 0, d_scratch, d_backup,
                                  stream);
}

int pcclb_local_allreduce_ex(void *const *h_bufs, uint32_t w, uint64_t n, int dtype, int op, int qformat,
                             void *d_scratch, void *d_backup, void *stream) {
  const int quantize = qformat != 0;
  if (!h_bufs || w < 1 || w > (uint32_t)kMaxWorld || !valid_dtype(dtype) || !valid_op(op) || qformat < 0 ||
      qformat > PCCLB_Q_U16_ZP)
    return PCCLB_EINVAL;
  if (quantize && dtype != PCCLB_F32) return PCCLB_EINVAL;  // client.py:818-819
  for (uint32_t i = 0; i < w; ++i)
    if (n && !h_bufs[i]) return PCCLB_EINVAL;
  cudaStream_t s = as_stream(stream);
  const size_t esz = dtype_size(dtype);
  if (n == 0) return PCCLB_OK;
  if (w == 1)  // client.py:896-900: finalize only, never quantized
    return pcclb_finalize(h_bufs[0], n, dtype, op, 1, stream);
  if (quantize && !d_scratch) return PCCLB_EINVAL;
  if (d_backup)  // collective.py:501-504
    for (uint32_t i = 0; i < w; ++i)
      PCCLB_CUDA(cudaMemcpyAsync(static_cast<char *>(d_backup) + (uint64_t)i * n * esz, h_bufs[i],
                                 n * esz, cudaMemcpyDeviceToDevice, s));
  const uint64_t n_c = (n + w - 1) / w;
  const int target = sm_count() * 8;
  unsigned per_chunk = (unsigned)std::max<int64_t>(1, target / (int)w);
  const uint64_t per_cta = (uint64_t)kLocalThreads * 4;
  uint64_t need = (n_c + per_cta - 1) / per_cta;
  if (need < per_chunk) per_chunk = (unsigned)std::max<uint64_t>(1, need);
  dim3 grid(per_chunk, w);
  const bool vec = same_alignment<float>(h_bufs, w);
  const uint32_t avg = (op == PCCLB_AVG) ? w : 0;
  if (!quantize) {
    if (dtype == PCCLB_F32) {
      LocalBufs<float> P{};
      for (uint32_t i = 0; i < w; ++i) P.b[i] = static_cast<float *>(h_bufs[i]);
      P.n = n, P.w = w, P.avg = avg;
      return local_plain<float>(P, op, vec, grid, s);
    }
    if (dtype == PCCLB_BF16) {
      LocalBufs<Bf16> P{};
      for (uint32_t i = 0; i < w; ++i) P.b[i] = static_cast<Bf16 *>(h_bufs[i]);
      P.n = n, P.w = w, P.avg = avg;
      return local_plain<Bf16>(P, op, vec, grid, s);
    }
    LocalBufs<double> P{};
    for (uint32_t i = 0; i < w; ++i) P.b[i] = static_cast<double *>(h_bufs[i]);
    P.n = n, P.w = w, P.avg = avg;
    return local_plain<double>(P, op, vec, grid, s);
  }
  LocalBufs<float> P{};
  for (uint32_t i = 0; i < w; ++i) P.b[i] = static_cast<float *>(h_bufs[i]);
  P.n = n, P.w = w, P.avg = avg;
  pcclb_range *ranges = static_cast<pcclb_range *>(d_scratch);
  PCCLB_CUDA(cudaMemsetAsync(ranges, 0, pcclb_local_scratch_bytes(w), s));
  local_q_range0_kernel<<<grid, kLocalThreads, 0, s>>>(P, ranges);
  PCCLB_LAUNCH_CHECK();
  int rcq = PCCLB_OK;
  switch (qformat) {
    case PCCLB_Q_U16:
      rcq = local_q_hops<PCCLB_Q_U16>(P, ranges, op, grid, s);
      break;
    case PCCLB_Q_U8_ZP:
      rcq = local_q_hops<PCCLB_Q_U8_ZP>(P, ranges, op, grid, s);
      break;
    case PCCLB_Q_U16_ZP:
      rcq = local_q_hops<PCCLB_Q_U16_ZP>(P, ranges, op, grid, s);
      break;
    default:
      rcq = local_q_hops<PCCLB_Q_U8>(P, ranges, op, grid, s);
      break;
  }
  if (rcq) return rcq;
  // every quantized span must have been finite (collective.py:117-118)
  std::vector<pcclb_range> host(w * w);
  PCCLB_CUDA(cudaMemcpyAsync(host.data(), ranges, pcclb_local_scratch_bytes(w),
                             cudaMemcpyDeviceToHost, s));
  PCCLB_CUDA(cudaStreamSynchronize(s));
  bool bad = false;
  for (auto &r : host) bad |= r.nonfinite != 0;
  if (!bad) return PCCLB_OK;
  if (d_backup) {  // restore instead of leaving inf/NaN behind (SURVEY §0 finding 5)
    for (uint32_t i = 0; i < w; ++i)
      PCCLB_CUDA(cudaMemcpyAsync(h_bufs[i], static_cast<char *>(d_backup) + (uint64_t)i * n * esz,
                                 n * esz, cudaMemcpyDeviceToDevice, s));
    PCCLB_CUDA(cudaStreamSynchronize(s));
  }
  return PCCLB_ENONFINITE;
}

}  // extern "C"
