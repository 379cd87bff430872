// Single-GPU kernel seams of the ring data plane.
//
//   pcclb_accumulate            K1  collective.py:66-71, :407, :416
//   pcclb_finalize              K8  collective.py:479-482
//   pcclb_range_f32             K2  collective.py:117-121
//   pcclb_quantize_u8           K3/K6 collective.py:119-129, :538-551
//   pcclb_dequantize_u8         K4/K7 collective.py:132-135, :445-452
//   pcclb_dequant_accumulate_u8 K5  collective.py:399-409
//
// All are HBM-bound streaming kernels: 128-bit vector loads/stores, grid
// sized to a multiple of the SM count, arithmetic from numerics.cuh.
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "elementwise.cuh"
#include "numerics.cuh"
#include "ew_ops.cuh"

namespace pcclb {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

// ---------------------------------------------------------------------------
// K1 accumulate
// ---------------------------------------------------------------------------
template <typename T, int OP>
struct AccumulateF {
  T *__restrict__ acc;
  const T *__restrict__ in;
  __device__ __forceinline__ void one(uint64_t i) { acc[i] = reduce_op<OP>(acc[i], in[i]); }
  struct In {
    Pack16<T> a, b;
  };
  __device__ __forceinline__ In vload(uint64_t i) {
    In v;
    v.a = ld16(acc + i);
    v.b = ld16_cs(in + i);
    return v;
  }
  __device__ __forceinline__ void vapply(uint64_t i, const In &v) {
    Pack16<T> a = v.a;
#pragma unroll
    for (int k = 0; k < Pack16<T>::N; ++k) a.e[k] = reduce_op<OP>(a.e[k], v.b.e[k]);
    st16(acc + i, a);
  }
};

template <typename T, int OP, int VEC>
__global__ void __launch_bounds__(kThreads, 4) accumulate_kernel(T *acc, const T *in, uint64_t n,
                                                               uint64_t head) {
  AccumulateF<T, OP> f{acc, in};
  ew_loop<VEC, kUnroll>(n, head, f);
}

template <typename T, int OP>
static int launch_accumulate(T *acc, const T *in, uint64_t n, cudaStream_t s) {
  if (n == 0) return PCCLB_OK;
  uint64_t head = peel16<T>(acc);
  bool vec_ok = peel16<T>(in) == head;
  unsigned grid = grid_for(n, (uint64_t)kThreads * kUnroll * (16 / sizeof(T)));
  if (vec_ok)
    accumulate_kernel<T, OP, 16 / sizeof(T)><<<grid, kThreads, 0, s>>>(acc, in, n, head);
  else
    accumulate_kernel<T, OP, 1><<<grid, kThreads, 0, s>>>(acc, in, n, 0);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

template <typename T>
static int dispatch_accumulate(void *acc, const void *in, uint64_t n, int op, cudaStream_t s) {
  T *a = static_cast<T *>(acc);
  const T *b = static_cast<const T *>(in);
  switch (op) {
    case PCCLB_SUM:
    case PCCLB_AVG:
      return launch_accumulate<T, PCCLB_SUM>(a, b, n, s);
    case PCCLB_MAX:
      return launch_accumulate<T, PCCLB_MAX>(a, b, n, s);
    case PCCLB_MIN:
      return launch_accumulate<T, PCCLB_MIN>(a, b, n, s);
    case PCCLB_PROD:
      return launch_accumulate<T, PCCLB_PROD>(a, b, n, s);
  }
  return PCCLB_EINVAL;
}

// ---------------------------------------------------------------------------
// K8 finalize: buf /= dtype(W)
// ---------------------------------------------------------------------------
template <typename T>
struct DivF {
  T *__restrict__ buf;
  T w;
  __device__ __forceinline__ void one(uint64_t i) { buf[i] = div_world(buf[i], w); }
  using In = Pack16<T>;
  __device__ __forceinline__ In vload(uint64_t i) { return ld16(buf + i); }
  __device__ __forceinline__ void vapply(uint64_t i, const In &v) {
    Pack16<T> a = v;
#pragma unroll
    for (int k = 0; k < Pack16<T>::N; ++k) a.e[k] = div_world(a.e[k], w);
    st16(buf + i, a);
  }
};

template <typename T, int VEC>
__global__ void __launch_bounds__(kThreads, 4) div_kernel(T *buf, uint64_t n, uint64_t head, T w) {
  DivF<T> f{buf, w};
  ew_loop<VEC, kUnroll>(n, head, f);
}

template <typename T>
static int launch_div(T *buf, uint64_t n, uint32_t w, cudaStream_t s) {
  if (n == 0) return PCCLB_OK;
  unsigned grid = grid_for(n, (uint64_t)kThreads * kUnroll * (16 / sizeof(T)));
  div_kernel<T, 16 / sizeof(T)><<<grid, kThreads, 0, s>>>(buf, n, peel16<T>(buf), (T)w);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

// K2 range
template <int VEC>
__global__ void __launch_bounds__(kThreads, 4) range_kernel(const float *x, uint64_t n, uint64_t head,
                                                          pcclb_range *out) {
  RangeF f{x, RangeAcc()};
  ew_loop<VEC, kUnroll>(n, head, f);
  range_block_commit(f.acc, out);
}

template <int VEC>
__global__ void __launch_bounds__(kThreads, 4)
    quantize_kernel(const float *x, uint64_t n, uint64_t head, const pcclb_range *range,
                    uint8_t *codes, pcclb_qmeta *meta, float *adopt, uint32_t avg_div) {
  QParams qp = qparams_from_range(*range);
  if (meta && blockIdx.x == 0 && threadIdx.x == 0) {
    meta->min_val = qp.mn;
    meta->scale = qp.scale;
  }
  QuantF f{x, codes, adopt, qp, (float)avg_div, avg_div > 1};
  ew_loop<VEC, kUnroll>(n, head, f);
}

template <int VEC>
__global__ void __launch_bounds__(kThreads, 4)
    dequantize_kernel(float *out, const uint8_t *codes, uint64_t n, uint64_t head,
                      const pcclb_qmeta *meta, uint32_t avg_div) {
  DequantF f{out, codes, meta->min_val, meta->scale, (float)avg_div, avg_div > 1};
  ew_loop<VEC, kUnroll>(n, head, f);
}

template <int OP, int VEC>
__global__ void __launch_bounds__(kThreads, 4)
    dequant_acc_kernel(float *acc, const uint8_t *codes, uint64_t n, uint64_t head,
                       const pcclb_qmeta *meta, pcclb_range *next) {
  DequantAccF<OP> f{acc, codes, meta->min_val, meta->scale, next != nullptr, RangeAcc()};
  ew_loop<VEC, kUnroll>(n, head, f);
  if (next) range_block_commit(f.r, next);
}

// ---------------------------------------------------------------------------
// quantization formats beyond u8 min-max (extensions, pcclb200.h PCCLB_Q_*):
// grid-stride kernels over the format's code type
// ---------------------------------------------------------------------------
template <int QF>
__global__ void __launch_bounds__(kThreads)
    quantize_q_kernel(const float *x, uint64_t n, const pcclb_range *range, void *codes_v, pcclb_qmeta *meta,
                      float *adopt, uint32_t avg_div) {
  using C = typename QFmt<QF>::Code;
  C *codes = static_cast<C *>(codes_v);
  const QParams qp = qparams_q<QF>(*range);
  if (meta && blockIdx.x == 0 && threadIdx.x == 0) {
    meta->min_val = qp.mn;  // the zero point for the _ZP formats
    meta->scale = qp.scale;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = quantq<QF>(x[i], qp);
    codes[i] = (C)q;
    if (adopt) {
      const float d = dequantq<QF>(q, qp);
      adopt[i] = avg_div > 1 ? div_world(d, (float)avg_div) : d;
    }
  }
}

template <int QF>
__global__ void __launch_bounds__(kThreads)
    dequantize_q_kernel(float *out, const void *codes_v, uint64_t n, const pcclb_qmeta *meta, uint32_t avg_div) {
  using C = typename QFmt<QF>::Code;
  const C *codes = static_cast<const C *>(codes_v);
  const QParams qp{meta->min_val, meta->scale, 0.0f};
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const float d = dequantq<QF>(codes[i], qp);
    out[i] = avg_div > 1 ? div_world(d, (float)avg_div) : d;
  }
}

template <int QF, int OP>
__global__ void __launch_bounds__(kThreads)
    dequant_acc_q_kernel(float *acc, const void *codes_v, uint64_t n, const pcclb_qmeta *meta, pcclb_range *next) {
  using C = typename QFmt<QF>::Code;
  const C *codes = static_cast<const C *>(codes_v);
  const QParams qp{meta->min_val, meta->scale, 0.0f};
  RangeAcc r;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const float v = reduce_op<OP>(acc[i], dequantq<QF>(codes[i], qp));
    acc[i] = v;
    if (next) r.add(v);
  }
  if (next) range_block_commit(r, next);
}

template <class F>
static int with_qformat(int qformat, F f) {
  switch (qformat) {
    case PCCLB_Q_U8:
      return f(std::integral_constant<int, PCCLB_Q_U8>());
    case PCCLB_Q_U16:
      return f(std::integral_constant<int, PCCLB_Q_U16>());
    case PCCLB_Q_U8_ZP:
      return f(std::integral_constant<int, PCCLB_Q_U8_ZP>());
    case PCCLB_Q_U16_ZP:
      return f(std::integral_constant<int, PCCLB_Q_U16_ZP>());
  }
  return PCCLB_EINVAL;
}

// float/code pointer pair vectorizable with the same peel?
static bool fc_vec_ok(const float *x, const uint8_t *codes, uint64_t *head) {
  uint64_t h = peel16<float>(x);
  *head = h;
  return ((reinterpret_cast<uintptr_t>(codes) + h) & 3) == 0;
}

}  // namespace pcclb

using namespace pcclb;

extern "C" {

int pcclb_accumulate(void *acc, const void *in, uint64_t n, int dtype, int op, void *stream) {
  if (!valid_dtype(dtype) || !valid_op(op) || (n && (!acc || !in))) return PCCLB_EINVAL;
  if (dtype == PCCLB_F32) return dispatch_accumulate<float>(acc, in, n, op, as_stream(stream));
  if (dtype == PCCLB_BF16) return dispatch_accumulate<Bf16>(acc, in, n, op, as_stream(stream));
  return dispatch_accumulate<double>(acc, in, n, op, as_stream(stream));
}

int pcclb_finalize(void *buf, uint64_t n, int dtype, int op, uint32_t world, void *stream) {
  if (!valid_dtype(dtype) || !valid_op(op) || world < 1 || (n && !buf)) return PCCLB_EINVAL;
  if (op != PCCLB_AVG) return PCCLB_OK;
  if (dtype == PCCLB_F32) return launch_div<float>((float *)buf, n, world, as_stream(stream));
  if (dtype == PCCLB_BF16) return launch_div<Bf16>((Bf16 *)buf, n, world, as_stream(stream));
  return launch_div<double>((double *)buf, n, world, as_stream(stream));
}

int pcclb_range_reset(pcclb_range *d_range, uint32_t count, void *stream) {
  if (!d_range) return PCCLB_EINVAL;
  PCCLB_CUDA(cudaMemsetAsync(d_range, 0, sizeof(pcclb_range) * count, as_stream(stream)));
  return PCCLB_OK;
}

int pcclb_range_f32(const float *x, uint64_t n, pcclb_range *d_range, void *stream) {
  if (!d_range || (n && !x)) return PCCLB_EINVAL;
  if (n == 0) return PCCLB_OK;
  cudaStream_t s = as_stream(stream);
  unsigned grid = grid_for(n, (uint64_t)kThreads * kUnroll * 4);
  range_kernel<4><<<grid, kThreads, 0, s>>>(x, n, peel16<float>(x), d_range);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

int pcclb_quantize_u8(const float *x, uint64_t n, const pcclb_range *d_range, uint8_t *codes,
                      pcclb_qmeta *d_meta, float *adopt_out, uint32_t avg_div, void *stream) {
  if (!d_range || (n && (!x || !codes)) || avg_div < 1) return PCCLB_EINVAL;
  cudaStream_t s = as_stream(stream);
  uint64_t head;
  bool ok = fc_vec_ok(x, codes, &head);
  if (adopt_out && peel16<float>(adopt_out) != head) ok = false;
  unsigned grid = grid_for(n ? n : 1, (uint64_t)kThreads * kUnroll * 4);
  if (ok)
    quantize_kernel<4><<<grid, kThreads, 0, s>>>(x, n, head, d_range, codes, d_meta, adopt_out,
                                                 avg_div);
  else
    quantize_kernel<1><<<grid, kThreads, 0, s>>>(x, n, 0, d_range, codes, d_meta, adopt_out,
                                                 avg_div);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

int pcclb_dequantize_u8(float *out, const uint8_t *codes, uint64_t n, const pcclb_qmeta *d_meta,
                        uint32_t avg_div, void *stream) {
  if (!d_meta || (n && (!out || !codes)) || avg_div < 1) return PCCLB_EINVAL;
  if (n == 0) return PCCLB_OK;
  cudaStream_t s = as_stream(stream);
  uint64_t head;
  bool ok = fc_vec_ok(out, codes, &head);
  unsigned grid = grid_for(n, (uint64_t)kThreads * kUnroll * 4);
  if (ok)
    dequantize_kernel<4><<<grid, kThreads, 0, s>>>(out, codes, n, head, d_meta, avg_div);
  else
    dequantize_kernel<1><<<grid, kThreads, 0, s>>>(out, codes, n, 0, d_meta, avg_div);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

int pcclb_dequant_accumulate_u8(float *acc, const uint8_t *codes, uint64_t n,
                                const pcclb_qmeta *d_meta, int op, pcclb_range *d_next_range,
                                void *stream) {
  if (!d_meta || !valid_op(op) || (n && (!acc || !codes))) return PCCLB_EINVAL;
  if (n == 0) return PCCLB_OK;
  cudaStream_t s = as_stream(stream);
  uint64_t head;
  bool ok = fc_vec_ok(acc, codes, &head);
  unsigned grid = grid_for(n, (uint64_t)kThreads * kUnroll * 4);
#define PCCLB_DQA(OPC)                                                                      \
  if (ok)                                                                                   \
    dequant_acc_kernel<OPC, 4><<<grid, kThreads, 0, s>>>(acc, codes, n, head, d_meta,       \
                                                         d_next_range);                     \
  else                                                                                      \
    dequant_acc_kernel<OPC, 1><<<grid, kThreads, 0, s>>>(acc, codes, n, 0, d_meta, d_next_range);
  switch (op) {
    case PCCLB_MAX:
      PCCLB_DQA(PCCLB_MAX);
      break;
    case PCCLB_MIN:
      PCCLB_DQA(PCCLB_MIN);
      break;
    case PCCLB_PROD:
      PCCLB_DQA(PCCLB_PROD);
      break;
    default:
      PCCLB_DQA(PCCLB_SUM);
      break;
  }
#undef PCCLB_DQA
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

int pcclb_quantize_ex(const float *x, uint64_t n, const pcclb_range *d_range, void *codes, pcclb_qmeta *d_meta,
                      float *adopt_out, uint32_t avg_div, int qformat, void *stream) {
  if (qformat == PCCLB_Q_U8)
    return pcclb_quantize_u8(x, n, d_range, static_cast<uint8_t *>(codes), d_meta, adopt_out, avg_div, stream);
  if (!d_range || (n && (!x || !codes)) || avg_div < 1) return PCCLB_EINVAL;
  cudaStream_t s = as_stream(stream);
  const unsigned grid = grid_for(n ? n : 1, (uint64_t)kThreads * 8);
  return with_qformat(qformat, [&](auto qf) -> int {
    quantize_q_kernel<decltype(qf)::value><<<grid, kThreads, 0, s>>>(x, n, d_range, codes, d_meta, adopt_out, avg_div);
    PCCLB_LAUNCH_CHECK();
    return PCCLB_OK;
  });
}

int pcclb_dequantize_ex(float *out, const void *codes, uint64_t n, const pcclb_qmeta *d_meta, uint32_t avg_div,
                        int qformat, void *stream) {
  if (qformat == PCCLB_Q_U8)
    return pcclb_dequantize_u8(out, static_cast<const uint8_t *>(codes), n, d_meta, avg_div, stream);
  if (!d_meta || (n && (!out || !codes)) || avg_div < 1) return PCCLB_EINVAL;
  if (n == 0) return PCCLB_OK;
  cudaStream_t s = as_stream(stream);
  const unsigned grid = grid_for(n, (uint64_t)kThreads * 8);
  return with_qformat(qformat, [&](auto qf) -> int {
    dequantize_q_kernel<decltype(qf)::value><<<grid, kThreads, 0, s>>>(out, codes, n, d_meta, avg_div);
    PCCLB_LAUNCH_CHECK();
    return PCCLB_OK;
  });
}

int pcclb_dequant_accumulate_ex(float *acc, const void *codes, uint64_t n, const pcclb_qmeta *d_meta, int op,
                                pcclb_range *d_next_range, int qformat, void *stream) {
  if (qformat == PCCLB_Q_U8)
    return pcclb_dequant_accumulate_u8(acc, static_cast<const uint8_t *>(codes), n, d_meta, op, d_next_range,
                                       stream);
  if (!d_meta || !valid_op(op) || (n && (!acc || !codes))) return PCCLB_EINVAL;
  if (n == 0) return PCCLB_OK;
  cudaStream_t s = as_stream(stream);
  const unsigned grid = grid_for(n, (uint64_t)kThreads * 8);
  return with_qformat(qformat, [&](auto qf) -> int {
    constexpr int QF = decltype(qf)::value;
    switch (op) {
      case PCCLB_MAX:
        dequant_acc_q_kernel<QF, PCCLB_MAX><<<grid, kThreads, 0, s>>>(acc, codes, n, d_meta, d_next_range);
        break;
      case PCCLB_MIN:
        dequant_acc_q_kernel<QF, PCCLB_MIN><<<grid, kThreads, 0, s>>>(acc, codes, n, d_meta, d_next_range);
        break;
      case PCCLB_PROD:
        dequant_acc_q_kernel<QF, PCCLB_PROD><<<grid, kThreads, 0, s>>>(acc, codes, n, d_meta, d_next_range);
        break;
      default:
        dequant_acc_q_kernel<QF, PCCLB_SUM><<<grid, kThreads, 0, s>>>(acc, codes, n, d_meta, d_next_range);
        break;
    }
    PCCLB_LAUNCH_CHECK();
    return PCCLB_OK;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Outer-optimizer steps around the all-reduce, with the
// reference's NumPy rounding sequence (algos.py:79-105, :236-239):
//   pseudo-gradient   delta = global - local
//   PlainSGD          params -= lr * grad                    (2 roundings)
//   NesterovOuter     v = v * mu; v = v + delta;
//                     params -= lr * (delta + mu * v)        (6 roundings, no FMA)
// ---------------------------------------------------------------------------
namespace pcclb {

struct SubF {  // out = a - b
  float *__restrict__ out;
  const float *__restrict__ a;
  const float *__restrict__ b;
  __device__ __forceinline__ void one(uint64_t i) { out[i] = x86_sub(a[i], b[i]); }
  struct In {
    Pack16<float> x, y;
  };
  __device__ __forceinline__ In vload(uint64_t i) { return In{ld16(a + i), ld16(b + i)}; }
  __device__ __forceinline__ void vapply(uint64_t i, const In &v) {
    Pack16<float> r;
#pragma unroll
    for (int k = 0; k < 4; ++k) r.e[k] = x86_sub(v.x.e[k], v.y.e[k]);
    st16(out + i, r);
  }
};

struct SgdF {  // p -= lr * g
  float *__restrict__ p;
  const float *__restrict__ g;
  float lr;
  __device__ __forceinline__ float upd(float pv, float gv) const { return x86_sub(pv, x86_mul(lr, gv)); }
  __device__ __forceinline__ void one(uint64_t i) { p[i] = upd(p[i], g[i]); }
  struct In {
    Pack16<float> p, g;
  };
  __device__ __forceinline__ In vload(uint64_t i) { return In{ld16(p + i), ld16(g + i)}; }
  __device__ __forceinline__ void vapply(uint64_t i, const In &v) {
    Pack16<float> r;
#pragma unroll
    for (int k = 0; k < 4; ++k) r.e[k] = upd(v.p.e[k], v.g.e[k]);
    st16(p + i, r);
  }
};

struct NesterovF {
  float *__restrict__ p;
  const float *__restrict__ d;
  float *__restrict__ vel;
  float lr, mu;
  __device__ __forceinline__ void upd(float &pv, float dv, float &vv) const {
    vv = x86_mul(vv, mu);
    vv = x86_add(vv, dv);
    pv = x86_sub(pv, x86_mul(lr, x86_add(dv, x86_mul(mu, vv))));
  }
  __device__ __forceinline__ void one(uint64_t i) {
    float pv = p[i], vv = vel[i];
    upd(pv, d[i], vv);
    p[i] = pv;
    vel[i] = vv;
  }
  struct In {
    Pack16<float> p, d, v;
  };
  __device__ __forceinline__ In vload(uint64_t i) { return In{ld16(p + i), ld16(d + i), ld16(vel + i)}; }
  __device__ __forceinline__ void vapply(uint64_t i, const In &in) {
    Pack16<float> pv = in.p, vv = in.v;
#pragma unroll
    for (int k = 0; k < 4; ++k) upd(pv.e[k], in.d.e[k], vv.e[k]);
    st16(p + i, pv);
    st16(vel + i, vv);
  }
};

template <typename F, int VEC>
__global__ void __launch_bounds__(kThreads, 4) functor_kernel(F f, uint64_t n, uint64_t head) {
  ew_loop<VEC, kUnroll>(n, head, f);
}

template <typename F>
static int launch_functor(F f, uint64_t n, bool vec, uint64_t head, cudaStream_t s) {
  if (n == 0) return PCCLB_OK;
  unsigned grid = grid_for(n, (uint64_t)kThreads * kUnroll * 4);
  if (vec)
    functor_kernel<F, 4><<<grid, kThreads, 0, s>>>(f, n, head);
  else
    functor_kernel<F, 1><<<grid, kThreads, 0, s>>>(f, n, 0);
  PCCLB_LAUNCH_CHECK();
  return PCCLB_OK;
}

}  // namespace pcclb

extern "C" {

int pcclb_pseudo_gradient_f32(float *delta, const float *global, const float *local, uint64_t n,
                              void *stream) {
  if (n && (!delta || !global || !local)) return PCCLB_EINVAL;
  const uint64_t h = peel16<float>(delta);
  const bool vec = peel16<float>(global) == h && peel16<float>(local) == h;
  return launch_functor(SubF{delta, global, local}, n, vec, h, as_stream(stream));
}

int pcclb_outer_sgd_f32(float *params, const float *grad, uint64_t n, float lr, void *stream) {
  if (n && (!params || !grad)) return PCCLB_EINVAL;
  const uint64_t h = peel16<float>(params);
  return launch_functor(SgdF{params, grad, lr}, n, peel16<float>(grad) == h, h, as_stream(stream));
}

int pcclb_outer_nesterov_f32(float *params, const float *delta, float *velocity, uint64_t n, float lr,
                             float momentum, void *stream) {
  if (n && (!params || !delta || !velocity)) return PCCLB_EINVAL;
  const uint64_t h = peel16<float>(params);
  const bool vec = peel16<float>(delta) == h && peel16<float>(velocity) == h;
  return launch_functor(NesterovF{params, delta, velocity, lr, momentum}, n, vec, h, as_stream(stream));
}

}  // extern "C"
