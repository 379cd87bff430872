// Element arithmetic that reproduces the reference's NumPy results bit for bit.
//
// The reference computes with NumPy ufuncs on x86 (collective.py:66-71,
// :119-135, :479-482). Probed behaviour (NumPy 2.3.5, see DESIGN.md
// §Numerics and tests/golden/edges.npz):
//   * add/sub/mul/div: IEEE binary32/64 round-to-nearest, no contraction, no
//     FTZ. A NaN operand propagates quieted (first operand wins); an invalid
//     operation yields the x86 default NaN (0xffc00000 / 0xfff8000000000000),
//     not the CUDA canonical 0x7fffffff.
//   * np.maximum(a, b): a if a > b or a is NaN, else b  -> ties and a NaN b
//     return b (the incoming operand); NaN returned unquieted.
//   * np.minimum(a, b): a if a < b or a is NaN, else b.
//   * rint: ties-to-even; f32 -> u8 cast of NaN gives 0 (cvttss2si path).
// The library is compiled with -fmad=false -prec-div=true -ftz=false; the
// explicit _rn intrinsics below keep that true regardless of flags.
#pragma once

#include <stdint.h>
#include <string.h>

#include <type_traits>

#include "pcclb200.h"

namespace pcclb {

template <typename T>
struct FTraits;
template <>
struct FTraits<float> {
  using U = uint32_t;
  static constexpr U kQuiet = 0x00400000u;
  static constexpr U kDefaultNaN = 0xffc00000u;
  static __device__ __forceinline__ U bits(float x) { return __float_as_uint(x); }
  static __device__ __forceinline__ float from(U u) { return __uint_as_float(u); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
};
template <>
struct FTraits<double> {
  using U = unsigned long long;
  static constexpr U kQuiet = 0x0008000000000000ull;
  static constexpr U kDefaultNaN = 0xfff8000000000000ull;
  static __device__ __forceinline__ U bits(double x) { return (U)__double_as_longlong(x); }
  static __device__ __forceinline__ double from(U u) { return __longlong_as_double((long long)u); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};

template <typename T>
__device__ __forceinline__ bool is_nan(T x) {
  return x != x;
}

template <typename T>
__device__ __forceinline__ T quiet(T x) {
  using F = FTraits<T>;
  return F::from(F::bits(x) | F::kQuiet);
}

// NaN result of a binary x86 SSE operation: first NaN operand quieted, else
// the default NaN (invalid operation).
template <typename T>
__device__ __noinline__ T x86_nan_result(T a, T b) {
  if (is_nan(a)) return quiet(a);
  if (is_nan(b)) return quiet(b);
  return FTraits<T>::from(FTraits<T>::kDefaultNaN);
}

template <typename T>
__device__ __forceinline__ T x86_add(T a, T b) {
  T r = FTraits<T>::add(a, b);
  if (__builtin_expect(is_nan(r), 0)) r = x86_nan_result(a, b);
  return r;
}
template <typename T>
__device__ __forceinline__ T x86_sub(T a, T b) {
  T r = FTraits<T>::sub(a, b);
  if (__builtin_expect(is_nan(r), 0)) r = x86_nan_result(a, b);
  return r;
}
template <typename T>
__device__ __forceinline__ T x86_mul(T a, T b) {
  T r = FTraits<T>::mul(a, b);
  if (__builtin_expect(is_nan(r), 0)) r = x86_nan_result(a, b);
  return r;
}
template <typename T>
__device__ __forceinline__ T x86_div(T a, T b) {
  T r = FTraits<T>::div(a, b);
  if (__builtin_expect(is_nan(r), 0)) r = x86_nan_result(a, b);
  return r;
}
// AVG finalize x / W (collective.py:482). For a power-of-two W the quotient is
// x * 2^-k exactly (the same real value rounded once, also for subnormal
// results), which avoids the IEEE division sequence; other W divide.
__device__ __forceinline__ float div_world(float x, float w) {
  const uint32_t b = __float_as_uint(w);
  if ((b & 0x007fffffu) == 0u) return x86_mul(x, __uint_as_float((254u << 23) - b));
  return x86_div(x, w);
}
__device__ __forceinline__ double div_world(double x, double w) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(w);
  if ((b & 0x000fffffffffffffull) == 0ull)
    return x86_mul(x, __longlong_as_double((long long)((2046ull << 52) - b)));
  return x86_div(x, w);
}

// np.maximum / np.minimum (collective.py:69-70)
template <typename T>
__device__ __forceinline__ T np_maximum(T a, T b) {
  return (a > b || is_nan(a)) ? a : b;
}
template <typename T>
__device__ __forceinline__ T np_minimum(T a, T b) {
  return (a < b || is_nan(a)) ? a : b;
}

// accumulate(local, incoming) for a reduce op code (AVG accumulates with add)
template <int OP, typename T>
__device__ __forceinline__ T reduce_op(T local, T incoming) {
  if constexpr (OP == PCCLB_MAX) {
    return np_maximum(local, incoming);
  } else if constexpr (OP == PCCLB_MIN) {
    return np_minimum(local, incoming);
  } else if constexpr (OP == PCCLB_PROD) {
    return x86_mul(local, incoming);  // np.multiply (extension op)
  } else {
    return x86_add(local, incoming);
  }
}

// ---------------------------------------------------------------------------
// bf16 buffers (extension: the reference's collectives take f32/f64 only,
// collective.py:73-74, so the definition is this repo's, oracle/bf16.py):
// every fold step computes in f32 with the rules above and rounds the result
// to bf16 (round to nearest even; a NaN keeps sign and payload, quieted);
// np.maximum/np.minimum select one of the two bf16 operands unchanged.
// ---------------------------------------------------------------------------
struct Bf16 {
  uint16_t b;
  Bf16() = default;
  // the world size as a bf16 (exact for W <= 256)
  __host__ __device__ explicit Bf16(uint32_t w) {
    float f = (float)w;
    uint32_t u;
    memcpy(&u, &f, 4);
    b = (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
  }
};

__device__ __forceinline__ float bf16_to_f32(Bf16 x) { return __uint_as_float((uint32_t)x.b << 16); }
__device__ __forceinline__ Bf16 f32_to_bf16(float f) {
  const uint32_t u = __float_as_uint(f);
  Bf16 r;
  if ((u & 0x7fffffffu) > 0x7f800000u) r.b = (uint16_t)((u >> 16) | 0x0040u);  // NaN: quieted
  else r.b = (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);              // RNE
  return r;
}
template <>
__device__ __forceinline__ bool is_nan<Bf16>(Bf16 x) {
  return (x.b & 0x7fffu) > 0x7f80u;
}

template <int OP>
__device__ __forceinline__ Bf16 reduce_op(Bf16 local, Bf16 incoming) {
  const float a = bf16_to_f32(local), b = bf16_to_f32(incoming);
  if constexpr (OP == PCCLB_MAX) return (a > b || is_nan(a)) ? local : incoming;
  else if constexpr (OP == PCCLB_MIN) return (a < b || is_nan(a)) ? local : incoming;
  else if constexpr (OP == PCCLB_PROD) return f32_to_bf16(x86_mul(a, b));
  else return f32_to_bf16(x86_add(a, b));
}
__device__ __forceinline__ Bf16 div_world(Bf16 x, Bf16 w) {
  return f32_to_bf16(div_world(bf16_to_f32(x), bf16_to_f32(w)));
}

// ---------------------------------------------------------------------------
// quantization (collective.py:109-135)
// ---------------------------------------------------------------------------
// order-preserving key of a float (-0 sorts just below +0)
__device__ __forceinline__ uint32_t fkey(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey_decode(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ bool finite_f(float x) { return fabsf(x) <= 3.402823466e38f; }

struct QParams {
  float mn;
  float scale;
  float inv;  // fl(1 / scale): fast path of quant1 (exactness-guarded)
};

// (min, scale) from a span range: scale = (max - min) / 255f, 1 when 0.
// Empty span -> (0, 1) (collective.py:115-116).
__device__ __forceinline__ QParams qparams_from_range(const pcclb_range &r) {
  QParams q;
  if (!r.seen) {
    q.mn = 0.0f;
    q.scale = 1.0f;
    q.inv = 1.0f;
    return q;
  }
  float mn = fkey_decode(~r.kmin_inv);
  float mx = fkey_decode(r.kmax);
  float s = x86_div(x86_sub(mx, mn), 255.0f);
  if (s == 0.0f) s = 1.0f;
  q.mn = mn;
  q.scale = s;
  q.inv = __fdiv_rn(1.0f, s);
  return q;
}

// q = u8(clip(rint((x - min) / scale), 0, 255)); NaN -> 0. A NaN's payload
// never reaches the code, so plain IEEE operations give the reference's codes.
__device__ __forceinline__ uint32_t quant1(float x, float mn, float scale) {
  float t = __fdiv_rn(__fsub_rn(x, mn), scale);
  t = rintf(t);
  if (is_nan(t)) return 0u;
  t = fminf(fmaxf(t, 0.0f), 255.0f);
  return (uint32_t)t;
}

// out-of-line exact path: keeps the division sequence's registers out of the
// hot loops (72 -> fewer registers per thread, higher occupancy)
static __device__ __noinline__ uint32_t quant1_exact(float x, float mn, float scale) {
  return quant1(x, mn, scale);
}

// Same result without a division per element. t = d * fl(1/scale) is within
// ~2^-22 (relative) of fl(d / scale); rint can only differ if a half-integer
// lies that close, so t is used unless its fractional part is within 2^-20
// (relative) of 0.5, where the exact division decides. Non-finite t (d or
// 1/scale overflowing) also takes the exact path.
__device__ __forceinline__ uint32_t quant1_fast(float x, float mn, float scale, float inv) {
  const float d = __fsub_rn(x, mn);
  const float t = __fmul_rn(d, inv);
  const float fl = floorf(t);
  const float h = __fsub_rn(t, fl);            // exact for t < 2^23
  const float m = fabsf(__fsub_rn(h, 0.5f));   // distance to the half-integer
  if (__builtin_expect(m > __fmul_rn(t, 1e-6f) + 1e-30f, 1)) {
    float q = (h > 0.5f) ? __fadd_rn(fl, 1.0f) : fl;
    q = fminf(fmaxf(q, 0.0f), 255.0f);
    return (uint32_t)q;
  }
  return quant1_exact(x, mn, scale);
}

// ---------------------------------------------------------------------------
// quantization formats beyond the reference's u8 min-max (extensions, see
// pcclb200.h PCCLB_Q_*): qparams_q / quantq / dequantq. For PCCLB_Q_U8 they
// are exactly qparams_from_range / quant1_fast / dequant1.
// ---------------------------------------------------------------------------
template <int QF>
struct QFmt {
  static constexpr float kLevels = (QF == PCCLB_Q_U16 || QF == PCCLB_Q_U16_ZP) ? 65535.0f : 255.0f;
  static constexpr bool kZp = QF == PCCLB_Q_U8_ZP || QF == PCCLB_Q_U16_ZP;
  using Code = typename std::conditional<(QF == PCCLB_Q_U16 || QF == PCCLB_Q_U16_ZP), uint16_t, uint8_t>::type;
};

// round t (finite or not) to an integer code in [0, L]; NaN -> 0
template <int QF>
__device__ __forceinline__ uint32_t clip_code(float t) {
  if (is_nan(t)) return 0u;
  return (uint32_t)fminf(fmaxf(t, 0.0f), QFmt<QF>::kLevels);
}

// QParams.mn holds the minimum (min-max) or the zero point (as a float)
template <int QF>
__device__ __forceinline__ QParams qparams_q(const pcclb_range &r) {
  if constexpr (QF == PCCLB_Q_U8) {
    return qparams_from_range(r);
  } else {
    QParams q;
    if (!r.seen) {
      q.mn = 0.0f;
      q.scale = 1.0f;
      q.inv = 1.0f;
      return q;
    }
    float mn = fkey_decode(~r.kmin_inv), mx = fkey_decode(r.kmax);
    if constexpr (QFmt<QF>::kZp) {
      // the range is widened to include 0, which the zero point then encodes
      // exactly (asymmetric affine quantization, like PyTorch's MinMaxObserver)
      mn = fminf(mn, 0.0f);
      mx = fmaxf(mx, 0.0f);
    }
    float s = x86_div(x86_sub(mx, mn), QFmt<QF>::kLevels);
    if (s == 0.0f) s = 1.0f;
    q.scale = s;
    q.inv = __fdiv_rn(1.0f, s);
    if constexpr (QFmt<QF>::kZp) q.mn = (float)clip_code<QF>(rintf(__fdiv_rn(-mn, s)));
    else q.mn = mn;
    return q;
  }
}

template <int QF>
__device__ __noinline__ uint32_t quantq_exact(float x, float mn, float scale) {
  if constexpr (QFmt<QF>::kZp) return clip_code<QF>(__fadd_rn(rintf(__fdiv_rn(x, scale)), mn));
  else return clip_code<QF>(rintf(__fdiv_rn(__fsub_rn(x, mn), scale)));
}

// exactness-guarded reciprocal like quant1_fast: the product is used unless
// it lies within ~2^-20 (relative) of a half-integer
template <int QF>
__device__ __forceinline__ uint32_t quantq(float x, const QParams &qp) {
  if constexpr (QF == PCCLB_Q_U8) {
    return quant1_fast(x, qp.mn, qp.scale, qp.inv);
  } else {
    const float d = QFmt<QF>::kZp ? x : __fsub_rn(x, qp.mn);
    const float t = __fmul_rn(d, qp.inv);
    const float fl = floorf(t);
    const float h = __fsub_rn(t, fl);
    const float m = fabsf(__fsub_rn(h, 0.5f));
    if (__builtin_expect(m > __fmul_rn(fabsf(t), 1e-6f) + 1e-30f && fabsf(t) < 8388608.0f, 1)) {
      float q = (h > 0.5f) ? __fadd_rn(fl, 1.0f) : fl;
      if constexpr (QFmt<QF>::kZp) q = __fadd_rn(q, qp.mn);
      return clip_code<QF>(q);
    }
    return quantq_exact<QF>(x, qp.mn, qp.scale);
  }
}

template <int QF>
__device__ __forceinline__ float dequantq(uint32_t q, const QParams &qp) {
  if constexpr (QFmt<QF>::kZp) return x86_mul(__fsub_rn((float)q, qp.mn), qp.scale);
  else return x86_add(x86_mul((float)q, qp.scale), qp.mn);
}

// x = f32(q) * scale (RN) + min (RN), x86 NaN rules
__device__ __forceinline__ float dequant1(uint32_t q, float mn, float scale) {
  return x86_add(x86_mul((float)q, scale), mn);
}
// X86 = false: plain IEEE operations, for kernels where a NaN cannot occur
// (finite scale and min) or can only occur in an op that is then aborted and
// restored (any NaN in a partial sum makes the next range non-finite), so
// the x86 payload rules cannot change a delivered result
template <bool X86>
__device__ __forceinline__ float dequant1x(uint32_t q, float mn, float scale) {
  if constexpr (X86) return dequant1(q, mn, scale);
  else return __fadd_rn(__fmul_rn((float)q, scale), mn);
}
template <bool X86>
__device__ __forceinline__ float div_world_x(float x, float w) {
  if constexpr (X86) {
    return div_world(x, w);
  } else {
    const uint32_t b = __float_as_uint(w);
    if ((b & 0x007fffffu) == 0u) return __fmul_rn(x, __uint_as_float((254u << 23) - b));
    return __fdiv_rn(x, w);
  }
}
template <int OP, bool X86, typename T>
__device__ __forceinline__ T reduce_op_x(T local, T incoming) {
  if constexpr (X86 || OP == PCCLB_MAX || OP == PCCLB_MIN) return reduce_op<OP>(local, incoming);
  else if constexpr (OP == PCCLB_PROD) return FTraits<T>::mul(local, incoming);
  else return FTraits<T>::add(local, incoming);
}

// block-wide range accumulation helpers
struct RangeAcc {
  uint32_t kmin_inv = 0;
  uint32_t kmax = 0;
  uint32_t nonfinite = 0;
  uint32_t seen = 0;
  __device__ __forceinline__ void add(float x) {
    uint32_t k = fkey(x);
    kmin_inv = max(kmin_inv, ~k);
    kmax = max(kmax, k);
    nonfinite |= finite_f(x) ? 0u : 1u;
    seen = 1u;
  }
};

// reduce a RangeAcc over the block and fold it into *dst with atomics
__device__ __forceinline__ void range_block_commit(RangeAcc a, pcclb_range *dst) {
  __shared__ uint32_t s_inv[32], s_max[32], s_nf[32], s_seen[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a.kmin_inv = max(a.kmin_inv, __shfl_xor_sync(0xffffffffu, a.kmin_inv, o));
    a.kmax = max(a.kmax, __shfl_xor_sync(0xffffffffu, a.kmax, o));
    a.nonfinite |= __shfl_xor_sync(0xffffffffu, a.nonfinite, o);
    a.seen |= __shfl_xor_sync(0xffffffffu, a.seen, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) {
    s_inv[warp] = a.kmin_inv;
    s_max[warp] = a.kmax;
    s_nf[warp] = a.nonfinite;
    s_seen[warp] = a.seen;
  }
  __syncthreads();
  if (warp == 0) {
    RangeAcc b;
    if (lane < nw) {
      b.kmin_inv = s_inv[lane];
      b.kmax = s_max[lane];
      b.nonfinite = s_nf[lane];
      b.seen = s_seen[lane];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      b.kmin_inv = max(b.kmin_inv, __shfl_xor_sync(0xffffffffu, b.kmin_inv, o));
      b.kmax = max(b.kmax, __shfl_xor_sync(0xffffffffu, b.kmax, o));
      b.nonfinite |= __shfl_xor_sync(0xffffffffu, b.nonfinite, o);
      b.seen |= __shfl_xor_sync(0xffffffffu, b.seen, o);
    }
    if (lane == 0 && b.seen) {
      atomicMax(&dst->kmin_inv, b.kmin_inv);
      atomicMax(&dst->kmax, b.kmax);
      if (b.nonfinite) atomicOr(&dst->nonfinite, 1u);
      atomicOr(&dst->seen, 1u);
    }
  }
}

}  // namespace pcclb
