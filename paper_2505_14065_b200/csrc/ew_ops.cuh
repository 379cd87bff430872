// Per-element functors of the quantization kernels, shared by the single-GPU
// seams (kernels.cu) and the NVLink ring (ring_ipc.cu). See ew_loop().
#pragma once

#include "elementwise.cuh"
#include "numerics.cuh"

namespace pcclb {

// ---------------------------------------------------------------------------
// K2 range
// ---------------------------------------------------------------------------
struct RangeF {
  const float *__restrict__ x;
  RangeAcc acc;
  __device__ __forceinline__ void one(uint64_t i) { acc.add(x[i]); }
  using In = Pack16<float>;
  __device__ __forceinline__ In vload(uint64_t i) { return ld16_cs(x + i); }
  __device__ __forceinline__ void vapply(uint64_t, const In &a) {
#pragma unroll
    for (int k = 0; k < 4; ++k) acc.add(a.e[k]);
  }
};

// ---------------------------------------------------------------------------
// K3/K6 quantize (+ optional adoption D(Q(x)) / avg_div)
// ---------------------------------------------------------------------------
struct QuantF {
  const float *__restrict__ x;
  uint8_t *__restrict__ codes;
  float *__restrict__ adopt;  // may alias x (adoption in place): same element, same thread
  QParams qp;
  float avg;  // 1 => no division
  bool do_div;
  __device__ __forceinline__ float adopt_val(uint32_t q) {
    float d = dequant1(q, qp.mn, qp.scale);
    return do_div ? div_world(d, avg) : d;
  }
  __device__ __forceinline__ void one(uint64_t i) {
    uint32_t q = quant1_fast(x[i], qp.mn, qp.scale, qp.inv);
    codes[i] = (uint8_t)q;
    if (adopt) adopt[i] = adopt_val(q);
  }
  using In = Pack16<float>;
  __device__ __forceinline__ In vload(uint64_t i) { return ld16(x + i); }
  __device__ __forceinline__ void vapply(uint64_t i, const In &a) {
    uint32_t q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = quant1_fast(a.e[k], qp.mn, qp.scale, qp.inv);
    *reinterpret_cast<uint32_t *>(codes + i) = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
    if (adopt) {
      Pack16<float> d;
#pragma unroll
      for (int k = 0; k < 4; ++k) d.e[k] = adopt_val(q[k]);
      st16(adopt + i, d);
    }
  }
};

// ---------------------------------------------------------------------------
// K4/K7 dequantize (+ optional AVG division)
// ---------------------------------------------------------------------------
struct DequantF {
  float *__restrict__ out;
  const uint8_t *__restrict__ codes;
  float mn, scale, avg;
  bool do_div;
  __device__ __forceinline__ float val(uint32_t q) {
    float d = dequant1(q, mn, scale);
    return do_div ? div_world(d, avg) : d;
  }
  __device__ __forceinline__ void one(uint64_t i) { out[i] = val(codes[i]); }
  using In = uint32_t;
  __device__ __forceinline__ In vload(uint64_t i) { return *reinterpret_cast<const uint32_t *>(codes + i); }
  __device__ __forceinline__ void vapply(uint64_t i, const In &q) {
    Pack16<float> d;
#pragma unroll
    for (int k = 0; k < 4; ++k) d.e[k] = val((q >> (8 * k)) & 0xffu);
    st16(out + i, d);
  }
};

// ---------------------------------------------------------------------------
// K5 dequant-accumulate (+ fused range of the result)
// ---------------------------------------------------------------------------
template <int OP>
struct DequantAccF {
  float *__restrict__ acc;
  const uint8_t *__restrict__ codes;
  float mn, scale;
  bool track;
  RangeAcc r;
  float *__restrict__ bak = nullptr;  // optional: save acc's old value first
  __device__ __forceinline__ float step(float local, uint32_t q) {
    float v = reduce_op<OP>(local, dequant1(q, mn, scale));
    if (track) r.add(v);
    return v;
  }
  __device__ __forceinline__ void one(uint64_t i) {
    const float old = acc[i];
    if (bak) bak[i] = old;
    acc[i] = step(old, codes[i]);
  }
  struct In {
    Pack16<float> a;
    uint32_t q;
  };
  __device__ __forceinline__ In vload(uint64_t i) {
    In v;
    v.a = ld16(acc + i);
    v.q = *reinterpret_cast<const uint32_t *>(codes + i);
    return v;
  }
  __device__ __forceinline__ void vapply(uint64_t i, const In &v) {
    Pack16<float> a = v.a;
    if (bak) st16(bak + i, a);
#pragma unroll
    for (int k = 0; k < 4; ++k) a.e[k] = step(a.e[k], (v.q >> (8 * k)) & 0xffu);
    st16(acc + i, a);
  }
};

// range of x, saving x into bak on the way (first read of a chunk)
struct RangeBakF {
  const float *__restrict__ x;
  float *__restrict__ bak;
  RangeAcc acc;
  __device__ __forceinline__ void one(uint64_t i) {
    const float v = x[i];
    bak[i] = v;
    acc.add(v);
  }
  using In = Pack16<float>;
  __device__ __forceinline__ In vload(uint64_t i) { return ld16(x + i); }
  __device__ __forceinline__ void vapply(uint64_t i, const In &a) {
    st16(bak + i, a);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc.add(a.e[k]);
  }
};

// plain copy src -> dst
struct CopyF {
  const float *__restrict__ src;
  float *__restrict__ dst;
  __device__ __forceinline__ void one(uint64_t i) { dst[i] = src[i]; }
  using In = Pack16<float>;
  __device__ __forceinline__ In vload(uint64_t i) { return ld16(src + i); }
  __device__ __forceinline__ void vapply(uint64_t i, const In &a) { st16(dst + i, a); }
};


// ---------------------------------------------------------------------------
// 16-element-wide forms for the NVLink ring: one 16-byte code load per 16
// floats keeps every remote request at 16 bytes per lane (u32 code loads
// gave ~460 GB/s over NVLink). Requires codes 16-byte aligned at the vector
// start (the ring places chunk codes at an offset congruent to the chunk's
// element offset modulo 16).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t code_byte(const uint4 &q, int k) {
  const uint32_t w = k < 4 ? q.x : k < 8 ? q.y : k < 12 ? q.z : q.w;
  return (w >> (8 * (k & 3))) & 0xffu;
}

template <int OP, bool X86 = true>
struct DequantAcc16F {
  float *__restrict__ acc;
  const uint8_t *__restrict__ codes;
  float mn, scale;
  RangeAcc r;
  float *__restrict__ bak;  // nullable: save acc's old value first
  __device__ __forceinline__ float step(float local, uint32_t q) {
    float v = reduce_op_x<OP, X86>(local, dequant1x<X86>(q, mn, scale));
    r.add(v);
    return v;
  }
  // codes are read with ld.global.cg (L2): a peer wrote them during this op
  __device__ __forceinline__ void one(uint64_t i) {
    const float old = acc[i];
    if (bak) bak[i] = old;
    acc[i] = step(old, __ldcg(codes + i));
  }
  struct In {
    Pack16<float> a[4];
    uint4 q;
  };
  __device__ __forceinline__ In vload(uint64_t i) {
    In v;
    v.q = __ldcg(reinterpret_cast<const uint4 *>(codes + i));
#pragma unroll
    for (int g = 0; g < 4; ++g) v.a[g] = ld16(acc + i + 4 * g);
    return v;
  }
  __device__ __forceinline__ void vapply(uint64_t i, const In &v) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      Pack16<float> a = v.a[g];
      if (bak) st16(bak + i + 4 * g, a);
#pragma unroll
      for (int k = 0; k < 4; ++k) a.e[k] = step(a.e[k], code_byte(v.q, 4 * g + k));
      st16(acc + i + 4 * g, a);
    }
  }
};

template <bool X86>
struct Dequant16T {
  float *__restrict__ out;
  const uint8_t *__restrict__ codes;
  float mn, scale, avg;
  bool do_div;
  __device__ __forceinline__ float val(uint32_t q) {
    float d = dequant1x<X86>(q, mn, scale);
    return do_div ? div_world_x<X86>(d, avg) : d;
  }
  __device__ __forceinline__ void one(uint64_t i) { out[i] = val(__ldcg(codes + i)); }
  using In = uint4;
  __device__ __forceinline__ In vload(uint64_t i) { return __ldcg(reinterpret_cast<const uint4 *>(codes + i)); }
  __device__ __forceinline__ void vapply(uint64_t i, const In &q) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      Pack16<float> d;
#pragma unroll
      for (int k = 0; k < 4; ++k) d.e[k] = val(code_byte(q, 4 * g + k));
      st16(out + i + 4 * g, d);
    }
  }
};

using Dequant16F = Dequant16T<true>;

// 4-element-wide form for local codes: a lane's 4-byte code load and 16-byte
// store are contiguous with its neighbours', so every store instruction
// writes whole sectors (the 16-wide form's four 16-byte stores per lane at a
// 64-byte stride measured ~25 % slower on this write-dominated stream)
template <bool X86>
struct Dequant4T {
  float *__restrict__ out;
  const uint8_t *__restrict__ codes;
  float mn, scale, avg;
  bool do_div;
  __device__ __forceinline__ float val(uint32_t q) {
    float d = dequant1x<X86>(q, mn, scale);
    return do_div ? div_world_x<X86>(d, avg) : d;
  }
  __device__ __forceinline__ void one(uint64_t i) { out[i] = val(__ldcg(codes + i)); }
  using In = uint32_t;
  __device__ __forceinline__ In vload(uint64_t i) { return __ldcg(reinterpret_cast<const uint32_t *>(codes + i)); }
  __device__ __forceinline__ void vapply(uint64_t i, In q) {
    Pack16<float> d;
#pragma unroll
    for (int k = 0; k < 4; ++k) d.e[k] = val((q >> (8 * k)) & 0xffu);
    st16(out + i, d);
  }
};

struct Quant16F {
  const float *__restrict__ x;
  uint8_t *__restrict__ codes;
  float *__restrict__ adopt;  // may alias x (adoption in place): same element, same thread
  QParams qp;
  float avg;
  bool do_div;
  __device__ __forceinline__ float adopt_val(uint32_t q) {
    float d = dequant1(q, qp.mn, qp.scale);
    return do_div ? div_world(d, avg) : d;
  }
  __device__ __forceinline__ void one(uint64_t i) {
    uint32_t q = quant1_fast(x[i], qp.mn, qp.scale, qp.inv);
    codes[i] = (uint8_t)q;
    if (adopt) adopt[i] = adopt_val(q);
  }
  struct In {
    Pack16<float> a[4];
  };
  __device__ __forceinline__ In vload(uint64_t i) {
    In v;
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
      for (int k = 0; k < 4; ++k) q[k] = quant1_fast(v.a[g].e[k], qp.mn, qp.scale, qp.inv);
      w[g] = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
      if (adopt) {
        Pack16<float> d;
#pragma unroll
        for (int k = 0; k < 4; ++k) d.e[k] = adopt_val(q[k]);
        st16(adopt + i + 4 * g, d);
      }
    }
    *reinterpret_cast<uint4 *>(codes + i) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};

// elements to peel before a float pointer is 64-byte aligned (16 floats)
__device__ __forceinline__ uint64_t dpeel64f(const float *p) {
  const uintptr_t x = reinterpret_cast<uintptr_t>(p);
  return (uint64_t)(((64 - (x & 63)) & 63) / 4);
}

}  // namespace pcclb
