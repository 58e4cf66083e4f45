// common.cuh — element-wise helpers shared by the fused kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include "sm100.cuh"

namespace wl {

enum Act : int { kIdentity = 0, kRelu = 1, kSilu = 2, kSigmoid = 3, kGelu = 4 };

// phi of machine.py:178-188 (+ GELU, exact erf form), fp32 on CUDA cores
template <int ACT>
__device__ __forceinline__ float act(float v) {
  if constexpr (ACT == kRelu) return fmaxf(v, 0.f);
  if constexpr (ACT == kSilu) return __fdividef(v, 1.f + __expf(-v));
  if constexpr (ACT == kSigmoid) return __fdividef(1.f, 1.f + __expf(-v));
  if constexpr (ACT == kGelu) return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
  return v;
}

// ---- packed-half activations (2 values per instruction; MUFU tanh.approx)
// silu(x) = x/2 (1 + tanh(x/2)); sigmoid(x) = 1/2 + tanh(x/2)/2;
// gelu(x) ~= x/2 (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))  (tanh form)
__device__ __forceinline__ __half2 tanh_h2(__half2 x) {
  uint32_t r, v = *reinterpret_cast<uint32_t*>(&x);
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(v));
  return *reinterpret_cast<__half2*>(&r);
}
template <int ACT>
__device__ __forceinline__ __half2 act_h2(__half2 x) {
  if constexpr (ACT == kRelu) return __hmax2(x, __float2half2_rn(0.f));
  if constexpr (ACT == kSilu) {
    const __half2 h = __hmul2(x, __float2half2_rn(0.5f));
    return __hfma2(h, tanh_h2(h), h);
  }
  if constexpr (ACT == kSigmoid) {
    const __half2 h = __float2half2_rn(0.5f);
    return __hfma2(h, tanh_h2(__hmul2(x, h)), h);
  }
  if constexpr (ACT == kGelu) {
    const __half2 x2 = __hmul2(x, x);
    const __half2 p = __hfma2(x2, __float2half2_rn(0.0356774081f), __float2half2_rn(0.7978845608f));
    const __half2 h = __hmul2(x, __float2half2_rn(0.5f));
    return __hfma2(h, tanh_h2(__hmul2(x, p)), h);
  }
  return x;
}
// fp32 accumulators (+ fp32 bias) -> packed-half activation: 8 values -> uint4
// (bias is 16-byte aligned: two vector loads instead of eight scalar ones —
// each scalar load of a broadcast bias costs a shared-memory wavefront)
template <int ACT>
__device__ __forceinline__ uint4 bias_act8(const uint32_t* acc, const float* bias) {
  uint4 q;
  uint32_t* o = reinterpret_cast<uint32_t*>(&q);
  const float4 b0 = *reinterpret_cast<const float4*>(bias), b1 = *reinterpret_cast<const float4*>(bias + 4);
  const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __half2 h = __floats2half2_rn(__uint_as_float(acc[2 * i]) + bv[2 * i],
                                  __uint_as_float(acc[2 * i + 1]) + bv[2 * i + 1]);
    h = act_h2<ACT>(h);
    o[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return q;
}

// ---- warp-level tensor path (mma.sync): ldmatrix fragments and the two HMMA shapes
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
// D += A(16x16) B(16x8), fp16 operands, fp32 accumulators
__device__ __forceinline__ void hmma16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void hmma8(float* d, uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0));
}

// named barrier over n threads (multiple of 32)
__device__ __forceinline__ void nbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// 16-byte read-only global load the compiler may neither sink to its use nor
// re-issue there (a prefetch meant to hide L2 latency behind other work)
__device__ __forceinline__ uint4 ldg_pinned(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// 16 consecutive fp32 values (16-byte aligned) as four vector loads
__device__ __forceinline__ void load16f(const float* p, float* out) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 v = reinterpret_cast<const float4*>(p)[k];
    out[4 * k] = v.x;
    out[4 * k + 1] = v.y;
    out[4 * k + 2] = v.z;
    out[4 * k + 3] = v.w;
  }
}

// one 16-byte shared-memory load (keeps the compiler from splitting a uint4
// read through a generic pointer into four 4-byte LDS, each replayed 4x)
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
  return v;
}

__device__ __forceinline__ void unpack8(const uint4& q, float* f) {
  const __half2* h = reinterpret_cast<const __half2*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __half22float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 q;
  q.x = pack_h2(f[0], f[1]);
  q.y = pack_h2(f[2], f[3]);
  q.z = pack_h2(f[4], f[5]);
  q.w = pack_h2(f[6], f[7]);
  return q;
}

// ---- storage-type helpers (fp16 / bf16 activations and weights, fp32 math)
template <typename T>
struct Dt;
template <>
struct Dt<__half> {
  static constexpr uint32_t kIdescAB = 0;  // kind::f16 A / B format: f16
  static __device__ __forceinline__ uint32_t pack2(float a, float b) { return pack_h2(a, b); }
  static __device__ __forceinline__ float2 unpack2(uint32_t v) {
    return __half22float2(*reinterpret_cast<const __half2*>(&v));
  }
};
template <>
struct Dt<__nv_bfloat16> {
  static constexpr uint32_t kIdescAB = (1u << 7) | (1u << 10);  // A / B format: bf16
  static __device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ float2 unpack2(uint32_t v) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v));
  }
};
template <typename T>
__device__ __forceinline__ uint4 pack8t(const float* f) {
  return make_uint4(Dt<T>::pack2(f[0], f[1]), Dt<T>::pack2(f[2], f[3]), Dt<T>::pack2(f[4], f[5]),
                    Dt<T>::pack2(f[6], f[7]));
}
template <typename T>
__device__ __forceinline__ void unpack8t(const uint4& q, float* f) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = Dt<T>::unpack2(w[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
// bias-added pair -> activation -> packed storage: packed half math for fp16
// (MUFU tanh form), fp32 math for bf16
template <typename T, int ACT>
__device__ __forceinline__ uint32_t act_pack2(float a, float b) {
  if constexpr (sizeof(T) == 2 && Dt<T>::kIdescAB == 0) {
    const __half2 h = act_h2<ACT>(__floats2half2_rn(a, b));
    return *reinterpret_cast<const uint32_t*>(&h);
  } else {
    return Dt<T>::pack2(act<ACT>(a), act<ACT>(b));
  }
}

__device__ __forceinline__ uint32_t tmem_lane_addr(uint32_t base, int quad, int col) {
  return base + ((uint32_t)(quad * 32) << 16) + (uint32_t)col;
}

}  // namespace wl
