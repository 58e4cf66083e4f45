// common.cuh — element-wise helpers shared by the fused kernels.
#pragma once
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

__device__ __forceinline__ uint32_t tmem_lane_addr(uint32_t base, int quad, int col) {
  return base + ((uint32_t)(quad * 32) << 16) + (uint32_t)col;
}

}  // namespace wl
