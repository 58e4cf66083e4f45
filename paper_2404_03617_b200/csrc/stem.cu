// stem.cu — the network's first unit (core.py:135-141; op count
// complexity.py:147-151), which the reference only costs: dense 3x3
// stride-2 conv (pad 1) from RGB + bias + phi. Each CTA owns R output rows;
// im2col rows (27 taps padded to K = 32) are assembled in shared memory and
// multiplied on tcgen05 (M = output pixels of a row, N = stem width).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include "common.cuh"
#include "plan.h"

namespace wl {

struct StemArgs {
  int H, W, Ho, Wo, Cs, Np, R, tiles_y;
  int s_in, s_a, s_w, s_bar, tmem_cols;
  const __half* x;          // (n, H, W, 3)
  const uint8_t* wpack;     // [B: Np x 32 core | bias fp32 Np]
  int w_bytes, o_bias;
  __half* z;                // (n, Ho, Wo, Cs)
};

template <int ACT>
__global__ void __launch_bounds__(256, 1) stem_kernel(const __grid_constant__ StemArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __half* s_in = reinterpret_cast<__half*>(smem + a.s_in);  // [(2R+1) rows][W][3]
  uint8_t* s_a = smem + a.s_a;                              // R tiles x [4][128][8]
  uint8_t* s_w = smem + a.s_w;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.s_bar);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int n = blockIdx.x / a.tiles_y, yo0 = (blockIdx.x % a.tiles_y) * a.R;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_n(tbase, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = *tbase;
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar[0], a.w_bytes);
    bulk_g2s(s_w, a.wpack, a.w_bytes, &bar[0]);
  }
  // input rows 2*yo0-1 .. 2*yo0+2R-1 (row -1 and rows >= H read as zero)
  const int rows = 2 * a.R + 1, row_vec = a.W * 3 * 2 / 16;  // 16-byte vectors per row
  for (int i = tid; i < rows * row_vec; i += blockDim.x) {
    const int rr = i / row_vec, v = i % row_vec, y = 2 * yo0 - 1 + rr;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (y >= 0 && y < a.H)
      val = reinterpret_cast<const uint4*>(a.x + ((size_t)n * a.H + y) * a.W * 3)[v];
    reinterpret_cast<uint4*>(s_in + (size_t)rr * a.W * 3)[v] = val;
  }
  __syncthreads();
  // im2col: tile t = output row yo0 + t, M row = output column
  for (int i = tid; i < a.R * 128; i += blockDim.x) {
    const int t = i / 128, xo = i % 128;
    float f[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) f[k] = 0.f;
    if (xo < a.Wo) {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int xx = 2 * xo - 1 + dx;
          if (xx < 0 || xx >= a.W) continue;
          const __half* px = s_in + ((size_t)(2 * t + dy) * a.W + xx) * 3;
#pragma unroll
          for (int c = 0; c < 3; ++c) f[(dy * 3 + dx) * 3 + c] = __half2float(px[c]);
        }
    }
#pragma unroll
    for (int k8 = 0; k8 < 4; ++k8)
      *reinterpret_cast<uint4*>(s_a + (size_t)t * 8192 + (k8 * 128 + xo) * 16) = pack8(f + 8 * k8);
  }
  fence_async_smem();
  __syncthreads();
  mbar_wait(&bar[0], 0);
  if (tid == 0) {
    tc_fence_after();
    const uint32_t idesc = make_idesc_f16(128, a.Np);
    for (int t = 0; t < a.R; ++t)
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t ad = make_sdesc(smem_u32(s_a) + t * 8192 + kk * 2 * 2048, 2048, 128);
        const uint64_t bd = make_sdesc(smem_u32(s_w) + kk * 2 * (a.Np * 16), a.Np * 16, 128);
        mma_ss(tmem + t * a.Np, ad, bd, idesc, kk > 0);
      }
    mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  const float* bias = reinterpret_cast<const float*>(s_w + a.o_bias);
  const int q = warp % 4;
  for (int t = warp / 4; t < a.R; t += 2) {
    const int xo = q * 32 + lane, yo = yo0 + t;
    for (int c0 = 0; c0 < a.Np; c0 += 16) {
      uint32_t v[16];
      WL_TMEM_LD16(tmem_lane_addr(tmem, q, t * a.Np + c0), v);
      tmem_ld_wait();
      if (xo >= a.Wo || yo >= a.Ho) continue;
      float f[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = act<ACT>(__uint_as_float(v[i]) + bias[c0 + i]);
      __half* zp = a.z + (((size_t)n * a.Ho + yo) * a.Wo + xo) * a.Cs + c0;
      for (int i = 0; i < 16 && c0 + i < a.Cs; i += 8) *reinterpret_cast<uint4*>(zp + i) = pack8(f + i);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc_n(tmem, a.tmem_cols);
}

}  // namespace wl

// =================================================================== host
#include <algorithm>
#include <cstring>
#include "launch.h"

namespace wl {
namespace {

constexpr int kSmemMaxSH = 232448;

// ------------------------------------------------------------------ stem
bool stem_plan(const wl_block_desc& d, StemArgs& a) {
  memset(&a, 0, sizeof(a));
  a.H = d.h;
  a.W = d.w;
  a.Ho = d.h / 2;
  a.Wo = d.w / 2;
  a.Cs = d.k;
  a.Np = align_up(d.k, 16);
  if (a.Wo > 128 || a.Np > 256 || d.k % 8 || (d.w * 3 * 2) % 16) return false;
  a.R = 4;  // measured: R = 2 and R = 8 are both slower (54-55 us vs 40 us at 224x224x16, b128)
  while (a.R * a.Np > 512) --a.R;
  a.tiles_y = (a.Ho + a.R - 1) / a.R;
  a.o_bias = a.Np * 32 * 2;
  a.w_bytes = align_up(a.o_bias + a.Np * 4, 16);
  int s = 0;
  a.s_a = s;
  s += a.R * 8192;
  a.s_in = s;
  s = align_up(s + (2 * a.R + 1) * a.W * 3 * 2, 128);
  a.s_w = s;
  s = align_up(s + a.w_bytes, 128);
  a.s_bar = s;
  a.tmem_cols = 32;
  while (a.tmem_cols < a.R * a.Np) a.tmem_cols *= 2;
  return true;
}
using StemK = void (*)(const StemArgs);
StemK stem_k(int act) {
  switch (act) {
    case kRelu: return stem_kernel<kRelu>;
    case kSilu: return stem_kernel<kSilu>;
    case kGelu: return stem_kernel<kGelu>;
    case kIdentity: return stem_kernel<kIdentity>;
  }
  return nullptr;
}
int stem_validate(const wl_block_desc& d) {
  if (d.n < 1 || d.h < 2 || d.w < 2 || d.k < 1) return set_error(WL_EINVAL, "dims must be positive");
  if (d.c != 3) return set_error(WL_EINVAL, "stem reads %d input channels; expected 3 (core.py:13)", d.c);
  if (d.h % 2 || d.w % 2) return set_error(WL_EINVAL, "stem stride 2 requires an even input resolution");
  if (!stem_k(d.act)) return set_error(WL_EUNSUPPORTED, "stem activation not supported");
  StemArgs a;
  if (!stem_plan(d, a)) return set_error(WL_EUNSUPPORTED, "no stem plan for %dx%d -> %d", d.h, d.w, d.k);
  return WL_OK;
}
int stem_wc(const wl_block_desc&) { return 2; }
int64_t stem_wn(const wl_block_desc& d, int i) {
  if (i == 0) return (int64_t)d.k * 27;
  if (i == 1) return d.k;
  return set_error(WL_EINVAL, "weight index out of range");
}
int64_t stem_pb(const wl_block_desc& d) {
  StemArgs a;
  stem_plan(d, a);
  return a.w_bytes;
}
int stem_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  StemArgs a;
  stem_plan(d, a);
  memset(out, 0, a.w_bytes);
  for (int n = 0; n < d.k; ++n)
    for (int k = 0; k < 27; ++k) put_h(out, core_off_h(n, k, a.Np * 16), w[0][(size_t)n * 27 + k]);
  float* b = reinterpret_cast<float*>(out + a.o_bias);
  for (int n = 0; n < d.k; ++n) b[n] = w[1][n];
  return WL_OK;
}
int64_t stem_ws(const wl_block_desc&) { return 0; }
int stem_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void*, cudaStream_t st) {
  StemArgs a;
  stem_plan(d, a);
  a.x = reinterpret_cast<const __half*>(x);
  a.wpack = reinterpret_cast<const uint8_t*>(p);
  a.z = reinterpret_cast<__half*>(z);
  return launch_pdl(stem_k(d.act), d.n * a.tiles_y, 256, a.s_bar + 64, st, "stem launch", a);
}
int stem_init() {
  for (int act : {kRelu, kSilu, kGelu, kIdentity})
    if (int e = check_cuda(cudaFuncSetAttribute(stem_k(act), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMaxSH),
                           "cudaFuncSetAttribute(stem)"))
      return e;
  return WL_OK;
}

}  // namespace

const Family kStemFamily = {stem_validate, stem_wc, stem_wn, stem_pb, stem_pack, stem_ws, stem_fwd, stem_init};

}  // namespace wl
