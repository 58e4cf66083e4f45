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
  int H, W, Ho, Wo, Cs, Np, R, tiles_y, nbands;
  int s_in, s_a, s_w, s_bar, tmem_cols, in_bytes, a_bytes;
  const __half* x;          // (n, H, W, 3)
  const uint8_t* wpack;     // [B: Np x 32 core | bias fp32 Np]
  int w_bytes, o_bias;
  __half* z;                // (n, Ho, Wo, Cs)
};

namespace stk {
constexpr int kNB = 3;  // input-row ring depth
struct Bars {
  uint64_t w_full, in_full[kNB], in_empty[kNB], a_full[2], mma_done[2];
  uint32_t tmem_base;
};
}  // namespace stk

// Persistent: each CTA walks bands of R output rows (stride gridDim). The
// band's 2R+1 input rows (contiguous in NHWC) arrive by ONE bulk copy, two
// bands ahead; im2col tiles and TMEM accumulators are double-buffered so the
// MMA of band b overlaps the epilogue of band b-1 and the loads run ahead.
template <int ACT>
__global__ void __launch_bounds__(256, 1) stem_kernel(const __grid_constant__ StemArgs a) {
  using namespace stk;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_in = smem + a.s_in;  // kNB x [(2R+1) rows][W][3]
  uint8_t* s_a = smem + a.s_a;    // 2 x R tiles x [4][128][8]
  uint8_t* s_w = smem + a.s_w;
  Bars& B = *reinterpret_cast<Bars*>(smem + a.s_bar);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int nb = a.nbands > (int)blockIdx.x ? (a.nbands - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int rows = 2 * a.R + 1, row_bytes = a.W * 6;
  if (tid == 0) {
    mbar_init(&B.w_full, 1);
    for (int i = 0; i < kNB; ++i) {
      mbar_init(&B.in_full[i], 1);
      mbar_init(&B.in_empty[i], 256);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.a_full[i], 256);
      mbar_init(&B.mma_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_n(&B.tmem_base, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  const uint32_t tmem = B.tmem_base;
  auto band_of = [&](int i, int& n, int& yo0) {
    const int band = (int)blockIdx.x + i * (int)gridDim.x;
    n = band / a.tiles_y;
    yo0 = (band % a.tiles_y) * a.R;
  };
  // rows [y0, y1) of the band that exist in the image; slot row r <-> input row 2*yo0 - 1 + r
  auto load = [&](int i) {
    const int sl = i % kNB;
    if (i >= kNB) mbar_wait(&B.in_empty[sl], ((i / kNB) - 1) & 1);
    int n, yo0;
    band_of(i, n, yo0);
    const int ya = max(0, 2 * yo0 - 1), yb = min(a.H, 2 * yo0 - 1 + rows);
    const uint32_t bytes = (uint32_t)(yb - ya) * row_bytes;
    mbar_arrive_expect_tx(&B.in_full[sl], bytes);
    bulk_g2s(s_in + sl * a.in_bytes + (size_t)(ya - (2 * yo0 - 1)) * row_bytes,
             a.x + ((size_t)n * a.H + ya) * a.W * 3, bytes, &B.in_full[sl]);
  };
  if (tid == 0) {
    mbar_arrive_expect_tx(&B.w_full, a.w_bytes);
    bulk_g2s(s_w, a.wpack, a.w_bytes, &B.w_full);
    for (int i = 0; i < nb && i < kNB - 1; ++i) load(i);
  }
  const float* bias = reinterpret_cast<const float*>(s_w + a.o_bias);
  const int q = warp % 4;
  auto epilogue = [&](int i) {
    const int ab = i & 1;
    mbar_wait(&B.mma_done[ab], (i >> 1) & 1);
    tc_fence_after();
    int n, yo0;
    band_of(i, n, yo0);
    for (int t = warp / 4; t < a.R; t += 2) {
      const int xo = q * 32 + lane, yo = yo0 + t;
      for (int c0 = 0; c0 < a.Np; c0 += 16) {
        uint32_t v[16];
        WL_TMEM_LD16(tmem_lane_addr(tmem, q, (ab * a.R + t) * a.Np + c0), v);
        tmem_ld_wait();
        if (xo >= a.Wo || yo >= a.Ho) continue;
        float f[16], b16[16];
        load16f(bias + c0, b16);
#pragma unroll
        for (int k = 0; k < 16; ++k) f[k] = act<ACT>(__uint_as_float(v[k]) + b16[k]);
        __half* zp = a.z + (((size_t)n * a.Ho + yo) * a.Wo + xo) * a.Cs + c0;
        for (int k = 0; k < 16 && c0 + k < a.Cs; k += 8) *reinterpret_cast<uint4*>(zp + k) = pack8(f + k);
      }
    }
    tc_fence_before();
  };
  mbar_wait(&B.w_full, 0);
  for (int i = 0; i < nb; ++i) {
    if (tid == 0 && i + kNB - 1 < nb) load(i + kNB - 1);
    const int sl = i % kNB, ab = i & 1;
    int n, yo0;
    band_of(i, n, yo0);
    mbar_wait(&B.in_full[sl], (i / kNB) & 1);
    const uint8_t* in = s_in + sl * a.in_bytes;
    // im2col: tile t = output row yo0 + t, M row = output column; rows outside
    // the image (y < 0 or y >= H) are never loaded and read as zero
    const int ylo = 1 - 2 * yo0, yhi = a.H - (2 * yo0 - 1);  // valid slot rows [ylo, yhi)
    uint8_t* sa = s_a + ab * a.a_bytes;
    for (int it = tid; it < a.R * 128; it += 256) {
      const int t = it >> 7, xo = it & 127;
      float f[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) f[k] = 0.f;
      if (xo < a.Wo) {
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
          const int r = 2 * t + dy;
          if (r < ylo || r >= yhi) continue;
          const __half* rowp = reinterpret_cast<const __half*>(in + (size_t)r * row_bytes);
          // the row's 9 halves (dx = -1..1 x 3 channels) start at half 6xo - 3: five
          // aligned 32-bit words from half 6xo - 4 cover them (the words left of the
          // image at xo = 0 are the zero padding) — 5 loads instead of 9
          const int h0 = 6 * xo - 4;
          float hv[10];
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            uint32_t wv = 0u;
            if (h0 + 2 * k >= 0) wv = *reinterpret_cast<const uint32_t*>(rowp + h0 + 2 * k);
            const float2 t2 = __half22float2(*reinterpret_cast<const __half2*>(&wv));
            hv[2 * k] = t2.x;
            hv[2 * k + 1] = t2.y;
          }
#pragma unroll
          for (int k = 0; k < 9; ++k) f[dy * 9 + k] = hv[k + 1];
        }
      }
#pragma unroll
      for (int k8 = 0; k8 < 4; ++k8)
        *reinterpret_cast<uint4*>(sa + (size_t)t * 8192 + (k8 * 128 + xo) * 16) = pack8(f + 8 * k8);
    }
    mbar_arrive(&B.in_empty[sl]);
    fence_async_smem();
    mbar_arrive(&B.a_full[ab]);
    if (tid == 32) {  // MMA issue for band i (its accumulators were drained by epilogue(i-2))
      mbar_wait(&B.a_full[ab], (i >> 1) & 1);
      tc_fence_after();
      const uint32_t idesc = make_idesc_f16(128, a.Np);
      for (int t = 0; t < a.R; ++t)
        for (int kk = 0; kk < 2; ++kk) {
          const uint64_t ad = make_sdesc(smem_u32(sa) + t * 8192 + kk * 2 * 2048, 2048, 128);
          const uint64_t bd = make_sdesc(smem_u32(s_w) + kk * 2 * (a.Np * 16), a.Np * 16, 128);
          mma_ss(tmem + (ab * a.R + t) * a.Np, ad, bd, idesc, kk > 0);
        }
      mma_commit(&B.mma_done[ab]);
    }
    if (i > 0) epilogue(i - 1);  // overlaps MMA(i)
    // s_a[ab ^ 1] is rewritten by im2col(i+1): epilogue(i-1) waited for MMA(i-1)
  }
  if (nb > 0) epilogue(nb - 1);
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
  a.R = 4;
  while (2 * a.R * a.Np > 512) --a.R;
  a.tiles_y = (a.Ho + a.R - 1) / a.R;
  a.nbands = d.n * a.tiles_y;
  a.o_bias = a.Np * 32 * 2;
  a.w_bytes = align_up(a.o_bias + a.Np * 4, 16);
  a.in_bytes = align_up((2 * a.R + 1) * a.W * 3 * 2, 128);
  a.a_bytes = a.R * 8192;
  int s = 0;
  a.s_a = s;
  s += 2 * a.a_bytes;
  a.s_in = s;
  s = align_up(s + stk::kNB * a.in_bytes, 128);
  a.s_w = s;
  s = align_up(s + a.w_bytes, 128);
  a.s_bar = s;
  a.tmem_cols = 32;
  while (a.tmem_cols < 2 * a.R * a.Np) a.tmem_cols *= 2;
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
  return launch_pdl(stem_k(d.act), std::min(a.nbands, 2 * kNumSMs), 256, a.s_bar + 128, st, "stem launch", a);
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
