// stem_head.cu — the network's first and last units (core.py:135-152; op
// counts complexity.py:147-157), which the reference only costs:
//   stem : dense 3x3 stride-2 conv (pad 1) from RGB + bias + phi. Each CTA
//          owns R output rows; im2col rows (27 taps padded to K = 32) are
//          assembled in shared memory and multiplied on tcgen05 (M = output
//          pixels of a row, N = stem width).
//   head : 1x1 conv to the embedding + bias + phi and the global average pool
//          fused in one kernel (the embedding never reaches HBM), then the
//          linear classifier as a second tcgen05 GEMM over the pooled batch.
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

// ---------------------------------------------------------------- head
// kernel 1: CTA = group of images (imgs * HW <= 128 pixels). embed in chunks
// of NE; z1 = phi(x W1 + b1) in TMEM; per-image column sums -> feat (fp16).
struct HeadArgs {
  int C, E, M, HW, imgs, P, NE, nce, npair;
  int s_a, s_w, s_pool, s_bar, tmem_cols, w1_chunk, o_b1;
  const uint8_t* w1;  // [b1 fp32 E (padded)][chunks: NE x C core]
  __half* feat;       // (n, E) pooled embedding
};

template <int ACT>
__global__ void __launch_bounds__(256, 1) head_pool_kernel(const __grid_constant__ CUtensorMap tmap_x,
                                                           const __grid_constant__ HeadArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_a = smem + a.s_a;  // [C/8][128][8]
  uint8_t* s_w = smem + a.s_w;  // 2 x chunk
  float* s_pool = reinterpret_cast<float*>(smem + a.s_pool);  // [imgs][NE]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.s_bar);  // 0 x, 1 mma, 2..3 w
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 4);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, q = warp % 4, half = warp / 4;
  const int p0 = blockIdx.x * a.imgs * a.HW;
  const float* b1 = reinterpret_cast<const float*>(a.w1 + a.o_b1);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_n(tbase, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  const uint8_t* chunks = a.w1 + a.o_b1 + align_up(a.E * 4, 128);
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar[0], 128 * a.C * 2);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(s_a)),
        "l"(&tmap_x), "r"(0), "r"(p0), "r"(0), "r"(smem_u32(&bar[0]))
        : "memory");
    mbar_arrive_expect_tx(&bar[2], a.w1_chunk);
    bulk_g2s(s_w, chunks, a.w1_chunk, &bar[2]);
  }
  const int npix = a.imgs * a.HW;
  for (int j = 0; j < a.nce; ++j) {
    for (int i = tid; i < a.imgs * a.NE; i += blockDim.x) s_pool[i] = 0.f;
    if (tid == 0) {
      if (j + 1 < a.nce) {  // prefetch next chunk into the other buffer (free: its MMA finished last iteration)
        mbar_arrive_expect_tx(&bar[2 + ((j + 1) & 1)], a.w1_chunk);
        bulk_g2s(s_w + ((j + 1) & 1) * a.w1_chunk, chunks + (size_t)(j + 1) * a.w1_chunk, a.w1_chunk,
                 &bar[2 + ((j + 1) & 1)]);
      }
      mbar_wait(&bar[0], 0);
      mbar_wait(&bar[2 + (j & 1)], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t idesc = make_idesc_f16(128, a.NE);
      const uint32_t wb = smem_u32(s_w) + (j & 1) * a.w1_chunk;
      for (int kk = 0; kk < a.C / 16; ++kk) {
        const uint64_t ad = make_sdesc(smem_u32(s_a) + kk * 2 * 2048, 2048, 128);
        const uint64_t bd = make_sdesc(wb + kk * 2 * (a.NE * 16), a.NE * 16, 128);
        mma_ss(tmem, ad, bd, idesc, kk > 0);
      }
      mma_commit(&bar[1]);
    }
    __syncthreads();  // s_pool zeroed
    mbar_wait(&bar[1], j & 1);
    tc_fence_after();
    const int m = q * 32 + lane;
    const int img = m / a.HW;
    const bool real = m < npix && (p0 + m) < a.P;
    // columns split between the two warps of a quadrant
    for (int c0 = half * 16; c0 < a.NE; c0 += 32) {
      uint32_t v[16];
      WL_TMEM_LD16(tmem_lane_addr(tmem, q, c0), v);
      tmem_ld_wait();
      for (int im = 0; im < a.imgs; ++im) {
        const unsigned msk = __ballot_sync(0xffffffffu, real && img == im);
        if (!msk) continue;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float val = (real && img == im) ? act<ACT>(__uint_as_float(v[i]) + b1[j * a.NE + c0 + i]) : 0.f;
#pragma unroll
          for (int s = 16; s >= 1; s >>= 1) val += __shfl_xor_sync(0xffffffffu, val, s);
          if (lane == 0) atomicAdd(&s_pool[im * a.NE + c0 + i], val);
        }
      }
    }
    tc_fence_before();
    __syncthreads();
    const float inv = 1.f / (float)a.HW;
    for (int i = tid; i < a.imgs * a.NE; i += blockDim.x) {
      const int im = i / a.NE, c = i % a.NE;
      const int nimg = blockIdx.x * a.imgs + im;
      if ((size_t)nimg * a.HW < (size_t)a.P)
        a.feat[(size_t)nimg * a.E + j * a.NE + c] = __float2half(s_pool[i] * inv);
    }
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc_n(tmem, a.tmem_cols);
}

// kernel 2: logits = feat W2 + b2. CTA = (128 rows of the batch, NC classes).
struct FcArgs {
  int E, classes, NC, nkc, N, nrows;
  int s_a, s_w, s_bar, tmem_cols, w_chunk, o_b2;
  const uint8_t* w2;  // [b2 fp32][class-chunk][k-chunk: NC x 64 core]
  __half* z;          // (n, classes)
};

__global__ void __launch_bounds__(128, 1) head_fc_kernel(const __grid_constant__ CUtensorMap tmap_f,
                                                         const __grid_constant__ FcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_a = smem + a.s_a;  // 2 x [8][128][8] (K chunk 64)
  uint8_t* s_w = smem + a.s_w;  // 2 x NC x 64
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.s_bar);  // full[2], empty[2], mma
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 5);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int row0 = (blockIdx.x / a.N) * 128, cc = blockIdx.x % a.N;
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_n(tbase, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  const uint8_t* wchunks = a.w2 + align_up(a.classes * 4, 128) + (size_t)cc * a.nkc * a.w_chunk;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_f16(128, a.NC);
    for (int k = 0; k < a.nkc + 1; ++k) {
      if (k < a.nkc) {  // load chunk k
        const int b = k & 1;
        if (k >= 2) mbar_wait(&bar[2 + b], ((k - 2) >> 1) & 1);
        mbar_arrive_expect_tx(&bar[b], 128 * 64 * 2 + a.w_chunk);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];" ::"r"(smem_u32(s_a + b * 16384)),
            "l"(&tmap_f), "r"(0), "r"(row0), "r"(k * 8), "r"(smem_u32(&bar[b]))
            : "memory");
        bulk_g2s(s_w + b * a.w_chunk, wchunks + (size_t)k * a.w_chunk, a.w_chunk, &bar[b]);
      }
      if (k >= 1) {  // multiply chunk k-1
        const int kk = k - 1, b = kk & 1;
        mbar_wait(&bar[b], (kk >> 1) & 1);
        tc_fence_after();
        for (int s = 0; s < 4; ++s) {
          const uint64_t ad = make_sdesc(smem_u32(s_a + b * 16384) + s * 2 * 2048, 2048, 128);
          const uint64_t bd = make_sdesc(smem_u32(s_w + b * a.w_chunk) + s * 2 * (a.NC * 16), a.NC * 16, 128);
          mma_ss(tmem, ad, bd, idesc, (kk > 0 || s > 0));
        }
        mma_commit(&bar[2 + b]);
      }
    }
    mma_commit(&bar[4]);
  }
  mbar_wait(&bar[4], 0);
  tc_fence_after();
  const float* b2 = reinterpret_cast<const float*>(a.w2);
  const int row = row0 + warp * 32 + lane;
  for (int c0 = 0; c0 < a.NC; c0 += 16) {
    uint32_t v[16];
    WL_TMEM_LD16(tmem_lane_addr(tmem, warp, c0), v);
    tmem_ld_wait();
    if (row >= a.nrows) continue;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int cls = cc * a.NC + c0 + i;
      if (cls < a.classes) a.z[(size_t)row * a.classes + cls] = __float2half(__uint_as_float(v[i]) + b2[cls]);
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
  a.R = 4;
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
  stem_k(d.act)<<<d.n * a.tiles_y, 256, a.s_bar + 64, st>>>(a);
  return check_cuda(cudaGetLastError(), "stem launch");
}
int stem_init() {
  for (int act : {kRelu, kSilu, kGelu, kIdentity})
    if (int e = check_cuda(cudaFuncSetAttribute(stem_k(act), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMaxSH),
                           "cudaFuncSetAttribute(stem)"))
      return e;
  return WL_OK;
}

// ------------------------------------------------------------------ head
struct HeadPlan {
  HeadArgs h;
  FcArgs f;
  int64_t w1_bytes, w2_bytes;
};
bool head_plan(const wl_block_desc& d, HeadPlan& P) {
  memset(&P, 0, sizeof(P));
  HeadArgs& h = P.h;
  FcArgs& f = P.f;
  h.C = d.c;
  h.E = d.embed;
  h.M = d.classes;
  h.HW = d.h * d.w;
  if (h.C % 16 || h.E % 64 || h.HW > 128 || h.C > 512) return false;
  h.imgs = std::max(1, 128 / h.HW);
  h.P = d.n * h.HW;
  h.NE = h.E % 256 == 0 ? 256 : (h.E % 128 == 0 ? 128 : 64);
  h.nce = h.E / h.NE;
  h.o_b1 = 0;
  h.w1_chunk = h.NE * h.C * 2;
  P.w1_bytes = align_up(h.E * 4, 128) + (int64_t)h.nce * h.w1_chunk;
  int s = 0;
  h.s_a = s;
  s += 128 * h.C * 2;
  h.s_w = s;
  s += 2 * h.w1_chunk;
  h.s_pool = s;
  s = align_up(s + h.imgs * h.NE * 4, 128);
  h.s_bar = s;
  if (s + 64 > kSmemMaxSH) return false;
  h.tmem_cols = std::max(32, h.NE);
  f.E = h.E;
  f.classes = h.M;
  f.NC = 128;
  f.N = (h.M + f.NC - 1) / f.NC;
  f.nkc = h.E / 64;
  f.nrows = d.n;
  f.w_chunk = f.NC * 64 * 2;
  f.o_b2 = 0;
  P.w2_bytes = align_up(h.M * 4, 128) + (int64_t)f.N * f.nkc * f.w_chunk;
  f.s_a = 0;
  f.s_w = 2 * 16384;
  f.s_bar = f.s_w + 2 * f.w_chunk;
  f.tmem_cols = 128;
  return true;
}
using HeadK = void (*)(const CUtensorMap, const HeadArgs);
HeadK head_k(int act) {
  switch (act) {
    case kRelu: return head_pool_kernel<kRelu>;
    case kSilu: return head_pool_kernel<kSilu>;
    case kGelu: return head_pool_kernel<kGelu>;
    case kIdentity: return head_pool_kernel<kIdentity>;
  }
  return nullptr;
}
int head_validate(const wl_block_desc& d) {
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.c < 1) return set_error(WL_EINVAL, "dims must be positive");
  if (d.embed < 1 || d.classes < 1) return set_error(WL_EINVAL, "head widths must be positive");
  if (!head_k(d.act)) return set_error(WL_EUNSUPPORTED, "head activation not supported");
  HeadPlan P;
  if (!head_plan(d, P))
    return set_error(WL_EUNSUPPORTED, "no head plan for C=%d %dx%d E=%d", d.c, d.h, d.w, d.embed);
  return WL_OK;
}
int head_wc(const wl_block_desc&) { return 4; }
int64_t head_wn(const wl_block_desc& d, int i) {
  switch (i) {
    case 0: return (int64_t)d.c * d.embed;
    case 1: return d.embed;
    case 2: return (int64_t)d.embed * d.classes;
    case 3: return d.classes;
  }
  return set_error(WL_EINVAL, "weight index out of range");
}
int64_t head_pb(const wl_block_desc& d) {
  HeadPlan P;
  head_plan(d, P);
  return P.w1_bytes + P.w2_bytes;
}
int head_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  HeadPlan P;
  head_plan(d, P);
  const HeadArgs& h = P.h;
  const FcArgs& f = P.f;
  memset(out, 0, (size_t)(P.w1_bytes + P.w2_bytes));
  float* b1 = reinterpret_cast<float*>(out);
  for (int e = 0; e < h.E; ++e) b1[e] = w[1][e];
  uint8_t* c1 = out + align_up(h.E * 4, 128);
  for (int j = 0; j < h.nce; ++j)
    for (int n = 0; n < h.NE; ++n)
      for (int k = 0; k < h.C; ++k)
        put_h(c1 + (size_t)j * h.w1_chunk, core_off_h(n, k, h.NE * 16), w[0][(size_t)k * h.E + j * h.NE + n]);
  uint8_t* o2 = out + P.w1_bytes;
  float* b2 = reinterpret_cast<float*>(o2);
  for (int m = 0; m < h.M; ++m) b2[m] = w[3][m];
  uint8_t* c2 = o2 + align_up(h.M * 4, 128);
  for (int cc = 0; cc < f.N; ++cc)
    for (int kc = 0; kc < f.nkc; ++kc) {
      uint8_t* blk = c2 + ((size_t)cc * f.nkc + kc) * f.w_chunk;
      for (int n = 0; n < f.NC; ++n) {
        const int cls = cc * f.NC + n;
        if (cls >= h.M) continue;
        for (int k = 0; k < 64; ++k) put_h(blk, core_off_h(n, k, f.NC * 16), w[2][(size_t)(kc * 64 + k) * h.M + cls]);
      }
    }
  return WL_OK;
}
// workspace: [4 KiB reserved counter header shared by all families][pooled embedding]
int64_t head_ws(const wl_block_desc& d) { return 4096 + align_up(d.n * d.embed * 2, 256); }
int head_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st) {
  HeadPlan P;
  head_plan(d, P);
  HeadArgs h = P.h;
  FcArgs f = P.f;
  CUtensorMap tx, tf;
  {
    const uint64_t dims[3] = {8, (uint64_t)h.P, (uint64_t)(h.C / 8)};
    const uint64_t strides[2] = {(uint64_t)h.C * 2, 16};
    const uint32_t box[3] = {8, 128, (uint32_t)(h.C / 8)};
    if (int e = encode_tmap(&tx, x, 3, dims, strides, box)) return e;
  }
  {
    const uint64_t dims[3] = {8, (uint64_t)d.n, (uint64_t)(h.E / 8)};
    const uint64_t strides[2] = {(uint64_t)h.E * 2, 16};
    const uint32_t box[3] = {8, 128, 8};
    if (int e = encode_tmap(&tf, reinterpret_cast<uint8_t*>(ws) + 4096, 3, dims, strides, box)) return e;
  }
  h.w1 = reinterpret_cast<const uint8_t*>(p);
  h.feat = reinterpret_cast<__half*>(reinterpret_cast<uint8_t*>(ws) + 4096);
  const int groups = (d.n + h.imgs - 1) / h.imgs;
  head_k(d.act)<<<groups, 256, h.s_bar + 64, st>>>(tx, h);
  if (int e = check_cuda(cudaGetLastError(), "head_pool launch")) return e;
  f.w2 = reinterpret_cast<const uint8_t*>(p) + P.w1_bytes;
  f.z = reinterpret_cast<__half*>(z);
  const int rows = (d.n + 127) / 128;
  head_fc_kernel<<<rows * f.N, 128, f.s_bar + 64, st>>>(tf, f);
  return check_cuda(cudaGetLastError(), "head_fc launch");
}
int head_init() {
  for (int act : {kRelu, kSilu, kGelu, kIdentity})
    if (int e = check_cuda(cudaFuncSetAttribute(head_k(act), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMaxSH),
                           "cudaFuncSetAttribute(head)"))
      return e;
  return check_cuda(cudaFuncSetAttribute(head_fc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMaxSH),
                    "cudaFuncSetAttribute(head_fc)");
}

}  // namespace

const Family kStemFamily = {stem_validate, stem_wc, stem_wn, stem_pb, stem_pack, stem_ws, stem_fwd, stem_init};
const Family kHeadFamily = {head_validate, head_wc, head_wn, head_pb, head_pack, head_ws, head_fwd, head_init};

}  // namespace wl
